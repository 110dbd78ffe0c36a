// Exact box-QP block minimizer on ONE CTA (engine.py:189-245 solve_block).
//
//   minimize 1/2 x'Mx - r'x  over lo <= x <= hi     (M SPD, s x s, row-major)
//
// Same finite active-set procedure as the reference: solve unconstrained;
// if outside the box clamp, then repeatedly re-solve on the free set and
// clamp violators (the active set only grows within a pass), then release the
// single worst wrong-sign multiplier; budget 10*s passes, then projected
// gradient to 1e-10 (engine.py:175-186).  Reduced systems M_FF are factored
// in shared memory (or a global scratch for large s) by the whole CTA; the
// triangular solves run warp-synchronously on warp 0.
#pragma once

#include "rac_common.cuh"

namespace rac {

struct BoxWork {
  double *x, *r, *lo, *hi, *grad, *xf, *rr;  // s each
  int* flag;   // 0 free, 1 at lower, 2 at upper
  int* F;      // free list
  int* B;      // bound list
  double* L;   // s x s (ld = s) factor workspace
  int* misc;   // [0] nf, [1] nb, [2] fail, [3] worst, [4..36) per-warp argmax scratch
  double* red; // >= nwarps
};

__device__ __forceinline__ bool isbounded_lo(double v) { return v > -INFINITY; }

// Cholesky of the leading n x n of L (row-major, ld) in place, lower; CTA-wide.
// Returns 0 or k+1 on a non-positive pivot.  misc[2] is used as the flag.
__device__ int cta_cholesky(double* L, int ld, int n, int* flag) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int tx = tid & 31, ty = tid >> 5, nty = nt >> 5;
  if (tid == 0) *flag = 0;
  __syncthreads();
  for (int k = 0; k < n; ++k) {
    if (tid == 0) {
      double d = L[k * ld + k];
      if (!(d > 0.0) || !isfinite(d)) *flag = k + 1;
      else L[k * ld + k] = sqrt(d);
    }
    __syncthreads();
    if (*flag) return *flag;
    const double piv = L[k * ld + k];
    for (int i = k + 1 + tid; i < n; i += nt) L[i * ld + k] /= piv;
    __syncthreads();
    for (int i = k + 1 + ty; i < n; i += nty) {
      const double lik = L[i * ld + k];
      for (int j = k + 1 + tx; j <= i; j += 32) L[i * ld + j] -= lik * L[j * ld + k];
    }
    __syncthreads();
  }
  return 0;
}

// Warp 0: solve L L' v = b in place (b -> v), L lower n x n.  Others idle.
__device__ void warp_chol_solve(const double* L, int ld, int n, double* v) {
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  // forward: L y = b
  for (int k = 0; k < n; ++k) {
    double yk = 0.0;
    if (lane == 0) {
      yk = v[k] / L[k * ld + k];
      v[k] = yk;
    }
    yk = __shfl_sync(0xffffffffu, yk, 0);
    for (int i = k + 1 + lane; i < n; i += 32) v[i] -= L[i * ld + k] * yk;
    __syncwarp();
  }
  // backward: L' x = y
  for (int k = n - 1; k >= 0; --k) {
    double xk = 0.0;
    if (lane == 0) {
      xk = v[k] / L[k * ld + k];
      v[k] = xk;
    }
    xk = __shfl_sync(0xffffffffu, xk, 0);
    for (int i = lane; i < k; i += 32) v[i] -= L[k * ld + i] * xk;
    __syncwarp();
  }
}

// out = M v (rows x s of row-major M, ld), warp per row.
__device__ __forceinline__ void cta_matvec(const double* M, int ld, int rows, int cols,
                                           const double* v, double* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int i = warp; i < rows; i += nw) {
    const double* row = M + (int64_t)i * ld;
    double acc = 0.0;
    for (int j = lane; j < cols; j += 32) acc += row[j] * v[j];
    acc = warp_sum(acc);
    if (lane == 0) out[i] = acc;
  }
}

// block max of a per-thread value (all threads get it)
__device__ __forceinline__ double cta_max(double v, double* red) {
  v = warp_max(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double m = red[0];
  for (int w = 1; w < nw; ++w) m = fmax(m, red[w]);
  __syncthreads();
  return m;
}

// Build the free/bound lists from flags (warp 0, ballot compaction; ordered).
__device__ void cta_lists(BoxWork& w, int s) {
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    int nf = 0, nb = 0;
    for (int base = 0; base < s; base += 32) {
      int i = base + lane;
      bool valid = i < s;
      bool fr = valid && w.flag[i] == 0;
      bool bd = valid && w.flag[i] != 0;
      unsigned mf = __ballot_sync(0xffffffffu, fr), mb = __ballot_sync(0xffffffffu, bd);
      unsigned below = (1u << lane) - 1u;
      if (fr) w.F[nf + __popc(mf & below)] = i;
      if (bd) w.B[nb + __popc(mb & below)] = i;
      nf += __popc(mf);
      nb += __popc(mb);
    }
    if (lane == 0) {
      w.misc[0] = nf;
      w.misc[1] = nb;
    }
  }
  __syncthreads();
}

// Solve M_FF xf = r_F - M_FB x_B on the current free set; result in w.xf[0..nf).
// Returns fail code (k+1) if M_FF is not PD.
__device__ int solve_free(const double* M, int ldm, BoxWork& w) {
  const int nf = w.misc[0], nb = w.misc[1];
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  for (int e = tid; e < nf * nf; e += nt) {
    int a = e / nf, b = e - a * nf;
    if (b <= a) w.L[a * nf + b] = M[(int64_t)w.F[a] * ldm + w.F[b]];
  }
  for (int a = warp; a < nf; a += nw) {
    const double* row = M + (int64_t)w.F[a] * ldm;
    double acc = 0.0;
    for (int k = lane; k < nb; k += 32) acc += row[w.B[k]] * w.x[w.B[k]];
    acc = warp_sum(acc);
    if (lane == 0) w.xf[a] = (nb > 0) ? w.r[w.F[a]] - acc : w.r[w.F[a]];
  }
  __syncthreads();
  int fail = cta_cholesky(w.L, nf, nf, &w.misc[2]);
  if (fail) return fail;
  warp_chol_solve(w.L, nf, nf, w.xf);
  __syncthreads();
  return 0;
}

// Projected-gradient fallback (engine.py:175-186).  The step uses the largest
// eigenvalue of M estimated by power iteration (the reference uses eigvalsh).
__device__ void projected_gradient(const double* M, int ldm, int s, BoxWork& w) {
  const int tid = threadIdx.x, nt = blockDim.x;
  // power iteration: xf <- M xf / |M xf|
  for (int i = tid; i < s; i += nt) w.xf[i] = 1.0;
  __syncthreads();
  double lam = 1.0;
  for (int it = 0; it < 200; ++it) {
    cta_matvec(M, ldm, s, s, w.xf, w.rr);
    __syncthreads();
    double loc = 0.0;
    for (int i = tid; i < s; i += nt) loc = fmax(loc, fabs(w.rr[i]));
    double nrm = cta_max(loc, w.red);
    lam = nrm;
    for (int i = tid; i < s; i += nt) w.xf[i] = w.rr[i] / (nrm > 0 ? nrm : 1.0);
    __syncthreads();
  }
  const double step = 1.0 / fmax(lam, 1e-12);
  for (int i = tid; i < s; i += nt) w.x[i] = fmin(fmax(w.x[i], w.lo[i]), w.hi[i]);
  __syncthreads();
  for (int it = 0; it < 200000; ++it) {
    cta_matvec(M, ldm, s, s, w.x, w.grad);
    __syncthreads();
    double loc = 0.0;
    for (int i = tid; i < s; i += nt) {
      double nx = fmin(fmax(w.x[i] - step * (w.grad[i] - w.r[i]), w.lo[i]), w.hi[i]);
      loc = fmax(loc, fabs(nx - w.x[i]));
      w.xf[i] = nx;
    }
    double d = cta_max(loc, w.red);
    for (int i = tid; i < s; i += nt) w.x[i] = w.xf[i];
    __syncthreads();
    if (d <= 1e-10 * step) break;
  }
}

// Entry: w.x holds the unconstrained solution M^{-1} r on input.  Returns 0 or
// the fail code of a non-PD reduced system.
__device__ int box_active_set(const double* M, int ldm, int s, BoxWork& w) {
  const int tid = threadIdx.x, nt = blockDim.x;
  int bnd = 0, out = 0;
  for (int i = tid; i < s; i += nt) {
    bnd |= (w.lo[i] > -INFINITY) || (w.hi[i] < INFINITY);
    out |= !(w.x[i] >= w.lo[i] && w.x[i] <= w.hi[i]);
  }
  bnd = __syncthreads_or(bnd);
  if (!bnd) return 0;
  out = __syncthreads_or(out);
  if (!out) return 0;
  for (int i = tid; i < s; i += nt) {
    double v = fmin(fmax(w.x[i], w.lo[i]), w.hi[i]);
    w.x[i] = v;
    w.flag[i] = (v <= w.lo[i]) ? 1 : ((v >= w.hi[i]) ? 2 : 0);
  }
  __syncthreads();
  for (int pass = 0; pass < 10 * s; ++pass) {
    for (int it = 0; it <= s; ++it) {
      for (int i = tid; i < s; i += nt) {
        if (w.flag[i] == 1) w.x[i] = w.lo[i];
        else if (w.flag[i] == 2) w.x[i] = w.hi[i];
      }
      __syncthreads();
      cta_lists(w, s);
      const int nf = w.misc[0];
      if (nf == 0) break;
      int fail = solve_free(M, ldm, w);
      if (fail) return fail;
      int viol = 0;
      for (int a = tid; a < nf; a += nt) {
        const int i = w.F[a];
        const double v = w.xf[a];
        if (v < w.lo[i]) { w.flag[i] = 1; viol = 1; }
        else if (v > w.hi[i]) { w.flag[i] = 2; viol = 1; }
        w.x[i] = fmin(fmax(v, w.lo[i]), w.hi[i]);
      }
      viol = __syncthreads_or(viol);
      if (!viol) break;
    }
    // multipliers: grad = M x - r
    cta_matvec(M, ldm, s, s, w.x, w.grad);
    __syncthreads();
    double loc = 0.0;
    for (int i = tid; i < s; i += nt) {
      w.grad[i] -= w.r[i];
      loc = fmax(loc, fabs(w.grad[i]));
    }
    const double scale = fmax(1.0, cta_max(loc, w.red));
    // worst offender: max score, lowest index on ties (np.argmax)
    double best = 0.0;
    int bi = -1;
    for (int i = tid; i < s; i += nt) {
      double sc = 0.0;
      if (w.flag[i] == 1 && w.grad[i] < -1e-14 * scale) sc = -w.grad[i];
      else if (w.flag[i] == 2 && w.grad[i] > 1e-14 * scale) sc = w.grad[i];
      if (sc > best) { best = sc; bi = i; }
    }
    // reduce (best, bi): max best, then min index
    const int lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
    for (int o = 16; o > 0; o >>= 1) {
      double ob = __shfl_xor_sync(0xffffffffu, best, o);
      int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi >= 0 && (bi < 0 || oi < bi))) { best = ob; bi = oi; }
    }
    __syncthreads();
    if (lane == 0) { w.red[warp] = best; w.misc[4 + warp] = bi; }
    __syncthreads();
    if (tid == 0) {
      double b0 = w.red[0];
      int i0 = w.misc[4];
      for (int q = 1; q < nw; ++q) {
        double bq = w.red[q];
        int iq = w.misc[4 + q];
        if (bq > b0 || (bq == b0 && iq >= 0 && (i0 < 0 || iq < i0))) { b0 = bq; i0 = iq; }
      }
      w.misc[3] = (b0 > 0.0) ? i0 : -1;
    }
    __syncthreads();
    const int worst = w.misc[3];
    if (worst < 0) return 0;
    if (tid == 0) w.flag[worst] = 0;
    __syncthreads();
  }
  projected_gradient(M, ldm, s, w);
  return 0;
}

}  // namespace rac
