// Exact box-QP block minimizer on ONE CTA (engine.py:189-245 solve_block).
//
//   minimize 1/2 x'Mx - r'x  over lo <= x <= hi     (M SPD, s x s, row-major)
//
// Same finite active-set procedure as the reference: solve unconstrained;
// if outside the box clamp, then repeatedly re-solve on the free set F and
// clamp violators (the active set only grows within a pass), then release the
// single worst wrong-sign multiplier; budget 10*s passes, then projected
// gradient to 1e-10 (engine.py:175-186).
//
// The reduced systems  M_FF x_F = r_F - M_FB x_B  are solved exactly in one of
// two ways:
//   Schur (well-conditioned M, |B| <= |F|): with N = M^{-1} precomputed for the
//     block,  M_FF^{-1} = N_FF - N_FB N_BB^{-1} N_BF,  so only the small
//     |B| x |B| system N_BB is factored;
//   direct (otherwise): Cholesky of M_FF, as the reference does.
// Both are exact minimizers of the same strictly convex subproblem, so the
// iterates agree to rounding.  Factorizations run CTA-wide with one barrier
// per column; triangular solves run on warp 0 with reciprocal pivots.
#pragma once

#include "rac_common.cuh"

namespace rac {

struct BoxWork {
  double *x, *r, *lo, *hi, *grad, *xf, *rr;  // s each
  int* flag;   // 0 free, 1 at lower, 2 at upper
  int* F;      // free list
  int* B;      // bound list
  double* L;   // factor workspace (capacity lcap doubles)
  int lcap;
  const double* N;  // M^{-1} (ld = s) or nullptr
  int ldn;
  int* misc;   // [0] nf, [1] nb, [2] fail, [3] worst, [4..36) per-warp argmax scratch
  double* red; // >= nwarps
  double* rinv;  // s: reciprocal pivots of the current factor
  long long* dbg;  // optional counters: [reduced solves, passes, ns in solves, ns total]
  long long* st;   // optional solve statistics: [sum nb, sum nf, direct solves, ns factor, ns tri-solve]
  double* symv_scratch;  // >= 4 s doubles for the split-row symv, or null
};

// Cholesky of the leading n x n of L (row-major, ld) in place, lower; CTA-wide.
// One barrier per column: step k reads the pivot d = a_kk and the UNSCALED
// column k, applies a_ij -= a_ik a_jk / d to the trailing triangle, and scales
// column k-1 (nobody reads it any more) in the same phase.  Returns 0 or k+1.
// rinv[k] = 1 / L_kk on success.
__device__ int cta_cholesky(double* L, int ld, int n, double* rinv) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int tx = tid & 31, ty = tid >> 5, nty = nt >> 5;
  __syncthreads();
  for (int k = 0; k < n; ++k) {
    const double d = L[k * ld + k];
    if (!(d > 0.0) || !isfinite(d)) {
      __syncthreads();
      return k + 1;   // uniform: every thread read the same pivot
    }
    // one reciprocal square root per pivot (no FP64 divide / sqrt on the chain)
    const double rs = rsqrt(d);
    const double dinv = rs * rs;
    if (k > 0) {
      const double rp = rinv[k - 1];
      for (int i = k + tid; i < n; i += nt) L[i * ld + (k - 1)] *= rp;
      if (tid == 0) {
        const double dp = L[(k - 1) * ld + (k - 1)];
        L[(k - 1) * ld + (k - 1)] = dp * rp;   // d_{k-1} -> L_{k-1,k-1} = sqrt(d_{k-1})
      }
    }
    for (int i = k + 1 + ty; i < n; i += nty) {
      const double lik = L[i * ld + k] * dinv;
      for (int j = k + 1 + tx; j <= i; j += 32) L[i * ld + j] -= lik * L[j * ld + k];
    }
    if (tid == 0) rinv[k] = rs;
    __syncthreads();
  }
  if (n > 0 && tid == 0) L[(n - 1) * ld + (n - 1)] *= rinv[n - 1];
  __syncthreads();
  return 0;
}

// Warp 0: solve L L' v = b in place (b -> v), L lower n x n (ld), rinv = 1/L_kk.
// The right-hand side lives in registers (lane l owns rows l, l+32, ...).
template <int MAXQ = 8>
__device__ void warp_chol_solve(const double* L, int ld, int n, double* v, const double* rinv) {
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  double reg[MAXQ];
#pragma unroll
  for (int q = 0; q < MAXQ; ++q) {
    const int i = lane + 32 * q;
    reg[q] = (i < n) ? v[i] : 0.0;
  }
  // forward: L y = b
  for (int k = 0; k < n; ++k) {
    const int ow = k & 31, oq = k >> 5;
    double yk = 0.0;
#pragma unroll
    for (int q = 0; q < MAXQ; ++q)
      if (q == oq) yk = reg[q] * rinv[k];
    __syncwarp();   // reconverge before the shuffle (a diverged warp takes a ~10x slower path)
    yk = __shfl_sync(0xffffffffu, yk, ow);
#pragma unroll
    for (int q = 0; q < MAXQ; ++q) {
      const int i = lane + 32 * q;
      if (i == k) reg[q] = yk;
      else if (i > k && i < n) reg[q] -= L[i * ld + k] * yk;
    }
  }
  // backward: L' x = y
  for (int k = n - 1; k >= 0; --k) {
    const int ow = k & 31, oq = k >> 5;
    double xk = 0.0;
#pragma unroll
    for (int q = 0; q < MAXQ; ++q)
      if (q == oq) xk = reg[q] * rinv[k];
    __syncwarp();
    xk = __shfl_sync(0xffffffffu, xk, ow);
#pragma unroll
    for (int q = 0; q < MAXQ; ++q) {
      const int i = lane + 32 * q;
      if (i == k) reg[q] = xk;
      else if (i < k) reg[q] -= L[k * ld + i] * xk;
    }
  }
#pragma unroll
  for (int q = 0; q < MAXQ; ++q) {
    const int i = lane + 32 * q;
    if (i < n) v[i] = reg[q];
  }
  __syncwarp();
}

// Warp 0 slow path for n > 256 (L in any memory): scalar substitution.
__device__ void warp_chol_solve_any(const double* L, int ld, int n, double* v) {
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  for (int k = 0; k < n; ++k) {
    double yk = 0.0;
    if (lane == 0) {
      yk = v[k] / L[(int64_t)k * ld + k];
      v[k] = yk;
    }
    yk = __shfl_sync(0xffffffffu, yk, 0);
    for (int i = k + 1 + lane; i < n; i += 32) v[i] -= L[(int64_t)i * ld + k] * yk;
    __syncwarp();
  }
  for (int k = n - 1; k >= 0; --k) {
    double xk = 0.0;
    if (lane == 0) {
      xk = v[k] / L[(int64_t)k * ld + k];
      v[k] = xk;
    }
    xk = __shfl_sync(0xffffffffu, xk, 0);
    for (int i = lane; i < k; i += 32) v[i] -= L[(int64_t)k * ld + i] * xk;
    __syncwarp();
  }
}

__device__ __forceinline__ void chol_solve(const double* L, int ld, int n, double* v, const double* rinv) {
  if (n <= 8 && rinv) {
    // tiny systems (the typical bound set of an SVM block): one thread, no warp traffic
    if (threadIdx.x == 0) {
      for (int k = 0; k < n; ++k) {
        double y = v[k];
        for (int j = 0; j < k; ++j) y -= L[k * ld + j] * v[j];
        v[k] = y * rinv[k];
      }
      for (int k = n - 1; k >= 0; --k) {
        double x = v[k];
        for (int j = k + 1; j < n; ++j) x -= L[j * ld + k] * v[j];
        v[k] = x * rinv[k];
      }
    }
    return;
  }
  if (n <= 256 && rinv) warp_chol_solve<8>(L, ld, n, v, rinv);
  else warp_chol_solve_any(L, ld, n, v);
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

// out = M v for a SYMMETRIC M (row-major, stride ld): thread per row reading
// column i (= row i), so consecutive threads touch consecutive words; four
// independent accumulators.  No cross-lane reduction.  With 4 * rows <= threads,
// four threads share a row (quarter of the columns each) and the quarters are
// combined in fixed order through `scratch` (>= 4 * rows doubles); the caller
// synchronizes before reading `out` either way.
__device__ __forceinline__ void cta_symv(const double* M, int ld, int rows, const double* v, double* out,
                                         double* scratch = nullptr) {
  if (scratch && 4 * rows <= (int)blockDim.x) {
    const int i = threadIdx.x % rows, qq = threadIdx.x / rows;
    if (qq < 4) {
      const int j0 = (rows * qq) / 4, j1 = (rows * (qq + 1)) / 4;
      double a0 = 0.0, a1 = 0.0;
      int j = j0;
      for (; j + 2 <= j1; j += 2) {
        a0 += M[(int64_t)j * ld + i] * v[j];
        a1 += M[(int64_t)(j + 1) * ld + i] * v[j + 1];
      }
      if (j < j1) a0 += M[(int64_t)j * ld + i] * v[j];
      scratch[qq * rows + i] = a0 + a1;
    }
    __syncthreads();
    for (int r = threadIdx.x; r < rows; r += blockDim.x)
      out[r] = (scratch[r] + scratch[rows + r]) + (scratch[2 * rows + r] + scratch[3 * rows + r]);
    return;
  }
  for (int i = threadIdx.x; i < rows; i += blockDim.x) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int j = 0;
    for (; j + 4 <= rows; j += 4) {
      a0 += M[(int64_t)j * ld + i] * v[j];
      a1 += M[(int64_t)(j + 1) * ld + i] * v[j + 1];
      a2 += M[(int64_t)(j + 2) * ld + i] * v[j + 2];
      a3 += M[(int64_t)(j + 3) * ld + i] * v[j + 3];
    }
    for (; j < rows; ++j) a0 += M[(int64_t)j * ld + i] * v[j];
    out[i] = (a0 + a1) + (a2 + a3);
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

// sum_{k < cnt} Mcol[list[k] * ld] * v[vi(k)] with four chains: the gathered column of a
// SYMMETRIC matrix read by one thread (consecutive threads -> consecutive columns).
template <class VI>
__device__ __forceinline__ double gathered_dot(const double* Mcol, int ld, const int* list, int cnt, VI vi) {
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int k = 0;
  for (; k + 4 <= cnt; k += 4) {
    a0 += Mcol[(int64_t)list[k] * ld] * vi(k);
    a1 += Mcol[(int64_t)list[k + 1] * ld] * vi(k + 1);
    a2 += Mcol[(int64_t)list[k + 2] * ld] * vi(k + 2);
    a3 += Mcol[(int64_t)list[k + 3] * ld] * vi(k + 3);
  }
  for (; k < cnt; ++k) a0 += Mcol[(int64_t)list[k] * ld] * vi(k);
  return (a0 + a1) + (a2 + a3);
}

// Solve M_FF xf = r_F - M_FB x_B on the current free set; result in w.xf[0..nf).
// M and N = M^{-1} are symmetric, so every product is one thread per output reading
// the output's column (no cross-lane reductions on the box solver's chain).
// Returns fail code (k+1) if the reduced matrix is not PD.
__device__ int solve_free(const double* M, int ldm, BoxWork& w, bool use_schur) {
  const int nf = w.misc[0], nb = w.misc[1];
  const int tid = threadIdx.x, nt = blockDim.x;
  // q = r_F - M_FB x_B
  for (int a = tid; a < nf; a += nt) {
    const int fa = w.F[a];
    const double acc = gathered_dot(M + fa, ldm, w.B, nb, [&](int k) { return w.x[w.B[k]]; });
    w.xf[a] = (nb > 0) ? w.r[fa] - acc : w.r[fa];
  }
  __syncthreads();
  const bool st = w.st && tid == 0;
  if (st) { w.st[0] += nb; w.st[1] += nf; }
  const int ldk = nb | 1;
  if (use_schur && w.N && nb <= nf && (size_t)ldk * nb <= (size_t)w.lcap) {
    const double* N = w.N;
    const int ldn = w.ldn;
    if (nb > 0) {
      // u = N_BF q ; N_BB (lower) into the workspace
      for (int c = tid; c < nb; c += nt)
        w.rr[c] = gathered_dot(N + w.B[c], ldn, w.F, nf, [&](int k) { return w.xf[k]; });
      for (int e = tid; e < nb * nb; e += nt) {
        const int c1 = e / nb, c2 = e - c1 * nb;
        if (c2 <= c1) w.L[c1 * ldk + c2] = N[(int64_t)w.B[c1] * ldn + w.B[c2]];
      }
      long long t0 = st ? gtimer() : 0;
      const int fail = cta_cholesky(w.L, ldk, nb, w.rinv);
      if (st) { const long long t1 = gtimer(); w.st[3] += t1 - t0; t0 = t1; }
      if (!fail) {
        chol_solve(w.L, ldk, nb, w.rr, w.rinv);   // rr <- N_BB^{-1} N_BF q
        __syncthreads();
        if (st) w.st[4] += gtimer() - t0;
        // x_F = N_FF q - N_FB (N_BB^{-1} N_BF q)
        for (int a2 = tid; a2 < nf; a2 += nt) {
          const double* col = N + w.F[a2];
          w.grad[a2] = gathered_dot(col, ldn, w.F, nf, [&](int k) { return w.xf[k]; }) -
                       gathered_dot(col, ldn, w.B, nb, [&](int k) { return w.rr[k]; });
        }
        __syncthreads();
        for (int a2 = tid; a2 < nf; a2 += nt) w.xf[a2] = w.grad[a2];
        __syncthreads();
        return 0;
      }
      // numerically indefinite N_BB: fall through to the direct factorization
    } else {
      for (int a2 = tid; a2 < nf; a2 += nt)
        w.grad[a2] = gathered_dot(N + w.F[a2], ldn, w.F, nf, [&](int k) { return w.xf[k]; });
      __syncthreads();
      for (int a2 = tid; a2 < nf; a2 += nt) w.xf[a2] = w.grad[a2];
      __syncthreads();
      return 0;
    }
  }
  // direct: Cholesky of M_FF (the reference's route)
  const int ldf = nf | 1;
  if ((size_t)ldf * nf > (size_t)w.lcap) return nf + 1;   // workspace too small (never for SPD M)
  for (int e = tid; e < nf * nf; e += nt) {
    const int a1 = e / nf, b1 = e - a1 * nf;
    if (b1 <= a1) w.L[a1 * ldf + b1] = M[(int64_t)w.F[a1] * ldm + w.F[b1]];
  }
  long long t0 = st ? gtimer() : 0;
  if (st) w.st[2] += 1;
  const int fail = cta_cholesky(w.L, ldf, nf, w.rinv);
  if (st) { const long long t1 = gtimer(); w.st[3] += t1 - t0; t0 = t1; }
  if (fail) return fail;
  chol_solve(w.L, ldf, nf, w.xf, w.rinv);
  __syncthreads();
  if (st) w.st[4] += gtimer() - t0;
  return 0;
}

// Projected-gradient fallback (engine.py:175-186).  The step uses the largest
// eigenvalue of M estimated by power iteration (the reference uses eigvalsh).
__device__ void projected_gradient(const double* M, int ldm, int s, BoxWork& w) {
  const int tid = threadIdx.x, nt = blockDim.x;
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
// `max_passes` < 0: the reference's budget ACTIVE_SET_PASS_FACTOR * s (engine.py:38,215);
// rac_box_block_min lowers it only to exercise the projected-gradient fallback in tests.
__device__ int box_active_set(const double* M, int ldm, int s, BoxWork& w, bool use_schur, int max_passes = -1) {
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
  const int budget = max_passes < 0 ? 10 * s : max_passes;
  for (int pass = 0; pass < budget; ++pass) {
    for (int it = 0; it <= s; ++it) {
      for (int i = tid; i < s; i += nt) {
        if (w.flag[i] == 1) w.x[i] = w.lo[i];
        else if (w.flag[i] == 2) w.x[i] = w.hi[i];
      }
      __syncthreads();
      cta_lists(w, s);
      const int nf = w.misc[0];
      if (nf == 0) break;
      long long t_s = (w.dbg && threadIdx.x == 0) ? gtimer() : 0;
      int fail = solve_free(M, ldm, w, use_schur);
      if (w.dbg && threadIdx.x == 0) { w.dbg[0] += 1; w.dbg[2] += gtimer() - t_s; }
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
    if (w.dbg && threadIdx.x == 0) w.dbg[1] += 1;
    // multipliers: grad = M x - r  (M symmetric: four threads per row)
    cta_symv(M, ldm, s, w.x, w.grad, w.symv_scratch);
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
    const int lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
    __syncwarp();
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
