// K3 — block systems of one partition: assembly, positive-definiteness check,
// and the factor the chain needs.  One CTA per block.
//
//   sys_b = (sum of split-K Gram partials) / div * mul  (+ H_bb)  + shift I
//           (+ ridge_rel * max diag I)
//     EN:  X_b'X_b / m + gamma I                      (elastic_net.py:210-212)
//     QP:  H_bb + beta A_b'A_b                         (engine.py:103-119)
//     SVM: Q_bb + beta y_b y_b' + 1e-9 max(diag) I     (svm.py:241-246)
//
// Modes
//   FACTOR_INVERSE (EN chain): explicit sys^{-1}, so the distributed chain
//     solves a block with one parallel mat-vec.  Fast path: blocked symmetric
//     sweep operator (Gauss-Jordan, 8 pivots per step) on the packed lower
//     triangle in shared memory.  If it meets a non-positive pivot the block
//     is re-done with Cholesky (backward stable) + triangular inverse, which
//     is the authoritative positive-definiteness test.
//   FACTOR_CHOL (QP/SVM chain): the lower Cholesky factor L (what the
//     reference's solve_block factors, engine.py:160-172); the single-CTA
//     box solver does the two triangular solves.
// A failing block reports k+1 for the first non-positive leading minor, as
// np.linalg.cholesky does (elastic_net.py:213-219).
#include "rac_internal.h"

#include <algorithm>

namespace rac {

constexpr int CTHREADS = 512;
constexpr int SB = 8;   // pivots per blocked sweep step

__device__ __forceinline__ int pk(int i, int j) { return i * (i + 1) / 2 + j; }  // j <= i

// gathered H_bb entry (0 for padding)
__device__ __forceinline__ double h_entry(const SysArgs& a, int b, const int32_t* bidx, int i, int j) {
  if (!(a.H || a.hblk) || !bidx || bidx[i] < 0 || bidx[j] < 0) return 0.0;
  if (a.hblk) return a.hblk[((int64_t)b * a.s + i) * a.s + j];
  return a.H[(int64_t)bidx[i] * a.ldh + bidx[j]];
}

// value of the assembled system at (i, j), j <= i (before the ridge)
__device__ __forceinline__ double sys_entry(const SysArgs& a, int b, const int32_t* bidx, int i, int j,
                                            double* h_out) {
  const bool pad = bidx && (bidx[i] < 0 || bidx[j] < 0);
  double h = 0.0;
  if (!pad) h = h_entry(a, b, bidx, i, j);
  if (h_out) *h_out = h;
  if (pad) return (i == j) ? 1.0 : 0.0;   // short last block: identity rows keep the leading part exact
  double v = 0.0;
  if (a.ws) {
    const int s = a.s;
    const double* src = a.ws + (int64_t)b * a.splits * s * s + (int64_t)i * s + j;
    double acc = src[0];
    for (int z = 1; z < a.splits; ++z) acc += src[(int64_t)z * s * s];
    if (a.div != 1.0) acc = acc / a.div;
    if (a.mul != 1.0) acc = a.mul * acc;
    v = acc;
  }
  if (a.H || a.hblk) v = a.ws ? h + v : h;
  if (i == j) v += a.shift;
  return v;
}

// ridge_rel * max over valid diagonal entries (all threads get it)
template <class DiagFn>
__device__ double cta_ridge(const SysArgs& a, const int32_t* bidx, int s, DiagFn diag, double* red) {
  const int tid = threadIdx.x;
  double mx = -INFINITY;
  for (int i = tid; i < s; i += CTHREADS)
    if (!bidx || bidx[i] >= 0) mx = fmax(mx, diag(i));
  mx = warp_max(mx);
  if ((tid & 31) == 0) red[tid >> 5] = mx;
  __syncthreads();
  double m2 = red[0];
  for (int w = 1; w < CTHREADS / 32; ++w) m2 = fmax(m2, red[w]);
  __syncthreads();
  return a.ridge_rel * m2;
}

// assemble the full square (row-major, stride ld) incl. ridge; optional copies out
__device__ void assemble_square(const SysArgs& a, int b, double* A, int ld, double* red) {
  const int s = a.s, tid = threadIdx.x;
  const int32_t* bidx = a.idx ? a.idx + (int64_t)b * s : nullptr;
  double* hbo = a.hbb_out ? a.hbb_out + (int64_t)b * s * s : nullptr;
  for (int e = tid; e < s * s; e += CTHREADS) {
    const int i = e / s, j = e - i * s;
    const double v = (j <= i) ? sys_entry(a, b, bidx, i, j, nullptr) : 0.0;
    if (hbo) hbo[e] = h_entry(a, b, bidx, i, j);
    A[(int64_t)i * ld + j] = v;
  }
  __syncthreads();
  if (a.ridge_rel > 0.0) {
    const double ridge = cta_ridge(a, bidx, s, [&](int i) { return A[(int64_t)i * ld + i]; }, red);
    for (int i = tid; i < s; i += CTHREADS)
      if (!bidx || bidx[i] >= 0) A[(int64_t)i * ld + i] += ridge;
    __syncthreads();
  }
  if (a.mat_out) {
    double* mo = a.mat_out + (int64_t)b * s * s;
    for (int e = tid; e < s * s; e += CTHREADS) {
      const int i = e / s, j = e - i * s;
      mo[e] = (j <= i) ? A[(int64_t)i * ld + j] : A[(int64_t)j * ld + i];
    }
  }
}

// right-looking Cholesky in place (lower, diag included); returns 0 or k+1
__device__ int cta_cholesky_sq(double* A, int ld, int s, int* flag) {
  const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
  if (tid == 0) *flag = 0;
  __syncthreads();
  for (int k = 0; k < s; ++k) {
    if (tid == 0) {
      const double d = A[(int64_t)k * ld + k];
      if (!(d > 0.0) || !isfinite(d)) *flag = k + 1;
      else A[(int64_t)k * ld + k] = sqrt(d);
    }
    __syncthreads();
    if (*flag) return *flag;
    const double piv = A[(int64_t)k * ld + k];
    for (int i = k + 1 + tid; i < s; i += CTHREADS) A[(int64_t)i * ld + k] /= piv;
    __syncthreads();
    for (int i = k + 1 + ty; i < s; i += CTHREADS / 32) {
      const double lik = A[(int64_t)i * ld + k];
      for (int j = k + 1 + tx; j <= i; j += 32) A[(int64_t)i * ld + j] -= lik * A[(int64_t)j * ld + k];
    }
    __syncthreads();
  }
  return 0;
}

// inverse from the Cholesky factor in the lower triangle of A: Y = L^{-1} in
// the strict upper triangle (transposed) + dY, then out = Y'Y (full, row-major)
__device__ void cta_chol_inverse(double* A, int ld, int s, double* dY, double* out) {
  const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
  for (int e = tid; e < s * s; e += CTHREADS) {
    const int c = e / s, i = e - c * s;
    if (c < i) A[(int64_t)c * ld + i] = 0.0;
  }
  __syncthreads();
  for (int k = 0; k < s; ++k) {
    const double lkk = A[(int64_t)k * ld + k];
    for (int c = tid; c < k; c += CTHREADS) A[(int64_t)c * ld + k] /= lkk;
    if (tid == 0) dY[k] = 1.0 / lkk;
    __syncthreads();
    for (int i = k + 1 + ty; i < s; i += CTHREADS / 32) {
      const double lik = A[(int64_t)i * ld + k];
      for (int c = tx; c <= k; c += 32) {
        const double ykc = (c == k) ? dY[k] : A[(int64_t)c * ld + k];
        A[(int64_t)c * ld + i] -= lik * ykc;
      }
    }
    __syncthreads();
  }
  // out[i][j] = sum_{r >= max(i,j)} Y[r][i] Y[r][j]; rows i by warps, cols j by lanes
  for (int i = ty; i < s; i += CTHREADS / 32) {
    for (int j = tx; j <= i; j += 32) {
      double acc = dY[i] * ((i == j) ? dY[j] : A[(int64_t)j * ld + i]);
      for (int r = i + 1; r < s; ++r) acc += A[(int64_t)i * ld + r] * A[(int64_t)j * ld + r];
      out[(int64_t)i * s + j] = acc;
      out[(int64_t)j * s + i] = acc;
    }
  }
}

// blocked symmetric sweep on the packed lower triangle P (-> -P^{-1}); 0 or k+1
__device__ int cta_sweep_packed(double* P, int s, double* Cm, double* CW, double* W, int* fail,
                                long long* tr) {
  const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
  if (tid == 0) *fail = 0;
  __syncthreads();
  int tp = 0;
  auto stamp = [&]() {
    if (tr && tid == 0) tr[tp] = gtimer();
    ++tp;
  };
  for (int k = 0; k < s; k += SB) {
    const int bb = min(SB, s - k);
    for (int e = tid; e < bb * s; e += CTHREADS) {
      const int q = e / s, i = e - q * s, c = k + q;
      Cm[q * s + i] = (i >= c) ? P[pk(i, c)] : P[pk(c, i)];
    }
    __syncthreads();
    stamp();
    if (ty == 0) {
      // 8x8 diagonal block swept in registers: lane l holds (r0 = l/8, c = l%8)
      // and (r0 + 4, c); pivot rows/columns move by warp shuffles.
      const int r0 = tx >> 3, c = tx & 7, r1 = r0 + 4;
      double v0 = (r0 < bb && c < bb) ? Cm[c * s + k + r0] : 0.0;
      double v1 = (r1 < bb && c < bb) ? Cm[c * s + k + r1] : 0.0;
      int f = 0;
      // branch-free (selects only) and fully unrolled: every lane runs the same
      // instruction stream; a non-positive pivot is recorded, the rest ignored
#pragma unroll
      for (int q = 0; q < SB; ++q) {
        if (q < bb) {
          const double d = __shfl_sync(0xffffffffu, (q < 4) ? v0 : v1, (q & 3) * 8 + q);  // W[q][q]
          const double wq0 = __shfl_sync(0xffffffffu, v0, r0 * 8 + q);     // W[r0][q]
          const double wq1 = __shfl_sync(0xffffffffu, v1, r0 * 8 + q);     // W[r1][q]
          const double wqc = __shfl_sync(0xffffffffu, (q < 4) ? v0 : v1, (q & 3) * 8 + c);  // W[q][c]
          const bool ok = (d > 0.0) && isfinite(d);
          if (!ok && !f) f = k + q + 1;
          const double dinv = __drcp_rn(ok ? d : 1.0);
          const double n0 = (r0 == q) ? ((c == q) ? -dinv : wqc * dinv)
                                      : ((c == q) ? wq0 * dinv : v0 - wq0 * wqc * dinv);
          const double n1 = (r1 == q) ? ((c == q) ? -dinv : wqc * dinv)
                                      : ((c == q) ? wq1 * dinv : v1 - wq1 * wqc * dinv);
          if (r0 < bb && c < bb) v0 = n0;
          if (r1 < bb && c < bb) v1 = n1;
        }
      }
      if (tx == 0 && f) *fail = f;
      W[tx] = -v0;
      W[tx + 32] = -v1;
    }
    __syncthreads();
    stamp();
    if (*fail) return *fail;
    for (int e = tid; e < bb * s; e += CTHREADS) {
      const int q = e / s, i = e - q * s;
      double acc = 0.0;
      for (int r = 0; r < bb; ++r) acc += Cm[r * s + i] * W[r * SB + q];
      CW[q * s + i] = acc;
    }
    __syncthreads();
    stamp();
    if ((s & 7) == 0 && bb == SB) {
      // rank-8 update  A_RR -= CW Cm'  on FP64 tensor cores: one m8n8k4 pair per
      // 8x8 lower tile (D = C - A B, A = CW rows, B = Cm rows); the K strip is
      // rewritten below.  lane (g, t): A[g][t], B[t][g], D[g][2t..2t+1].
      const int nt = s >> 3, ntiles = nt * (nt + 1) / 2;
      const int g = tx >> 2, t4 = tx & 3;
      int I = 0, J = ty;   // tile ty in row-major lower-triangle order, advanced by 16
      while (J > I) { J -= I + 1; ++I; }
      for (int tile = ty; tile < ntiles; tile += CTHREADS / 32) {
        const int r = 8 * I + g, c0 = 8 * J + 2 * t4;
        const int off = pk(r, 0);
        double d0 = (c0 <= r) ? P[off + c0] : 0.0;
        double d1 = (c0 + 1 <= r) ? P[off + c0 + 1] : 0.0;
        dmma884(d0, d1, -CW[t4 * s + 8 * I + g], Cm[t4 * s + 8 * J + g]);
        dmma884(d0, d1, -CW[(t4 + 4) * s + 8 * I + g], Cm[(t4 + 4) * s + 8 * J + g]);
        if (c0 <= r) P[off + c0] = d0;
        if (c0 + 1 <= r) P[off + c0 + 1] = d1;
        J += CTHREADS / 32;
        while (J > I) { J -= I + 1; ++I; }
      }
      __syncthreads();
      // K strip: rows >= k of columns K, and the K rows left of the strip
      for (int e = tid; e < (s - k) * SB; e += CTHREADS) {
        const int i = k + e / SB, q = e % SB, j = k + q;
        if (j > i) continue;
        P[pk(i, j)] = (i < k + SB) ? -W[(i - k) * SB + q] : CW[q * s + i];
      }
      for (int e = tid; e < k * SB; e += CTHREADS) {
        const int q = e / k, j = e - q * k, i = k + q;
        P[pk(i, j)] = CW[q * s + j];
      }
    } else {
      for (int pr = ty; pr < (s + 1) / 2; pr += CTHREADS / 32) {
        for (int half = 0; half < 2; ++half) {
          const int i = half ? s - 1 - pr : pr;
          if (half && i == pr) break;
          const int off = pk(i, 0);
          const bool iK = (i >= k && i < k + bb);
          double cw[SB];
#pragma unroll
          for (int q = 0; q < SB; ++q) cw[q] = (q < bb) ? CW[q * s + i] : 0.0;
          for (int j = tx; j <= i; j += 32) {
            const bool jK = (j >= k && j < k + bb);
            double v;
            if (iK && jK) {
              v = -W[(i - k) * SB + (j - k)];
            } else if (jK) {
              v = CW[(j - k) * s + i];
            } else if (iK) {
              v = CW[(i - k) * s + j];
            } else {
              v = P[off + j];
#pragma unroll
              for (int q = 0; q < SB; ++q)
                if (q < bb) v -= cw[q] * Cm[q * s + j];
            }
            P[off + j] = v;
          }
        }
      }
    }
    __syncthreads();
    stamp();
  }
  return 0;
}

struct FactorSmemPlan {
  bool packed;   // blocked sweep on the packed triangle fits
  bool square;   // full square (Cholesky path) fits
};

constexpr size_t kMaxDyn = 227 * 1024 - 2048;
__host__ __device__ inline size_t packed_bytes(int s) {
  const size_t s8 = (s + 7) & ~7;
  return (s8 * (s8 + 1) / 2 + 2 * SB * s8) * sizeof(double);
}
__host__ __device__ inline size_t square_bytes(int s) { return ((size_t)s * (s + 1) + s) * sizeof(double); }

__global__ void __launch_bounds__(CTHREADS) factor_kernel(SysArgs a, int mode, int use_packed, int use_square) {
  extern __shared__ __align__(16) double fsm[];
  if (a.done && *a.done) return;
  const int s = a.s;
  const int b = a.blk_list ? a.blk_list[blockIdx.x] : blockIdx.x;
  if (a.only_failed && a.info[b] == 0) return;   // re-do pass for blocks the blocked path rejected
  __shared__ int fail;
  __shared__ double red[CTHREADS / 32];
  __shared__ double W[SB * SB];
  const int tid = threadIdx.x;
  const int32_t* bidx = a.idx ? a.idx + (int64_t)b * s : nullptr;
  double* out = a.inv + (int64_t)b * s * s;

  if (a.trace && blockIdx.x == 0 && tid == 0) a.trace[0] = gtimer();
  if (mode == FACTOR_INVERSE && use_packed) {
    // padded to a multiple of 8 (identity rows) so the update runs on DMMA tiles
    const int s8 = (s + 7) & ~7;
    double* P = fsm;
    double* Cm = fsm + (size_t)s8 * (s8 + 1) / 2;
    double* CW = Cm + SB * s8;
    double* hbo = a.hbb_out ? a.hbb_out + (int64_t)b * s * s : nullptr;
    const int tx = tid & 31, ty = tid >> 5;
    // block indices staged in smem (Cm is free until the sweep), then every row's
    // entries fetched as one batch of independent loads per lane (s8 <= 256)
    int* sbi = reinterpret_cast<int*>(Cm);
    for (int i = tid; i < s; i += CTHREADS) sbi[i] = bidx ? bidx[i] : i;
    __syncthreads();
    const double* wsb = a.ws ? a.ws + (int64_t)b * a.splits * s * s : nullptr;
    // packed lower triangle, 8 independent gathers per thread in flight (one L2
    // round trip per 8 * CTHREADS entries instead of one per row and warp)
    const int ntri = s8 * (s8 + 1) / 2;
    for (int e0 = 0; e0 < ntri; e0 += 8 * CTHREADS) {
      double v[8];
      int pos[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + u * CTHREADS + tid;
        pos[u] = e;
        double val = 0.0;
        if (e < ntri) {
          int i = (int)((sqrtf(8.0f * (float)e + 1.0f) - 1.0f) * 0.5f);
          while (pk(i + 1, 0) <= e) ++i;
          while (pk(i, 0) > e) --i;
          const int j = e - pk(i, 0);
          val = (i == j) ? 1.0 : 0.0;
          if (i < s && j < s) {
            const int gi = sbi[i], gj = sbi[j];
            if (!(bidx && (gi < 0 || gj < 0))) {
              double acc = 0.0;
              if (wsb) {
                const double* src = wsb + (int64_t)i * s + j;
                acc = src[0];
                for (int z = 1; z < a.splits; ++z) acc += src[(int64_t)z * s * s];
                if (a.div != 1.0) acc = acc / a.div;
                if (a.mul != 1.0) acc = a.mul * acc;
              }
              if (a.H || a.hblk) {
                const double h = a.hblk ? a.hblk[((int64_t)b * s + i) * s + j] : a.H[(int64_t)gi * a.ldh + gj];
                acc = wsb ? h + acc : h;
              }
              if (i == j) acc += a.shift;
              val = acc;
            }
          }
        }
        v[u] = val;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (pos[u] < ntri) P[pos[u]] = v[u];
    }
    if (hbo)
      for (int e = tid; e < s * s; e += CTHREADS) {
        const int i = e / s, j = e - i * s;
        hbo[e] = h_entry(a, b, bidx, i, j);
      }
    __syncthreads();
    if (a.ridge_rel > 0.0) {
      const double ridge = cta_ridge(a, bidx, s, [&](int i) { return P[pk(i, i)]; }, red);
      for (int i = tid; i < s; i += CTHREADS)
        if (!bidx || bidx[i] >= 0) P[pk(i, i)] += ridge;
      __syncthreads();
    }
    if (a.mat_out) {
      double* mo = a.mat_out + (int64_t)b * s * s;
      for (int e = tid; e < s * s; e += CTHREADS) {
        const int i = e / s, j = e - i * s;
        mo[e] = (j <= i) ? P[pk(i, j)] : P[pk(j, i)];
      }
    }
    long long* tr = (a.trace && blockIdx.x == 0) ? a.trace + 2 : nullptr;
    if (tr && tid == 0) a.trace[1] = gtimer();
    const int f = cta_sweep_packed(P, s8, Cm, CW, W, &fail, tr);
    __syncthreads();
    if (!f) {
      if (tid == 0) a.info[b] = 0;
      for (int e = tid; e < s * s; e += CTHREADS) {
        const int i = e / s, j = e - i * s;
        out[e] = -((j <= i) ? P[pk(i, j)] : P[pk(j, i)]);
      }
      return;
    }
    // fall through: authoritative Cholesky path
  }
  const int ld = s + 1;
  double* A = use_square ? fsm : a.scratch + (int64_t)b * ((int64_t)s * ld + s);
  double* dY = A + (size_t)s * ld;
  assemble_square(a, b, A, ld, red);
  const int f = cta_cholesky_sq(A, ld, s, &fail);
  if (tid == 0) a.info[b] = f;
  if (f) return;
  if (mode == FACTOR_CHOL) {
    for (int e = tid; e < s * s; e += CTHREADS) {
      const int i = e / s, j = e - i * s;
      out[e] = (j <= i) ? A[(int64_t)i * ld + j] : 0.0;
    }
    if (a.cond_out) {
      // pivot-ratio estimate of cond(sys): (max L_ii / min L_ii)^2
      double mx = 0.0, mn = INFINITY;
      for (int i = tid; i < s; i += CTHREADS) {
        const double d = A[(int64_t)i * ld + i];
        mx = fmax(mx, d);
        mn = fmin(mn, d);
      }
      mx = warp_max(mx);
      mn = -warp_max(-mn);
      __shared__ double redmin[CTHREADS / 32];
      if ((tid & 31) == 0) { red[tid >> 5] = mx; redmin[tid >> 5] = mn; }
      __syncthreads();
      if (tid == 0) {
        double M1 = red[0], m1 = redmin[0];
        for (int w = 1; w < CTHREADS / 32; ++w) { M1 = fmax(M1, red[w]); m1 = fmin(m1, redmin[w]); }
        a.cond_out[b] = (M1 / m1) * (M1 / m1);
      }
      __syncthreads();
    }
    if (!a.inv2) return;
    cta_chol_inverse(A, ld, s, dY, a.inv2 + (int64_t)b * s * s);
    return;
  }
  cta_chol_inverse(A, ld, s, dY, out);
}

int launch_chol_system(const SysArgs& a, int p, cudaStream_t st) {
  if (p <= 0) return RAC_OK;
  const int s = a.s;
  const int mode = a.mode;
  const int use_packed = (mode == FACTOR_INVERSE && packed_bytes(s) <= kMaxDyn) ? 1 : 0;
  const int use_square = (square_bytes(s) <= kMaxDyn) ? 1 : 0;
  if (!use_square && !a.scratch) return set_error(RAC_ERR_ARG, "factor: scratch required for s=%d", s);
  if (mode == FACTOR_INVERSE && !use_packed && !a.only_failed) {
    // large blocks: blocked sweep over all blocks at once, then the Cholesky
    // route only for blocks it rejected (authoritative PD test)
    int rc = launch_inverse_large(a, p, st);
    if (rc) return rc;
    SysArgs b2 = a;
    b2.only_failed = 1;
    return launch_chol_system(b2, p, st);
  }
  size_t smem = 0;
  if (use_packed) smem = packed_bytes(s);
  if (use_square) smem = std::max(smem, square_bytes(s));
  int rc = check_cuda(cudaFuncSetAttribute(factor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                      "factor smem attribute");
  if (rc) return rc;
  factor_kernel<<<p, CTHREADS, smem, st>>>(a, mode, use_packed, use_square);
  note_launch();
  return check_launch("factor");
}

size_t chol_scratch_bytes(int s, int p) {
  if (square_bytes(s) <= kMaxDyn) return 0;
  const size_t chol = (size_t)p * ((size_t)s * (s + 1) + s) * sizeof(double);
  return packed_bytes(s) <= kMaxDyn ? chol : std::max(chol, large_scratch_bytes(s, p));
}

}  // namespace rac
