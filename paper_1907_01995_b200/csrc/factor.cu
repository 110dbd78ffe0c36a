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

// The lower triangle is kept as 8 x 8 tiles: tile (I, J), J <= I, at (I (I + 1) / 2 + J) * 64
// doubles, row-major inside (diagonal tiles are stored whole; their upper part is never read
// as a value).  The rank-8 update then loads and stores a tile's DMMA fragment as one 16-byte
// access per lane, 512 contiguous bytes per warp: conflict-free, where rows of the packed
// triangle collided 3-4 ways (the update is bound by shared-memory wavefronts).
__host__ __device__ __forceinline__ int tri_tiles(int s8) { return (s8 >> 3) * ((s8 >> 3) + 1) / 2; }
__device__ __forceinline__ int pk(int i, int j) {   // j <= i
  const int I = i >> 3, J = j >> 3;
  return ((I * (I + 1) / 2 + J) << 6) + ((i & 7) << 3) + (j & 7);
}
// stride of the 8-row panel buffers Cm / CW: = 4 mod 16 doubles, so the update's fragment loads
// (lane (g, t): row t or t + 4, column 8 I + g) fall on 32 distinct bank pairs
__host__ __device__ __forceinline__ int panel_stride(int s8) { return s8 + ((4 - (s8 & 15)) + 16) % 16; }

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

// blocked symmetric sweep on the tiled lower triangle P (-> -P^{-1}); 0 or k+1.  s % 8 == 0
// (the caller pads with identity rows); sp = panel_stride(s).
__device__ int cta_sweep_packed(double* P, int s, int sp, double* Cm, double* CW, double* W, int* fail,
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
    for (int e = tid; e < SB * s; e += CTHREADS) {
      const int q = e / s, i = e - q * s, c = k + q;
      Cm[q * sp + i] = (i >= c) ? P[pk(i, c)] : P[pk(c, i)];
    }
    __syncthreads();
    stamp();
    if (ty == 0) {
      // 8x8 diagonal block swept in registers: lane l holds (r0 = l/8, c = l%8)
      // and (r0 + 4, c); pivot rows/columns move by warp shuffles.
      const int r0 = tx >> 3, c = tx & 7, r1 = r0 + 4;
      double v0 = Cm[c * sp + k + r0];
      double v1 = Cm[c * sp + k + r1];
      int f = 0;
      // branch-free (selects only) and fully unrolled: every lane runs the same
      // instruction stream; a non-positive pivot is recorded, the rest ignored
#pragma unroll
      for (int q = 0; q < SB; ++q) {
        const double d = __shfl_sync(0xffffffffu, (q < 4) ? v0 : v1, (q & 3) * 8 + q);  // W[q][q]
        const double wq0 = __shfl_sync(0xffffffffu, v0, r0 * 8 + q);     // W[r0][q]
        const double wq1 = __shfl_sync(0xffffffffu, v1, r0 * 8 + q);     // W[r1][q]
        const double wqc = __shfl_sync(0xffffffffu, (q < 4) ? v0 : v1, (q & 3) * 8 + c);  // W[q][c]
        const bool ok = (d > 0.0) && isfinite(d);
        if (!ok && !f) f = k + q + 1;
        const double dinv = __drcp_rn(ok ? d : 1.0);
        v0 = (r0 == q) ? ((c == q) ? -dinv : wqc * dinv) : ((c == q) ? wq0 * dinv : v0 - wq0 * wqc * dinv);
        v1 = (r1 == q) ? ((c == q) ? -dinv : wqc * dinv) : ((c == q) ? wq1 * dinv : v1 - wq1 * wqc * dinv);
      }
      if (tx == 0 && f) *fail = f;
      W[tx] = -v0;
      W[tx + 32] = -v1;
    }
    __syncthreads();
    stamp();
    if (*fail) return *fail;
    for (int e = tid; e < SB * s; e += CTHREADS) {
      const int q = e / s, i = e - q * s;
      double acc = 0.0;
#pragma unroll
      for (int r = 0; r < SB; ++r) acc += Cm[r * sp + i] * W[r * SB + q];
      CW[q * sp + i] = acc;
    }
    __syncthreads();
    stamp();
    {
      // rank-8 update  A_RR -= CW Cm'  on FP64 tensor cores: one m8n8k4 pair per
      // 8x8 lower tile (D = C - A B, A = CW rows, B = Cm rows); the K strip is
      // rewritten below.  lane (g, t): A[g][t], B[t][g], D[g][2t..2t+1].
      const int ntiles = tri_tiles(s);
      const int g = tx >> 2, t4 = tx & 3;
      int I = 0, J = ty;   // tile ty in row-major lower-triangle order, advanced by 16
      while (J > I) { J -= I + 1; ++I; }
      for (int tile = ty; tile < ntiles; tile += CTHREADS / 32) {
        double2* pt = reinterpret_cast<double2*>(P + (tile << 6) + (g << 3) + 2 * t4);
        double2 d = *pt;
        const double a0 = -CW[t4 * sp + 8 * I + g], a1 = -CW[(t4 + 4) * sp + 8 * I + g];
        const double b0 = Cm[t4 * sp + 8 * J + g], b1 = Cm[(t4 + 4) * sp + 8 * J + g];
        dmma884(d.x, d.y, a0, b0);
        dmma884(d.x, d.y, a1, b1);
        *pt = d;
        J += CTHREADS / 32;
        while (J > I) { J -= I + 1; ++I; }
      }
      __syncthreads();
      // K strip: rows >= k of columns K, and the K rows left of the strip
      for (int e = tid; e < (s - k) * SB; e += CTHREADS) {
        const int i = k + e / SB, q = e % SB, j = k + q;
        if (j > i) continue;
        P[pk(i, j)] = (i < k + SB) ? -W[(i - k) * SB + q] : CW[q * sp + i];
      }
      for (int e = tid; e < k * SB; e += CTHREADS) {
        const int q = e / k, j = e - q * k, i = k + q;
        P[pk(i, j)] = CW[q * sp + j];
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
  const int s8 = (s + 7) & ~7;
  return ((size_t)tri_tiles(s8) * 64 + 2 * SB * (size_t)panel_stride(s8)) * sizeof(double);
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
    const int sp = panel_stride(s8);
    const int ntri = tri_tiles(s8) * 64;   // doubles of the tiled triangle
    double* P = fsm;
    double* Cm = fsm + ntri;
    double* CW = Cm + SB * sp;
    double* hbo = a.hbb_out ? a.hbb_out + (int64_t)b * s * s : nullptr;
    const int tx = tid & 31, ty = tid >> 5;
    // block indices staged in smem (Cm is free until the sweep), then every thread fetches
    // batches of 8 independent entries (one L2 round trip per 8 * CTHREADS entries)
    int* sbi = reinterpret_cast<int*>(Cm);
    for (int i = tid; i < s; i += CTHREADS) sbi[i] = bidx ? bidx[i] : i;
    __syncthreads();
    const double* wsb = a.ws ? a.ws + (int64_t)b * a.splits * s * s : nullptr;
    for (int e0 = 0; e0 < ntri; e0 += 8 * CTHREADS) {
      double v[8];
      int pos[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + u * CTHREADS + tid;
        pos[u] = e;
        double val = 0.0;
        if (e < ntri) {
          // tile T = I (I + 1) / 2 + J of the triangle, element (w / 8, w % 8) inside
          const int T = e >> 6, w = e & 63;
          int I = (int)((sqrtf(8.0f * (float)T + 1.0f) - 1.0f) * 0.5f);
          while ((I + 1) * (I + 2) / 2 <= T) ++I;
          while (I * (I + 1) / 2 > T) --I;
          const int J = T - I * (I + 1) / 2;
          const int i = 8 * I + (w >> 3), j = 8 * J + (w & 7);
          val = (i == j) ? 1.0 : 0.0;
          if (i < s && j <= i) {
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
          } else if (j > i) {
            val = 0.0;   // upper part of a diagonal tile: carried along by the update, never used
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
    const int f = cta_sweep_packed(P, s8, sp, Cm, CW, W, &fail, tr);
    __syncthreads();
    if (!f) {
      if (tid == 0) a.info[b] = 0;
      // inv = -P, both orientations from each lower tile: a warp per tile, lane (g, t) holds
      // (8 I + g, 8 J + 2 t .. + 1): 64 contiguous bytes per row either way
      {
        const int g = tx >> 2, t4 = tx & 3;
        int I = 0, J = ty;
        while (J > I) { J -= I + 1; ++I; }
        for (int tile = ty; tile < tri_tiles(s8); tile += CTHREADS / 32) {
          const double2 d = *reinterpret_cast<const double2*>(P + (tile << 6) + (g << 3) + 2 * t4);
          const int i = 8 * I + g;
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int j = 8 * J + 2 * t4 + u;
            if (i < s && j <= i) {
              const double v = -(u ? d.y : d.x);
              out[(int64_t)i * s + j] = v;
              if (j < i) out[(int64_t)j * s + i] = v;
            }
          }
          J += CTHREADS / 32;
          while (J > I) { J -= I + 1; ++I; }
        }
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
