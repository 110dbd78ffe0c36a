// K2/K3 — batched block systems of one partition.
//
//   K2  sys_b  = V_b' V_b for every block b of the sweep (elastic_net.py:210,
//       engine.py:114 `Ab.T @ Ab`, svm.py:241 via the label Gram), computed on
//       FP64 tensor cores (mma.sync m8n8k4 f64 -> SASS DMMA.8x8x4).  Block
//       systems depend only on the block indices, never on the iterates, so
//       all p blocks of a sweep are formed in one launch before the sequential
//       Gauss-Seidel chain starts.
//   K3  L_b = chol(sys_b), inv_b = sys_b^{-1} = L^-T L^-1 (elastic_net.py:213-222,
//       engine.py:160-172).  The chain then solves each block with one
//       parallel mat-vec instead of two dependent triangular sweeps.
#include "rac_internal.h"

#include <algorithm>

namespace rac {

constexpr int GT = 64;        // CTA tile (rows/cols of the block Gram)
constexpr int GKC = 32;       // k-chunk (rows of V per pipeline stage)
constexpr int GLD = GKC + 4;  // padded smem row: conflict-free DMMA fragment loads
constexpr int GTHREADS = 256;

GramPlan plan_gram(int64_t len, int s, int p) {
  GramPlan pl;
  pl.tiles = (s + GT - 1) / GT;
  pl.pairs = pl.tiles * (pl.tiles + 1) / 2;
  const int64_t nchunks = (len + GKC - 1) / GKC;
  const int64_t ctas = (int64_t)p * pl.pairs;
  const int64_t target = 2LL * num_sms();
  int64_t splits = (target + ctas - 1) / ctas;
  splits = std::max<int64_t>(1, std::min<int64_t>(splits, std::max<int64_t>(1, nchunks / 8)));
  splits = std::min<int64_t>(splits, 64);
  int64_t per = (nchunks + splits - 1) / splits;
  splits = (nchunks + per - 1) / per;
  pl.splits = (int)splits;
  pl.chunk = per * GKC;
  return pl;
}

size_t gram_ws_bytes(int64_t len, int s, int p) {
  GramPlan pl = plan_gram(len, s, p);
  return (size_t)p * pl.splits * s * s * sizeof(double);
}

// ws[b][z][i][j] (j <= i) = sum_{k in split z} V[idx_b[i]][k] * V[idx_b[j]][k]
__global__ void __launch_bounds__(GTHREADS) gram_kernel(const double* __restrict__ V, int64_t ldv,
                                                       int64_t len, const int32_t* __restrict__ idx,
                                                       const int32_t* __restrict__ blk_list, int s,
                                                       int splits, int64_t chunk,
                                                       double* __restrict__ ws,
                                                       const int32_t* __restrict__ done) {
  if (done && *done) return;
  extern __shared__ __align__(16) double gsm[];
  double* sA[2] = {gsm, gsm + GT * GLD};
  double* sB[2] = {gsm + 2 * GT * GLD, gsm + 3 * GT * GLD};

  const int pair = blockIdx.x;
  int I = 0;
  while ((I + 1) * (I + 2) / 2 <= pair) ++I;
  const int J = pair - I * (I + 1) / 2;
  const int b = blk_list ? blk_list[blockIdx.y] : blockIdx.y;
  const int z = blockIdx.z;
  const bool diag = (I == J);
  const int32_t* bidx = idx + (int64_t)b * s;

  const int64_t k_begin = (int64_t)z * chunk;
  const int64_t k_end = min(len, k_begin + chunk);
  const int nck = (int)((k_end - k_begin + GKC - 1) / GKC);

  const int tid = threadIdx.x;
  // Column sources for the two tiles (-1: padding column -> zeros).
  __shared__ int64_t colA[GT], colB[GT];
  if (tid < GT) {
    int gi = I * GT + tid;
    int v = (gi < s) ? bidx[gi] : -1;
    colA[tid] = (v >= 0) ? (int64_t)v * ldv : -1;
    int gj = J * GT + tid;
    int w = (gj < s) ? bidx[gj] : -1;
    colB[tid] = (w >= 0) ? (int64_t)w * ldv : -1;
  }
  __syncthreads();
  // zero padding columns once (both stages); they are never loaded
  for (int e = tid; e < GT * GLD; e += GTHREADS) {
    int c = e / GLD;
    if (colA[c] < 0) { sA[0][e] = 0.0; sA[1][e] = 0.0; }
    if (!diag && colB[c] < 0) { sB[0][e] = 0.0; sB[1][e] = 0.0; }
  }

  auto load_stage = [&](int stage, int64_t k0) {
    // 64 columns x 32 doubles = 64 x 16 16-byte pieces per tile
    for (int e = tid; e < GT * (GKC / 2); e += GTHREADS) {
      int c = e >> 4, q = e & 15;
      int64_t a = colA[c];
      if (a >= 0) cp_async16(sA[stage] + c * GLD + 2 * q, V + a + k0 + 2 * q);
      if (!diag) {
        int64_t bb = colB[c];
        if (bb >= 0) cp_async16(sB[stage] + c * GLD + 2 * q, V + bb + k0 + 2 * q);
      }
    }
    cp_async_commit();
  };

  // warp units: 16x16 sub-tiles of the 64x64 tile; warp w -> units w, w+8
  const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  int ur[2], uc[2];
  bool act[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    int u = warp + 8 * q;
    ur[q] = u >> 2;
    uc[q] = u & 3;
    act[q] = (I * GT + ur[q] * 16 < s) && (J * GT + uc[q] * 16 < s) && (!diag || uc[q] <= ur[q]);
  }
  double acc[2][4][2];
#pragma unroll
  for (int q = 0; q < 2; ++q)
#pragma unroll
    for (int r = 0; r < 4; ++r) acc[q][r][0] = acc[q][r][1] = 0.0;

  if (nck > 0) load_stage(0, k_begin);
  for (int ck = 0; ck < nck; ++ck) {
    const int cur = ck & 1;
    if (ck + 1 < nck) {
      load_stage(cur ^ 1, k_begin + (int64_t)(ck + 1) * GKC);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* A = sA[cur];
    const double* B = diag ? sA[cur] : sB[cur];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      if (!act[q]) continue;
      const double* a0p = A + (ur[q] * 16 + g) * GLD + t;
      const double* a1p = a0p + 8 * GLD;
      const double* b0p = B + (uc[q] * 16 + g) * GLD + t;
      const double* b1p = b0p + 8 * GLD;
#pragma unroll
      for (int kk = 0; kk < GKC; kk += 4) {
        double a0 = a0p[kk], a1 = a1p[kk], b0 = b0p[kk], b1 = b1p[kk];
        dmma884(acc[q][0][0], acc[q][0][1], a0, b0);
        dmma884(acc[q][1][0], acc[q][1][1], a0, b1);
        dmma884(acc[q][2][0], acc[q][2][1], a1, b0);
        dmma884(acc[q][3][0], acc[q][3][1], a1, b1);
      }
    }
    __syncthreads();
  }

  double* out = ws + ((int64_t)b * splits + z) * (int64_t)s * s;
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    if (!act[q]) continue;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      int row = I * GT + ur[q] * 16 + (r >> 1) * 8 + g;
      int col0 = J * GT + uc[q] * 16 + (r & 1) * 8 + 2 * t;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        int col = col0 + e;
        if (row < s && col < s && col <= row) out[(int64_t)row * s + col] = acc[q][r][e];
      }
    }
  }
}

int launch_gram(const double* V, int64_t ldv, int64_t len, const int32_t* idx,
                const int32_t* blk_list, int s, int p, double* ws, const GramPlan& pl,
                cudaStream_t st, const int32_t* done) {
  if (p <= 0) return RAC_OK;
  const size_t smem = 4 * GT * GLD * sizeof(double);
  int rc = check_cuda(cudaFuncSetAttribute(gram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                      "gram smem attribute");
  if (rc) return rc;
  dim3 grid(pl.pairs, p, pl.splits);
  gram_kernel<<<grid, GTHREADS, smem, st>>>(V, ldv, len, idx, blk_list, s, pl.splits, pl.chunk, ws, done);
  return check_launch("gram");
}

// ---------------------------------------------------------------------------
// K3: Cholesky + explicit inverse of each block system, one CTA per block.
//     sys = (sum_z ws_z) / div * mul  (+ H_bb)  + shift*I  (+ ridge_rel*max diag * I)
// The matrix lives in shared memory when it fits, else in a global scratch.
// ---------------------------------------------------------------------------


constexpr int CTHREADS = 512;

template <bool SMEM>
__global__ void __launch_bounds__(CTHREADS) chol_inverse_kernel(SysArgs a) {
  extern __shared__ __align__(16) double csm[];
  if (a.done && *a.done) return;
  const int s = a.s;
  const int slot = blockIdx.x;
  const int b = a.blk_list ? a.blk_list[slot] : slot;
  const int ld = s + 1;
  double* A = SMEM ? csm : a.scratch + (int64_t)b * s * ld;
  double* dY = SMEM ? csm + (int64_t)s * ld : a.inv + (int64_t)b * s * s;  // diag of L^-1 (uses inv row 0 as scratch in global mode)
  __shared__ int fail;
  __shared__ double red[CTHREADS / 32];
  const int tid = threadIdx.x;
  if (tid == 0) fail = 0;

  // ---- assemble
  const int32_t* bidx = a.idx ? a.idx + (int64_t)b * s : nullptr;
  double* hbo = a.hbb_out ? a.hbb_out + (int64_t)b * s * s : nullptr;
  for (int e = tid; e < s * s; e += CTHREADS) {
    int i = e / s, j = e - i * s;
    const bool pad = bidx && (bidx[i] < 0 || bidx[j] < 0);
    double v = 0.0;
    double h = 0.0;
    if (a.H && !pad) h = a.H[(int64_t)bidx[i] * a.ldh + bidx[j]];
    if (hbo) hbo[e] = h;
    if (pad) {
      v = (i == j) ? 1.0 : 0.0;   // keeps the short last block's leading part exact
    } else if (j <= i) {
      if (a.ws) {
        const double* src = a.ws + (int64_t)b * a.splits * s * s + (int64_t)i * s + j;
        double acc = src[0];
        for (int z = 1; z < a.splits; ++z) acc += src[(int64_t)z * s * s];
        if (a.div != 1.0) acc = acc / a.div;
        if (a.mul != 1.0) acc = a.mul * acc;
        v = acc;
      }
      if (a.H) v = a.ws ? h + v : h;
      if (i == j) v += a.shift;
    }
    A[(int64_t)i * ld + j] = v;
  }
  __syncthreads();
  if (a.ridge_rel > 0.0) {
    double mx = -INFINITY;
    for (int i = tid; i < s; i += CTHREADS)
      if (!bidx || bidx[i] >= 0) mx = fmax(mx, A[(int64_t)i * ld + i]);
    mx = warp_max(mx);
    if ((tid & 31) == 0) red[tid >> 5] = mx;
    __syncthreads();
    if (tid == 0) {
      double m2 = red[0];
      for (int w = 1; w < CTHREADS / 32; ++w) m2 = fmax(m2, red[w]);
      red[0] = a.ridge_rel * m2;
    }
    __syncthreads();
    const double ridge = red[0];
    for (int i = tid; i < s; i += CTHREADS)
      if (!bidx || bidx[i] >= 0) A[(int64_t)i * ld + i] += ridge;
    __syncthreads();
  }
  if (a.mat_out) {
    double* mo = a.mat_out + (int64_t)b * s * s;
    for (int e = tid; e < s * s; e += CTHREADS) {
      int i = e / s, j = e - i * s;
      mo[e] = (j <= i) ? A[(int64_t)i * ld + j] : A[(int64_t)j * ld + i];
    }
  }

  // ---- Cholesky (right-looking), L in the lower triangle (diag included)
  const int tx = tid & 31, ty = tid >> 5;  // 32 x 16 thread grid
  for (int k = 0; k < s; ++k) {
    if (tid == 0) {
      double d = A[(int64_t)k * ld + k];
      if (!(d > 0.0) || !isfinite(d)) {
        fail = k + 1;
      } else {
        A[(int64_t)k * ld + k] = sqrt(d);
      }
    }
    __syncthreads();
    if (fail) break;
    const double piv = A[(int64_t)k * ld + k];
    for (int i = k + 1 + tid; i < s; i += CTHREADS) A[(int64_t)i * ld + k] /= piv;
    __syncthreads();
    for (int i = k + 1 + ty; i < s; i += CTHREADS / 32) {
      const double lik = A[(int64_t)i * ld + k];
      for (int j = k + 1 + tx; j <= i; j += 32) A[(int64_t)i * ld + j] -= lik * A[(int64_t)j * ld + k];
    }
    __syncthreads();
  }
  if (fail) {
    if (tid == 0) a.info[b] = fail;
    return;
  }
  if (tid == 0) a.info[b] = 0;

  // ---- Y = L^{-1}: Y[i][c] (c < i) stored at A[c][i] (strict upper), diag in dY
  for (int e = tid; e < s * s; e += CTHREADS) {
    int c = e / s, i = e - c * s;
    if (c < i) A[(int64_t)c * ld + i] = 0.0;
  }
  __syncthreads();
  for (int k = 0; k < s; ++k) {
    const double lkk = A[(int64_t)k * ld + k];
    for (int c = tid; c < k; c += CTHREADS) A[(int64_t)c * ld + k] /= lkk;
    if (tid == 0) dY[k] = 1.0 / lkk;
    __syncthreads();
    // Y[i][c] -= L[i][k] * Y[k][c]   for i > k, c <= k
    for (int i = k + 1 + ty; i < s; i += CTHREADS / 32) {
      const double lik = A[(int64_t)i * ld + k];
      for (int c = tx; c <= k; c += 32) {
        const double ykc = (c == k) ? dY[k] : A[(int64_t)c * ld + k];
        A[(int64_t)c * ld + i] -= lik * ykc;
      }
    }
    __syncthreads();
  }

  // ---- inv = Y' Y :  inv[i][j] = sum_{r >= max(i,j)} Y[r][i] Y[r][j]
  double* out = a.inv + (int64_t)b * s * s;
  const int total = s * (s + 1) / 2;
  for (int e = tid; e < total; e += CTHREADS) {
    // e -> (i, j), j <= i, row-major over the lower triangle
    int i = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
    while ((i + 1) * (i + 2) / 2 <= e) ++i;
    while (i * (i + 1) / 2 > e) --i;
    int j = e - i * (i + 1) / 2;
    double acc = dY[i] * ((i == j) ? dY[j] : A[(int64_t)j * ld + i]);
    for (int r = i + 1; r < s; ++r) acc += A[(int64_t)i * ld + r] * A[(int64_t)j * ld + r];
    if (SMEM) {
      out[(int64_t)i * s + j] = acc;
      out[(int64_t)j * s + i] = acc;
    } else {
      // dY aliases out row 0 in global mode: stage through A's lower triangle (dead now)
      A[(int64_t)i * ld + j] = acc;
    }
  }
  if (!SMEM) {
    __syncthreads();
    for (int e = tid; e < s * s; e += CTHREADS) {
      int i = e / s, j = e - i * s;
      out[e] = (j <= i) ? A[(int64_t)i * ld + j] : A[(int64_t)j * ld + i];
    }
  }
}

// ---------------------------------------------------------------------------
// K3 (s <= 236): the block system is assembled into the PACKED lower triangle
// in shared memory and inverted in place by the symmetric sweep operator
// (Gauss-Jordan without pivoting, valid for SPD):  for each pivot k
//     d = a_kk;  a_ij -= a_ik a_kj / d;  a_ik /= d;  a_kk = -1/d
// which leaves -A^{-1}.  The pivots are the Cholesky pivots L_kk^2, so a
// non-positive pivot reports exactly the leading minor np.linalg.cholesky
// rejects (elastic_net.py:213-219, engine.py:160-167).  One CTA per block,
// s steps of two barriers each; no global round trips.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int pk(int i, int j) { return i * (i + 1) / 2 + j; }  // j <= i

__global__ void __launch_bounds__(CTHREADS) sweep_inverse_kernel(SysArgs a) {
  extern __shared__ __align__(16) double psm[];
  if (a.done && *a.done) return;
  const int s = a.s;
  const int b = a.blk_list ? a.blk_list[blockIdx.x] : blockIdx.x;
  double* P = psm;                                 // s(s+1)/2
  double* col = psm + (size_t)s * (s + 1) / 2;     // s
  __shared__ int fail;
  __shared__ double red[CTHREADS / 32];
  const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
  if (tid == 0) fail = 0;
  const int32_t* bidx = a.idx ? a.idx + (int64_t)b * s : nullptr;
  double* hbo = a.hbb_out ? a.hbb_out + (int64_t)b * s * s : nullptr;
  // ---- assemble (lower, packed)
  for (int i = ty; i < s; i += CTHREADS / 32) {
    const int off = pk(i, 0);
    for (int j = tx; j < s; j += 32) {
      const bool pad = bidx && (bidx[i] < 0 || bidx[j] < 0);
      double h = 0.0;
      if (a.H && !pad) h = a.H[(int64_t)bidx[i] * a.ldh + bidx[j]];
      if (hbo) hbo[(int64_t)i * s + j] = h;
      if (j > i) continue;
      double v;
      if (pad) {
        v = (i == j) ? 1.0 : 0.0;
      } else {
        v = 0.0;
        if (a.ws) {
          const double* src = a.ws + (int64_t)b * a.splits * s * s + (int64_t)i * s + j;
          double acc = src[0];
          for (int z = 1; z < a.splits; ++z) acc += src[(int64_t)z * s * s];
          if (a.div != 1.0) acc = acc / a.div;
          if (a.mul != 1.0) acc = a.mul * acc;
          v = acc;
        }
        if (a.H) v = a.ws ? h + v : h;
        if (i == j) v += a.shift;
      }
      P[off + j] = v;
    }
  }
  __syncthreads();
  if (a.ridge_rel > 0.0) {
    double mx = -INFINITY;
    for (int i = tid; i < s; i += CTHREADS)
      if (!bidx || bidx[i] >= 0) mx = fmax(mx, P[pk(i, i)]);
    mx = warp_max(mx);
    if (tx == 0) red[ty] = mx;
    __syncthreads();
    double m2 = red[0];
    for (int w = 1; w < CTHREADS / 32; ++w) m2 = fmax(m2, red[w]);
    const double ridge = a.ridge_rel * m2;
    __syncthreads();
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
  // ---- sweep every pivot
  for (int k = 0; k < s; ++k) {
    const double d = P[pk(k, k)];
    if (!(d > 0.0) || !isfinite(d)) {
      if (tid == 0) fail = k + 1;
      break;   // uniform: every thread read the same d
    }
    for (int i = tid; i < s; i += CTHREADS) col[i] = (i >= k) ? P[pk(i, k)] : P[pk(k, i)];
    __syncthreads();
    const double dinv = 1.0 / d;
    for (int i = ty; i < s; i += CTHREADS / 32) {
      const int off = pk(i, 0);
      const double ci = col[i];
      const double cid = ci * dinv;
      for (int j = tx; j <= i; j += 32) {
        double v;
        if (i == k) {
          v = (j == k) ? -dinv : col[j] * dinv;
        } else if (j == k) {
          v = cid;
        } else {
          v = P[off + j] - cid * col[j];
        }
        P[off + j] = v;
      }
    }
    __syncthreads();
  }
  __syncthreads();
  if (fail) {
    if (tid == 0) a.info[b] = fail;
    return;
  }
  if (tid == 0) a.info[b] = 0;
  double* out = a.inv + (int64_t)b * s * s;
  for (int e = tid; e < s * s; e += CTHREADS) {
    const int i = e / s, j = e - i * s;
    out[e] = -((j <= i) ? P[pk(i, j)] : P[pk(j, i)]);
  }
}

static size_t sweep_smem_bytes(int s) { return ((size_t)s * (s + 1) / 2 + s) * sizeof(double); }
static size_t chol_smem_bytes(int s) { return ((size_t)s * (s + 1) + s) * sizeof(double); }
static constexpr size_t kMaxSmem = 227 * 1024 - 2048;  // dynamic budget (static smem is extra)

int launch_chol_system(const SysArgs& a, int p, cudaStream_t st) {
  if (p <= 0) return RAC_OK;
  const size_t pmem = sweep_smem_bytes(a.s);
  if (pmem <= kMaxSmem) {
    int rc = check_cuda(cudaFuncSetAttribute(sweep_inverse_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)pmem),
                        "sweep_inverse smem attribute");
    if (rc) return rc;
    sweep_inverse_kernel<<<p, CTHREADS, pmem, st>>>(a);
    return check_launch("sweep_inverse");
  }
  const size_t smem = chol_smem_bytes(a.s);
  if (smem <= kMaxSmem) {
    int rc = check_cuda(cudaFuncSetAttribute(chol_inverse_kernel<true>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                        "chol_inverse smem attribute");
    if (rc) return rc;
    chol_inverse_kernel<true><<<p, CTHREADS, smem, st>>>(a);
  } else {
    if (!a.scratch) return set_error(RAC_ERR_ARG, "chol: scratch required for s=%d", a.s);
    chol_inverse_kernel<false><<<p, CTHREADS, 0, st>>>(a);
  }
  return check_launch("chol_inverse");
}

size_t chol_scratch_bytes(int s, int p) {
  if (sweep_smem_bytes(s) <= kMaxSmem || chol_smem_bytes(s) <= kMaxSmem) return 0;
  return (size_t)p * s * (s + 1) * sizeof(double);
}

}  // namespace rac

extern "C" size_t rac_gram_workspace_bytes(int64_t len, int32_t s, int32_t p) {
  return rac::gram_ws_bytes(len, s, p) + rac::chol_scratch_bytes(s, p);
}

extern "C" int rac_gram_inverse(const double* V, int64_t ldv, int64_t len, const int32_t* idx,
                                int32_t s, int32_t p, int64_t n_valid, double scale, double shift,
                                double* ws, double* inv, int32_t* info, void* stream) {
  using namespace rac;
  (void)n_valid;
  clear_error();
  if (!V || !idx || !ws || !inv || !info || s < 1 || p < 1 || len < 1)
    return set_error(RAC_ERR_ARG, "rac_gram_inverse: bad arguments");
  if ((ldv % 32) != 0 || ldv < len || (((uintptr_t)V) & 15))
    return set_error(RAC_ERR_ARG, "rac_gram_inverse: V must be 16B aligned with ldv %% 32 == 0");
  cudaStream_t st = (cudaStream_t)stream;
  GramPlan pl = plan_gram(len, s, p);
  int rc = launch_gram(V, ldv, len, idx, nullptr, s, p, ws, pl, st, nullptr);
  if (rc) return rc;
  SysArgs a{};
  a.ws = ws;
  a.splits = pl.splits;
  a.div = 1.0;
  a.mul = scale;
  a.shift = shift;
  a.s = s;
  a.inv = inv;
  a.info = info;
  a.scratch = ws + gram_ws_bytes(len, s, p) / sizeof(double);
  return launch_chol_system(a, p, st);
}
