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
  // Pick the K split that minimises (CTAs on the busiest SM) x (chunks per CTA + epilogue):
  // the DMMA pipe of an SM is shared by its resident CTAs, so a partially filled last
  // wave costs as much as a full one.  Ties go to fewer splits (less partial traffic).
  const int64_t sms = num_sms();
  const int64_t max_splits = std::max<int64_t>(1, std::min<int64_t>(64, nchunks / 4));
  int64_t best = 1;
  double best_cost = 1e300;
  for (int64_t sp = 1; sp <= max_splits; ++sp) {
    const int64_t per = (nchunks + sp - 1) / sp;
    const int64_t eff = (nchunks + per - 1) / per;
    const int64_t waves = (ctas * eff + sms - 1) / sms;
    const double cost = (double)waves * (double)(per + 2);
    if (cost < best_cost * 0.995) { best_cost = cost; best = eff; }
  }
  const int64_t per = (nchunks + best - 1) / best;
  pl.splits = (int)((nchunks + per - 1) / per);
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
                                                       const int32_t* __restrict__ done, double sym_div,
                                                       int sym_accum) {
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
        if (row < s && col < s && col <= row) {
          if (sym_accum) {
            // streaming ingest: raw sums accumulated chunk after chunk (fixed order)
            const double v = acc[q][r][e];
            out[(int64_t)row * s + col] += v;
            if (col != row) out[(int64_t)col * s + row] += v;
          } else if (sym_div > 0.0) {
            // single split, full symmetric output scaled like X_b'X_b / m (dot, then divide)
            const double v = acc[q][r][e] / sym_div;
            out[(int64_t)row * s + col] = v;
            out[(int64_t)col * s + row] = v;
          } else {
            out[(int64_t)row * s + col] = acc[q][r][e];
          }
        }
      }
    }
  }
}

int launch_gram(const double* V, int64_t ldv, int64_t len, const int32_t* idx,
                const int32_t* blk_list, int s, int p, double* ws, const GramPlan& pl,
                cudaStream_t st, const int32_t* done, double sym_div, int sym_accum) {
  if (p <= 0) return RAC_OK;
  const size_t smem = 4 * GT * GLD * sizeof(double);
  // maximal shared-memory carveout: the SM configuration then matches the chain kernels,
  // so Gram CTAs of the next sweep can co-reside with a latency-bound chain
  cudaFuncSetAttribute(gram_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  int rc = check_cuda(cudaFuncSetAttribute(gram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                      "gram smem attribute");
  if (rc) return rc;
  dim3 grid(pl.pairs, p, pl.splits);
  gram_kernel<<<grid, GTHREADS, smem, st>>>(V, ldv, len, idx, blk_list, s, pl.splits, pl.chunk, ws, done,
                                            sym_div, sym_accum);
  note_launch();
  return check_launch("gram");
}

// G[i][j] = G[j][i] = (sum_z ws[z][i][j]) / div for j <= i: the split-K partials of a
// single full Gram summed in fixed split order (deterministic), scaled, mirrored.
__global__ void gram_reduce_sym_kernel(const double* __restrict__ ws, int64_t n, int splits, double div,
                                       double* __restrict__ G) {
  const int64_t nn = n * n;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nn; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / n, j = e - i * n;
    if (j > i) continue;
    double acc = ws[e];
    for (int z = 1; z < splits; ++z) acc += ws[(int64_t)z * nn + e];
    const double v = acc / div;
    G[e] = v;
    G[j * n + i] = v;
  }
}

int launch_gram_reduce_sym(const double* ws, int64_t n, int splits, double div, double* G, cudaStream_t st) {
  gram_reduce_sym_kernel<<<num_sms() * 8, 256, 0, st>>>(ws, n, splits, div, G);
  note_launch();
  return check_launch("gram reduce");
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
