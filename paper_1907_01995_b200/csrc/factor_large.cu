// K3 for large blocks (s > 236, e.g. BASELINE config 5 with s = 500): the
// explicit block inverse by a BLOCKED symmetric sweep (Gauss-Jordan) run as a
// sequence of GPU-wide launches over all p blocks of the sweep at once.
//
// The block system lives in global memory as 64 x 64 lower tiles of an
// S x S matrix (S = s rounded up to 64, padding = identity).  For each pivot
// tile K:
//   (a) W   = A_KK^{-1}              one CTA per block, packed sweep in smem
//   (b) CW_I = A_IK W                 one CTA per (block, tile row I != K)
//   (c) A_IJ -= CW_I A_JK'            one CTA per (block, lower tile I>=J, I,J != K)
//   (d) A_IK = CW_I, A_KK = -W        K row / column rewritten
// and finally inv = -A.  (b) and (c) are 64x64x64 products on FP64 tensor
// cores (DMMA.8x8x4).  A non-positive pivot marks the block; such blocks are
// re-done by the authoritative Cholesky kernel (factor.cu).
#include "rac_internal.h"

#include <algorithm>

namespace rac {

constexpr int LT = 64;           // tile side
constexpr int LLD = LT + 4;      // smem stride (conflict-free fragment loads)
constexpr int LTHREADS = 256;

size_t large_scratch_bytes(int s, int p) {
  const size_t S = (size_t)(s + LT - 1) / LT * LT;
  return (size_t)p * (S * S + S * LT + 2 * LT * LT) * sizeof(double);
}

struct LargeBufs {
  int p;
  double* A;    // [p][S][S]   (only lower tiles maintained)
  double* CW;   // [p][S][LT]
  double* W;    // [2][p][LT][LT]: W of pivot step kt in half kt & 1 (the look-ahead pivot of
                //   step kt + 1 is written while step kt's strip still reads W_kt)
  int S, nt;
};

__device__ __forceinline__ LargeBufs large_bufs(double* scratch, int s, int p) {
  LargeBufs L;
  L.p = p;
  L.S = (s + LT - 1) / LT * LT;
  L.nt = L.S / LT;
  L.A = scratch;
  L.CW = L.A + (size_t)p * L.S * L.S;
  L.W = L.CW + (size_t)p * L.S * LT;
  return L;
}

// (0) assemble the padded block systems (lower part) from the split-K partials: one warp per
// row i, lanes over the columns j <= i (coalesced reads of the Gram row, writes of A's row)
__global__ void large_assemble_kernel(SysArgs a, int p) {
  if (a.done && *a.done) return;
  const int s = a.s;
  const LargeBufs L = large_bufs(a.scratch, s, p);
  const int b = blockIdx.y;
  const int32_t* bidx = a.idx ? a.idx + (int64_t)b * s : nullptr;
  double* A = L.A + (size_t)b * L.S * L.S;
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < L.S; i += nw) {
    const bool ivalid = i < s && !(bidx && bidx[i] < 0);
    const int64_t gi = ivalid && bidx ? (int64_t)bidx[i] * a.ldh : 0;
    for (int j = lane; j <= i; j += 32) {
      double v;
      if (!ivalid || j >= s || (bidx && bidx[j] < 0)) {
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
        if (a.H || a.hblk) {
          const double h = a.hblk ? a.hblk[((int64_t)b * s + i) * s + j] : a.H[gi + bidx[j]];
          v = a.ws ? h + v : h;
        }
        if (i == j) v += a.shift;
      }
      A[(int64_t)i * L.S + j] = v;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) a.info[b] = 0;
}

// (a) W = inv(A_KK): symmetric sweep of the 64x64 diagonal block held in REGISTERS: thread
// (i, quarter) owns row i's 16 columns 16*quarter..; per pivot q the owner of column q
// publishes it (double-buffered in smem, one barrier per pivot), and every thread updates
// its 16 entries.  The sweep keeps the matrix symmetric, so column q is also row q.
__device__ void pivot_sweep(const SysArgs& a, const LargeBufs& L, int b, int kt) {
  static_assert(LTHREADS == 4 * LT, "thread = (row, quarter of the columns)");
  __shared__ __align__(16) double col[2][LT];
  const double* A = L.A + (size_t)b * L.S * L.S;
  const int tid = threadIdx.x, i = tid >> 2, j0 = (tid & 3) * 16, k0 = kt * LT;
  double v[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    const int j = j0 + u;
    v[u] = (j <= i) ? A[(int64_t)(k0 + i) * L.S + k0 + j] : A[(int64_t)(k0 + j) * L.S + k0 + i];
  }
  if ((tid & 3) == 0) col[0][i] = v[0];   // column 0 = row i's entry 0 (owner: quarter 0)
  __syncthreads();
  int fail = 0;
  for (int q = 0; q < LT; ++q) {
    const double* c = col[q & 1];
    const double d = c[q];
    if (!(d > 0.0) || !isfinite(d)) {
      fail = k0 + q + 1;    // uniform: every thread read the same pivot
      break;
    }
    const double dinv = __drcp_rn(d);   // correctly rounded: the same value as 1.0 / d, no division slow path
    const double ri = c[i] * dinv;
    double cj[16];
#pragma unroll
    for (int u = 0; u < 16; u += 2) {
      const double2 t = *reinterpret_cast<const double2*>(c + j0 + u);
      cj[u] = t.x;
      cj[u + 1] = t.y;
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int j = j0 + u;
      if (j == q) v[u] = (i == q) ? -dinv : ri;
      else if (i == q) v[u] = cj[u] * dinv;
      else v[u] = v[u] - ri * cj[u];
    }
    // publish column q + 1 (owned by quarter (q + 1) / 16) for the next pivot
    if (q + 1 < LT && (tid & 3) == ((q + 1) >> 4)) {
#pragma unroll
      for (int u = 0; u < 16; ++u)
        if (j0 + u == q + 1) col[(q + 1) & 1][i] = v[u];
    }
    __syncthreads();
  }
  if (fail) {
    if (tid == 0) a.info[b] = fail;
    return;
  }
  double* W = L.W + ((size_t)(kt & 1) * L.p + b) * LT * LT;
#pragma unroll
  for (int u = 0; u < 16; ++u) W[i * LT + j0 + u] = -v[u];   // +inv
}

__global__ void __launch_bounds__(LTHREADS) large_pivot_kernel(SysArgs a, int p, int kt) {
  if (a.done && *a.done) return;
  const LargeBufs L = large_bufs(a.scratch, a.s, p);
  const int b = blockIdx.x;
  if (a.info[b]) return;
  pivot_sweep(a, L, b, kt);
}

// load a 64x64 tile (row-major, ld) into smem [r][c] (optionally transposed).
// Straight tiles: 16-byte cp.async (all 8 per thread in flight; the caller's
// cp_async_wait + __syncthreads completes them).  Transposed tiles: all 16
// loads per thread issued before the shared-memory stores.
__device__ __forceinline__ void load_tile(double (*dst)[LLD], const double* src, int64_t ld, bool trans) {
  if (!trans) {
#pragma unroll
    for (int u = 0; u < (LT * LT / 2) / LTHREADS; ++u) {
      const int e = threadIdx.x + u * LTHREADS;
      const int r = e / (LT / 2), c = 2 * (e - r * (LT / 2));
      cp_async16(&dst[r][c], src + (int64_t)r * ld + c);
    }
    cp_async_commit();
  } else {
    double v[LT * LT / LTHREADS];
#pragma unroll
    for (int u = 0; u < LT * LT / LTHREADS; ++u) {
      const int e = threadIdx.x + u * LTHREADS;
      v[u] = src[(int64_t)(e / LT) * ld + (e % LT)];
    }
#pragma unroll
    for (int u = 0; u < LT * LT / LTHREADS; ++u) {
      const int e = threadIdx.x + u * LTHREADS;
      dst[e % LT][e / LT] = v[u];
    }
  }
}

// C(64x64, in registers of the warp tiles) += alpha * X(64x64) * Y(64x64)'
// sX[i][k], sY[j][k]; warp w computes rows 16*(w/2).., cols 32*(w%2)..
__device__ __forceinline__ void tile_mma(const double (*sX)[LLD], const double (*sY)[LLD], double acc[2][4][2],
                                         double alpha) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int r0 = (warp >> 1) * 16, c0 = (warp & 1) * 32;
#pragma unroll 4
  for (int k = 0; k < LT; k += 4) {
    double af[2], bf[4];
#pragma unroll
    for (int i = 0; i < 2; ++i) af[i] = alpha * sX[r0 + i * 8 + g][k + t];
#pragma unroll
    for (int j = 0; j < 4; ++j) bf[j] = sY[c0 + j * 8 + g][k + t];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
  }
}

// (b) CW_I = A_IK * W for every tile row I != K
__global__ void __launch_bounds__(LTHREADS) large_cw_kernel(SysArgs a, int p, int kt) {
  if (a.done && *a.done) return;
  const LargeBufs L = large_bufs(a.scratch, a.s, p);
  const int b = blockIdx.y;
  int I = blockIdx.x;
  if (I >= kt) ++I;   // skip K
  if (a.info[b]) return;
  extern __shared__ __align__(16) double lsm[];
  double(*sX)[LLD] = reinterpret_cast<double(*)[LLD]>(lsm);
  double(*sY)[LLD] = reinterpret_cast<double(*)[LLD]>(lsm + LT * LLD);
  const double* A = L.A + (size_t)b * L.S * L.S;
  // X = A_IK (rows i of tile I, k of tile K); Y rows j = W columns: W symmetric, Y[j][k] = W[j][k]
  if (I > kt) load_tile(sX, A + (int64_t)I * LT * L.S + kt * LT, L.S, false);
  else load_tile(sX, A + (int64_t)kt * LT * L.S + I * LT, L.S, true);
  load_tile(sY, L.W + ((size_t)(kt & 1) * p + b) * LT * LT, LT, false);
  cp_async_wait<0>();
  __syncthreads();
  double acc[2][4][2] = {};
  tile_mma(sX, sY, acc, 1.0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int r0 = (warp >> 1) * 16, c0 = (warp & 1) * 32;
  double* CW = L.CW + ((size_t)b * L.S + (size_t)I * LT) * LT;
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) CW[(size_t)(r0 + i * 8 + g) * LT + c0 + j * 8 + 2 * t + e] = acc[i][j][e];
}

// (c) A_IJ -= CW_I * A_JK'   for lower tiles I >= J with I, J != K
// grid (p, tiles): the first tile of every block is the NEXT pivot tile (K+1, K+1), so those
// CTAs are dispatched first; after its update the CTA also inverts it (the next step's pivot,
// look-ahead), overlapping that latency-bound sweep with the rest of this update.
__global__ void __launch_bounds__(LTHREADS) large_update_kernel(SysArgs a, int p, int kt) {
  if (a.done && *a.done) return;
  const LargeBufs L = large_bufs(a.scratch, a.s, p);
  const int b = blockIdx.x;
  if (a.info[b]) return;
  // tile index over the lower triangle of the (nt-1) x (nt-1) grid without K; index 0 is
  // remapped to the next diagonal tile (reduced index (kt, kt)) when there is a next step
  const int m = L.nt - 1;
  const bool lookahead = kt + 1 < L.nt;
  const int dnext = kt * (kt + 1) / 2 + kt;
  int e = blockIdx.y;
  if (lookahead) e = (e == 0) ? dnext : (e <= dnext ? e - 1 : e);
  int I = 0, J = e;
  while (J > I) { J -= I + 1; ++I; }
  if (I >= m) return;
  if (I >= kt) ++I;
  if (J >= kt) ++J;
  extern __shared__ __align__(16) double lsm[];
  double(*sX)[LLD] = reinterpret_cast<double(*)[LLD]>(lsm);
  double(*sY)[LLD] = reinterpret_cast<double(*)[LLD]>(lsm + LT * LLD);
  double* A = L.A + (size_t)b * L.S * L.S;
  load_tile(sX, L.CW + ((size_t)b * L.S + (size_t)I * LT) * LT, LT, false);
  // Y[j][k] = A[J*64 + j][K*64 + k]
  if (J > kt) load_tile(sY, A + (int64_t)J * LT * L.S + kt * LT, L.S, false);
  else load_tile(sY, A + (int64_t)kt * LT * L.S + J * LT, L.S, true);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int r0 = (warp >> 1) * 16, c0 = (warp & 1) * 32;
  double* C = A + (int64_t)I * LT * L.S + J * LT;
  double acc[2][4][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) acc[i][j][e] = C[(int64_t)(r0 + i * 8 + g) * L.S + c0 + j * 8 + 2 * t + e];
  cp_async_wait<0>();
  __syncthreads();
  tile_mma(sX, sY, acc, -1.0);
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) C[(int64_t)(r0 + i * 8 + g) * L.S + c0 + j * 8 + 2 * t + e] = acc[i][j][e];
  if (lookahead && I == kt + 1 && J == kt + 1) {
    __syncthreads();   // the updated tile (global, written by this CTA) is the next pivot
    pivot_sweep(a, L, b, kt + 1);
  }
}

// (d) K strip: A_IK = CW_I (lower tiles, transposed above K), A_KK = -W
__global__ void large_strip_kernel(SysArgs a, int p, int kt) {
  if (a.done && *a.done) return;
  const LargeBufs L = large_bufs(a.scratch, a.s, p);
  const int b = blockIdx.y;
  if (a.info[b]) return;
  const int I = blockIdx.x;   // 0..nt-1
  double* A = L.A + (size_t)b * L.S * L.S;
  for (int e = threadIdx.x; e < LT * LT; e += blockDim.x) {
    const int i = e / LT, j = e - i * LT;
    if (I == kt) {
      if (j <= i) A[(int64_t)(kt * LT + i) * L.S + kt * LT + j] = -L.W[((size_t)(kt & 1) * p + b) * LT * LT + e];
    } else {
      const double v = L.CW[((size_t)b * L.S + (size_t)I * LT + i) * LT + j];   // CW_I[i][j] = A'_{I i, K j}
      if (I > kt) A[(int64_t)(I * LT + i) * L.S + kt * LT + j] = v;
      else A[(int64_t)(kt * LT + j) * L.S + I * LT + i] = v;          // lower tile (K, I)
    }
  }
}

// (e) inv = -A (symmetric, s x s)
__global__ void large_out_kernel(SysArgs a, int p) {
  if (a.done && *a.done) return;
  const int s = a.s;
  const LargeBufs L = large_bufs(a.scratch, s, p);
  const int b = blockIdx.y;
  if (a.info[b]) return;
  const double* A = L.A + (size_t)b * L.S * L.S;
  double* out = a.inv + (int64_t)b * s * s;
  const int64_t total = (int64_t)s * s;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / s), j = (int)(e - (int64_t)i * s);
    out[e] = -((j <= i) ? A[(int64_t)i * L.S + j] : A[(int64_t)j * L.S + i]);
  }
}

int launch_inverse_large(const SysArgs& a, int p, cudaStream_t st) {
  const int S = (a.s + LT - 1) / LT * LT, nt = S / LT;
  const size_t smem = 2 * LT * LLD * sizeof(double);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(large_cw_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    cudaFuncSetAttribute(large_update_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                         cudaSharedmemCarveoutMaxShared);
    int rc = check_cuda(cudaFuncSetAttribute(large_cw_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                        "large_cw smem");
    if (rc) return rc;
    rc = check_cuda(cudaFuncSetAttribute(large_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                    "large_update smem");
    if (rc) return rc;
    attr = true;
  }
  large_assemble_kernel<<<dim3((S + 7) / 8, p), 256, 0, st>>>(a, p);
  // the first pivot is its own launch; every later one runs inside the previous step's update
  large_pivot_kernel<<<p, LTHREADS, 0, st>>>(a, p, 0);
  for (int kt = 0; kt < nt; ++kt) {
    if (nt > 1) {
      large_cw_kernel<<<dim3(nt - 1, p), LTHREADS, smem, st>>>(a, p, kt);
      const int m = nt - 1;
      const int ntiles = m * (m + 1) / 2;
      if (ntiles > 0) large_update_kernel<<<dim3(p, ntiles), LTHREADS, smem, st>>>(a, p, kt);
    }
    large_strip_kernel<<<dim3(nt, p), 256, 0, st>>>(a, p, kt);
  }
  large_out_kernel<<<dim3(32, p), 256, 0, st>>>(a, p);
  note_launch(3 + nt * (nt > 1 ? 3 : 1));
  return check_launch("inverse_large");
}

}  // namespace rac
