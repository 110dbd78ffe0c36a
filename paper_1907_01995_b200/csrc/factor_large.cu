// K3 for large blocks (s > 236, e.g. BASELINE config 5 with s = 500): the
// explicit block inverse by a BLOCKED symmetric sweep (Gauss-Jordan) run as a
// sequence of GPU-wide launches over all p blocks of the sweep at once.
//
// The block system lives in global memory as 64 x 64 lower tiles of an
// S x S matrix (S = s rounded up to 64, padding = identity).  For each pivot
// tile K:
//   (a) W   = A_KK^{-1}              one CTA per block, sweep held in registers
//   (b) CW_I = A_IK W                 one CTA per (block, tile row I != K); the same CTA rewrites
//                                     the K strip in place (A_IK = CW_I, A_KK = -W) and keeps the
//                                     old strip tile in OLD_I for (c)
//   (c) A_IJ -= CW_I OLD_J'           one CTA per (block, lower tile I>=J, I,J != K)
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
  return (size_t)p * (S * S + 2 * S * LT + 2 * LT * LT) * sizeof(double);
}

struct LargeBufs {
  int p;
  double* A;    // [p][S][S]   (only lower tiles maintained)
  double* CW;   // [p][S][LT]
  double* OLD;  // [p][S][LT]: the K strip before step K rewrote it (OLD_I[i][k] = A_IK[i][k])
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
  L.OLD = L.CW + (size_t)p * L.S * LT;
  L.W = L.OLD + (size_t)p * L.S * LT;
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
// A warp = 32 rows of ONE quarter: its lanes read the same 16 pivot-column entries (pure
// broadcasts; with the four quarters inside a warp every vector load was a 4-way bank
// conflict per quarter-warp, ~1000 shared-memory cycles per pivot).
__device__ void pivot_sweep(const SysArgs& a, const LargeBufs& L, int b, int kt) {
  static_assert(LTHREADS == 4 * LT, "thread = (row, quarter of the columns)");
  __shared__ __align__(16) double col[2][LT];
  const double* A = L.A + (size_t)b * L.S * L.S;
  const int tid = threadIdx.x, quarter = (tid >> 5) & 3, i = (tid >> 7) * 32 + (tid & 31), j0 = quarter * 16, k0 = kt * LT;
  double v[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    const int j = j0 + u;
    v[u] = (j <= i) ? A[(int64_t)(k0 + i) * L.S + k0 + j] : A[(int64_t)(k0 + j) * L.S + k0 + i];
  }
  if (quarter == 0) col[0][i] = v[0];   // column 0 = row i's entry 0 (owner: quarter 0)
  __syncthreads();
  int fail = 0;
  // pivots in groups of 16 = one quarter's columns: inside a group the pivot's position in
  // its owner's registers is a compile-time index, so a pivot costs the 16 FMAs, 8 vector
  // loads of the pivot column and a handful of predicated moves (the sweep is a chain of 64
  // dependent pivots: its latency, not its flop count, is what the look-ahead has to hide)
#pragma unroll 1
  for (int Q = 0; Q < LT / 16 && !fail; ++Q) {
#pragma unroll
    for (int uq = 0; uq < 16; ++uq) {
      const int q = Q * 16 + uq;
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
      if (i == q) {   // the pivot row (4 threads)
#pragma unroll
        for (int u = 0; u < 16; ++u) v[u] = cj[u] * dinv;
      } else {
#pragma unroll
        for (int u = 0; u < 16; ++u) v[u] = v[u] - ri * cj[u];
      }
      if (quarter == Q) v[uq] = (i == q) ? -dinv : ri;   // the pivot column
      // publish column q + 1 (owned by quarter (q + 1) / 16) for the next pivot
      if (q + 1 < LT && quarter == ((q + 1) >> 4)) col[(q + 1) & 1][i] = v[(uq + 1) & 15];
      __syncthreads();
    }
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

// (b) CW_I = A_IK * W for every tile row I != K.  The CTA also rewrites the K strip in place
// (A_IK = CW_I in the lower-tile orientation) after saving the old tile to OLD_I, and the first
// CTA of a block writes A_KK = -W.  Nothing else reads the K strip during this launch.
__global__ void __launch_bounds__(LTHREADS) large_cw_kernel(SysArgs a, int p, int kt) {
  const LargeBufs L = large_bufs(a.scratch, a.s, p);
  const int b = blockIdx.y;
  int I = blockIdx.x;
  if (I >= kt) ++I;   // skip K
  const int dn = a.done ? *a.done : 0;
  if (dn | a.info[b]) return;
  extern __shared__ __align__(16) double lsm[];
  double(*sX)[LLD] = reinterpret_cast<double(*)[LLD]>(lsm);
  double(*sY)[LLD] = reinterpret_cast<double(*)[LLD]>(lsm + LT * LLD);
  double* A = L.A + (size_t)b * L.S * L.S;
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
  double* OLD = L.OLD + ((size_t)b * L.S + (size_t)I * LT) * LT;
  const bool lastk = kt == L.nt - 1;   // last step: the strip is final, inv = -A goes straight out
  const int s = a.s;
  double* out = a.inv + (int64_t)b * s * s;
  // the old strip tile, as loaded
#pragma unroll
  for (int u = 0; u < (LT * LT / 2) / LTHREADS; ++u) {
    const int e = threadIdx.x + u * LTHREADS;
    const int r = e / (LT / 2), c = 2 * (e - r * (LT / 2));
    *reinterpret_cast<double2*>(OLD + (size_t)r * LT + c) = make_double2(sX[r][c], sX[r][c + 1]);
  }
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int row = r0 + i * 8 + g, col = c0 + j * 8 + 2 * t;
      const double2 v = make_double2(acc[i][j][0], acc[i][j][1]);
      *reinterpret_cast<double2*>(CW + (size_t)row * LT + col) = v;
      if (lastk) {   // I < K: inv[K k][I i] = inv[I i][K k] = -CW_I[i][k]
        const int gi = I * LT + row, gk = kt * LT + col;
        if (gi < s) {
          if (gk < s) {
            out[(int64_t)gk * s + gi] = -v.x;
            out[(int64_t)gi * s + gk] = -v.x;
          }
          if (gk + 1 < s) {
            out[(int64_t)(gk + 1) * s + gi] = -v.y;
            out[(int64_t)gi * s + gk + 1] = -v.y;
          }
        }
      } else if (I > kt) {
        *reinterpret_cast<double2*>(A + (int64_t)(I * LT + row) * L.S + kt * LT + col) = v;
      } else {   // lower tile (K, I): A[K k][I i] = CW_I[i][k]
        A[(int64_t)(kt * LT + col) * L.S + I * LT + row] = v.x;
        A[(int64_t)(kt * LT + col + 1) * L.S + I * LT + row] = v.y;
      }
    }
  if (blockIdx.x == 0) {   // A_KK = -W (lower part); last step: inv_KK = W
    for (int e = threadIdx.x; e < LT * LT; e += LTHREADS) {
      const int i = e / LT, j = e - i * LT;
      if (lastk) {
        const int gi = kt * LT + i, gj = kt * LT + j;
        if (gi < s && gj < s) out[(int64_t)gi * s + gj] = sY[max(i, j)][min(i, j)];
      } else if (j <= i) {
        A[(int64_t)(kt * LT + i) * L.S + kt * LT + j] = -sY[i][j];
      }
    }
  }
}

// (c) A_IJ -= CW_I * OLD_J'   for lower tiles I >= J with I, J != K   (OLD_J = A_JK before (b))
// grid (p, tiles): the first tile of every block is the NEXT pivot tile (K+1, K+1), so those
// CTAs are dispatched first; after its update the CTA also inverts it (the next step's pivot,
// look-ahead), overlapping that latency-bound sweep with the rest of this update.
__global__ void __launch_bounds__(LTHREADS) large_update_kernel(SysArgs a, int p, int kt) {
  const LargeBufs L = large_bufs(a.scratch, a.s, p);
  const int b = blockIdx.x;
  const int dn = a.done ? *a.done : 0;
  if (dn | a.info[b]) return;
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
  load_tile(sY, L.OLD + ((size_t)b * L.S + (size_t)J * LT) * LT, LT, false);   // Y[j][k] = A_JK[j][k]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int r0 = (warp >> 1) * 16, c0 = (warp & 1) * 32;
  double* C = A + (int64_t)I * LT * L.S + J * LT;
  double acc[2][4][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const double2 v = *reinterpret_cast<const double2*>(C + (int64_t)(r0 + i * 8 + g) * L.S + c0 + j * 8 + 2 * t);
      acc[i][j][0] = v.x;
      acc[i][j][1] = v.y;
    }
  cp_async_wait<0>();
  __syncthreads();
  tile_mma(sX, sY, acc, -1.0);
  if (kt == L.nt - 1) {
    // last step: the tile is final; inv = -A goes straight out, both orientations (the lower
    // part of a diagonal tile serves both, so inv is exactly symmetric)
    const int s = a.s;
    double* out = a.inv + (int64_t)b * s * s;
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int row = r0 + i * 8 + g, col = c0 + j * 8 + 2 * t + u;
          const int gi = I * LT + row, gj = J * LT + col;
          if (gi >= s || gj >= s || (I == J && col > row)) continue;
          const double v = -acc[i][j][u];
          out[(int64_t)gi * s + gj] = v;
          if (gi != gj) out[(int64_t)gj * s + gi] = v;
        }
    return;
  }
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
      *reinterpret_cast<double2*>(C + (int64_t)(r0 + i * 8 + g) * L.S + c0 + j * 8 + 2 * t) =
          make_double2(acc[i][j][0], acc[i][j][1]);
  if (lookahead && I == kt + 1 && J == kt + 1) {
    __syncthreads();   // the updated tile (global, written by this CTA) is the next pivot
    pivot_sweep(a, L, b, kt + 1);
  }
}

// nt == 1 (s <= 64 forced onto this path): A = -W
__global__ void large_strip1_kernel(SysArgs a, int p) {
  const LargeBufs L = large_bufs(a.scratch, a.s, p);
  const int b = blockIdx.x;
  const int dn = a.done ? *a.done : 0;
  if (dn | a.info[b]) return;
  double* A = L.A + (size_t)b * L.S * L.S;
  for (int e = threadIdx.x; e < LT * LT; e += blockDim.x) {
    const int i = e / LT, j = e - i * LT;
    if (j <= i) A[(int64_t)i * L.S + j] = -L.W[(size_t)b * LT * LT + e];
  }
}

// (e) inv = -A (symmetric, s x s): one CTA per 64 x 64 output tile, the upper tiles through a
// shared-memory transpose of the stored lower tile (coalesced on both sides)
__global__ void __launch_bounds__(LTHREADS) large_out_kernel(SysArgs a, int p) {
  const int s = a.s;
  const LargeBufs L = large_bufs(a.scratch, s, p);
  const int b = blockIdx.y;
  const int dn = a.done ? *a.done : 0;
  if (dn | a.info[b]) return;
  const int I = blockIdx.x / L.nt, J = blockIdx.x - I * L.nt;
  const int hi = max(I, J), lo = min(I, J);
  __shared__ double T[LT][LT + 1];
  const double* A = L.A + (size_t)b * L.S * L.S + (int64_t)hi * LT * L.S + lo * LT;
  for (int e = threadIdx.x; e < LT * LT; e += LTHREADS) {
    const int i = e / LT, j = e - i * LT;
    T[i][j] = A[(int64_t)i * L.S + j];
  }
  __syncthreads();
  double* out = a.inv + (int64_t)b * s * s;
  for (int e = threadIdx.x; e < LT * LT; e += LTHREADS) {
    const int i = e / LT, j = e - i * LT;
    const int gi = I * LT + i, gj = J * LT + j;
    if (gi >= s || gj >= s) continue;
    const double v = (I > J) ? T[i][j] : (I < J) ? T[j][i] : T[max(i, j)][min(i, j)];
    out[(int64_t)gi * s + gj] = -v;
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
    else large_strip1_kernel<<<p, LTHREADS, 0, st>>>(a, p);   // single tile: A = -W
  }
  // nt > 1: the last step's kernels write inv = -A themselves
  if (nt == 1) large_out_kernel<<<dim3(nt * nt, p), LTHREADS, 0, st>>>(a, p);
  note_launch(2 + (nt == 1) + nt * (nt > 1 ? 2 : 1));
  return check_launch("inverse_large");
}

}  // namespace rac
