// Label-weighted kernel strips  strip[i][j] = y_{r_i} y_j K(x_{r_i}, x_j)  (svm.py:121-143
// assemble_kernel_block; svm.py:82-93 kernel_cross) on the FP64 tensor cores.
//
// The reference never forms the N x N matrix Q: per block it assembles the s x N strip
// Q_{b,.} from data rows through an LRU of kernel rows (svm.py:96-118).  Here one launch
// forms the strip rows of a whole block (or of several blocks) as a rectangular DMMA
// GEMM  X_rows (s x d) . X' (d x N)  with the kernel / label epilogue fused: 64 x 64
// output tiles, K = d staged through shared memory in 32-wide chunks by 16-byte cp.async,
// mma.sync m8n8k4 f64 (SASS DMMA.8x8x4), FP64 accumulation in a fixed order.
#include "rac_internal.h"

#include <algorithm>

namespace rac {

constexpr int ST = 64;          // tile edge
constexpr int SKC = 32;         // k chunk (doubles of a sample row per stage)
constexpr int SLD = SKC + 4;    // padded smem row (conflict-free fragment loads)
constexpr int STHREADS = 256;

// squared row norms, one warp per row, fixed order (the Gaussian epilogue's |x|^2 terms)
__global__ void row_sqnorm_kernel(const double* __restrict__ Xp, int64_t ldd, int64_t N, int64_t d,
                                  double* __restrict__ sq) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < N; i += nw) {
    const double* x = Xp + i * ldd;
    double acc = 0.0;
    for (int64_t k = lane; k < d; k += 32) acc = fma(x[k], x[k], acc);
    acc = warp_sum(acc);
    if (lane == 0) sq[i] = acc;
  }
}

// out[i * ldo + j], i < s (rows[i] = sample index; -1 = padding row -> zeros), j < N; the
// output columns are samples 0..N-1, or cols[j] when given (-1 = zero column).  blockIdx.z
// batches independent problems: rows / cols / out advance by the given strides.
__global__ void __launch_bounds__(STHREADS) strip_kernel(const double* __restrict__ Xp, int64_t ldd, int64_t d,
                                                        const int32_t* __restrict__ rows, int s, int64_t N,
                                                        const double* __restrict__ y,
                                                        const double* __restrict__ sq, int kind,
                                                        double two_sigma2, double* __restrict__ out,
                                                        int64_t ldo, const int32_t* __restrict__ cols,
                                                        int64_t zstride_rc, int64_t zstride_out) {
  extern __shared__ __align__(16) double ssm[];
  rows += blockIdx.z * zstride_rc;
  if (cols) cols += blockIdx.z * zstride_rc;
  out += blockIdx.z * zstride_out;
  double* sA[2] = {ssm, ssm + ST * SLD};
  double* sB[2] = {ssm + 2 * ST * SLD, ssm + 3 * ST * SLD};
  const int I = blockIdx.y;                 // tile of strip rows
  const int64_t J = blockIdx.x;             // tile of samples
  const int tid = threadIdx.x;
  __shared__ int64_t srcA[ST], srcB[ST];
  __shared__ double yA[ST], yB[ST], qA[ST], qB[ST];
  if (tid < ST) {
    const int gi = I * ST + tid;
    const int r = gi < s ? rows[gi] : -1;
    srcA[tid] = r >= 0 ? (int64_t)r * ldd : -1;
    yA[tid] = r >= 0 ? y[r] : 0.0;
    qA[tid] = (r >= 0 && kind == RAC_KERNEL_GAUSSIAN) ? sq[r] : 0.0;
    const int64_t gj0 = J * ST + tid;
    const int64_t gj = gj0 < N ? (cols ? (int64_t)cols[gj0] : gj0) : -1;
    srcB[tid] = gj >= 0 ? gj * ldd : -1;
    yB[tid] = gj >= 0 ? y[gj] : 0.0;
    qB[tid] = (gj >= 0 && kind == RAC_KERNEL_GAUSSIAN) ? sq[gj] : 0.0;
  }
  __syncthreads();
  for (int e = tid; e < ST * SLD; e += STHREADS) {
    const int c = e / SLD;
    if (srcA[c] < 0) { sA[0][e] = 0.0; sA[1][e] = 0.0; }
    if (srcB[c] < 0) { sB[0][e] = 0.0; sB[1][e] = 0.0; }
  }
  const int nck = (int)((d + SKC - 1) / SKC);     // Xp rows are zero-padded to ldd >= nck * SKC
  auto load_stage = [&](int stage, int64_t k0) {
    for (int e = tid; e < ST * (SKC / 2); e += STHREADS) {
      const int c = e >> 4, q = e & 15;
      const int64_t a = srcA[c], b = srcB[c];
      if (a >= 0) cp_async16(sA[stage] + c * SLD + 2 * q, Xp + a + k0 + 2 * q);
      if (b >= 0) cp_async16(sB[stage] + c * SLD + 2 * q, Xp + b + k0 + 2 * q);
    }
    cp_async_commit();
  };
  const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  int ur[2], uc[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int u = warp + 8 * q;
    ur[q] = u >> 2;
    uc[q] = u & 3;
  }
  double acc[2][4][2];
#pragma unroll
  for (int q = 0; q < 2; ++q)
#pragma unroll
    for (int r = 0; r < 4; ++r) acc[q][r][0] = acc[q][r][1] = 0.0;
  if (nck > 0) load_stage(0, 0);
  for (int ck = 0; ck < nck; ++ck) {
    const int cur = ck & 1;
    if (ck + 1 < nck) {
      load_stage(cur ^ 1, (int64_t)(ck + 1) * SKC);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const double* a0p = sA[cur] + (ur[q] * 16 + g) * SLD + t;
      const double* a1p = a0p + 8 * SLD;
      const double* b0p = sB[cur] + (uc[q] * 16 + g) * SLD + t;
      const double* b1p = b0p + 8 * SLD;
#pragma unroll
      for (int kk = 0; kk < SKC; kk += 4) {
        const double a0 = a0p[kk], a1 = a1p[kk], b0 = b0p[kk], b1 = b1p[kk];
        dmma884(acc[q][0][0], acc[q][0][1], a0, b0);
        dmma884(acc[q][1][0], acc[q][1][1], a0, b1);
        dmma884(acc[q][2][0], acc[q][2][1], a1, b0);
        dmma884(acc[q][3][0], acc[q][3][1], a1, b1);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < 2; ++q)
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int lr = ur[q] * 16 + (r >> 1) * 8 + g;
      const int row = I * ST + lr;
      if (row >= s) continue;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int lc = uc[q] * 16 + (r & 1) * 8 + 2 * t + e;
        const int64_t col = J * ST + lc;
        if (col >= N) continue;
        double k = acc[q][r][e];
        if (kind == RAC_KERNEL_GAUSSIAN) {
          const double d2 = fmax(sub(add(qA[lr], qB[lc]), mul(2.0, k)), 0.0);
          k = exp(-d2 / two_sigma2);
        }
        out[(int64_t)row * ldo + col] = mul(mul(yA[lr], k), yB[lc]);
      }
    }
}

int launch_kernel_strip(const double* Xp, int64_t ldd, int64_t d, const int32_t* rows, int s, int64_t N,
                        const double* y, const double* sq, int kind, double sigma, double* out, int64_t ldo,
                        cudaStream_t st, const int32_t* cols, int batch) {
  if (s <= 0 || N <= 0 || batch <= 0) return RAC_OK;
  const size_t smem = 4 * ST * SLD * sizeof(double);
  int rc = check_cuda(cudaFuncSetAttribute(strip_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                      "strip smem attribute");
  if (rc) return rc;
  dim3 grid((unsigned)((N + ST - 1) / ST), (unsigned)((s + ST - 1) / ST), (unsigned)batch);
  strip_kernel<<<grid, STHREADS, smem, st>>>(Xp, ldd, d, rows, s, N, y, sq, kind, 2.0 * sigma * sigma, out, ldo,
                                             cols, (int64_t)s, (int64_t)s * ldo);
  note_launch();
  return check_launch("kernel strip");
}

int launch_row_sqnorm(const double* Xp, int64_t ldd, int64_t N, int64_t d, double* sq, cudaStream_t st) {
  const int blocks = (int)std::min<int64_t>((N + 7) / 8, (int64_t)num_sms() * 8);
  row_sqnorm_kernel<<<std::max(1, blocks), 256, 0, st>>>(Xp, ldd, N, d, sq);
  note_launch();
  return check_launch("row sqnorm");
}

}  // namespace rac

// One call: pad X (N x d row-major) to 32-double rows, |x|^2 for the Gaussian kernel, then
// the strip rows.  Replaces svm.py:121-143 assemble_kernel_block(..., with_strip=True).
extern "C" int rac_svm_kernel_strip(const double* X, int64_t N, int64_t d, const double* labels, const int32_t* rows,
                                    int32_t s, int32_t kind, double sigma, double* strip, void* stream) {
  using namespace rac;
  clear_error();
  if (!X || !labels || !rows || !strip || N < 1 || d < 1 || s < 1)
    return set_error(RAC_ERR_ARG, "rac_svm_kernel_strip: bad arguments");
  if (kind == RAC_KERNEL_GAUSSIAN && !(sigma > 0)) return set_error(RAC_ERR_ARG, "sigma must be > 0");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t ldd = (d + 31) / 32 * 32;
  double *Xp = nullptr, *sq = nullptr;
  int rc = check_cuda(cudaMallocAsync((void**)&Xp, (size_t)N * ldd * sizeof(double), st), "malloc Xp");
  if (rc) return rc;
  rc = check_cuda(cudaMallocAsync((void**)&sq, (size_t)N * sizeof(double), st), "malloc sq");
  if (rc) {
    cudaFreeAsync(Xp, st);
    return rc;
  }
  cudaMemsetAsync(Xp, 0, (size_t)N * ldd * sizeof(double), st);
  cudaMemcpy2DAsync(Xp, ldd * sizeof(double), X, d * sizeof(double), d * sizeof(double), N,
                    cudaMemcpyDeviceToDevice, st);
  if (kind == RAC_KERNEL_GAUSSIAN) rc = launch_row_sqnorm(Xp, ldd, N, d, sq, st);
  if (!rc) rc = launch_kernel_strip(Xp, ldd, d, rows, s, N, labels, sq, kind, sigma, strip, N, st, nullptr, 1);
  cudaFreeAsync(Xp, st);
  cudaFreeAsync(sq, st);
  return rc;
}
