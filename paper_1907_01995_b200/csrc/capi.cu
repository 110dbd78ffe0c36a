// C ABI plumbing: error reporting, version, device checks, small kernels.
#include <stdarg.h>
#include <algorithm>
#include <atomic>
#include <stdio.h>
#include <stdlib.h>

#include "rac_internal.h"

namespace rac {

static thread_local char g_err[512] = {0};

void clear_error() { g_err[0] = 0; }

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int check_cuda(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return RAC_OK;
  return set_error(RAC_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

int check_launch(const char* what) { return check_cuda(cudaGetLastError(), what); }

// Context buffers come from each device's default stream-ordered memory pool.
// The pool keeps up to POOL_KEEP bytes of freed memory mapped (release
// threshold), so re-creating a context of a seen shape (one per fit/train/solve
// call) neither maps memory nor synchronises the device; anything above that is
// returned at the next synchronisation, and rac_trim_pool() / a context's
// destruction trims the pool back to the threshold so that PyTorch's caching
// allocator (e.g. an N x N SVM Q after a large fit) can have the memory.
const uint64_t POOL_KEEP = 8ULL << 30;
static std::atomic<uint64_t> g_pool_ready{0};   // bit per configured device

static cudaMemPool_t device_pool(int dev) {
  cudaMemPool_t pool = nullptr;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  const uint64_t bit = 1ULL << (dev & 63);
  if (!(g_pool_ready.load() & bit)) {
    uint64_t thr = POOL_KEEP;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    cudaGetLastError();
    g_pool_ready.fetch_or(bit);
  }
  return pool;
}

int dev_alloc(void** p, size_t bytes, cudaStream_t st) {
  int dev = 0;
  cudaGetDevice(&dev);
  device_pool(dev);
  return check_cuda(cudaMallocAsync(p, bytes, st), "cudaMallocAsync");
}

void dev_free(void* p, cudaStream_t st) {
  if (p) cudaFreeAsync(p, st);
}

void trim_pool(size_t keep) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (cudaMemPool_t pool = device_pool(dev)) cudaMemPoolTrimTo(pool, keep);
  cudaGetLastError();
}

// Nsight Compute cannot replay cooperative (grid-synchronised) launches, cluster ones
// least of all.  Under the profiler (ncu exports NV_NSIGHT_INJECTION_TRANSPORT_TYPE and
// NV_COMPUTE_PROFILER_PERFWORKS_DIR into the target; other injectors CUDA_INJECTION64_PATH)
// or with RAC_PROFILE_NONCOOP=1, the persistent chain kernels are launched without
// the cooperative attribute: every such grid is sized to one co-resident wave (checked
// with the occupancy API when the context is planned) and the other kernels sharing
// the GPU never wait on the chain, so all its CTAs still become resident and the
// software grid barriers hold.  RAC_PROFILE_NONCOOP=0 forces cooperative launches.
bool profile_noncoop() {
  static const int v = [] {
    if (const char* e = getenv("RAC_PROFILE_NONCOOP")) return atoi(e) == 1 ? 1 : 0;
    for (const char* k : {"NV_NSIGHT_INJECTION_TRANSPORT_TYPE", "NV_COMPUTE_PROFILER_PERFWORKS_DIR",
                          "CUDA_INJECTION64_PATH"}) {
      const char* v = getenv(k);
      if (v && *v) return 1;
    }
    return 0;
  }();
  return v == 1;
}

cudaError_t launch_coop(const void* f, dim3 grid, dim3 block, void** args, size_t smem, cudaStream_t st) {
  if (profile_noncoop()) return cudaLaunchKernel(f, grid, block, args, smem, st);
  return cudaLaunchCooperativeKernel(f, grid, block, args, smem, st);
}

static std::atomic<unsigned long long> g_launches{0};
void note_launch(int k) { g_launches.fetch_add((unsigned long long)k, std::memory_order_relaxed); }
unsigned long long launch_count() { return g_launches.load(std::memory_order_relaxed); }

int num_sms() {
  static int cached = 0;
  if (!cached) {
    int dev = 0;
    cudaGetDevice(&dev);
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0)
      v = 148;
    cached = v;
  }
  return cached;
}

// out = Q w  (rows x cols row-major): one warp per row, fixed-order reduction.
__global__ void gemv_rows_kernel(const double* __restrict__ Q, int64_t rows, int64_t cols,
                                 const double* __restrict__ w, double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < rows; i += nw) {
    const double* q = Q + i * cols;
    double acc = 0.0;
    for (int64_t j = lane; j < cols; j += 32) acc += q[j] * w[j];
    acc = warp_sum(acc);
    if (lane == 0) out[i] = acc;
  }
}

int launch_gemv_rows(const double* Q, int64_t rows, int64_t cols, const double* w, double* out,
                     cudaStream_t st) {
  int blocks = (int)std::min<int64_t>((rows + 7) / 8, (int64_t)num_sms() * 8);
  if (blocks < 1) blocks = 1;
  gemv_rows_kernel<<<blocks, 256, 0, st>>>(Q, rows, cols, w, out);
  note_launch();
  return check_launch("gemv_rows");
}

__global__ void z_prox_kernel(const double* __restrict__ beta, const double* __restrict__ xi,
                              int64_t n, double gamma, double thr, double den,
                              double* __restrict__ z) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double a = sub(xi[i], mul(gamma, beta[i]));
    z[i] = __ddiv_rn(neg_shrink(a, thr), den);
  }
}

}  // namespace rac

extern "C" int rac_trim_pool(uint64_t keep_bytes) {
  rac::clear_error();
  rac::trim_pool((size_t)keep_bytes);
  return RAC_OK;
}

extern "C" uint64_t rac_launch_count(void) { return (uint64_t)rac::launch_count(); }

extern "C" const char* rac_version(void) { return "rac_b200 0.1.0 (sm_100a, fp64)"; }

extern "C" const char* rac_last_error(void) { return rac::g_err; }

extern "C" int rac_device_check(int device) {
  using namespace rac;
  clear_error();
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count <= device || device < 0)
    return set_error(RAC_ERR_CUDA, "no CUDA device %d (%s)", device, cudaGetErrorString(e));
  cudaDeviceProp prop;
  e = cudaGetDeviceProperties(&prop, device);
  if (e != cudaSuccess) return check_cuda(e, "cudaGetDeviceProperties");
  if (prop.major != 10 || prop.minor != 0)
    return set_error(RAC_ERR_CUDA, "device %d is sm_%d%d; this library is built for sm_100a",
                     device, prop.major, prop.minor);
  return RAC_OK;
}

extern "C" int rac_z_prox(const double* beta, const double* xi, int64_t n, double gamma,
                          double thr, double den, double* z, void* stream) {
  using namespace rac;
  clear_error();
  if (!beta || !xi || !z || n < 0) return set_error(RAC_ERR_ARG, "rac_z_prox: bad arguments");
  if (n == 0) return RAC_OK;
  int blocks = (int)std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 8);
  z_prox_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(beta, xi, n, gamma, thr, den, z);
  note_launch();
  return check_launch("z_prox");
}

extern "C" int rac_gemv(const double* Q, int64_t rows, int64_t cols, const double* w, double* out,
                        void* stream) {
  using namespace rac;
  clear_error();
  if (!Q || !w || !out || rows < 0 || cols < 0) return set_error(RAC_ERR_ARG, "rac_gemv: bad arguments");
  if (rows == 0) return RAC_OK;
  return launch_gemv_rows(Q, rows, cols, w, out, (cudaStream_t)stream);
}
