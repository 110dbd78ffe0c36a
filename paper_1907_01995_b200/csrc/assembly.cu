// K1 — random without-replacement block assembly.
//
// Replaces problems.py:234-243 (chunk_indices) applied to the host PCG64
// permutation (elastic_net.py:195, svm.py:231, engine.py:318-319): the
// permutation is cut into consecutive chunks of s and each chunk is sorted.
// One CTA per chunk; a rank sort (values are distinct) gives the sorted
// position of every element with s^2 comparisons in shared memory, which is
// exact and branch-free.  Output int32 rows of length s, -1 padded.
#include "rac_internal.h"

namespace rac {

template <int NT>
__global__ void __launch_bounds__(NT) chunk_sort_kernel(const int64_t* __restrict__ perms,
                                                        int64_t n, int s, int p,
                                                        int32_t* __restrict__ out) {
  extern __shared__ int32_t vals[];
  const int b = blockIdx.x;          // chunk within a permutation
  const int q = blockIdx.y;          // which permutation
  const int64_t base = (int64_t)b * s;
  const int len = (int)rac::min64(s, n - base);
  const int64_t* src = perms + (int64_t)q * n + base;
  int32_t* dst = out + ((int64_t)q * p + b) * s;
  for (int i = threadIdx.x; i < len; i += NT) vals[i] = (int32_t)src[i];
  __syncthreads();
  for (int i = threadIdx.x; i < len; i += NT) {
    const int32_t v = vals[i];
    int rank = 0;
    for (int k = 0; k < len; ++k) rank += (vals[k] < v);
    dst[rank] = v;
  }
  for (int i = len + threadIdx.x; i < s; i += NT) dst[i] = -1;
}

int launch_chunk_sort(const int64_t* perms, int64_t n, int s, int count, int32_t* out,
                      cudaStream_t st) {
  const int p = (int)((n + s - 1) / s);
  dim3 grid(p, count);
  chunk_sort_kernel<256><<<grid, 256, s * sizeof(int32_t), st>>>(perms, n, s, p, out);
  note_launch();
  return check_launch("chunk_sort");
}

// RP / CYCLIC block visit order: perms of p -> int32 order arrays.
__global__ void order_cast_kernel(const int64_t* __restrict__ src, int64_t total,
                                  int32_t* __restrict__ dst) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = (int32_t)src[i];
}

int launch_order_cast(const int64_t* src, int64_t total, int32_t* dst, cudaStream_t st) {
  if (total <= 0) return RAC_OK;
  int blocks = (int)rac::min64((total + 255) / 256, 1184);
  order_cast_kernel<<<blocks, 256, 0, st>>>(src, total, dst);
  note_launch();
  return check_launch("order_cast");
}

}  // namespace rac

extern "C" int rac_chunk_sort(const int64_t* perms, int64_t n, int32_t s, int32_t count,
                              int32_t* idx_out, void* stream) {
  using namespace rac;
  clear_error();
  if (!perms || !idx_out || n < 1 || s < 1 || count < 0) return set_error(RAC_ERR_ARG, "rac_chunk_sort: bad arguments");
  if (s > 12000) return set_error(RAC_ERR_UNSUPPORTED, "rac_chunk_sort: block_size > 12000");
  if (count == 0) return RAC_OK;
  return launch_chunk_sort(perms, n, s, count, idx_out, (cudaStream_t)stream);
}
