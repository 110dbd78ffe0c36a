// Which reconvergence restores fast shuffles after single-thread waits?
// warp 0 (of 8 "main" warps): thread 0 polls an mbarrier (already complete),
// then bar.sync 1,256; then a 13-row warp_sum loop.  Variants:
//   0: nothing     1: __syncwarp()     2: __syncthreads-style bar.sync 1 twice
//   3: all threads poll (no single-thread branch)   4: __syncwarp + predicated store in loop
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double wsum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ bool test(unsigned bar) {
  unsigned ok;
  asm volatile("{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p; }" : "=r"(ok) : "r"(bar) : "memory");
  return ok;
}
__global__ void probe(int mode, long long* out, double* sink, int* idx) {
  __shared__ unsigned long long bar;
  __shared__ double buf[64];
  const int tid = threadIdx.x, lane = tid & 31;
  const unsigned ba = (unsigned)__cvta_generic_to_shared(&bar);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(ba));
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(ba));   // phase 0 complete
  }
  __syncthreads();
  if (tid >= 256) return;
  double acc = lane;
  long long c0 = clock64();
  for (int it = 0; it < 100; ++it) {
    if (mode == 3) { while (!test(ba)) {} }
    else if (tid == 0) { while (!test(ba)) {} if (idx[it & 7] == -5) sink[3] = 1; }
    asm volatile("bar.sync 1, 256;" ::: "memory");
    if (mode == 2) asm volatile("bar.sync 1, 256;" ::: "memory");
    if (mode == 1 || mode == 4) __syncwarp();
    for (int r = 0; r < 13; ++r) {
      double a = wsum(acc + r);
      if (mode == 4) { if (lane == 0) buf[r] = a; }
      acc += 1e-3 * a;
    }
  }
  long long c1 = clock64();
  if (tid == 0) { out[mode] = c1 - c0; sink[0] = acc; sink[1] = buf[3]; }
}
int main() {
  long long* out; double* sink; int* idx;
  cudaMalloc(&out, 64); cudaMalloc(&sink, 64); cudaMalloc(&idx, 64); cudaMemset(idx, 0, 64);
  const char* names[] = {"thread0 spin, no resync", "+ __syncwarp", "bar.sync twice", "all threads spin", "+ __syncwarp, lane0 store"};
  for (int mode = 0; mode < 5; ++mode) {
    for (int rep = 0; rep < 3; ++rep) { probe<<<1, 512>>>(mode, out, sink, idx); cudaDeviceSynchronize(); }
    long long h[8]; cudaMemcpy(h, out, 64, cudaMemcpyDeviceToHost);
    printf("%-28s %9lld cycles / 1300 warp_sums = %.1f\n", names[mode], h[mode], h[mode] / 1300.0);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
