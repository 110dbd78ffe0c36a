// Microbenchmark: cost of a 13-row warp_sum loop in warp 8 while other warps
// of the CTA (a) idle at a barrier, (b) spin on ld.relaxed.gpu global loads,
// (c) spin on mbarrier.test_wait, (d) spin on mbarrier.try_wait.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ long long gt() { long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
__device__ __forceinline__ double wsum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__global__ void probe(int mode, unsigned long long* flag, long long* out, double* sink) {
  __shared__ unsigned long long bar;
  __shared__ double buf[64];
  __shared__ volatile int done;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&bar)));
    done = 0;
  }
  __syncthreads();
  if (warp == 8) {
    if (mode >= 7) {   // diverge the warp first: lanes < 13 poll global memory a few times, lane 0 waits on mbarrier
      if (lane < 13) { for (int i = 0; i < 3 + lane; ++i) { unsigned long long v; asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(flag + lane)); if (v == 777) break; } }
      if (lane == 0) { unsigned ok = 0; asm volatile("{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], 1; selp.u32 %0,1,0,p; }" : "=r"(ok) : "r"((unsigned)__cvta_generic_to_shared(&bar)) : "memory"); if (ok) sink[1] = 1; }
      if (mode == 8) __syncwarp();
    }
    long long t0 = gt(), c0 = clock64();
    double acc = lane;
    for (int it = 0; it < 100; ++it)
      for (int r = 0; r < 13; ++r) {
        double a = wsum(acc + r);
        if (lane == 0) buf[r] = a;
        acc += 1e-3 * a;
      }
    long long t1 = gt(), c1 = clock64();
    if (lane == 0) { out[0] = t1 - t0; out[1] = c1 - c0; sink[0] = acc; done = 1; }
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((unsigned)__cvta_generic_to_shared(&bar)));
  } else if (warp < 8 && mode > 0) {
    const bool me = (mode >= 4) ? (tid == 0) : true;   // modes 4-6: one thread spins
    const int m = (mode >= 4) ? mode - 3 : mode;
    if (me) {
      if (m == 1) {
        while (!done) { unsigned long long v; asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(flag + tid)); if (v == 12345) break; }
      } else if (m == 2) {
        unsigned ok = 0;
        while (!ok) asm volatile("{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p; }" : "=r"(ok) : "r"((unsigned)__cvta_generic_to_shared(&bar)) : "memory");
      } else {
        asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0; @!p bra W; }" ::"r"((unsigned)__cvta_generic_to_shared(&bar)) : "memory");
      }
    }
  }
  __syncthreads();
}
int main() {
  unsigned long long* flag; long long* out; double* sink;
  cudaMalloc(&flag, 4096); cudaMemset(flag, 0, 4096); cudaMalloc(&out, 64); cudaMalloc(&sink, 64);
  const char* names[] = {"idle", "256 thr ld.relaxed spin", "256 thr test_wait spin", "256 thr try_wait spin",
                         "1 thr ld.relaxed spin", "1 thr test_wait spin", "1 thr try_wait spin",
                         "diverged, no syncwarp", "diverged + syncwarp"};
  for (int mode = 0; mode < 9; ++mode) {
    for (int rep = 0; rep < 3; ++rep) {
      probe<<<1, 512>>>(mode, flag, out, sink);
      cudaDeviceSynchronize();
    }
    long long h[2]; cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
    printf("%-26s 1300 warp_sums: %8.2f us  %9lld cycles  (%.1f cycles / warp_sum)\n", names[mode], h[0] / 1e3, h[1], h[1] / 1300.0);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
