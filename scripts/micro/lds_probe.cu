// Calibrate: the helper's T-term loop (13 rows x 8 threads, 2 tiles of 100 doubles,
// two accumulators) on 96 threads, in isolation, vs variants.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void probe(int mode, long long* out, double* sink) {
  extern __shared__ double sm[];
  const int s = 100, sl = 13, D = 3;
  double* tile = sm;                       // (1 + D) * sl * s
  double* sDelta = tile + (1 + D) * sl * s;  // 4 * s
  double* hpart = sDelta + 4 * s;          // 256
  const int tid = threadIdx.x;
  for (int i = tid; i < (1 + D) * sl * s + 4 * s; i += blockDim.x) sm[i] = 1.0 + 1e-3 * i;
  __syncthreads();
  if (tid >= 96) return;
  const int gid = tid, rows = 13, u = 7, nd = 3;
  long long c0 = clock64();
  for (int rep = 0; rep < 100; ++rep) {
    if (mode == 0) {
      for (int e = gid; e < rows * 8; e += 96) {
        const int r = e >> 3, part = e & 7;
        double a0 = 0.0, a1 = 0.0;
        for (int d = 2; d <= nd; ++d) {
          const double* Td = tile + ((size_t)d * sl + r) * s;
          const double* dv = sDelta + (size_t)((u - d) & 3) * s;
          int c = part;
          for (; c + 8 < s; c += 16) { a0 += Td[c] * dv[c]; a1 += Td[c + 8] * dv[c + 8]; }
          if (c < s) a0 += Td[c] * dv[c];
        }
        hpart[e] = a0 + a1 + rep;
      }
    } else {
      // fully unrolled fixed-trip variant
      for (int e = gid; e < rows * 8; e += 96) {
        const int r = e >> 3, part = e & 7;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
        for (int d = 2; d <= 3; ++d) {
          const double* Td = tile + (d * sl + r) * s + part;
          const double* dv = sDelta + ((u - d) & 3) * s + part;
#pragma unroll
          for (int i = 0; i < 12; i += 2) { a0 += Td[8 * i] * dv[8 * i]; a1 += Td[8 * i + 8] * dv[8 * i + 8]; }
          if (part < 4) a2 += Td[96] * dv[96];
        }
        hpart[e] = (a0 + a1) + (a2 + a3) + rep;
      }
    }
    asm volatile("bar.sync 2, 96;" ::: "memory");
  }
  long long c1 = clock64();
  if (tid == 0) { out[mode] = c1 - c0; sink[0] = hpart[5]; }
}
int main() {
  long long* out; double* sink;
  cudaMalloc(&out, 64); cudaMalloc(&sink, 64);
  int smem = ((1 + 3) * 13 * 100 + 400 + 256) * 8;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int mode = 0; mode < 2; ++mode) {
    for (int rep = 0; rep < 3; ++rep) { probe<<<1, 512, smem>>>(mode, out, sink); cudaDeviceSynchronize(); }
    long long h[4]; cudaMemcpy(h, out, 32, cudaMemcpyDeviceToHost);
    printf("mode %d: %.1f cycles per T-term pass (incl. bar)\n", mode, h[mode] / 100.0);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
