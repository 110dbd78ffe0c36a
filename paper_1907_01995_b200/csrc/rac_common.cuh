// Shared device helpers for the RAC-MBADMM sweep kernels (sm_100a, FP64).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#define RAC_WARP 32

namespace rac {

__host__ __device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }

__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// ---------------------------------------------------------------------------
// memory-model helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void red_release_add_u32(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Loads of data produced by OTHER CTAs inside the same launch: bypass L1.
__device__ __forceinline__ double ldcg(const double* p) { return __ldcg(p); }
__device__ __forceinline__ int ldcg(const int* p) { return __ldcg(p); }

// Grid-wide barrier for a cooperative (all-CTAs-resident) launch.  The
// counter is monotonic within a launch and must be zero at launch start;
// every CTA keeps its own running target.
__device__ __forceinline__ void grid_barrier(unsigned* counter, unsigned& target,
                                             unsigned nblocks) {
  // bar.sync orders the CTA's writes before thread 0's release (release is
  // cumulative); the acquire load that sees the final count orders everything
  // after it, and the second bar.sync extends that to the whole CTA.
  __syncthreads();
  if (threadIdx.x == 0) {
    target += nblocks;
    red_release_add_u32(counter, 1u);
    while (ld_acquire_u32(counter) < target) {
    }
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// reductions (fixed order => bitwise run-to-run determinism)
// ---------------------------------------------------------------------------
// Callers are always all 32 lanes.  The __syncwarp reconverges a warp that
// arrives diverged (measured: a diverged double warp_sum costs ~2350 cycles
// instead of ~200 — scripts/micro/shfl_probe.cu).
__device__ __forceinline__ double warp_sum(double v) {
  __syncwarp();
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// max that propagates NaN like numpy's np.max (fmax drops it): a residual that went
// non-finite must not read as converged
__device__ __forceinline__ double nanmax(double a, double b) {
  return (a != a) ? a : ((b != b) ? b : fmax(a, b));
}

__device__ __forceinline__ double warp_nanmax(double v) {
  __syncwarp();
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = nanmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ double warp_max(double v) {
  __syncwarp();
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// ---------------------------------------------------------------------------
// FP64 tensor-core tile: D(8x8) += A(8x4, row) * B(4x8, col)  -> SASS DMMA.8x8x4
//   lane = 4*g + t:  a = A[g][t], b = B[t][g], d0/d1 = D[g][2t], D[g][2t+1]
// ---------------------------------------------------------------------------
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// ---------------------------------------------------------------------------
// cp.async (LDGSTS) 16-byte copies global -> shared
// ---------------------------------------------------------------------------
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// ---------------------------------------------------------------------------
// TMA bulk copies (cp.async.bulk -> SASS UBLKCP) completing on an mbarrier
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "RAC_MBAR_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra RAC_MBAR_WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// global -> own shared memory, `bytes` multiple of 16, both addresses 16B aligned
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// order prior generic-proxy shared accesses before subsequent async-proxy (TMA) writes
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// non-suspending poll (mbarrier.test_wait): for waits that are usually already
// satisfied, where try_wait's suspend/wake latency would dominate
__device__ __forceinline__ void mbar_spin(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "RAC_MBAR_SPIN_%=:\n"
      " mbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra RAC_MBAR_SPIN_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// test_wait poll with a nanosleep back-off: keeps a waiting thread from taking
// issue / MIO slots from the warps that produce what it waits for
__device__ __forceinline__ bool mbar_test(uint64_t* bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred p;\n"
      " mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_spin_sleep(uint64_t* bar, unsigned parity, unsigned ns = 64) {
  while (!mbar_test(bar, parity)) __nanosleep(ns);
}
__device__ __forceinline__ void mbar_spin_cluster(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "RAC_MBAR_SPINC_%=:\n"
      " mbarrier.test_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra RAC_MBAR_SPINC_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// wait with cluster-scope acquire: data pushed by peer CTAs (st.async) is visible afterwards
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "RAC_MBAR_WAITC_%=:\n"
      " mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra RAC_MBAR_WAITC_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// ---------------------------------------------------------------------------
// distributed shared memory: push 16 bytes into a peer CTA's shared memory,
// completing `bytes` on the peer's mbarrier (no cluster-wide barrier needed)
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned mapa_u32(unsigned saddr, unsigned rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_async_f64(unsigned raddr, double x, unsigned rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(raddr), "d"(x),
               "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void st_async_f64x2(unsigned raddr, double x, double y, unsigned rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(raddr),
               "d"(x), "d"(y), "r"(rbar)
               : "memory");
}

// bulk copy own shared memory -> a peer CTA's shared memory (TMA engine), completing
// `bytes` on the peer's mbarrier; dst / bar are shared::cluster addresses (mapa)
__device__ __forceinline__ void bulk_s2peer(unsigned dst, const void* src, unsigned bytes, unsigned bar) {
  asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   dst),
               "r"(smem_u32(src)), "r"(bytes), "r"(bar)
               : "memory");
}

__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// named barrier for a subset of the CTA's warps (id 1..15)
__device__ __forceinline__ void named_bar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// ---------------------------------------------------------------------------
// self-validating ("low-latency") messages between CTAs of one launch: a double
// travels as two 64-bit words {32 data bits | 32-bit tag}; a reader accepts the
// value once both words carry the expected tag.  Aligned 64-bit accesses are
// single-copy atomic, so no flag / fence round trip is needed.
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void ll_store(unsigned long long* p, double v, unsigned tag) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(v);
  const unsigned long long hi = (unsigned long long)tag << 32;
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"((u & 0xffffffffull) | hi),
               "l"((u >> 32) | hi)
               : "memory");
}
// both words of a tagged pair in one 16-byte access (each 64-bit half is single-copy atomic)
__device__ __forceinline__ void ll_load2(const unsigned long long* p, unsigned long long& w0, unsigned long long& w1) {
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(p) : "memory");
}
__device__ __forceinline__ bool ll_ok(unsigned long long w, unsigned tag) { return (unsigned)(w >> 32) == tag; }
__device__ __forceinline__ double ll_value(unsigned lo, unsigned hi) {
  return __longlong_as_double((long long)(((unsigned long long)hi << 32) | lo));
}

// IEEE operations without FMA contraction (numpy evaluates a*b+c as two
// rounded ops; use these where bitwise agreement with the oracle matters).
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }

// numpy's  -sign(a) * max(|a| - b, 0) + 0.0   (elastic_net.py:112)
__device__ __forceinline__ double neg_shrink(double a, double b) {
  double mag = fmax(sub(fabs(a), b), 0.0);
  double sg = (a > 0.0) ? 1.0 : ((a < 0.0) ? -1.0 : (a == 0.0 ? 0.0 : a));
  return add(mul(-sg, mag), 0.0);
}

}  // namespace rac
