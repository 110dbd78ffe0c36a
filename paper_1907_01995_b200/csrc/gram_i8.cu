// Covariance Gram G = X'X (features x features) on the 5th-generation tensor cores in
// exact integer arithmetic (tcgen05.mma kind::i8, int32 accumulators in TMEM).
//
// Replaces, for the covariance mode, the FP64 DMMA Gram of csrc/gram.cu: the same
// quantity the reference forms per block as X[:, b].T @ X[:, b] (elastic_net.py:199-224,
// the G = X'X/m restatement in DESIGN.md §4).
//
// Digit slicing (Ozaki scheme): every feature column j gets the power-of-two scale
// 2^{e_j} > max_i |x_ij|, and x·2^{6-e_j} is split into S balanced digits
//     x·2^{6-e_j} = d_1 + d_2 2^-7 + ... + d_S 2^{-7(S-1)} + rest,  d_s in [-64, 64], |rest| <= 2^{-7(S-1)-1}
// (N = rint(x·2^{6+7(S-1)-e_j}) once, then N's balanced base-128 digits in integer arithmetic).  Then
//     G_jk = 2^{e_j+e_k-12} Σ_{w=2..S+1} 2^{-7(w-2)} C_w[j,k],
//     C_w = Σ_{s+t=w} D_s' D_t      (int8 GEMMs, exact int32 sums)
// The dropped products (s+t > S+1) and the rest terms are below 2^-52.8 of
// max|x_j|·max|x_k| per sample for S = 8 — the rounding level of an FP64 dot product — and
// below 2^-45.8 for S = 7.  S is chosen per data set on the device (i8_colexp_kernel): S = 7
// (28 slice products instead of 36) when every column's max/rms ratio r is at most
// I8_NARROW_RATIO, so that the S = 7 error relative to |x_j| |x_k| (≈ 2^-48 r_j r_k / sqrt(m)
// typical) stays at the FP64 DMMA tiles' measured level (Gaussian columns, m = 5000,
// tests/test_digit_slices.py: S = 7 max 4.5e-15, median 2.9e-16; S = 8 3.2e-16 / 2.5e-18;
// numpy FP64 3.9e-16 / 6.3e-18; DMMA tiles 2e-15 .. 2e-14); else S = 8.
// Each group's int32 sum is exact while K·S·64² < 2^31 (K segments of 65472 samples,
// combined in FP64).  The FP64 combination runs in a fixed order, so the
// result is deterministic and G is exactly symmetric (each unordered pair is formed once
// and mirrored).
//
// Tiles are 128 x 128 (M = N = 128 MMAs: 16 operand bytes per 1024 MACs, under the shared-memory
// read rate that capped 128 x 64 tiles); the S weight groups need up to 1024 TMEM columns, so
// each tile makes two passes over K with up to 4 groups (512 columns) each — the small weights
// w = S-2..S+1 (S = 8: 26 slice products, S = 7: 22; all S slices) first, then w = 2..S-3
// (S = 8: 10 products from slices 1-4, S = 7: 6 from slices 1-3).  Each pass's FP64 partial is
// added to the tile's upper-triangle entries of G, the last one also writes the mirror.
//
// Data layout: slice s is stored in the UMMA "no swizzle, K-major" canonical layout so
// that one pipeline stage of a tile is ONE contiguous 4 KB block fetched by one TMA bulk copy:
//   byte ((kst * ngrp + g) * 2 + c) * 128 + r * 16 + b
//   kst = sample / 32, g = feature / 8, c = (sample % 32) / 16, r = feature % 8, b = sample % 16
// i.e. 8 x 16 B core matrices, LBO (K direction) = 128 B, SBO (8-feature groups) = 256 B.
#include "rac_common.cuh"
#include "rac_internal.h"

namespace rac {
namespace {

constexpr int I8_S = 8;                       // digit slices
constexpr int I8_TM = 128;                    // features per A tile (TMEM lanes)
constexpr int I8_TN = 128;                    // features per B tile (TMEM columns per group)
constexpr int I8_KS = 32;                     // samples per stage (bytes per row) = one MMA K step
constexpr int I8_NST = 3;                     // pipeline stages
constexpr int I8_OP = I8_TM * I8_KS;          // 4 KB per slice operand per stage
constexpr int I8_STAGE = 2 * I8_S * I8_OP;    // 64 KB: 8 A + 8 B slice operands
constexpr int I8_SEGST = 2046;                // stages per exact int32 segment (65472 samples)
constexpr int I8_SMEM = I8_NST * I8_STAGE + 1024;
constexpr int I8_EPI = 8;                     // epilogue warps: warp w drains TMEM lanes 32 (w % 4).., column half w / 4
constexpr int I8_THREADS = (I8_EPI + 2) * 32;  // warps 0-7 epilogue, 8 TMA producer, 9 MMA issuer
static_assert(I8_S * 64 * 64 * (I8_SEGST * (double)I8_KS) < 2147483648.0, "int32 group sums must stay exact");
static_assert(4 * I8_TN <= 512, "a pass's weight groups must fit the 512 TMEM columns");
static_assert(I8_S == 8, "storage for up to 8 slices; the two passes split the groups w = 2..S+1");
// pass 0: groups w = S-2 .. S+1 (all S slices), pass 1: groups w = 2 .. S-3 (slices 1 .. S-4)

struct I8Args {
  const uint8_t* sl;     // S slices
  size_t slice_bytes;
  int ngrp;              // 8-feature groups (padded to a multiple of 16)
  int nstg;              // 32-sample stages
  int n;
  int JT;                // 128-feature tiles per side
  const int* ex;         // per-feature exponents
  double* G;             // n x n row-major
  double div;            // > 0: G = sum / div ; accumulate: G += sum
  int accum;
  size_t blk_sl;         // block mode (blockIdx.y = block): slice, output and exponent strides
  int64_t blk_g;
  int blk_ex;
  const int* flags;      // i8_colexp_kernel's flags: bit 1 = some column's max/rms > I8_NARROW_RATIO
  int force8;            // RAC_I8_SLICES=8: always 8 slices
  int lower_only;        // block mode: only the lower triangle (incl. the diagonal) is consumed
};

// slices of this data set: 8 when a column is wide (or forced), else 7
__device__ __forceinline__ int slice_count(const int* flags, int force8) {
  return (force8 || (*flags & 2)) ? 8 : 7;
}

// ---- tcgen05 helpers ------------------------------------------------------------------
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_mma_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
// K-major, no swizzle: LBO = 128 B between the two 16-byte K chunks, SBO = 256 B between 8-row groups
__device__ __forceinline__ uint64_t umma_desc(unsigned saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) |
         (1ull << 46);
}
// kind::i8, D = s32 (bits 4-5 = 2), A / B signed int8 (bits 7-9, 10-12 = 1), both K-major,
// N >> 3 at bits 17-22, M >> 4 at bits 24-28
constexpr uint32_t I8_IDESC = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(I8_TN >> 3) << 17) |
                              ((uint32_t)(I8_TM >> 4) << 24);

// 16 TMEM lanes x 32 columns: thread t receives, for i = 0..3, v[4i + 0..1] = lane t / 4, columns
// 8i + 2 (t % 4) + {0, 1} and v[4i + 2..3] = lane t / 4 + 8, the same columns (the accumulator
// fragment layout of mma: rows over lane / 4, column pairs over lane % 4).  With it both the
// direct stores G[j][k..k+1] (4 lanes = 64 contiguous bytes per row) and the mirror stores
// G[k][j] (8 lanes = 64 contiguous bytes per row) fill whole sectors; the 32x32b shape
// (thread = row) made every direct store touch 32 sectors.
__device__ __forceinline__ void tmem_ld_16x256b_x4(uint32_t taddr, int* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.16x256b.x4.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// v 2^(ea + eb): two exact multiplications by powers of two while both are far inside the
// double range (any realistic column scale), ldexp otherwise
__device__ __forceinline__ double scale_pow2(double v, int ea, int eb) {
  if (abs(ea) <= 400 && abs(eb) <= 400)
    return v * __longlong_as_double((long long)(ea + 1023) << 52) * __longlong_as_double((long long)(eb + 1023) << 52);
  return ldexp(v, ea + eb);
}

// ---- per-feature exponent: 2^e > max |x_j| ---------------------------------------------
// The dropped digit products bound a Gram entry's error by 2^-52.8 max|x_j| max|x_k| per
// sample, i.e. by 2^-52.8 r_j r_k relative to |x_j| |x_k| where r = max / rms of a column.
// A column with r > I8_MAX_RATIO (heavy outliers: r_j r_k > 2^16 leaves > 2^-37 of relative
// error) raises *bad, and the caller forms that Gram on the FP64 DMMA tiles instead.
constexpr double I8_MAX_RATIO = 256.0;
// 7 slices while every column's r <= I8_NARROW_RATIO (flags bit 1 raised otherwise: 8 slices)
constexpr double I8_NARROW_RATIO = 8.0;

// flags: bit 0 = r > I8_MAX_RATIO somewhere (also raised in *bad when given), bit 1 = r >
// I8_NARROW_RATIO somewhere
__global__ void i8_colexp_kernel(const double* __restrict__ Xc, int64_t ld, int64_t len, int n, int nfeat,
                                 int* __restrict__ ex, int* __restrict__ flags, int* __restrict__ bad) {
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; j < nfeat; j += warps) {
    double mx = 0.0, ss = 0.0;
    if (j < n) {
      const double* col = Xc + (int64_t)j * ld;
      for (int64_t k = lane; k < len; k += 32) {
        const double v = __ldg(col + k);
        mx = fmax(mx, fabs(v));
        ss = fma(v, v, ss);
      }
    }
    mx = warp_max(mx);
    ss = warp_sum(ss);
    if (lane == 0) {
      int e = 0;
      if (mx > 0.0) frexp(mx, &e);
      ex[j] = e;
      const double rms = sqrt(ss / (double)len);
      if (mx > 0.0 && mx > I8_NARROW_RATIO * rms) atomicOr(flags, 2);
      if (mx > 0.0 && mx > I8_MAX_RATIO * rms) {
        atomicOr(flags, 1);
        if (bad) atomicOr(bad, 1);
      }
    }
  }
}

// The S balanced base-128 digits of 8 values, packed[s] byte i = digit s of x[i] (int8).
// x 2^(7S-1-e) (exact, |.| <= 2^(7S-1)) is rounded once to an integer N; adding the bias
// 64 (1 + 128 + ... + 128^(S-2)) turns the balanced digits d in [-64, 63] of the S-1 lower
// positions into the plain 7-bit fields u = d + 64 of N + bias, and leaves the signed top
// digit (|d_1| <= 64) in the bits above.  Each field is moved straight to its byte by one
// (funnel) shift and one masked OR; u - 64 as an int8 is u ^ 0x40 sign-extended from bit 6,
// done on four bytes at a time.  (The slicing pass was instruction-bound, not memory-bound,
// with the digit recurrence in 64-bit arithmetic: ~140 instructions per value.)
template <int S>
__device__ __forceinline__ void slice_digits(const double (&x)[8], int e, unsigned long long (&packed)[I8_S]) {
  long long bias = 0;
#pragma unroll
  for (int k = 0; k < S - 1; ++k) bias |= 64ll << (7 * k);
  const int sc = 7 * S - 1 - e;
  const bool fast = sc >= -1022 && sc <= 1023;   // 2^sc is a normal double: one exact multiplication
  const double scale = fast ? __longlong_as_double((long long)(sc + 1023) << 52) : 1.0;
  double xs[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) xs[i] = x[i];
  if (!fast) {   // columns with a maximum near the ends of the double range
#pragma unroll 1
    for (int i = 0; i < 8; ++i) xs[i] = ldexp(xs[i], sc);
  }
  uint32_t w[I8_S][2];
#pragma unroll
  for (int s = 0; s < I8_S; ++s) w[s][0] = w[s][1] = 0u;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const long long N = __double2ll_rn(xs[i] * scale) + bias;
    const uint32_t nlo = (uint32_t)(unsigned long long)N, nhi = (uint32_t)((unsigned long long)N >> 32);
    const int half = i >> 2, sh8 = 8 * (i & 3);
#pragma unroll
    for (int k = 0; k < S - 1; ++k) {   // field k from the bottom = slice index S - 1 - k
      const int r = 7 * k - sh8;        // bit 7k of N lands on bit sh8 of the word
      const uint32_t v = r >= 32 ? nhi >> (r - 32) : (r >= 0 ? __funnelshift_r(nlo, nhi, r) : nlo << (-r));
      w[S - 1 - k][half] |= v & (0x7fu << sh8);
    }
    const int r = 7 * (S - 1) - sh8;    // top digit: 8 bits from bit 7(S-1)
    const uint32_t v = r >= 32 ? nhi >> (r - 32) : __funnelshift_r(nlo, nhi, r);
    w[0][half] |= v & (0xffu << sh8);
  }
#pragma unroll
  for (int s = 0; s < I8_S; ++s) {
    if (s >= 1 && s < S) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t t = w[s][h] ^ 0x40404040u;
        w[s][h] = t | ((t & 0x40404040u) << 1);
      }
    }
    packed[s] = (unsigned long long)w[s][0] | ((unsigned long long)w[s][1] << 32);
  }
}

// ---- digit slices in the canonical UMMA layout -----------------------------------------
// CTA = one 8-feature group x 8 stages (256 samples); thread = (feature f, 4 pairs of samples).
// Covariance: features 0..n-1 of Xc.  Block mode (idx != null): blockIdx.z = block b, whose
// features are idx[b*n ..] (n = s, -1 = padding), exponents ex[feature], and the block's
// per-position exponents are written to ex_blk[b * nfeat + position].
__global__ void __launch_bounds__(256) i8_slice_kernel(const double* __restrict__ Xc, int64_t ld, int64_t len,
                                                       int n, const int* __restrict__ ex, uint8_t* __restrict__ sl,
                                                       size_t slice_bytes, int ngrp, int nstg,
                                                       const int32_t* __restrict__ idx, int* __restrict__ ex_blk,
                                                       const int* __restrict__ flags, int force8) {
  __shared__ __align__(16) uint8_t buf[I8_S][8 * 256];
  const int S = slice_count(flags, force8);
  const int f = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = blockIdx.x;
  const int pos = g * 8 + f;
  int j = pos < n ? pos : -1;
  if (idx) {
    j = pos < n ? __ldg(idx + (size_t)blockIdx.z * n + pos) : -1;
    sl += (size_t)blockIdx.z * I8_S * slice_bytes;
  }
  // load i of a lane: the pair of samples 64 i + 2 lane, + 1 of the CTA's 256 (a warp's load is
  // 512 contiguous bytes of its feature column)
  const int64_t kc = (int64_t)blockIdx.y * 256;
  double x[8];
  if (j >= 0) {
    const double* col = Xc + (int64_t)j * ld + kc;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int k = 64 * i + 2 * lane;
      if (kc + k + 2 <= len) {
        const double2 t = __ldg(reinterpret_cast<const double2*>(col + k));
        x[2 * i] = t.x;
        x[2 * i + 1] = t.y;
      } else {
        x[2 * i] = (kc + k < len) ? col[k] : 0.0;
        x[2 * i + 1] = 0.0;
      }
    }
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = 0.0;
  }
  const int e = (j >= 0) ? __ldg(ex + j) : 0;
  if (idx && blockIdx.y == 0 && lane == 0) ex_blk[(size_t)blockIdx.z * ngrp * 8 + pos] = e;
  unsigned long long packed[I8_S];
  if (S == 8) slice_digits<8>(x, e, packed);
  else slice_digits<7>(x, e, packed);
  // pair i -> stage 2 i + lane / 16, K chunk (lane / 8) % 2, bytes 2 (lane % 8), + 1 of feature f's
  // 16-byte row: logical 16-byte chunk C = stage * 16 + chunk * 8 + f, stored at C ^ ((C >> 3) & 7)
  // (the 8 rows of a core matrix spread over the 8 bank groups: conflict-free stores and loads)
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int C = (2 * i + (lane >> 4)) * 16 + ((lane >> 3) & 1) * 8 + f;
    const int off = (C ^ ((C >> 3) & 7)) * 16 + 2 * (lane & 7);
#pragma unroll
    for (int s = 0; s < I8_S; ++s)
      if (s < S) *reinterpret_cast<uint16_t*>(&buf[s][off]) = (uint16_t)(packed[s] >> (16 * i));
  }
  __syncthreads();
  // 8 slices x 8 stages x 256 B, 16 B per thread per pass
  const int kst0 = blockIdx.y * 8;
  for (int q = threadIdx.x; q < I8_S * 8 * 16; q += 256) {
    const int s = q >> 7, kl = (q >> 4) & 7, o = q & 15;
    if (kst0 + kl >= nstg || s >= S) continue;
    const int C = kl * 16 + o;
    const uint4 v = *reinterpret_cast<const uint4*>(&buf[s][(C ^ ((C >> 3) & 7)) * 16]);
    *reinterpret_cast<uint4*>(sl + s * slice_bytes + ((size_t)(kst0 + kl) * ngrp + g) * 256 + o * 16) = v;
  }
}

// ---- the tensor-core Gram ----------------------------------------------------------------
// one pipeline stage's MMAs.  Pass 0: groups w = S-2 .. S+1 (TMEM group w - S + 2) from the
// stage's S slice operands; pass 1: groups w = 2 .. S-3 from nk packed K steps of S-4 slices.
template <int S>
__device__ __forceinline__ void issue_stage(uint32_t tmem, unsigned sA, unsigned sB, bool p0, int nk, bool first) {
  if (p0) {
#pragma unroll
    for (int w = S - 2; w <= S + 1; ++w)
#pragma unroll
      for (int s = 1; s < w; ++s)
        tc_mma_i8(tmem + (uint32_t)((w - S + 2) * I8_TN), umma_desc(sA + (s - 1) * I8_OP),
                  umma_desc(sB + (w - s - 1) * I8_OP), I8_IDESC, (first && s == 1) ? 0u : 1u);
  } else {
#pragma unroll 1
    for (int h = 0; h < nk; ++h)
#pragma unroll
      for (int w = 2; w <= S - 3; ++w)
#pragma unroll
        for (int s = 1; s < w; ++s)
          tc_mma_i8(tmem + (uint32_t)((w - 2) * I8_TN), umma_desc(sA + (h * 4 + s - 1) * I8_OP),
                    umma_desc(sB + (h * 4 + w - s - 1) * I8_OP), I8_IDESC, (first && h == 0 && s == 1) ? 0u : 1u);
  }
}

// phases: pass 0 (groups w = S-2 .. S+1) then pass 1 (w = 2 .. S-3), each over the K segments
__global__ void __launch_bounds__(I8_THREADS, 1) gram_i8_kernel(I8Args a) {
  a.sl += blockIdx.y * a.blk_sl;
  a.G += blockIdx.y * a.blk_g;
  a.ex += blockIdx.y * a.blk_ex;
  const int S = slice_count(a.flags, a.force8);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t bar_full[I8_NST], bar_free[I8_NST], bar_acc, bar_tfree;
  __shared__ uint32_t tmem_slot;
  __shared__ int ek_s[I8_TN];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // tile (J, Kt), Kt >= J: row features 128J.., column features 128Kt..
  int t = blockIdx.x, J = 0;
  while (t >= a.JT - J) {
    t -= a.JT - J;
    ++J;
  }
  const int Kt = J + t;

  if (threadIdx.x == 0) {
    for (int i = 0; i < I8_NST; ++i) {
      mbar_init(&bar_full[i], 1);
      mbar_init(&bar_free[i], 1);
    }
    mbar_init(&bar_acc, 1);
    mbar_init(&bar_tfree, I8_EPI * 32);
    mbar_fence_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  const int nseg = (a.nstg + I8_SEGST - 1) / I8_SEGST;
  const int nphase = 2 * nseg;

  if (warp == I8_EPI) {
    if (lane == 0) {
      // TMA producer: one 4 KB bulk copy per slice operand per stage
      const size_t offA = (size_t)J * 16 * 256, offB = (size_t)Kt * 16 * 256;
      const bool diag = J == Kt;   // diagonal tile: B is the A operand, loaded once
      int q = 0;
      for (int ph = 0; ph < nphase; ++ph) {
        const int ns = (ph < nseg) ? S : S - 4;   // pass 0 reads all slices, pass 1 slices 1 .. S-4
        const int sg = ph % nseg;
        const int q1 = min(a.nstg, (sg + 1) * I8_SEGST);
        // pass 1 packs two 32-sample steps (4 slices each) into one slot
        const int kpack = (ph < nseg) ? 1 : 2;
        for (int kst = sg * I8_SEGST; kst < q1; kst += kpack, ++q) {
          const int slot = q % I8_NST;
          const int nk = min(kpack, q1 - kst);
          if (q >= I8_NST) mbar_wait(&bar_free[slot], ((q / I8_NST) - 1) & 1);
          mbar_arrive_expect_tx(&bar_full[slot], (unsigned)((diag ? 1 : 2) * ns * nk * I8_OP));
          uint8_t* sA = smem + slot * I8_STAGE;
          uint8_t* sB = sA + I8_S * I8_OP;
#pragma unroll 1
          for (int h = 0; h < nk; ++h) {
            const size_t row = (size_t)(kst + h) * a.ngrp * 256;
#pragma unroll 1
            for (int s = 0; s < ns; ++s) {
              const uint8_t* src = a.sl + s * a.slice_bytes + row;
              bulk_g2s(sA + (h * 4 + s) * I8_OP, src + offA, I8_OP, &bar_full[slot]);
              if (!diag) bulk_g2s(sB + (h * 4 + s) * I8_OP, src + offB, I8_OP, &bar_full[slot]);
            }
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == I8_EPI + 1) {
    if (lane == 0) {
      // MMA issuer: per stage the phase's slice products into their weight groups
      int q = 0;
      for (int ph = 0; ph < nphase; ++ph) {
        const bool p0 = ph < nseg;
        const int sg = ph % nseg;
        const int q1 = min(a.nstg, (sg + 1) * I8_SEGST);
        if (ph > 0) mbar_wait(&bar_tfree, (ph - 1) & 1);   // previous phase drained from TMEM
        tc_fence_after();
        const int kpack = p0 ? 1 : 2;
        for (int kst = sg * I8_SEGST; kst < q1; kst += kpack, ++q) {
          const int slot = q % I8_NST;
          const int nk = min(kpack, q1 - kst);
          const bool first = kst == sg * I8_SEGST;
          mbar_wait(&bar_full[slot], (q / I8_NST) & 1);
          tc_fence_after();
          const unsigned sA = smem_u32(smem + slot * I8_STAGE);
          const unsigned sB = (J == Kt) ? sA : sA + I8_S * I8_OP;
          if (S == 8) issue_stage<8>(tmem, sA, sB, p0, nk, first);
          else issue_stage<7>(tmem, sA, sB, p0, nk, first);
          tc_commit(&bar_free[slot]);
        }
        tc_commit(&bar_acc);
      }
    }
    __syncwarp();
  } else {
    // epilogue: warp w drains TMEM lanes 32 (w % 4).. (row features 128J + 32 (w % 4) ..) and the
    // column half w / 4 (two 32-column chunks) of every group.  Per phase the FP64 partial
    // sum_g 2^{-7(w-2)} C_w · 2^{e_j + e_k - 12} of both chunks is formed in registers, TMEM is
    // handed back to the MMA issuer, and only then the partial goes to G[j][k] (k >= j) and its
    // mirror — the global-memory part of the epilogue runs under the next phase's MMAs.
    const int wq = warp & 3, half = warp >> 2;
    const int tr = lane >> 2, tc = (lane & 3) * 2;
    const uint32_t trow = tmem + ((uint32_t)(wq * 32) << 16);
    const int jb = J * I8_TM + wq * 32 + tr;   // this thread's rows: jb + 8 rr + 16 h
    int ejr[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) ejr[r] = (jb + 8 * r < a.n) ? __ldg(a.ex + jb + 8 * r) - 12 : 0;
    // the column features' exponents, once per tile
    {
      const int t = threadIdx.x;
      if (t < I8_TN) ek_s[t] = (Kt * I8_TN + t < a.n) ? __ldg(a.ex + Kt * I8_TN + t) : 0;
      asm volatile("bar.sync 1, %0;" ::"n"(I8_EPI * 32) : "memory");
    }
    const bool vec_ok = Kt > J && (a.n & 1) == 0 && (reinterpret_cast<uintptr_t>(a.G) & 15) == 0;
    // mode 0: G = sum / div (read-modify-write, the division follows the last phase's sum);
    // raw sums: 1 = first phase stores, 2 = later phases (and accumulation) add with
    // fire-and-forget reductions — same thread, same address: ordered, the same sum as a
    // read-modify-write but no load latency; the mirror gets the same terms
    for (int ph = 0; ph < nphase; ++ph) {
      const int w0 = (ph < nseg) ? S - 2 : 2;   // groups w0 .. w0 + ng - 1 in TMEM columns 0..511
      const int ng = (ph < nseg) ? 4 : S - 4;
      const bool last = ph == nphase - 1;
      const int mode = (a.div > 0.0 && !a.accum) ? 0 : ((ph == 0 && !a.accum) ? 1 : 2);
      mbar_wait(&bar_acc, ph & 1);
      tc_fence_after();
      double acc[2][32];
#pragma unroll
      for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int c = 0; c < 32; ++c) acc[q][c] = 0.0;
#pragma unroll 1
      for (int g = ng - 1; g >= 0; --g) {   // smallest weight first, fixed order
        const double wgt = ldexp(1.0, -7 * (w0 + g - 2));
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          int v[32];
          const uint32_t col = (uint32_t)(g * I8_TN + (half * 2 + q) * 32);
          tmem_ld_16x256b_x4(trow + col, v);
          tmem_ld_16x256b_x4(trow + (16u << 16) + col, v + 16);
          tmem_ld_wait();
#pragma unroll
          for (int c = 0; c < 32; ++c) acc[q][c] = fma((double)v[c], wgt, acc[q][c]);
        }
      }
      tc_fence_before();
      mbar_arrive(&bar_tfree);   // TMEM drained: the next phase's MMAs may overwrite it
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int kl0 = (half * 2 + q) * 32 + tc;   // tile-local column of i = 0, u = 0
#pragma unroll
        for (int r = 0; r < 4; ++r) {               // r = 2 h + rr
          const int j = jb + 8 * r;
          if (j >= a.n) continue;
          double* Grow = a.G + (int64_t)j * a.n;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int kl = kl0 + 8 * i, k = Kt * I8_TN + kl;
            const int e = (r >> 1) * 16 + 4 * i + 2 * (r & 1);
            const double v0 = scale_pow2(acc[q][e], ejr[r], ek_s[kl]);
            const double v1 = scale_pow2(acc[q][e + 1], ejr[r], ek_s[kl + 1]);
            if (mode == 1 && vec_ok && k + 1 < a.n) {
              if (!a.lower_only) *reinterpret_cast<double2*>(Grow + k) = make_double2(v0, v1);
              a.G[(int64_t)k * a.n + j] = v0;
              a.G[(int64_t)(k + 1) * a.n + j] = v1;
              continue;
            }
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const int ku = k + u;
              const double val = u ? v1 : v0;
              if (ku >= a.n || ku < j) continue;
              const bool direct = !a.lower_only || ku == j;
              if (mode == 1) {
                if (direct) Grow[ku] = val;
                if (ku > j) a.G[(int64_t)ku * a.n + j] = val;
              } else if (mode == 2) {
                if (direct) atomicAdd(Grow + ku, val);
                if (ku > j) atomicAdd(a.G + (int64_t)ku * a.n + j, val);
              } else {
                const double cur = (ph == 0) ? 0.0 : Grow[ku];
                double t = cur + val;
                if (last) {
                  t = t / a.div;
                  if (ku > j) a.G[(int64_t)ku * a.n + j] = t;
                }
                Grow[ku] = t;
              }
            }
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

// one-time: the GEMM's shared memory, and the maximal carveout for all three kernels so
// that they co-reside with each other and with the ingest / chain kernels
void set_i8_attributes() {
  static bool done = false;
  if (done) return;
  cudaFuncSetAttribute(gram_i8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, I8_SMEM);
  for (const void* k : {(const void*)gram_i8_kernel, (const void*)i8_slice_kernel, (const void*)i8_colexp_kernel})
    cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  done = true;
}

}  // namespace

// RAC_I8_SLICES=8: always 8 slices (read per launch)
static int force8_env() {
  const char* e = getenv("RAC_I8_SLICES");
  return (e && atoi(e) == 8) ? 1 : 0;
}

size_t gram_i8_ws_bytes(int64_t len, int n) {
  const int64_t nstg = (len + I8_KS - 1) / I8_KS;
  const int64_t ngrp = (int64_t)((n + I8_TM - 1) / I8_TM) * 16;
  return (size_t)I8_S * nstg * ngrp * 256 + (size_t)ngrp * 8 * sizeof(int) + 256;
}

// G (n x n, row-major) = Xc[:, :n]' Xc[:, :n] over samples [0, len) of the column-major Xc
// (ld >= len): written / div (div > 0), or ADDED (accum) for row-chunk streaming.
int launch_gram_i8(const double* Xc, int64_t ld, int64_t len, int n, double* G, double div, int accum, void* ws,
                   size_t ws_bytes, cudaStream_t st, int* bad) {
  if (n < 1 || len < 1) return RAC_OK;
  if (!ws || ws_bytes < gram_i8_ws_bytes(len, n)) return set_error(RAC_ERR_ARG, "gram_i8: workspace too small");
  const int nstg = (int)((len + I8_KS - 1) / I8_KS);
  const int ngrp = ((n + I8_TM - 1) / I8_TM) * 16;
  const size_t slice_bytes = (size_t)nstg * ngrp * 256;
  int* flags = static_cast<int*>(ws);   // the workspace's first 256 bytes (gram_i8_ws_flags)
  uint8_t* sl = static_cast<uint8_t*>(ws) + 256;
  int* ex = reinterpret_cast<int*>(sl + I8_S * slice_bytes);
  const int nfeat = ngrp * 8;
  set_i8_attributes();
  cudaMemsetAsync(flags, 0, sizeof(int), st);
  note_launch();
  i8_colexp_kernel<<<std::min(num_sms() * 8, (nfeat + 7) / 8), 256, 0, st>>>(Xc, ld, len, n, nfeat, ex, flags, bad);
  if ((nstg + 7) / 8 > 65535) return set_error(RAC_ERR_UNSUPPORTED, "gram_i8: too many samples");
  note_launch();
  i8_slice_kernel<<<dim3((unsigned)ngrp, (unsigned)((nstg + 7) / 8)), 256, 0, st>>>(
      Xc, ld, len, n, ex, sl, slice_bytes, ngrp, nstg, nullptr, nullptr, flags, force8_env());
  set_i8_attributes();
  I8Args a{};
  a.sl = sl;
  a.slice_bytes = slice_bytes;
  a.ngrp = ngrp;
  a.nstg = nstg;
  a.n = n;
  a.JT = (n + I8_TM - 1) / I8_TM;
  a.ex = ex;
  a.G = G;
  a.div = div;
  a.accum = accum;
  a.flags = flags;
  a.force8 = force8_env();
  const int tiles = a.JT * (a.JT + 1) / 2;
  note_launch();
  gram_i8_kernel<<<tiles, I8_THREADS, I8_SMEM, st>>>(a);
  return check_launch("gram_i8");
}

const int* gram_i8_ws_flags(const void* ws) { return static_cast<const int*>(ws); }

size_t gram_i8_blocks_ws_bytes(int64_t len, int s, int p) {
  const int64_t nstg = (len + I8_KS - 1) / I8_KS;
  const int64_t ngrp = (int64_t)((s + I8_TM - 1) / I8_TM) * 16;
  return (size_t)p * I8_S * nstg * ngrp * 256 + (size_t)p * ngrp * 8 * sizeof(int) + 256;
}

int launch_i8_colexp(const double* Xc, int64_t ld, int64_t len, int n, int* ex, cudaStream_t st, int* flags) {
  set_i8_attributes();
  note_launch();
  i8_colexp_kernel<<<std::min(num_sms() * 8, (n + 7) / 8), 256, 0, st>>>(Xc, ld, len, n, n, ex, flags, nullptr);
  return check_launch("i8 exponents");
}

// block mode: the p block Grams (s x s raw sums, out[b][s][s], LOWER triangle incl. diagonal) of the
// feature lists idx[b*s ..] (-1 = padding), ex_all = per-feature exponents of Xc
int launch_gram_i8_blocks(const double* Xc, int64_t ld, int64_t len, const int32_t* idx, int s, int p,
                          const int* ex_all, const int* flags, double* out, void* ws, size_t ws_bytes,
                          cudaStream_t st, cudaEvent_t after_slicing) {
  if (!ws || ws_bytes < gram_i8_blocks_ws_bytes(len, s, p))
    return set_error(RAC_ERR_ARG, "gram_i8 blocks: workspace too small");
  const int nstg = (int)((len + I8_KS - 1) / I8_KS);
  const int ngrp = ((s + I8_TM - 1) / I8_TM) * 16;
  const size_t slice_bytes = (size_t)nstg * ngrp * 256;
  uint8_t* sl = static_cast<uint8_t*>(ws);
  int* ex_blk = reinterpret_cast<int*>(sl + (size_t)p * I8_S * slice_bytes);
  if ((nstg + 7) / 8 > 65535 || p > 65535) return set_error(RAC_ERR_UNSUPPORTED, "gram_i8 blocks: shape");
  set_i8_attributes();
  note_launch();
  i8_slice_kernel<<<dim3((unsigned)ngrp, (unsigned)((nstg + 7) / 8), (unsigned)p), 256, 0, st>>>(
      Xc, ld, len, s, ex_all, sl, slice_bytes, ngrp, nstg, idx, ex_blk, flags, force8_env());
  if (after_slicing) cudaEventRecord(after_slicing, st);   // stage timing: slicing | GEMM
  set_i8_attributes();
  I8Args a{};
  a.sl = sl;
  a.slice_bytes = slice_bytes;
  a.ngrp = ngrp;
  a.nstg = nstg;
  a.n = s;
  a.JT = (s + I8_TM - 1) / I8_TM;
  a.ex = ex_blk;
  a.G = out;
  a.div = 0.0;
  a.accum = 0;
  a.blk_sl = (size_t)I8_S * slice_bytes;
  a.blk_g = (int64_t)s * s;
  a.blk_ex = ngrp * 8;
  a.lower_only = 1;   // the block systems are assembled from the lower triangle
  a.flags = flags;
  a.force8 = force8_env();
  note_launch();
  gram_i8_kernel<<<dim3((unsigned)(a.JT * (a.JT + 1) / 2), (unsigned)p), I8_THREADS, I8_SMEM, st>>>(a);
  return check_launch("gram_i8 blocks");
}

}  // namespace rac
