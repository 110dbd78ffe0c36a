// Row phase of the Gauss-Seidel chain (shared by the EN and QP engines).
//
// Rows of a column-major matrix V (m x n, leading dim ld, zero rows past m)
// are split into chunks of RC rows; chunk ch belongs to CTA ch % gridDim.x
// for the whole launch, so the running row vector `acc` (EN: r = X beta,
// QP: ax = A x) is only ever touched by its owner CTA.
//
//   acc_i += V[i, blk_prev] . delta                    (running residual update)
//   t_i    = T(i, acc_i, V[i, blk_next] . x_next)      (engine-specific)
//   partial[cta][j] = sum_i V[i, blk_next[j]] t_i      (coupling term, reduced later)
#pragma once

#include "rac_common.cuh"

namespace rac {

constexpr int RP_THREADS = 256;
constexpr int RP_QMAX = 4;  // s <= RP_QMAX * RP_THREADS

template <int RC>
struct RowPhase {
  static constexpr int NG = (RP_THREADS / 32) * (32 / RC);  // row groups of the tile reduction
  // shared-memory doubles needed (tile + reductions), plus 2*s int32 of indices
  // two tiles (prev + next block) + delta + x_next + reduction scratch
  static __host__ __device__ size_t smem_doubles(int s) { return 2 * (size_t)s * (RC + 1) + 2 * (size_t)s + NG * RC + RC; }
};

struct RowPhaseSmem {
  double* tile;
  double* tile2;
  double* sDel;
  double* sXn;
  double* red;
  double* sT;
  int32_t* sIdxP;
  int32_t* sIdxN;
};

template <int RC>
__device__ __forceinline__ RowPhaseSmem carve_rowphase(double* base, int s) {
  RowPhaseSmem w;
  w.tile = base;
  w.tile2 = w.tile + (size_t)s * (RC + 1);
  w.sDel = w.tile2 + (size_t)s * (RC + 1);
  w.sXn = w.sDel + s;
  w.red = w.sXn + s;
  w.sT = w.red + RowPhase<RC>::NG * RC;
  w.sIdxP = (int32_t*)(w.sT + RC);
  w.sIdxN = w.sIdxP + s;
  return w;
}

// sum_{j = j0, j0 + step, ...} col[j * ld] * v[j] with four independent chains (the row
// phase is latency-bound: few warps, dependent shared-memory loads); fixed order, so
// results stay deterministic
__device__ __forceinline__ double strided_dot(const double* col, const double* v, int j0, int s, int step,
                                              int ld) {
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int j = j0;
  for (; j + 3 * step < s; j += 4 * step) {
    a0 += col[j * ld] * v[j];
    a1 += col[(j + step) * ld] * v[j + step];
    a2 += col[(j + 2 * step) * ld] * v[j + 2 * step];
    a3 += col[(j + 3 * step) * ld] * v[j + 3 * step];
  }
  for (; j < s; j += step) a0 += col[j * ld] * v[j];
  return (a0 + a1) + (a2 + a3);
}

// sum_{q < NG} red[q * ld + t], four chains
template <int NG>
__device__ __forceinline__ double group_sum(const double* red, int ld, int t) {
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
  for (int q = 0; q < NG; q += 4) {
    a0 += red[q * ld + t];
    if (q + 1 < NG) a1 += red[(q + 1) * ld + t];
    if (q + 2 < NG) a2 += red[(q + 2) * ld + t];
    if (q + 3 < NG) a3 += red[(q + 3) * ld + t];
  }
  return (a0 + a1) + (a2 + a3);
}

// T(i, acc_i, u_i) -> t_i
template <int RC, class TFn>
__device__ void row_phase(const double* __restrict__ V, int64_t ld, int64_t m, int nrc,
                          const int32_t* __restrict__ idx, int s, int bprev, int bnext,
                          const double* delta, const double* xsrc, double* acc,
                          double* partial, const RowPhaseSmem& w, TFn tfn) {
  constexpr int NG = RowPhase<RC>::NG;
  const int tid = threadIdx.x;
  const int P = gridDim.x;
  if (bprev >= 0)
    for (int j = tid; j < s; j += RP_THREADS) {
      w.sIdxP[j] = idx[(int64_t)bprev * s + j];
      w.sDel[j] = ldcg(delta + j);
    }
  if (bnext >= 0)
    for (int j = tid; j < s; j += RP_THREADS) {
      int g = idx[(int64_t)bnext * s + j];
      w.sIdxN[j] = g;
      w.sXn[j] = (g >= 0) ? ldcg(xsrc + g) : 0.0;
    }
  __syncthreads();
  const int lane = tid & 31, warp = tid >> 5;
  const int grp = warp * (32 / RC) + lane / RC;
  const int ri = lane % RC;
  double part[RP_QMAX];
#pragma unroll
  for (int q = 0; q < RP_QMAX; ++q) part[q] = 0.0;

  // Both tiles of a row chunk are fetched with asynchronous 8-byte copies
  // (LDGSTS): every thread has ~s*RC/256 loads in flight instead of one.
  auto issue = [&](double* dst, const int32_t* sIdx, int64_t i0) {
    for (int e = tid; e < s * RC; e += RP_THREADS) {
      int j = e / RC, i = e - j * RC;
      int g = sIdx[j];
      double* d = dst + j * (RC + 1) + i;
      if (g >= 0) cp_async8(d, V + (int64_t)g * ld + i0 + i);
      else *d = 0.0;
    }
  };
  for (int ch = blockIdx.x; ch < nrc; ch += P) {
    const int64_t i0 = (int64_t)ch * RC;
    const int rows = (int)min64(RC, m - i0);
    if (bprev >= 0) issue(w.tile, w.sIdxP, i0);
    if (bnext >= 0) issue(w.tile2, w.sIdxN, i0);
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    if (bprev >= 0) {
      w.red[grp * RC + ri] = strided_dot(w.tile + ri, w.sDel, grp, s, NG, RC + 1);
      __syncthreads();
      if (tid < rows) acc[i0 + tid] += group_sum<NG>(w.red, RC, tid);
      __syncthreads();
    }
    if (bnext >= 0) {
      w.red[grp * RC + ri] = strided_dot(w.tile2 + ri, w.sXn, grp, s, NG, RC + 1);
      __syncthreads();
      if (tid < RC) {
        const double tot = group_sum<NG>(w.red, RC, tid);
        w.sT[tid] = (tid < rows) ? tfn(i0 + tid, acc[i0 + tid], tot) : 0.0;
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < RP_QMAX; ++q) {
        int j = tid + q * RP_THREADS;
        if (j < s) {
          const double* col = w.tile2 + j * (RC + 1);
          double a = 0.0, b = 0.0;
#pragma unroll
          for (int i = 0; i < RC; i += 2) {
            a += col[i] * w.sT[i];
            b += col[i + 1] * w.sT[i + 1];
          }
          part[q] += a + b;
        }
      }
    }
    __syncthreads();
  }
  if (bnext >= 0) {
#pragma unroll
    for (int q = 0; q < RP_QMAX; ++q) {
      int j = tid + q * RP_THREADS;
      if (j < s) partial[(int64_t)blockIdx.x * s + j] = part[q];
    }
  }
}

}  // namespace rac

namespace rac {

// ---------------------------------------------------------------------------
// One-tile resident row phase (EN streaming chain, RC == 0 mode): CTA k owns the
// contiguous rows [r0, r0 + nr) for the whole launch and keeps X[rows, b] of the
// current block resident in shared memory from the row phase that loaded it as
// "next" to the one that applies its delta, so every block's columns are read
// once per sweep and the work is balanced (no row chunks to distribute).
//   (a) r += X[rows, b_prev] delta   (resident tile)
//   (b) X[rows, b_next] -> the tile  (8-byte cp.async, odd row stride: conflict-free
//                                     along rows and along columns)
//   (c) t = T(r, X[rows, b_next] x_next)
//   (d) partial[cta][j] = X[rows, b_next[j]]' t
// ---------------------------------------------------------------------------
struct Row1tSmem {
  double* tile;   // [s][rwp]
  double* sR;     // [rw] r at this CTA's rows (kept for the launch)
  double* sT;     // [rw]
  double* sX;     // [s]
  double* sDel;   // [s]
  double* red;    // [G][rw]
  int32_t* sIdx;  // [s]
  int rwp;
  int redcap;     // doubles in `red` (sized for rw rows; a CTA with fewer rows must not use more)
};

__host__ __device__ inline int row1t_groups(int rw) { return rw >= RP_THREADS ? 1 : RP_THREADS / rw; }
// row stride of the tile in doubles: even (16-byte cp.async rows); phase (d) reads it
// column-parallel (lane j at j * stride), which is 2-way bank-conflicted for a stride of
// 2 mod 4 and 4-way for 0 mod 4, so rw (even) is padded to the next 2 mod 4
__host__ __device__ inline int row1t_stride(int rw) { return (rw % 4 == 2) ? rw : rw + 2; }
__host__ __device__ inline size_t row1t_smem_bytes(int s, int rw) {
  const int rwp = row1t_stride(rw);
  return ((size_t)s * rwp + 2 * (size_t)rw + 2 * (size_t)s + (size_t)row1t_groups(rw) * rw) * sizeof(double) +
         (size_t)s * sizeof(int32_t);
}
__device__ __forceinline__ Row1tSmem carve_row1t(double* base, int s, int rw) {
  Row1tSmem w;
  w.rwp = row1t_stride(rw);
  w.tile = base;
  w.sR = w.tile + (size_t)s * w.rwp;
  w.sT = w.sR + rw;
  w.sX = w.sT + rw;
  w.sDel = w.sX + s;
  w.red = w.sDel + s;
  w.sIdx = reinterpret_cast<int32_t*>(w.red + (size_t)row1t_groups(rw) * rw);
  w.redcap = row1t_groups(rw) * rw;
  return w;
}

// sum over j = j0, j0 + step, ... < s of tile[j * rwp + row] * v[j], four chains
__device__ __forceinline__ double row1t_dot(const double* tile, int rwp, int row, const double* v, int j0, int s,
                                            int step) {
  return strided_dot(tile + row, v, j0, s, step, rwp);
}

// indices and current beta of block b (the row phase's next block) into shared memory while
// the chain waits on grid barriers (b's beta is final: b is solved later), asynchronously:
// (1) the indices (cp.async, one group), (2) after they landed, beta gathered by them
// (cp.async, one group that the row phase's wait completes)
__device__ __forceinline__ void row1t_gather_idx(const int32_t* __restrict__ idx, int s, int b, const Row1tSmem& w) {
  for (int j = threadIdx.x; j < s; j += RP_THREADS) cp_async4(w.sIdx + j, idx + (int64_t)b * s + j);
  cp_async_commit();
}
__device__ __forceinline__ void row1t_gather_beta(int s, const double* xsrc, const Row1tSmem& w) {
  cp_async_wait<0>();   // this thread's index copies (the same threads read them back)
  for (int j = threadIdx.x; j < s; j += RP_THREADS) {
    const int g = w.sIdx[j];
    if (g >= 0) cp_async8(w.sX + j, xsrc + g);
    else w.sX[j] = 0.0;
  }
  cp_async_commit();
}

// The resident-tile dot products in column chunks: the same operations in the same order as
// strided_dot (four chains over j = j0, j0 + step, ...; the tail into chain 0), cut at chunk ends
// that are multiples of 4 * step, so the chains run on across chunks and the result is
// bit-identical to the unchunked sum.
struct Dot4 {
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int j = 0;
};
__device__ __forceinline__ void dot4_chunk(Dot4& d, const double* col, const double* v, int ce, int step, int ld) {
  int j = d.j;
  for (; j + 3 * step < ce; j += 4 * step) {
    d.a0 += col[j * ld] * v[j];
    d.a1 += col[(j + step) * ld] * v[j + step];
    d.a2 += col[(j + 2 * step) * ld] * v[j + 2 * step];
    d.a3 += col[(j + 3 * step) * ld] * v[j + 3 * step];
  }
  d.j = j;
}
__device__ __forceinline__ double dot4_finish(Dot4& d, const double* col, const double* v, int s, int step, int ld) {
  for (int j = d.j; j < s; j += step) d.a0 += col[j * ld] * v[j];
  return (d.a0 + d.a1) + (d.a2 + d.a3);
}

constexpr int R1T_NC = 3;   // column chunks of the tile pipeline (measured on config 5: chain 3.26 ms with 4, 3.13 with 3, 3.25 with 2)

// Columns of the tile are released chunk by chunk while (a) runs and refilled at once with
// the next block's columns (16-byte cp.async, one group per chunk); (c) consumes the chunks as
// they land.  The tile's HBM read (D once per sweep) thereby overlaps both reductions instead
// of standing between them.
template <class TFn>
__device__ void row_phase_1t(const double* __restrict__ V, int64_t ld, int64_t r0, int nr,
                             const int32_t* __restrict__ idx, int s, int bprev, int bnext, const double* delta,
                             const double* xsrc, double* partial, const Row1tSmem& w, TFn tfn,
                             long long* rt = nullptr, bool pre_gathered = false,
                             unsigned long long* ll_part = nullptr, unsigned tag_next = 0u) {
  // ll_part != nullptr: the partials leave as tagged words (rac_common.cuh ll_store, tag_next) that
  // the S phase spins on
  // rt (tracing, CTA 0 thread 0): %globaltimer after (a) + the issue of the loads, after the
  // first chunk landed, after (c), after (d)
  const int tid = threadIdx.x;
  // groups of the row reductions; the last CTA's shorter row range (nr < rw) must stay
  // inside the reduction buffer sized for rw rows
  const int G = min(row1t_groups(nr), w.redcap / nr);
  const int row = tid % nr, grp = tid / nr;
  const bool act = grp < G;
  // chunk width: a multiple of 4 G columns (the dot products' four chains of stride G)
  const int CH = (((s + R1T_NC - 1) / R1T_NC + 4 * G - 1) / (4 * G)) * (4 * G);
  if (bprev >= 0)
    for (int j = tid; j < s; j += RP_THREADS) w.sDel[j] = ldcg(delta + j);
  if (bnext >= 0 && !pre_gathered)
    for (int j = tid; j < s; j += RP_THREADS) {
      const int g = idx[(int64_t)bnext * s + j];
      w.sIdx[j] = g;
      w.sX[j] = (g >= 0) ? ldcg(xsrc + g) : 0.0;
    }
  if (bnext >= 0 && pre_gathered) cp_async_wait<0>();   // this thread's beta gathers (row1t_gather_beta)
  __syncthreads();
  const int h = nr >> 1;   // 16-byte pieces per column (nr, r0, ld and the row stride are even)
  // piece e = tid + k RP_THREADS of a chunk is (column e / h, piece e % h): walked incrementally
  // (one division per row phase instead of one per piece; the issue of the ~8 pieces per thread
  // and chunk was ~0.45 us of instructions per chunk)
  const int pj0 = tid / h, pi0 = tid - pj0 * h;
  const int pdj = RP_THREADS / h, pdi = RP_THREADS - pdj * h;
  // h <= RP_THREADS (always, for tiles that fit): thread = (column lane pj0 < pdj, FIXED piece pi0),
  // columns in steps of pdj — per piece one index load, one 64-bit multiply-add and the copy
  const double* const vsrc = V + r0 + 2 * pi0;
  double* const vdst = w.tile + 2 * pi0;
  auto issue_chunk = [&](int c) {
    const int cb = min(c * CH, s), ce = min(cb + CH, s);
    if (bnext >= 0 && pdj >= 1) {
      if (pj0 < pdj)
        for (int j = cb + pj0; j < ce; j += pdj) {
          const int g = w.sIdx[j];
          double* d = vdst + (size_t)j * w.rwp;
          if (g >= 0) cp_async16(d, vsrc + (int64_t)g * ld);
          else d[0] = d[1] = 0.0;
        }
    } else if (bnext >= 0) {
      const int ncol = ce - cb;
      int jj = pj0, ii = pi0;
      while (jj < ncol) {
        const int j = cb + jj;
        const int g = w.sIdx[j];
        double* d = w.tile + (size_t)j * w.rwp + 2 * ii;
        if (g >= 0) cp_async16(d, V + (int64_t)g * ld + r0 + 2 * ii);
        else d[0] = d[1] = 0.0;
        jj += pdj;
        ii += pdi;
        if (ii >= h) {
          ii -= h;
          ++jj;
        }
      }
    }
    cp_async_commit();
  };
  if (bprev >= 0) {   // (a) resident tile holds X[rows, b_prev]
    Dot4 d;
    d.j = grp;
#pragma unroll
    for (int c = 0; c < R1T_NC; ++c) {
      const int ce = (c == R1T_NC - 1) ? s : min((c + 1) * CH, s);
      const bool fin = ce == s && (c == 0 || c * CH < s);   // the chunk that holds the last columns (and the tail)
      if (act) dot4_chunk(d, w.tile + row, w.sDel, ce, G, w.rwp);
      if (fin && act) w.red[grp * nr + row] = dot4_finish(d, w.tile + row, w.sDel, s, G, w.rwp);
      __syncthreads();   // every thread is done with the chunk's columns
      issue_chunk(c);
    }
    if (tid < nr) {
      double u = 0.0;
      for (int q = 0; q < G; ++q) u += w.red[q * nr + tid];
      w.sR[tid] += u;
    }
    __syncthreads();
  } else {
#pragma unroll
    for (int c = 0; c < R1T_NC; ++c) issue_chunk(c);
  }
  if (rt) rt[0] = gtimer();
  if (bnext < 0) {
    cp_async_wait<0>();
    return;
  }
  // (c) chunk c is complete when at most NC - 1 - c groups are pending
  {
    Dot4 d;
    d.j = grp;
#pragma unroll
    for (int c = 0; c < R1T_NC; ++c) {
      if (c == 0) cp_async_wait<R1T_NC - 1>();
      else if (c == 1) cp_async_wait<(R1T_NC >= 2 ? R1T_NC - 2 : 0)>();
      else if (c == 2) cp_async_wait<(R1T_NC >= 3 ? R1T_NC - 3 : 0)>();
      else cp_async_wait<0>();
      __syncthreads();
      if (rt && c == 0) rt[1] = gtimer();
      const int ce = (c == R1T_NC - 1) ? s : min((c + 1) * CH, s);
      const bool fin = ce == s && (c == 0 || c * CH < s);
      if (act) dot4_chunk(d, w.tile + row, w.sX, ce, G, w.rwp);
      if (fin && act) w.red[grp * nr + row] = dot4_finish(d, w.tile + row, w.sX, s, G, w.rwp);
    }
  }
  __syncthreads();
  if (tid < nr) {
    double u = 0.0;
    for (int q = 0; q < G; ++q) u += w.red[q * nr + tid];
    w.sT[tid] = tfn(r0 + tid, w.sR[tid], u);
  }
  __syncthreads();
  if (rt) rt[2] = gtimer();
  // (d)
  for (int j = tid; j < s; j += RP_THREADS) {
    const double* col = w.tile + (size_t)j * w.rwp;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int i = 0;
    // 16-byte loads (the row stride and the tile base are even): lane j at j * rwp * 8 bytes is
    // conflict-free for 16-byte accesses when rwp = 2 mod 4, and 2-way conflicted for 8-byte ones
    const double2* col2 = reinterpret_cast<const double2*>(col);
    const double2* t2 = reinterpret_cast<const double2*>(w.sT);
    for (; i + 4 <= nr; i += 4) {
      const double2 c0 = col2[i >> 1], c1 = col2[(i >> 1) + 1];
      const double2 u0 = t2[i >> 1], u1 = t2[(i >> 1) + 1];
      a0 += c0.x * u0.x;
      a1 += c0.y * u0.y;
      a2 += c1.x * u1.x;
      a3 += c1.y * u1.y;
    }
    for (; i < nr; ++i) a0 += col[i] * w.sT[i];
    // column-major partials [j][cta]: the S1 reduction then reads each column's P partials
    // as one contiguous run
    const double pv = (a0 + a1) + (a2 + a3);
    if (ll_part) ll_store(ll_part + 2 * ((size_t)j * gridDim.x + blockIdx.x), pv, tag_next);
    else partial[(int64_t)j * gridDim.x + blockIdx.x] = pv;
  }
  __syncthreads();
  if (rt) rt[3] = gtimer();
}

}  // namespace rac
