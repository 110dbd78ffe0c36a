// Elastic-net / LASSO / ridge sweep engine behind elastic_net.fit
// (elastic_net.py:150-232), sm_100a, FP64, everything HBM-resident.
//
// Per sweep (RAC):  K1 chunk-sort the host permutation -> K2 batched DMMA
// block Grams -> K3 batched Cholesky/inverse -> K4 one cooperative launch
// that runs the whole Gauss-Seidel chain over the p blocks:
//
//   R  (row phase, all CTAs, rows split across CTAs)
//        r_i += X[i, blk_prev] . delta_prev            (elastic_net.py:223)
//        t_i  = r_i - X[i, blk_next] . beta[blk_next]
//        partial_cta[j] = sum_i X[i, blk_next[j]] t_i  (elastic_net.py:205)
//   -- grid barrier --
//   S1 rhs_j = -(c + (sum_cta partial)/m - xi - gamma z)   (elastic_net.py:206)
//   -- grid barrier --
//   S2 beta_new = inv_b rhs (elastic_net.py:222); delta = beta_new - beta;
//      fused z-prox / dual / residual for the block's coordinates
//      (elastic_net.py:225-228; bitwise-equivalent since every coordinate
//      belongs to exactly one block and z/xi of other blocks are untouched)
//   -- grid barrier --
//
// The one-tile streaming chain (RC == 0, config 5) keeps only the last of these barriers: the
// partials reach the S phase as tagged words, and S1 / S2 are one fused phase (EnChainArgs::ll,
// ::fuse below).
//
// X is stored column-major with a leading dimension padded to 32 rows (zero
// rows), so a block's column gather is a set of contiguous, coalesced reads.
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "rac_internal.h"
#include "rac_rowphase.cuh"

namespace rac {

constexpr int ENT = RP_THREADS;   // threads per chain CTA
constexpr int EN_QMAX = RP_QMAX;   // block_size <= EN_QMAX * ENT

struct EnChainArgs {
  const double* Xc;
  int64_t ld, m, n;
  int s, p, nrc;        // block size, blocks, row chunks
  const int32_t* idx;   // [p][s] block table of this sweep
  const int32_t* order; // [p] visit order (nullptr: identity)
  const double* inv;    // [p][s][s]
  const int32_t* info;  // [p]
  const double* c;
  double *beta, *z, *xi, *r;
  double *partial, *rhs, *delta;
  double *wsum, *wmax;  // per global warp
  unsigned* bar;
  int32_t* ctrl;        // [0] done, [1] iterations, [2] failed block + 1, [3] converged
  double gamma, thr, den, mdiv, tol;
  int sweep;
  double *hist_p, *hist_d;
  long long* trace;     // optional: %globaltimer at every phase boundary (CTA 0)
  int rw;               // RC == 0 (one-tile resident row phase): rows per CTA
  // RC == 0: the row phase's partials reach the S phase as tagged 64-bit word pairs (rac_common.cuh
  // ll_store) that the reader spins on, instead of behind a grid barrier.  Layout: partials
  // [s][P][2], then the fused S phase's CTA sums [s][ceil(s / 8)][2]; tag of block step t =
  // tag0 + t + 1 (unique per launch and step).  Each buffer is rewritten for step t + 1 only
  // after every reader of step t is done: a writer of step t + 1 data depends, through the chain
  // itself, on all of step t's readers' outputs.  Every tagged word has ONE reader; the broadcast
  // hand-offs (rhs to all S warps, delta to all CTAs) were measured slower as tagged words — the
  // pollers of a shared 8 KB delay its writers — and stay behind a grid barrier.
  unsigned long long* ll;
  unsigned tag0;
  int ll_mask;   // 1: tagged partials (0: grid barrier)
  // fused S phase (needs the tagged partials; one pass: every column has its own warp, s <= 512):
  // warp j scales row j of the symmetric inverse by rhs_j, the CTA sums its 8 scaled rows in shared
  // memory (fuse_off: byte offset of the [8][s] buffer) and publishes them as tagged words
  // [s][ceil(s / 8)][2] (behind the words above); warp i then sums row i's CTA partials.  Every
  // tagged word has one reader, and the rhs broadcast with its grid barrier is gone.
  int fuse;
  unsigned fuse_off;
};


// RC > 0: row chunks of RC rows streamed through shared memory; RC == 0: each CTA owns
// `rw` contiguous rows and keeps the current block's tile resident (row_phase_1t)
template <int RC>
__global__ void __maxnreg__(192) en_chain_kernel(EnChainArgs a) {
  if (a.ctrl[0]) return;
  extern __shared__ __align__(16) double esm[];
  const int s = a.s;
  constexpr int RCC = RC > 0 ? RC : 8;   // (unused layout parameter in the one-tile mode)
  const RowPhaseSmem w = carve_rowphase<RCC>(esm, s);
  const Row1tSmem w1 = carve_row1t(esm, s, a.rw > 0 ? a.rw : 1);
  const int64_t r0 = (int64_t)blockIdx.x * a.rw;
  const int nr1 = (RC == 0) ? (int)min64(a.rw, a.ld - r0) : 0;
  __shared__ int bad;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int P = gridDim.x;
  const int gw = blockIdx.x * (ENT / 32) + warp, GW = P * (ENT / 32);
  unsigned target = 0;

  if (tid == 0) {
    bad = 0;
    for (int t = 0; t < a.p; ++t) {
      int b = a.order ? a.order[t] : t;
      if (a.info[b]) { bad = b + 1; break; }
    }
  }
  __syncthreads();
  if (bad) {
    if (blockIdx.x == 0 && tid == 0) { a.ctrl[2] = bad; a.ctrl[0] = 1; }
    return;
  }

  double my_sum = 0.0, my_max = 0.0;
  const double m = a.mdiv, gamma = a.gamma;

  auto tfn = [&](int64_t, double r_i, double u) { return r_i - u; };
  const bool tr = a.trace && blockIdx.x == 0 && tid == 0;
  int tp = 0;
  if (tr) a.trace[tp++] = gtimer();
  int bnext = a.order ? a.order[0] : 0;
  const bool LL = (RC == 0) && a.ll != nullptr;
  const bool LLP = LL && (a.ll_mask & 1);
  unsigned long long* const llp = LLP ? a.ll : nullptr;
  const bool s_cta = blockIdx.x * (ENT / 32) < s;   // this CTA has S1 / S2 rows
  const bool FUSE = LLP && a.fuse;
  if constexpr (RC == 0) {
    for (int i = threadIdx.x; i < nr1; i += ENT) w1.sR[i] = a.r[r0 + i];
    __syncthreads();
    row_phase_1t(a.Xc, a.ld, r0, nr1, a.idx, s, -1, bnext, a.delta, a.beta, a.partial, w1, tfn, nullptr, false,
                 llp, a.tag0 + 1u);
  } else {
    row_phase<RC>(a.Xc, a.ld, a.m, a.nrc, a.idx, s, -1, bnext, a.delta, a.beta, a.r, a.partial, w, tfn);
  }
  if (tr) a.trace[tp++] = gtimer();
  for (int t = 0; t < a.p; ++t) {
    const int b = bnext;
    const unsigned tg = a.tag0 + (unsigned)t + 1u;
    if (!LLP) grid_barrier(a.bar, target, P);
    if (tr) a.trace[tp++] = gtimer();
    // this CTA's S2 rows of inv_b -> L2 while S1 runs (one 128-byte line per thread)
    {
      const double* Ib = a.inv + (int64_t)b * s * s;
      const int lines = (s * (int)sizeof(double) + 127) / 128;
      for (int e = threadIdx.x; e < (ENT / 32) * lines; e += ENT) {
        const int i = blockIdx.x * (ENT / 32) + e / lines;   // global warp of row i (loop below, first round)
        if (i < s) prefetch_l2(Ib + (int64_t)i * s + 16 * (e % lines));
      }
    }
    if constexpr (RC == 0)
      if (t + 1 < a.p) row1t_gather_idx(a.idx, s, a.order ? a.order[t + 1] : t + 1, w1);
    if (FUSE) {
      if (s_cta) {
        const int NSC = (s + ENT / 32 - 1) / (ENT / 32);
        unsigned long long* const ypart = a.ll + 2 * (size_t)s * P;
        const double* Ibf = a.inv + (int64_t)b * s * s;
        const int j = gw;
        const bool mine = j < s;
        const int g = mine ? a.idx[(int64_t)b * s + j] : -1;
        double cg = 0.0, xg = 0.0, zg = 0.0, bo = 0.0;
        if (g >= 0) {
          cg = a.c[g];
          xg = ldcg(a.xi + g);
          zg = ldcg(a.z + g);
          bo = ldcg(a.beta + g);
        }
        // row j of the symmetric inverse (= its column j), in flight behind the partials' poll
        constexpr int KM = 16;   // s <= 512
        double rowv[KM];
#pragma unroll
        for (int k = 0; k < KM; ++k) {
          const int i = lane + 32 * k;
          rowv[k] = (mine && i < s) ? Ibf[(int64_t)j * s + i] : 0.0;
        }
        double acc = 0.0;
        if (mine) {
          const unsigned long long* pj = llp + 2 * (size_t)j * P;
          constexpr int QM = 8;   // P <= 256 CTAs
          unsigned long long w0[QM], w1[QM];
#pragma unroll
          for (int u = 0; u < QM; ++u) {
            const int q = lane + 32 * u;
            if (q < P) ll_load2(pj + 2 * q, w0[u], w1[u]);
          }
#pragma unroll
          for (int u = 0; u < QM; ++u) {
            const int q = lane + 32 * u;
            if (q < P) {
              while (!(ll_ok(w0[u], tg) && ll_ok(w1[u], tg))) ll_load2(pj + 2 * q, w0[u], w1[u]);
              acc += ll_value((unsigned)w0[u], (unsigned)w1[u]);
            }
          }
        }
        acc = warp_sum(acc);
        double rhs = 0.0;
        if (g >= 0) {
          double cross = acc / m;
          rhs = -(sub(sub(add(cg, cross), xg), mul(gamma, zg)));
        }
        double* sV = reinterpret_cast<double*>(reinterpret_cast<char*>(esm) + a.fuse_off);
#pragma unroll
        for (int k = 0; k < KM; ++k) {
          const int i = lane + 32 * k;
          if (i < s) sV[warp * s + i] = rowv[k] * rhs;
        }
        if (tr) a.trace[tp++] = gtimer();
        __syncthreads();
        for (int i = threadIdx.x; i < s; i += ENT) {
          double y = 0.0;
#pragma unroll
          for (int w8 = 0; w8 < ENT / 32; ++w8) y += sV[w8 * s + i];
          ll_store(ypart + 2 * ((size_t)i * NSC + blockIdx.x), y, tg);
        }
        if (tr) a.trace[tp++] = gtimer();
        if (mine) {
          const unsigned long long* yi = ypart + 2 * (size_t)j * NSC;
          unsigned long long w0[2], w1[2];   // NSC <= 64
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int q = lane + 32 * u;
            if (q < NSC) ll_load2(yi + 2 * q, w0[u], w1[u]);
          }
          double bsum = 0.0;
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int q = lane + 32 * u;
            if (q < NSC) {
              while (!(ll_ok(w0[u], tg) && ll_ok(w1[u], tg))) ll_load2(yi + 2 * q, w0[u], w1[u]);
              bsum += ll_value((unsigned)w0[u], (unsigned)w1[u]);
            }
          }
          bsum = warp_sum(bsum);
          if (lane == 0) {
            if (g >= 0) {
              const double bn = bsum;
              a.delta[j] = bn - bo;
              a.beta[g] = bn;
              const double av = sub(xg, mul(gamma, bn));
              const double zn = __ddiv_rn(neg_shrink(av, a.thr), a.den);
              a.z[g] = zn;
              a.xi[g] = sub(xg, mul(gamma, sub(bn, zn)));
              my_sum += fabs(sub(bn, zn));
              my_max = fmax(my_max, fabs(sub(zn, zg)));
            } else {
              a.delta[j] = 0.0;
            }
          }
        }
        __syncthreads();   // sV is rewritten by the next block's S phase
      } else if (tr) {
        tp += 2;
      }
      if constexpr (RC == 0)
        if (t + 1 < a.p) row1t_gather_beta(s, a.beta, w1);
      if (tr) a.trace[tp++] = gtimer();
    } else {
    // ---- S1: reduce the per-CTA partials -> block right-hand side
    for (int j = gw; j < s; j += GW) {
      // the coordinate's scalars (final since the previous sweep) are requested before the
      // reduction, so their L2 round trips overlap it instead of following it
      const int g = a.idx[(int64_t)b * s + j];
      double cg = 0.0, xg = 0.0, zg = 0.0;
      if (g >= 0) {
        cg = a.c[g];
        xg = ldcg(a.xi + g);
        zg = ldcg(a.z + g);
      }
      double acc = 0.0;
      if (LLP) {
        // the column's P tagged partials: all loads in flight, then re-poll the late ones; summed
        // in the same order as the plain path
        const unsigned long long* pj = llp + 2 * (size_t)j * P;
        constexpr int QM = 8;   // P <= 256 CTAs
        unsigned long long w0[QM], w1[QM];
#pragma unroll
        for (int u = 0; u < QM; ++u) {
          const int q = lane + 32 * u;
          if (q < P) ll_load2(pj + 2 * q, w0[u], w1[u]);
        }
#pragma unroll
        for (int u = 0; u < QM; ++u) {
          const int q = lane + 32 * u;
          if (q < P) {
            while (!(ll_ok(w0[u], tg) && ll_ok(w1[u], tg))) ll_load2(pj + 2 * q, w0[u], w1[u]);
            acc += ll_value((unsigned)w0[u], (unsigned)w1[u]);
          }
        }
      } else {
        // RC == 0: partials are [j][cta] (row_phase_1t), else [cta][j]
        for (int q = lane; q < P; q += 32)
          acc += ldcg(a.partial + (RC == 0 ? (int64_t)j * P + q : (int64_t)q * s + j));
      }
      acc = warp_sum(acc);
      if (lane == 0) {
        double rhs = 0.0;
        if (g >= 0) {
          double cross = acc / m;
          rhs = -(sub(sub(add(cg, cross), xg), mul(gamma, zg)));
        }
        a.rhs[j] = rhs;
      }
    }
    if (tr) a.trace[tp++] = gtimer();
    grid_barrier(a.bar, target, P);
    if (tr) a.trace[tp++] = gtimer();
    // ---- S2: beta_b = inv_b rhs, fused prox/dual/residual per coordinate
    const double* Ib = a.inv + (int64_t)b * s * s;
    for (int i = gw; i < s; i += GW) {
      int g = a.idx[(int64_t)b * s + i];
      const double* row = Ib + (int64_t)i * s;
      // old beta / z / xi requested before the dot product (see S1)
      double bo = 0.0, zo = 0.0, x0 = 0.0;
      if (g >= 0) {
        bo = ldcg(a.beta + g);
        zo = ldcg(a.z + g);
        x0 = ldcg(a.xi + g);
      }
      double acc = 0.0;
      for (int j = lane; j < s; j += 32) acc += row[j] * ldcg(a.rhs + j);
      acc = warp_sum(acc);
      if (lane == 0) {
        if (g >= 0) {
          const double bn = acc;
          a.delta[i] = bn - bo;
          a.beta[g] = bn;
          const double av = sub(x0, mul(gamma, bn));
          const double zn = __ddiv_rn(neg_shrink(av, a.thr), a.den);
          a.z[g] = zn;
          a.xi[g] = sub(x0, mul(gamma, sub(bn, zn)));
          my_sum += fabs(sub(bn, zn));
          my_max = fmax(my_max, fabs(sub(zn, zo)));
        } else {
          a.delta[i] = 0.0;
        }
      }
    }
    // the next row phase's block: its beta (final until its own solve) gathered into shared
    // memory behind this CTA's S2 work, landing during the barrier (indices issued before S1)
    if constexpr (RC == 0)
      if (t + 1 < a.p) row1t_gather_beta(s, a.beta, w1);
    if (tr) a.trace[tp++] = gtimer();
    }   // !FUSE
    grid_barrier(a.bar, target, P);
    if (tr) a.trace[tp++] = gtimer();
    bnext = (t + 1 < a.p) ? (a.order ? a.order[t + 1] : t + 1) : -1;
    if constexpr (RC == 0)
      row_phase_1t(a.Xc, a.ld, r0, nr1, a.idx, s, b, bnext, a.delta, a.beta, a.partial, w1, tfn,
                   tr ? a.trace + 16 + 16 * (size_t)a.p + s + 4 * (size_t)t : nullptr, true, llp, tg + 1u);
    else
      row_phase<RC>(a.Xc, a.ld, a.m, a.nrc, a.idx, s, b, bnext, a.delta, a.beta, a.r, a.partial, w, tfn);
    if (tr) a.trace[tp++] = gtimer();
  }
  if constexpr (RC == 0)
    for (int i = threadIdx.x; i < nr1; i += ENT) a.r[r0 + i] = w1.sR[i];
  if (lane == 0) {
    a.wsum[gw] = my_sum;
    a.wmax[gw] = my_max;
  }
  grid_barrier(a.bar, target, P);
  if (blockIdx.x == 0 && warp == 0) {
    double tot = 0.0, mx = 0.0;
    for (int q = lane; q < GW; q += 32) {
      tot += ldcg(a.wsum + q);
      mx = fmax(mx, ldcg(a.wmax + q));
    }
    tot = warp_sum(tot);
    mx = warp_max(mx);
    if (lane == 0) {
      a.hist_p[a.sweep] = tot;
      a.hist_d[a.sweep] = gamma * mx;
      a.ctrl[1] = a.sweep + 1;
      if (a.tol >= 0.0 && tot <= a.tol) {
        a.ctrl[0] = 1;
        a.ctrl[3] = 1;
      }
    }
  }
}

}  // namespace rac

#include "en_res.cuh"
#include "en_cov.cuh"
#include "en_cla.cuh"

namespace rac {

// ---------------------------------------------------------------------------
// prologue kernels
// ---------------------------------------------------------------------------
// row-major X (m x n) -> column-major Xc (ld x n), rows m..ld-1 zero
__global__ void transpose_pad_kernel(const double* __restrict__ X, int64_t m, int64_t n, int64_t ld,
                                     double* __restrict__ Xc) {
  __shared__ double t[32][33];
  const int64_t i0 = (int64_t)blockIdx.y * 32, j0 = (int64_t)blockIdx.x * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    int64_t i = i0 + r, j = j0 + threadIdx.x;
    t[r][threadIdx.x] = (i < m && j < n) ? X[i * n + j] : 0.0;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    int64_t j = j0 + r, i = i0 + threadIdx.x;
    if (j < n && i < ld) Xc[j * ld + i] = t[threadIdx.x][r];
  }
}

int launch_transpose_pad(const double* X, int64_t m, int64_t n, int64_t ld, double* Xc, cudaStream_t st) {
  dim3 grid((unsigned)((n + 31) / 32), (unsigned)((ld + 31) / 32));
  if (grid.y > 65535) return set_error(RAC_ERR_UNSUPPORTED, "transpose: too many rows (%lld)", (long long)m);
  transpose_pad_kernel<<<grid, dim3(32, 8), 0, st>>>(X, m, n, ld, Xc);
  note_launch();
  return check_launch("transpose_pad");
}

// rows [row0, row0 + rows) of a row-major chunk -> column-major Xc; the last
// chunk also zero-fills the padding rows up to ld
__global__ void transpose_rows_kernel(const double* __restrict__ X, int64_t rows, int64_t n, int64_t ld,
                                      int64_t row0, int64_t rows_out, double* __restrict__ Xc) {
  __shared__ double t[32][33];
  const int64_t i0 = (int64_t)blockIdx.y * 32, j0 = (int64_t)blockIdx.x * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    int64_t i = i0 + r, j = j0 + threadIdx.x;
    t[r][threadIdx.x] = (i < rows && j < n) ? X[i * n + j] : 0.0;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    int64_t j = j0 + r, i = i0 + threadIdx.x;
    if (j < n && i < rows_out) Xc[j * ld + row0 + i] = t[threadIdx.x][r];
  }
}

__global__ void scale_kernel(double* v, int64_t total, double div) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x)
    v[e] = v[e] / div;
}

// c_j = -(X[:, j] . y) / m      (elastic_net.py:177)
__global__ void neg_xty_kernel(const double* __restrict__ Xc, int64_t ld, int64_t m, int64_t n,
                               const double* __restrict__ y, double mdiv, double* __restrict__ c) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t j = w; j < n; j += nw) {
    const double* col = Xc + j * ld;
    double acc = 0.0;
    for (int64_t i = lane; i < m; i += 32) acc += col[i] * y[i];
    acc = warp_sum(acc);
    if (lane == 0) c[j] = (-acc) / mdiv;
  }
}

}  // namespace rac

// ---------------------------------------------------------------------------
// context
// ---------------------------------------------------------------------------
struct rac_en_ctx {
  int64_t m = 0, n = 0, ld = 0;
  int s = 0, p = 0, mode = 0;
  double lam = 0, alpha = 0, gamma = 1;
  cudaStream_t st = nullptr;
  int P = 0, RC = 32, nrc = 0;
  int variant = 0, nch = 0;   // 1: resident-tile cluster chain (en_chain_res_kernel)
  int rw = 0;                 // streaming chain with RC == 0: rows per CTA (one resident tile)
  int cs = 2;                 // its cluster size (2, 4 or 8)
  rac::GramPlan gp{};
  bool have_data = false, have_partition = false;
  int sweeps = 0;        // sweeps enqueued so far (history index; reset by rac_en_reset)
  unsigned msg_tag = 0;  // lookahead-chain launches so far: tag of the tagged messages (never reset)
  unsigned long long* ll = nullptr;   // streaming one-tile chain: tagged hand-off words (EnChainArgs::ll)
  unsigned ll_epoch = 0;              // chain launches with tagged hand-offs so far (tag0 = epoch (p + 1))
  int ll_mask = 1;                    // tagged partials (RAC_EN_LL bit 1; EnChainArgs::ll_mask)
  bool fuse = false;                  // fused S phase (EnChainArgs::fuse; RAC_EN_LL bit 8, on by default)
  int hist_cap = 0;
  // device buffers
  double *Xc = nullptr, *y = nullptr, *c = nullptr, *beta = nullptr, *z = nullptr, *xi = nullptr,
         *r = nullptr;
  int32_t* idx = nullptr;     // [p][s]
  int32_t* order = nullptr;   // [p] (RP)
  double *gram_ws = nullptr, *scratch = nullptr, *inv = nullptr;
  int32_t* info = nullptr;
  double *partial = nullptr, *rhs = nullptr, *delta = nullptr, *wsum = nullptr, *wmax = nullptr;
  unsigned* bar = nullptr;
  int32_t* ctrl = nullptr;
  double *hist_p = nullptr, *hist_d = nullptr;
  std::vector<void*> allocs;
  // Sweep pipeline (RAC): the block systems of sweep k+1 (sort, Gram, inverses) only
  // depend on the permutation, so they are prepared on a low-priority stream while
  // the chain of sweep k runs on a high-priority one; idx/inv/info are double-buffered.
  bool pipe = false;
  cudaStream_t sprep = nullptr, schain = nullptr;
  cudaEvent_t ev_start = nullptr, ev_end = nullptr, ev_prep[2] = {nullptr, nullptr},
              ev_chain[2] = {nullptr, nullptr}, ev_gram = nullptr;
  bool look_gram = false;     // block mode: gram(k+1) before chain(k), factor(k+1) beside it (RAC_EN_LOOKGRAM=1;
                              // measured no faster on config 5)
  bool chain_rec[2] = {false, false};
  int32_t* idx_b[2] = {nullptr, nullptr};
  double* inv_b[2] = {nullptr, nullptr};
  int32_t* info_b[2] = {nullptr, nullptr};
  // covariance mode (en_cov.cuh): G = X'X/m formed once, chain on G in one cluster
  int gram_mode = 0;          // 0: per-sweep block Grams from X; 1: covariance
  bool have_G = false;
  int cov_k = 16;
  int cov_full = 0;           // whole inverse per CTA (en_cov.cuh full_inv)
  double *G = nullptr, *q = nullptr, *q2 = nullptr, *cwsum = nullptr, *cwmax = nullptr;
  int32_t* G_ids = nullptr;   // 0..n-1 (the single "block" of the full Gram)
  double* G_ws = nullptr;     // split-K partials of G
  size_t G_ws_cap = 0;
  void* i8_ws = nullptr;      // digit slices of the tensor-core Gram (gram_i8.cu), null = DMMA Gram
  size_t i8_ws_cap = 0;
  int64_t g_rows_done = 0;    // row-chunk ingest: samples already summed into G
  void* bg_ws = nullptr;      // block mode: per-sweep digit slices of the int8 block Grams, null = DMMA
  size_t bg_cap = 0;
  int* ex_all = nullptr;      // block mode: per-feature exponents of Xc (set with the data)
  int* i8_bad = nullptr;      // raised by the exponent passes when a column's max/rms makes the int8
                              // digit slices lose FP64-level accuracy (then: DMMA Grams for this data)
  bool i8_checked = true;
  bool i8_off = false;        // this data set's Grams on the DMMA tiles (set from i8_bad)
  int32_t* h_ctrl = nullptr;  // pinned: ctrl snapshot after each run (2 slots), for rac_en_poll
  cudaEvent_t ev_ctrl[2] = {nullptr, nullptr};
  int64_t ctrl_n = 0;         // runs snapshotted
  // lookahead covariance chain (en_cla.cuh); cla_L = leader cluster size, 0 = not used
  int cla_L = 0, cla_D = 3, cla_W = 0, cla_segw = 1, cla_R = 2, cla_NS = 2;
  size_t cla_smem = 0;
  double* T = nullptr;        // [p][D][s][s] tiles of the current sweep
  double* T_b[2] = {nullptr, nullptr};
  unsigned long long *dpub = nullptr, *qst = nullptr;   // [cla_B p][s][2] tagged messages (delta, base)
  double* snap = nullptr;     // [cla_B][3][n] per-sweep beta/z/xi (speculative sweeps after convergence)
  int32_t* conv = nullptr;    // [2] launch's first sweep, converged sweep within it
  unsigned* ccnt = nullptr;   // [CLA_BMAX] per-sweep commit counters of one launch
  // batched preparation (pipelined RAC): the block systems and tiles of cla_B sweeps are
  // formed by one launch on the prep stream, ring of 2 batches
  int cla_B = 1, batch_ctr = 0;
  int32_t *idx_r = nullptr, *info_r = nullptr;
  double *inv_r = nullptr, *T_r = nullptr;
  // optional per-stage CUDA-event timing: [assembly, gram, factor, chain]
  bool timing = false;
  std::vector<cudaEvent_t> events;  // 5 per timed sweep
  std::vector<cudaEvent_t> slice_events;   // int8 block Grams: after the slicing pass, one per timed sweep
  double slice_ms = 0.0;                    // summed by rac_en_timing, read by rac_en_timing_slicing
  long long* trace = nullptr;       // phase timestamps of the last traced sweep (chain | factor)
  long long* trace_buf = nullptr;
};

namespace {

template <typename T>
int dalloc(rac_en_ctx* c, T** p, size_t count) {
  if (count == 0) count = 1;
  void* q = nullptr;
  const int rc = rac::dev_alloc(&q, count * sizeof(T), c->st);
  if (rc) return rc;
  c->allocs.push_back(q);
  // zero-filled: the chains read padding entries (tiles of absent lookahead steps, short
  // last blocks) that are multiplied by zero and must therefore be finite
  cudaMemsetAsync(q, getenv("RAC_POISON") ? 0xff : 0, count * sizeof(T), c->st);
  *p = (T*)q;
  return RAC_OK;
}

void* res_kernel(int cs) {
  return cs == 8 ? (void*)rac::en_chain_res_kernel<8>
                 : (cs == 4 ? (void*)rac::en_chain_res_kernel<4> : (void*)rac::en_chain_res_kernel<2>);
}

size_t res_smem(int cs, int s, int nch, int p) {
  return cs == 8 ? rac::res_smem_bytes<8>(s, nch, p)
                 : (cs == 4 ? rac::res_smem_bytes<4>(s, nch, p) : rac::res_smem_bytes<2>(s, nch, p));
}

size_t en_chain_smem(int s, int RC) {
  size_t d = RC == 32 ? rac::RowPhase<32>::smem_doubles(s)
                      : (RC == 16 ? rac::RowPhase<16>::smem_doubles(s) : rac::RowPhase<8>::smem_doubles(s));
  return d * sizeof(double) + 2 * s * sizeof(int32_t);
}

int en_grow_history(rac_en_ctx* c, int need) {
  if (need <= c->hist_cap) return RAC_OK;
  int cap = std::max(need, std::max(64, 2 * c->hist_cap));
  double *hp = nullptr, *hd = nullptr;
  int rc = dalloc(c, &hp, cap);
  if (rc) return rc;
  rc = dalloc(c, &hd, cap);
  if (rc) return rc;
  if (c->hist_cap) {
    cudaMemcpyAsync(hp, c->hist_p, c->hist_cap * sizeof(double), cudaMemcpyDeviceToDevice, c->st);
    cudaMemcpyAsync(hd, c->hist_d, c->hist_cap * sizeof(double), cudaMemcpyDeviceToDevice, c->st);
  }
  c->hist_p = hp;
  c->hist_d = hd;
  c->hist_cap = cap;
  return RAC_OK;
}

void* cov_kernel(int k) { return k == 16 ? (void*)rac::en_cov_kernel<16> : (void*)rac::en_cov_kernel<8>; }

size_t cov_smem(int k, int s, int64_t n, int p, int full) {
  return k == 16 ? rac::cov_smem_bytes<16>(s, n, p, full) : rac::cov_smem_bytes<8>(s, n, p, full);
}

// largest cluster size (16, else 8) whose single-cluster chain fits, preferring
// the whole-inverse-per-CTA form (one cluster barrier per block) when it fits;
// returns k * 2 + full, or 0 if nothing fits
int cov_plan(int s, int64_t n, int p) {
  const char* env = getenv("RAC_COV_FULL");
  const bool allow_full = !(env && atoi(env) == 0);
  for (int full : {1, 0})
  for (int k : {16, 8}) {
    if (full && !allow_full) continue;
    const size_t smem = cov_smem(k, s, n, p, full);
    if (smem > 226 * 1024) continue;
    void* kf = cov_kernel(k);
    if (cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess ||
        (k > 8 && cudaFuncSetAttribute(kf, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)) {
      cudaGetLastError();
      continue;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(k);
    cfg.blockDim = dim3(rac::COVT);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = k;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int clusters = 0;
    if (cudaOccupancyMaxActiveClusters(&clusters, kf, &cfg) == cudaSuccess && clusters >= 1) return k * 2 + full;
    cudaGetLastError();
  }
  return 0;
}

volatile long long* g_cla_dbg = nullptr;   // rac_debug_buffer (mapped host memory)

void* cla_kernel(int L) { return L == 16 ? (void*)rac::en_cla_kernel<16> : (void*)rac::en_cla_kernel<8>; }

// Lookahead chain plan: leader cluster L (8, else 16) with at most 32 rows per
// rank, tile slots NS (4 if they fit, else 2), workers owning 32-column segments
// of q, G-row ring R; the whole grid (L + W CTAs, a multiple of L) must be
// co-resident.  Needs even s and n (16-byte TMA granules).  Returns false if
// nothing fits.
bool cla_plan(rac_en_ctx* c) {
  using namespace rac;
  const char* env = getenv("RAC_COV_LA");
  if (env && atoi(env) == 0) return false;
  const int s = c->s;
  const int64_t n = c->n;
  if ((s & 1) || (n & 1) || s > 256 || n > 20000) return false;
  const char* envd = getenv("RAC_CLA_D");
  const int Dwant = envd ? std::max(1, std::min(CLA_DMAX, atoi(envd))) : 3;
  const int nseg = (int)((n + 31) / 32);
  const size_t lim = 226 * 1024;
  for (int L : {8, 16}) {
    const int sl = (s + L - 1) / L;
    if (sl > 16) continue;   // main warps hold 16 rows of the step's operands in registers
    // deepest lookahead (then most tile slots) whose leader tiles fit in shared memory
    int NS = 0, D = 0;
    for (int dd = Dwant; dd >= 1 && !NS; --dd)
      for (int ns : {4, 2})
        if (cla_leader_doubles(L, s, dd, ns) * sizeof(double) <= lim) { NS = ns; D = dd; break; }
    if (!NS) continue;
    void* kf = cla_kernel(L);
    if ((L > 8 && cudaFuncSetAttribute(kf, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) ||
        cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lim) != cudaSuccess) {
      cudaGetLastError();
      continue;
    }
    // co-resident clusters at the largest shared-memory footprint we may pick
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(L);
    cfg.blockDim = dim3(CLA_T);
    cfg.dynamicSmemBytes = lim;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = L;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int clusters = 0;
    if (cudaOccupancyMaxActiveClusters(&clusters, kf, &cfg) != cudaSuccess || clusters < 2) {
      cudaGetLastError();
      continue;
    }
    int wclusters = std::min(clusters - 1, (nseg + L - 1) / L);
    const int segw = (nseg + wclusters * L - 1) / (wclusters * L);
    // fewest worker clusters with the same segments per worker: the SMs they leave free
    // run the next sweeps' block factorisations
    wclusters = std::min(wclusters, (nseg + segw * L - 1) / (segw * L));
    const int W = wclusters * L;
    int R = 0;
    for (int r : {4, 3, 2})
      if (cla_worker_doubles(s, segw, r) * sizeof(double) <= lim) { R = r; break; }
    if (!R) continue;
    c->cla_L = L;
    c->cla_D = D;
    c->cla_W = W;
    c->cla_segw = segw;
    c->cla_R = R;
    c->cla_NS = NS;
    c->cla_smem = cla_smem_bytes(L, s, D, NS, segw, R);   // the attribute stays at `lim` (shared by contexts)
    return true;
  }
  return false;
}

int launch_cla_tiles(rac_en_ctx* c, cudaStream_t st, int sweeps = 1) {
  using namespace rac;
  if (!c->cla_L || c->p < 2) return RAC_OK;
  cla_tiles_kernel<<<c->p * c->cla_D * sweeps, 256, 0, st>>>(
      c->G, c->n, c->s, c->p, c->cla_D, c->idx, (c->mode == RAC_MODE_RP) ? c->order : nullptr, c->T, c->ctrl);
  note_launch();
  return check_launch("cla tiles");
}

// G = X'X/m (full, row-major) on the FP64 tensor cores, one K split (each tile
// pair writes its block and the mirror), then q = G beta
int en_compute_G(rac_en_ctx* c, cudaStream_t st) {
  using namespace rac;
  const int64_t n = c->n;
  GramPlan pl = plan_gram(c->m, (int)n, 1);
  int rc = RAC_OK;
  if (c->i8_ws && !c->i8_off) {
    // int8 tensor-core Gram in exact digit-slice arithmetic (FP64-level accuracy)
    if ((rc = launch_gram_i8(c->Xc, c->ld, c->m, (int)n, c->G, (double)c->m, 0, c->i8_ws, c->i8_ws_cap, st, c->i8_bad)) ||
        (rc = launch_gemv_rows(c->G, n, n, c->beta, c->q, st)))
      return rc;
    c->have_G = true;
    return check_launch("covariance Gram (int8 slices)");
  }
  // K split (better filled waves) when rac_en_set_gram_mode could reserve its workspace
  const size_t wsb = (size_t)pl.splits * n * n * sizeof(double);
  if (pl.splits > 1 && c->G_ws && c->G_ws_cap >= wsb) {
    if ((rc = launch_gram(c->Xc, c->ld, c->m, c->G_ids, nullptr, (int)n, 1, c->G_ws, pl, st, nullptr)) ||
        (rc = launch_gram_reduce_sym(c->G_ws, n, pl.splits, (double)c->m, c->G, st)))
      return rc;
  } else {
    pl.splits = 1;
    pl.chunk = (c->m + 31) / 32 * 32;
    if ((rc = launch_gram(c->Xc, c->ld, c->m, c->G_ids, nullptr, (int)n, 1, c->G, pl, st, nullptr, (double)c->m)))
      return rc;
  }
  rc = launch_gemv_rows(c->G, n, n, c->beta, c->q, st);
  if (rc) return rc;
  c->have_G = true;
  return check_launch("covariance Gram");
}

int en_factor(rac_en_ctx* c, cudaStream_t st, int sweeps = 1) {
  using namespace rac;
  SysArgs a{};
  if (c->gram_mode == 1) {
    a.H = c->G;          // sys_b = G[b, b] + gamma I (padding of a short last block -> identity)
    a.ldh = c->n;
    a.idx = c->idx;
    a.div = 1.0;
    a.mul = 1.0;
  } else {
    a.ws = c->gram_ws;
    a.splits = (c->bg_ws && !c->i8_off) ? 1 : c->gp.splits;   // the int8 block Grams are complete (one split)
    a.div = (double)c->m;
    a.mul = 1.0;
  }
  a.shift = c->gamma;
  a.s = c->s;
  a.inv = c->inv;
  a.scratch = c->scratch;
  a.info = c->info;
  a.done = c->ctrl;
  a.trace = c->trace ? c->trace + 8 + 16 * (size_t)c->p : nullptr;
  // `sweeps` consecutive partitions in idx / inv / info (batched preparation): the
  // kernel treats them as sweeps * p independent blocks
  int rc = launch_chol_system(a, c->p * sweeps, st);
  if (rc) return rc;
  // RAC: the lookahead chain's tiles G[b_t, b_{t-d}] depend on this sweep's blocks only
  if (c->gram_mode == 1 && c->mode == RAC_MODE_RAC) return launch_cla_tiles(c, st, sweeps);
  return RAC_OK;
}

// block mode: the p block Grams of the partition in c->idx into gram_ws — int8 tensor
// cores (exact digit slices, gram_i8.cu) when reserved, else the FP64 DMMA tiles
int en_block_gram(rac_en_ctx* c, cudaStream_t st, cudaEvent_t after_slicing = nullptr) {
  if (c->bg_ws && !c->i8_off)
    return rac::launch_gram_i8_blocks(c->Xc, c->ld, c->m, c->idx, c->s, c->p, c->ex_all, c->i8_bad, c->gram_ws,
                                      c->bg_ws, c->bg_cap, st, after_slicing);
  return rac::launch_gram(c->Xc, c->ld, c->m, c->idx, nullptr, c->s, c->p, c->gram_ws, c->gp, st, c->ctrl);
}

int en_block_systems(rac_en_ctx* c) {
  if (c->gram_mode != 1) {
    int rc = en_block_gram(c, c->st);
    if (rc) return rc;
  }
  return en_factor(c, c->st);
}

int en_chain_cla(rac_en_ctx* c, double tol, cudaStream_t st, int nsw) {
  using namespace rac;
  EnClaArgs a{};
  a.G = c->G;
  a.n = c->n;
  a.s = c->s;
  a.p = c->p;
  a.nsw = nsw;
  a.tag = ++c->msg_tag;
  a.snap = (nsw > 1 && tol >= 0.0) ? c->snap : nullptr;
  a.conv = c->conv;
  a.ccnt = c->ccnt;
  a.dbg = g_cla_dbg;
  cudaMemsetAsync(c->ccnt, 0, CLA_BMAX * sizeof(unsigned), st);
  a.idx = c->idx;
  a.order = (c->mode == RAC_MODE_RP) ? c->order : nullptr;
  a.inv = c->inv;
  a.T = c->T;
  a.info = c->info;
  a.c = c->c;
  a.beta = c->beta;
  a.z = c->z;
  a.xi = c->xi;
  a.q = c->q;
  a.dpub = c->dpub;
  a.qst = c->qst;
  a.ctrl = c->ctrl;
  a.gamma = c->gamma;
  a.thr = c->lam * c->alpha;
  a.den = (1.0 - c->alpha) * c->lam + c->gamma;
  a.tol = tol;
  a.sweep = c->sweeps;
  a.hist_p = c->hist_p;
  a.hist_d = c->hist_d;
  a.trace = c->trace;
  a.D = c->cla_D;
  a.W = c->cla_W;
  a.segw = c->cla_segw;
  a.R = c->cla_R;
  a.NS = c->cla_NS;
  void* args[] = {&a};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(c->cla_L + c->cla_W);
  cfg.blockDim = dim3(CLA_T);
  cfg.dynamicSmemBytes = c->cla_smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = c->cla_L;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeCooperative;
  at[1].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = profile_noncoop() ? 1 : 2;
  note_launch();
  int rc = check_cuda(cudaLaunchKernelExC(&cfg, cla_kernel(c->cla_L), args), "en_cla (cluster cooperative launch)");
  if (rc || !a.snap) return rc;
  cla_restore_kernel<<<std::max(1, std::min(num_sms(), (int)((c->n + 255) / 256))), 256, 0, st>>>(
      c->conv, c->sweeps, nsw, c->n, c->snap, c->beta, c->z, c->xi);
  note_launch();
  return check_launch("cla restore");
}

int en_chain_cov(rac_en_ctx* c, double tol, cudaStream_t st, int nsw = 1) {
  using namespace rac;
  if (c->cla_L) return en_chain_cla(c, tol, st, nsw);
  EnCovArgs a{};
  a.G = c->G;
  a.n = c->n;
  a.s = c->s;
  a.p = c->p;
  a.idx = c->idx;
  a.order = (c->mode == RAC_MODE_RP) ? c->order : nullptr;
  a.inv = c->inv;
  a.info = c->info;
  a.c = c->c;
  a.beta = c->beta;
  a.z = c->z;
  a.xi = c->xi;
  a.q = c->q;
  a.wsum = c->cwsum;
  a.wmax = c->cwmax;
  a.ctrl = c->ctrl;
  a.gamma = c->gamma;
  a.thr = c->lam * c->alpha;
  a.den = (1.0 - c->alpha) * c->lam + c->gamma;
  a.tol = tol;
  a.sweep = c->sweeps;
  a.hist_p = c->hist_p;
  a.hist_d = c->hist_d;
  a.trace = c->trace;
  a.q2 = c->q2;
  a.full_inv = c->cov_full;
  void* args[] = {&a};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(c->cov_k);
  cfg.blockDim = dim3(COVT);
  cfg.dynamicSmemBytes = cov_smem(c->cov_k, c->s, c->n, c->p, c->cov_full);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = c->cov_k;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaFuncSetAttribute(cov_kernel(c->cov_k), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cfg.dynamicSmemBytes);
  note_launch();
  return check_cuda(cudaLaunchKernelExC(&cfg, cov_kernel(c->cov_k), args), "en_cov (cluster launch)");
}

int en_chain(rac_en_ctx* c, double tol, cudaStream_t st, int nsw = 1) {
  using namespace rac;
  if (c->gram_mode == 1) return en_chain_cov(c, tol, st, nsw);
  cudaMemsetAsync(c->bar, 0, sizeof(unsigned), st);
  EnChainArgs a{};
  a.Xc = c->Xc;
  a.ld = c->ld;
  a.n = c->n;
  a.m = c->m;
  a.s = c->s;
  a.p = c->p;
  a.nrc = c->nrc;
  a.idx = c->idx;
  a.order = (c->mode == RAC_MODE_RP) ? c->order : nullptr;
  a.inv = c->inv;
  a.info = c->info;
  a.c = c->c;
  a.beta = c->beta;
  a.z = c->z;
  a.xi = c->xi;
  a.r = c->r;
  a.partial = c->partial;
  a.rhs = c->rhs;
  a.delta = c->delta;
  a.wsum = c->wsum;
  a.wmax = c->wmax;
  a.bar = c->bar;
  a.ctrl = c->ctrl;
  a.gamma = c->gamma;
  a.thr = c->lam * c->alpha;
  a.den = (1.0 - c->alpha) * c->lam + c->gamma;
  a.mdiv = (double)c->m;
  a.tol = tol;
  a.sweep = c->sweeps;
  a.hist_p = c->hist_p;
  a.hist_d = c->hist_d;
  a.trace = c->trace;
  a.rw = c->rw;
  if (c->ll && c->RC == 0 && c->variant != 1) {
    if ((unsigned long long)(c->ll_epoch + 2u) * (unsigned)(c->p + 1) >= 0xfffffff0ull) {
      // tag space used up (2^32 / (p + 1) launches): clear the words and start over
      const size_t nsc = (size_t)(c->s + ENT / 32 - 1) / (ENT / 32);
      cudaMemsetAsync(c->ll, 0,
                      2 * ((size_t)c->s * c->P + c->s * nsc) *
                          sizeof(unsigned long long), st);
      c->ll_epoch = 0;
    }
    ++c->ll_epoch;
    a.ll = c->ll;
    a.tag0 = c->ll_epoch * (unsigned)(c->p + 1);
    a.ll_mask = c->ll_mask;
    a.fuse = c->fuse ? 1 : 0;
    a.fuse_off = (unsigned)((row1t_smem_bytes(c->s, c->rw) + 15) / 16 * 16);
  }
  void* args[] = {&a};
  if (c->variant == 1) {
    int nch = c->nch;
    void* rargs[] = {&a, &nch};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(c->P);
    cfg.blockDim = dim3(ENT);
    cfg.dynamicSmemBytes = res_smem(c->cs, c->s, c->nch, c->p);
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = c->cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeCooperative;
    at[1].val.cooperative = 1;
    cfg.attrs = at;
    // Nsight Compute cannot replay a cooperative *cluster* launch; for profiling only,
    // RAC_PROFILE_NONCOOP=1 drops the cooperative attribute (the grid is one wave of
    // one CTA per SM either way, and ncu serialises kernels, so the barrier still holds).
    cfg.numAttrs = profile_noncoop() ? 1 : 2;
    // the function attribute is process-wide: another context's plan may have lowered it
    cudaFuncSetAttribute(res_kernel(c->cs), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cfg.dynamicSmemBytes);
    note_launch();
    return check_cuda(cudaLaunchKernelExC(&cfg, (const void*)res_kernel(c->cs), rargs),
                      "en_chain_res (cluster cooperative launch)");
  }
  size_t smem = c->RC == 0 ? row1t_smem_bytes(c->s, c->rw) : en_chain_smem(c->s, c->RC);
  if (c->RC == 0 && c->fuse) smem = (smem + 15) / 16 * 16 + (size_t)(ENT / 32) * c->s * sizeof(double);
  cudaError_t e;
  {
    // the function attribute is process-wide: another context's plan may have lowered it
    void* kf = c->RC == 0 ? (void*)en_chain_kernel<0>
                          : (c->RC == 32 ? (void*)en_chain_kernel<32>
                                         : (c->RC == 16 ? (void*)en_chain_kernel<16> : (void*)en_chain_kernel<8>));
    if (smem > 48 * 1024) cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  }
  if (c->RC == 0)
    e = launch_coop((void*)en_chain_kernel<0>, dim3(c->P), dim3(ENT), args, smem, st);
  else if (c->RC == 32)
    e = launch_coop((void*)en_chain_kernel<32>, dim3(c->P), dim3(ENT), args, smem, st);
  else if (c->RC == 16)
    e = launch_coop((void*)en_chain_kernel<16>, dim3(c->P), dim3(ENT), args, smem, st);
  else
    e = launch_coop((void*)en_chain_kernel<8>, dim3(c->P), dim3(ENT), args, smem, st);
  note_launch();
  return check_cuda(e, "en_chain (cooperative launch)");
}

}  // namespace

extern "C" int rac_en_create(rac_en_ctx** out, int64_t m, int64_t n, int32_t block_size,
                             int32_t mode, double lam, double alpha, double gamma, void* stream) {
  using namespace rac;
  clear_error();
  if (!out || m < 1 || n < 1 || block_size < 1 || !(gamma > 0) || lam < 0 || alpha < 0 || alpha > 1)
    return set_error(RAC_ERR_ARG, "rac_en_create: bad arguments");
  if (mode != RAC_MODE_RAC && mode != RAC_MODE_RP)
    return set_error(RAC_ERR_ARG, "rac_en_create: mode must be rac or rp");
  const int s = (int)std::min<int64_t>(block_size, n);
  if (s > EN_QMAX * ENT) return set_error(RAC_ERR_UNSUPPORTED, "block_size %d > %d", s, EN_QMAX * ENT);
  rac_en_ctx* c = new rac_en_ctx();
  c->m = m;
  c->n = n;
  c->ld = (m + 31) / 32 * 32;
  c->s = s;
  c->p = (int)((n + s - 1) / s);
  c->mode = mode;
  c->lam = lam;
  c->alpha = alpha;
  c->gamma = gamma;
  c->st = (cudaStream_t)stream;
  // rows per chunk: biggest that keeps the tile within ~110 KB of shared memory
  c->RC = (en_chain_smem(s, 32) <= 150 * 1024) ? 32 : (en_chain_smem(s, 16) <= 150 * 1024 ? 16 : 8);
  c->nrc = (int)((m + c->RC - 1) / c->RC);
  c->gp = plan_gram(m, s, c->p);
  int rc = RAC_OK;
  size_t smem = en_chain_smem(s, c->RC);
  void* kfn = (c->RC == 32) ? (void*)en_chain_kernel<32>
                            : (c->RC == 16 ? (void*)en_chain_kernel<16> : (void*)en_chain_kernel<8>);
  if ((rc = check_cuda(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                       "chain smem attribute"))) {
    delete c;
    return rc;
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, ENT, smem);
  if (per_sm < 1) {
    delete c;
    return set_error(RAC_ERR_UNSUPPORTED, "chain kernel does not fit (smem %zu)", smem);
  }
  c->P = std::max(1, std::min(num_sms(), c->nrc));
  // resident-tile cluster chain when the row tiles of every CTA fit in shared memory
  {
    const char* env = getenv("RAC_EN_VARIANT");
    const int want = env ? atoi(env) : 1;
    const int nrc32 = (int)((m + 31) / 32);
    const int pblocks = (int)((n + s - 1) / s);
    // the largest co-resident grid (multiple of cs) of the resident chain; false if it does not fit
    auto plan_res = [&](int cs, int* P_out, int* nch_out) -> bool {
      int Pc = std::max(cs, std::min(num_sms(), (nrc32 + cs - 1) / cs * cs) / cs * cs);
      void* rk = res_kernel(cs);
      if (Pc > 148 || cudaFuncSetAttribute(rk, cudaFuncAttributeNonPortableClusterSizeAllowed, 0) != cudaSuccess)
        return false;
      for (int tries = 0; tries < 4 && Pc >= cs; ++tries) {
        const int nch = (nrc32 + Pc - 1) / Pc;
        const size_t rs = res_smem(cs, s, nch, pblocks);
        if (rs > 226 * 1024 || cudaFuncSetAttribute(rk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rs) != cudaSuccess)
          return false;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(Pc);
        cfg.blockDim = dim3(ENT);
        cfg.dynamicSmemBytes = rs;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int clusters = 0;
        if (cudaOccupancyMaxActiveClusters(&clusters, rk, &cfg) != cudaSuccess) return false;
        if (clusters * cs >= Pc) {
          *P_out = Pc;
          *nch_out = nch;
          return true;
        }
        Pc = clusters * cs;
      }
      return false;
    };
    if (want == 1 && s <= ENT) {
      // cluster size: RAC_EN_CS if set; otherwise 8 (fewer partials to reduce per
      // block) unless it would give CTAs more row chunks than pairs do.
      const char* envcs = getenv("RAC_EN_CS");
      int P2 = 0, n2 = 0, P8 = 0, n8 = 0, Pe = 0, ne = 0;
      int pick = 0;
      if (envcs) {
        const int e = atoi(envcs);
        const int cs = (e >= 8) ? 8 : (e >= 4 ? 4 : 2);
        if (plan_res(cs, &Pe, &ne)) pick = cs;
      } else {
        const bool ok2 = plan_res(2, &P2, &n2);
        const bool ok8 = plan_res(8, &P8, &n8);
        if (ok8 && (!ok2 || n8 <= n2)) { pick = 8; Pe = P8; ne = n8; }
        else if (ok2) { pick = 2; Pe = P2; ne = n2; }
      }
      if (pick) {
        c->variant = 1;
        c->cs = pick;
        c->RC = 32;
        c->nrc = nrc32;
        c->nch = ne;
        c->P = Pe;
        cudaFuncSetAttribute(res_kernel(pick), cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)res_smem(pick, s, ne, pblocks));
      }
      cudaGetLastError();
    }
  }
  // streaming chain, one-tile resident row phase (RC == 0) when a CTA's contiguous rows
  // of one block fit in shared memory: every block's columns read once per sweep, no
  // row-chunk imbalance (RAC_EN_1T=0 keeps the chunked schedule)
  if (c->variant == 0) {
    const char* env = getenv("RAC_EN_1T");
    const int rw = (int)(((c->ld + num_sms() - 1) / num_sms() + 1) / 2 * 2);
    const size_t sm1 = row1t_smem_bytes(s, rw);
    if (!(env && atoi(env) == 0) && sm1 <= 200 * 1024 &&
        cudaFuncSetAttribute((void*)en_chain_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1) ==
            cudaSuccess) {
      cudaFuncSetAttribute((void*)en_chain_kernel<0>, cudaFuncAttributePreferredSharedMemoryCarveout,
                           cudaSharedmemCarveoutMaxShared);
      c->RC = 0;
      c->rw = rw;
      c->P = (int)((c->ld + rw - 1) / rw);
    }
    cudaGetLastError();
  }
  const int GW = c->P * (ENT / 32);
  const size_t sqs = (size_t)c->p * s * s;
  if ((rc = dalloc(c, &c->Xc, (size_t)c->ld * n)) || (rc = dalloc(c, &c->c, n)) ||
      (rc = dalloc(c, &c->beta, n)) || (rc = dalloc(c, &c->z, n)) || (rc = dalloc(c, &c->xi, n)) ||
      (rc = dalloc(c, &c->r, c->ld)) || (rc = dalloc(c, &c->idx, (size_t)c->p * s)) ||
      (rc = dalloc(c, &c->order, c->p)) ||
      (rc = dalloc(c, &c->gram_ws, gram_ws_bytes(m, s, c->p) / sizeof(double))) ||
      (rc = dalloc(c, &c->inv, sqs)) || (rc = dalloc(c, &c->info, c->p)) ||
      (rc = dalloc(c, &c->partial, (size_t)c->P * s)) || (rc = dalloc(c, &c->rhs, s)) || (rc = dalloc(c, &c->i8_bad, 1)) ||
      (rc = dalloc(c, &c->delta, s)) || (rc = dalloc(c, &c->wsum, GW)) ||
      (rc = dalloc(c, &c->wmax, GW)) || (rc = dalloc(c, &c->bar, 1)) || (rc = dalloc(c, &c->ctrl, 4))) {
    rac_en_destroy(c);
    return rc;
  }
  if (c->RC == 0 && c->P <= 256) {
    // RAC_EN_LL: 1 tagged partials, + 8 the fused S phase (default 9); 0: three grid barriers per block
    const char* e = getenv("RAC_EN_LL");
    int want_fuse = 1;
    if (e) {
      c->ll_mask = atoi(e) & 1;
      want_fuse = (atoi(e) & 8) ? 1 : 0;
    }
    const int nsc = (s + ENT / 32 - 1) / (ENT / 32);
    if (c->ll_mask != 0 &&
        (rc = dalloc(c, &c->ll, 2 * ((size_t)s * c->P + (size_t)s * nsc)))) {
      rac_en_destroy(c);
      return rc;
    }
    const size_t smf = (row1t_smem_bytes(s, c->rw) + 15) / 16 * 16 + (size_t)(ENT / 32) * s * sizeof(double);
    if (want_fuse && (c->ll_mask & 1) && s <= 512 && c->P * (ENT / 32) >= s && smf <= 200 * 1024 &&
        cudaFuncSetAttribute((void*)en_chain_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smf) ==
            cudaSuccess)
      c->fuse = true;
    cudaGetLastError();
  }
  {
    // int8 tensor-core block Grams when a sweep's 128 x 128 tiles fill the SMs several times
    // (RAC_BG_I8=2 forces them, =0 keeps the DMMA tiles)
    const char* e8 = getenv("RAC_BG_I8");
    const int mode8 = e8 ? atoi(e8) : 1;
    const int64_t jt = (s + 127) / 128;
    const int64_t tiles = (int64_t)c->p * jt * (jt + 1) / 2;
    if (mode8 == 2 || (mode8 == 1 && s >= 128 && tiles >= 4 * (int64_t)num_sms())) {
      const size_t need = gram_i8_blocks_ws_bytes(c->ld, s, c->p);
      uint8_t* w = nullptr;
      if (dalloc(c, &w, need) == RAC_OK && dalloc(c, &c->ex_all, n) == RAC_OK) {
        c->bg_ws = w;
        c->bg_cap = need;
      } else {
        cudaGetLastError();
        clear_error();
      }
    }
  }
  size_t scr = chol_scratch_bytes(s, c->p);
  if (scr && (rc = dalloc(c, &c->scratch, scr / sizeof(double)))) {
    rac_en_destroy(c);
    return rc;
  }
  c->idx_b[0] = c->idx;
  c->inv_b[0] = c->inv;
  c->info_b[0] = c->info;
  {
    const char* env = getenv("RAC_EN_PIPE");
    c->pipe = (mode == RAC_MODE_RAC) && !(env && atoi(env) == 0);
  }
  if (c->pipe) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    if ((rc = dalloc(c, &c->idx_b[1], (size_t)c->p * s)) || (rc = dalloc(c, &c->inv_b[1], sqs)) ||
        (rc = dalloc(c, &c->info_b[1], c->p)) ||
        (rc = check_cuda(cudaStreamCreateWithPriority(&c->sprep, cudaStreamNonBlocking, lo), "prep stream")) ||
        (rc = check_cuda(cudaStreamCreateWithPriority(&c->schain, cudaStreamNonBlocking, hi), "chain stream"))) {
      rac_en_destroy(c);
      return rc;
    }
    cudaEvent_t* evs[] = {&c->ev_start, &c->ev_end, &c->ev_prep[0], &c->ev_prep[1], &c->ev_chain[0], &c->ev_chain[1],
                          &c->ev_gram};
    if (const char* el = getenv("RAC_EN_LOOKGRAM")) c->look_gram = atoi(el) != 0;
    for (cudaEvent_t* e : evs)
      if ((rc = check_cuda(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "pipeline event"))) {
        rac_en_destroy(c);
        return rc;
      }
    cudaMemsetAsync(c->info_b[1], 0, c->p * sizeof(int32_t), c->st);
  }
  if ((rc = en_grow_history(c, 256))) {
    rac_en_destroy(c);
    return rc;
  }
  cudaMemsetAsync(c->beta, 0, n * sizeof(double), c->st);
  cudaMemsetAsync(c->z, 0, n * sizeof(double), c->st);
  cudaMemsetAsync(c->xi, 0, n * sizeof(double), c->st);
  cudaMemsetAsync(c->r, 0, c->ld * sizeof(double), c->st);
  cudaMemsetAsync(c->ctrl, 0, 4 * sizeof(int32_t), c->st);
  cudaMemsetAsync(c->info, 0, c->p * sizeof(int32_t), c->st);
  rc = check_launch("rac_en_create");
  if (rc) {
    rac_en_destroy(c);
    return rc;
  }
  if (cudaHostAlloc((void**)&c->h_ctrl, 8 * sizeof(int32_t), cudaHostAllocDefault) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_ctrl[0], cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_ctrl[1], cudaEventDisableTiming) != cudaSuccess) {
    rac_en_destroy(c);
    return set_error(RAC_ERR_CUDA, "rac_en_create: pinned control snapshot");
  }
  *out = c;
  return RAC_OK;
}

namespace rac {
// CSC (canonical: sorted, no duplicate entries) -> the column-major Xc: one warp per column
// scatters its stored entries into the zeroed column (a block's columns are then exactly
// what the reference's X[:, block].todense() gives, elastic_net.py:144-147)
__global__ void csc_scatter_kernel(const int64_t* __restrict__ indptr, const int32_t* __restrict__ rows,
                                   const double* __restrict__ vals, int64_t n, int64_t ld, double* __restrict__ Xc) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t j = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; j < n; j += nw) {
    double* col = Xc + j * ld;
    for (int64_t k = indptr[j] + lane; k < indptr[j + 1]; k += 32) col[rows[k]] = vals[k];
  }
}
}  // namespace rac

// Sparse X: the nnz stored entries travel (12 bytes each instead of 8 m n for the dense
// matrix) and are expanded on the device; everything after is the dense block path.
extern "C" int rac_en_set_data_csc(rac_en_ctx* c, const int64_t* indptr, const int32_t* rows, const double* vals,
                                   const double* y) {
  using namespace rac;
  clear_error();
  if (!c || !indptr || !y || (!rows && vals) || (rows && !vals))
    return set_error(RAC_ERR_ARG, "rac_en_set_data_csc: null pointer");
  cudaMemsetAsync(c->Xc, 0, (size_t)c->ld * c->n * sizeof(double), c->st);
  if (rows) {
    const int blocks = (int)std::min<int64_t>((c->n + 7) / 8, (int64_t)num_sms() * 16);
    csc_scatter_kernel<<<blocks, 256, 0, c->st>>>(indptr, rows, vals, c->n, c->ld, c->Xc);
    note_launch();
  }
  int blocks = (int)std::min<int64_t>((c->n + 7) / 8, (int64_t)num_sms() * 16);
  note_launch();
  neg_xty_kernel<<<blocks, 256, 0, c->st>>>(c->Xc, c->ld, c->m, c->n, y, (double)c->m, c->c);
  cudaMemsetAsync(c->i8_bad, 0, sizeof(int), c->st);
  c->i8_checked = false;
  c->i8_off = false;
  if (c->bg_ws) {
    int rc = launch_i8_colexp(c->Xc, c->ld, c->m, (int)c->n, c->ex_all, c->st, c->i8_bad);
    if (rc) return rc;
  }
  c->have_data = true;
  return check_launch("rac_en_set_data_csc");
}

extern "C" int rac_en_set_data(rac_en_ctx* c, const double* X, int32_t layout, const double* y) {
  using namespace rac;
  clear_error();
  if (!c || !X || !y) return set_error(RAC_ERR_ARG, "rac_en_set_data: null pointer");
  if (layout == RAC_LAYOUT_ROW_MAJOR) {
    int rc = launch_transpose_pad(X, c->m, c->n, c->ld, c->Xc, c->st);
    if (rc) return rc;
  } else if (layout == RAC_LAYOUT_COL_MAJOR) {
    cudaMemcpy2DAsync(c->Xc, c->ld * sizeof(double), X, c->m * sizeof(double), c->m * sizeof(double),
                      c->n, cudaMemcpyDeviceToDevice, c->st);
    if (c->ld > c->m)
      cudaMemset2DAsync(c->Xc + c->m, c->ld * sizeof(double), 0, (c->ld - c->m) * sizeof(double), c->n,
                        c->st);
  } else {
    return set_error(RAC_ERR_ARG, "rac_en_set_data: unknown layout %d", layout);
  }
  int blocks = (int)std::min<int64_t>((c->n + 7) / 8, (int64_t)num_sms() * 16);
  note_launch();
  neg_xty_kernel<<<blocks, 256, 0, c->st>>>(c->Xc, c->ld, c->m, c->n, y, (double)c->m, c->c);
  cudaMemsetAsync(c->i8_bad, 0, sizeof(int), c->st);
  c->i8_checked = false;
  c->i8_off = false;
  if (c->bg_ws) {
    int rc = launch_i8_colexp(c->Xc, c->ld, c->m, (int)c->n, c->ex_all, c->st, c->i8_bad);
    if (rc) return rc;
  }
  c->have_data = true;
  return check_launch("rac_en_set_data");
}

extern "C" int rac_en_set_data_rows(rac_en_ctx* c, const double* X_rows, int64_t row0, int64_t rows,
                                    const double* y) {
  using namespace rac;
  clear_error();
  if (!c || !X_rows || rows < 1 || row0 < 0 || row0 + rows > c->m || (row0 % 32) != 0)
    return set_error(RAC_ERR_ARG, "rac_en_set_data_rows: bad arguments");
  const bool last = (row0 + rows == c->m);
  if (!last && (rows % 32) != 0) return set_error(RAC_ERR_ARG, "rac_en_set_data_rows: rows must be a multiple of 32");
  if (last && !y) return set_error(RAC_ERR_ARG, "rac_en_set_data_rows: the last chunk needs y");
  if (row0 == 0) {
    c->have_data = false;
    c->have_G = false;
    cudaMemsetAsync(c->i8_bad, 0, sizeof(int), c->st);
    c->i8_checked = false;
  c->i8_off = false;
    c->g_rows_done = 0;
    if (c->gram_mode == 1) cudaMemsetAsync(c->G, 0, (size_t)c->n * c->n * sizeof(double), c->st);
  }
  const int64_t rows_out = last ? (c->ld - row0) : rows;
  dim3 grid((unsigned)((c->n + 31) / 32), (unsigned)((rows_out + 31) / 32));
  if (grid.y > 65535) return set_error(RAC_ERR_UNSUPPORTED, "rac_en_set_data_rows: chunk too tall");
  static bool carve = false;
  if (!carve) {
    // co-reside with the int8 Gram pieces (198 KB of shared memory per CTA) on the prep stream
    cudaFuncSetAttribute(transpose_rows_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                         cudaSharedmemCarveoutMaxShared);
    carve = true;
  }
  transpose_rows_kernel<<<grid, dim3(32, 8), 0, c->st>>>(X_rows, rows, c->n, c->ld, row0, rows_out, c->Xc);
  note_launch();
  int rc = check_launch("transpose_rows");
  if (rc) return rc;
  if (c->gram_mode == 1) {
    // G += X_chunk' X_chunk on the column-major rows just written (len rounded up to 32:
    // the zero padding of the last chunk, or rows that are a multiple of 32)
    const int64_t len = (rows + 31) / 32 * 32;
    GramPlan pl = plan_gram(len, (int)c->n, 1);
    pl.splits = 1;
    pl.chunk = len;
    if (c->i8_ws) {
      // tensor-core Gram over pieces of >= 4096 samples (full tiles' worth of K per launch),
      // each overlapping the transfer of the following chunks
      const int64_t done = c->g_rows_done, upto = row0 + rows;
      if (last || upto - done >= 4096) {
        const int64_t plen = last ? (c->m - done) : (upto - done);
        // on the prep stream, so the transposes of the next chunks (c->st) keep draining
        // the staging ring while the piece runs
        cudaStream_t gs = c->sprep ? c->sprep : c->st;
        if (gs != c->st) {
          cudaEventRecord(c->ev_start, c->st);
          cudaStreamWaitEvent(gs, c->ev_start, 0);
        }
        rc = launch_gram_i8(c->Xc + done, c->ld, plen, (int)c->n, c->G, 0.0, 1, c->i8_ws, c->i8_ws_cap, gs, c->i8_bad);
        c->g_rows_done = upto;
        if (last && gs != c->st) {
          cudaEventRecord(c->ev_end, gs);
          cudaStreamWaitEvent(c->st, c->ev_end, 0);
        }
      }
    } else {
      rc = launch_gram(c->Xc + row0, c->ld, len, c->G_ids, nullptr, (int)c->n, 1, c->G, pl, c->st, nullptr, 0.0, 1);
    }
    if (rc) return rc;
  }
  if (!last) return RAC_OK;
  int blocks = (int)std::min<int64_t>((c->n + 7) / 8, (int64_t)num_sms() * 16);
  note_launch();
  neg_xty_kernel<<<blocks, 256, 0, c->st>>>(c->Xc, c->ld, c->m, c->n, y, (double)c->m, c->c);
  if (c->bg_ws && (rc = launch_i8_colexp(c->Xc, c->ld, c->m, (int)c->n, c->ex_all, c->st, c->i8_bad))) return rc;
  if (c->gram_mode == 1) {
    scale_kernel<<<num_sms() * 8, 256, 0, c->st>>>(c->G, c->n * c->n, (double)c->m);   // dot, then / m
    note_launch();
    rc = launch_gemv_rows(c->G, c->n, c->n, c->beta, c->q, c->st);
    if (rc) return rc;
    c->have_G = true;
  }
  c->have_data = true;
  return check_launch("rac_en_set_data_rows");
}

extern "C" int rac_en_set_gram_mode(rac_en_ctx* c, int32_t mode) {
  using namespace rac;
  clear_error();
  if (!c || (mode != RAC_GRAM_BLOCKS && mode != RAC_GRAM_COVARIANCE))
    return set_error(RAC_ERR_ARG, "rac_en_set_gram_mode: bad arguments");
  c->have_G = false;
  c->have_partition = false;   // RP block systems must be re-formed
  if (mode == RAC_GRAM_BLOCKS) {
    c->gram_mode = 0;
    return RAC_OK;
  }
  const int plan = cov_plan(c->s, c->n, c->p);
  const int k = plan / 2;
  if (!k) return set_error(RAC_ERR_UNSUPPORTED, "covariance mode does not fit (n=%lld, s=%d)", (long long)c->n, c->s);
  int rc = RAC_OK;
  if (!c->G) {
    if ((rc = dalloc(c, &c->G, (size_t)c->n * c->n)) || (rc = dalloc(c, &c->q, c->n)) ||
        (rc = dalloc(c, &c->q2, c->n)) ||
        (rc = dalloc(c, &c->cwsum, 16)) || (rc = dalloc(c, &c->cwmax, 16)) || (rc = dalloc(c, &c->G_ids, c->n)))
      return rc;
    iota_kernel<<<(int)std::min<int64_t>((c->n + 255) / 256, 4096), 256, 0, c->st>>>(c->G_ids, c->n);
    note_launch();
  }
  c->cov_k = k;
  c->cov_full = plan & 1;
  c->gram_mode = 1;
  {
    // digit-slice workspace of the int8 tensor-core Gram (RAC_G_I8=0: the FP64 DMMA Gram)
    // (used when its 128 x 64 output tiles fill the SMs; RAC_G_I8=2 forces it, =0 disables it)
    const char* e8 = getenv("RAC_G_I8");
    const int mode8 = e8 ? atoi(e8) : 1;
    const int64_t kt = (c->n + 63) / 64;
    int64_t tiles = 0;
    for (int64_t J = 0; 2 * J < kt; ++J) tiles += kt - 2 * J;
    const size_t need = gram_i8_ws_bytes(c->ld, (int)c->n);
    if ((mode8 == 2 || (mode8 == 1 && tiles >= num_sms())) && c->i8_ws_cap < need) {
      uint8_t* w = nullptr;
      if (dalloc(c, &w, need) == RAC_OK) {
        c->i8_ws = w;
        c->i8_ws_cap = need;
      } else {
        cudaGetLastError();
        clear_error();
      }
    }
  }
  if (!c->i8_ws) {
    // split-K workspace of G (en_compute_G), reserved here so no fit allocates in its sweep loop
    const GramPlan pl = plan_gram(c->m, (int)c->n, 1);
    const size_t wsb = (size_t)pl.splits * c->n * c->n * sizeof(double);
    const char* env = getenv("RAC_G_SPLIT");
    if (pl.splits > 1 && wsb <= ((size_t)1 << 30) && !(env && atoi(env) == 0) && c->G_ws_cap < wsb) {
      double* w = nullptr;
      if (dalloc(c, &w, wsb / sizeof(double)) == RAC_OK) {
        c->G_ws = w;
        c->G_ws_cap = wsb;
      } else {
        cudaGetLastError();
        clear_error();
      }
    }
  }
  if (!c->cla_L && cla_plan(c)) {
    const size_t tq = (size_t)c->p * c->cla_D * c->s * c->s;
    if ((rc = dalloc(c, &c->T_b[0], tq)) || (c->pipe && (rc = dalloc(c, &c->T_b[1], tq)))) {
      c->cla_L = 0;
      return rc;
    }
    if (c->pipe) {
      // sweeps per preparation batch: the factor CTAs (one per block) of a batch should fit
      // on the SMs the chain leaves free
      const int free_sms = std::max(0, num_sms() - (c->cla_L + c->cla_W));
      c->cla_B = std::max(1, std::min(CLA_BMAX, free_sms / std::max(1, c->p)));
      if (const char* eb = getenv("RAC_CLA_B")) c->cla_B = std::max(1, std::min(CLA_BMAX, atoi(eb)));
      // the factor's global scratch (Cholesky re-check / large-s path) must cover the batch
      const size_t scr = chol_scratch_bytes(c->s, c->p * c->cla_B);
      if (c->cla_B > 1 && scr > chol_scratch_bytes(c->s, c->p)) {
        double* w = nullptr;
        if ((rc = dalloc(c, &w, scr / sizeof(double)))) c->cla_B = 1;
        else c->scratch = w;
        cudaGetLastError();
        clear_error();
        rc = RAC_OK;
      }
      const int nb = 2 * c->cla_B;
      if ((rc = dalloc(c, &c->idx_r, (size_t)nb * c->p * c->s)) || (rc = dalloc(c, &c->info_r, (size_t)nb * c->p)) ||
          (rc = dalloc(c, &c->inv_r, (size_t)nb * c->p * c->s * c->s)) || (rc = dalloc(c, &c->T_r, (size_t)nb * tq))) {
        c->cla_L = 0;
        return rc;
      }
      cudaMemsetAsync(c->info_r, 0, (size_t)nb * c->p * sizeof(int32_t), c->st);
    }
    // tagged message slots for every global step of one launch (cla_B sweeps), snapshots
    const size_t ps = (size_t)c->cla_B * c->p * c->s;
    if ((rc = dalloc(c, &c->dpub, ps * 2)) || (rc = dalloc(c, &c->qst, ps * 2)) || (rc = dalloc(c, &c->conv, 2)) ||
        (rc = dalloc(c, &c->ccnt, CLA_BMAX)) ||
        (c->cla_B > 1 && (rc = dalloc(c, &c->snap, (size_t)c->cla_B * 3 * c->n)))) {
      c->cla_L = 0;
      return rc;
    }
    cudaMemsetAsync(c->dpub, 0, ps * 2 * sizeof(unsigned long long), c->st);
    cudaMemsetAsync(c->qst, 0, ps * 2 * sizeof(unsigned long long), c->st);
    cudaMemsetAsync(c->conv, 0xff, 2 * sizeof(int32_t), c->st);
    c->T = c->T_b[0];
  }
  return RAC_OK;
}

extern "C" int rac_en_set_partition(rac_en_ctx* c, const int64_t* perm) {
  using namespace rac;
  clear_error();
  if (!c || !perm) return set_error(RAC_ERR_ARG, "rac_en_set_partition: null pointer");
  if (c->mode != RAC_MODE_RP) return set_error(RAC_ERR_ARG, "rac_en_set_partition: mode is not rp");
  if (!c->have_data) return set_error(RAC_ERR_ARG, "rac_en_set_partition: call rac_en_set_data first");
  int rc = RAC_OK;
  if (c->gram_mode == 1 && !c->have_G && (rc = en_compute_G(c, c->st))) return rc;
  rc = launch_chunk_sort(perm, c->n, c->s, 1, c->idx, c->st);
  if (rc) return rc;
  rc = en_block_systems(c);
  if (rc) return rc;
  c->have_partition = true;
  return RAC_OK;
}

static int en_run(rac_en_ctx* c, const int64_t* perms, int32_t count, double tol);

extern "C" int rac_en_run(rac_en_ctx* c, const int64_t* perms, int32_t count, double tol) {
  const int rc = en_run(c, perms, count, tol);
  if (rc == RAC_OK && c->h_ctrl) {
    // snapshot of the control word once this run's work is done (rac_en_poll)
    const int slot = (int)(c->ctrl_n & 1);
    cudaMemcpyAsync(c->h_ctrl + 4 * slot, c->ctrl, 4 * sizeof(int32_t), cudaMemcpyDeviceToHost, c->st);
    cudaEventRecord(c->ev_ctrl[slot], c->st);
    c->ctrl_n++;
  }
  return rc;
}

extern "C" int rac_en_poll(rac_en_ctx* c, int32_t lag, int32_t* iterations, int32_t* converged,
                           int32_t* failed_block) {
  using namespace rac;
  clear_error();
  if (!c || lag < 0 || lag > 1 || c->ctrl_n - 1 - lag < 0)
    return set_error(RAC_ERR_ARG, "rac_en_poll: no such run");
  const int slot = (int)((c->ctrl_n - 1 - lag) & 1);
  int rc = check_cuda(cudaEventSynchronize(c->ev_ctrl[slot]), "poll");
  if (rc) return rc;
  const int32_t* h = c->h_ctrl + 4 * slot;
  if (iterations) *iterations = h[1];
  if (converged) *converged = h[3];
  if (failed_block) *failed_block = h[2] - 1;
  return RAC_OK;
}

static int en_run(rac_en_ctx* c, const int64_t* perms, int32_t count, double tol) {
  using namespace rac;
  clear_error();
  if (!c || (!perms && count > 0) || count < 0) return set_error(RAC_ERR_ARG, "rac_en_run: bad arguments");
  if (!c->have_data) return set_error(RAC_ERR_ARG, "rac_en_run: call rac_en_set_data first");
  if (c->mode == RAC_MODE_RP && !c->have_partition)
    return set_error(RAC_ERR_ARG, "rac_en_run: rp mode needs rac_en_set_partition");
  int rc = en_grow_history(c, c->sweeps + count);
  if (rc) return rc;
  if (!c->i8_checked && (c->bg_ws || c->i8_ws) && count > 0) {
    // heavy-tailed columns (max/rms above gram_i8.cu's bound): this data set's Grams go to
    // the FP64 DMMA tiles (G is re-formed; the block Grams switch for the whole fit)
    if (c->gram_mode == 1 && !c->have_G && (rc = en_compute_G(c, c->st))) return rc;   // raises the flag
    int bad = 0;
    if ((rc = check_cuda(cudaMemcpyAsync(&bad, c->i8_bad, sizeof(int), cudaMemcpyDeviceToHost, c->st),
                         "int8 accuracy flag")) ||
        (rc = check_cuda(cudaStreamSynchronize(c->st), "int8 accuracy flag")))
      return rc;
    if (bad & 1) {   // bit 1 (8 instead of 7 slices) is read by the kernels themselves
      c->i8_off = true;
      c->have_G = false;
    }
    c->i8_checked = true;
  }
  if (c->gram_mode == 1 && !c->have_G && count > 0 && (rc = en_compute_G(c, c->st))) return rc;
  if (c->pipe && !c->timing && count > 0 && c->gram_mode == 1 && c->cla_L && c->idx_r) {
    // batched preparation: sort + factor + tiles of B sweeps in one launch each on sprep
    // (filling the SMs the lookahead chain leaves free), chains on schain; batch slot j of
    // the 2-slot ring is rewritten only after the last chain that read it.
    cudaEventRecord(c->ev_start, c->st);
    cudaStreamWaitEvent(c->sprep, c->ev_start, 0);
    cudaStreamWaitEvent(c->schain, c->ev_start, 0);
    const int B = c->cla_B;
    const size_t ps = (size_t)c->p * c->s, pss = ps * c->s, pT = pss * c->cla_D;
    for (int k0 = 0; k0 < count; k0 += B) {
      const int bs = std::min(B, count - k0);
      const int j = c->batch_ctr & 1;
      if (c->chain_rec[j]) cudaStreamWaitEvent(c->sprep, c->ev_chain[j], 0);
      c->idx = c->idx_r + (size_t)j * B * ps;
      c->inv = c->inv_r + (size_t)j * B * pss;
      c->info = c->info_r + (size_t)j * B * c->p;
      c->T = c->T_r + (size_t)j * B * pT;
      if ((rc = launch_chunk_sort(perms + (int64_t)k0 * c->n, c->n, c->s, bs, c->idx, c->sprep))) return rc;
      if ((rc = en_factor(c, c->sprep, bs))) return rc;
      cudaEventRecord(c->ev_prep[j], c->sprep);
      cudaStreamWaitEvent(c->schain, c->ev_prep[j], 0);
      // the batch's sweeps run as one chain launch (c->idx/inv/info/T: batch base)
      if ((rc = en_chain(c, tol, c->schain, bs))) return rc;
      c->sweeps += bs;
      cudaEventRecord(c->ev_chain[j], c->schain);
      c->chain_rec[j] = true;
      c->batch_ctr++;
    }
    cudaEventRecord(c->ev_end, c->schain);
    cudaStreamWaitEvent(c->st, c->ev_end, 0);
    return check_launch("rac_en_run (batched)");
  }
  if (c->pipe && !c->timing && count > 0 && c->gram_mode != 1 && c->mode == RAC_MODE_RAC && c->look_gram) {
    // block mode: gram(k+1) runs BEFORE chain(k) (the int8 Gram's shared memory cannot sit
    // beside the chain), so the factorisations of sweep k+1 start together with chain(k) and
    // fill the room the latency-bound chain leaves on every SM:
    //   sprep: sort(k+1) gram(k+1) [ev_gram] factor(k+1) [ev_prep(k+1)]
    //   schain: wait ev_prep(k), ev_gram -> chain(k) [ev_chain(k)]
    // gram_ws is single-buffered: factor(k) precedes gram(k+1) on sprep.
    cudaEventRecord(c->ev_start, c->st);
    cudaStreamWaitEvent(c->sprep, c->ev_start, 0);
    cudaStreamWaitEvent(c->schain, c->ev_start, 0);
    const int base = c->sweeps;
    auto prep_gram = [&](int k) -> int {
      const int j = (base + k) & 1;
      if (c->chain_rec[j]) cudaStreamWaitEvent(c->sprep, c->ev_chain[j], 0);   // chain(k-2) done
      c->idx = c->idx_b[j];
      c->inv = c->inv_b[j];
      c->info = c->info_b[j];
      int r = launch_chunk_sort(perms + (int64_t)k * c->n, c->n, c->s, 1, c->idx, c->sprep);
      return r ? r : en_block_gram(c, c->sprep);
    };
    auto prep_factor = [&](int k) -> int {
      const int j = (base + k) & 1;
      c->idx = c->idx_b[j];
      c->inv = c->inv_b[j];
      c->info = c->info_b[j];
      int r = en_factor(c, c->sprep);
      cudaEventRecord(c->ev_prep[j], c->sprep);
      return r;
    };
    if ((rc = prep_gram(0)) || (rc = prep_factor(0))) return rc;
    for (int k = 0; k < count; ++k) {
      const int j = c->sweeps & 1;
      if (k + 1 < count) {
        if ((rc = prep_gram(k + 1))) return rc;
        cudaEventRecord(c->ev_gram, c->sprep);
        cudaStreamWaitEvent(c->schain, c->ev_gram, 0);
      }
      cudaStreamWaitEvent(c->schain, c->ev_prep[j], 0);
      c->idx = c->idx_b[j];
      c->inv = c->inv_b[j];
      c->info = c->info_b[j];
      if ((rc = en_chain(c, tol, c->schain))) return rc;
      cudaEventRecord(c->ev_chain[j], c->schain);
      c->chain_rec[j] = true;
      c->sweeps++;
      if (k + 1 < count && (rc = prep_factor(k + 1))) return rc;
    }
    cudaEventRecord(c->ev_end, c->schain);
    cudaStreamWaitEvent(c->st, c->ev_end, 0);
    return check_launch("rac_en_run (pipelined, gram ahead)");
  }
  if (c->pipe && !c->timing && count > 0) {
    // prep(k+1) on sprep overlaps chain(k) on schain; prep(k) may only overwrite the
    // buffers of sweep k-2 once that chain is done.
    cudaEventRecord(c->ev_start, c->st);
    cudaStreamWaitEvent(c->sprep, c->ev_start, 0);
    cudaStreamWaitEvent(c->schain, c->ev_start, 0);
    for (int k = 0; k < count; ++k) {
      const int j = c->sweeps & 1;
      if (c->chain_rec[j]) cudaStreamWaitEvent(c->sprep, c->ev_chain[j], 0);
      c->idx = c->idx_b[j];
      c->inv = c->inv_b[j];
      c->info = c->info_b[j];
      c->T = c->T_b[j];
      if ((rc = launch_chunk_sort(perms + (int64_t)k * c->n, c->n, c->s, 1, c->idx, c->sprep))) return rc;
      if (c->gram_mode != 1 && (rc = en_block_gram(c, c->sprep))) return rc;
      if ((rc = en_factor(c, c->sprep))) return rc;
      cudaEventRecord(c->ev_prep[j], c->sprep);
      cudaStreamWaitEvent(c->schain, c->ev_prep[j], 0);
      if ((rc = en_chain(c, tol, c->schain))) return rc;
      cudaEventRecord(c->ev_chain[j], c->schain);
      c->chain_rec[j] = true;
      c->sweeps++;
    }
    cudaEventRecord(c->ev_end, c->schain);
    cudaStreamWaitEvent(c->st, c->ev_end, 0);
    return check_launch("rac_en_run (pipelined)");
  }
  for (int k = 0; k < count; ++k) {
    cudaEvent_t ev[5] = {};
    if (c->timing) {
      for (auto& e : ev) cudaEventCreate(&e);
      cudaEventRecord(ev[0], c->st);
    }
    if (c->mode == RAC_MODE_RAC) {
      rc = launch_chunk_sort(perms + (int64_t)k * c->n, c->n, c->s, 1, c->idx, c->st);
      if (rc) return rc;
      if (c->timing) cudaEventRecord(ev[1], c->st);
      if (c->gram_mode != 1) {
        cudaEvent_t mid = nullptr;
        if (c->timing && c->bg_ws && !c->i8_off) cudaEventCreate(&mid);
        rc = en_block_gram(c, c->st, mid);
        if (rc) return rc;
        if (mid) c->slice_events.push_back(mid);
      }
      if (c->timing) cudaEventRecord(ev[2], c->st);
      rc = en_factor(c, c->st);
      if (rc) return rc;
    } else {
      rc = launch_order_cast(perms + (int64_t)k * c->p, c->p, c->order, c->st);
      if (rc) return rc;
      if (c->gram_mode == 1 && (rc = launch_cla_tiles(c, c->st))) return rc;   // tiles follow the visit order
      if (c->timing) { cudaEventRecord(ev[1], c->st); cudaEventRecord(ev[2], c->st); }
    }
    if (c->timing) cudaEventRecord(ev[3], c->st);
    rc = en_chain(c, tol, c->st);
    if (rc) return rc;
    if (c->timing) {
      cudaEventRecord(ev[4], c->st);
      c->events.insert(c->events.end(), ev, ev + 5);
    }
    c->sweeps++;
  }
  return RAC_OK;
}

extern "C" int rac_en_progress(rac_en_ctx* c, int32_t* iterations, int32_t* converged,
                               double* residual, int32_t* failed_block) {
  using namespace rac;
  clear_error();
  if (!c) return set_error(RAC_ERR_ARG, "rac_en_progress: null context");
  int32_t h[4];
  int rc = check_cuda(cudaMemcpyAsync(h, c->ctrl, sizeof(h), cudaMemcpyDeviceToHost, c->st), "progress");
  if (rc) return rc;
  rc = check_cuda(cudaStreamSynchronize(c->st), "progress sync");
  if (rc) return rc;
  if (iterations) *iterations = h[1];
  if (converged) *converged = h[3];
  if (failed_block) *failed_block = h[2] - 1;
  if (residual) {
    *residual = INFINITY;
    if (h[1] > 0) {
      rc = check_cuda(cudaMemcpy(residual, c->hist_p + (h[1] - 1), sizeof(double), cudaMemcpyDeviceToHost),
                      "progress residual");
      if (rc) return rc;
    }
  }
  return RAC_OK;
}

extern "C" int rac_en_get(rac_en_ctx* c, double* beta, double* z, double* xi, double* r) {
  using namespace rac;
  clear_error();
  if (!c) return set_error(RAC_ERR_ARG, "rac_en_get: null context");
  const size_t nb = c->n * sizeof(double);
  if (beta) cudaMemcpyAsync(beta, c->beta, nb, cudaMemcpyDeviceToDevice, c->st);
  if (z) cudaMemcpyAsync(z, c->z, nb, cudaMemcpyDeviceToDevice, c->st);
  if (xi) cudaMemcpyAsync(xi, c->xi, nb, cudaMemcpyDeviceToDevice, c->st);
  if (r) cudaMemcpyAsync(r, c->r, c->m * sizeof(double), cudaMemcpyDeviceToDevice, c->st);
  return check_launch("rac_en_get");
}

extern "C" int rac_en_history(rac_en_ctx* c, double* primal, double* dual, int32_t capacity) {
  using namespace rac;
  clear_error();
  if (!c || capacity < 0) return set_error(RAC_ERR_ARG, "rac_en_history: bad arguments");
  int k = std::min(capacity, c->hist_cap);
  if (k <= 0) return RAC_OK;
  if (primal) cudaMemcpyAsync(primal, c->hist_p, k * sizeof(double), cudaMemcpyDeviceToDevice, c->st);
  if (dual) cudaMemcpyAsync(dual, c->hist_d, k * sizeof(double), cudaMemcpyDeviceToDevice, c->st);
  return check_launch("rac_en_history");
}

extern "C" int rac_en_set_timing(rac_en_ctx* c, int32_t enable) {
  using namespace rac;
  clear_error();
  if (!c) return set_error(RAC_ERR_ARG, "rac_en_set_timing: null context");
  c->timing = enable != 0;
  if (enable >= 2 && !c->trace) {
    // chain stamps, then the factor kernel's (block 0): 8 + 16p | 8 + s
    int rc = dalloc(c, &c->trace, 16 + 28 * (size_t)c->p + c->s);   // + 8p clock64 stamps (lookahead chain)
    if (rc) return rc;
    c->trace_buf = c->trace;
  }
  c->trace = (enable >= 2) ? c->trace_buf : nullptr;
  return RAC_OK;
}

extern "C" int rac_en_info(rac_en_ctx* c, int32_t* info4) {
  using namespace rac;
  clear_error();
  if (!c || !info4) return set_error(RAC_ERR_ARG, "rac_en_info: bad arguments");
  info4[0] = (c->gram_mode == 1) ? (c->cla_L ? 3 : 2) : c->variant;
  info4[1] = (c->gram_mode == 1) ? (c->cla_L ? c->cla_L + c->cla_W : c->cov_k) : c->P;
  // lookahead chain: [3, grid CTAs, sweeps per preparation batch, lookahead depth]
  info4[2] = (c->gram_mode == 1 && c->cla_L) ? (c->pipe && c->idx_r ? c->cla_B : 1) : c->RC;
  info4[3] = (c->gram_mode == 1 && c->cla_L) ? c->cla_D : c->nch;
  return RAC_OK;
}

extern "C" int rac_en_gram_slices(rac_en_ctx* c, int32_t* slices) {
  using namespace rac;
  clear_error();
  if (!c || !slices) return set_error(RAC_ERR_ARG, "rac_en_gram_slices: bad arguments");
  *slices = 0;
  const int* flags = c->bg_ws ? c->i8_bad : (c->i8_ws ? gram_i8_ws_flags(c->i8_ws) : nullptr);
  if (!flags || c->i8_off || (!c->bg_ws && !c->have_G)) return RAC_OK;
  int f = 0;
  int rc = check_cuda(cudaMemcpyAsync(&f, flags, sizeof(int), cudaMemcpyDeviceToHost, c->st), "slices flag");
  if (!rc) rc = check_cuda(cudaStreamSynchronize(c->st), "slices flag");
  if (rc) return rc;
  const char* e = getenv("RAC_I8_SLICES");
  *slices = ((f & 2) || (e && atoi(e) == 8)) ? 8 : 7;
  return RAC_OK;
}

extern "C" int rac_en_trace(rac_en_ctx* c, int64_t* host, int32_t capacity) {
  using namespace rac;
  clear_error();
  if (!c || !host || !c->trace) return set_error(RAC_ERR_ARG, "rac_en_trace: tracing not enabled");
  int k = std::min<int>(capacity, 16 + 28 * c->p + c->s);
  return check_cuda(cudaMemcpy(host, c->trace, k * sizeof(int64_t), cudaMemcpyDeviceToHost), "trace copy");
}

extern "C" int rac_en_timing(rac_en_ctx* c, double* stage_ms, int32_t* sweeps) {
  using namespace rac;
  clear_error();
  if (!c || !stage_ms) return set_error(RAC_ERR_ARG, "rac_en_timing: bad arguments");
  int rc = check_cuda(cudaStreamSynchronize(c->st), "timing sync");
  if (rc) return rc;
  for (int q = 0; q < 4; ++q) stage_ms[q] = 0.0;
  const size_t k = c->events.size() / 5;
  for (size_t i = 0; i < k; ++i) {
    for (int q = 0; q < 4; ++q) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, c->events[5 * i + q], c->events[5 * i + q + 1]);
      stage_ms[q] += ms;
    }
  }
  // slicing share of the gram stage (int8 block Grams; one mid event per timed sweep)
  c->slice_ms = 0.0;
  if (c->slice_events.size() == k)
    for (size_t i = 0; i < k; ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, c->events[5 * i + 1], c->slice_events[i]);
      c->slice_ms += ms;
    }
  for (auto e : c->slice_events) cudaEventDestroy(e);
  c->slice_events.clear();
  for (auto e : c->events) cudaEventDestroy(e);
  c->events.clear();
  if (sweeps) *sweeps = (int32_t)k;
  return RAC_OK;
}

extern "C" int rac_en_timing_slicing(rac_en_ctx* c, double* slice_ms) {
  using namespace rac;
  clear_error();
  if (!c || !slice_ms) return set_error(RAC_ERR_ARG, "rac_en_timing_slicing: bad arguments");
  *slice_ms = c->slice_ms;
  return RAC_OK;
}

extern "C" int rac_en_reset(rac_en_ctx* c, double lam, double alpha, double gamma) {
  using namespace rac;
  clear_error();
  if (!c || !(gamma > 0) || lam < 0 || alpha < 0 || alpha > 1) return set_error(RAC_ERR_ARG, "rac_en_reset: bad arguments");
  cudaStream_t st = c->st;
  if (c->pipe) {
    // previous work on the helper streams completes before their buffers are reused
    cudaEventRecord(c->ev_end, c->schain);
    cudaStreamWaitEvent(st, c->ev_end, 0);
    cudaEventRecord(c->ev_start, c->sprep);
    cudaStreamWaitEvent(st, c->ev_start, 0);
  }
  c->lam = lam;
  c->alpha = alpha;
  c->gamma = gamma;
  c->sweeps = 0;
  c->have_data = false;
  c->have_partition = false;
  c->have_G = false;
  cudaMemsetAsync(c->beta, 0, c->n * sizeof(double), st);
  cudaMemsetAsync(c->z, 0, c->n * sizeof(double), st);
  cudaMemsetAsync(c->xi, 0, c->n * sizeof(double), st);
  cudaMemsetAsync(c->r, 0, c->ld * sizeof(double), st);
  cudaMemsetAsync(c->ctrl, 0, 4 * sizeof(int32_t), st);
  for (int32_t* inf : {c->info_b[0], c->info_b[1]})
    if (inf) cudaMemsetAsync(inf, 0, c->p * sizeof(int32_t), st);
  if (c->info_r) cudaMemsetAsync(c->info_r, 0, (size_t)2 * c->cla_B * c->p * sizeof(int32_t), st);
  if (c->conv) cudaMemsetAsync(c->conv, 0xff, 2 * sizeof(int32_t), st);
  return check_launch("rac_en_reset");
}

extern "C" int rac_en_destroy(rac_en_ctx* c) {
  if (!c) return RAC_OK;
  if (c->st) cudaStreamSynchronize(c->st);
  if (c->schain) cudaStreamSynchronize(c->schain);
  if (c->sprep) cudaStreamSynchronize(c->sprep);
  for (auto e : c->events) cudaEventDestroy(e);
  for (cudaEvent_t e : {c->ev_start, c->ev_end, c->ev_prep[0], c->ev_prep[1], c->ev_chain[0], c->ev_chain[1], c->ev_gram,
                        c->ev_ctrl[0], c->ev_ctrl[1]})
    if (e) cudaEventDestroy(e);
  if (c->h_ctrl) cudaFreeHost(c->h_ctrl);
  if (c->schain) cudaStreamDestroy(c->schain);
  if (c->sprep) cudaStreamDestroy(c->sprep);
  for (void* q : c->allocs) rac::dev_free(q, c->st);
  // release the freed memory above the pool's threshold now (a later synchronisation would
  // otherwise pay for unmapping gigabytes at an unrelated point, e.g. inside the next fit)
  if (c->st) cudaStreamSynchronize(c->st);
  rac::trim_pool(rac::POOL_KEEP);
  delete c;
  return RAC_OK;
}

// Debugging aid: progress markers of the lookahead chain are written to this
// device-accessible (mapped, pinned) host buffer of >= 16 int64 (null: off).
extern "C" int rac_debug_buffer(void* mapped_host) {
  g_cla_dbg = (volatile long long*)mapped_host;
  return RAC_OK;
}

extern "C" int rac_gram_covariance(const double* Xc, int64_t ld, int64_t len, int32_t n, double* G, double div,
                                   int32_t method) {
  using namespace rac;
  clear_error();
  if (!Xc || !G || n < 1 || len < 1 || ld < len || (method != 0 && method != 1))
    return set_error(RAC_ERR_ARG, "rac_gram_covariance: bad arguments");
  cudaStream_t st = 0;
  int rc = RAC_OK;
  if (method == 1) {
    // grow-only workspace kept between calls (a utility for tests and measurements)
    static void* ws = nullptr;
    static size_t cap = 0;
    const size_t need = gram_i8_ws_bytes(len, n);
    if (cap < need) {
      cudaDeviceSynchronize();
      if (ws) cudaFree(ws);
      ws = nullptr;
      cap = 0;
      if (cudaMalloc(&ws, need) != cudaSuccess) return set_error(RAC_ERR_CUDA, "rac_gram_covariance: out of memory");
      cap = need;
    }
    rc = launch_gram_i8(Xc, ld, len, n, G, div, div > 0.0 ? 0 : 1, ws, cap, st);
    cudaStreamSynchronize(st);
  } else {
    GramPlan pl = plan_gram(len, n, 1);
    pl.splits = 1;
    pl.chunk = (len + 31) / 32 * 32;
    int32_t* ids = nullptr;
    if (cudaMalloc(&ids, sizeof(int32_t) * n) != cudaSuccess) return set_error(RAC_ERR_CUDA, "out of memory");
    iota_kernel<<<(n + 255) / 256, 256, 0, st>>>(ids, n);
    rc = launch_gram(Xc, ld, pl.chunk, ids, nullptr, n, 1, G, pl, st, nullptr, div > 0.0 ? div : 0.0,
                     div > 0.0 ? 0 : 1);
    cudaStreamSynchronize(st);
    cudaFree(ids);
  }
  if (rc) return rc;
  return check_launch("rac_gram_covariance");
}
