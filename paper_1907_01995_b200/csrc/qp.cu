// Dense box-QP sweep engine behind engine.solve (engine.py:322-405) and
// svm.train (svm.py:181-284), sm_100a, FP64, HBM-resident.
//
//   min 1/2 x'Hx + c'x   s.t.  Ax = b,  lo <= x <= hi
//
// Per sweep (RAC): K1 chunk-sort -> K2 batched A_b'A_b on FP64 tensor cores
// -> K3 block matrices M_b = H_bb + beta A_b'A_b (+ ridge), their inverses
// -> one cooperative launch for the whole Gauss-Seidel chain:
//
//   G  (all CTAs) hx += H[blk_prev, :]' delta   (column-parallel, one HBM pass
//      over the strip; svm.py:255 `qz += strip.T @ delta`)
//      ax += A[:, blk_prev] delta; partial = A_b'(y - beta(ax_rest - b)) rows
//   -- grid barrier --
//   S  (CTA 0) rhs = -c_b - (hx_b - H_bb x_b) + A_b'(...)   (engine.py:122-133,
//      svm.py:247-249), x_b = exact box minimizer (engine.py:189-245)
//   -- grid barrier --
//
// then y <- y - beta(Ax - b) and the residuals of engine.py:259-281 /
// svm.py:258-262 with the divergence / convergence tests of engine.py:385-397.
// The SVM is the instance H = Q, A = y', b = 0, c = -1, box [0, C], with the
// 1e-9 relative ridge of svm.py:242-246.
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "boxqp.cuh"
#include "rac_internal.h"
#include "rac_rowphase.cuh"

namespace rac {

constexpr int QPT = RP_THREADS;  // 256 threads per chain CTA
constexpr int QCOLS = 128;       // column tile of the strip update

struct QpChainArgs {
  int64_t n, m, lda;
  int s, p, nrc;
  const double* H;     // n x n row-major (ldh = n), may be null
  const double* Ac;    // column-major A (lda x n), may be null
  const double *b, *c, *lo, *hi;
  const int32_t* idx;
  const int32_t* order;
  const double *Mb, *Hbb, *inv;
  const int32_t* info;
  double *x, *y, *hx, *ax;
  double *partial, *delta;
  double *pmax, *psum, *dmax;  // per CTA
  double* lscratch;            // s x s global factor scratch (large s)
  double* hbx;                 // [s] H_bb x_b of the next block (computed in the G phase)
  const double* Ninv;          // [p][s][s] block inverses M_b^{-1}
  const double* cond;          // [p] pivot-ratio condition estimate of M_b
  long long* trace;            // optional %globaltimer stamps (CTA 0): per block [S start, S end, G start, G end]
  unsigned* bar;
  int32_t* ctrl;  // [0] done, [1] iterations, [2] failed block+1, [3] status
  double beta, tol_p, tol_d, div_bar;
  int fixed, sweep, lsmem;
  double *hist_p, *hist_l1, *hist_d;
  // blocks [t0, t1) of the sweep's visit order run in this launch (the dual step and the
  // residuals only when t1 == p).  strips: H holds the kernel strips of exactly these blocks,
  // row (t - t0) * s + i for member i of block t (formed on the fly, svm.py:121-143), instead
  // of the full N x N matrix indexed by sample
  int t0, t1, strips;
  // One grid barrier per block instead of two (resident strips staged in shared memory, no or few
  // constraint rows): the workers publish hx at the NEXT block's coordinates as tagged word pairs
  // right where they apply delta (each coordinate has one owner CTA and one reader, CTA 0), and the
  // constraint-row owner publishes the block's partial the same way; CTA 0 spins on those words
  // instead of waiting for the whole grid.  llq: hx words [s][2], partial words [s][2]; tag of
  // block step t = tagq0 + t + 1.  delta is double-buffered by step parity.
  unsigned long long* llq;
  unsigned tagq0;
};

// H row of member i (global index g) of the block visited at step t
__device__ __forceinline__ const double* h_row(const QpChainArgs& a, int t, int i, int g) {
  return a.strips ? a.H + ((int64_t)(t - a.t0) * a.s + i) * a.n : a.H + (int64_t)g * a.n;
}

// hx[cols of this CTA] += sum_i H[blk[i], col] * delta[i]
__device__ void strip_update(const QpChainArgs& a, int t, const int32_t* sIdx, const double* sDel,
                             double* red, int s) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = QPT / 32;
  const int P = gridDim.x;
  const int64_t per = ((a.n + P - 1) / P + 31) / 32 * 32;
  const int64_t c0 = (int64_t)blockIdx.x * per, c1 = min64(a.n, c0 + per);
  for (int64_t t0 = c0; t0 < c1; t0 += QCOLS) {
    double acc[QCOLS / 32];
#pragma unroll
    for (int q = 0; q < QCOLS / 32; ++q) acc[q] = 0.0;
    // rows in batches of 4: 4 x (QCOLS/32) independent loads in flight per lane
    for (int i0 = warp; i0 < s; i0 += 4 * nw) {
      double v[4][QCOLS / 32];
      double dd[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + u * nw;
        const int g = (i < s) ? sIdx[i] : -1;
        dd[u] = (g >= 0) ? sDel[i] : 0.0;
        const double* row = h_row(a, t, (g >= 0) ? i : 0, g >= 0 ? g : 0);
#pragma unroll
        for (int q = 0; q < QCOLS / 32; ++q) {
          const int64_t j = t0 + q * 32 + lane;
          v[u][q] = (g >= 0 && j < c1) ? __ldg(row + j) : 0.0;
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int q = 0; q < QCOLS / 32; ++q) acc[q] += v[u][q] * dd[u];
    }
#pragma unroll
    for (int q = 0; q < QCOLS / 32; ++q) red[warp * QCOLS + q * 32 + lane] = acc[q];
    __syncthreads();
    for (int e = tid; e < QCOLS; e += QPT) {
      int64_t j = t0 + e;
      if (j < c1) {
        double tot = red[e];
        for (int w = 1; w < nw; ++w) tot += red[w * QCOLS + e];
        a.hx[j] += tot;
      }
    }
    __syncthreads();
  }
}

struct QpSmem {
  RowPhaseSmem rp;
  BoxWork bw;
  double* red;     // nw * QCOLS
  int32_t* sIdx;   // s
  double* sDel;    // s
  double *sxb, *shx, *sc;
  double* sM;      // s x s block matrix M_b (smem-resident when lsmem)
  double* sN;      // s x s M_b^{-1} (smem-resident when lsmem)
  double* Lsmall;  // small factor workspace ((s/2+1)^2) for the Schur / small direct solves
  uint64_t* bar;   // mbarrier of the M_b / N_b prefetch
};

__host__ __device__ inline size_t qp_lsmall(int s) { return (size_t)(s / 2 + 2) * (s / 2 + 2); }

template <int RC>
__host__ __device__ size_t qp_smem_bytes(int s, bool rowphase, bool lsmem) {
  size_t d = 0;
  if (rowphase) d += RowPhase<RC>::smem_doubles(s) + s;  // + int idx (as doubles, generous)
  d += (QPT / 32) * QCOLS;                               // strip reduction
  d += 15 * (size_t)s + 64;                              // box vectors, rinv, sDel, sxb, shx, sc, symv scratch
  if (lsmem) d += 2 * (size_t)s * s + qp_lsmall(s) + 3;  // M_b, N_b, small workspace, mbarrier, align
  size_t ints = 4 * (size_t)s + 64;                      // flag, F, B, sIdx, misc
  return d * sizeof(double) + ints * sizeof(int);
}

template <int RC>
__device__ QpSmem carve_qp(double* base, int s, bool rowphase, bool lsmem, double* lscratch) {
  QpSmem q;
  double* p = base;
  if (rowphase) {
    q.rp = carve_rowphase<RC>(p, s);
    p += RowPhase<RC>::smem_doubles(s) + s;
  }
  q.red = p;
  p += (QPT / 32) * QCOLS;
  q.bw.x = p; p += s;
  q.bw.r = p; p += s;
  q.bw.lo = p; p += s;
  q.bw.hi = p; p += s;
  q.bw.grad = p; p += s;
  q.bw.xf = p; p += s;
  q.bw.rr = p; p += s;
  q.sDel = p; p += s;
  q.sxb = p; p += s;
  q.shx = p; p += s;
  q.bw.red = p; p += 32;
  q.sc = p; p += 32;  // scalars
  q.bw.rinv = p; p += s;
  q.bw.symv_scratch = p; p += 4 * s;
  q.bw.dbg = nullptr;
  q.bw.st = nullptr;
  q.bw.N = nullptr;
  q.bw.ldn = s;
  q.bw.L = lscratch;                       // large workspace (global): s(s+1) doubles
  q.bw.lcap = s * (s + 1);
  if (lsmem) {
    p += (p - base) & 1;   // 16-byte alignment for the TMA destinations
    q.sM = p;
    p += (size_t)s * s;
    q.sN = p;
    p += (size_t)s * s;
    q.Lsmall = p;
    p += qp_lsmall(s);
    q.bar = reinterpret_cast<uint64_t*>(p);
    p += 2;
  } else {
    q.sM = nullptr;
    q.sN = nullptr;
    q.Lsmall = nullptr;
    q.bar = nullptr;
  }
  int* ip = (int*)p;
  q.bw.flag = ip; ip += s;
  q.bw.F = ip; ip += s;
  q.bw.B = ip; ip += s;
  q.sIdx = ip; ip += s;
  q.bw.misc = ip;
  return q;
}

// end of a sweep (all CTAs): dual step y -= beta (Ax - b) with the primal residuals, the dual
// residual per column, the history and the stop / divergence flags (engine.py:248-281,
// 385-397).  Rows of A are owned by the CTA that owns their row chunk (RC rows).
template <int RC>
__device__ void qp_sweep_end(const QpChainArgs& a, QpSmem& w, unsigned& target) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = QPT / 32;
  const int P = gridDim.x;
  const bool has_a = a.m > 0;
  const double beta = a.beta;
  grid_barrier(a.bar, target, P);
  // ------------------------------------------------------------ dual step + primal residual
  // rows of A are owned by the CTA that owns their row chunk
  double pm = 0.0, ps = 0.0;
  if (has_a) {
    for (int ch = blockIdx.x; ch < a.nrc; ch += P) {
      const int64_t i0 = (int64_t)ch * RC;
      for (int r = tid; r < RC; r += QPT) {
        const int64_t i = i0 + r;
        if (i < a.m) {
          const double res = ldcg(a.ax + i) - a.b[i];
          a.y[i] = a.y[i] - beta * res;
          pm = nanmax(pm, fabs(res));
          ps += fabs(res);
        }
      }
    }
  }
  pm = warp_nanmax(pm);
  ps = warp_sum(ps);
  if (lane == 0) { w.bw.red[warp] = pm; w.sc[warp] = ps; }
  __syncthreads();
  if (tid == 0) {
    double m1 = 0.0, s1 = 0.0;
    for (int q = 0; q < nw; ++q) { m1 = nanmax(m1, w.bw.red[q]); s1 += w.sc[q]; }
    a.pmax[blockIdx.x] = m1;
    a.psum[blockIdx.x] = s1;
  }
  grid_barrier(a.bar, target, P);
  // ------------------------------------------------------------ dual residual (columns)
  double dm = 0.0;
  {
    const int gw = blockIdx.x * nw + warp, GW = P * nw;
    for (int64_t j = gw; j < a.n; j += GW) {
      double aty = 0.0;
      if (has_a) {
        const double* col = a.Ac + j * a.lda;
        for (int64_t r = lane; r < a.m; r += 32) aty += col[r] * ldcg(a.y + r);
        aty = warp_sum(aty);
      }
      if (lane == 0) {
        double grad = a.c[j];
        if (a.H) grad = grad + ldcg(a.hx + j);
        if (has_a) grad = grad - aty;
        const double xj = ldcg(a.x + j);
        const double v = xj - grad;
        const double pr = (v != v) ? v : fmin(fmax(v, a.lo[j]), a.hi[j]);   // np.clip keeps NaN
        dm = nanmax(dm, fabs(pr - xj));
      }
    }
  }
  dm = warp_nanmax(dm);
  if (lane == 0) w.bw.red[warp] = dm;
  __syncthreads();
  if (tid == 0) {
    double m1 = 0.0;
    for (int q = 0; q < nw; ++q) m1 = nanmax(m1, w.bw.red[q]);
    a.dmax[blockIdx.x] = m1;
  }
  grid_barrier(a.bar, target, P);
  if (blockIdx.x == 0 && warp == 0) {
    double pmx = 0.0, psm = 0.0, dmx = 0.0;
    for (int q = lane; q < P; q += 32) {
      pmx = nanmax(pmx, ldcg(a.pmax + q));
      psm += ldcg(a.psum + q);
      dmx = nanmax(dmx, ldcg(a.dmax + q));
    }
    pmx = warp_nanmax(pmx);
    psm = warp_sum(psm);
    dmx = warp_nanmax(dmx);
    if (lane == 0) {
      a.hist_p[a.sweep] = pmx;
      a.hist_l1[a.sweep] = psm;
      a.hist_d[a.sweep] = dmx;
      a.ctrl[1] = a.sweep + 1;
      if (pmx > a.div_bar) {
        a.ctrl[3] = RAC_STATUS_DIVERGED;
        a.ctrl[0] = 1;
      } else if (!a.fixed && pmx <= a.tol_p && dmx <= a.tol_d) {
        a.ctrl[3] = RAC_STATUS_CONVERGED;
        a.ctrl[0] = 1;
      }
    }
  }
}

template <int RC>
__global__ void __launch_bounds__(QPT, 1) qp_chain_kernel(QpChainArgs a) {
  if (a.ctrl[0]) return;
  extern __shared__ __align__(16) double qsm[];
  const int s = a.s;
  const bool has_a = a.m > 0;
  QpSmem w = carve_qp<RC>(qsm, s, has_a, a.lsmem != 0, a.lscratch);
  __shared__ int bad;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = QPT / 32;
  const int P = gridDim.x;
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
  const double beta = a.beta;
  // rest_r = ax_r - (A_b x_b)_r ;  t_r = y_r - beta * (rest_r - b_r)
  auto tfn = [&](int64_t r, double ax_r, double u) {
    return ldcg(a.y + r) - beta * ((ax_r - u) - a.b[r]);
  };
  // CTA 0 keeps M_b and the Cholesky factor L_b of the block it solves in
  // shared memory; the next block's pair is fetched by TMA bulk copies while
  // every CTA runs the G phase.
  unsigned mpar = 0u;
  const bool bulkML = (w.sM != nullptr) && ((s * s) % 2 == 0);
  if (blockIdx.x == 0 && w.sM && tid == 0) {
    mbar_init(w.bar, 1);       // N_b = M_b^{-1} (needed first: x0 = N_b r)
    mbar_init(w.bar + 1, 1);   // M_b (needed by the box solve; its copy runs under x0)
    mbar_fence_init();
  }
  auto prefetch_ML = [&](int b) {
    if (blockIdx.x != 0 || !w.sM) return;
    const double* Mg = a.Mb + (int64_t)b * s * s;
    const double* Ng = a.Ninv + (int64_t)b * s * s;
    __syncthreads();
    if (bulkML) {
      if (tid == 0) {
        fence_proxy_async();
        const unsigned bytes = (unsigned)(s * s * sizeof(double));
        mbar_arrive_expect_tx(w.bar, bytes);
        for (unsigned off = 0; off < bytes; off += 32768u)
          bulk_g2s(w.sN + off / 8, Ng + off / 8, min(32768u, bytes - off), w.bar);
        mbar_arrive_expect_tx(w.bar + 1, bytes);
        for (unsigned off = 0; off < bytes; off += 32768u)
          bulk_g2s(w.sM + off / 8, Mg + off / 8, min(32768u, bytes - off), w.bar + 1);
      }
    } else {
      for (int e = tid; e < s * s; e += QPT) {
        cp_async8(w.sM + e, Mg + e);
        cp_async8(w.sN + e, Ng + e);
      }
      cp_async_commit();
    }
  };
  auto wait_N = [&]() {   // N_b resident (also M_b when the copies are not bulk copies)
    if (bulkML) mbar_spin(w.bar, mpar);   // on the critical path: poll, no suspend / wake latency
    else if (w.sM) cp_async_wait<0>();
    __syncthreads();
  };
  auto wait_M = [&]() {
    if (bulkML) {
      mbar_spin(w.bar + 1, mpar);
      mpar ^= 1u;
      __syncthreads();
    }
  };
  // hbx = H_bb x_b for block b (rows spread over all warps of the grid)
  // Strip staging: while CTA 0 solves block b, every other CTA bulk-copies
  // its column slice of the block's H rows into its (otherwise unused)
  // M/N shared-memory region, so the G phase is pure shared-memory math.
  // With few constraint rows, CTA 1 keeps them (small_pre/small_post below) and
  // gets no strip, so its G-phase work does not add to a strip.
  const bool few_rows = has_a && a.m <= 8 && a.nrc == 1 && 2 * a.m * s <= 1024 && P > 2;
  const int sfirst = few_rows ? 2 : 1;                           // first CTA with a strip
  const int64_t sper = (a.n + (P - sfirst - 1)) / max(1, P - sfirst);
  const int64_t sper2 = (sper + 1) & ~1LL;                      // even: 16-byte row segments
  const bool strip_smem = a.H && w.sM && P > sfirst && (sper2 * s <= 2LL * s * s + (int64_t)qp_lsmall(s)) &&
                          (a.n % 2 == 0);
  const int64_t sc0 = ((int)blockIdx.x < sfirst) ? 0 : min64(a.n, (int64_t)(blockIdx.x - sfirst) * sper2);
  const int64_t sc1 = ((int)blockIdx.x < sfirst) ? 0 : min64(a.n, sc0 + sper2);
  const bool lla = a.llq != nullptr && strip_smem && ((few_rows && strip_smem) || !has_a) && P > sfirst;
  unsigned long long* const hxLL = a.llq;
  unsigned long long* const paLL = a.llq ? a.llq + 2 * (size_t)s : nullptr;
  // workers: position of each owned column in the next block (-1: not a member); w.red is free
  // on the strip CTAs when the strips are staged in shared memory
  int* posmap = reinterpret_cast<int*>(w.red);
  // a strip CTA owns its columns of hx for the whole launch: kept in shared memory (second half of
  // w.red), written through to global memory, so the G phase has no load of hx on its path
  double* sHx = w.red + (QPT / 32) * QCOLS / 2;
  const bool hx_cached = strip_smem && blockIdx.x >= (unsigned)sfirst && sc1 > sc0 &&
                         (sc1 - sc0) <= (QPT / 32) * QCOLS / 2;
  if (hx_cached)
    for (int jj = tid; jj < (int)(sc1 - sc0); jj += QPT) sHx[jj] = ldcg(a.hx + sc0 + jj);
  auto build_posmap = [&](int bn) {
    if (blockIdx.x < (unsigned)sfirst || sc1 <= sc0) return;
    const int W = (int)(sc1 - sc0);
    for (int jj = tid; jj < W; jj += QPT) posmap[jj] = -1;
    __syncthreads();
    if (bn >= 0) {
      const int32_t* bi = a.idx + (int64_t)bn * s;
      for (int i = tid; i < s; i += QPT) {
        const int g = bi[i];
        if (g >= sc0 && g < sc1) posmap[g - sc0] = i;
      }
    }
    __syncthreads();
  };
  unsigned spar = 0u;
  if (strip_smem && blockIdx.x != 0 && tid == 0) {
    mbar_init(w.bar, 1);
    mbar_fence_init();
  }
  auto issue_strip = [&](int b, int t) {
    if (!strip_smem || blockIdx.x == 0 || sc1 <= sc0) return;
    const int32_t* bi = a.idx + (int64_t)b * s;
    const unsigned seg = (unsigned)((sc1 - sc0) * sizeof(double));
    // valid rows: padding only at the end of a short last block -> count in parallel
    int mine = 0;
    for (int i = tid; i < s; i += QPT) mine += (bi[i] >= 0);
    if (tid == 0) w.bw.misc[1] = 0;
    __syncthreads();
    if (mine) atomicAdd(&w.bw.misc[1], mine);
    __syncthreads();
    if (tid == 0) {
      fence_proxy_async();
      mbar_arrive_expect_tx(w.bar, seg * (unsigned)w.bw.misc[1]);
    }
    __syncthreads();
    for (int i = tid; i < s; i += QPT) {
      const int g = bi[i];
      if (g >= 0) bulk_g2s(w.sM + (size_t)i * sper2, h_row(a, t, i, g) + sc0, seg, w.bar);
      else
        for (int64_t jj = 0; jj < sc1 - sc0; ++jj) w.sM[(size_t)i * sper2 + jj] = 0.0;   // padding row
    }
  };
  auto strip_from_smem = [&](unsigned pub_tag) {   // pub_tag != 0: publish hx at the next block's coordinates
    if (blockIdx.x == 0 || sc1 <= sc0) return;
    mbar_wait(w.bar, spar);
    spar ^= 1u;
    __syncthreads();
    const int W = (int)(sc1 - sc0);
    for (int jj = tid; jj < W; jj += QPT) {
      // padding rows are zero-filled and their delta is 0: no branch; 4 partial sums
      const double hx0 = hx_cached ? sHx[jj] : ldcg(a.hx + sc0 + jj);
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      int i = 0;
      for (; i + 4 <= s; i += 4) {
        a0 += w.sM[(size_t)i * sper2 + jj] * w.sDel[i];
        a1 += w.sM[(size_t)(i + 1) * sper2 + jj] * w.sDel[i + 1];
        a2 += w.sM[(size_t)(i + 2) * sper2 + jj] * w.sDel[i + 2];
        a3 += w.sM[(size_t)(i + 3) * sper2 + jj] * w.sDel[i + 3];
      }
      for (; i < s; ++i) a0 += w.sM[(size_t)i * sper2 + jj] * w.sDel[i];
      const double hnew = hx0 + ((a0 + a1) + (a2 + a3));
      a.hx[sc0 + jj] = hnew;
      if (hx_cached) sHx[jj] = hnew;
      if (pub_tag && posmap[jj] >= 0) ll_store(hxLL + 2 * (size_t)posmap[jj], hnew, pub_tag);
    }
    __syncthreads();
  };
  // Rows go to CTAs 1..P-1 (CTA 0 solves the box QPs); every lane issues all its
  // index loads, then all its H_bb / x loads, so a row costs two round trips.
  auto compute_hbx = [&](int b, int slot) {
    if (!a.H) return;
    const int32_t* bi = a.idx + (int64_t)b * s;
    const double* Hb = a.Hbb + (int64_t)b * s * s;
    const int P1 = max(1, P - 1), c1 = (P > 1) ? (int)blockIdx.x - 1 : 0;
    if (c1 < 0) return;
    for (int i = c1 * nw + warp; i < s; i += P1 * nw) {
      constexpr int U = 8;                 // columns per lane per round
      double acc = 0.0;
      for (int j0 = 0; j0 < s; j0 += 32 * U) {
        int gs[U];
        double hv[U], xv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int j = j0 + lane + 32 * u;
          gs[u] = (j < s) ? bi[j] : -1;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int j = j0 + lane + 32 * u;
          hv[u] = (gs[u] >= 0) ? Hb[(int64_t)i * s + j] : 0.0;
          xv[u] = (gs[u] >= 0) ? ldcg(a.x + gs[u]) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc += hv[u] * xv[u];
      }
      acc = warp_sum(acc);
      if (lane == 0) a.hbx[(int64_t)slot * s + i] = acc;
    }
  };
  // Few constraint rows (SVM: the single row y'): one owner CTA (CTA 1, idle while
  // CTA 0 solves) keeps them, with ax and the A columns of the current and next
  // block in shared memory.  small_pre(bn, slot) (during the S phase: x of the
  // next block is final) gathers A[:, bn] and forms u = A_bn x_bn;
  // small_post(slot_b, slot_bn) (G phase) is shared-memory arithmetic only:
  // ax += A_b delta, t = y - beta(ax - u - b), partial = A_bn' t.
  const bool small_a = few_rows && strip_smem;
  const int a_owner = (P > 1) ? 1 : 0;
  __shared__ double sred[8][QPT / 32];
  __shared__ double sUn[2][8], sUp[8], sAx[8];
  double* aS = w.red;   // [2][m][s] (w.red is free when the strips are staged in smem)
  auto block_rows_sum = [&](double* v, int mr, double* out) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
      if (r < mr) {
        const double u = warp_sum(v[r]);
        if (lane == 0) sred[r][warp] = u;
      }
    __syncthreads();
    if (tid < mr) {
      double u = 0.0;
      for (int w2 = 0; w2 < nw; ++w2) u += sred[tid][w2];
      out[tid] = u;
    }
    __syncthreads();
  };
  if (small_a && (int)blockIdx.x == a_owner && tid < a.m) sAx[tid] = ldcg(a.ax + tid);
  auto small_pre = [&](int bn, int slot) {
    if ((int)blockIdx.x != a_owner) return;
    const int mr = (int)a.m;
    double un[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) un[r] = 0.0;
    double* dst = aS + (size_t)slot * mr * s;
    for (int j = tid; j < s; j += QPT) {
      const int gn = a.idx[(int64_t)bn * s + j];
      const double xn = (gn >= 0) ? ldcg(a.x + gn) : 0.0;
#pragma unroll
      for (int r = 0; r < 8; ++r)
        if (r < mr) {
          const double av = (gn >= 0) ? a.Ac[(int64_t)gn * a.lda + r] : 0.0;
          dst[(size_t)r * s + j] = av;
          un[r] += av * xn;
        }
    }
    block_rows_sum(un, mr, sUn[slot]);
  };
  auto small_post = [&](int slot_b, int slot_bn, bool has_prev, bool has_next, unsigned pub_tag) {
    if ((int)blockIdx.x != a_owner) return;
    const int mr = (int)a.m;
    if (has_prev) {
      double up[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) up[r] = 0.0;
      const double* ab = aS + (size_t)slot_b * mr * s;
      for (int j = tid; j < s; j += QPT) {
        const double d = w.sDel[j];
#pragma unroll
        for (int r = 0; r < 8; ++r)
          if (r < mr) up[r] += ab[(size_t)r * s + j] * d;
      }
      block_rows_sum(up, mr, sUp);
    }
    if (tid < mr) {
      const double axr = has_prev ? sAx[tid] + sUp[tid] : sAx[tid];
      sAx[tid] = axr;
      a.ax[tid] = axr;
      w.rp.sT[tid] = tfn(tid, axr, sUn[slot_bn][tid]);
    }
    __syncthreads();
    if (has_next) {
      const double* an = aS + (size_t)slot_bn * mr * s;
      for (int j = tid; j < s; j += QPT) {
        double acc = 0.0;
        for (int r = 0; r < mr; ++r) acc += an[(size_t)r * s + j] * w.rp.sT[r];
        if (pub_tag) ll_store(paLL + 2 * (size_t)j, acc, pub_tag);
        else a.partial[j] = acc;
      }
    }
  };
  // CTA 0 is idle in the G phase: it gathers everything of the next block that is
  // final by then (indices, c, bounds, x, H_bb x_b, the condition estimate) into
  // the strip-reduction smem it never uses, so the next S phase only loads hx and
  // the partial (one round trip).
  const bool pf_on = (blockIdx.x == 0) && strip_smem && !(small_a && a_owner == 0) && 6 * s <= (QPT / 32) * QCOLS;
  double* pf = w.red;   // [6][s]: idx (as double), c, lo, hi, x, hbx
  __shared__ double pf_cond;
  auto prefetch_next = [&](int bn, int slot) {
    if (!pf_on) return;
    const int32_t* bi = a.idx + (int64_t)bn * s;
    for (int i = tid; i < s; i += QPT) {
      const int g = bi[i];
      pf[i] = (double)g;
      if (g >= 0) {
        pf[s + i] = a.c[g];
        pf[2 * s + i] = a.lo[g];
        pf[3 * s + i] = a.hi[g];
        pf[4 * s + i] = ldcg(a.x + g);
        pf[5 * s + i] = a.H ? ldcg(a.hbx + (int64_t)slot * s + i) : 0.0;
      }
    }
    if (tid == 0) pf_cond = ldcg(a.cond + bn);
  };
  int bnext = a.order ? a.order[a.t0] : a.t0;
  const int s0 = a.t0 & 1;   // parity slot of the launch's first block
  prefetch_ML(bnext);
  compute_hbx(bnext, s0);
  if (small_a) {
    small_pre(bnext, s0);
    __syncthreads();
    small_post(s0, s0, false, true, 0u);
  }
  else if (has_a)
    row_phase<RC>(a.Ac, a.lda, a.m, a.nrc, a.idx, s, -1, bnext, a.delta, a.x, a.ax, a.partial, w.rp, tfn);
  const bool tr = a.trace && blockIdx.x == 0 && tid == 0;
  // per-CTA arrival stamps at both grid barriers of every block (tracing only)
  long long* arr = a.trace ? a.trace + 14 * (size_t)a.p : nullptr;
  for (int t = a.t0; t < a.t1; ++t) {
    const int b = bnext;
    if (arr && tid == 0) arr[((size_t)t * P + blockIdx.x) * 2 + 1] = gtimer();
    const bool lla_t = lla && t > a.t0;   // this block's hx / partial arrive as tagged words: no barrier
    const unsigned tagq = a.tagq0 + (unsigned)t + 1u;
    if (!lla_t) grid_barrier(a.bar, target, P);
    if (tr) a.trace[10 * t + 0] = gtimer();
    // While CTA 0 solves block t, the others prepare block t+1's terms that do not
    // depend on block t's solution: H_bb x_b (double-buffered by parity) and, on the
    // constraint-row owner, A_b x_b.
    {
      const int bn1 = (t + 1 < a.t1) ? (a.order ? a.order[t + 1] : t + 1) : -1;
      if (lla && blockIdx.x != 0) build_posmap(bn1);   // for the G phase's publication of hx at block t+1
      if (bn1 >= 0 && blockIdx.x != 0) {
        compute_hbx(bn1, (t + 1) & 1);
        if (small_a) small_pre(bn1, (t + 1) & 1);
        // M_{t+1} and M_{t+1}^{-1} -> L2 (spread over the idle CTAs) so CTA 0's bulk copy
        // of them after this block's box solve hits L2
        if (w.sM || a.Mb) {
          const int lines = (int)(((int64_t)s * s * sizeof(double) + 127) / 128);
          const int per = (lines + P - 2) / (P - 1);
          const int l0 = (blockIdx.x - 1) * per, l1 = min(lines, l0 + per);
          const char* Mg = reinterpret_cast<const char*>(a.Mb + (int64_t)bn1 * s * s);
          const char* Ng = reinterpret_cast<const char*>(a.Ninv ? a.Ninv + (int64_t)bn1 * s * s : nullptr);
          for (int l = l0 + tid; l < l1; l += QPT) {
            prefetch_l2(Mg + (size_t)l * 128);
            if (Ng) prefetch_l2(Ng + (size_t)l * 128);
          }
        }
      }
    }
    // the strip's 8 s n bytes are requested AFTER the latency-bound preparation above: without a
    // grid barrier in front of this point they would otherwise start right behind the previous
    // G phase and delay CTA 0's copy of M_b / N_b, which is on the critical path
    issue_strip(b, t);
    // ------------------------------------------------------------ S (CTA 0)
    if (blockIdx.x == 0) {
      const int32_t* bidx = a.idx + (int64_t)b * s;
      // one parallel gather pass (all loads independent), then the rhs
      // (engine.py:126-132):  -c_b - (hx_b - H_bb x_b) + A_b'(y - beta(Ax_rest - b))
      const int Pa = min(P, a.nrc);   // CTAs that own constraint rows (others' partials are 0)
      // valid entries (padding only at the end of a short last block)
      if (tid == 0) w.bw.misc[0] = 0;
      __syncthreads();
      int nval = 0;
      const bool use_pf = pf_on && t > a.t0;
      for (int i = tid; i < s; i += QPT) {
        const int g = use_pf ? (int)pf[i] : bidx[i];
        w.sIdx[i] = g;
        nval += (g >= 0);
        if (g >= 0) {
          // all of the block's loads in flight, then the spins on the tagged words
          unsigned long long h0 = 0, h1 = 0, p0 = 0, p1 = 0;
          if (lla_t) {
            ll_load2(hxLL + 2 * (size_t)i, h0, h1);
            if (has_a) ll_load2(paLL + 2 * (size_t)i, p0, p1);
          }
          const double hb = a.H ? (use_pf ? pf[5 * s + i] : ldcg(a.hbx + (int64_t)(t & 1) * s + i)) : 0.0;
          double hxg;
          if (lla_t) {   // published by the column's owner while it applied the previous delta
            while (!(ll_ok(h0, tagq) && ll_ok(h1, tagq))) ll_load2(hxLL + 2 * (size_t)i, h0, h1);
            hxg = ll_value((unsigned)h0, (unsigned)h1);
          } else {
            hxg = ldcg(a.hx + g);
          }
          const double xg = use_pf ? pf[4 * s + i] : ldcg(a.x + g);
          const double cg_ = use_pf ? pf[s + i] : a.c[g];
          const double lo = use_pf ? pf[2 * s + i] : a.lo[g], hi = use_pf ? pf[3 * s + i] : a.hi[g];
          double pa = 0.0;
          if (has_a && lla_t) {   // small_a: the constraint-row owner's tagged partial
            while (!(ll_ok(p0, tagq) && ll_ok(p1, tagq))) ll_load2(paLL + 2 * (size_t)i, p0, p1);
            pa = ll_value((unsigned)p0, (unsigned)p1);
          } else if (has_a) {
            for (int q = 0; q < Pa; ++q) pa += ldcg(a.partial + (int64_t)q * s + i);
          }
          w.sxb[i] = xg;
          w.shx[i] = hxg;
          w.bw.lo[i] = lo;
          w.bw.hi[i] = hi;
          double rhs = -cg_;
          if (a.H) rhs = rhs - (hxg - hb);
          if (has_a) rhs = rhs + pa;
          w.bw.r[i] = rhs;
        }
      }
      if (nval) atomicAdd(&w.bw.misc[0], nval);
      __syncthreads();
      if (tr) a.trace[10 * t + 1] = gtimer();
      const int seff = w.bw.misc[0];
      const double cond_b = use_pf ? pf_cond : ldcg(a.cond + b);

      // unconstrained solution (engine.py:201-203).  Well-conditioned blocks:
      // x = N_b r with the smem-resident inverse, reduced systems by Schur
      // complements of N_b.  Otherwise: cho_solve with the block's Cholesky
      // factor and direct reduced factorizations, exactly as the reference.
      const bool schur = (w.sM != nullptr) && (cond_b < 1e6);
      const double* Mblk;
      if (w.sM) wait_N();   // N_b resident (ld = s); M_b may still be landing under x0
      if (tr) a.trace[10 * t + 2] = gtimer();
      if (schur) {
        cta_symv(w.sN, s, seff, w.bw.r, w.bw.x, w.bw.symv_scratch);   // M_b^{-1} is exactly symmetric (Y'Y)
        w.bw.N = w.sN;
        w.bw.ldn = s;
        w.bw.L = w.Lsmall;
        w.bw.lcap = (int)qp_lsmall(s);
        Mblk = w.sM;
      } else {
        const double* Lb = a.inv + (int64_t)b * s * s;
        for (int i = tid; i < seff; i += QPT) w.bw.x[i] = w.bw.r[i];
        __syncthreads();
        warp_chol_solve_any(Lb, s, seff, w.bw.x);
        w.bw.N = nullptr;
        w.bw.L = a.lscratch;
        w.bw.lcap = s * (s + 1);
        Mblk = w.sM ? w.sM : a.Mb + (int64_t)b * s * s;
      }
      if (w.sM) wait_M();   // M_b resident
      __syncthreads();
      long long t_box = tr ? gtimer() : 0;
      if (tr) a.trace[10 * t + 3] = t_box;
      w.bw.dbg = a.trace ? (a.trace + 10 * a.p + 4 * t) : nullptr;
      w.bw.st = a.trace ? (a.trace + 14 * (size_t)a.p + 2 * (size_t)a.p * gridDim.x + 8 * t) : nullptr;
      if (tr) {
        w.bw.dbg[0] = 0; w.bw.dbg[1] = 0; w.bw.dbg[2] = 0;
        for (int q = 0; q < 8; ++q) w.bw.st[q] = 0;
      }
      __syncthreads();
      int fail = box_active_set(Mblk, s, seff, w.bw, schur);
      if (tr) {
        const long long t_end = gtimer();
        w.bw.dbg[3] = t_end - t_box;
        a.trace[10 * t + 4] = t_end;
      }
      if (fail) {
        if (tid == 0) { a.ctrl[2] = b + 1; a.ctrl[0] = 1; }
      }
      for (int i = tid; i < s; i += QPT) {
        double d = 0.0;
        if (i < seff) {
          d = w.bw.x[i] - w.sxb[i];
          a.x[w.sIdx[i]] = w.bw.x[i];
        }
        a.delta[(lla ? (size_t)(t & 1) * s : 0) + i] = d;
      }
      if (t + 1 < a.t1) prefetch_ML(a.order ? a.order[t + 1] : t + 1);
    }
    if (tr) a.trace[10 * t + 5] = gtimer();
    if (arr && tid == 0) arr[((size_t)t * P + blockIdx.x) * 2 + 0] = gtimer();
    grid_barrier(a.bar, target, P);
    if (tr) a.trace[10 * t + 6] = gtimer();
    // ------------------------------------------------------------ G (all CTAs)
    // block data + the non-PD abort flag in one round trip
    for (int i = tid; i < s; i += QPT) {
      w.sIdx[i] = a.idx[(int64_t)b * s + i];
      w.sDel[i] = ldcg(a.delta + (lla ? (size_t)(t & 1) * s : 0) + i);
    }
    if (tid == 0) bad = ldcg(a.ctrl + 0);
    __syncthreads();
    if (bad) return;
    bnext = (t + 1 < a.t1) ? (a.order ? a.order[t + 1] : t + 1) : -1;
    if (P == 1 && bnext >= 0) {   // single CTA: nobody could prepare during S
      compute_hbx(bnext, (t + 1) & 1);
      if (small_a) small_pre(bnext, (t + 1) & 1);
    }
    if (tr) a.trace[10 * t + 8] = gtimer();
    if (strip_smem) strip_from_smem((lla && bnext >= 0) ? tagq + 1u : 0u);
    else if (a.H) strip_update(a, t, w.sIdx, w.sDel, w.red, s);
    if (tr) a.trace[10 * t + 9] = gtimer();
    if (small_a) small_post(t & 1, (t + 1) & 1, true, bnext >= 0, lla ? tagq + 1u : 0u);
    else if (has_a && (int)blockIdx.x < a.nrc)   // CTAs without row chunks have no partial to write
      row_phase<RC>(a.Ac, a.lda, a.m, a.nrc, a.idx, s, b, bnext, a.delta, a.x, a.ax, a.partial, w.rp, tfn);
    if (bnext >= 0) prefetch_next(bnext, (t + 1) & 1);
    if (tr) a.trace[10 * t + 7] = gtimer();
  }
  if (a.t1 < a.p) return;   // a later launch continues the sweep (running Hx / Ax are global)
  qp_sweep_end<RC>(a, w, target);
}

// x0 = clip(0, lo, hi)
__global__ void clip0_kernel(const double* lo, const double* hi, int64_t n, double* x) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = fmin(fmax(0.0, lo[i]), hi[i]);
}

// single-CTA test entry for the box solver (inverse-free first solve)
__global__ void __launch_bounds__(QPT) box_test_kernel(const double* M, const double* r, const double* lo,
                                                       const double* hi, int s, double* xout,
                                                       int32_t* info, double* L, int max_passes) {
  extern __shared__ __align__(16) double bsm[];
  QpSmem w = carve_qp<32>(bsm, s, false, false, L);   // workspace L: global, s(s+1)
  for (int i = threadIdx.x; i < s; i += QPT) {
    w.bw.r[i] = r[i];
    w.bw.lo[i] = lo[i];
    w.bw.hi[i] = hi[i];
    w.bw.flag[i] = 0;
  }
  __syncthreads();
  cta_lists(w.bw, s);  // all free
  for (int i = threadIdx.x; i < s; i += QPT) w.bw.x[i] = 0.0;
  __syncthreads();
  int fail = solve_free(M, s, w.bw, false);
  if (!fail) {
    for (int i = threadIdx.x; i < s; i += QPT) w.bw.x[i] = w.bw.xf[i];
    __syncthreads();
    fail = box_active_set(M, s, s, w.bw, false, max_passes);
  }
  for (int i = threadIdx.x; i < s; i += QPT) xout[i] = w.bw.x[i];
  if (threadIdx.x == 0) *info = fail;
}

// Q_ij = y_i y_j K(x_i, x_j) from the full symmetric raw Gram, in place:
// row-major tiles, coalesced reads and writes (y = +-1 makes the products exact,
// so both triangles are bitwise what the reference's (i, j) / (j, i) order gives)
__global__ void svm_kernel_epilogue(double* Q, int64_t N, const double* y, const double* sq,
                                    int kind, double two_sigma2) {
  for (int64_t i = blockIdx.y; i < N; i += gridDim.y) {
    const double yi = y[i], si = (kind == RAC_KERNEL_GAUSSIAN) ? sq[i] : 0.0;
    double* row = Q + i * N;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < N; j += (int64_t)gridDim.x * blockDim.x) {
      double k = row[j];
      if (kind == RAC_KERNEL_GAUSSIAN) {
        const double d2 = fmax(sub(add(si, sq[j]), mul(2.0, k)), 0.0);
        k = exp(-d2 / two_sigma2);
      }
      row[j] = mul(mul(yi, k), y[j]);
    }
  }
}

__global__ void diag_copy_kernel(const double* Q, int64_t N, double* d) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
    d[i] = Q[i * N + i];
}

__global__ void iota_kernel(int32_t* v, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v[i] = (int32_t)i;
}

}  // namespace rac

// ---------------------------------------------------------------------------
struct rac_qp_ctx {
  int64_t n = 0, m = 0, lda = 0;
  int s = 0, p = 0, mode = 0;
  double beta = 1, ridge_rel = 0;
  cudaStream_t st = nullptr;
  int P = 0, nrc = 0;
  bool lsmem = true, ready = false, have_partition = false;
  rac::GramPlan gp{};
  int sweeps = 0, hist_cap = 0;
  double* H = nullptr;  // owned or borrowed
  bool own_h = false;
  double *Ac = nullptr, *b = nullptr, *c = nullptr, *lo = nullptr, *hi = nullptr;
  double *x = nullptr, *y = nullptr, *hx = nullptr, *ax = nullptr;
  int32_t *idx = nullptr, *order = nullptr, *info = nullptr;
  double *gram_ws = nullptr, *Mb = nullptr, *Hbb = nullptr, *inv = nullptr, *scratch = nullptr;
  double *partial = nullptr, *delta = nullptr, *pmax = nullptr, *psum = nullptr, *dmax = nullptr;
  double* lscratch = nullptr;
  double* hbx = nullptr;
  unsigned long long* llq = nullptr;   // tagged hand-off words of the chain (QpChainArgs::llq)
  unsigned llq_epoch = 0;              // chain launches so far (tagq0 = epoch (p + 1))
  double *Ninv = nullptr, *cond = nullptr;
  unsigned* bar = nullptr;
  int32_t* ctrl = nullptr;
  double *hist_p = nullptr, *hist_l1 = nullptr, *hist_d = nullptr;
  double div_bar = INFINITY;
  int rc = 32;   // rows per chunk of the A row phase (8 for few constraint rows)
  long long* trace = nullptr;   // 4 stamps per block of the last traced sweep
  // kernel strips on the fly (rac_qp_set_kernel_strips): no N x N matrix; per sweep the
  // blocks' H_bb and, batch by batch, the strip rows of sb blocks are formed from the samples
  bool strips = false;
  double *Xp = nullptr, *sq = nullptr, *lab = nullptr, *Hs = nullptr, *hblk = nullptr;
  int64_t ldd = 0, dfeat = 0;
  int kkind = 0, sb = 1;
  double ksigma = 1.0;
  std::vector<void*> allocs;
};

namespace {

template <typename T>
int qalloc(rac_qp_ctx* c, T** p, size_t count) {
  if (count == 0) count = 1;
  void* q = nullptr;
  const int rc = rac::dev_alloc(&q, count * sizeof(T), c->st);
  if (rc) return rc;
  c->allocs.push_back(q);
  *p = (T*)q;
  return RAC_OK;
}

size_t qp_smem_for(int rc, int s, bool rowphase, bool lsmem) {
  return rc == 8 ? rac::qp_smem_bytes<8>(s, rowphase, lsmem) : rac::qp_smem_bytes<32>(s, rowphase, lsmem);
}
size_t qp_smem(const rac_qp_ctx* c) { return qp_smem_for(c->rc, c->s, c->m > 0, c->lsmem); }
const void* qp_kernel(const rac_qp_ctx* c) {
  return c->rc == 8 ? (const void*)rac::qp_chain_kernel<8> : (const void*)rac::qp_chain_kernel<32>;
}

int qp_grow_history(rac_qp_ctx* c, int need) {
  if (need <= c->hist_cap) return RAC_OK;
  int cap = std::max(need, std::max(64, 2 * c->hist_cap));
  double *hp, *hl, *hd;
  int rc;
  if ((rc = qalloc(c, &hp, cap)) || (rc = qalloc(c, &hl, cap)) || (rc = qalloc(c, &hd, cap))) return rc;
  if (c->hist_cap) {
    cudaMemcpyAsync(hp, c->hist_p, c->hist_cap * sizeof(double), cudaMemcpyDeviceToDevice, c->st);
    cudaMemcpyAsync(hl, c->hist_l1, c->hist_cap * sizeof(double), cudaMemcpyDeviceToDevice, c->st);
    cudaMemcpyAsync(hd, c->hist_d, c->hist_cap * sizeof(double), cudaMemcpyDeviceToDevice, c->st);
  }
  c->hist_p = hp;
  c->hist_l1 = hl;
  c->hist_d = hd;
  c->hist_cap = cap;
  return RAC_OK;
}

int qp_block_systems(rac_qp_ctx* c) {
  using namespace rac;
  int rc;
  if (c->m > 0) {
    rc = launch_gram(c->Ac, c->lda, c->m, c->idx, nullptr, c->s, c->p, c->gram_ws, c->gp, c->st, c->ctrl);
    if (rc) return rc;
  }
  SysArgs a{};
  if (c->strips) {
    // H_bb of every block straight from the samples (gathered rows and columns), one launch
    rc = launch_kernel_strip(c->Xp, c->ldd, c->dfeat, c->idx, c->s, c->s, c->lab, c->sq, c->kkind, c->ksigma,
                             c->hblk, c->s, c->st, c->idx, c->p);
    if (rc) return rc;
    a.hblk = c->hblk;
  }
  a.ws = (c->m > 0) ? c->gram_ws : nullptr;
  a.splits = c->gp.splits;
  a.div = 1.0;
  a.mul = c->beta;
  a.H = c->strips ? nullptr : c->H;
  a.ldh = c->n;
  a.idx = c->idx;
  a.shift = 0.0;
  a.ridge_rel = c->ridge_rel;
  a.s = c->s;
  a.inv = c->inv;
  a.mat_out = c->Mb;
  a.hbb_out = c->Hbb;
  a.inv2 = c->Ninv;
  a.cond_out = c->cond;
  a.scratch = c->scratch;
  a.info = c->info;
  a.mode = FACTOR_CHOL;
  a.done = c->ctrl;
  return launch_chol_system(a, c->p, c->st);
}

int qp_chain(rac_qp_ctx* c, double tol_p, double tol_d, int fixed, int t0, int t1) {
  using namespace rac;
  cudaMemsetAsync(c->bar, 0, sizeof(unsigned), c->st);
  QpChainArgs a{};
  if (c->llq) {
    if ((unsigned long long)(c->llq_epoch + 2u) * (unsigned)(c->p + 1) >= 0xfffffff0ull) {
      cudaMemsetAsync(c->llq, 0, 4 * (size_t)c->s * sizeof(unsigned long long), c->st);   // tag space used up
      c->llq_epoch = 0;
    }
    ++c->llq_epoch;
    a.llq = c->llq;
    a.tagq0 = c->llq_epoch * (unsigned)(c->p + 1);
  }
  a.n = c->n;
  a.m = c->m;
  a.lda = c->lda;
  a.s = c->s;
  a.p = c->p;
  a.nrc = c->nrc;
  a.H = c->strips ? c->Hs : c->H;
  a.strips = c->strips ? 1 : 0;
  a.t0 = t0;
  a.t1 = t1;
  a.Ac = c->Ac;
  a.b = c->b;
  a.c = c->c;
  a.lo = c->lo;
  a.hi = c->hi;
  a.idx = c->idx;
  a.order = (c->mode == RAC_MODE_RP) ? c->order : nullptr;
  a.Mb = c->Mb;
  a.Hbb = c->Hbb;
  a.inv = c->inv;
  a.info = c->info;
  a.x = c->x;
  a.y = c->y;
  a.hx = c->hx;
  a.ax = c->ax;
  a.partial = c->partial;
  a.delta = c->delta;
  a.pmax = c->pmax;
  a.psum = c->psum;
  a.dmax = c->dmax;
  a.lscratch = c->lscratch;
  a.bar = c->bar;
  a.ctrl = c->ctrl;
  a.beta = c->beta;
  a.tol_p = tol_p;
  a.tol_d = tol_d;
  a.div_bar = c->div_bar;
  a.fixed = fixed;
  a.sweep = c->sweeps;
  a.lsmem = c->lsmem ? 1 : 0;
  a.hist_p = c->hist_p;
  a.hist_l1 = c->hist_l1;
  a.hist_d = c->hist_d;
  a.hbx = c->hbx;
  a.trace = c->trace;
  a.Ninv = c->Ninv;
  a.cond = c->cond;
  void* args[] = {&a};
  cudaError_t e = launch_coop((const void*)qp_kernel(c), dim3(c->P), dim3(QPT), args, qp_smem(c), c->st);
  note_launch();
  return check_cuda(e, "qp_chain (cooperative launch)");
}

}  // namespace

extern "C" int rac_qp_create(rac_qp_ctx** out, int64_t n, int64_t m, int32_t block_size, int32_t mode,
                             double beta, double ridge_rel, void* stream) {
  using namespace rac;
  clear_error();
  if (!out || n < 1 || m < 0 || block_size < 1 || block_size > n || !(beta > 0) || ridge_rel < 0)
    return set_error(RAC_ERR_ARG, "rac_qp_create: bad arguments");
  if (mode != RAC_MODE_RAC && mode != RAC_MODE_RP && mode != RAC_MODE_CYCLIC)
    return set_error(RAC_ERR_ARG, "rac_qp_create: bad mode");
  if (block_size > RP_QMAX * RP_THREADS)
    return set_error(RAC_ERR_UNSUPPORTED, "block_size %d > %d", block_size, RP_QMAX * RP_THREADS);
  rac_qp_ctx* c = new rac_qp_ctx();
  c->n = n;
  c->m = m;
  c->lda = (m + 31) / 32 * 32;
  c->s = block_size;
  c->p = (int)((n + block_size - 1) / block_size);
  c->mode = mode;
  c->beta = beta;
  c->ridge_rel = ridge_rel;
  c->st = (cudaStream_t)stream;
  c->rc = (m <= 256) ? 8 : 32;
  c->nrc = (int)((std::max<int64_t>(m, 1) + c->rc - 1) / c->rc);
  c->lsmem = qp_smem_for(c->rc, c->s, m > 0, true) <= 224 * 1024;
  if (const char* e = getenv("RAC_QP_RESIDENT")) c->lsmem = c->lsmem && atoi(e) != 0;
  int rc = check_cuda(cudaFuncSetAttribute(qp_kernel(c), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)qp_smem(c)),
                      "qp chain smem attribute");
  if (rc) {
    delete c;
    return rc;
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, qp_kernel(c), QPT, qp_smem(c));
  if (per_sm < 1) {
    delete c;
    return set_error(RAC_ERR_UNSUPPORTED, "qp chain kernel does not fit (smem %zu)", qp_smem(c));
  }
  c->P = num_sms();
  if (m > 0) c->gp = plan_gram(m, c->s, c->p);
  const size_t sqs = (size_t)c->p * c->s * c->s;
  if ((rc = qalloc(c, &c->c, n)) || (rc = qalloc(c, &c->lo, n)) || (rc = qalloc(c, &c->hi, n)) ||
      (rc = qalloc(c, &c->x, n)) || (rc = qalloc(c, &c->hx, n)) || (rc = qalloc(c, &c->b, std::max<int64_t>(m, 1))) ||
      (rc = qalloc(c, &c->y, std::max<int64_t>(m, 1))) || (rc = qalloc(c, &c->ax, std::max<int64_t>(c->lda, 1))) ||
      (rc = qalloc(c, &c->idx, (size_t)c->p * c->s)) || (rc = qalloc(c, &c->order, c->p)) ||
      (rc = qalloc(c, &c->info, c->p)) || (rc = qalloc(c, &c->Mb, sqs)) || (rc = qalloc(c, &c->Hbb, sqs)) ||
      (rc = qalloc(c, &c->inv, sqs)) || (rc = qalloc(c, &c->partial, (size_t)c->P * c->s)) ||
      (rc = qalloc(c, &c->delta, 2 * (size_t)c->s)) || (rc = qalloc(c, &c->pmax, c->P)) || (rc = qalloc(c, &c->psum, c->P)) ||
      (rc = qalloc(c, &c->dmax, c->P)) || (rc = qalloc(c, &c->bar, 1)) || (rc = qalloc(c, &c->ctrl, 4)) ||
      (rc = qalloc(c, &c->hbx, 2 * (size_t)c->s)) || (rc = qalloc(c, &c->Ninv, sqs)) || (rc = qalloc(c, &c->cond, c->p))) {
    rac_qp_destroy(c);
    return rc;
  }
  if (m > 0 && (rc = qalloc(c, &c->gram_ws, gram_ws_bytes(m, c->s, c->p) / sizeof(double)))) {
    rac_qp_destroy(c);
    return rc;
  }
  size_t scr = chol_scratch_bytes(c->s, c->p);
  if (scr && (rc = qalloc(c, &c->scratch, scr / sizeof(double)))) {
    rac_qp_destroy(c);
    return rc;
  }
  {
    // tagged hx / partial hand-off of the chain (one grid barrier per block); RAC_QP_LL=0: two barriers
    const char* e = getenv("RAC_QP_LL");
    if (!(e && atoi(e) == 0)) {
      if ((rc = qalloc(c, &c->llq, 4 * (size_t)c->s))) {
        rac_qp_destroy(c);
        return rc;
      }
      cudaMemsetAsync(c->llq, 0, 4 * (size_t)c->s * sizeof(unsigned long long), c->st);
    }
  }
  if ((rc = qalloc(c, &c->lscratch, (size_t)c->s * (c->s + 1)))) {
    rac_qp_destroy(c);
    return rc;
  }
  if ((rc = qp_grow_history(c, 256))) {
    rac_qp_destroy(c);
    return rc;
  }
  cudaMemsetAsync(c->ctrl, 0, 4 * sizeof(int32_t), c->st);
  cudaMemsetAsync(c->info, 0, c->p * sizeof(int32_t), c->st);
  cudaMemsetAsync(c->y, 0, std::max<int64_t>(m, 1) * sizeof(double), c->st);
  cudaMemsetAsync(c->ax, 0, std::max<int64_t>(c->lda, 1) * sizeof(double), c->st);
  cudaMemsetAsync(c->hx, 0, n * sizeof(double), c->st);
  *out = c;
  return check_launch("rac_qp_create");
}

extern "C" int rac_qp_set_problem(rac_qp_ctx* c, const double* H, const double* A, const double* b,
                                  const double* cvec, const double* lower, const double* upper) {
  using namespace rac;
  clear_error();
  if (!c || !cvec || !lower || !upper) return set_error(RAC_ERR_ARG, "rac_qp_set_problem: null pointer");
  if ((c->m > 0) != (A != nullptr) || (c->m > 0 && !b))
    return set_error(RAC_ERR_ARG, "rac_qp_set_problem: A/b must be given iff m > 0");
  const size_t nb = c->n * sizeof(double);
  if (H && c->strips) return set_error(RAC_ERR_ARG, "rac_qp_set_problem: H given to a kernel-strip context");
  if (H) {
    if (!c->own_h) {
      int rc = qalloc(c, &c->H, (size_t)c->n * c->n);
      if (rc) return rc;
      c->own_h = true;
    }
    cudaMemcpyAsync(c->H, H, nb * c->n, cudaMemcpyDeviceToDevice, c->st);
  }
  if (c->m > 0) {
    int rc = qalloc(c, &c->Ac, (size_t)c->lda * c->n);
    if (rc) return rc;
    rc = launch_transpose_pad(A, c->m, c->n, c->lda, c->Ac, c->st);
    if (rc) return rc;
    cudaMemcpyAsync(c->b, b, c->m * sizeof(double), cudaMemcpyDeviceToDevice, c->st);
  }
  cudaMemcpyAsync(c->c, cvec, nb, cudaMemcpyDeviceToDevice, c->st);
  cudaMemcpyAsync(c->lo, lower, nb, cudaMemcpyDeviceToDevice, c->st);
  cudaMemcpyAsync(c->hi, upper, nb, cudaMemcpyDeviceToDevice, c->st);
  note_launch();
  clip0_kernel<<<(int)std::min<int64_t>((c->n + 255) / 256, 1184), 256, 0, c->st>>>(c->lo, c->hi, c->n, c->x);
  // running products at x0 and the divergence bar (engine.py:361-362)
  if (c->strips) {
    // strip mode serves the SVM dual: x0 = clip(0, 0, C) = 0, so Hx0 = 0 (checked below)
    std::vector<double> lo(c->n), hi(c->n);
    cudaMemcpyAsync(lo.data(), c->lo, nb, cudaMemcpyDeviceToHost, c->st);
    cudaMemcpyAsync(hi.data(), c->hi, nb, cudaMemcpyDeviceToHost, c->st);
    int rc = check_cuda(cudaStreamSynchronize(c->st), "qp set_problem sync");
    if (rc) return rc;
    for (int64_t i = 0; i < c->n; ++i)
      if (lo[i] > 0.0 || hi[i] < 0.0)
        return set_error(RAC_ERR_UNSUPPORTED, "kernel strips need 0 inside every box (x0 = 0)");
    cudaMemsetAsync(c->hx, 0, nb, c->st);
  } else if (c->H) {
    int rc = launch_gemv_rows(c->H, c->n, c->n, c->x, c->hx, c->st);
    if (rc) return rc;
  }
  double primal0 = 0.0;
  if (c->m > 0) {
    int rc = launch_gemv_rows(A, c->m, c->n, c->x, c->ax, c->st);
    if (rc) return rc;
    std::vector<double> ax(c->m), bh(c->m);
    cudaMemcpyAsync(ax.data(), c->ax, c->m * sizeof(double), cudaMemcpyDeviceToHost, c->st);
    cudaMemcpyAsync(bh.data(), c->b, c->m * sizeof(double), cudaMemcpyDeviceToHost, c->st);
    rc = check_cuda(cudaStreamSynchronize(c->st), "qp set_problem sync");
    if (rc) return rc;
    for (int64_t i = 0; i < c->m; ++i) primal0 = std::max(primal0, std::fabs(ax[i] - bh[i]));
  }
  c->div_bar = 1e8 * std::max(primal0, 1.0);
  c->ready = true;
  return check_launch("rac_qp_set_problem");
}

namespace rac {
// out = A x for the column-major (lda x n) copy of A: one thread per row, columns in order
__global__ void gemv_colmajor_kernel(const double* __restrict__ Ac, int64_t lda, int64_t m, int64_t n,
                                     const double* __restrict__ x, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int64_t j = 0; j < n; ++j) acc = fma(Ac[j * lda + i], x[j], acc);
    out[i] = acc;
  }
}
}  // namespace rac

// Start the next sweep from (x, y) instead of (clip(0, lo, hi), 0): the running products
// Hx and Ax are recomputed from x.  engine.run_sweep (engine.py:284-315) goes through this.
extern "C" int rac_qp_set_state(rac_qp_ctx* c, const double* x, const double* y) {
  using namespace rac;
  clear_error();
  if (!c || !x || (c->m > 0 && !y)) return set_error(RAC_ERR_ARG, "rac_qp_set_state: null pointer");
  if (!c->ready) return set_error(RAC_ERR_ARG, "rac_qp_set_state: call rac_qp_set_problem first");
  if (c->strips) return set_error(RAC_ERR_UNSUPPORTED, "rac_qp_set_state: not with kernel strips");
  cudaMemcpyAsync(c->x, x, c->n * sizeof(double), cudaMemcpyDeviceToDevice, c->st);
  if (c->m > 0) cudaMemcpyAsync(c->y, y, c->m * sizeof(double), cudaMemcpyDeviceToDevice, c->st);
  if (c->H) {
    int rc = launch_gemv_rows(c->H, c->n, c->n, c->x, c->hx, c->st);
    if (rc) return rc;
  }
  if (c->m > 0) {
    gemv_colmajor_kernel<<<(int)std::min<int64_t>((c->m + 127) / 128, 1184), 128, 0, c->st>>>(
        c->Ac, c->lda, c->m, c->n, c->x, c->ax);
    note_launch();
  }
  return check_launch("rac_qp_set_state");
}

// Kernel strips on the fly instead of a resident N x N matrix (svm.py:96-143): H_ij =
// labels_i labels_j K(x_i, x_j) is formed per sweep for the blocks' H_bb and batch by batch for
// the strip rows (at most max_strip_bytes of strips at a time).  Call before set_problem.
extern "C" int rac_qp_set_kernel_strips(rac_qp_ctx* c, const double* X, int64_t d, const double* labels,
                                        int32_t kind, double sigma, uint64_t max_strip_bytes) {
  using namespace rac;
  clear_error();
  if (!c || !X || !labels || d < 1) return set_error(RAC_ERR_ARG, "rac_qp_set_kernel_strips: bad arguments");
  if (kind == RAC_KERNEL_GAUSSIAN && !(sigma > 0)) return set_error(RAC_ERR_ARG, "sigma must be > 0");
  if (c->mode == RAC_MODE_RP)
    return set_error(RAC_ERR_UNSUPPORTED, "kernel strips: rp mode visits blocks out of table order");
  if (c->H || c->strips) return set_error(RAC_ERR_ARG, "rac_qp_set_kernel_strips: context already has H");
  const int64_t n = c->n, s = c->s;
  c->ldd = (d + 31) / 32 * 32;
  c->dfeat = d;
  c->kkind = kind;
  c->ksigma = sigma;
  const size_t row = (size_t)s * n * sizeof(double);
  c->sb = (int)std::max<int64_t>(1, std::min<int64_t>(c->p, (int64_t)(max_strip_bytes / std::max<size_t>(row, 1))));
  int rc;
  if ((rc = qalloc(c, &c->Xp, (size_t)n * c->ldd)) || (rc = qalloc(c, &c->sq, n)) || (rc = qalloc(c, &c->lab, n)) ||
      (rc = qalloc(c, &c->hblk, (size_t)c->p * s * s)) || (rc = qalloc(c, &c->Hs, (size_t)c->sb * s * n)))
    return rc;
  cudaMemsetAsync(c->Xp, 0, (size_t)n * c->ldd * sizeof(double), c->st);
  cudaMemcpy2DAsync(c->Xp, c->ldd * sizeof(double), X, d * sizeof(double), d * sizeof(double), n,
                    cudaMemcpyDeviceToDevice, c->st);
  cudaMemcpyAsync(c->lab, labels, n * sizeof(double), cudaMemcpyDeviceToDevice, c->st);
  if (kind == RAC_KERNEL_GAUSSIAN && (rc = launch_row_sqnorm(c->Xp, c->ldd, n, d, c->sq, c->st))) return rc;
  c->strips = true;
  return check_launch("rac_qp_set_kernel_strips");
}

extern "C" int rac_qp_borrow_h(rac_qp_ctx* c, const double* H) {
  using namespace rac;
  clear_error();
  if (!c || !H) return set_error(RAC_ERR_ARG, "rac_qp_borrow_h: null pointer");
  if (c->own_h) return set_error(RAC_ERR_ARG, "rac_qp_borrow_h: context already owns H");
  c->H = const_cast<double*>(H);
  return RAC_OK;
}

extern "C" int rac_qp_set_divergence_bar(rac_qp_ctx* c, double bar) {
  using namespace rac;
  clear_error();
  if (!c) return set_error(RAC_ERR_ARG, "null context");
  c->div_bar = bar;
  return RAC_OK;
}

extern "C" int rac_qp_set_partition(rac_qp_ctx* c, const int64_t* perm) {
  using namespace rac;
  clear_error();
  if (!c || !perm) return set_error(RAC_ERR_ARG, "rac_qp_set_partition: null pointer");
  if (!c->ready) return set_error(RAC_ERR_ARG, "rac_qp_set_partition: call rac_qp_set_problem first");
  int rc = launch_chunk_sort(perm, c->n, c->s, 1, c->idx, c->st);
  if (rc) return rc;
  rc = qp_block_systems(c);
  if (rc) return rc;
  c->have_partition = true;
  return RAC_OK;
}

extern "C" int rac_qp_run(rac_qp_ctx* c, const int64_t* perms, int32_t count, double tol_p, double tol_d,
                          int32_t fixed) {
  using namespace rac;
  clear_error();
  if (!c || count < 0) return set_error(RAC_ERR_ARG, "rac_qp_run: bad arguments");
  if (!c->ready) return set_error(RAC_ERR_ARG, "rac_qp_run: call rac_qp_set_problem first");
  if (c->mode == RAC_MODE_RAC && !perms && count > 0) return set_error(RAC_ERR_ARG, "rac_qp_run: perms required");
  if (c->mode == RAC_MODE_RP && !perms && count > 0) return set_error(RAC_ERR_ARG, "rac_qp_run: perms required");
  if (c->mode != RAC_MODE_RAC && !c->have_partition)
    return set_error(RAC_ERR_ARG, "rac_qp_run: rp/cyclic need rac_qp_set_partition");
  int rc = qp_grow_history(c, c->sweeps + count);
  if (rc) return rc;
  for (int k = 0; k < count; ++k) {
    if (c->mode == RAC_MODE_RAC) {
      rc = launch_chunk_sort(perms + (int64_t)k * c->n, c->n, c->s, 1, c->idx, c->st);
      if (rc) return rc;
      rc = qp_block_systems(c);
      if (rc) return rc;
    } else if (c->mode == RAC_MODE_RP) {
      rc = launch_order_cast(perms + (int64_t)k * c->p, c->p, c->order, c->st);
      if (rc) return rc;
    }
    if (c->strips) {
      // the sweep in batches of sb blocks: their kernel strips, then the chain over them
      for (int t0 = 0; t0 < c->p && !rc; t0 += c->sb) {
        const int t1 = std::min(c->p, t0 + c->sb);
        rc = launch_kernel_strip(c->Xp, c->ldd, c->dfeat, c->idx + (int64_t)t0 * c->s, (t1 - t0) * c->s, c->n,
                                 c->lab, c->sq, c->kkind, c->ksigma, c->Hs, c->n, c->st);
        if (!rc) rc = qp_chain(c, tol_p, tol_d, fixed, t0, t1);
      }
    } else {
      rc = qp_chain(c, tol_p, tol_d, fixed, 0, c->p);
    }
    if (rc) return rc;
    c->sweeps++;
  }
  return RAC_OK;
}

extern "C" int rac_qp_progress(rac_qp_ctx* c, int32_t* iterations, int32_t* status, int32_t* failed_block) {
  using namespace rac;
  clear_error();
  if (!c) return set_error(RAC_ERR_ARG, "rac_qp_progress: null context");
  int32_t h[4];
  int rc = check_cuda(cudaMemcpyAsync(h, c->ctrl, sizeof(h), cudaMemcpyDeviceToHost, c->st), "qp progress");
  if (rc) return rc;
  rc = check_cuda(cudaStreamSynchronize(c->st), "qp progress sync");
  if (rc) return rc;
  if (iterations) *iterations = h[1];
  if (status) *status = h[3];
  if (failed_block) *failed_block = h[2] - 1;
  return RAC_OK;
}

extern "C" int rac_qp_get(rac_qp_ctx* c, double* x, double* y, double* hx, double* ax) {
  using namespace rac;
  clear_error();
  if (!c) return set_error(RAC_ERR_ARG, "rac_qp_get: null context");
  if (x) cudaMemcpyAsync(x, c->x, c->n * sizeof(double), cudaMemcpyDeviceToDevice, c->st);
  if (y && c->m) cudaMemcpyAsync(y, c->y, c->m * sizeof(double), cudaMemcpyDeviceToDevice, c->st);
  if (hx) cudaMemcpyAsync(hx, c->hx, c->n * sizeof(double), cudaMemcpyDeviceToDevice, c->st);
  if (ax && c->m) cudaMemcpyAsync(ax, c->ax, c->m * sizeof(double), cudaMemcpyDeviceToDevice, c->st);
  return check_launch("rac_qp_get");
}

extern "C" int rac_qp_history(rac_qp_ctx* c, double* primal, double* primal_l1, double* dual, int32_t capacity) {
  using namespace rac;
  clear_error();
  if (!c || capacity < 0) return set_error(RAC_ERR_ARG, "rac_qp_history: bad arguments");
  int k = std::min(capacity, c->hist_cap);
  if (k <= 0) return RAC_OK;
  if (primal) cudaMemcpyAsync(primal, c->hist_p, k * sizeof(double), cudaMemcpyDeviceToDevice, c->st);
  if (primal_l1) cudaMemcpyAsync(primal_l1, c->hist_l1, k * sizeof(double), cudaMemcpyDeviceToDevice, c->st);
  if (dual) cudaMemcpyAsync(dual, c->hist_d, k * sizeof(double), cudaMemcpyDeviceToDevice, c->st);
  return check_launch("rac_qp_history");
}

extern "C" int rac_qp_set_trace(rac_qp_ctx* c, int32_t enable) {
  using namespace rac;
  clear_error();
  if (!c) return set_error(RAC_ERR_ARG, "rac_qp_set_trace: null context");
  if (enable && !c->trace) {
    int rc = qalloc(c, &c->trace, 22 * (size_t)c->p + 2 * (size_t)c->p * c->P);   // + 8 solve stats per block
    if (rc) return rc;
  }
  if (!enable) c->trace = nullptr;
  return RAC_OK;
}

extern "C" int rac_qp_trace(rac_qp_ctx* c, int64_t* host, int32_t capacity) {
  using namespace rac;
  clear_error();
  if (!c || !host || !c->trace) return set_error(RAC_ERR_ARG, "rac_qp_trace: tracing not enabled");
  const int k = std::min<int>(capacity, 22 * c->p + 2 * c->p * c->P);
  return check_cuda(cudaMemcpy(host, c->trace, k * sizeof(int64_t), cudaMemcpyDeviceToHost), "qp trace copy");
}

extern "C" int rac_qp_destroy(rac_qp_ctx* c) {
  if (!c) return RAC_OK;
  if (c->st) cudaStreamSynchronize(c->st);
  for (void* q : c->allocs) rac::dev_free(q, c->st);
  if (c->st) cudaStreamSynchronize(c->st);
  rac::trim_pool(rac::POOL_KEEP);   // see rac_en_destroy
  delete c;
  return RAC_OK;
}

extern "C" int rac_svm_build_q(const double* X, int64_t N, int64_t d, const double* labels, int32_t kind,
                               double sigma, double* Q, void* stream) {
  using namespace rac;
  clear_error();
  if (!X || !labels || !Q || N < 1 || d < 1) return set_error(RAC_ERR_ARG, "rac_svm_build_q: bad arguments");
  if (kind == RAC_KERNEL_GAUSSIAN && !(sigma > 0)) return set_error(RAC_ERR_ARG, "sigma must be > 0");
  if (N > 2000000000LL) return set_error(RAC_ERR_UNSUPPORTED, "N too large");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t ldd = (d + 31) / 32 * 32;
  double *Xp = nullptr, *sq = nullptr;
  int32_t* ids = nullptr;
  int rc = check_cuda(cudaMallocAsync((void**)&Xp, (size_t)N * ldd * sizeof(double), st), "malloc Xp");
  if (rc) return rc;
  cudaMallocAsync((void**)&sq, N * sizeof(double), st);
  cudaMallocAsync((void**)&ids, N * sizeof(int32_t), st);
  cudaMemsetAsync(Xp, 0, (size_t)N * ldd * sizeof(double), st);
  cudaMemcpy2DAsync(Xp, ldd * sizeof(double), X, d * sizeof(double), d * sizeof(double), N,
                    cudaMemcpyDeviceToDevice, st);
  iota_kernel<<<(int)std::min<int64_t>((N + 255) / 256, 4096), 256, 0, st>>>(ids, N);
  // full symmetric X X': on the int8 tensor cores (exact digit slices, gram_i8.cu) when its
  // 128 x 128 tiles fill the SMs (RAC_Q_I8=2 forces it, =0 keeps the FP64 DMMA tiles)
  const char* e8 = getenv("RAC_Q_I8");
  const int mode8 = e8 ? atoi(e8) : 1;
  const int64_t jt = (N + 127) / 128;
  void* ws8 = nullptr;
  size_t ws8b = 0;
  if (mode8 == 2 || (mode8 == 1 && jt * (jt + 1) / 2 >= num_sms())) {
    ws8b = gram_i8_ws_bytes(ldd, (int)N);
    if (cudaMallocAsync(&ws8, ws8b, st) != cudaSuccess) {
      cudaGetLastError();
      ws8 = nullptr;
    }
  }
  int* bad = nullptr;
  if (ws8 && cudaMallocAsync((void**)&bad, sizeof(int), st) != cudaSuccess) {
    cudaGetLastError();
    bad = nullptr;
  }
  if (ws8 && bad) {
    cudaMemsetAsync(bad, 0, sizeof(int), st);
    rc = launch_gram_i8(Xp, ldd, d, (int)N, Q, 1.0, 0, ws8, ws8b, st, bad);
    cudaFreeAsync(ws8, st);
    int hbad = 0;
    if (!rc) rc = check_cuda(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, st), "int8 flag");
    if (!rc) rc = check_cuda(cudaStreamSynchronize(st), "int8 flag");
    cudaFreeAsync(bad, st);
    if (!rc && hbad) {
      // heavy-tailed samples: the digit slices would lose FP64-level accuracy (gram_i8.cu)
      GramPlan pl = plan_gram(d, (int)N, 1);
      pl.splits = 1;
      pl.chunk = ldd;
      rc = launch_gram(Xp, ldd, d, ids, nullptr, (int)N, 1, Q, pl, st, nullptr, 1.0);
    }
  } else {
    if (ws8) cudaFreeAsync(ws8, st);
    GramPlan pl = plan_gram(d, (int)N, 1);
    pl.splits = 1;
    pl.chunk = ldd;
    rc = launch_gram(Xp, ldd, d, ids, nullptr, (int)N, 1, Q, pl, st, nullptr, 1.0);
  }
  if (rc) return rc;
  diag_copy_kernel<<<(int)std::min<int64_t>((N + 255) / 256, 4096), 256, 0, st>>>(Q, N, sq);
  {
    const int gx = (int)std::min<int64_t>((N + 255) / 256, 8);
    const int gy = (int)std::min<int64_t>(N, 148 * 64);
    svm_kernel_epilogue<<<dim3(gx, gy), 256, 0, st>>>(Q, N, labels, sq, kind, 2.0 * sigma * sigma);
  }
  cudaFreeAsync(Xp, st);
  cudaFreeAsync(sq, st);
  cudaFreeAsync(ids, st);
  note_launch(3);
  return check_launch("rac_svm_build_q");
}

extern "C" int rac_box_block_min(const double* M, const double* r, const double* lo, const double* hi, int32_t s,
                                 double* x, int32_t* info, void* stream) {
  using namespace rac;
  clear_error();
  if (!M || !r || !lo || !hi || !x || !info || s < 1) return set_error(RAC_ERR_ARG, "rac_box_block_min: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  double* L = nullptr;
  {
    int rc = check_cuda(cudaMallocAsync((void**)&L, (size_t)s * (s + 1) * sizeof(double), st), "malloc L");
    if (rc) return rc;
  }
  size_t smem = qp_smem_bytes<32>(s, false, false);
  int rc = check_cuda(cudaFuncSetAttribute(box_test_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                      "box smem attribute");
  if (rc) return rc;
  // RAC_BOX_PASSES (tests only): active-set pass budget instead of 10 s, e.g. 0 to run the
  // projected-gradient fallback of engine.py:175-186 directly from the clipped solution
  const char* ep = getenv("RAC_BOX_PASSES");
  const int passes = ep ? atoi(ep) : -1;
  box_test_kernel<<<1, QPT, smem, st>>>(M, r, lo, hi, s, x, info, L, passes);
  if (L) cudaFreeAsync(L, st);
  note_launch();
  return check_launch("rac_box_block_min");
}
