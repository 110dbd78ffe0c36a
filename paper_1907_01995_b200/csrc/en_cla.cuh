// Lookahead covariance chain for the elastic-net sweep (included by en.cu).
//
// Same block step as en_cov.cuh (covariance-update form of elastic_net.py:199-224):
//
//   v_t  = -c_b - q_b + xi_b + gamma (z_b - beta_b)        b = block visited at step t
//   D_t  = sys_b^{-1} v_t ,  beta_b += D_t                  (then z / xi prox, elastic_net.py:225-227)
//   q   += G[:, b] D_t                                      (q = G beta kept current)
//
// but the q update is taken off the critical path.  Step t only needs q at the
// s indices of block t.  Write base_t = q[b_t] including the deltas of steps
// < t - D; then
//
//   q[b_t] = base_t + sum_{d=1..D} T_{t,d} D_{t-d},   T_{t,d} = G[b_t, b_{t-d}]   (s x s tiles)
//
// so one step is two s x s mat-vecs (T_{t,1} D_{t-1}, sys^{-1} v) plus one
// exchange.  A launch runs `nsw` consecutive sweeps as ONE sequence of global
// steps u = q p + t (the tiles of a sweep's first blocks reach into the
// previous sweep of the batch), so a sweep boundary costs nothing.  Roles:
//
//   leader cluster (CTAs 0..L-1): rank k owns rows S_k of every block.  Main
//     warps: [A] T_1 term from register-resident rows, [B] v, [C] the rank's
//     partial inv[S_k,:]' v[S_k] (the inverse is symmetric) bulk-copied into
//     every rank's shared memory (mbarrier completion, no cluster barrier),
//     [D] D_t = sum_k P_k in fixed rank order.  Helper warps: TMA of the
//     coming steps' inverse rows and T tiles, gathers of c/xi/z/beta, base_t
//     (polled from the workers' messages), the T_{d>=2} terms.  Commit warps:
//     publish D_t[S_k] for the workers, commit beta/z/xi, and reduce each
//     sweep's residuals (rank 0 writes the history and the stop flag).
//   workers (CTAs L..): each owns whole 32-column segments of q (kept in
//     shared memory) and applies every D_j:  q[cols] += G[b_j, cols]' D_j
//     from cp.async-staged rows of G.  Right after D_j it publishes q at the
//     columns of the block visited at step j+D+1: exactly base_{j+D+1}.  The
//     leader's q_t (base + tiles) only feeds v_t; the workers' q is the
//     running state.
//
// With a tolerance, the sweeps after the converging one in the same launch run
// speculatively; every sweep snapshots beta/z/xi and cla_restore_kernel puts the
// converged sweep's values back (bitwise the state a per-sweep launch stops at;
// q is not restored: nothing sweeps after convergence and q is re-formed with G).
// All cross-CTA traffic on the chain is tagged 64-bit words
// (rac_common.cuh ll_store / ll_ok): a reader spins on the data itself.
// Results are deterministic (fixed reduction orders).
#pragma once

#include <cooperative_groups.h>

namespace rac {

constexpr int CLA_T = 512;     // threads per CTA (leader: 256 main + helper / commit warps; worker: all)
constexpr int CLA_MAIN = 256;  // leader critical-path threads (8 warps)
constexpr int CLA_HELP = 96;   // threads per leader helper group (3 warps; up to 2 groups, then 2 commit warps)
constexpr int CLA_DMAX = 3;
constexpr int CLA_BMAX = 4;    // sweeps per launch (batched preparation)
#ifndef RAC_CLA_BULK_PUSH
#define RAC_CLA_BULK_PUSH 1
#endif
constexpr bool kBulkPush = RAC_CLA_BULK_PUSH != 0;   // partial exchange by TMA bulk copies (else st.async)

struct EnClaArgs {
  const double* G;  // n x n row-major, X'X/m
  int64_t n;
  int s, p;
  int nsw;               // sweeps in this launch (RP: 1)
  const int32_t* idx;    // [nsw][p][s] block indices (by block id)
  const int32_t* order;  // RP visit order or null
  const double* inv;     // [nsw][p][s][s] by block id
  const double* T;       // [nsw p][D][s][s] by global step: T[u][d-1] = G[b_u, b_{u-d}]
  const int32_t* info;   // [nsw][p]
  const double* c;
  double *beta, *z, *xi, *q;
  unsigned long long* dpub;  // [nsw p][s][2]: delta lo/hi (tagged)
  unsigned long long* qst;   // [nsw p][s][2]: base q lo/hi (tagged)
  double* snap;              // [nsw][3][n] beta, z, xi after every sweep (null: no snapshots)
  int32_t* conv;             // [2] (launch's first sweep, converged sweep within the launch)
  unsigned* ccnt;            // [nsw] commits per sweep (all ranks), zero at launch: a coordinate
                             // revisited in the next sweep is gathered only after its commit
  int32_t* ctrl;
  double gamma, thr, den, tol;
  int sweep;                 // history index of the launch's first sweep
  unsigned tag;              // message tag, unique per launch of a context (never reused, never 0)
  double *hist_p, *hist_d;
  long long* trace;  // optional (rank 0): first sweep's phase stamps
  int D;             // lookahead depth 1..3
  int W;             // worker CTAs
  int segw;          // max 32-column segments per worker
  int R;             // worker ring slots of staged G rows
  int NS;            // leader tile slots (2 or 4; NS/2 helper groups)
  volatile long long* dbg;   // optional progress markers (mapped host memory; RAC debugging)
};

__host__ __device__ inline size_t cla_leader_doubles(int L, int s, int D, int NS) {
  const size_t sl = (size_t)(s + L - 1) / L;
  return (size_t)NS * (1 + D) * sl * s + (size_t)NS * 4 * sl + 3 * (size_t)NS * sl + 4 * (size_t)s +
         2 * (size_t)L * s + 21 * sl + 8 + 32 + 512 + 2 * (size_t)s + 16 + 4 * (size_t)L +
         (3 * (size_t)NS + 12) + ((size_t)NS * sl + 1) / 2 + 1;   // + residual slots, mbarriers, idx
}
__host__ __device__ inline size_t cla_worker_doubles(int s, int segw, int R) {
  const size_t cw = 32 * (size_t)segw;
  return (size_t)R * s * cw + 16 * cw + cw + 2 * (size_t)s + 2 * (size_t)s + (size_t)CLA_BMAX * cw;
  //      ring             partials  q    D x2          raw words (4s u32)  maps (2 ints x BMAX)
}
__host__ inline size_t cla_smem_bytes(int L, int s, int D, int NS, int segw, int R) {
  const size_t a = cla_leader_doubles(L, s, D, NS), b = cla_worker_doubles(s, segw, R);
  return (a > b ? a : b) * sizeof(double);
}

// global block id (row of idx / inv / info) of global step u
__device__ __forceinline__ int cla_gb(const EnClaArgs& a, int u) {
  const int q = u / a.p, t = u - q * a.p;
  return q * a.p + (a.order ? a.order[t] : t);
}

// T[u][d-1] = G[b_u, b_{u-d}] for the `nsw` sweeps of a batch (global steps u = q p + t,
// contiguous idx rows; RP: nsw == 1 and the visit order).  grid.x = nsw * p * D, 256
// threads: indices staged in shared memory, then 8 independent gathers per thread in
// flight (the kernel is L2-latency bound otherwise).
__global__ void __launch_bounds__(256) cla_tiles_kernel(const double* __restrict__ G, int64_t n, int s, int p,
                                                        int D, const int32_t* __restrict__ idx,
                                                        const int32_t* __restrict__ order, double* __restrict__ T,
                                                        const int32_t* done) {
  __shared__ int ri[256], ci[256];
  if (done && *done) return;
  const int u = blockIdx.x / D, d = blockIdx.x % D + 1;
  if (u - d < 0) return;
  auto gb = [&](int v) {
    const int q = v / p, t = v - q * p;
    return q * p + (order ? order[t] : t);
  };
  const int32_t* rsrc = idx + (int64_t)gb(u) * s;
  const int32_t* csrc = idx + (int64_t)gb(u - d) * s;
  for (int i = threadIdx.x; i < s; i += 256) {
    ri[i] = rsrc[i];
    ci[i] = csrc[i];
  }
  __syncthreads();
  double* out = T + ((int64_t)u * D + d - 1) * s * s;
  const int ss = s * s;
  for (int e0 = 0; e0 < ss; e0 += 8 * 256) {
    double v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int e = e0 + k * 256 + threadIdx.x;
      v[k] = 0.0;
      if (e < ss) {
        const int i = e / s, c = e - i * s;
        const int g = ri[i], h = ci[c];
        if (g >= 0 && h >= 0) v[k] = __ldg(G + (int64_t)g * n + h);
      }
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int e = e0 + k * 256 + threadIdx.x;
      if (e < ss) out[e] = v[k];
    }
  }
}

// after a multi-sweep launch with a tolerance: if sweep qc < nsw - 1 of the launch
// starting at `sweep0` converged, the later (speculative) sweeps are undone by
// restoring the snapshot of sweep qc
__global__ void cla_restore_kernel(const int32_t* conv, int sweep0, int nsw, int64_t n, const double* snap,
                                   double* beta, double* z, double* xi) {
  if (conv[0] != sweep0) return;
  const int qc = conv[1];
  if (qc < 0 || qc >= nsw - 1) return;
  const double* sn = snap + (int64_t)qc * 3 * n;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    beta[i] = sn[i];
    z[i] = sn[n + i];
    xi[i] = sn[2 * n + i];
  }
}

template <int L>
__device__ __forceinline__ void cla_leader(const EnClaArgs& a, double* sm, int U) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int s = a.s, p = a.p, D = a.D, NS = a.NS, NH = a.NS / 2;
  const int64_t n = a.n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int k = (int)cl.block_rank();
  const int sl = (s + L - 1) / L, j0 = min(s, k * sl), rows = min(s, j0 + sl) - j0;
  const int nswE = U / p;   // sweeps this launch runs
  const size_t tileD = (size_t)(1 + D) * sl * s;
  double* sTile = sm;                            // [NS][inv rows | T_1 rows | ... | T_D rows]
  double* sVec = sTile + (size_t)NS * tileD;     // [NS][4][sl]  c, xi, z, beta
  double* sBase = sVec + (size_t)NS * 4 * sl;    // [NS][sl]
  double* sTq = sBase + (size_t)NS * sl;         // [NS][sl]  sum_{d>=2} T_d D_{t-d}
  double* sK = sTq + (size_t)NS * sl;            // [NS][sl]  -c - base + xi + gamma (z - beta) - tq
  double* sDelta = sK + (size_t)NS * sl;         // [4][s]    ring of full deltas
  double* sRecv = sDelta + 4 * (size_t)s;        // [2][L][s] partials pushed by the ranks
  const int sl2 = (sl + 1) & ~1;                 // keeps the double2 views below 16-byte aligned
  double* sV = sRecv + 2 * (size_t)L * s;        // [sl2]
  double* wred = sV + sl2;                       // [32]
  double* sPart = wred + 32;                     // [16 * sl] T_1 partials (16 threads per row)
  double* sHPart = sPart + 16 * sl;              // [2][256] helper partials (8 per row, rows <= 32)
  double* sOut = sHPart + 512;                   // [2][s] this rank's partial (bulk-push source)
  double* sRes = sOut + 2 * s;                   // [2 sweeps][2 commit warps][sum, max]
  double* sAll = sRes + 8;                       // [2][L][2] per-rank sweep residuals (rank 0 receives)
  sAll = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(sAll) + 15) & ~uintptr_t(15));
  uint64_t* mb = reinterpret_cast<uint64_t*>(sAll + 4 * L);
  uint64_t *mb_tma = mb, *mb_tq = mb + NS, *mb_free = mb + 2 * NS, *mb_x = mb + 3 * NS, *mb_dl = mb + 3 * NS + 2,
           *mb_res = mb + 3 * NS + 6, *mb_all = mb + 3 * NS + 8;
  int* sIdx = reinterpret_cast<int*>(mb + 3 * NS + 10);   // [NS][sl] indices of this rank's rows
  if (tid == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(mb_tma + i, 1);
      mbar_init(mb_tq + i, CLA_HELP);
      mbar_init(mb_free + i, CLA_MAIN + 32);   // main warps + the step's commit warp
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(mb_x + i, 1);
      mbar_init(mb_res + i, 2);   // both commit warps flushed the sweep
      mbar_init(mb_all + i, 1);   // rank 0: every rank's residuals arrived
    }
    for (int i = 0; i < 4; ++i) mbar_init(mb_dl + i, CLA_MAIN);
    mbar_fence_init();
  }
  // the delta ring starts at zero: step 0's T_1 term (zero tile rows) reads slot 3, and
  // 0 * (stale shared memory left by an earlier kernel) must not become NaN
  for (int i = tid; i < 4 * s; i += blockDim.x) sDelta[i] = 0.0;
  cl.sync();   // every rank's barriers exist before anyone pushes into them
  const unsigned tag = a.tag;
  const double gamma = a.gamma;
  constexpr int HW0 = CLA_MAIN / 32;               // first helper warp
  constexpr int CW0 = HW0 + 2 * (CLA_HELP / 32);   // first commit warp

  if (warp < HW0) {
    // ------------------------------------------------------------ main warps: the critical path
    // step u: [A] T_1 term partials | [B] q_u, v | [C] P_k = inv[S_k,:]' v -> every rank |
    //         [D] D_u = sum_k P_k, signal the commit warp, wait for step u+1's inputs
    const bool tr = a.trace && k == 0 && tid == 0;
    long long* ck = a.trace ? a.trace + 16 + 16 * (size_t)p + s : nullptr;   // clock64 stamps, 8 per step
    // register-resident operands of the coming step (rows <= 16, s <= 256):
    //   t1r[i] = T_1[r][part + 16 i]   (16 threads per row)      ivr[q] = inv[q][tid]  (column tid)
    const int r16 = tid >> 4, part = tid & 15;
    double t1r[16], ivr[16];
    auto preload = [&](int u) {
      const int slot = u % NS;
      const double* I = sTile + (size_t)slot * tileD;
      const double* T1 = I + (size_t)sl * s;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int c = part + 16 * i;
        t1r[i] = (u >= 1 && r16 < rows && c < s) ? T1[(size_t)r16 * s + c] : 0.0;
      }
#pragma unroll
      for (int q = 0; q < 16; ++q) ivr[q] = (q < rows && tid < s) ? I[(size_t)q * s + tid] : 0.0;
    };
    if (tr) a.trace[0] = gtimer();
    if (tid == 0) mbar_spin_sleep(mb_tq + 0, 0u, 32);
    mbar_spin(mb_tma + 0, 0u);
    preload(0);
    named_bar_sync(1, CLA_MAIN);
    for (int u = 0; u < U; ++u) {
      const int slot = u % NS, xs = u & 1;
      const bool trs = tr && u < p;
      if (a.dbg && k == 0 && tid == 0) a.dbg[0] = u;
      if (trs) { a.trace[1 + 5 * u] = gtimer(); ck[8 * u + 0] = clock64(); }
      const double* dprev = sDelta + (size_t)((u - 1) & 3) * s;
      // [A] T_1 D_{u-1}: 16 threads per row, operands in registers, four chains
      if (r16 < rows) {
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
        for (int i = 0; i < 16; i += 4) {
          const int c = part + 16 * i;
          if (c < s) a0 += t1r[i] * dprev[c];
          if (c + 16 < s) a1 += t1r[i + 1] * dprev[c + 16];
          if (c + 32 < s) a2 += t1r[i + 2] * dprev[c + 32];
          if (c + 48 < s) a3 += t1r[i + 3] * dprev[c + 48];
        }
        sPart[tid] = (a0 + a1) + (a2 + a3);
      }
      if (trs) ck[8 * u + 1] = clock64();
      named_bar_sync(1, CLA_MAIN);
      if (trs) { a.trace[2 + 5 * u] = gtimer(); ck[8 * u + 2] = clock64(); }
      // [B] corr = tq + T_1 term;  v = (-c - base + xi + gamma (z - beta) - tq) - T_1 term
      if (tid < rows) {
        const int r = tid;
        const double2* pp = reinterpret_cast<const double2*>(sPart + 16 * r);
        double q8[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const double2 w = pp[i];
          q8[i] = w.x + w.y;
        }
        const double acc = ((q8[0] + q8[1]) + (q8[2] + q8[3])) + ((q8[4] + q8[5]) + (q8[6] + q8[7]));
        sV[r] = (sIdx[slot * sl + r] >= 0) ? sK[slot * sl + r] - acc : 0.0;
      }
      if (trs) ck[8 * u + 3] = clock64();
      named_bar_sync(1, CLA_MAIN);
      if (trs) { a.trace[3 + 5 * u] = gtimer(); ck[8 * u + 4] = clock64(); }
      // [C] P_k[j] = sum_q inv[q][j] v[q] (inverse symmetric), pushed to every rank
      if (tid < s) {
        double p0 = 0.0, p1 = 0.0, p2 = 0.0, p3 = 0.0;
#pragma unroll
        for (int q = 0; q < 16; q += 4) {
          if (q < rows) p0 += ivr[q] * sV[q];
          if (q + 1 < rows) p1 += ivr[q + 1] * sV[q + 1];
          if (q + 2 < rows) p2 += ivr[q + 2] * sV[q + 2];
          if (q + 3 < rows) p3 += ivr[q + 3] * sV[q + 3];
        }
        const double pj = (p0 + p1) + (p2 + p3);
        if (kBulkPush) {
          sOut[xs * s + tid] = pj;
          fence_proxy_async();   // generic writes -> visible to the bulk copy (async proxy)
        } else {
          const unsigned la = smem_u32(sRecv + ((size_t)xs * L + k) * s + tid);
          const unsigned lb = smem_u32(mb_x + xs);
#pragma unroll
          for (int pr = 0; pr < L; ++pr) st_async_f64(mapa_u32(la, pr), pj, mapa_u32(lb, pr));
        }
      }
      if (kBulkPush) named_bar_sync(1, CLA_MAIN);
      if (tid == 0) {
        mbar_arrive_expect_tx(mb_x + xs, (unsigned)(L * s * sizeof(double)));
        if (kBulkPush) {
          const unsigned la = smem_u32(sRecv + ((size_t)xs * L + k) * s);
          const unsigned lb = smem_u32(mb_x + xs);
#pragma unroll
          for (int pr = 0; pr < L; ++pr)
            bulk_s2peer(mapa_u32(la, pr), sOut + xs * s, (unsigned)(s * sizeof(double)), mapa_u32(lb, pr));
        }
        if (trs) { a.trace[4 + 5 * u] = gtimer(); ck[8 * u + 5] = clock64(); }
      }
      // while the exchange is in flight: operands of step u+1 into registers
      if (u + 1 < U) {
        mbar_spin(mb_tma + (u + 1) % NS, (unsigned)((u + 1) / NS) & 1u);
        preload(u + 1);
      }
      if (tid == 0) {
        mbar_spin_cluster(mb_x + xs, (unsigned)(u >> 1) & 1u);
        if (trs) { a.trace[5 + 5 * u] = gtimer(); ck[8 * u + 6] = clock64(); }
      }
      named_bar_sync(1, CLA_MAIN);
      // [D] D_u in fixed rank order
      double* dcur = sDelta + (size_t)(u & 3) * s;
      for (int j = tid; j < s; j += CLA_MAIN) {
        const double* rv = sRecv + (size_t)xs * L * s + j;
        double d = rv[0];
#pragma unroll
        for (int pr = 1; pr < L; ++pr) d += rv[(size_t)pr * s];
        dcur[j] = d;
      }
      mbar_arrive(mb_dl + (u & 3));     // the commit warp publishes D_u
      mbar_arrive(mb_free + slot);      // this slot is no longer read by the main warps
      if (tid == 0 && u + 1 < U) mbar_spin_sleep(mb_tq + (u + 1) % NS, (unsigned)((u + 1) / NS) & 1u, 32);
      if (trs) ck[8 * u + 7] = clock64();
      named_bar_sync(1, CLA_MAIN);
    }
  } else if (warp < CW0 && (warp - HW0) / (CLA_HELP / 32) < NH) {
    // ------------------------------------------------------------ helper groups: inputs of step u
    const int h = (warp - HW0) / (CLA_HELP / 32);
    const int gid = tid - CLA_MAIN - CLA_HELP * h;
    const int hb = 2 + h;                       // named barrier of this group
    double* hpart = sHPart + 256 * h;
    int ready_q = 0;
    for (int u = h; u < U; u += NH) {
      const int gbu = cla_gb(a, u), slot = u % NS;
      const unsigned ph = (unsigned)(u / NS) & 1u;
      const int32_t* bi = a.idx + (int64_t)gbu * s;
      if (u >= NS && gid == 0) mbar_spin_sleep(mb_free + slot, (unsigned)((u - NS) / NS) & 1u);
      named_bar_sync(hb, CLA_HELP);
      const int nd = min(D, u);
      double* tile = sTile + (size_t)slot * tileD;
      const bool htr = a.trace && k == 0 && gid == 0 && u < p;
      if (gid == 0) {
        fence_proxy_async();
        const unsigned bytes = (unsigned)(rows * s * sizeof(double));
        mbar_arrive_expect_tx(mb_tma + slot, bytes * (unsigned)(1 + nd));
        if (rows > 0) {
          bulk_g2s(tile, a.inv + (int64_t)gbu * s * s + (int64_t)j0 * s, bytes, mb_tma + slot);
          for (int d = 1; d <= nd; ++d)
            bulk_g2s(tile + (size_t)d * sl * s, a.T + (((int64_t)u * D + d - 1) * s + j0) * s, bytes, mb_tma + slot);
        }
        if (htr) a.trace[1 + 5 * p + 4 * u] = gtimer();
      }
      // beta / z / xi of this block may have been committed (by any rank) in the previous sweep
      // of this launch: gather only after all of its commits (the TMA above does not wait:
      // main's preload of this step needs it while it finishes the previous sweep)
      const int qu = u / p;
      if (qu >= 1 && ready_q < qu) {
        if (gid == 0) {
          if (a.dbg && k == 0) { a.dbg[1 + h] = u; a.dbg[3 + h] = 1; }
          while (ld_acquire_u32(a.ccnt + qu - 1) < (unsigned)(L * p)) __nanosleep(32);
        }
        ready_q = qu;
        named_bar_sync(hb, CLA_HELP);
      }
      double* vec = sVec + (size_t)slot * 4 * sl;
      if (gid < rows) {
        const int r = gid;
        const int g = bi[j0 + r];
        sIdx[slot * sl + r] = g;
        double base = 0.0;
        if (g >= 0) {
          // L1-bypassing loads (values written by other CTAs in this launch), consumed after the poll
          const double vc = ldcg(a.c + g), vx = ldcg(a.xi + g), vz = ldcg(a.z + g), vb = ldcg(a.beta + g);
          // base of step u (q with the deltas of steps < u - D), published by the owning worker
          const unsigned long long* w = a.qst + ((size_t)u * s + j0 + r) * 2;
          unsigned long long w0, w1;
          do {
            w0 = ld_relaxed_u64(w);
            w1 = ld_relaxed_u64(w + 1);
          } while (!(ll_ok(w0, tag) && ll_ok(w1, tag)));
          base = ll_value((unsigned)w0, (unsigned)w1);
          vec[r] = vc;
          vec[sl + r] = vx;
          vec[2 * sl + r] = vz;
          vec[3 * sl + r] = vb;
        } else {
          vec[r] = vec[sl + r] = vec[2 * sl + r] = vec[3 * sl + r] = 0.0;
        }
        sBase[slot * sl + r] = base;
      }
      cp_async_commit();
      if (gid == 0) {
        if (htr) a.trace[2 + 5 * p + 4 * u] = gtimer();
        // D_{u-2} in the ring: main's signal to the commit warp (phase of step u-2 of a 4-ring;
        // main cannot lap it: step u+2 needs this helper's tq(u+2))
        if (u >= 2 && nd >= 2) mbar_spin_sleep(mb_dl + ((u - 2) & 3), (unsigned)((u - 2) >> 2) & 1u, 32);
        mbar_spin_sleep(mb_tma + slot, ph, 32);
        if (htr) a.trace[3 + 5 * p + 4 * u] = gtimer();
      }
      cp_async_wait<0>();
      named_bar_sync(hb, CLA_HELP);
      // T_{d>=2} terms: 8 threads per row, partials combined in fixed order
      for (int e = gid; e < rows * 8; e += CLA_HELP) {
        const int r = e >> 3, pt = e & 7;
        double a0 = 0.0, a1 = 0.0;
        for (int d = 2; d <= nd; ++d) {
          const double* Td = tile + ((size_t)d * sl + r) * s;
          const double* dv = sDelta + (size_t)((u - d) & 3) * s;
          int c = pt;
          for (; c + 8 < s; c += 16) {
            a0 += Td[c] * dv[c];
            a1 += Td[c + 8] * dv[c + 8];
          }
          if (c < s) a0 += Td[c] * dv[c];
        }
        hpart[e] = a0 + a1;
      }
      named_bar_sync(hb, CLA_HELP);
      if (gid < rows) {
        const int r = gid;
        const double* pp = hpart + 8 * r;
        const double tq = ((pp[0] + pp[1]) + (pp[2] + pp[3])) + ((pp[4] + pp[5]) + (pp[6] + pp[7]));
        sTq[slot * sl + r] = tq;
        const double k1 = add(sub(-vec[r], sBase[slot * sl + r]), vec[sl + r]);   // -c - base + xi
        sK[slot * sl + r] = sub(add(k1, mul(gamma, sub(vec[2 * sl + r], vec[3 * sl + r]))), tq);
      }
      if (htr) a.trace[4 + 5 * p + 4 * u] = gtimer();
      mbar_arrive(mb_tq + slot);
    }
  } else if (warp >= CW0) {
    // ------------------------------------------------------------ commit warps (alternate steps):
    // publish D_u[S_k] and corr for the workers, commit beta / z / xi, and per sweep
    // reduce the residuals (rank 0: history, stop flag)
    const int cw = warp - CW0;
    double my_sum = 0.0, my_max = 0.0;
    bool converged = false;   // rank 0, commit warp 0
    auto flush = [&](int q) {
      const double ssum = warp_sum(my_sum), smax = warp_max(my_max);
      my_sum = 0.0;
      my_max = 0.0;
      if (lane == 0) {
        sRes[((q & 1) * 2 + cw) * 2 + 0] = ssum;
        sRes[((q & 1) * 2 + cw) * 2 + 1] = smax;
        mbar_arrive(mb_res + (q & 1));
      }
      if (cw != 0 || lane != 0) return;
      // rank total (fixed commit-warp order) -> rank 0
      mbar_spin(mb_res + (q & 1), (unsigned)(q >> 1) & 1u);
      const double* rs = sRes + (q & 1) * 4;
      const double tot_k = rs[0] + rs[2], mx_k = fmax(rs[1], rs[3]);
      const unsigned la = smem_u32(sAll + ((q & 1) * L + k) * 2);
      st_async_f64x2(mapa_u32(la, 0), tot_k, mx_k, mapa_u32(smem_u32(mb_all + (q & 1)), 0));
      if (k != 0) return;
      mbar_arrive_expect_tx(mb_all + (q & 1), (unsigned)(L * 2 * sizeof(double)));
      mbar_spin_cluster(mb_all + (q & 1), (unsigned)(q >> 1) & 1u);
      double tot = 0.0, mx = 0.0;
      for (int r = 0; r < L; ++r) {
        tot += sAll[((q & 1) * L + r) * 2];
        mx = fmax(mx, sAll[((q & 1) * L + r) * 2 + 1]);
      }
      const int sw = a.sweep + q;
      a.hist_p[sw] = tot;
      a.hist_d[sw] = gamma * mx;
      if (!converged) {
        a.ctrl[1] = sw + 1;
        if (a.tol >= 0.0 && tot <= a.tol) {
          converged = true;
          a.conv[0] = a.sweep;
          a.conv[1] = q;
          a.ctrl[0] = 1;
          a.ctrl[3] = 1;
        }
      }
    };
    int qcur = 0;
    for (int u = cw; u < U; u += 2) {
      const int qu = u / p;
      while (qcur < qu) flush(qcur++);
      const int slot = u % NS;
      if (a.dbg && k == 0 && lane == 0) a.dbg[5 + cw] = u;
      if (lane == 0) mbar_spin_sleep(mb_dl + (u & 3), (unsigned)(u >> 2) & 1u, 32);
      __syncwarp();
      const double* vec = sVec + (size_t)slot * 4 * sl;
      const double* dcur = sDelta + (size_t)(u & 3) * s;
      double* snap = a.snap ? a.snap + (int64_t)qu * 3 * n : nullptr;
      for (int r = lane; r < rows; r += 32) {
        const int jj = j0 + r, g = sIdx[slot * sl + r];
        const double d = dcur[jj];
        ll_store(a.dpub + ((size_t)u * s + jj) * 2, d, tag);
        if (g >= 0) {
          const double bn = add(vec[3 * sl + r], d);
          const double x0 = vec[sl + r], zo = vec[2 * sl + r];
          const double av = sub(x0, mul(gamma, bn));
          const double zn = __ddiv_rn(neg_shrink(av, a.thr), a.den);
          const double xn = sub(x0, mul(gamma, sub(bn, zn)));
          a.beta[g] = bn;
          a.z[g] = zn;
          a.xi[g] = xn;
          if (snap) {
            snap[g] = bn;
            snap[n + g] = zn;
            snap[2 * n + g] = xn;
          }
          my_sum += fabs(sub(bn, zn));
          my_max = fmax(my_max, fabs(sub(zn, zo)));
        }
      }
      __syncwarp();
      if (lane == 0) red_release_add_u32(a.ccnt + qu, 1u);   // this rank's rows of step u committed
      mbar_arrive(mb_free + slot);
    }
    while (qcur < nswE) flush(qcur++);
  }
  __syncthreads();
  cl.sync();   // peers' pushes into this CTA are complete before it exits
}

__device__ __forceinline__ void cla_worker(const EnClaArgs& a, double* sm, int w, int U) {
  const int s = a.s, p = a.p, D = a.D, R = a.R;
  const int64_t n = a.n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nseg = (int)((n + 31) / 32);
  const int sg0 = (int)((int64_t)nseg * w / a.W), sg1 = (int)((int64_t)nseg * (w + 1) / a.W);
  const int ns = sg1 - sg0;
  if (ns <= 0) return;
  const int64_t c0 = (int64_t)sg0 * 32, c1 = min64(n, (int64_t)sg1 * 32);
  const int ncol = (int)(c1 - c0);
  const int CW = 32 * a.segw;
  const int nswE = U / p;
  const unsigned tag = a.tag;

  double* sG = sm;                               // [R][s][CW]
  double* part = sG + (size_t)R * s * CW;        // [16][CW]
  double* sQ = part + 16 * (size_t)CW;           // [CW]
  double* sD = sQ + CW;                          // [2][s]
  unsigned* sW = reinterpret_cast<unsigned*>(sD + 2 * (size_t)s);   // [2][2s]
  int* stepmap = reinterpret_cast<int*>(sW + 4 * (size_t)s);         // [BMAX][CW] global step of the column's block
  int* posmap = stepmap + CLA_BMAX * CW;                              // [BMAX][CW] position in that block

  for (int e = tid; e < nswE * p * s; e += CLA_T) {
    const int u = e / s, i = e - u * s;
    const int g = a.idx[(int64_t)cla_gb(a, u) * s + i];
    if (g >= c0 && g < c1) {
      const int q = u / p;
      stepmap[q * CW + (g - c0)] = u;
      posmap[q * CW + (g - c0)] = i;
    }
  }
  for (int l = tid; l < ncol; l += CLA_T) sQ[l] = a.q[c0 + l];
  __syncthreads();
  // bases of steps 0..D: q as the launch starts
  for (int l = tid; l < ncol; l += CLA_T)
    for (int q = 0; q < nswE; ++q)
      if (stepmap[q * CW + l] <= D)
        ll_store(a.qst + ((size_t)stepmap[q * CW + l] * s + posmap[q * CW + l]) * 2, sQ[l], tag);

  // rows G[b_j, my columns] -> ring slot j % R, 16-byte cp.async by all threads
  // (one commit group per slot; padding rows read row 0, their delta is 0)
  const int chunks = ncol / 2;   // 16-byte pieces per row (ncol is even)
  auto issue = [&](int j) {
    const int slot = j % R;
    const int32_t* bi = a.idx + (int64_t)cla_gb(a, j) * s;
    for (int e = tid; e < s * chunks; e += CLA_T) {
      const int c = e / chunks, q2 = e - c * chunks;
      const int g = max(0, bi[c]);
      cp_async16(sG + ((size_t)slot * s + c) * CW + 2 * q2, a.G + (int64_t)g * n + c0 + 2 * q2);
    }
    cp_async_commit();
  };
  for (int j = 0; j < min(R, U); ++j) issue(j);

  int j = 0;
  while (j < U) {
    const int nw = min(2, U - j);
    const int nwords = nw * 2 * s;
    int ok1 = 0;
    // poll the tagged words of D_j (and D_{j+1}) in one round trip
    for (;;) {
      unsigned long long v[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int e = tid + i * CLA_T;
        v[i] = (e < nwords) ? ld_relaxed_u64(a.dpub + (size_t)j * 2 * s + e) : 0ull;
      }
      int bad0 = 0, bad1 = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int e = tid + i * CLA_T;
        if (e < nwords) {
          const int bad = !ll_ok(v[i], tag);
          if (e < 2 * s) bad0 |= bad; else bad1 |= bad;
          sW[e] = (unsigned)v[i];
        }
      }
      const int any0 = __syncthreads_or(bad0);
      const int any1 = __syncthreads_or(bad1);
      if (!any0) {
        ok1 = (nw > 1) && !any1;
        break;
      }
    }
    if (a.dbg && w == a.W - 1 && tid == 0) a.dbg[8] = j;
    if (a.trace && w == a.W - 1 && tid == 0 && j < p) {
      a.trace[1 + 9 * p + 2 * j] = gtimer();
      if (ok1 && j + 1 < p) a.trace[1 + 9 * p + 2 * (j + 1)] = -1;
    }
    for (int qd = 0; qd <= ok1; ++qd) {
      const int jj = j + qd, slot = jj % R;
      const unsigned* Wd = sW + (size_t)qd * 2 * s;
      double* dD = sD + (size_t)qd * s;
      for (int c = tid; c < s; c += CLA_T) dD[c] = ll_value(Wd[2 * c], Wd[2 * c + 1]);
      // ring slot jj landed: groups committed after it = slots issued ahead
      {
        const int ahead = min(U - 1, jj + R - 1) - jj;
        if (ahead >= 3) cp_async_wait<3>(); else if (ahead == 2) cp_async_wait<2>();
        else if (ahead == 1) cp_async_wait<1>(); else cp_async_wait<0>();
      }
      __syncthreads();
      const double* Gs = sG + (size_t)slot * s * CW;
      for (int sg = 0; sg < ns; ++sg) {
        double acc = 0.0, a1 = 0.0;
        int c = warp;
        for (; c + 16 < s; c += 32) {
          acc += Gs[(size_t)c * CW + sg * 32 + lane] * dD[c];
          a1 += Gs[(size_t)(c + 16) * CW + sg * 32 + lane] * dD[c + 16];
        }
        if (c < s) acc += Gs[(size_t)c * CW + sg * 32 + lane] * dD[c];
        part[warp * CW + sg * 32 + lane] = acc + a1;
      }
      __syncthreads();
      for (int l = tid; l < ncol; l += CLA_T) {
        double sum = part[l];
#pragma unroll
        for (int w2 = 1; w2 < 16; ++w2) sum += part[w2 * CW + l];
        const double qv = sQ[l] + sum;
        sQ[l] = qv;
        // base of the visit at step jj+D+1 (a column is visited once per sweep)
        for (int q = 0; q < nswE; ++q)
          if (stepmap[q * CW + l] == jj + D + 1)
            ll_store(a.qst + ((size_t)(jj + D + 1) * s + posmap[q * CW + l]) * 2, qv, tag);
      }
      __syncthreads();
      if (jj + R < U) issue(jj + R);
      if (a.trace && w == a.W - 1 && tid == 0 && jj < p) a.trace[2 + 9 * p + 2 * jj] = gtimer();
    }
    j += 1 + ok1;
  }
  for (int l = tid; l < ncol; l += CLA_T) a.q[c0 + l] = sQ[l];
}

template <int L>
__global__ void __launch_bounds__(CLA_T, 1) en_cla_kernel(EnClaArgs a) {
  if (a.ctrl[0]) return;
  extern __shared__ __align__(128) double cla_sm[];
  __shared__ int bad, nrun;
  if (threadIdx.x == 0) {
    // sweeps run: up to (not including) the first sweep with a non-PD block
    bad = 0;
    nrun = a.nsw;
    for (int q = 0; q < a.nsw && !bad; ++q)
      for (int t = 0; t < a.p; ++t) {
        const int b = q * a.p + (a.order ? a.order[t] : t);
        if (a.info[b]) {
          bad = b - q * a.p + 1;
          nrun = q;
          break;
        }
      }
  }
  __syncthreads();
  const int U = nrun * a.p;
  if (U > 0) {
    if ((int)blockIdx.x < L)
      cla_leader<L>(a, cla_sm, U);
    else
      cla_worker(a, cla_sm, (int)blockIdx.x - L, U);
  }
  if (bad && blockIdx.x == 0 && threadIdx.x == 0) {
    // after the sweeps before it: ordered behind rank 0's history writes (same thread
    // block, __syncthreads + cluster barrier at the leader's end)
    if (!(a.ctrl[0] && a.ctrl[3])) {
      a.ctrl[2] = bad;
      a.ctrl[0] = 1;
    }
  }
}

}  // namespace rac
