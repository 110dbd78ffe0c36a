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
// exchange.  Roles in one cooperative launch:
//
//   leader cluster (CTAs 0..L-1): rank k owns rows S_k of every block.  Main
//     warps: q_t[S_k] (T_1 term), v[S_k], partial P_k = inv[S_k,:]' v[S_k]
//     (the inverse is symmetric), P_k pushed into every peer's shared memory
//     with st.async (mbarrier completion, no cluster barrier), D_t = sum_k P_k
//     in fixed rank order, commit of beta/z/xi for S_k, D_t[S_k] and the
//     correction corr = q_t - base_t published as tagged messages.  Helper
//     warps: TMA of the next steps' inverse rows and T tiles, gathers of
//     c/xi/z/beta, base_t (polled from the workers' messages) and the
//     T_{d>=2} terms.
//   workers (CTAs L..): each owns whole 32-column segments of q (kept in
//     shared memory) and applies every D_j:  q[cols] += G[b_j, cols]' D_j
//     from TMA-staged rows of G, except for the columns of blocks j+1..j+D
//     (the leader accounts for those through the tiles; the worker adds the
//     leader's correction when it reaches that block).  After D_j it
//     publishes the base of block j+D+1 for the leader.
//
// All cross-CTA traffic on the chain is tagged 64-bit words (rac_common.cuh
// ll_store / ll_ok): a reader spins on the data itself.  Results are
// deterministic (fixed reduction orders) and equal the serial chain to
// rounding.
#pragma once

#include <cooperative_groups.h>

namespace rac {

constexpr int CLA_T = 512;     // threads per CTA (leader: 256 main + helper warps; worker: all)
constexpr int CLA_MAIN = 256;  // leader critical-path threads (8 warps)
constexpr int CLA_HELP = 96;   // threads per leader helper group (3 warps; up to 2 groups, then 2 commit warps)
constexpr int CLA_DMAX = 3;

struct EnClaArgs {
  const double* G;  // n x n row-major, X'X/m
  int64_t n;
  int s, p;
  const int32_t* idx;    // [p][s] block indices (by block id)
  const int32_t* order;  // RP visit order or null
  const double* inv;     // [p][s][s] by block id
  const double* T;       // [p][D][s][s] by visit position: T[t][d-1] = G[b_t, b_{t-d}]
  const int32_t* info;
  const double* c;
  double *beta, *z, *xi, *q;
  unsigned long long* dpub;  // [p][s][4]: delta lo/hi, corr lo/hi (tagged)
  unsigned long long* qst;   // [p][s][2]: base q lo/hi (tagged)
  double *wsum, *wmax;       // [L]
  int32_t* ctrl;
  double gamma, thr, den, tol;
  int sweep;
  double *hist_p, *hist_d;
  long long* trace;  // optional (rank 0, thread 0): 1 + 5 per step
  int D;             // lookahead depth 1..3
  int W;             // worker CTAs
  int segw;          // max 32-column segments per worker
  int R;             // worker ring slots of staged G rows
  int NS;            // leader tile slots (2 or 4; NS/2 helper warps)
};

__host__ __device__ inline size_t cla_leader_doubles(int L, int s, int D, int NS) {
  const size_t sl = (size_t)(s + L - 1) / L;
  return (size_t)NS * (1 + D) * sl * s + (size_t)NS * 4 * sl + 3 * (size_t)NS * sl + 4 * (size_t)s +
         2 * (size_t)L * s + 21 * sl + 8 + 32 + 512 + (3 * (size_t)NS + 6) + ((size_t)NS * sl + 1) / 2 + 1;   // + mbarriers, idx
}
__host__ __device__ inline size_t cla_worker_doubles(int s, int segw, int R) {
  const size_t cw = 32 * (size_t)segw;
  return (size_t)R * s * cw + 16 * cw + cw + 4 * (size_t)s + 4 * (size_t)s + cw + 2 * (size_t)R;
  //      ring             partials  q    D/corr x2     raw words (8s u32)    maps  mbar
}
__host__ inline size_t cla_smem_bytes(int L, int s, int D, int NS, int segw, int R) {
  const size_t a = cla_leader_doubles(L, s, D, NS), b = cla_worker_doubles(s, segw, R);
  return (a > b ? a : b) * sizeof(double);
}

// blockIdx.y = sweep of a batch: idx + y * p * s, T + y * p * D * s * s
__global__ void cla_tiles_kernel(const double* __restrict__ G, int64_t n, int s, int p, int D,
                                 const int32_t* __restrict__ idx, const int32_t* __restrict__ order,
                                 double* __restrict__ T, const int32_t* done) {
  if (done && *done) return;
  idx += (int64_t)blockIdx.y * p * s;
  T += (int64_t)blockIdx.y * p * D * s * s;
  const int t = blockIdx.x / D, d = blockIdx.x % D + 1;
  if (t - d < 0) return;
  const int b = order ? order[t] : t, b2 = order ? order[t - d] : t - d;
  const int32_t* ri = idx + (int64_t)b * s;
  const int32_t* ci = idx + (int64_t)b2 * s;
  double* out = T + ((int64_t)t * D + d - 1) * s * s;
  for (int i = threadIdx.y; i < s; i += blockDim.y) {
    const int g = ri[i];
    for (int c = threadIdx.x; c < s; c += blockDim.x) {
      const int h = ci[c];
      out[(int64_t)i * s + c] = (g >= 0 && h >= 0) ? G[(int64_t)g * n + h] : 0.0;
    }
  }
}

template <int L>
__device__ __forceinline__ void cla_leader(const EnClaArgs& a, double* sm) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int s = a.s, p = a.p, D = a.D, NS = a.NS, NH = a.NS / 2;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int k = (int)cl.block_rank();
  const int sl = (s + L - 1) / L, j0 = min(s, k * sl), rows = min(s, j0 + sl) - j0;
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
  double* sCorr = sV + sl2;                      // [4][sl2]  q_t - base_t (ring: read by the commit warps)
  double* wred = sCorr + 4 * sl2;                // [32]
  double* sPart = wred + 32;                     // [16 * sl] T_1 partials (16 threads per row)
  double* sHPart = sPart + 16 * sl;              // [2][256] helper partials (8 per row, rows <= 32)
  uint64_t* mb = reinterpret_cast<uint64_t*>(sHPart + 512);
  uint64_t *mb_tma = mb, *mb_tq = mb + NS, *mb_free = mb + 2 * NS, *mb_x = mb + 3 * NS, *mb_dl = mb + 3 * NS + 2;
  int* sIdx = reinterpret_cast<int*>(mb + 3 * NS + 6);   // [NS][sl] indices of this rank's rows
  if (tid == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(mb_tma + i, 1);
      mbar_init(mb_tq + i, CLA_HELP);
      mbar_init(mb_free + i, CLA_MAIN + 32);   // main warps + the step's commit warp
    }
    for (int i = 0; i < 2; ++i) mbar_init(mb_x + i, 1);
    for (int i = 0; i < 4; ++i) mbar_init(mb_dl + i, CLA_MAIN);
    mbar_fence_init();
  }
  cl.sync();   // every rank's barriers exist before anyone pushes into them
  const unsigned tag = (unsigned)a.sweep + 1u;
  const double gamma = a.gamma;
  auto blk = [&](int t) { return a.order ? a.order[t] : t; };
  double my_sum = 0.0, my_max = 0.0;
  constexpr int HW0 = CLA_MAIN / 32;               // first helper warp
  constexpr int CW0 = HW0 + 2 * (CLA_HELP / 32);   // first commit warp

  if (warp < HW0) {
    // ------------------------------------------------------------ main warps: the critical path
    // step t: [A] T_1 term partials | [B] q_t, v | [C] P_k = inv[S_k,:]' v -> every rank |
    //         [D] D_t = sum_k P_k, signal the commit warp, wait for step t+1's inputs
    const bool tr = a.trace && k == 0 && tid == 0;
    long long* ck = a.trace ? a.trace + 16 + 16 * (size_t)p + s : nullptr;   // clock64 stamps, 8 per step
    // register-resident operands of the coming step (rows <= 16, s <= 256):
    //   t1r[i] = T_1[r][part + 16 i]   (16 threads per row)      ivr[q] = inv[q][tid]  (column tid)
    const int r16 = tid >> 4, part = tid & 15;
    double t1r[16], ivr[16];
    auto preload = [&](int t) {
      const int slot = t % NS;
      const double* I = sTile + (size_t)slot * tileD;
      const double* T1 = I + (size_t)sl * s;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int c = part + 16 * i;
        t1r[i] = (t >= 1 && r16 < rows && c < s) ? T1[(size_t)r16 * s + c] : 0.0;
      }
#pragma unroll
      for (int q = 0; q < 16; ++q) ivr[q] = (q < rows && tid < s) ? I[(size_t)q * s + tid] : 0.0;
    };
    if (tr) a.trace[0] = gtimer();
    if (p > 0) {
      if (tid == 0) mbar_spin_sleep(mb_tq + 0, 0u, 32);
      mbar_spin(mb_tma + 0, 0u);
      preload(0);
    }
    named_bar_sync(1, CLA_MAIN);
    for (int t = 0; t < p; ++t) {
      const int slot = t % NS, xs = t & 1;
      if (tr) { a.trace[1 + 5 * t] = gtimer(); ck[8 * t + 0] = clock64(); }
      const double* dprev = sDelta + (size_t)((t - 1) & 3) * s;
      // [A] T_1 D_{t-1}: 16 threads per row, operands in registers, four chains
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
      if (tr) ck[8 * t + 1] = clock64();
      named_bar_sync(1, CLA_MAIN);
      if (tr) { a.trace[2 + 5 * t] = gtimer(); ck[8 * t + 2] = clock64(); }
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
        sCorr[(t & 3) * sl2 + r] = sTq[slot * sl + r] + acc;
        sV[r] = (sIdx[slot * sl + r] >= 0) ? sK[slot * sl + r] - acc : 0.0;
      }
      if (tr) ck[8 * t + 3] = clock64();
      named_bar_sync(1, CLA_MAIN);
      if (tr) { a.trace[3 + 5 * t] = gtimer(); ck[8 * t + 4] = clock64(); }
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
        const unsigned la = smem_u32(sRecv + ((size_t)xs * L + k) * s + tid);
        const unsigned lb = smem_u32(mb_x + xs);
#pragma unroll
        for (int pr = 0; pr < L; ++pr) st_async_f64(mapa_u32(la, pr), pj, mapa_u32(lb, pr));
      }
      if (tid == 0) {
        mbar_arrive_expect_tx(mb_x + xs, (unsigned)(L * s * sizeof(double)));
        if (tr) { a.trace[4 + 5 * t] = gtimer(); ck[8 * t + 5] = clock64(); }
      }
      // while the exchange is in flight: operands of step t+1 into registers
      if (t + 1 < p) {
        mbar_spin(mb_tma + (t + 1) % NS, (unsigned)((t + 1) / NS) & 1u);
        preload(t + 1);
      }
      if (tid == 0) {
        mbar_spin_cluster(mb_x + xs, (unsigned)(t >> 1) & 1u);
        if (tr) { a.trace[5 + 5 * t] = gtimer(); ck[8 * t + 6] = clock64(); }
      }
      named_bar_sync(1, CLA_MAIN);
      // [D] D_t in fixed rank order
      double* dcur = sDelta + (size_t)(t & 3) * s;
      for (int j = tid; j < s; j += CLA_MAIN) {
        const double* rv = sRecv + (size_t)xs * L * s + j;
        double d = rv[0];
#pragma unroll
        for (int pr = 1; pr < L; ++pr) d += rv[(size_t)pr * s];
        dcur[j] = d;
      }
      mbar_arrive(mb_dl + (t & 3));     // the commit warp publishes D_t
      mbar_arrive(mb_free + slot);      // this slot is no longer read by the main warps
      if (tid == 0 && t + 1 < p) mbar_spin_sleep(mb_tq + (t + 1) % NS, (unsigned)((t + 1) / NS) & 1u, 32);
      if (tr) ck[8 * t + 7] = clock64();
      named_bar_sync(1, CLA_MAIN);
    }
  } else if (warp < CW0 && (warp - HW0) / (CLA_HELP / 32) < NH) {
    // ------------------------------------------------------------ helper groups: inputs of step u
    const int h = (warp - HW0) / (CLA_HELP / 32);
    const int gid = tid - CLA_MAIN - CLA_HELP * h;
    const int hb = 2 + h;                       // named barrier of this group
    double* hpart = sHPart + 256 * h;
    for (int u = h; u < p; u += NH) {
      const int b = blk(u), slot = u % NS;
      const unsigned ph = (unsigned)(u / NS) & 1u;
      const int32_t* bi = a.idx + (int64_t)b * s;
      if (u >= NS && gid == 0) mbar_spin_sleep(mb_free + slot, (unsigned)((u - NS) / NS) & 1u);
      named_bar_sync(hb, CLA_HELP);
      const int nd = min(D, u);
      double* tile = sTile + (size_t)slot * tileD;
      const bool htr = a.trace && k == 0 && gid == 0;
      if (gid == 0) {
        fence_proxy_async();
        const unsigned bytes = (unsigned)(rows * s * sizeof(double));
        mbar_arrive_expect_tx(mb_tma + slot, bytes * (unsigned)(1 + nd));
        if (rows > 0) {
          bulk_g2s(tile, a.inv + (int64_t)b * s * s + (int64_t)j0 * s, bytes, mb_tma + slot);
          for (int d = 1; d <= nd; ++d)
            bulk_g2s(tile + (size_t)d * sl * s, a.T + (((int64_t)u * D + d - 1) * s + j0) * s, bytes, mb_tma + slot);
        }
        if (htr) a.trace[1 + 5 * p + 4 * u] = gtimer();
      }
      double* vec = sVec + (size_t)slot * 4 * sl;
      if (gid < rows) {
        const int r = gid;
        const int g = bi[j0 + r];
        sIdx[slot * sl + r] = g;
        double base = 0.0;
        if (g >= 0) {
          cp_async8(vec + r, a.c + g);
          cp_async8(vec + sl + r, a.xi + g);
          cp_async8(vec + 2 * sl + r, a.z + g);
          cp_async8(vec + 3 * sl + r, a.beta + g);
          // base of block u (q with the deltas of steps < u - D), published by the owning worker
          const unsigned long long* w = a.qst + ((size_t)u * s + j0 + r) * 2;
          unsigned long long w0, w1;
          do {
            w0 = ld_relaxed_u64(w);
            w1 = ld_relaxed_u64(w + 1);
          } while (!(ll_ok(w0, tag) && ll_ok(w1, tag)));
          base = ll_value((unsigned)w0, (unsigned)w1);
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
      long long* hk = (htr) ? a.trace + 16 + 24 * (size_t)p + s + 4 * u : nullptr;
      if (hk) hk[0] = clock64();
      cp_async_wait<0>();
      named_bar_sync(hb, CLA_HELP);
      if (hk) hk[1] = clock64();
      // T_{d>=2} terms: 8 threads per row, partials combined in fixed order
      for (int e = gid; e < rows * 8; e += CLA_HELP) {
        const int r = e >> 3, part = e & 7;
        double a0 = 0.0, a1 = 0.0;
        for (int d = 2; d <= nd; ++d) {
          const double* Td = tile + ((size_t)d * sl + r) * s;
          const double* dv = sDelta + (size_t)((u - d) & 3) * s;
          int c = part;
          for (; c + 8 < s; c += 16) {
            a0 += Td[c] * dv[c];
            a1 += Td[c + 8] * dv[c + 8];
          }
          if (c < s) a0 += Td[c] * dv[c];
        }
        hpart[e] = a0 + a1;
      }
      if (hk) hk[2] = clock64();
      named_bar_sync(hb, CLA_HELP);
      if (hk) hk[3] = clock64();
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
    // publish D_t[S_k] and corr for the workers, then beta / z / xi and the residuals
    for (int t = warp - CW0; t < p; t += 2) {
      const int slot = t % NS;
      if (lane == 0) mbar_spin_sleep(mb_dl + (t & 3), (unsigned)(t >> 2) & 1u, 32);
      __syncwarp();
      const double* vec = sVec + (size_t)slot * 4 * sl;
      const double* dcur = sDelta + (size_t)(t & 3) * s;
      for (int r = lane; r < rows; r += 32) {
        const int jj = j0 + r, g = sIdx[slot * sl + r];
        const double d = dcur[jj];
        unsigned long long* w = a.dpub + ((size_t)t * s + jj) * 4;
        ll_store(w, d, tag);
        ll_store(w + 2, sCorr[(t & 3) * sl2 + r], tag);
        if (g >= 0) {
          const double bn = add(vec[3 * sl + r], d);
          const double x0 = vec[sl + r], zo = vec[2 * sl + r];
          a.beta[g] = bn;
          const double av = sub(x0, mul(gamma, bn));
          const double zn = __ddiv_rn(neg_shrink(av, a.thr), a.den);
          a.z[g] = zn;
          a.xi[g] = sub(x0, mul(gamma, sub(bn, zn)));
          my_sum += fabs(sub(bn, zn));
          my_max = fmax(my_max, fabs(sub(zn, zo)));
        }
      }
      __syncwarp();
      mbar_arrive(mb_free + slot);
    }
  }
  // residuals: warp -> CTA -> rank 0
  __syncwarp();
  my_sum = warp_sum(my_sum);
  my_max = warp_max(my_max);
  __syncthreads();
  if (lane == 0) {
    wred[warp] = my_sum;
    wred[16 + warp] = my_max;
  }
  __syncthreads();
  if (tid == 0) {
    double tot = 0.0, mx = 0.0;
    for (int w2 = 0; w2 < CLA_T / 32; ++w2) {
      tot += wred[w2];
      mx = fmax(mx, wred[16 + w2]);
    }
    a.wsum[k] = tot;
    a.wmax[k] = mx;
  }
  cl.sync();
  if (k == 0 && tid == 0) {
    double tot = 0.0, mx = 0.0;
    for (int r = 0; r < L; ++r) {
      tot += ldcg(a.wsum + r);
      mx = fmax(mx, ldcg(a.wmax + r));
    }
    a.hist_p[a.sweep] = tot;
    a.hist_d[a.sweep] = gamma * mx;
    a.ctrl[1] = a.sweep + 1;
    if (a.tol >= 0.0 && tot <= a.tol) {
      a.ctrl[0] = 1;
      a.ctrl[3] = 1;
    }
  }
}

__device__ __forceinline__ void cla_worker(const EnClaArgs& a, double* sm, int w) {
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
  const unsigned tag = (unsigned)a.sweep + 1u;
  auto blk = [&](int t) { return a.order ? a.order[t] : t; };

  double* sG = sm;                               // [R][s][CW]
  double* part = sG + (size_t)R * s * CW;        // [16][CW]
  double* sQ = part + 16 * (size_t)CW;           // [CW]
  double* sD = sQ + CW;                          // [2][s]
  double* sC = sD + 2 * (size_t)s;               // [2][s]
  unsigned* sW = reinterpret_cast<unsigned*>(sC + 2 * (size_t)s);   // [2][4s]
  int* blkmap = reinterpret_cast<int*>(sW + 8 * (size_t)s);          // [CW]
  int* posmap = blkmap + CW;                                          // [CW]
  uint64_t* mb_g = reinterpret_cast<uint64_t*>(sC + 2 * (size_t)s + 4 * (size_t)s + CW);   // [R]

  if (tid == 0) {
    for (int i = 0; i < R; ++i) mbar_init(mb_g + i, 1);
    mbar_fence_init();
  }
  for (int e = tid; e < p * s; e += CLA_T) {
    const int t = e / s, i = e - t * s;
    const int g = a.idx[(int64_t)blk(t) * s + i];
    if (g >= c0 && g < c1) {
      blkmap[g - c0] = t;
      posmap[g - c0] = i;
    }
  }
  for (int l = tid; l < ncol; l += CLA_T) sQ[l] = a.q[c0 + l];
  __syncthreads();
  // bases of the first D+1 blocks: q as the sweep starts
  for (int l = tid; l < ncol; l += CLA_T)
    if (blkmap[l] <= D) ll_store(a.qst + ((size_t)blkmap[l] * s + posmap[l]) * 2, sQ[l], tag);

  // rows G[b_j, my columns] -> ring slot j % R, 16-byte cp.async by all threads
  // (one commit group per slot; padding rows read row 0, their delta is 0)
  const int chunks = ncol / 2;   // 16-byte pieces per row (ncol is even)
  auto issue = [&](int j) {
    const int slot = j % R;
    const int32_t* bi = a.idx + (int64_t)blk(j) * s;
    for (int e = tid; e < s * chunks; e += CLA_T) {
      const int c = e / chunks, q2 = e - c * chunks;
      const int g = max(0, bi[c]);
      cp_async16(sG + ((size_t)slot * s + c) * CW + 2 * q2, a.G + (int64_t)g * n + c0 + 2 * q2);
    }
    cp_async_commit();
  };
  for (int j = 0; j < min(R, p); ++j) issue(j);

  int j = 0;
  while (j < p) {
    const int nw = min(2, p - j);
    const int nwords = nw * 4 * s;
    int ok1 = 0;
    // poll the tagged words of D_j (and D_{j+1}) in one round trip
    for (;;) {
      unsigned long long v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = tid + u * CLA_T;
        v[u] = (e < nwords) ? ld_relaxed_u64(a.dpub + (size_t)j * 4 * s + e) : 0ull;
      }
      int bad0 = 0, bad1 = 0;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = tid + u * CLA_T;
        if (e < nwords) {
          const int bad = !ll_ok(v[u], tag);
          if (e < 4 * s) bad0 |= bad; else bad1 |= bad;
          sW[e] = (unsigned)v[u];
        }
      }
      const int any0 = __syncthreads_or(bad0);
      const int any1 = __syncthreads_or(bad1);
      if (!any0) {
        ok1 = (nw > 1) && !any1;
        break;
      }
    }
    if (a.trace && w == a.W - 1 && tid == 0) {
      a.trace[1 + 9 * p + 2 * j] = gtimer();
      if (ok1) a.trace[1 + 9 * p + 2 * (j + 1)] = -1;
    }
    for (int qd = 0; qd <= ok1; ++qd) {
      const int jj = j + qd, slot = jj % R;
      const unsigned* Wd = sW + (size_t)qd * 4 * s;
      double* dD = sD + (size_t)qd * s;
      double* dC = sC + (size_t)qd * s;
      for (int c = tid; c < s; c += CLA_T) {
        dD[c] = ll_value(Wd[4 * c], Wd[4 * c + 1]);
        dC[c] = ll_value(Wd[4 * c + 2], Wd[4 * c + 3]);
      }
      // ring slot jj landed: groups committed after it = min(R, p) - 1 - ... (slots issued ahead)
      {
        const int ahead = min(p - 1, jj + R - 1) - jj;   // groups issued after slot jj
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
        const int t = blkmap[l];
        double qv = sQ[l];
        if (t == jj) qv = qv + dC[posmap[l]];   // the leader's q_t for this block's columns
        if (!(t > jj && t <= jj + D)) {
          double sum = part[l];
#pragma unroll
          for (int w2 = 1; w2 < 16; ++w2) sum += part[w2 * CW + l];
          qv += sum;
        }
        sQ[l] = qv;
        if (t == jj + D + 1) ll_store(a.qst + ((size_t)t * s + posmap[l]) * 2, qv, tag);
      }
      __syncthreads();
      if (jj + R < p) issue(jj + R);
      if (a.trace && w == a.W - 1 && tid == 0) a.trace[2 + 9 * p + 2 * jj] = gtimer();
    }
    j += 1 + ok1;
  }
  for (int l = tid; l < ncol; l += CLA_T) a.q[c0 + l] = sQ[l];
}

template <int L>
__global__ void __launch_bounds__(CLA_T, 1) en_cla_kernel(EnClaArgs a) {
  if (a.ctrl[0]) return;
  extern __shared__ __align__(128) double cla_sm[];
  __shared__ int bad;
  if (threadIdx.x == 0) {
    bad = 0;
    for (int t = 0; t < a.p; ++t) {
      const int b = a.order ? a.order[t] : t;
      if (a.info[b]) {
        bad = b + 1;
        break;
      }
    }
  }
  __syncthreads();
  if (bad) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      a.ctrl[2] = bad;
      a.ctrl[0] = 1;
    }
    return;
  }
  if ((int)blockIdx.x < L)
    cla_leader<L>(a, cla_sm);
  else
    cla_worker(a, cla_sm, (int)blockIdx.x - L);
}

}  // namespace rac
