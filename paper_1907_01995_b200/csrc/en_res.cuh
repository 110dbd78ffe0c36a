// Resident-tile cluster chain for the elastic-net sweep (included by en.cu).
//
// Every CTA owns a fixed set of 32-row chunks of X.  The columns of the
// current block stay RESIDENT in shared memory from the row phase that used
// them as "next" to the one that applies their update, and everything the
// next blocks need — X column segments (one 256-byte TMA bulk copy each,
// SASS UBLKCP, completing on an mbarrier), rows of inv_b (one bulk copy),
// beta/c/xi/z at the block's indices (cp.async gathers) — is prefetched while
// the current block is solved.  The sweep's whole block table sits in shared
// memory.  CTAs form clusters of CS that pre-reduce partials through DSMEM and
// split the s x s mat-vec.  Per block: two cluster barriers + one grid
// barrier; the row phase is pure shared-memory arithmetic.
//
//   R(t)   r += X[rows, b_t] delta_t ;  partial_{t+1} = X[rows, b_{t+1}]'(r - X beta)
//   cl.sync; rank slice of the cluster sum -> global (double-buffered by parity)
//   grid barrier
//   every CTA: full rhs (elastic_net.py:205-206) from the C cluster partials
//   rank: delta rows of its slice = inv_b rhs - beta (smem-resident inv rows)
//   cl.sync; gather delta from the cluster
// Cluster 0 commits beta/z/xi of block t after the grid barrier of block t+1
// (nobody reads block t's coordinates after that point in the sweep).
#pragma once

#include <cooperative_groups.h>

namespace rac {

namespace cg = cooperative_groups;

constexpr int RES_RC = 32;        // rows per chunk (one 256-byte segment per column)
constexpr int RES_PAD = 4;        // tile column padding (doubles): column stride = 8 banks mod 32

struct ResSmem {
  double* tiles;   // [2][s][nch*32+4]  (column segments: TMA destination)
  double* ginv;    // [sl][s]            inv_b rows of this rank's slice
  double* cxz;     // [3][s]             c, xi, z at the block's indices
  double* sX;      // [2][s]             beta at a block's indices, by block parity
  double* sDel;    // [s]                full delta of the current block
  double* sRhs;    // [s]
  double* sPart;   // [s]                this CTA's partial (cluster peers read it)
  double* sSlice;  // [2s]               this rank's delta | new beta (global block positions)
  double* cm;      // [3s]               block awaiting commit: new beta, old xi, old z
  double* sR;      // [nch*32]           resident rows of r
  double* red;     // [2][nch][8 warps][32]  row-phase reductions; [s] rhs sums
  double* sT;      // [nch*32]
  uint64_t* bars;  // [3]                tile slot 0/1, solve data
  int* pend;       // [s]
  int* sIdx;       // [p*s]              this sweep's block table
};

// row-phase reductions; for CS >= 4 also the staged [s][C] cluster partials
template <int CS>
__host__ __device__ size_t res_red_doubles(int s, int nch) {
  const size_t rp = 2 * (size_t)nch * (ENT / 32) * RES_RC;
  const size_t st = (CS >= 4) ? (size_t)s * (148 / CS + 1) : 0;
  return rp > st ? rp : st;
}

template <int CS>
__host__ __device__ size_t res_smem_bytes(int s, int nch, int p) {
  const size_t sl = (s + CS - 1) / CS;
  return (2 * (size_t)s * (nch * RES_RC + RES_PAD) + sl * s + 13 * (size_t)s + (size_t)nch * RES_RC +
          res_red_doubles<CS>(s, nch) + (size_t)nch * RES_RC + 6) *
             sizeof(double) +
         ((size_t)s + (size_t)p * s) * sizeof(int);
}

template <int CS>
__device__ __forceinline__ ResSmem carve_res(double* base, int s, int nch) {
  const int sl = (s + CS - 1) / CS;
  ResSmem w;
  double* p = base;
  w.tiles = p; p += 2 * (size_t)s * (nch * RES_RC + RES_PAD);
  w.ginv = p; p += (size_t)sl * s;
  w.cxz = p; p += 3 * s;
  w.sX = p; p += 2 * s;
  w.sDel = p; p += s;
  w.sRhs = p; p += s;
  w.sPart = p; p += s;
  w.sSlice = p; p += 2 * s;
  w.cm = p; p += 3 * s;
  w.sR = p; p += (size_t)nch * RES_RC;
  w.red = p; p += res_red_doubles<CS>(s, nch);
  p = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(p) + 15) & ~uintptr_t(15));  // double2 loads
  w.sT = p; p += (size_t)nch * RES_RC;
  w.bars = reinterpret_cast<uint64_t*>(p); p += 4;
  w.pend = reinterpret_cast<int*>(p);
  w.sIdx = w.pend + s;
  return w;
}

template <int CS>
__global__ void __launch_bounds__(ENT) en_chain_res_kernel(EnChainArgs a, int nch) {
  if (a.ctrl[0]) return;
  constexpr int RC = RES_RC;
  extern __shared__ __align__(128) double rsm[];
  cg::cluster_group cl = cg::this_cluster();
  const int s = a.s;
  const ResSmem w = carve_res<CS>(rsm, s, nch);
  __shared__ int bad;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = ENT / 32;
  const int P = gridDim.x, C = P / CS;
  const int rank = (int)cl.block_rank(), cid = blockIdx.x / CS;
  const int sl = (s + CS - 1) / CS, j0 = min(s, rank * sl), j1 = min(s, j0 + sl);
  unsigned target = 0;
  if (tid == 0) {
    bad = 0;
    for (int t = 0; t < a.p; ++t) {
      int b = a.order ? a.order[t] : t;
      if (a.info[b]) { bad = b + 1; break; }
    }
    for (int q = 0; q < 3; ++q) mbar_init(w.bars + q, 1);
    mbar_fence_init();
  }
  for (int e = tid; e < a.p * s; e += ENT) w.sIdx[e] = a.idx[e];
  __syncthreads();
  if (bad) {
    if (blockIdx.x == 0 && tid == 0) { a.ctrl[2] = bad; a.ctrl[0] = 1; }
    return;
  }
  const double m = a.mdiv, gamma = a.gamma;
  const bool tr = a.trace && blockIdx.x == 0 && tid == 0;
  int tp = 0;
  if (tr) a.trace[tp++] = gtimer();
  auto blk = [&](int t) { return a.order ? a.order[t] : t; };
  auto bidx = [&](int b) { return w.sIdx + (size_t)b * s; };
  // CTA q owns the contiguous chunks q*nch .. q*nch+nchv-1, so one column of a
  // block is ONE bulk copy of nchv*256 bytes; slot layout T[j][nch*RC].
  // column stride padded by 2 doubles: 16-byte loads of 8 consecutive columns hit
  // 8 distinct bank quads (pass 3 is column-per-thread)
  const int RCN = nch * RC + RES_PAD;
  auto tile = [&](int slot) { return w.tiles + (size_t)slot * s * RCN; };
  const int nchv = max(0, min(nch, a.nrc - (int)blockIdx.x * nch));  // valid chunks of this CTA
  const int64_t row0 = (int64_t)blockIdx.x * nch * RC;
  for (int k = 0; k < nchv; ++k) {
    const int64_t i0 = row0 + (int64_t)k * RC;
    for (int i = tid; i < RC; i += ENT) w.sR[k * RC + i] = (i0 + i < a.m) ? a.r[i0 + i] : 0.0;
  }
  unsigned par[3] = {0u, 0u, 0u};
  const bool bulk_inv = ((s & 1) == 0);  // 16-byte aligned rows of inv
  // TMA fetch of block b's column segments into a tile slot, plus beta at the
  // block's indices (cp.async) into sX[parity].  The slot must be dead.
  auto issue_tile = [&](int slot, int b, double* xdst) {
    const int nvalid = (int)min64(s, a.n - (int64_t)b * s);
    if (tid == 0) {
      fence_proxy_async();
      mbar_arrive_expect_tx(w.bars + slot, (unsigned)(nchv * nvalid * RC * sizeof(double)));
    }
    __syncthreads();
    const int* bi = bidx(b);
    if (nchv > 0)
      for (int j = tid; j < s; j += ENT) {
        double* dst = tile(slot) + (size_t)j * RCN;
        const int g = bi[j];
        if (g >= 0) bulk_g2s(dst, a.Xc + (int64_t)g * a.ld + row0, (unsigned)(nchv * RC * sizeof(double)), w.bars + slot);
        else
          for (int i = 0; i < nchv * RC; ++i) dst[i] = 0.0;
      }
    for (int j = tid; j < s; j += ENT) {
      const int g = bi[j];
      if (g >= 0) cp_async8(xdst + j, a.beta + g);
      else xdst[j] = 0.0;
    }
  };
  auto wait_tile = [&](int slot) {
    mbar_wait(w.bars + slot, par[slot]);
    par[slot] ^= 1u;
  };
  // inv rows of the slice (bulk) + c/xi/z at the block's indices (cp.async); commits the group
  auto issue_solve = [&](int b) {
    const int* bi = bidx(b);
    const double* Ib = a.inv + (int64_t)b * s * s + (int64_t)j0 * s;
    const int rows = j1 - j0;
    if (bulk_inv) {
      if (tid == 0) {
        mbar_arrive_expect_tx(w.bars + 2, (unsigned)(rows * s * sizeof(double)));
        if (rows > 0) bulk_g2s(w.ginv, Ib, (unsigned)(rows * s * sizeof(double)), w.bars + 2);
      }
    } else {
      for (int e = tid; e < rows * s; e += ENT) cp_async8(w.ginv + e, Ib + e);
    }
    for (int j = tid; j < s; j += ENT) {
      const int g = bi[j];
      if (g >= 0) {
        cp_async8(w.cxz + j, a.c + g);
        cp_async8(w.cxz + s + j, a.xi + g);
        cp_async8(w.cxz + 2 * s + j, a.z + g);
      } else {
        w.cxz[j] = 0.0;
        w.cxz[s + j] = 0.0;
        w.cxz[2 * s + j] = 0.0;
      }
    }
    cp_async_commit();
  };
  auto wait_solve = [&]() {
    if (bulk_inv) {
      mbar_wait(w.bars + 2, par[2]);
      par[2] ^= 1u;
    }
    cp_async_wait<0>();
  };
  // one row phase: optional r-update with slot sp (delta in sDel) and optional
  // partial for slot sn (x values in xs) -> sPart.  Layout T[j][i], lanes = rows.
  // All chunks of the CTA go through each pass together: two __syncthreads per
  // row phase whatever nch is.
  auto row_phase_res = [&](int sp, int sn, const double* xs) {
    double* redp = w.red;                              // [nch][nw][RC]
    double* redn = w.red + (size_t)nch * nw * RC;      // [nch][nw][RC]
    // up to 4 chunks per pass over j: independent accumulators, same j order per chunk
    for (int kb = 0; kb < nchv; kb += 4) {
      const int kn = min(4, nchv - kb);
      double up[4] = {0.0, 0.0, 0.0, 0.0}, un[4] = {0.0, 0.0, 0.0, 0.0};
      if (sp >= 0) {
        const double* T = tile(sp) + kb * RC + lane;
        for (int j = warp; j < s; j += nw) {
          const double d = w.sDel[j];
          const double* Tj = T + (size_t)j * RCN;
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (u < kn) up[u] += Tj[u * RC] * d;
        }
      }
      if (sn >= 0) {
        const double* T = tile(sn) + kb * RC + lane;
        for (int j = warp; j < s; j += nw) {
          const double x = xs[j];
          const double* Tj = T + (size_t)j * RCN;
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (u < kn) un[u] += Tj[u * RC] * x;
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (u < kn) {
          redp[((kb + u) * nw + warp) * RC + lane] = up[u];
          redn[((kb + u) * nw + warp) * RC + lane] = un[u];
        }
    }
    if (tr) a.trace[tp++] = gtimer();
    __syncthreads();
    if (tr) a.trace[tp++] = gtimer();
    for (int e = tid; e < nchv * RC; e += ENT) {
      const int k = e / RC, i = e - k * RC;
      const int64_t i0 = row0 + (int64_t)k * RC;
      const int rows = (int)min64(RC, a.m - i0);
      double* rr = w.sR + k * RC;
      if (sp >= 0 && i < rows) {
        double tot = redp[(k * nw) * RC + i];
        for (int q = 1; q < nw; ++q) tot += redp[(k * nw + q) * RC + i];
        rr[i] += tot;
      }
      if (sn >= 0) {
        double tot = redn[(k * nw) * RC + i];
        for (int q = 1; q < nw; ++q) tot += redn[(k * nw + q) * RC + i];
        w.sT[k * RC + i] = (i < rows) ? rr[i] - tot : 0.0;
      }
    }
    __syncthreads();
    if (tr) a.trace[tp++] = gtimer();
    if (sn >= 0) {
      // partial_j = sum_i T[j][i] t_i : two lanes per column (s <= 128) taking
      // alternate 16-byte row pairs; combined with one shuffle
      const double* T = tile(sn);
      const int nr2 = nchv * RC / 2;
      const int tpc = (2 * s <= ENT) ? 2 : 1;
      const double2* tt = reinterpret_cast<const double2*>(w.sT);
      for (int e0 = 0; e0 < s * tpc; e0 += ENT) {
        const int e = e0 + tid;
        const int j = e / tpc, h = e - j * tpc;
        double v = 0.0;
        if (j < s) {
          const double2* col = reinterpret_cast<const double2*>(T + (size_t)j * RCN);
          double a0 = 0.0, a1 = 0.0;
          for (int k = h; k < nr2; k += tpc) {
            const double2 x = col[k], y = tt[k];
            a0 += x.x * y.x;
            a1 += x.y * y.y;
          }
          v = a0 + a1;
        }
        if (tpc == 2) v += __shfl_xor_sync(0xffffffffu, v, 1);
        if (j < s && h == 0) w.sPart[j] = v;
      }
    }
  };

  double my_sum = 0.0, my_max = 0.0;
  // beta/z/xi of the block whose new values sit in cm; coordinate j of the
  // block is written by CTA j mod P
  auto commit = [&](const int* bip) {
    for (int j = (int)blockIdx.x + tid * P; j < s; j += ENT * P) {
      const int g = bip[j];
      if (g < 0) continue;
      const double bn = w.cm[j];
      a.beta[g] = bn;
      const double x0 = w.cm[s + j], zo = w.cm[2 * s + j];
      const double av = sub(x0, mul(gamma, bn));
      const double zn = __ddiv_rn(neg_shrink(av, a.thr), a.den);
      a.z[g] = zn;
      a.xi[g] = sub(x0, mul(gamma, sub(bn, zn)));
      my_sum += fabs(sub(bn, zn));
      my_max = fmax(my_max, fabs(sub(zn, zo)));
    }
  };
  // rhs reduction over the C cluster partials: the global partials are laid
  // out [s][C], so one warp reads the C partials of an entry as contiguous
  // 256-byte lines; 4 entries x RES_QL loads per lane are in flight at once.
  constexpr int RES_QL = (148 / CS + 31) / 32;

  // ---- prologue: tiles (+ beta) of blocks 0 and 1, solve data of block 0
  issue_tile(0, blk(0), w.sX);
  cp_async_commit();
  if (a.p > 1) issue_tile(1, blk(1), w.sX + s);
  issue_solve(blk(0));
  wait_tile(0);
  cp_async_wait<1>();   // beta of block 0
  __syncthreads();
  row_phase_res(-1, 0, w.sX);
  if (tr) a.trace[tp++] = gtimer();

  for (int t = 0; t < a.p; ++t) {
    const int b = blk(t);
    const int* bi = bidx(b);
    const double* xb = w.sX + (t & 1) * s;         // beta of block t
    // ---- cluster pre-reduction, grid barrier
    cl.sync();
    if (tr) a.trace[tp++] = gtimer();
    double* gpart = a.partial + (int64_t)(t & 1) * C * s;
    for (int j = j0 + tid; j < j1; j += ENT) {
      double acc = 0.0;
      for (int q = 0; q < CS; ++q) acc += cl.map_shared_rank(w.sPart, q)[j];
      gpart[(int64_t)j * C + cid] = acc;
    }
    if (tr) a.trace[tp++] = gtimer();
    grid_barrier(a.bar, target, P);
    if (tr) a.trace[tp++] = gtimer();
    if (t > 0) commit(bidx(blk(t - 1)));
    if (tr) a.trace[tp++] = gtimer();
    // ---- full rhs
    if constexpr (CS >= 4) {
      // s*C partials (<= 19 per thread for s <= 256) staged into smem in one round
      // trip, then entry j sums its C partials in cluster order
      const int tot = s * C;
      for (int f0 = tid; f0 < tot; f0 += 8 * ENT) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int f = f0 + u * ENT;
          v[u] = (f < tot) ? ldcg(gpart + f) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int f = f0 + u * ENT;
          if (f < tot) w.red[f] = v[u];
        }
      }
    } else
    for (int jb = warp; jb < s; jb += 4 * nw) {
      double v[4][RES_QL];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int j = jb + u * nw;
#pragma unroll
        for (int ql = 0; ql < RES_QL; ++ql) {
          const int q = lane + 32 * ql;
          v[u][ql] = (j < s && q < C) ? ldcg(gpart + (int64_t)j * C + q) : 0.0;
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        double acc = v[u][0];
#pragma unroll
        for (int ql = 1; ql < RES_QL; ++ql) acc += v[u][ql];
        acc = warp_sum(acc);
        const int j = jb + u * nw;
        if (lane == 0 && j < s) w.red[j] = acc;
      }
    }
    if (tr) a.trace[tp++] = gtimer();
    wait_solve();
    if (tr) a.trace[tp++] = gtimer();
    __syncthreads();
    for (int j = tid; j < s; j += ENT) {
      double acc;
      if constexpr (CS >= 4) {
        const double* pj = w.red + (size_t)j * C;
        acc = pj[0];
        for (int q = 1; q < C; ++q) acc += pj[q];
      } else {
        acc = w.red[j];
      }
      double rhs = 0.0;
      if (bi[j] >= 0) {
        const double cross = acc / m;
        rhs = -(sub(sub(add(w.cxz[j], cross), w.cxz[s + j]), mul(gamma, w.cxz[2 * s + j])));
      }
      w.sRhs[j] = rhs;
    }
    __syncthreads();
    if (tr) a.trace[tp++] = gtimer();
    // ---- delta rows of this rank's slice: 4 lanes-groups of 8 per row
    {
      const int rows = j1 - j0;
      const int sub8 = lane >> 3, l8 = lane & 7;      // 4 rows per warp, 8 lanes per row
      for (int r0 = warp * 4; r0 < rows; r0 += nw * 4) {
        const int i = j0 + r0 + sub8;
        double acc = 0.0;
        if (r0 + sub8 < rows) {
          const double* row = w.ginv + (int64_t)(i - j0) * s;
          for (int j = l8; j < s; j += 8) acc += row[j] * w.sRhs[j];
        }
        acc += __shfl_xor_sync(0xffffffffu, acc, 4);
        acc += __shfl_xor_sync(0xffffffffu, acc, 2);
        acc += __shfl_xor_sync(0xffffffffu, acc, 1);
        if (l8 == 0 && r0 + sub8 < rows) {
          const int g = bi[i];
          w.sSlice[i] = (g >= 0) ? acc - xb[i] : 0.0;
          w.sSlice[s + i] = acc;
        }
      }
    }
    cl.sync();
    if (tr) a.trace[tp++] = gtimer();
    for (int i = tid; i < s; i += ENT) {
      const double* peer = cl.map_shared_rank(w.sSlice, i / sl);
      w.sDel[i] = peer[i];
      w.cm[i] = peer[s + i];            // new beta
      w.cm[s + i] = w.cxz[s + i];       // xi, z of block t before its update
      w.cm[2 * s + i] = w.cxz[2 * s + i];
    }
    // ---- row phase (tile of b resident, tile + beta of the next block prefetched)
    const bool more = t + 1 < a.p;
    if (more) {
      wait_tile((t + 1) & 1);
      cp_async_wait<1>();   // beta of block t+1 (committed before the last solve group)
    }
    __syncthreads();
    if (tr) a.trace[tp++] = gtimer();
    row_phase_res(t & 1, more ? ((t + 1) & 1) : -1, w.sX + ((t + 1) & 1) * s);
    if (tr) a.trace[tp++] = gtimer();
    if (more) {
      __syncthreads();   // slot t&1, sX[t&1], ginv, cxz are dead for every thread
      if (t + 2 < a.p) issue_tile(t & 1, blk(t + 2), w.sX + (t & 1) * s);
      cp_async_commit();
      issue_solve(blk(t + 1));
    }
    if (tr) a.trace[tp++] = gtimer();
  }
  for (int k = 0; k < nchv; ++k) {
    const int64_t i0 = row0 + (int64_t)k * RC;
    for (int i = tid; i < RC; i += ENT)
      if (i0 + i < a.m) a.r[i0 + i] = w.sR[k * RC + i];
  }
  __syncthreads();
  commit(bidx(blk(a.p - 1)));   // last block: nobody reads its coordinates any more
  my_sum = warp_sum(my_sum);
  my_max = warp_max(my_max);
  if (lane == 0) {
    a.wsum[blockIdx.x * nw + warp] = my_sum;
    a.wmax[blockIdx.x * nw + warp] = my_max;
  }
  cl.sync();  // peers may still read our shared memory
  grid_barrier(a.bar, target, P);
  if (blockIdx.x == 0 && warp == 0) {
    double tot = 0.0, mx = 0.0;
    for (int q = lane; q < P * nw; q += 32) {
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
