// Covariance-mode chain for the elastic-net sweep (included by en.cu).
//
// When n is moderate, G = X'X/m (n x n) is formed once per fit and the
// Gauss-Seidel chain runs on G instead of X (the covariance-update form of
// the same block step, cf. elastic_net.py:199-224):
//
//   reference:  sys_b beta_b' = -(c_b + X_b'(r - X_b beta_b)/m - xi_b - gamma z_b),  r = X beta
//   here:       q = G beta is kept current, and with v = -c_b - q_b + xi_b + gamma (z_b - beta_b)
//               beta_b' = beta_b + sys_b^{-1} v            (since X_b'X_b/m = sys_b - gamma I)
//               q      += G[:, b] (beta_b' - beta_b)
//
// The whole chain runs in ONE thread-block cluster of up to 16 CTAs (no grid
// barrier): CTA k owns rows R_k of q (n/K entries) and rows S_k of every
// block's inverse (s/K).  Per block: cluster barrier, v from q (L2),
// delta slice from the smem-resident inverse rows (TMA bulk, prefetched one
// block ahead), commit of the slice's beta/z/xi, cluster barrier, DSMEM
// gather of the full delta, then q[R_k] += G[b, R_k]' delta (coalesced rows
// of G, L2-resident for the BASELINE configs that use this mode).  The other
// SMs stay free for the next sweep's block factorisations.
#pragma once

#include <cooperative_groups.h>

namespace rac {

constexpr int COVT = 512;              // threads per CTA
constexpr int COV_NW = COVT / 32;
constexpr int COV_UNR = 32;            // independent G loads in flight per lane

struct EnCovArgs {
  const double* G;      // n x n row-major, X'X/m
  int64_t n;
  int s, p;
  const int32_t* idx;   // [p][s]
  const int32_t* order; // RP visit order or null
  const double* inv;    // [p][s][s]
  const int32_t* info;
  const double* c;
  double *beta, *z, *xi, *q;
  double* q2;           // second published copy of q (full_inv mode double-buffers it)
  double *wsum, *wmax;  // [K]
  int32_t* ctrl;
  double gamma, thr, den, tol;
  int sweep;
  double *hist_p, *hist_d;
  long long* trace;     // optional: %globaltimer per phase (CTA 0): 1 + 7 per block
  int full_inv;         // 1: every CTA stages the whole inverse and computes the whole delta
                        //    (one cluster barrier per block instead of two, no DSMEM gather)
};

// phase-A partials: GA x RT x 32 with GA = ceil(16 / RT)  ->  <= 512 + RT * 32
__host__ __device__ inline size_t cov_red_doubles(size_t rn) { return 512 + (rn + 31) / 32 * 32; }

template <int K>
__host__ __device__ inline size_t cov_smem_bytes(int s, int64_t n, int p, int full_inv) {
  const size_t sl = full_inv ? (size_t)s : (size_t)(s + K - 1) / K;
  const size_t rn = (size_t)((n + K - 1) / K);
  return (2 * sl * s + 8 * (size_t)s + (size_t)s + s + sl + rn + cov_red_doubles(rn) + 2 * COV_NW + 4) *
             sizeof(double) +
         (size_t)p * s * sizeof(int32_t);
}

template <int K>
__global__ void __launch_bounds__(COVT, 1) en_cov_kernel(EnCovArgs a) {
  if (a.ctrl[0]) return;
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ __align__(128) double csm[];
  const int s = a.s, p = a.p;
  const int64_t n = a.n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rank = (int)cl.block_rank();
  const int sl = (s + K - 1) / K, j0 = min(s, rank * sl), j1 = min(s, j0 + sl), rows = j1 - j0;
  const bool full = a.full_inv != 0;
  const int ir = full ? s : sl;            // inverse rows staged per CTA
  const int ij0 = full ? 0 : j0, irows = full ? s : rows;
  const int64_t rn = (n + K - 1) / K, r0 = min(n, (int64_t)rank * rn), r1 = min(n, r0 + rn);
  const int nr = (int)(r1 - r0);

  double* sInv = csm;                          // [2][ir*s]
  double* sVec = sInv + 2 * (size_t)ir * s;    // [2][4][s]  c, xi, z, beta at the block's indices
  double* sV = sVec + 8 * (size_t)s;           // [s]
  double* sDel = sV + s;                       // [s]  full delta of the last solved block
  double* sD = sDel + s;                       // [sl] this rank's delta slice (peers read it)
  double* qR = sD + sl;                        // [rn] q rows owned by this CTA
  double* red = qR + rn;                       // phase-A partials [GA][RT*32]
  double* wred = red + cov_red_doubles((size_t)rn);   // [2*COV_NW]
  uint64_t* bars = reinterpret_cast<uint64_t*>(wred + 2 * COV_NW);   // [2]
  int* sIdx = reinterpret_cast<int*>(bars + 4);                      // [p*s]
  __shared__ int bad;

  if (tid == 0) {
    bad = 0;
    for (int t = 0; t < p; ++t) {
      const int b = a.order ? a.order[t] : t;
      if (a.info[b]) { bad = b + 1; break; }
    }
    mbar_init(bars + 0, 1);
    mbar_init(bars + 1, 1);
    mbar_fence_init();
  }
  for (int e = tid; e < p * s; e += COVT) sIdx[e] = a.idx[e];
  for (int r = tid; r < nr; r += COVT) qR[r] = a.q[r0 + r];
  __syncthreads();
  if (bad) {
    if (rank == 0 && tid == 0) { a.ctrl[2] = bad; a.ctrl[0] = 1; }
    return;
  }
  const double gamma = a.gamma;
  auto blk = [&](int t) { return a.order ? a.order[t] : t; };
  auto bidx = [&](int b) { return sIdx + (size_t)b * s; };
  const bool bulk_inv = ((s & 1) == 0);
  unsigned par[2] = {0u, 0u};

  // prefetch of block t's inverse rows (this rank's slice) and c/xi/z/beta at its indices
  auto issue = [&](int t) {
    const int b = blk(t), buf = t & 1;
    const int* bi = bidx(b);
    const double* Ib = a.inv + (int64_t)b * s * s + (int64_t)ij0 * s;
    double* dInv = sInv + (size_t)buf * ir * s;
    if (bulk_inv) {
      if (tid == 0) {
        fence_proxy_async();
        const unsigned bytes = (unsigned)(irows * s * sizeof(double));
        mbar_arrive_expect_tx(bars + buf, bytes);
        for (unsigned off = 0; off < bytes; off += 65536u)
          bulk_g2s(dInv + off / 8, Ib + off / 8, min(65536u, bytes - off), bars + buf);
      }
    } else {
      for (int e = tid; e < irows * s; e += COVT) cp_async8(dInv + e, Ib + e);
    }
    double* dv = sVec + (size_t)buf * 4 * s;
    for (int j = tid; j < s; j += COVT) {
      const int g = bi[j];
      if (g >= 0) {
        cp_async8(dv + j, a.c + g);
        cp_async8(dv + s + j, a.xi + g);
        cp_async8(dv + 2 * s + j, a.z + g);
        cp_async8(dv + 3 * s + j, a.beta + g);
      } else {
        dv[j] = dv[s + j] = dv[2 * s + j] = dv[3 * s + j] = 0.0;
      }
    }
    cp_async_commit();
  };
  auto wait = [&](int t) {
    const int buf = t & 1;
    if (bulk_inv) {
      mbar_wait(bars + buf, par[buf]);
      par[buf] ^= 1u;
    }
  };

  // q[R] += G[b, R]' delta  (rows of G = columns by symmetry; lanes = consecutive rows)
  const int RT = (nr + 31) / 32;
  // j-groups per row tile so that every warp has a task: at most ceil(RT*s/16) loads per lane
  const int GA = max(1, (COV_NW + max(1, RT) - 1) / max(1, RT));
  const int tasks = RT * GA;
  const int per = (s + GA - 1) / GA;
  auto phase_a = [&](int b, double* qdst) {
    const int* bi = bidx(b);
    for (int task = warp; task < tasks; task += COV_NW) {
      const int rt = task % RT, ga = task / RT;
      const int r = rt * 32 + lane;
      const bool live = r < nr;
      const int64_t col = r0 + (live ? r : 0);
      const int ja = ga * per, jb = min(s, ja + per);
      double acc = 0.0;
      for (int jj = ja; jj < jb; jj += COV_UNR) {
        double gv[COV_UNR];
#pragma unroll
        for (int u = 0; u < COV_UNR; ++u) {
          const int j = jj + u;
          const int g = (j < jb) ? bi[j] : -1;
          gv[u] = (g >= 0) ? ldcg(a.G + (int64_t)g * n + col) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < COV_UNR; ++u) {
          const int j = jj + u;
          if (j < jb) acc += gv[u] * sDel[j];
        }
      }
      if (live) red[ga * (RT * 32) + r] = acc;
    }
    __syncthreads();
    for (int r = tid; r < nr; r += COVT) {
      double tot = red[r];
      for (int ga = 1; ga < GA; ++ga) tot += red[ga * (RT * 32) + r];
      const double qn = qR[r] + tot;
      qR[r] = qn;
      qdst[r0 + r] = qn;
    }
  };

  double my_sum = 0.0, my_max = 0.0;
  const bool tr = a.trace && rank == 0 && tid == 0;
  int tp = 0;
  if (tr) a.trace[tp++] = gtimer();
  issue(0);
  for (int t = 0; t < p; ++t) {
    const int b = blk(t), buf = t & 1;
    const int* bi = bidx(b);
    // the q published at block t: full_inv mode alternates two global copies, so a
    // rank already updating for block t+1 never overwrites what a slower rank reads
    double* qpub = (full && (t & 1)) ? a.q2 : a.q;
    if (t > 0) phase_a(blk(t - 1), qpub);
    if (tr) a.trace[tp++] = gtimer();
    cl.sync();   // q rows of every rank are current; every rank is done with sDel / sD
    if (tr) a.trace[tp++] = gtimer();
    if (t + 1 < p) issue(t + 1);
    wait(t);
    if (t + 1 < p) cp_async_wait<1>(); else cp_async_wait<0>();
    __syncthreads();
    if (tr) a.trace[tp++] = gtimer();
    // v = -c - q + xi + gamma (z - beta) at the block's indices
    const double* dv = sVec + (size_t)buf * 4 * s;
    for (int j = tid; j < s; j += COVT) {
      const int g = bi[j];
      sV[j] = (g >= 0) ? add(add(sub(-dv[j], ldcg(qpub + g)), dv[s + j]), mul(gamma, sub(dv[2 * s + j], dv[3 * s + j])))
                       : 0.0;
    }
    __syncthreads();
    if (tr) a.trace[tp++] = gtimer();
    if (full) {
      // whole delta in every CTA: (row i, part k) threads, column reads of the
      // symmetric inverse (conflict-free), parts summed in order
      const double* I = sInv + (size_t)buf * s * s;
      const int rs = (s + 31) / 32 * 32;
      const int parts = max(1, min(COVT / rs, 8));
      const int per = (s + parts - 1) / parts;
      for (int e = tid; e < parts * rs; e += COVT) {
        const int k = e / rs, i = e - k * rs;
        double acc = 0.0;
        if (i < s) {
          const int ja = k * per, jb = min(s, ja + per);
          double a1 = 0.0, a2 = 0.0, a3 = 0.0;   // four independent chains
          int j = ja;
          for (; j + 4 <= jb; j += 4) {
            acc += I[(size_t)j * s + i] * sV[j];
            a1 += I[(size_t)(j + 1) * s + i] * sV[j + 1];
            a2 += I[(size_t)(j + 2) * s + i] * sV[j + 2];
            a3 += I[(size_t)(j + 3) * s + i] * sV[j + 3];
          }
          for (; j < jb; ++j) acc += I[(size_t)j * s + i] * sV[j];
          acc = (acc + a1) + (a2 + a3);
        }
        red[k * rs + i] = acc;
      }
      __syncthreads();
      for (int i = tid; i < s; i += COVT) {
        double d = red[i];
        for (int k = 1; k < parts; ++k) d += red[k * rs + i];
        sDel[i] = (bi[i] >= 0) ? d : 0.0;
      }
      __syncthreads();
      if (tr) a.trace[tp++] = gtimer();
      for (int jj = j0 + tid; jj < j1; jj += COVT) {
        const int g = bi[jj];
        if (g < 0) continue;
        const double bn = add(dv[3 * s + jj], sDel[jj]);
        const double x0 = dv[s + jj], zo = dv[2 * s + jj];
        a.beta[g] = bn;
        const double av = sub(x0, mul(gamma, bn));
        const double zn = __ddiv_rn(neg_shrink(av, a.thr), a.den);
        a.z[g] = zn;
        a.xi[g] = sub(x0, mul(gamma, sub(bn, zn)));
        my_sum += fabs(sub(bn, zn));
        my_max = fmax(my_max, fabs(sub(zn, zo)));
      }
      if (tr) { a.trace[tp++] = gtimer(); a.trace[tp++] = gtimer(); }
      continue;
    }
    // delta slice = inv rows . v ; commit beta/z/xi of the slice
    const double* I = sInv + (size_t)buf * sl * s;
    for (int i = warp; i < rows; i += COV_NW) {
      const double* row = I + (size_t)i * s;
      double acc = 0.0;
      for (int j = lane; j < s; j += 32) acc += row[j] * sV[j];
      acc = warp_sum(acc);
      if (lane == 0) {
        const int jj = j0 + i;
        const int g = bi[jj];
        double d = 0.0;
        if (g >= 0) {
          d = acc;
          const double bn = add(dv[3 * s + jj], d);
          const double x0 = dv[s + jj], zo = dv[2 * s + jj];
          a.beta[g] = bn;
          const double av = sub(x0, mul(gamma, bn));
          const double zn = __ddiv_rn(neg_shrink(av, a.thr), a.den);
          a.z[g] = zn;
          a.xi[g] = sub(x0, mul(gamma, sub(bn, zn)));
          my_sum += fabs(sub(bn, zn));
          my_max = fmax(my_max, fabs(sub(zn, zo)));
        }
        sD[i] = d;
      }
    }
    if (tr) a.trace[tp++] = gtimer();
    cl.sync();
    if (tr) a.trace[tp++] = gtimer();
    for (int j = tid; j < s; j += COVT) {
      const int rk = j / sl;
      sDel[j] = cl.map_shared_rank(sD, rk)[j - rk * sl];
    }
    __syncthreads();
    if (tr) a.trace[tp++] = gtimer();
  }
  if (full) cl.sync();   // every rank is past its last read of the published q
  phase_a(blk(p - 1), a.q);   // q current for the next sweep
  // residuals: warp -> CTA -> rank 0
  my_sum = warp_sum(my_sum);
  my_max = warp_max(my_max);
  if (lane == 0) {
    wred[warp] = my_sum;
    wred[COV_NW + warp] = my_max;
  }
  __syncthreads();
  if (tid == 0) {
    double tot = 0.0, mx = 0.0;
    for (int w2 = 0; w2 < COV_NW; ++w2) {
      tot += wred[w2];
      mx = fmax(mx, wred[COV_NW + w2]);
    }
    a.wsum[rank] = tot;
    a.wmax[rank] = mx;
  }
  cl.sync();   // also: peers may still read our sD
  if (rank == 0 && tid == 0) {
    double tot = 0.0, mx = 0.0;
    for (int k = 0; k < K; ++k) {
      tot += ldcg(a.wsum + k);
      mx = fmax(mx, ldcg(a.wmax + k));
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

}  // namespace rac
