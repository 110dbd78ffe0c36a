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
#include <vector>

#include "boxqp.cuh"
#include "rac_internal.h"
#include "rac_rowphase.cuh"

namespace rac {

constexpr int QPT = RP_THREADS;  // 256 threads per chain CTA
constexpr int QCOLS = 256;       // column tile of the strip update

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
  unsigned* bar;
  int32_t* ctrl;  // [0] done, [1] iterations, [2] failed block+1, [3] status
  double beta, tol_p, tol_d, div_bar;
  int fixed, sweep, lsmem;
  double *hist_p, *hist_l1, *hist_d;
};

// hx[cols of this CTA] += sum_i H[blk[i], col] * delta[i]
__device__ void strip_update(const QpChainArgs& a, const int32_t* sIdx, const double* sDel,
                             double* red, int s) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = QPT / 32;
  const int P = gridDim.x;
  const int64_t per = ((a.n + P - 1) / P + 31) / 32 * 32;
  const int64_t c0 = (int64_t)blockIdx.x * per, c1 = min64(a.n, c0 + per);
  for (int64_t t0 = c0; t0 < c1; t0 += QCOLS) {
    double acc[QCOLS / 32];
#pragma unroll
    for (int q = 0; q < QCOLS / 32; ++q) acc[q] = 0.0;
    for (int i = warp; i < s; i += nw) {
      const int g = sIdx[i];
      if (g < 0) continue;
      const double d = sDel[i];
      const double* row = a.H + (int64_t)g * a.n;
#pragma unroll
      for (int q = 0; q < QCOLS / 32; ++q) {
        int64_t j = t0 + q * 32 + lane;
        if (j < c1) acc[q] += __ldg(row + j) * d;
      }
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
};

template <int RC>
__host__ __device__ size_t qp_smem_bytes(int s, bool rowphase, bool lsmem) {
  size_t d = 0;
  if (rowphase) d += RowPhase<RC>::smem_doubles(s) + s;  // + int idx (as doubles, generous)
  d += (QPT / 32) * QCOLS;                               // strip reduction
  d += 10 * (size_t)s + 64;                              // box vectors + sDel, sxb, shx, sc
  if (lsmem) d += (size_t)s * s;                         // factor workspace
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
  if (lsmem) {
    q.bw.L = p;
    p += (size_t)s * s;
  } else {
    q.bw.L = lscratch;
  }
  int* ip = (int*)p;
  q.bw.flag = ip; ip += s;
  q.bw.F = ip; ip += s;
  q.bw.B = ip; ip += s;
  q.sIdx = ip; ip += s;
  q.bw.misc = ip;
  return q;
}

template <int RC>
__global__ void __launch_bounds__(QPT) qp_chain_kernel(QpChainArgs a) {
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
  int bnext = a.order ? a.order[0] : 0;
  if (has_a)
    row_phase<RC>(a.Ac, a.lda, a.m, a.nrc, a.idx, s, -1, bnext, a.delta, a.x, a.ax, a.partial, w.rp, tfn);
  for (int t = 0; t < a.p; ++t) {
    const int b = bnext;
    grid_barrier(a.bar, target, P);
    // ------------------------------------------------------------ S (CTA 0)
    if (blockIdx.x == 0) {
      const int32_t* bidx = a.idx + (int64_t)b * s;
      for (int i = tid; i < s; i += QPT) {
        int g = bidx[i];
        w.sIdx[i] = g;
        if (g >= 0) {
          w.sxb[i] = ldcg(a.x + g);
          w.shx[i] = ldcg(a.hx + g);
          w.bw.lo[i] = a.lo[g];
          w.bw.hi[i] = a.hi[g];
        }
      }
      int seff;
      if (tid == 0) {
        int k = 0;
        while (k < s && bidx[k] >= 0) ++k;
        w.bw.misc[0] = k;
      }
      __syncthreads();
      seff = w.bw.misc[0];
      // (A_b' t) from the per-CTA partials, then H_bb x_b
      const double* Hb = a.Hbb + (int64_t)b * s * s;
      for (int i = warp; i < seff; i += nw) {
        double pa = 0.0;
        if (has_a) {
          for (int q = lane; q < P; q += 32) pa += ldcg(a.partial + (int64_t)q * s + i);
          pa = warp_sum(pa);
        }
        double hb = 0.0;
        if (a.H) {
          const double* row = Hb + (int64_t)i * s;
          for (int j = lane; j < seff; j += 32) hb += row[j] * w.sxb[j];
          hb = warp_sum(hb);
        }
        if (lane == 0) {
          const int g = w.sIdx[i];
          double rhs = -a.c[g];
          if (a.H) rhs = rhs - (w.shx[i] - hb);
          if (has_a) rhs = rhs + pa;
          w.bw.r[i] = rhs;
        }
      }
      __syncthreads();
      // unconstrained solution x = L^-T L^-1 r with the block's Cholesky factor
      // (engine.py:201-203: cho_solve with the full-block factor)
      {
        const double* Lb = a.inv + (int64_t)b * s * s;
        for (int e = tid; e < seff * seff; e += QPT) {
          const int i = e / seff, j = e - i * seff;
          w.bw.L[e] = Lb[(int64_t)i * s + j];
        }
        for (int i = tid; i < seff; i += QPT) w.bw.x[i] = w.bw.r[i];
        __syncthreads();
        warp_chol_solve(w.bw.L, seff, seff, w.bw.x);
        __syncthreads();
      }
      int fail = box_active_set(a.Mb + (int64_t)b * s * s, s, seff, w.bw);
      if (fail) {
        if (tid == 0) { a.ctrl[2] = b + 1; a.ctrl[0] = 1; }
      }
      for (int i = tid; i < s; i += QPT) {
        double d = 0.0;
        if (i < seff) {
          d = w.bw.x[i] - w.sxb[i];
          a.x[w.sIdx[i]] = w.bw.x[i];
        }
        a.delta[i] = d;
      }
    }
    grid_barrier(a.bar, target, P);
    if (ldcg(a.ctrl + 0)) return;  // non-PD reduced system: abort the sweep
    // ------------------------------------------------------------ G (all CTAs)
    for (int i = tid; i < s; i += QPT) {
      w.sIdx[i] = a.idx[(int64_t)b * s + i];
      w.sDel[i] = ldcg(a.delta + i);
    }
    __syncthreads();
    if (a.H) strip_update(a, w.sIdx, w.sDel, w.red, s);
    bnext = (t + 1 < a.p) ? (a.order ? a.order[t + 1] : t + 1) : -1;
    if (has_a)
      row_phase<RC>(a.Ac, a.lda, a.m, a.nrc, a.idx, s, b, bnext, a.delta, a.x, a.ax, a.partial, w.rp, tfn);
  }
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
          const double res = a.ax[i] - a.b[i];
          a.y[i] = a.y[i] - beta * res;
          pm = fmax(pm, fabs(res));
          ps += fabs(res);
        }
      }
    }
  }
  pm = warp_max(pm);
  ps = warp_sum(ps);
  if (lane == 0) { w.bw.red[warp] = pm; w.sc[warp] = ps; }
  __syncthreads();
  if (tid == 0) {
    double m1 = 0.0, s1 = 0.0;
    for (int q = 0; q < nw; ++q) { m1 = fmax(m1, w.bw.red[q]); s1 += w.sc[q]; }
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
        const double pr = fmin(fmax(xj - grad, a.lo[j]), a.hi[j]);
        dm = fmax(dm, fabs(pr - xj));
      }
    }
  }
  dm = warp_max(dm);
  if (lane == 0) w.bw.red[warp] = dm;
  __syncthreads();
  if (tid == 0) {
    double m1 = 0.0;
    for (int q = 0; q < nw; ++q) m1 = fmax(m1, w.bw.red[q]);
    a.dmax[blockIdx.x] = m1;
  }
  grid_barrier(a.bar, target, P);
  if (blockIdx.x == 0 && warp == 0) {
    double pmx = 0.0, psm = 0.0, dmx = 0.0;
    for (int q = lane; q < P; q += 32) {
      pmx = fmax(pmx, ldcg(a.pmax + q));
      psm += ldcg(a.psum + q);
      dmx = fmax(dmx, ldcg(a.dmax + q));
    }
    pmx = warp_max(pmx);
    psm = warp_sum(psm);
    dmx = warp_max(dmx);
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

// x0 = clip(0, lo, hi)
__global__ void clip0_kernel(const double* lo, const double* hi, int64_t n, double* x) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = fmin(fmax(0.0, lo[i]), hi[i]);
}

// single-CTA test entry for the box solver (inverse-free first solve)
__global__ void __launch_bounds__(QPT) box_test_kernel(const double* M, const double* r, const double* lo,
                                                       const double* hi, int s, double* xout,
                                                       int32_t* info, double* L) {
  extern __shared__ __align__(16) double bsm[];
  QpSmem w = carve_qp<32>(bsm, s, false, L == nullptr, L);
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
  int fail = solve_free(M, s, w.bw);
  if (!fail) {
    for (int i = threadIdx.x; i < s; i += QPT) w.bw.x[i] = w.bw.xf[i];
    __syncthreads();
    fail = box_active_set(M, s, s, w.bw);
  }
  for (int i = threadIdx.x; i < s; i += QPT) xout[i] = w.bw.x[i];
  if (threadIdx.x == 0) *info = fail;
}

// Q_ij = y_i y_j K(x_i, x_j) from the raw Gram (lower triangle in G, full write)
__global__ void svm_kernel_epilogue(double* Q, int64_t N, const double* y, const double* sq,
                                    int kind, double two_sigma2) {
  const int64_t total = N * (N + 1) / 2;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = (int64_t)((sqrt(8.0 * (double)e + 1.0) - 1.0) * 0.5);
    while ((i + 1) * (i + 2) / 2 <= e) ++i;
    while (i * (i + 1) / 2 > e) --i;
    const int64_t j = e - i * (i + 1) / 2;
    double k = Q[i * N + j];
    if (kind == RAC_KERNEL_GAUSSIAN) {
      double d2 = fmax(sub(add(sq[i], sq[j]), mul(2.0, k)), 0.0);
      k = exp(-d2 / two_sigma2);
    }
    Q[i * N + j] = mul(mul(y[i], k), y[j]);
    Q[j * N + i] = mul(mul(y[j], k), y[i]);
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
  unsigned* bar = nullptr;
  int32_t* ctrl = nullptr;
  double *hist_p = nullptr, *hist_l1 = nullptr, *hist_d = nullptr;
  double div_bar = INFINITY;
  std::vector<void*> allocs;
};

namespace {

template <typename T>
int qalloc(rac_qp_ctx* c, T** p, size_t count) {
  if (count == 0) count = 1;
  void* q = nullptr;
  cudaError_t e = cudaMalloc(&q, count * sizeof(T));
  if (e != cudaSuccess) return rac::check_cuda(e, "cudaMalloc");
  c->allocs.push_back(q);
  *p = (T*)q;
  return RAC_OK;
}

constexpr int kQpRC = 32;

size_t qp_smem(const rac_qp_ctx* c) { return rac::qp_smem_bytes<kQpRC>(c->s, c->m > 0, c->lsmem); }

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
  a.ws = (c->m > 0) ? c->gram_ws : nullptr;
  a.splits = c->gp.splits;
  a.div = 1.0;
  a.mul = c->beta;
  a.H = c->H;
  a.ldh = c->n;
  a.idx = c->idx;
  a.shift = 0.0;
  a.ridge_rel = c->ridge_rel;
  a.s = c->s;
  a.inv = c->inv;
  a.mat_out = c->Mb;
  a.hbb_out = c->Hbb;
  a.scratch = c->scratch;
  a.info = c->info;
  a.mode = FACTOR_CHOL;
  a.done = c->ctrl;
  return launch_chol_system(a, c->p, c->st);
}

int qp_chain(rac_qp_ctx* c, double tol_p, double tol_d, int fixed) {
  using namespace rac;
  cudaMemsetAsync(c->bar, 0, sizeof(unsigned), c->st);
  QpChainArgs a{};
  a.n = c->n;
  a.m = c->m;
  a.lda = c->lda;
  a.s = c->s;
  a.p = c->p;
  a.nrc = c->nrc;
  a.H = c->H;
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
  void* args[] = {&a};
  cudaError_t e = cudaLaunchCooperativeKernel((void*)qp_chain_kernel<kQpRC>, dim3(c->P), dim3(QPT), args,
                                              qp_smem(c), c->st);
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
  c->nrc = (int)((std::max<int64_t>(m, 1) + kQpRC - 1) / kQpRC);
  c->lsmem = rac::qp_smem_bytes<kQpRC>(c->s, m > 0, true) <= 200 * 1024;
  int rc = check_cuda(cudaFuncSetAttribute(qp_chain_kernel<kQpRC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)qp_smem(c)),
                      "qp chain smem attribute");
  if (rc) {
    delete c;
    return rc;
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, qp_chain_kernel<kQpRC>, QPT, qp_smem(c));
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
      (rc = qalloc(c, &c->delta, c->s)) || (rc = qalloc(c, &c->pmax, c->P)) || (rc = qalloc(c, &c->psum, c->P)) ||
      (rc = qalloc(c, &c->dmax, c->P)) || (rc = qalloc(c, &c->bar, 1)) || (rc = qalloc(c, &c->ctrl, 4))) {
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
  if (!c->lsmem && (rc = qalloc(c, &c->lscratch, (size_t)c->s * c->s))) {
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
  clip0_kernel<<<(int)std::min<int64_t>((c->n + 255) / 256, 1184), 256, 0, c->st>>>(c->lo, c->hi, c->n, c->x);
  // running products at x0 and the divergence bar (engine.py:361-362)
  if (c->H) {
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
    rc = qp_chain(c, tol_p, tol_d, fixed);
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

extern "C" int rac_qp_destroy(rac_qp_ctx* c) {
  if (!c) return RAC_OK;
  if (c->st) cudaStreamSynchronize(c->st);
  for (void* q : c->allocs) cudaFree(q);
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
  GramPlan pl = plan_gram(d, (int)N, 1);
  pl.splits = 1;
  pl.chunk = ldd;
  rc = launch_gram(Xp, ldd, d, ids, nullptr, (int)N, 1, Q, pl, st, nullptr);
  if (rc) return rc;
  diag_copy_kernel<<<(int)std::min<int64_t>((N + 255) / 256, 4096), 256, 0, st>>>(Q, N, sq);
  const int64_t total = N * (N + 1) / 2;
  svm_kernel_epilogue<<<(int)std::min<int64_t>((total + 255) / 256, 148 * 32), 256, 0, st>>>(
      Q, N, labels, sq, kind, 2.0 * sigma * sigma);
  cudaFreeAsync(Xp, st);
  cudaFreeAsync(sq, st);
  cudaFreeAsync(ids, st);
  return check_launch("rac_svm_build_q");
}

extern "C" int rac_box_block_min(const double* M, const double* r, const double* lo, const double* hi, int32_t s,
                                 double* x, int32_t* info, void* stream) {
  using namespace rac;
  clear_error();
  if (!M || !r || !lo || !hi || !x || !info || s < 1) return set_error(RAC_ERR_ARG, "rac_box_block_min: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  bool lsmem = qp_smem_bytes<32>(s, false, true) <= 200 * 1024;
  double* L = nullptr;
  if (!lsmem) {
    int rc = check_cuda(cudaMallocAsync((void**)&L, (size_t)s * s * sizeof(double), st), "malloc L");
    if (rc) return rc;
  }
  size_t smem = qp_smem_bytes<32>(s, false, lsmem);
  int rc = check_cuda(cudaFuncSetAttribute(box_test_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                      "box smem attribute");
  if (rc) return rc;
  box_test_kernel<<<1, QPT, smem, st>>>(M, r, lo, hi, s, x, info, L);
  if (L) cudaFreeAsync(L, st);
  return check_launch("rac_box_block_min");
}
