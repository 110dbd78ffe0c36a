// Two-block consensus baseline (elastic_net.py:252-316 consensus_fit), per-sweep part.
//
// N coefficient copies (one per sample group).  Per sweep:
//   w_i      = w0_i + duals_i + gamma z                       (elastic_net.py:300)
//   copy_i   = S_i^{-1} w_i                          direct   (p <= n_i, :301-302)
//            = (w_i - X_i' W_i^{-1} X_i w_i) / gamma  Woodbury (p > n_i,  :303-305)
//   agg      = sum_i duals_i - gamma sum_i copy_i                  (:306)
//   z        = S(agg, lam alpha) / ((1 - alpha) lam + N gamma)     (:307-308, negated shrink)
//   duals_i -= gamma (copy_i - z)                                  (:309)
//   residual = mean_i ||copy_i - z||_1                             (:311)
// S_i^{-1} / W_i^{-1} are formed once per fit (host side, paper_1907_01995_b200/consensus.py).
// Kernels: (1) direct groups: one warp per output row of the batched symmetric mat-vec, w_i
// formed on the fly (HBM-bound: N p^2 doubles per sweep); (2) Woodbury groups: u = X_i w_i,
// inner = W_i^{-1} u, copy_i = (w_i - X_i' inner) / gamma; (3) the z / dual / residual step,
// one thread per feature over the N copies, block partial sums reduced in a fixed order, and
// an on-device stop flag so that a batch of sweeps runs without a host round trip.
#include "rac_internal.h"

#include <algorithm>

namespace rac {
namespace {

struct ConsArgs {
  int N;
  int64_t p;
  const int32_t* kind;      // [N] 0 direct, 1 Woodbury
  const int32_t* ni;        // [N] samples per group
  const int64_t* off_inv;   // [N] offset of S_i^{-1} (p x p) or W_i^{-1} (n_i x n_i) in inv
  const int64_t* off_x;     // [N] offset of X_i (n_i x p, row-major) in xg (Woodbury groups)
  const int64_t* off_u;     // [N] offset of group i's n_i-vectors in u / inner
  const double* inv;
  const double* xg;
  const double* w0;         // [N][p]
  double* copies;           // [N][p]
  double* duals;            // [N][p]
  double* z;                // [p]
  double* u;
  double* inner;
  double* part;             // [grid of the z step] residual partials
  double* hist;             // [max sweeps] residual per sweep
  int32_t* state;           // [0] sweeps done, [1] stop flag
  double gamma, thr, denom, tol;
};

__device__ __forceinline__ double w_of(const ConsArgs& a, int i, int64_t c) {
  return add(add(a.w0[(int64_t)i * a.p + c], a.duals[(int64_t)i * a.p + c]), mul(a.gamma, a.z[c]));
}

// (1) direct groups: copies[i][r] = sum_c S_i^{-1}[r][c] w_i[c]
__global__ void cons_direct_kernel(ConsArgs a) {
  if (a.state[1]) return;
  const int lane = threadIdx.x & 31;
  const int64_t rows = (int64_t)a.N * a.p;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t gr = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; gr < rows; gr += nw) {
    const int i = (int)(gr / a.p);
    if (a.kind[i] != 0) continue;
    const int64_t r = gr - (int64_t)i * a.p;
    const double* row = a.inv + a.off_inv[i] + r * a.p;
    double acc = 0.0;
    for (int64_t c = lane; c < a.p; c += 32) acc = fma(row[c], w_of(a, i, c), acc);
    acc = warp_sum(acc);
    if (lane == 0) a.copies[gr] = acc;
  }
}

// (2a) Woodbury: u_i[k] = X_i[k, :] . w_i   (one warp per (group, sample))
__global__ void cons_wb_u_kernel(ConsArgs a, int64_t total_rows) {
  if (a.state[1]) return;
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t gk = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; gk < total_rows; gk += nw) {
    // group of this row: off_u is increasing
    int i = 0;
    while (i + 1 < a.N && a.off_u[i + 1] <= gk) ++i;
    if (a.kind[i] != 1) continue;
    const int64_t k = gk - a.off_u[i];
    const double* xr = a.xg + a.off_x[i] + k * a.p;
    double acc = 0.0;
    for (int64_t c = lane; c < a.p; c += 32) acc = fma(xr[c], w_of(a, i, c), acc);
    acc = warp_sum(acc);
    if (lane == 0) a.u[gk] = acc;
  }
}

// (2b) inner_i = W_i^{-1} u_i   (one warp per (group, sample))
__global__ void cons_wb_inner_kernel(ConsArgs a, int64_t total_rows) {
  if (a.state[1]) return;
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t gk = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; gk < total_rows; gk += nw) {
    int i = 0;
    while (i + 1 < a.N && a.off_u[i + 1] <= gk) ++i;
    if (a.kind[i] != 1) continue;
    const int n = a.ni[i];
    const int64_t k = gk - a.off_u[i];
    const double* wr = a.inv + a.off_inv[i] + k * n;
    double acc = 0.0;
    for (int q = lane; q < n; q += 32) acc = fma(wr[q], a.u[a.off_u[i] + q], acc);
    acc = warp_sum(acc);
    if (lane == 0) a.inner[gk] = acc;
  }
}

// (2c) copies[i][c] = (w_i[c] - sum_k X_i[k][c] inner_i[k]) / gamma   (thread per (group, feature))
__global__ void cons_wb_copy_kernel(ConsArgs a) {
  if (a.state[1]) return;
  const int64_t total = (int64_t)a.N * a.p;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / a.p);
    if (a.kind[i] != 1) continue;
    const int64_t c = e - (int64_t)i * a.p;
    const double* xc = a.xg + a.off_x[i] + c;
    const double* in = a.inner + a.off_u[i];
    double acc = 0.0;
    for (int k = 0; k < a.ni[i]; ++k) acc = fma(xc[(int64_t)k * a.p], in[k], acc);
    a.copies[e] = __ddiv_rn(sub(w_of(a, i, c), acc), a.gamma);
  }
}

// (3) z, duals, residual partials (thread per feature), block sums in shared memory
constexpr int CZT = 256;
__global__ void __launch_bounds__(CZT) cons_z_kernel(ConsArgs a) {
  if (a.state[1]) return;
  __shared__ double red[CZT / 32];
  double loc = 0.0;
  for (int64_t c = blockIdx.x * (int64_t)CZT + threadIdx.x; c < a.p; c += (int64_t)gridDim.x * CZT) {
    double ds = 0.0, cs = 0.0;
    for (int i = 0; i < a.N; ++i) {
      ds = add(ds, a.duals[(int64_t)i * a.p + c]);
      cs = add(cs, a.copies[(int64_t)i * a.p + c]);
    }
    const double agg = sub(ds, mul(a.gamma, cs));
    const double zc = __ddiv_rn(neg_shrink(agg, a.thr), a.denom);
    a.z[c] = zc;
    for (int i = 0; i < a.N; ++i) {
      const int64_t e = (int64_t)i * a.p + c;
      const double d = sub(a.copies[e], zc);
      a.duals[e] = sub(a.duals[e], mul(a.gamma, d));
      loc += fabs(d);
    }
  }
  loc = warp_sum(loc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = loc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < CZT / 32; ++w) t += red[w];
    a.part[blockIdx.x] = t;
  }
}

__global__ void cons_finish_kernel(ConsArgs a, int nblk) {
  if (a.state[1]) return;
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int b = 0; b < nblk; ++b) t += a.part[b];
    const double res = t / (double)a.N;
    const int k = a.state[0];
    a.hist[k] = res;
    a.state[0] = k + 1;
    if (a.tol >= 0.0 && res <= a.tol) a.state[1] = 1;
  }
}

}  // namespace
}  // namespace rac

extern "C" int rac_consensus_run(const rac_consensus_args* d, int32_t count, void* stream) {
  using namespace rac;
  clear_error();
  if (!d || d->N < 1 || d->p < 1 || !d->kind || !d->ni || !d->off_inv || !d->inv || !d->w0 || !d->copies ||
      !d->duals || !d->z || !d->part || !d->hist || !d->state || count < 0 || !(d->gamma > 0))
    return set_error(RAC_ERR_ARG, "rac_consensus_run: bad arguments");
  if (d->wb_rows > 0 && (!d->xg || !d->off_x || !d->off_u || !d->u || !d->inner))
    return set_error(RAC_ERR_ARG, "rac_consensus_run: Woodbury groups need xg / off_x / off_u / u / inner");
  cudaStream_t st = (cudaStream_t)stream;
  ConsArgs a{};
  a.N = d->N;
  a.p = d->p;
  a.kind = d->kind;
  a.ni = d->ni;
  a.off_inv = d->off_inv;
  a.off_x = d->off_x;
  a.off_u = d->off_u;
  a.inv = d->inv;
  a.xg = d->xg;
  a.w0 = d->w0;
  a.copies = d->copies;
  a.duals = d->duals;
  a.z = d->z;
  a.u = d->u;
  a.inner = d->inner;
  a.part = d->part;
  a.hist = d->hist;
  a.state = d->state;
  a.gamma = d->gamma;
  a.thr = d->thr;
  a.denom = d->denom;
  a.tol = d->tol;
  const int sms = num_sms();
  const int zblk = (int)std::min<int64_t>((d->p + CZT - 1) / CZT, (int64_t)d->part_cap);
  for (int k = 0; k < count; ++k) {
    if (d->direct_groups > 0) {
      const int64_t rows = (int64_t)d->N * d->p;
      cons_direct_kernel<<<(int)std::min<int64_t>((rows + 7) / 8, (int64_t)sms * 16), 256, 0, st>>>(a);
      note_launch();
    }
    if (d->wb_rows > 0) {
      const int g1 = (int)std::min<int64_t>((d->wb_rows + 7) / 8, (int64_t)sms * 16);
      cons_wb_u_kernel<<<g1, 256, 0, st>>>(a, d->wb_rows);
      cons_wb_inner_kernel<<<g1, 256, 0, st>>>(a, d->wb_rows);
      const int64_t tot = (int64_t)d->N * d->p;
      cons_wb_copy_kernel<<<(int)std::min<int64_t>((tot + 255) / 256, (int64_t)sms * 16), 256, 0, st>>>(a);
      note_launch(3);
    }
    cons_z_kernel<<<zblk, CZT, 0, st>>>(a);
    cons_finish_kernel<<<1, 32, 0, st>>>(a, zblk);
    note_launch(2);
  }
  return check_launch("consensus sweep");
}
