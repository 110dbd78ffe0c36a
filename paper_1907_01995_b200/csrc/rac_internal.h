// Internal declarations shared by the .cu translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/rac_b200.h"
#include "rac_common.cuh"

namespace rac {

// thread-local error reporting (rac_last_error)
void clear_error();
int set_error(int code, const char* fmt, ...);
int check_cuda(cudaError_t e, const char* what);
int check_launch(const char* what);
// count of kernels this library launched (rac_launch_count)
void note_launch(int k = 1);
unsigned long long launch_count();

int num_sms();
int dev_alloc(void** p, size_t bytes, cudaStream_t st);
void dev_free(void* p, cudaStream_t st);
void trim_pool(size_t keep);
extern const uint64_t POOL_KEEP;   // bytes the device pool keeps mapped across synchronisations
// launch the persistent (software grid-barrier) kernels without the cooperative
// attribute: under Nsight Compute or with RAC_PROFILE_NONCOOP=1 (capi.cu)
bool profile_noncoop();
// cudaLaunchCooperativeKernel, or a plain launch when profile_noncoop()
cudaError_t launch_coop(const void* f, dim3 grid, dim3 block, void** args, size_t smem, cudaStream_t st);
int launch_gemv_rows(const double* Q, int64_t rows, int64_t cols, const double* w, double* out,
                     cudaStream_t st);

// K1
int launch_chunk_sort(const int64_t* perms, int64_t n, int s, int count, int32_t* out,
                      cudaStream_t st);
int launch_order_cast(const int64_t* src, int64_t total, int32_t* dst, cudaStream_t st);

// K2/K3: batched Gram (DMMA) and Cholesky/inverse of the block systems.
struct GramPlan {
  int tiles;      // 64-wide tiles per block side
  int pairs;      // lower-triangular tile pairs
  int splits;     // split-K factor
  int64_t chunk;  // rows per split (multiple of 32)
};
GramPlan plan_gram(int64_t len, int s, int p);
size_t gram_ws_bytes(int64_t len, int s, int p);
// ws receives `splits` partial Grams per block ([p][splits][s][s], lower part valid)
int launch_gram(const double* V, int64_t ldv, int64_t len, const int32_t* idx, const int32_t* blk_list,
                int s, int p, double* ws, const GramPlan& plan, cudaStream_t st,
                const int32_t* done, double sym_div = 0.0, int sym_accum = 0);
// sym_div > 0 (requires plan.splits == 1): ws receives the FULL symmetric s x s
// matrix divided by sym_div (the covariance G = X'X/m).  sym_accum: the full
// symmetric raw sums are ADDED to ws (row-chunk streaming of G).
// fixed-order sum of the split partials of ONE full Gram (ws [splits][n][n], lower part
// valid), divided by div, written as the full symmetric n x n matrix
// covariance Gram on the tensor cores in exact int8 digit-slice arithmetic (gram_i8.cu):
// G = Xc' Xc over samples [0, len) written / div, or added (accum); ws >= gram_i8_ws_bytes
size_t gram_i8_ws_bytes(int64_t len, int n);
// the flags word of the last launch_gram_i8 on this workspace (bits as launch_i8_colexp's)
const int* gram_i8_ws_flags(const void* ws);
// bad (optional): raised when a column's max/rms ratio makes the digit-slice error exceed the
// FP64 level (gram_i8.cu I8_MAX_RATIO) — the caller then forms that Gram on the DMMA tiles
int launch_gram_i8(const double* Xc, int64_t ld, int64_t len, int n, double* G, double div, int accum, void* ws,
                   size_t ws_bytes, cudaStream_t st, int* bad = nullptr);
// block mode: per-feature exponents once per data set, then per sweep the p block Grams
// (raw sums out[b][s][s], lower triangle incl. the diagonal valid) of idx[b*s ..] in one slicing + one GEMM launch
size_t gram_i8_blocks_ws_bytes(int64_t len, int s, int p);
// flags (required): bit 0 = a column too heavy-tailed for the digit slices (the caller switches
// to the DMMA tiles), bit 1 = a column wide enough to need 8 slices (else 7); read on the device
// by launch_gram_i8_blocks
int launch_i8_colexp(const double* Xc, int64_t ld, int64_t len, int n, int* ex, cudaStream_t st, int* flags);
int launch_gram_i8_blocks(const double* Xc, int64_t ld, int64_t len, const int32_t* idx, int s, int p,
                          const int* ex_all, const int* flags, double* out, void* ws, size_t ws_bytes,
                          cudaStream_t st, cudaEvent_t after_slicing = nullptr);
int launch_gram_reduce_sym(const double* ws, int64_t n, int splits, double div, double* G, cudaStream_t st);
// K3: assemble block systems, Cholesky, explicit inverse.
struct SysArgs {
  const double* ws;   // [p][splits][s][s] partial Grams (lower), may be null
  int splits;
  double div, mul;    // val = (sum / div) * mul  (div==1/mul==1 skip the op)
  const double* H;    // optional dense H (row-major, ldh) -> + H[idx_i][idx_j]
  int64_t ldh;
  const double* hblk; // optional [p][s][s] precomputed H_bb per block (kernel strips on the fly):
                      // used instead of gathering H (H may then be null)
  const int32_t* idx;  // block indices (-1 = padding of the short last block -> identity row)
  const int32_t* blk_list;
  double shift, ridge_rel;
  int s;
  double* inv;        // [p][s][s] out
  double* mat_out;    // optional [p][s][s] copy of the assembled block matrix
  double* hbb_out;    // optional [p][s][s] copy of H_bb (gathered H block)
  double* scratch;    // [p][s][s] global scratch for the large-s path
  int32_t* info;
  const int32_t* done;  // skip when *done (converged / failed)
  int mode;             // FACTOR_INVERSE: sys^{-1} into inv; FACTOR_CHOL: lower L into inv
  double* inv2;         // FACTOR_CHOL: optional sys^{-1} as well
  double* cond_out;     // FACTOR_CHOL: optional per-block (max L_ii / min L_ii)^2
  int only_failed;      // factor only blocks whose info[b] != 0 (re-do pass)
  long long* trace;     // optional (block 0): [start, sweep start, 4 stamps per 8-pivot step ...]
};
int launch_inverse_large(const SysArgs& a, int p, cudaStream_t st);
size_t large_scratch_bytes(int s, int p);
constexpr int FACTOR_INVERSE = 0;
constexpr int FACTOR_CHOL = 1;
int launch_chol_system(const SysArgs& a, int p, cudaStream_t st);
size_t chol_scratch_bytes(int s, int p);

__global__ void iota_kernel(int32_t* v, int64_t n);

// label-weighted kernel strips (strips.cu): out[i][j] = y_{rows_i} y_j K(x_{rows_i}, x_{c_j}) from
// the zero-padded row-major samples Xp (N x ldd, ldd % 32 == 0); sq = |x_j|^2 (Gaussian only);
// c_j = j, or cols[j]; `batch` problems along blockIdx.z (rows / cols advance by s, out by s*ldo)
int launch_kernel_strip(const double* Xp, int64_t ldd, int64_t d, const int32_t* rows, int s, int64_t N,
                        const double* y, const double* sq, int kind, double sigma, double* out, int64_t ldo,
                        cudaStream_t st, const int32_t* cols = nullptr, int batch = 1);
int launch_row_sqnorm(const double* Xp, int64_t ldd, int64_t N, int64_t d, double* sq, cudaStream_t st);

// row-major X (m x n) -> column-major (ld x n), rows m..ld-1 zero
int launch_transpose_pad(const double* X, int64_t m, int64_t n, int64_t ld, double* Xc, cudaStream_t st);

}  // namespace rac
