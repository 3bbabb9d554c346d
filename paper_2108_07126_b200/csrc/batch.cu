// C ABI of the device batch layer (kernels_batch.cuh): expansion, batched
// exponential and batched GEMM over caller-owned device buffers on the
// caller's stream.  Context-free: the caller (the Python MatrixBatch /
// Workspace layer, or a C user) owns every buffer, including the scratch of
// sp_expm_batch_device, so back-to-back calls never allocate
// (chebyshev.py:221-246 Workspace contract).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>

#include "internal.h"
#include "kernels_batch.cuh"

using namespace sp;
using namespace sp::batch;

namespace {

#define BATCH_TRY(call)                                                                    \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      return set_error(SP_E_INTERNAL, "CUDA error %s (%s) at %s:%d", cudaGetErrorName(e_), \
                       cudaGetErrorString(e_), __FILE__, __LINE__);                        \
  } while (0)

int grid_stride_blocks(int64_t total) {
  int64_t b = (total + 255) / 256;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, 148 * 32));
}

int check_bits(int bits) {
  if (bits != 32 && bits != 64)
    return set_error(SP_E_CONFIG, "precision bits must be 32 or 64, got %d", bits);
  return SP_OK;
}

// fused on-chip Clenshaw for d <= 64: register tile and padded dimension
void fused_shape(int d, int* rt, int* dp) {
  *rt = d <= 16 ? 1 : (d <= 32 ? 2 : 4);
  *dp = (d + *rt - 1) / *rt * *rt;
}

template <class R, int RT>
int launch_fused(const ExpmParams& p, const void* g, void* u, cudaStream_t st) {
  const int nb = p.DP / RT, tpm = nb * nb, mpc = std::max(1, 256 / tpm);
  const size_t smem = (size_t)mpc * 2 * p.DP * p.DP * sizeof(cplx<R>);
  auto kern = expm_fused_kernel<R, RT>;
  if (smem > 48 * 1024)
    BATCH_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem));
  const int64_t blocks = (p.count + mpc - 1) / mpc;
  if (blocks > 0x7fffffff) return set_error(SP_E_CONFIG, "batch too large");
  kern<<<(unsigned)blocks, 256, smem, st>>>(p, (const cplx<R>*)g, (cplx<R>*)u);
  BATCH_TRY(cudaGetLastError());
  return SP_OK;
}

template <class R>
int gemm_launch(const GemmParams& p, const void* a, const void* b, const void* cin, void* c,
                cudaStream_t st) {
  const int tiles = (p.d + 63) / 64;
  const int64_t blocks = p.count * tiles * tiles;
  if (blocks == 0) return SP_OK;
  if (blocks > 0x7fffffff) return set_error(SP_E_CONFIG, "batch too large");
  gemm_batched_kernel<R><<<(unsigned)blocks, 256, 0, st>>>(
      p, (const cplx<R>*)a, (const cplx<R>*)b, (const cplx<R>*)cin, (cplx<R>*)c);
  BATCH_TRY(cudaGetLastError());
  return SP_OK;
}

template <class R>
int expm_impl(int dim, int64_t count, const void* g, int64_t stride_in, const sp_plan* plan,
              void* u, int64_t stride_out, void* scratch, cudaStream_t st) {
  const double span = plan->beta - plan->alpha;
  ExpmParams p;
  std::memset(&p, 0, sizeof(p));
  p.d = dim;
  p.m = plan->m_max;
  p.xscale = span == 0.0 ? 0.0 : 2.0 / span;
  p.center = 0.5 * (plan->alpha + plan->beta);
  std::memcpy(p.coef, plan->coeffs, sizeof(double) * 2 * (plan->m_max + 1));
  p.phase[0] = plan->phase[0];
  p.phase[1] = plan->phase[1];
  p.phase_one = (plan->phase[0] == 1.0 && plan->phase[1] == 0.0) ? 1 : 0;
  p.count = count;
  p.stride_in = stride_in;
  p.stride_out = stride_out;
  if (dim <= 64) {
    int rt, dp;
    fused_shape(dim, &rt, &dp);
    p.DP = dp;
    if (rt == 1) return launch_fused<R, 1>(p, g, u, st);
    if (rt == 2) return launch_fused<R, 2>(p, g, u, st);
    return launch_fused<R, 4>(p, g, u, st);
  }
  // d > 64: X and D1 in the caller's scratch, D0 = a compact staging of the
  // output (scratch too when the output is strided), m + 1 GEMM launches as
  // in the reference (the first multiplies zero)
  if (!scratch) return set_error(SP_E_CONFIG, "expm_batch for dim > 64 needs scratch");
  const int64_t dd = (int64_t)dim * dim;
  cplx<R>* x = (cplx<R>*)scratch;
  cplx<R>* d1 = x + count * dd;
  cplx<R>* d0 = d1 + count * dd;
  const int blocks = grid_stride_blocks(count * dd);
  xprep_kernel<R><<<blocks, 256, 0, st>>>((const cplx<R>*)g, stride_in, dim, count, p.xscale,
                                          p.center, x);
  BATCH_TRY(cudaGetLastError());
  BATCH_TRY(cudaMemsetAsync(d0, 0, (size_t)count * dd * sizeof(cplx<R>), st));
  BATCH_TRY(cudaMemsetAsync(d1, 0, (size_t)count * dd * sizeof(cplx<R>), st));
  GemmParams gp;
  std::memset(&gp, 0, sizeof(gp));
  gp.d = dim;
  gp.count = count;
  gp.sa = gp.sb = gp.sc = gp.scin = dd;
  gp.alpha[0] = 2.0;
  for (int k = plan->m_max; k >= 1; k -= 2) {
    const bool last = k == 1;
    gp.beta[0] = -1.0;
    gp.gamma[0] = plan->coeffs[2 * k];
    gp.gamma[1] = plan->coeffs[2 * k + 1];
    int rc = gemm_launch<R>(gp, x, d0, d1, d1, st);
    if (rc) return rc;
    const int k2 = last ? 0 : k - 1;
    gp.beta[0] = last ? -2.0 : -1.0;
    gp.gamma[0] = plan->coeffs[2 * k2];
    gp.gamma[1] = plan->coeffs[2 * k2 + 1];
    rc = gemm_launch<R>(gp, x, d1, d0, d0, st);
    if (rc) return rc;
  }
  phase_copy_kernel<R><<<blocks, 256, 0, st>>>(d0, dim, count, p.phase[0], p.phase[1],
                                               p.phase_one, (cplx<R>*)u, stride_out);
  BATCH_TRY(cudaGetLastError());
  return SP_OK;
}

}  // namespace

extern "C" {

int sp_expand_batch_device(int precision_bits, int dim, int n_terms, const void* d_terms,
                           int64_t count, const double* d_coeffs, double scale, void* d_out,
                           void* stream) {
  int rc = check_bits(precision_bits);
  if (rc) return rc;
  if (dim < 1 || n_terms < 1 || count < 0)
    return set_error(SP_E_SHAPE, "expansion needs dim >= 1, n_terms >= 1, count >= 0");
  if (count == 0) return SP_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t dd = (int64_t)dim * dim;
  const int blocks = grid_stride_blocks(count * dd);
  if (precision_bits == 64)
    expand_kernel<double><<<blocks, 256, 0, st>>>((const double2*)d_terms, n_terms, dd,
                                                  d_coeffs, count, scale,
                                                  (cplx<double>*)d_out);
  else
    expand_kernel<float><<<blocks, 256, 0, st>>>((const double2*)d_terms, n_terms, dd,
                                                 d_coeffs, count, scale, (cplx<float>*)d_out);
  BATCH_TRY(cudaGetLastError());
  return SP_OK;
}

size_t sp_expm_batch_scratch_bytes(int precision_bits, int dim, int64_t count) {
  if (dim <= 64 || count <= 0) return 0;
  const size_t el = precision_bits == 32 ? 8 : 16;
  return 3 * (size_t)count * dim * dim * el;
}

int sp_expm_batch_device(int precision_bits, int dim, int64_t count, const void* d_g,
                         int64_t stride_in, const sp_plan* plan, void* d_u, int64_t stride_out,
                         void* d_scratch, void* stream) {
  int rc = check_bits(precision_bits);
  if (rc) return rc;
  if (!plan) return set_error(SP_E_CONFIG, "null plan");
  if (dim < 1 || count < 0) return set_error(SP_E_SHAPE, "expm_batch needs dim >= 1, count >= 0");
  if (plan->m_max < 1 || plan->m_max > SP_MAX_ORDER || plan->m_max % 2 == 0)
    return set_error(SP_E_CONFIG, "plan order %d is not an odd order in 1..25", plan->m_max);
  if (stride_in < (int64_t)dim * dim || stride_out < (int64_t)dim * dim)
    return set_error(SP_E_SHAPE, "stride smaller than one matrix");
  if (count == 0) return SP_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (precision_bits == 64)
    return expm_impl<double>(dim, count, d_g, stride_in, plan, d_u, stride_out, d_scratch, st);
  return expm_impl<float>(dim, count, d_g, stride_in, plan, d_u, stride_out, d_scratch, st);
}

int sp_gemm_batched_device(int precision_bits, int dim, int64_t count, const void* d_a,
                           int64_t stride_a, const void* d_b, int64_t stride_b,
                           const double* alpha, const double* beta, const double* gamma,
                           void* d_c, int64_t stride_c, void* stream) {
  int rc = check_bits(precision_bits);
  if (rc) return rc;
  if (dim < 1 || count < 0) return set_error(SP_E_SHAPE, "gemm needs dim >= 1, count >= 0");
  if (count == 0) return SP_OK;
  GemmParams gp;
  std::memset(&gp, 0, sizeof(gp));
  gp.d = dim;
  gp.count = count;
  gp.sa = stride_a;
  gp.sb = stride_b;
  gp.sc = gp.scin = stride_c;
  gp.alpha[0] = alpha ? alpha[0] : 1.0;
  gp.alpha[1] = alpha ? alpha[1] : 0.0;
  gp.beta[0] = beta ? beta[0] : 0.0;
  gp.beta[1] = beta ? beta[1] : 0.0;
  gp.gamma[0] = gamma ? gamma[0] : 0.0;
  gp.gamma[1] = gamma ? gamma[1] : 0.0;
  gp.beta_zero = (gp.beta[0] == 0.0 && gp.beta[1] == 0.0) ? 1 : 0;
  cudaStream_t st = (cudaStream_t)stream;
  if (precision_bits == 64) return gemm_launch<double>(gp, d_a, d_b, d_c, d_c, st);
  return gemm_launch<float>(gp, d_a, d_b, d_c, d_c, st);
}

size_t sp_apply_batch_scratch_bytes(int precision_bits, int dim, int64_t count, int kind) {
  if (kind != 1 || dim < 1 || count < 0) return 0;
  const size_t el = precision_bits == 32 ? 8 : 16;
  return ((size_t)count + 1) * dim * dim * el;
}

int sp_apply_batch_device(int precision_bits, int dim, const void* d_u, int64_t count, int kind,
                          const void* d_states, void* d_out, void* d_scratch, void* stream) {
  int rc = check_bits(precision_bits);
  if (rc) return rc;
  if (dim < 1 || count < 0) return set_error(SP_E_SHAPE, "apply needs dim >= 1, count >= 0");
  if (kind != 0 && kind != 1)
    return set_error(SP_E_SHAPE, "state kind must be 0 (vectors) or 1 (density matrices)");
  if (count == 0) return SP_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (kind == 0) {
    const int blocks = grid_stride_blocks(count * dim);
    if (precision_bits == 64)
      apply_vec_kernel<double><<<blocks, 256, 0, st>>>(dim, count, (const cplx<double>*)d_u,
                                                       (const cplx<double>*)d_states,
                                                       (cplx<double>*)d_out);
    else
      apply_vec_kernel<float><<<blocks, 256, 0, st>>>(dim, count, (const cplx<float>*)d_u,
                                                      (const cplx<float>*)d_states,
                                                      (cplx<float>*)d_out);
    BATCH_TRY(cudaGetLastError());
    return SP_OK;
  }
  if (!d_scratch) return set_error(SP_E_CONFIG, "density-matrix apply needs scratch");
  // rho' = (U rho) U^+: two batched GEMMs (U and U^+ broadcast, stride 0)
  const size_t el = precision_bits == 32 ? 8 : 16;
  const size_t dd = (size_t)dim * dim;
  char* tmp = (char*)d_scratch;
  char* uadj = tmp + (size_t)count * dd * el;
  const int ablocks = grid_stride_blocks((int64_t)dd);
  if (precision_bits == 64)
    adjoint_kernel<double><<<ablocks, 256, 0, st>>>(dim, (const cplx<double>*)d_u,
                                                    (cplx<double>*)uadj);
  else
    adjoint_kernel<float><<<ablocks, 256, 0, st>>>(dim, (const cplx<float>*)d_u,
                                                   (cplx<float>*)uadj);
  BATCH_TRY(cudaGetLastError());
  rc = sp_gemm_batched_device(precision_bits, dim, count, d_u, 0, d_states, (int64_t)dd,
                              nullptr, nullptr, nullptr, tmp, (int64_t)dd, stream);
  if (rc) return rc;
  return sp_gemm_batched_device(precision_bits, dim, count, tmp, (int64_t)dd, uadj, 0, nullptr,
                                nullptr, nullptr, d_out, (int64_t)dd, stream);
}

}  // extern "C"
