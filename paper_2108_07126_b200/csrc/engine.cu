// C ABI + device orchestration of the equiprop hot path (sm_100a).
//
// Replaces, behind include/sliceprop_b200.h, the reference's
// IntegratorContext._slice_propagators + reduce_pairwise + equiprop +
// equiprop_all (sliceprop/propagator.py:132-331) with one streaming kernel
// pass per call (kernels.cuh) plus a short ordered-product tail.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "internal.h"
#include "kernels.cuh"
#include "kernels_tc.cuh"
#include "kernels_ps.cuh"
#include "kernels_ps3.cuh"
#include "kernels_ps3g.cuh"
#include "kernels_apply.cuh"
#include "kernels_d8.cuh"
#include "kernels_f32.cuh"

using namespace sp;

namespace {

const char* kVersion = "sliceprop_b200 0.1.0 (sm_100a)";
thread_local char g_err[512] = "";

enum Family {
  FAM_NONE = 0, FAM_S2, FAM_S4, FAM_T16, FAM_T32, FAM_T64, FAM_T128, FAM_T256, FAM_T512,
  FAM_T8
};

// families whose lane products / prefixes use the plain row-major layout
// (ordered tree, fold and prefix application shared with the small families)
bool plain_family(int fam) { return fam == FAM_S2 || fam == FAM_S4 || fam == FAM_T8; }

// tensor-core configurations (see TCCfg): D, WC, MT, NT, WPL, LPC, GPL, X-in-smem
using Cfg16 = TCCfg<16, 16, 1, 2, 1, 4, 1, true>;
using Cfg32 = TCCfg<32, 32, 1, 2, 4, 1, 1, true>;
using Cfg64 = TCCfg<64, 64, 1, 4, 8, 1, 1, true>;
using Cfg128 = TCCfg<128, 32, 1, 4, 8, 1, 4, false>;
using Cfg256 = TCCfg<256, 16, 2, 2, 8, 1, 16, false>;
// d <= 512: 64 CTAs x 8 columns per lane (2 lanes on 148 SMs); each CTA reads
// the whole A operand per GEMM for 8 columns, so this family is L2-bound
using Cfg512 = TCCfg<512, 8, 4, 1, 8, 1, 64, false>;
// Paterson-Stockmeyer configurations (A operands: smem for D <= 32, else L2)
using PS16 = PSCfg<16, 16, 1, 2, 1, 4, 1, true>;
using PS32 = PSCfg<32, 32, 1, 2, 4, 1, 1, true>;
using PS64 = PSCfg<64, 32, 1, 4, 4, 1, 2, false>;
using PS128 = PSCfg<128, 32, 1, 4, 8, 1, 4, false>;
using PS256 = PSCfg<256, 16, 2, 2, 8, 1, 16, false>;
using PS512 = PSCfg<512, 8, 4, 1, 8, 1, 64, false>;
// ... and with 3-multiplication complex products (3-plane operands)
using P3_16 = PS3Cfg<16, 16, 1, 2, 1, 4, 1, true>;
using P3_32 = PS3Cfg<32, 32, 1, 2, 4, 1, 1, true>;
// D=64: 2 CTAs x 32 columns, 8 warps of 16 x 16 (measured: +2% over 4 warps
// of 16 x 32; 4 CTAs x 16 columns -38%)
using P3_64 = PS3Cfg<64, 32, 1, 2, 8, 1, 2, false>;
// D=64 as ONE CTA per lane (all 64 columns, 8 warps of 16 x 32): CTA
// barriers instead of group barriers, 4x the MMA work per step
using P3_64s = PS3Cfg<64, 64, 1, 4, 8, 1, 1, false>;
// D=128: 4 CTAs x 32 columns per lane, 8 warps, 1 CTA per SM.  (Measured:
// 8 CTAs x 16 columns with 2 CTAs/SM is 1.4x slower — twice the L2 operand
// traffic and an 8-way group barrier outweigh the barrier overlap.)
using P3_128 = PS3Cfg<128, 32, 1, 4, 8, 1, 4, false>;
using P3_256 = PS3Cfg<256, 16, 2, 2, 8, 1, 16, false>;
using P3_512 = PS3Cfg<512, 8, 4, 1, 8, 1, 64, false>;

enum Algo { ALGO_AUTO = 0, ALGO_CLENSHAW = 1, ALGO_PS = 2, ALGO_PS3 = 3,
            ALGO_F32 = 4 /* reported only: the complex64-arithmetic lane kernel */,
            ALGO_SU2 = 5 /* reported only: the su(2) quaternion lane kernel */,
            ALGO_SU2_F32 = 6 /* reported only: the same in float32 arithmetic */,
            ALGO_U2 = 7 /* reported only: the same lanes for u(2) systems */,
            ALGO_U2_F32 = 8 /* reported only: u(2) lanes in float32 arithmetic */ };

// GEMMs per slice: Clenshaw m; PS (s-1) + (r-1) + 1, r = ceil((m+1)/s)
int ps_cost(int m, int s) {
  const int r = (m + 1 + s - 1) / s;
  return (s - 1) + (r - 1) + 1;
}

int ps_choose(int m) {
  // s <= 4: the power blocks T_1..T_{s-1} live in TMEM (4 blocks per
  // thread); larger s never lowers the cost for m <= 25.  SP_PS_S=<s>
  // forces the split (A/B timing)
  static const int s_env = [] {
    const char* e = getenv("SP_PS_S");
    return e ? atoi(e) : 0;
  }();
  if (s_env >= 2 && s_env <= 4 && (m + 1 + s_env - 1) / s_env >= 2) return s_env;
  int best = 0, cost = m;
  for (int s = 2; s <= 4; ++s) {
    const int r = (m + 1 + s - 1) / s;
    if (r < 2 || r * s > PS_MAXC) continue;
    if (ps_cost(m, s) < cost) {
      cost = ps_cost(m, s);
      best = s;
    }
  }
  return best;  // 0: no saving over Clenshaw
}

// alpha_{j,i} of p = sum_j Q_j T_j(T_s), Q_j = sum_i alpha_{j,i} T_i, from
// the plan's Chebyshev coefficients a'_0 = a_0, a'_k = 2 a_k (the
// reference series p = a_0 + 2 sum a_k T_k), by the top-down solve of
// T_i T_js = (T_{js+i} + T_{|js-i|}) / 2; 80-bit accumulation.
void ps_coefficients(const double* coef, int m, int s, double* alpha, int* r_out) {
  typedef long double ld;
  const int r = (m + 1 + s - 1) / s;
  std::vector<ld> ar((r + 1) * s, 0.0L), ai((r + 1) * s, 0.0L);
  auto apr = [&](int k) -> ld { return k > m ? 0.0L : (k == 0 ? 1.0L : 2.0L) * (ld)coef[2 * k]; };
  auto api = [&](int k) -> ld {
    return k > m ? 0.0L : (k == 0 ? 1.0L : 2.0L) * (ld)coef[2 * k + 1];
  };
  for (int j = r - 1; j >= 0; --j)
    for (int i = 0; i < s; ++i) {
      const int k = j * s + i;
      ld vr, vi;
      if (j >= 1 && i >= 1) {
        vr = 2.0L * apr(k) - ar[(j + 1) * s + (s - i)];
        vi = 2.0L * api(k) - ai[(j + 1) * s + (s - i)];
      } else if (j >= 1) {
        vr = apr(k);
        vi = api(k);
      } else if (i >= 1) {
        vr = apr(i) - ar[1 * s + (s - i)] / 2.0L;
        vi = api(i) - ai[1 * s + (s - i)] / 2.0L;
      } else {
        vr = apr(0);
        vi = api(0);
      }
      ar[j * s + i] = vr;
      ai[j * s + i] = vi;
    }
  for (int q = 0; q < r * s; ++q) {
    alpha[2 * q] = (double)ar[q];
    alpha[2 * q + 1] = (double)ai[q];
  }
  *r_out = r;
}

// alpha alternates exactly real / imaginary with the parity of j*s + i
int ps_alpha_alt(const double* alpha, int count) {
  for (int q = 0; q < count; ++q)
    if (alpha[2 * q + ((q & 1) ? 0 : 1)] != 0.0) return 0;
  return 1;
}

int family_for(int d, int* D) {
  if (d <= 2) { *D = 2; return FAM_S2; }
  if (d <= 4) { *D = 4; return FAM_S4; }
  if (d <= 8) { *D = 8; return FAM_T8; }
  if (d <= 16) { *D = 16; return FAM_T16; }
  if (d <= 32) { *D = 32; return FAM_T32; }
  if (d <= 64) { *D = 64; return FAM_T64; }
  if (d <= 128) { *D = 128; return FAM_T128; }
  if (d <= 256) { *D = 256; return FAM_T256; }
  if (d <= 512) { *D = 512; return FAM_T512; }
  *D = 0;
  return FAM_NONE;
}

bool d64_single();

const char* family_kernel_name(int fam, int algo) {
  if (algo == 5) return "lane_su2_kernel";
  if (algo == 6) return "lane_su2_f32_kernel";
  if (algo == 7) return "lane_u2_kernel";
  if (algo == 8) return "lane_u2_f32_kernel";
  if (algo == 4)  // complex64 arithmetic (kernels_f32.cuh)
    return fam == FAM_S2 ? "lane_f32_kernel<2>" : fam == FAM_S4 ? "lane_f32_kernel<4>"
                                                                : "lane_f32_kernel<8>";
  if (fam == FAM_T8)
    return algo == 3 ? "lane_d8_kernel<ps3m>" : algo == 2 ? "lane_d8_kernel<ps>"
                                                          : "lane_d8_kernel<clenshaw>";
  if (algo == 3) {
    switch (fam) {
      case FAM_T16: return "lane_ps3_kernel<D16>";
      case FAM_T32: return "lane_ps3_kernel<D32>";
      case FAM_T64:
        return d64_single() ? "lane_ps3g_kernel<D64,group1>" : "lane_ps3g_kernel<D64,group2>";
      case FAM_T128: return "lane_ps3g_kernel<D128,group4>";
      case FAM_T256: return "lane_ps3g_kernel<D256,group16>";
      case FAM_T512: return "lane_ps3g_kernel<D512,group64>";
    }
  }
  if (algo == 2) {
    switch (fam) {
      case FAM_T16: return "lane_ps_kernel<D16>";
      case FAM_T32: return "lane_ps_kernel<D32>";
      case FAM_T64: return "lane_ps_kernel<D64,group2>";
      case FAM_T128: return "lane_ps_kernel<D128,group4>";
      case FAM_T256: return "lane_ps_kernel<D256,group16>";
      case FAM_T512: return "lane_ps_kernel<D512,group64>";
    }
  }
  switch (fam) {
    case FAM_S2: return "lane_small_kernel<2,1>";
    case FAM_S4: return "lane_small_kernel<4,4>";
    case FAM_T16: return "lane_tc_kernel<D16>";
    case FAM_T32: return "lane_tc_kernel<D32>";
    case FAM_T64: return "lane_tc_kernel<D64>";
    case FAM_T128: return "lane_tc_kernel<D128,group4>";
    case FAM_T256: return "lane_tc_kernel<D256,group16>";
    case FAM_T512: return "lane_tc_kernel<D512,group64>";
  }
  return "none";
}

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
};

}  // namespace

struct sp_ctx {
  int bits = 64;
  int device = 0;
  char err[512] = "";
  // host-side system
  bool loaded = false;
  int dim = 0, n_ctrl = 0, n_terms = 0, mode = 0;
  std::vector<double> terms_host;  // T x d x d complex128 interleaved
  bool herm_exact = false;         // every term bitwise Hermitian
  bool su2_terms = false;          // d = 2, every term bitwise Hermitian and traceless
  bool u2_terms = false;           // d = 2, every term bitwise Hermitian, some with a trace
  // device-side
  bool dev_ready = false;
  bool terms_uploaded = false;
  int sms = 0;
  cudaStream_t stream = nullptr;
  int fam = FAM_NONE, D = 0;
  DevBuf terms, amps, lanes, ctab, tree0, tree1, xglob, gctr, result, out, cumP, cumE, cumO,
      fold_scratch, psA, tpriv, viol, terms3, tailctr, seqA, scanEin, lstarts, scanS, scanA;
  cudaStream_t viol_stream = nullptr;
  int64_t viol_pts = 0;
  // page-locked copy of the violation slots: the host entry points fetch it
  // with the result before their one stream synchronisation
  unsigned long long* viol_host = nullptr;
  // page-locked staging of the d x d result of the host entry points
  void* out_host = nullptr;
  size_t out_host_bytes = 0;
  int algo = 0;          // Algo
  int last_algo = 0;     // algorithm of the last lane pass
  int last_gemms = 0;    // GEMMs per slice of the last lane pass
  int last_lanes = 0;    // lanes of the last lane pass
  // profiling
  bool prof = false;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  bool ev_pending = false;
  float last_ms = 0.f;
  int launches = 0;
  double flops = 0.0;
  const char* kname = "none";
  // single-process multi-device context (sp_create with num_gpus > 1): the
  // per-device child contexts, each propagating one contiguous block of
  // slices; the block products are gathered by peer copies onto the first
  // device and multiplied there in time order
  std::vector<sp_ctx*> kids;
  bool block64 = false;  // child: write its block product in complex128
  DevBuf gather;         // first child: P x d x d complex128 block products
  DevBuf result2;        // first child: the d x d result of the gather product
  int64_t multi_viol = -1;  // first offender of the last multi-device call
  bool last_multi = false;  // the last call was a multi-device equiprop
  std::vector<cudaEvent_t> kid_done;
};

namespace {

// the call's d x d output in complex64 (fp32 contexts, except a multi-device
// child writing its block for the complex128 gather)
bool out32(const sp_ctx* ctx) { return ctx->bits == 32 && !ctx->block64; }

int fail(sp_ctx* ctx, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  if (ctx) snprintf(ctx->err, sizeof(ctx->err), "%s", buf);
  snprintf(g_err, sizeof(g_err), "%s", buf);
  return code;
}

}  // namespace

int sp::set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

namespace {

#define CUDA_TRY(ctx, call)                                                              \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return fail(ctx, SP_E_INTERNAL, "CUDA error %s (%s) at %s:%d", cudaGetErrorName(e_), \
                  cudaGetErrorString(e_), __FILE__, __LINE__);                           \
  } while (0)

int ensure(sp_ctx* ctx, DevBuf& b, size_t bytes) {
  if (bytes == 0) bytes = 16;
  if (b.cap >= bytes) return SP_OK;
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.cap = 0;
  CUDA_TRY(ctx, cudaMalloc(&b.p, bytes));
  b.cap = bytes;
  return SP_OK;
}

int device_init(sp_ctx* ctx) {
  if (ctx->dev_ready) return SP_OK;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0)
    return fail(ctx, SP_E_INTERNAL,
                "no CUDA device available (%s): the sliceprop_b200 propagation path is "
                "GPU-only and has no CPU fallback",
                e == cudaSuccess ? "device count 0" : cudaGetErrorString(e));
  if (ctx->device < 0 || ctx->device >= n)
    return fail(ctx, SP_E_CONFIG, "device ordinal %d out of range (have %d)", ctx->device, n);
  CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  cudaDeviceProp prop;
  CUDA_TRY(ctx, cudaGetDeviceProperties(&prop, ctx->device));
  if (prop.major < 10)
    return fail(ctx, SP_E_INTERNAL, "device %s (sm_%d%d) is not a Blackwell sm_100 part",
                prop.name, prop.major, prop.minor);
  ctx->sms = prop.multiProcessorCount;
  CUDA_TRY(ctx, cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
  CUDA_TRY(ctx, cudaEventCreate(&ctx->ev0));
  CUDA_TRY(ctx, cudaEventCreate(&ctx->ev1));
  ctx->dev_ready = true;
  return SP_OK;
}

template <class C>
int tc_prepare(sp_ctx* ctx) {
  CUDA_TRY(ctx, cudaFuncSetAttribute(lane_tc_kernel<C>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)C::SMEM));
  return SP_OK;
}

template <class C, bool M3 = false>
int ps_prepare(sp_ctx* ctx);
template <class C>
int ps3_prepare(sp_ctx* ctx);

int d8_prepare(sp_ctx* ctx);

// permute + pad the host terms into the family's device layout
int upload_terms(sp_ctx* ctx) {
  const int d = ctx->dim, D = ctx->D, T = ctx->n_terms;
  std::vector<double> h;
  if (ctx->fam == FAM_T8) {
    // m8n8k4 A-fragment order (kernels_d8.cuh d8_apos), complex interleaved
    h.assign((size_t)T * 64 * 2, 0.0);
    for (int t = 0; t < T; ++t)
      for (int r = 0; r < d; ++r)
        for (int c = 0; c < d; ++c) {
          const double* src = &ctx->terms_host[(((size_t)t * d + r) * d + c) * 2];
          const int pos = (c >> 2) * 32 + ((r << 2) | (c & 3));
          h[((size_t)t * 64 + pos) * 2] = src[0];
          h[((size_t)t * 64 + pos) * 2 + 1] = src[1];
        }
  } else if (ctx->fam == FAM_S2 || ctx->fam == FAM_S4) {
    h.assign((size_t)T * D * D * 2, 0.0);
    for (int t = 0; t < T; ++t)
      for (int r = 0; r < d; ++r)
        for (int c = 0; c < d; ++c) {
          const double* src = &ctx->terms_host[(((size_t)t * d + r) * d + c) * 2];
          double* dst = &h[(((size_t)t * D + r) * D + c) * 2];
          dst[0] = src[0];
          dst[1] = src[1];
        }
  } else {
    const size_t xd = (size_t)2 * D * D;
    h.assign((size_t)T * xd, 0.0);
    for (int t = 0; t < T; ++t)
      for (int r = 0; r < d; ++r)
        for (int c = 0; c < d; ++c) {
          const double* src = &ctx->terms_host[(((size_t)t * d + r) * d + c) * 2];
          h[t * xd + xfrag_index(D, r, c, 0)] = src[0];
          h[t * xd + xfrag_index(D, r, c, 1)] = src[1];
        }
  }
  int rc = ensure(ctx, ctx->terms, h.size() * sizeof(double));
  if (rc) return rc;
  CUDA_TRY(ctx, cudaMemcpy(ctx->terms.p, h.data(), h.size() * sizeof(double),
                           cudaMemcpyHostToDevice));
  if (!plain_family(ctx->fam)) {
    // 3-plane (re, im, re+im) copy for the 3-multiplication kernels
    const size_t xd3 = (size_t)3 * D * D;
    std::vector<double> h3((size_t)T * xd3, 0.0);
    for (int t = 0; t < T; ++t)
      for (int r = 0; r < d; ++r)
        for (int c = 0; c < d; ++c) {
          const double* src = &ctx->terms_host[(((size_t)t * d + r) * d + c) * 2];
          h3[t * xd3 + xfrag3_index(D, r, c, 0)] = src[0];
          h3[t * xd3 + xfrag3_index(D, r, c, 1)] = src[1];
          h3[t * xd3 + xfrag3_index(D, r, c, 2)] = src[0] + src[1];
        }
    rc = ensure(ctx, ctx->terms3, h3.size() * sizeof(double));
    if (rc) return rc;
    CUDA_TRY(ctx, cudaMemcpy(ctx->terms3.p, h3.data(), h3.size() * sizeof(double),
                             cudaMemcpyHostToDevice));
  }
  if (ctx->fam == FAM_T8) {
    rc = d8_prepare(ctx);
    if (rc) return rc;
  }
  switch (ctx->fam) {
    case FAM_T16: rc = ps3_prepare<P3_16>(ctx); break;
    case FAM_T32: rc = ps3_prepare<P3_32>(ctx); break;
    case FAM_T64:
      rc = ps3_prepare<P3_64>(ctx);
      if (!rc) rc = ps3_prepare<P3_64s>(ctx);
      break;
    case FAM_T128: rc = ps3_prepare<P3_128>(ctx); break;
    case FAM_T256: rc = ps3_prepare<P3_256>(ctx); break;
    case FAM_T512: rc = ps3_prepare<P3_512>(ctx); break;
    default: break;
  }
  if (rc) return rc;
  switch (ctx->fam) {
    case FAM_T16: rc = tc_prepare<Cfg16>(ctx); break;
    case FAM_T32: rc = tc_prepare<Cfg32>(ctx); break;
    case FAM_T64: rc = tc_prepare<Cfg64>(ctx); break;
    case FAM_T128: rc = tc_prepare<Cfg128>(ctx); break;
    case FAM_T256: rc = tc_prepare<Cfg256>(ctx); break;
    case FAM_T512: rc = tc_prepare<Cfg512>(ctx); break;
    default: break;
  }
  if (rc) return rc;
  switch (ctx->fam) {
    case FAM_T16: rc = ps_prepare<PS16>(ctx); break;
    case FAM_T32: rc = ps_prepare<PS32>(ctx); break;
    case FAM_T64: rc = ps_prepare<PS64>(ctx); break;
    case FAM_T128: rc = ps_prepare<PS128>(ctx); break;
    case FAM_T256: rc = ps_prepare<PS256>(ctx); break;
    case FAM_T512: rc = ps_prepare<PS512>(ctx); break;
    default: break;
  }
  if (rc) return rc;
  ctx->terms_uploaded = true;
  return SP_OK;
}

int64_t slice_count_for(int mode, int64_t pts, int* code) {
  *code = SP_OK;
  if (mode == SP_MODE_MIDPOINT) return pts;
  if (mode >= SP_MODE_GAUSS2) {  // two Gauss-Legendre nodes per slice
    if (pts < 2 || pts % 2 != 0) {
      *code = SP_E_SAMPLING_PARITY;
      return -1;
    }
    return pts / 2;
  }
  if (pts < 3 || pts % 2 == 0) {
    *code = SP_E_SAMPLING_PARITY;
    return -1;
  }
  return (pts - 1) / 2;
}

const char* parity_message(int mode) {
  return mode >= SP_MODE_GAUSS2
             ? "Gauss-Legendre quadrature needs an even number of samples >= 2"
             : "three-point quadrature needs an odd number of samples >= 3";
}

int grid_for(int64_t total, int threads) {
  int64_t b = (total + threads - 1) / threads;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, 148 * 64));
}

template <class C>
int tc_lanes(sp_ctx* ctx, int64_t n) {
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, lane_tc_kernel<C>, C::THREADS, C::SMEM);
  if (occ < 1) occ = 1;
  int64_t ctas = (int64_t)ctx->sms * occ;
  int64_t units = (C::GPL > 1) ? ctas / C::GPL : ctas * C::LPC;
  return (int)std::max<int64_t>(1, std::min<int64_t>(units, n));
}

template <class C>
int tc_launch(sp_ctx* ctx, const SliceJob& job, int lanes, double2* lane_out,
              double2* prefix_out, cudaStream_t st) {
  const int groups = (lanes + C::LPC - 1) / C::LPC;
  const int grid = groups * C::GPL;
  double* xg = nullptr;
  unsigned* ctr = nullptr;
  if (C::GPL > 1) {
    int rc = ensure(ctx, ctx->xglob, (size_t)groups * 2 * C::XDBL * sizeof(double));
    if (rc) return rc;
    rc = ensure(ctx, ctx->gctr, (size_t)groups * sizeof(unsigned));
    if (rc) return rc;
    CUDA_TRY(ctx, cudaMemsetAsync(ctx->gctr.p, 0, (size_t)groups * sizeof(unsigned), st));
    xg = (double*)ctx->xglob.p;
    ctr = (unsigned*)ctx->gctr.p;
    const double* terms = (const double*)ctx->terms.p;
    void* args[] = {(void*)&job, (void*)&terms, (void*)&lanes, (void*)&xg,
                    (void*)&ctr,  (void*)&lane_out, (void*)&prefix_out};
    // co-residency of a lane's GPL CTAs is required by the group barrier
    if (ctx->prof) CUDA_TRY(ctx, cudaEventRecord(ctx->ev0, st));
    CUDA_TRY(ctx, cudaLaunchCooperativeKernel((const void*)lane_tc_kernel<C>, dim3(grid),
                                              dim3(C::THREADS), args, C::SMEM, st));
  } else {
    if (ctx->prof) CUDA_TRY(ctx, cudaEventRecord(ctx->ev0, st));
    lane_tc_kernel<C><<<grid, C::THREADS, C::SMEM, st>>>(
        job, (const double*)ctx->terms.p, lanes, xg, ctr, lane_out, prefix_out);
  }
  CUDA_TRY(ctx, cudaGetLastError());
  if (ctx->prof) CUDA_TRY(ctx, cudaEventRecord(ctx->ev1, st));
  ++ctx->launches;
  return SP_OK;
}

// lane_ps_kernel (4 real products per complex product) or lane_ps3_kernel (3)
template <class C, bool M3>
constexpr auto ps_kernel() {
  if constexpr (M3 && (C::GPL > 1 || !C::XS))
    return lane_ps3g_kernel<C>;  // group families: pipelined slice loop
  else if constexpr (M3)
    return lane_ps3_kernel<C>;
  else
    return lane_ps_kernel<C>;
}

template <class C, bool M3>
int ps_prepare(sp_ctx* ctx) {
  CUDA_TRY(ctx, cudaFuncSetAttribute(ps_kernel<C, M3>(),
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)C::SMEM));
  if constexpr (!M3 && C::GPL == 1) {
    CUDA_TRY(ctx, cudaFuncSetAttribute(lane_ps_kernel<C, 3, 5>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
    CUDA_TRY(ctx, cudaFuncSetAttribute(lane_ps_kernel<C, 4, 4>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
    CUDA_TRY(ctx, cudaFuncSetAttribute(lane_ps_kernel<C, 2, 4>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
  }
  return SP_OK;
}

template <class C, bool M3 = false>
int ps_lanes(sp_ctx* ctx, int64_t n) {
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, ps_kernel<C, M3>(), C::THREADS, C::SMEM);
  if constexpr (M3) occ = std::min(occ, 512 / C::TMEM_COLS);  // TMEM columns per SM
  if (occ < 1) occ = 1;
  int64_t ctas = (int64_t)ctx->sms * occ;
  int64_t units = (C::GPL > 1) ? ctas / C::GPL : ctas * C::LPC;
  return (int)std::max<int64_t>(1, std::min<int64_t>(units, n));
}

template <class C>
int ps3_prepare(sp_ctx* ctx) { return ps_prepare<C, true>(ctx); }
// D = 64 lane shape: one CTA (default) or a group of two (SP_D64_GROUP=2, A/B)
bool d64_single() {
  static const bool single = [] {
    const char* e = getenv("SP_D64_GROUP");
    return !(e && e[0] == '2');
  }();
  return single;
}
template <class C>
int ps3_lanes(sp_ctx* ctx, int64_t n) { return ps_lanes<C, true>(ctx, n); }

template <class C, bool M3 = false>
int ps_launch(sp_ctx* ctx, const PSJob& pj, int lanes, double2* lane_out, double2* prefix_out,
              cudaStream_t st) {
  const int groups = (lanes + C::LPC - 1) / C::LPC;
  const int grid = groups * C::GPL;
  constexpr int NE = C::MT * C::NT * 4;
  int rc = ensure(ctx, ctx->tpriv,
                  (size_t)grid * (pj.s - 1) * NE * C::THREADS * sizeof(double2));
  if (rc) return rc;
  double2* tpriv = (double2*)ctx->tpriv.p;
  // the group PS3 kernel assembles from the 2-plane terms (and forms the sum
  // plane itself); the single-CTA PS3 kernel reads the 3-plane copy
  const double* terms =
      (const double*)((M3 && C::GPL == 1 && C::XS) ? ctx->terms3.p : ctx->terms.p);
  double* ga = nullptr;
  unsigned* ctr = nullptr;
  if (C::GPL > 1 || (M3 && !C::XS)) {
    rc = ensure(ctx, ctx->psA, (size_t)groups * 3 * C::XDBL * sizeof(double));
    if (rc) return rc;
    ga = (double*)ctx->psA.p;
    if (C::GPL > 1) {  // co-resident lane groups, arrival counters zeroed
      rc = ensure(ctx, ctx->gctr, (size_t)groups * sizeof(unsigned));
      if (rc) return rc;
      CUDA_TRY(ctx, cudaMemsetAsync(ctx->gctr.p, 0, (size_t)groups * sizeof(unsigned), st));
      ctr = (unsigned*)ctx->gctr.p;
    }
    void* args[] = {(void*)&pj, (void*)&terms, (void*)&lanes, (void*)&ga, (void*)&ctr,
                    (void*)&tpriv, (void*)&lane_out, (void*)&prefix_out};
    if (ctx->prof) CUDA_TRY(ctx, cudaEventRecord(ctx->ev0, st));
    if (C::GPL > 1)
      CUDA_TRY(ctx, cudaLaunchCooperativeKernel((const void*)ps_kernel<C, M3>(), dim3(grid),
                                                dim3(C::THREADS), args, C::SMEM, st));
    else
      CUDA_TRY(ctx, cudaLaunchKernel((const void*)ps_kernel<C, M3>(), dim3(grid),
                                     dim3(C::THREADS), args, C::SMEM, st));
  } else {
    if (ctx->prof) CUDA_TRY(ctx, cudaEventRecord(ctx->ev0, st));
    // smem-resident 4-product families: the (s, r) split of the common
    // orders (m = 13 -> (3, 5), m = 15 -> (4, 4), fp32 m = 7 -> (2, 4))
    // compiled in
    auto kern = ps_kernel<C, M3>();
    if constexpr (!M3 && C::GPL == 1) {
      if (pj.s == 3 && pj.r == 5) kern = lane_ps_kernel<C, 3, 5>;
      if (pj.s == 4 && pj.r == 4) kern = lane_ps_kernel<C, 4, 4>;
      if (pj.s == 2 && pj.r == 4) kern = lane_ps_kernel<C, 2, 4>;
    }
    kern<<<grid, C::THREADS, C::SMEM, st>>>(pj, terms, lanes, ga, ctr, tpriv, lane_out,
                                            prefix_out);
  }
  CUDA_TRY(ctx, cudaGetLastError());
  if (ctx->prof) CUDA_TRY(ctx, cudaEventRecord(ctx->ev1, st));
  ++ctx->launches;
  return SP_OK;
}

template <class C>
int ps3_launch(sp_ctx* ctx, const PSJob& pj, int lanes, double2* lane_out, double2* prefix_out,
               cudaStream_t st) {
  return ps_launch<C, true>(ctx, pj, lanes, lane_out, prefix_out, st);
}

// ---- tensor-core prefix application (equiprop_all / sequential total)
using AP16 = TCCfg<16, 16, 1, 2, 1, 1, 1, false>;
using AP32 = TCCfg<32, 32, 1, 2, 4, 1, 1, false>;
using AP64 = TCCfg<64, 64, 1, 4, 8, 1, 1, false>;
using AP128 = TCCfg<128, 32, 1, 4, 8, 1, 4, false>;
using AP256 = TCCfg<256, 16, 2, 2, 8, 1, 16, false>;
using AP512 = TCCfg<512, 8, 4, 1, 8, 1, 64, false>;

template <class C>
int ap_launch(sp_ctx* ctx, const double* P, const double2* E, int64_t n, int lanes, void* out,
              cudaStream_t st, int out_d = -1, int out_fp32 = -1) {
  const size_t smem = (size_t)C::BDBL * sizeof(double);
  CUDA_TRY(ctx, cudaFuncSetAttribute(apply_prefix_tc_kernel<C>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t target = std::max<int64_t>(1, (int64_t)ctx->sms * 4 / C::GPL);
  const int64_t spb = std::max<int64_t>(1, (n + target - 1) / target);
  const int64_t chunks = (n + spb - 1) / spb;
  apply_prefix_tc_kernel<C><<<dim3((unsigned)chunks, C::GPL), C::THREADS, smem, st>>>(
      P, E, n, lanes, spb, out_d >= 0 ? out_d : ctx->dim,
      out_fp32 >= 0 ? out_fp32 : (out32(ctx) ? 1 : 0), out);
  CUDA_TRY(ctx, cudaGetLastError());
  ++ctx->launches;
  return SP_OK;
}

// (out_d / out_fp32: the output block size and dtype, default the context's d
// and working dtype; the scan below writes full D x D complex128 blocks)
int tc_apply(sp_ctx* ctx, const double* P, const double2* E, int64_t n, int lanes, void* out,
             cudaStream_t st, int out_d = -1, int out_fp32 = -1) {
  switch (ctx->fam) {
    case FAM_T16: return ap_launch<AP16>(ctx, P, E, n, lanes, out, st, out_d, out_fp32);
    case FAM_T32: return ap_launch<AP32>(ctx, P, E, n, lanes, out, st, out_d, out_fp32);
    case FAM_T64: return ap_launch<AP64>(ctx, P, E, n, lanes, out, st, out_d, out_fp32);
    case FAM_T128: return ap_launch<AP128>(ctx, P, E, n, lanes, out, st, out_d, out_fp32);
    case FAM_T256: return ap_launch<AP256>(ctx, P, E, n, lanes, out, st, out_d, out_fp32);
    case FAM_T512: return ap_launch<AP512>(ctx, P, E, n, lanes, out, st, out_d, out_fp32);
  }
  return fail(ctx, SP_E_INTERNAL, "no tensor-core apply for this family");
}

// count row-major complex D x D matrices -> A-native 2-plane layout (exact)
__global__ void batch_afrag_kernel(const double2* __restrict__ in, int64_t count, int D,
                                   double* __restrict__ out) {
  const int64_t dd = (int64_t)D * D, total = count * dd;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t mtx = e / dd;
    const int rc = (int)(e % dd), r = rc / D, c = rc % D;
    double* o = out + mtx * 2 * dd;
    o[xfrag_index(D, r, c, 0)] = in[e].x;
    o[xfrag_index(D, r, c, 1)] = in[e].y;
  }
}

// Exclusive prefixes of the lane products on tensor cores (tensor-core
// families): E_0 = I, E_l = M_{l-1} ... M_0 into ctx->cumE, by a
// Hillis-Steele scan: S <- (I, M_0, ..., M_{L-2}), then for o = 1, 2, 4, ...
// S_l <- S_l S_{l-o} (l >= o) as one batched DMMA launch per level (the
// prefix-application kernel with one "lane" per item).  log2(L) levels of
// parallel GEMMs instead of L dependent ones on one SM (the SIMT fold: 13.6 ms
// for 37 lanes of D = 128).  The sequential reduction uses the same E_{L-1},
// so equiprop_all's last entry stays bitwise equal to it.
int tc_scan(sp_ctx* ctx, const double2* prods, int L, cudaStream_t st) {
  const int D = ctx->D;
  const size_t dd = (size_t)D * D;
  int rc = ensure(ctx, ctx->cumE, (size_t)L * dd * sizeof(double2));
  if (rc) return rc;
  rc = ensure(ctx, ctx->scanS, (size_t)L * dd * sizeof(double2));
  if (rc) return rc;
  rc = ensure(ctx, ctx->scanA, (size_t)L * 2 * dd * sizeof(double));
  if (rc) return rc;
  double2* S = (double2*)ctx->scanS.p;
  double2* T = (double2*)ctx->cumE.p;
  embed_kernel<<<grid_for((int64_t)dd, 256), 256, 0, st>>>(nullptr, 1, 0, D, S);
  CUDA_TRY(ctx, cudaGetLastError());
  ++ctx->launches;
  if (L > 1)
    CUDA_TRY(ctx, cudaMemcpyAsync(S + dd, prods, (size_t)(L - 1) * dd * sizeof(double2),
                                  cudaMemcpyDeviceToDevice, st));
  for (int o = 1; o < L; o <<= 1) {
    const int64_t m = L - o;
    batch_afrag_kernel<<<grid_for(m * (int64_t)dd, 256), 256, 0, st>>>(
        S + (size_t)o * dd, m, D, (double*)ctx->scanA.p);
    CUDA_TRY(ctx, cudaGetLastError());
    ++ctx->launches;
    CUDA_TRY(ctx, cudaMemcpyAsync(T, S, (size_t)o * dd * sizeof(double2),
                                  cudaMemcpyDeviceToDevice, st));
    rc = tc_apply(ctx, (const double*)ctx->scanA.p, S, m, (int)m, T + (size_t)o * dd, st, D, 0);
    if (rc) return rc;
    std::swap(S, T);
  }
  if (S != (double2*)ctx->cumE.p)
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->cumE.p, S, (size_t)L * dd * sizeof(double2),
                                  cudaMemcpyDeviceToDevice, st));
  return SP_OK;
}

// one CTA folds a chunk of CH consecutive products by the level-order smem
// tree (later on the left, odd leftovers carried): log2(CH) levels per launch
__global__ void chunk_reduce_kernel(const double2* __restrict__ in, int cnt, int D, int CH,
                                    double2* __restrict__ out) {
  extern __shared__ double2 cbuf[];
  const int dd = D * D;
  double2* buf[2] = {cbuf, cbuf + (size_t)CH * dd};
  const int base = blockIdx.x * CH;
  const int here = min(CH, cnt - base);
  for (int e = threadIdx.x; e < here * dd; e += blockDim.x)
    buf[0][e] = in[(size_t)base * dd + e];
  __syncthreads();
  int c = here, src = 0;
  while (c > 1) {
    const int pairs = c >> 1;
    for (int e = threadIdx.x; e < pairs * dd; e += blockDim.x) {
      const int p = e / dd, rc = e % dd, r = rc / D, cc = rc % D;
      buf[src ^ 1][p * dd + rc] =
          cdot(&buf[src][(2 * p + 1) * dd + r * D], &buf[src][(2 * p) * dd], D, cc, D);
    }
    if (c & 1)
      for (int e = threadIdx.x; e < dd; e += blockDim.x)
        buf[src ^ 1][pairs * dd + e] = buf[src][(c - 1) * dd + e];
    __syncthreads();
    c = pairs + (c & 1);
    src ^= 1;
  }
  for (int e = threadIdx.x; e < dd; e += blockDim.x) out[(size_t)blockIdx.x * dd + e] = buf[src][e];
}

// pairwise tree over cnt matrices (in place ping-pong); returns the buffer
// holding the single result
int reduce_pairwise_dev(sp_ctx* ctx, const double2* in, int cnt, int D, cudaStream_t st,
                        const double2** result) {
  const size_t dd = (size_t)D * D;
  if (cnt == 1) {
    *result = in;
    return SP_OK;
  }
  int rc = ensure(ctx, ctx->tree0, ((cnt + 1) / 2) * dd * sizeof(double2));
  if (rc) return rc;
  rc = ensure(ctx, ctx->tree1, ((cnt + 3) / 4 + 1) * dd * sizeof(double2));
  if (rc) return rc;
  const double2* src = in;
  DevBuf* bufs[2] = {&ctx->tree0, &ctx->tree1};
  int which = 0;
  while (cnt > 1) {
    const int nxt = cnt / 2 + (cnt & 1);
    double2* dst = (double2*)bufs[which]->p;
    // chunks of CH products per CTA (smem budget 96 KB: D <= 32) cut the
    // launches of a deep tree to log_CH(cnt); larger D: one level per launch
    const int ch = std::min(256, 98304 / (int)(dd * 2 * sizeof(double2)));
    if (ch >= 3 && cnt > 2) {
      const int blocks = (cnt + ch - 1) / ch;
      const size_t sm = (size_t)2 * ch * dd * sizeof(double2);
      if (sm > 48 * 1024)
        CUDA_TRY(ctx, cudaFuncSetAttribute(chunk_reduce_kernel,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      chunk_reduce_kernel<<<blocks, 256, sm, st>>>(src, cnt, D, ch, dst);
      CUDA_TRY(ctx, cudaGetLastError());
      ++ctx->launches;
      cnt = blocks;
    } else {
      pair_level_kernel<<<grid_for((int64_t)nxt * dd, 256), 256, 0, st>>>(src, cnt, D, dst);
      CUDA_TRY(ctx, cudaGetLastError());
      ++ctx->launches;
      cnt = nxt;
    }
    src = dst;
    which ^= 1;
  }
  *result = src;
  return SP_OK;
}

// ---- family D8: one warp per lane, m8n8k4 DMMA (kernels_d8.cuh)
constexpr int D8_WPC = 8;  // lanes (warps) per CTA
// 3 planes for the 3-multiplication form, 2 otherwise (3 CTAs/SM for the latter)
constexpr size_t d8_smem(int alg) {
  return ((size_t)D8_WPC * d8_slot(alg == D8_PS3 ? 3 : 2) + 2 * 64 * D8_TSM) * sizeof(double);
}

template <int ALG, int SC = 0, int RC = 0>
int d8_prepare_one(sp_ctx* ctx) {
  CUDA_TRY(ctx, cudaFuncSetAttribute(lane_d8_kernel<D8_WPC, ALG, SC, RC>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)d8_smem(ALG)));
  return SP_OK;
}

template <int ALG>
int d8_prepare_ps(sp_ctx* ctx) {
  int rc = d8_prepare_one<ALG>(ctx);
  if (!rc) rc = d8_prepare_one<ALG, 3, 5>(ctx);
  if (!rc) rc = d8_prepare_one<ALG, 4, 4>(ctx);
  if (!rc) rc = d8_prepare_one<ALG, 2, 4>(ctx);
  return rc;
}

int d8_prepare(sp_ctx* ctx) {
  int rc = d8_prepare_one<D8_CLENSHAW>(ctx);
  if (!rc) rc = d8_prepare_ps<D8_PS>(ctx);
  if (!rc) rc = d8_prepare_ps<D8_PS3>(ctx);
  return rc;
}

// one launch of a D8 kernel variant: lanes = its resident capacity (one wave)
template <int ALG, int SC = 0, int RC = 0>
int d8_run(sp_ctx* ctx, const PSJob& pj, double2* prefix_out, cudaStream_t st, int* lanes_out) {
  auto kern = lane_d8_kernel<D8_WPC, ALG, SC, RC>;
  const size_t sm = d8_smem(ALG);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 32 * D8_WPC, sm);
  occ = std::max(occ, 1);
  const int lanes = (int)std::max<int64_t>(
      1, std::min<int64_t>((int64_t)ctx->sms * occ * D8_WPC, pj.base.n_slices));
  int rc = ensure(ctx, ctx->lanes, (size_t)lanes * 64 * sizeof(double2));
  if (rc) return rc;
  const int grid = (lanes + D8_WPC - 1) / D8_WPC;
  if (ctx->prof) CUDA_TRY(ctx, cudaEventRecord(ctx->ev0, st));
  kern<<<grid, 32 * D8_WPC, sm, st>>>(pj, (const double2*)ctx->terms.p, lanes,
                                      (double2*)ctx->lanes.p, prefix_out);
  CUDA_TRY(ctx, cudaGetLastError());
  if (ctx->prof) CUDA_TRY(ctx, cudaEventRecord(ctx->ev1, st));
  *lanes_out = lanes;
  return SP_OK;
}

// PS forms: the (s, r) split compiled in where it is one of the common ones
template <int ALG>
int d8_run_ps(sp_ctx* ctx, const PSJob& pj, double2* prefix_out, cudaStream_t st, int* lanes) {
  if (pj.s == 3 && pj.r == 5) return d8_run<ALG, 3, 5>(ctx, pj, prefix_out, st, lanes);
  if (pj.s == 4 && pj.r == 4) return d8_run<ALG, 4, 4>(ctx, pj, prefix_out, st, lanes);
  if (pj.s == 2 && pj.r == 4) return d8_run<ALG, 2, 4>(ctx, pj, prefix_out, st, lanes);
  return d8_run<ALG>(ctx, pj, prefix_out, st, lanes);
}

int d8_launch(sp_ctx* ctx, const SliceJob& job, double2* prefix_out, cudaStream_t st,
              const double2** prods, int* count) {
  const int ps_s = (ctx->algo == ALGO_CLENSHAW) ? 0
                   : (ctx->algo == ALGO_PS || ctx->algo == ALGO_PS3)
                         ? std::max(2, ps_choose(job.m) ? ps_choose(job.m) : 2)
                         : ps_choose(job.m);
  const int alg = ps_s == 0 ? D8_CLENSHAW : (ctx->algo == ALGO_PS3 ? D8_PS3 : D8_PS);
  PSJob pj;
  std::memset(&pj, 0, sizeof(pj));
  pj.base = job;
  if (ps_s > 0) {
    pj.s = ps_s;
    ps_coefficients(job.coef, job.m, ps_s, pj.alpha, &pj.r);
    pj.alt = ps_alpha_alt(pj.alpha, pj.r * pj.s);
  }
  int lanes = 0;
  const int rc = alg == D8_CLENSHAW ? d8_run<D8_CLENSHAW>(ctx, pj, prefix_out, st, &lanes)
                 : alg == D8_PS     ? d8_run_ps<D8_PS>(ctx, pj, prefix_out, st, &lanes)
                                    : d8_run_ps<D8_PS3>(ctx, pj, prefix_out, st, &lanes);
  if (rc) return rc;
  ++ctx->launches;
  ctx->last_algo = alg == D8_CLENSHAW ? ALGO_CLENSHAW : alg == D8_PS ? ALGO_PS : ALGO_PS3;
  ctx->last_gemms = ps_s == 0 ? job.m : ps_cost(job.m, ps_s);
  *prods = (const double2*)ctx->lanes.p;
  *count = lanes;
  ctx->last_lanes = lanes;
  return SP_OK;
}

// the device-resident and cumulative entry points of a multi-device context
// run on its first device
sp_ctx* primary(sp_ctx* ctx) { return ctx->kids.empty() ? ctx : ctx->kids[0]; }

// complex64 contexts of the plain families (d <= 8) run in complex64
// arithmetic on the FP32 pipe (kernels_f32.cuh); d >= 9 complex64 contexts
// use the FP64 tensor-core kernels and round
bool f32_path(const sp_ctx* ctx) { return ctx->bits == 32 && plain_family(ctx->fam); }

template <int D>
int f32_run(sp_ctx* ctx, const SliceJob& job, double2* prefix_out, cudaStream_t st,
            int* lanes_out) {
  const size_t smem = f32_smem_bytes<D>(job.n_terms);
  CUDA_TRY(ctx, cudaFuncSetAttribute(lane_f32_kernel<D>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, lane_f32_kernel<D>, F32_THREADS, smem);
  occ = std::max(occ, 1);
  constexpr int LPC = F32_THREADS / D;
  // one wave of resident lanes, at least 16 slices per lane
  const int64_t cap = (int64_t)ctx->sms * occ * LPC;
  const int64_t want = std::max<int64_t>(1024, (job.n_slices + 15) / 16);
  const int lanes = (int)std::max<int64_t>(1, std::min<int64_t>(std::min(cap, want),
                                                                 job.n_slices));
  int rc = ensure(ctx, ctx->lanes, (size_t)lanes * D * D * sizeof(double2));
  if (rc) return rc;
  const int grid = (lanes + LPC - 1) / LPC;
  if (ctx->prof) CUDA_TRY(ctx, cudaEventRecord(ctx->ev0, st));
  lane_f32_kernel<D><<<grid, F32_THREADS, smem, st>>>(job, (const double2*)ctx->terms.p, lanes,
                                                      (double2*)ctx->lanes.p, prefix_out);
  CUDA_TRY(ctx, cudaGetLastError());
  if (ctx->prof) CUDA_TRY(ctx, cudaEventRecord(ctx->ev1, st));
  *lanes_out = lanes;
  return SP_OK;
}

// D = 2: one thread per lane, everything in registers (lane_f32_reg2_kernel)
int f32_run_reg2(sp_ctx* ctx, const SliceJob& job, double2* prefix_out, cudaStream_t st,
                 int* lanes_out) {
  const size_t smem = (size_t)job.n_terms * 4 * sizeof(float2);
  if (smem > 48 * 1024)
    CUDA_TRY(ctx, cudaFuncSetAttribute(lane_f32_reg2_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, lane_f32_reg2_kernel, F32_THREADS, smem);
  occ = std::max(occ, 1);
  // one wave of resident lanes, at least 16 slices per lane
  const int64_t cap = (int64_t)ctx->sms * occ * F32_THREADS;
  const int64_t want = std::max<int64_t>(1024, (job.n_slices + 15) / 16);
  const int lanes = (int)std::max<int64_t>(1, std::min<int64_t>(std::min(cap, want),
                                                                 job.n_slices));
  int rc = ensure(ctx, ctx->lanes, (size_t)lanes * 4 * sizeof(double2));
  if (rc) return rc;
  const int grid = (lanes + F32_THREADS - 1) / F32_THREADS;
  if (ctx->prof) CUDA_TRY(ctx, cudaEventRecord(ctx->ev0, st));
  lane_f32_reg2_kernel<<<grid, F32_THREADS, smem, st>>>(job, (const double2*)ctx->terms.p, lanes,
                                                         (double2*)ctx->lanes.p, prefix_out);
  CUDA_TRY(ctx, cudaGetLastError());
  if (ctx->prof) CUDA_TRY(ctx, cudaEventRecord(ctx->ev1, st));
  *lanes_out = lanes;
  return SP_OK;
}

int f32_launch(sp_ctx* ctx, const SliceJob& job, double2* prefix_out, cudaStream_t st,
               const double2** prods, int* count) {
  int lanes = 0;
  // D = 2: register lanes from 2^19 slices (1e7: 309 vs 380 us); below,
  // the two-thread lanes give twice the threads for the same lane count
  // (1e5: 25 vs 34 us).  SP_F32_REG2=0 / 1 forces either (A/B, tests)
  static const int reg2_env = [] {
    const char* e = getenv("SP_F32_REG2");
    return e ? (e[0] == '0' ? 0 : 1) : -1;
  }();
  const bool reg2 = reg2_env >= 0 ? reg2_env == 1 : job.n_slices >= (1 << 19);
  const int rc = ctx->D == 2 ? (reg2 ? f32_run_reg2(ctx, job, prefix_out, st, &lanes)
                                     : f32_run<2>(ctx, job, prefix_out, st, &lanes))
                 : ctx->D == 4 ? f32_run<4>(ctx, job, prefix_out, st, &lanes)
                               : f32_run<8>(ctx, job, prefix_out, st, &lanes);
  if (rc) return rc;
  ++ctx->launches;
  ctx->last_algo = ALGO_F32;
  ctx->last_gemms = job.m + 1;
  *prods = (const double2*)ctx->lanes.p;
  *count = lanes;
  ctx->last_lanes = lanes;
  return SP_OK;
}

// su(2) family: d = 2 traceless Hermitian terms, symmetric plan with
// alternating coefficients (phase 1), fp64, pairwise, one fused launch
// (kernels_su2.cuh); u(2) systems (Hermitian terms with a trace part) on the
// same lanes with complex Clenshaw pairs and 2 x 2 complex products (any
// coefficients, phase 1).  SP_SU2=0 / SP_U2=0 in the environment disable
// them (A/B timing).
bool su2_applies(const sp_ctx* ctx, const SliceJob& job) {
  static const int enabled = [] {
    const char* e = getenv("SP_SU2");
    return (e && e[0] == '0') ? 0 : 1;
  }();
  static const int u2_enabled = [] {
    const char* e = getenv("SP_U2");
    return (e && e[0] == '0') ? 0 : 1;
  }();
  if (!enabled) return false;
  const bool su2 = ctx->su2_terms && job.coef_alt;
  // u(2): complex128 (complex64 keeps the reference's float32 sequence of
  // lane_f32_kernel<2>: the u(2) float32 pairs land 1-3x outside the
  // complex64 gate)
  const bool u2 = u2_enabled && ctx->u2_terms && ctx->bits == 64 && job.m <= SP_MAX_ORDER;
  if (!su2 && !u2) return false;
  if (job.mode > SP_MODE_MAGNUS) return false;  // Gauss-Legendre: general d = 2 kernel
  if (!(job.phase[0] == 1.0 && job.phase[1] == 0.0)) return false;
  if (job.n_ctrl % 2 == 0 && ((uintptr_t)job.amps & 15u)) return false;  // vector row loads
  return true;
}

int su2_launch(sp_ctx* ctx, const SliceJob& job, cudaStream_t st, void* fused_out,
               const double2** prods, int* count, double2* prefix_out = nullptr) {
  Su2Job sj;
  std::memset(&sj, 0, sizeof(sj));
  sj.amps = job.amps;
  sj.n_slices = job.n_slices;
  sj.n_ctrl = job.n_ctrl;
  sj.mode = job.mode;
  sj.m = job.m;
  sj.dt6 = job.dt / 6.0;
  // u(2): the terms carry a trace part (su(2) terms are traceless, and then
  // (H00 - H11) / 2 is H00 exactly)
  sj.u2 = ctx->su2_terms ? 0 : 1;
  for (int t = 0; t < ctx->n_terms; ++t) {
    const double* h = &ctx->terms_host[(size_t)t * 8];  // 2 x 2 complex128, row-major
    sj.ta[t] = job.xs * (0.5 * (h[0] + h[6]));          // (H00 + H11) / 2
    sj.tz[t][0] = job.xs * (0.5 * (h[0] - h[6]));       // (H00 - H11) / 2
    sj.tz[t][1] = job.xs * h[2];                        // Re H01
    sj.tz[t][2] = job.xs * h[3];                        // Im H01
  }
  for (int k = 0; k <= job.m; ++k) {
    sj.cr[k] = job.coef[2 * k + (k & 1)];
    sj.cz[2 * k] = job.coef[2 * k];
    sj.cz[2 * k + 1] = job.coef[2 * k + 1];
  }
  sj.viol = job.viol;
  sj.viol_epoch = job.viol_epoch;
  sj.out = fused_out;
  sj.to_fp32 = out32(ctx) ? 1 : 0;
  sj.arith32 = ctx->bits == 32 ? 1 : 0;
  // lanes: >= SPT slices each (tree and tail amortised), one CTA per SM
  static const int spt = [] {
    const char* e = getenv("SP_SU2_SPT");
    return e ? std::max(1, atoi(e)) : 4;
  }();
  static const int tpb_env = [] {
    const char* e = getenv("SP_SU2_TPB");
    return e ? atoi(e) : 0;
  }();
  int tpb_max = su2_max_block(sj);
  if (tpb_env >= 32) tpb_max = std::min(tpb_max, tpb_env & ~31);
  // (lane mode: >= 16 slices per lane, the two-level scan of the lane
  // products sizes its groups for that)
  const int spt_eff = fused_out ? spt : std::max(spt, 16);
  const int64_t want = std::max<int64_t>(1, (job.n_slices + spt_eff - 1) / spt_eff);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ctx->sms, (want + 31) / 32));
  const int64_t per = (want + grid - 1) / grid;
  const int block = (int)std::min<int64_t>(tpb_max, ((per + 31) / 32) * 32);
  const bool lane_mode = fused_out == nullptr;
  int rc = ensure(ctx, ctx->lanes, lane_mode ? (size_t)grid * block * 4 * sizeof(double2)
                                             : (size_t)grid * 8 * sizeof(double));
  if (rc) return rc;
  if (lane_mode) {  // lane products, per-slice running products, initial products
    sj.lane_out = ctx->lanes.p;
    sj.prefix_out = prefix_out;
    sj.vinit = job.vinit;
  }
  sj.cta_out = ctx->lanes.p;
  if (!ctx->tailctr.p) {
    rc = ensure(ctx, ctx->tailctr, sizeof(unsigned));
    if (rc) return rc;
    CUDA_TRY(ctx, cudaMemsetAsync(ctx->tailctr.p, 0, sizeof(unsigned), st));
  }
  sj.ctr = (unsigned*)ctx->tailctr.p;
  // tools only: phase timestamps printed to stderr (SP_SU2_PROF=1)
  static const bool phase_prof = getenv("SP_SU2_PROF") && getenv("SP_SU2_PROF")[0] == '1';
  static unsigned long long* d_prof = nullptr;
  if (phase_prof) {
    if (!d_prof) CUDA_TRY(ctx, cudaMalloc(&d_prof, 16 * sizeof(unsigned long long)));
    std::vector<unsigned long long> init(16);
    for (int i = 0; i < 16; ++i) init[i] = (i & 1) ? 0ull : ~0ull;
    CUDA_TRY(ctx, cudaMemcpyAsync(d_prof, init.data(), 16 * 8, cudaMemcpyHostToDevice, st));
    sj.prof = d_prof;
  }
  if (ctx->prof) CUDA_TRY(ctx, cudaEventRecord(ctx->ev0, st));
  CUDA_TRY(ctx, su2_run(sj, grid, block, st));
  if (ctx->prof) CUDA_TRY(ctx, cudaEventRecord(ctx->ev1, st));
  if (phase_prof) {
    unsigned long long h[16];
    CUDA_TRY(ctx, cudaMemcpyAsync(h, d_prof, sizeof(h), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(ctx, cudaStreamSynchronize(st));
    fprintf(stderr, "[su2 phases ns] n=%lld grid=%d block=%d", (long long)job.n_slices, grid,
            block);
    for (int k = 0; k < 6; ++k)
      if (h[2 * k] != ~0ull)
        fprintf(stderr, " p%d=[%lld,%lld]", k, (long long)(h[2 * k] - h[0]),
                (long long)(h[2 * k + 1] - h[0]));
    fprintf(stderr, "\n");
  }
  ++ctx->launches;
  ctx->last_algo = sj.u2 ? (ctx->bits == 32 ? ALGO_U2_F32 : ALGO_U2)
                         : (ctx->bits == 32 ? ALGO_SU2_F32 : ALGO_SU2);
  ctx->last_gemms = job.m;
  ctx->last_lanes = grid * block;
  *prods = (const double2*)ctx->lanes.p;
  *count = lane_mode ? grid * block : grid;
  return SP_OK;
}

// Run the lane pass.  Returns the lane products (lane_count of them) on the
// device, or (small families, pairwise) the per-CTA products.
int run_lanes(sp_ctx* ctx, const SliceJob& job, bool cta_reduce, double2* prefix_out,
              cudaStream_t st, const double2** prods, int* count, void* fused_out = nullptr) {
  const int64_t n = job.n_slices;
  const int D = ctx->D;
  const size_t dd = (size_t)D * D;
  int lanes = 1;
  if (ctx->fam == FAM_S2 && fused_out && cta_reduce && !prefix_out && !job.vinit &&
      su2_applies(ctx, job))
    return su2_launch(ctx, job, st, fused_out, prods, count);
  // lane mode (sequential reduction, the d = 2 two-pass equiprop_all): the
  // su(2) lanes write lane products / running products in the plain layout
  if (ctx->fam == FAM_S2 && !cta_reduce && ctx->bits == 64 && su2_applies(ctx, job))
    return su2_launch(ctx, job, st, nullptr, prods, count, prefix_out);
  if (f32_path(ctx)) return f32_launch(ctx, job, prefix_out, st, prods, count);
  if (ctx->fam == FAM_T8) return d8_launch(ctx, job, prefix_out, st, prods, count);
  if (ctx->fam == FAM_S2 || ctx->fam == FAM_S4) {
    const int tpl = (ctx->fam == FAM_S2) ? 1 : 4;
    // pairwise: at least 4 slices per lane (short CTA tree and tail for the
    // latency-bound small n), at most one full wave of resident threads (no
    // second partial wave); sequential / cumulative: at least 16 slices per
    // lane (the two-level scan of the lane products)
    int occ = 0;
    if (ctx->fam == FAM_S2)
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, lane_small_kernel<2, 1>, 256, 0);
    else
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, lane_small_kernel<4, 4>, 256, 0);
    occ = std::max(occ, 1);
    int64_t cap = (int64_t)ctx->sms * occ * 256 / tpl;
    int64_t want = cta_reduce ? std::max<int64_t>((int64_t)ctx->sms * 256 / tpl, (n + 3) / 4)
                              : std::max<int64_t>(1024, (n + 15) / 16);
    lanes = (int)std::max<int64_t>(1, std::min<int64_t>(std::min(cap, want), n));
    const int blocks = (int)(((int64_t)lanes * tpl + 255) / 256);
    int rc = ensure(ctx, ctx->lanes, (size_t)(cta_reduce ? blocks : lanes) * dd * sizeof(double2));
    if (rc) return rc;
    double2* lane_out = (double2*)ctx->lanes.p;
    double2* cta_out = cta_reduce ? lane_out : nullptr;
    SmallTail tail{nullptr, nullptr, ctx->dim, out32(ctx)};
    if (fused_out) {
      // arrival counter: zeroed once at allocation, reset by the last CTA
      if (!ctx->tailctr.p) {
        rc = ensure(ctx, ctx->tailctr, sizeof(unsigned));
        if (rc) return rc;
        CUDA_TRY(ctx, cudaMemsetAsync(ctx->tailctr.p, 0, sizeof(unsigned), st));
      }
      tail.ctr = (unsigned*)ctx->tailctr.p;
      tail.out = fused_out;
    }
    if (ctx->prof) CUDA_TRY(ctx, cudaEventRecord(ctx->ev0, st));
    const double2* tp = (const double2*)ctx->terms.p;
    if (ctx->fam == FAM_S2) {
      // the common series orders compiled in (qubit fine steps 3, fp32 7,
      // beta = 0.5 fp64 13, magnus 15)
      // and, for two controls in midpoint mode (the driven qubit), the
      // control count of the fast path
      // (its rows are read as 16-byte vectors: aligned tables only)
      const bool two = job.n_ctrl == 2 && job.mode == SP_MODE_MIDPOINT &&
                       ((uintptr_t)job.amps & 15u) == 0;
#define SP_S2(MCV)                                                                          \
  (two ? lane_small_kernel<2, 1, MCV, 2><<<blocks, 256, 0, st>>>(job, tp, lanes, lane_out,  \
                                                                 cta_out, prefix_out, tail) \
       : lane_small_kernel<2, 1, MCV><<<blocks, 256, 0, st>>>(job, tp, lanes, lane_out,     \
                                                              cta_out, prefix_out, tail))
      switch (job.m) {
        case 3: SP_S2(3); break;
        case 7: SP_S2(7); break;
        case 13: SP_S2(13); break;
        case 15: SP_S2(15); break;
        default: SP_S2(0);
      }
#undef SP_S2
    }
    else {
      // d = 3, 4: the series order compiled in for every order of the plan
      // grid (odd 3..25; the Clenshaw loop unrolls, no spills) with the
      // alternating-coefficient products when the plan has them
#define SP_S4(MCV)                                                                            \
  lane_small_kernel<4, 4, MCV, 0, true><<<blocks, 256, 0, st>>>(job, tp, lanes, lane_out,   \
                                                                cta_out, prefix_out, tail)
      switch (job.coef_alt ? job.m : 0) {
        case 3: SP_S4(3); break;
        case 5: SP_S4(5); break;
        case 7: SP_S4(7); break;
        case 9: SP_S4(9); break;
        case 11: SP_S4(11); break;
        case 13: SP_S4(13); break;
        case 15: SP_S4(15); break;
        case 17: SP_S4(17); break;
        case 19: SP_S4(19); break;
        case 21: SP_S4(21); break;
        case 23: SP_S4(23); break;
        case 25: SP_S4(25); break;
        default:
          lane_small_kernel<4, 4><<<blocks, 256, 0, st>>>(job, tp, lanes, lane_out, cta_out,
                                                          prefix_out, tail);
      }
#undef SP_S4
    }
    CUDA_TRY(ctx, cudaGetLastError());
    if (ctx->prof) CUDA_TRY(ctx, cudaEventRecord(ctx->ev1, st));
    ++ctx->launches;
    ctx->last_algo = ALGO_CLENSHAW;
    ctx->last_gemms = job.m;
    *prods = lane_out;
    *count = cta_reduce ? blocks : lanes;
    ctx->last_lanes = lanes;
    return SP_OK;
  }
  const int ps_s = (ctx->algo == ALGO_CLENSHAW) ? 0
                   : (ctx->algo == ALGO_PS || ctx->algo == ALGO_PS3)
                         ? std::max(2, ps_choose(job.m) ? ps_choose(job.m) : 2)
                         : ps_choose(job.m);
  // auto: the 3-multiplication/TMEM form where it measured faster (the
  // group families, D >= 128: 165% vs 149% of canonical FP64 peak at D128;
  // D64 with 8 warps of 16 x 16: +2% for fp64 plans, -4% for the fp32 m = 7
  // plan); for the smem-resident D <= 32 its 1.5x operands cost occupancy
  // and the 4-product PS wins
  // (D = 64 as one CTA per lane: PS3 measured 18% faster than the group-of-2
  // form for fp64 and 17% faster than the 4-product PS for the fp32 plan)
  const bool three_m =
      ps_s > 0 && (ctx->algo == ALGO_PS3 ||
                   (ctx->algo == ALGO_AUTO &&
                    (ctx->D >= 128 ||
                     (ctx->D == 64 && (ctx->bits == 64 || d64_single())))));
  if (ps_s > 0 && three_m) {
    PSJob pj;
    std::memset(&pj, 0, sizeof(pj));
    pj.base = job;
    pj.s = ps_s;
    ps_coefficients(job.coef, job.m, ps_s, pj.alpha, &pj.r);
    pj.alt = ps_alpha_alt(pj.alpha, pj.r * pj.s);
    switch (ctx->fam) {
      case FAM_T16: lanes = ps3_lanes<P3_16>(ctx, n); break;
      case FAM_T32: lanes = ps3_lanes<P3_32>(ctx, n); break;
      case FAM_T64:
        lanes = d64_single() ? ps3_lanes<P3_64s>(ctx, n) : ps3_lanes<P3_64>(ctx, n);
        break;
      case FAM_T128: lanes = ps3_lanes<P3_128>(ctx, n); break;
      case FAM_T256: lanes = ps3_lanes<P3_256>(ctx, n); break;
      case FAM_T512: lanes = ps3_lanes<P3_512>(ctx, n); break;
    }
    int rc = ensure(ctx, ctx->lanes, (size_t)lanes * dd * sizeof(double2));
    if (rc) return rc;
    double2* lane_out = (double2*)ctx->lanes.p;
    switch (ctx->fam) {
      case FAM_T16: rc = ps3_launch<P3_16>(ctx, pj, lanes, lane_out, prefix_out, st); break;
      case FAM_T32: rc = ps3_launch<P3_32>(ctx, pj, lanes, lane_out, prefix_out, st); break;
      case FAM_T64:
        rc = d64_single() ? ps3_launch<P3_64s>(ctx, pj, lanes, lane_out, prefix_out, st)
                          : ps3_launch<P3_64>(ctx, pj, lanes, lane_out, prefix_out, st);
        break;
      case FAM_T128: rc = ps3_launch<P3_128>(ctx, pj, lanes, lane_out, prefix_out, st); break;
      case FAM_T256: rc = ps3_launch<P3_256>(ctx, pj, lanes, lane_out, prefix_out, st); break;
      case FAM_T512: rc = ps3_launch<P3_512>(ctx, pj, lanes, lane_out, prefix_out, st); break;
    }
    if (rc) return rc;
    ctx->last_algo = ALGO_PS3;
    ctx->last_gemms = ps_cost(job.m, ps_s);
    *prods = lane_out;
    *count = lanes;
    ctx->last_lanes = lanes;
    return SP_OK;
  }
  if (ps_s > 0) {
    PSJob pj;
    std::memset(&pj, 0, sizeof(pj));
    pj.base = job;
    pj.s = ps_s;
    ps_coefficients(job.coef, job.m, ps_s, pj.alpha, &pj.r);
    pj.alt = ps_alpha_alt(pj.alpha, pj.r * pj.s);
    switch (ctx->fam) {
      case FAM_T16: lanes = ps_lanes<PS16>(ctx, n); break;
      case FAM_T32: lanes = ps_lanes<PS32>(ctx, n); break;
      case FAM_T64: lanes = ps_lanes<PS64>(ctx, n); break;
      case FAM_T128: lanes = ps_lanes<PS128>(ctx, n); break;
      case FAM_T256: lanes = ps_lanes<PS256>(ctx, n); break;
      case FAM_T512: lanes = ps_lanes<PS512>(ctx, n); break;
    }
    int rc = ensure(ctx, ctx->lanes, (size_t)lanes * dd * sizeof(double2));
    if (rc) return rc;
    double2* lane_out = (double2*)ctx->lanes.p;
    switch (ctx->fam) {
      case FAM_T16: rc = ps_launch<PS16>(ctx, pj, lanes, lane_out, prefix_out, st); break;
      case FAM_T32: rc = ps_launch<PS32>(ctx, pj, lanes, lane_out, prefix_out, st); break;
      case FAM_T64: rc = ps_launch<PS64>(ctx, pj, lanes, lane_out, prefix_out, st); break;
      case FAM_T128: rc = ps_launch<PS128>(ctx, pj, lanes, lane_out, prefix_out, st); break;
      case FAM_T256: rc = ps_launch<PS256>(ctx, pj, lanes, lane_out, prefix_out, st); break;
      case FAM_T512: rc = ps_launch<PS512>(ctx, pj, lanes, lane_out, prefix_out, st); break;
    }
    if (rc) return rc;
    ctx->last_algo = ALGO_PS;
    ctx->last_gemms = ps_cost(job.m, ps_s);
    *prods = lane_out;
    *count = lanes;
    ctx->last_lanes = lanes;
    return SP_OK;
  }
  ctx->last_algo = ALGO_CLENSHAW;
  ctx->last_gemms = job.m;
  switch (ctx->fam) {
    case FAM_T16: lanes = tc_lanes<Cfg16>(ctx, n); break;
    case FAM_T32: lanes = tc_lanes<Cfg32>(ctx, n); break;
    case FAM_T64: lanes = tc_lanes<Cfg64>(ctx, n); break;
    case FAM_T128: lanes = tc_lanes<Cfg128>(ctx, n); break;
    case FAM_T256: lanes = tc_lanes<Cfg256>(ctx, n); break;
    case FAM_T512: lanes = tc_lanes<Cfg512>(ctx, n); break;
  }
  int rc = ensure(ctx, ctx->lanes, (size_t)lanes * dd * sizeof(double2));
  if (rc) return rc;
  double2* lane_out = (double2*)ctx->lanes.p;
  switch (ctx->fam) {
    case FAM_T16: rc = tc_launch<Cfg16>(ctx, job, lanes, lane_out, prefix_out, st); break;
    case FAM_T32: rc = tc_launch<Cfg32>(ctx, job, lanes, lane_out, prefix_out, st); break;
    case FAM_T64: rc = tc_launch<Cfg64>(ctx, job, lanes, lane_out, prefix_out, st); break;
    case FAM_T128: rc = tc_launch<Cfg128>(ctx, job, lanes, lane_out, prefix_out, st); break;
    case FAM_T256: rc = tc_launch<Cfg256>(ctx, job, lanes, lane_out, prefix_out, st); break;
    case FAM_T512: rc = tc_launch<Cfg512>(ctx, job, lanes, lane_out, prefix_out, st); break;
  }
  if (rc) return rc;
  *prods = lane_out;
  *count = lanes;
  ctx->last_lanes = lanes;
  return SP_OK;
}

int check_loaded(sp_ctx* ctx) {
  if (!ctx) return fail(nullptr, SP_E_STATE_MACHINE, "null context");
  if (!ctx->loaded)
    return fail(ctx, SP_E_STATE_MACHINE, "no Hamiltonian loaded; call set_hamiltonian first");
  return SP_OK;
}

int build_job(sp_ctx* ctx, const double* d_amps, int64_t pts, int n_ctrl, double dt,
              const sp_plan* plan, SliceJob* job) {
  if (n_ctrl != ctx->n_ctrl)
    return fail(ctx, SP_E_SHAPE, "amplitude table has %d controls, system has %d", n_ctrl,
                ctx->n_ctrl);
  if (!(dt > 0.0)) return fail(ctx, SP_E_CONFIG, "time step must be > 0, got %g", dt);
  if (!plan) return fail(ctx, SP_E_CONFIG, "missing plan");
  if (plan->m_max < 3 || plan->m_max > SP_MAX_ORDER || plan->m_max % 2 == 0)
    return fail(ctx, SP_E_CONFIG, "plan order %d not on the odd grid 3..25", plan->m_max);
  if (plan->alpha != -plan->beta)
    return fail(ctx, SP_E_CONFIG, "equiprop plans are symmetric (alpha = -beta)");
  int code;
  const int64_t n = slice_count_for(ctx->mode, pts, &code);
  if (code)
    return fail(ctx, code, "%s, got %lld", parity_message(ctx->mode), (long long)pts);
  std::memset(job, 0, sizeof(*job));
  job->amps = d_amps;
  job->pts = pts;
  job->n_ctrl = n_ctrl;
  job->n_terms = ctx->n_terms;
  job->mode = ctx->mode;
  job->dt = dt;
  const double scale = (ctx->mode == SP_MODE_MIDPOINT) ? dt : 2.0 * dt;
  const double span = plan->beta - plan->alpha;
  job->xs = (span == 0.0) ? 0.0 : 2.0 * scale * (2.0 / span);
  job->scale = scale;
  job->xspan = (span == 0.0) ? 0.0 : 2.0 / span;
  job->gl = std::sqrt(3.0) * dt / 6.0;
  job->m = plan->m_max;
  std::memcpy(job->coef, plan->coeffs, sizeof(job->coef));
  job->phase[0] = plan->phase[0];
  job->phase[1] = plan->phase[1];
  job->n_slices = n;
  job->herm_exact = ctx->herm_exact ? 1 : 0;
  job->coef_alt = 1;
  for (int k = 0; k <= job->m; ++k)
    if (job->coef[2 * k + ((k & 1) ? 0 : 1)] != 0.0) job->coef_alt = 0;
  return SP_OK;
}

// amplitude validation fused into the lane kernels: reset the device flag
// (fused: a single-launch call whose last CTA rotates the slots, no memset)
int arm_validation(sp_ctx* ctx, SliceJob* job, cudaStream_t st, bool fused = false) {
  const bool fresh = ctx->viol.p == nullptr;
  int rc = ensure(ctx, ctx->viol, 4 * sizeof(unsigned long long));
  if (rc) return rc;
  if (fresh || !fused)
    CUDA_TRY(ctx, cudaMemsetAsync(ctx->viol.p, 0xFF,
                                  (fresh ? 4 : 3) * sizeof(unsigned long long), st));
  job->viol = (unsigned long long*)ctx->viol.p;
  job->viol_epoch = fused ? 1 : 0;
  ctx->viol_stream = st;
  ctx->viol_pts = job->pts;
  return SP_OK;
}

// after the stream work: SP_E_AMPLITUDE_BOUND with the reference's message
// (hamiltonian.py:165-174) if any sample was outside [-1, 1]
// (fetched: the slots were copied into ctx->viol_host on the call's stream and
// that stream has been synchronised)
int read_violation(sp_ctx* ctx, const double* host_amps, int64_t* index_out,
                   bool fetched = false) {
  unsigned long long v = ~0ull;
  if (ctx->viol.p) {
    unsigned long long slots[3];
    if (fetched) {
      for (int i = 0; i < 3; ++i) slots[i] = ctx->viol_host[i];
    } else {
      CUDA_TRY(ctx, cudaStreamSynchronize(ctx->viol_stream));
      CUDA_TRY(ctx, cudaMemcpy(slots, ctx->viol.p, sizeof(slots), cudaMemcpyDeviceToHost));
    }
    v = std::min(slots[0], std::min(slots[1], slots[2]));
  }
  if (index_out) *index_out = (v == ~0ull) ? -1 : (int64_t)v;
  if (v == ~0ull) return SP_OK;
  const int N = std::max(1, ctx->n_ctrl);
  const long long k = (long long)(v / N), i = (long long)(v % N);
  if (host_amps)
    return fail(ctx, SP_E_AMPLITUDE_BOUND,
                "control amplitude %.17g at sample %lld, control %lld lies outside [-1, 1]",
                host_amps[v], k, i);
  return fail(ctx, SP_E_AMPLITUDE_BOUND,
              "control amplitude at sample %lld, control %lld lies outside [-1, 1]", k, i);
}

// queue the copy of the violation slots into page-locked host memory
int fetch_violation(sp_ctx* ctx, cudaStream_t st) {
  if (!ctx->viol.p) return SP_OK;
  if (!ctx->viol_host) CUDA_TRY(ctx, cudaMallocHost((void**)&ctx->viol_host, 4 * sizeof(unsigned long long)));
  CUDA_TRY(ctx, cudaMemcpyAsync(ctx->viol_host, ctx->viol.p, 3 * sizeof(unsigned long long),
                                cudaMemcpyDeviceToHost, st));
  return SP_OK;
}

int prepare_device(sp_ctx* ctx) {
  int rc = device_init(ctx);
  if (rc) return rc;
  CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  if (!ctx->terms_uploaded) {
    rc = upload_terms(ctx);
    if (rc) return rc;
  }
  return SP_OK;
}

double executed_flops(const sp_ctx* ctx, int64_t n, int m) {
  const double D = ctx->D;
  // complex64 lane kernel (FP32): per slice, D threads each run m
  // matrix-vector products of the Clenshaw recurrence (the first of the
  // reference's m + 1 multiplies zero and is skipped), one of V <- U V, and
  // the assembly of T terms
  if (ctx->last_algo == ALGO_F32)
    return (double)n * (8.0 * D * D * D * (m + 1) + 4.0 * D * D * (ctx->n_terms - 1));
  // register families: FP64 flops per slice (DFMA = 2, DADD / DMUL = 1)
  // calibrated on the SASS instruction counts of ncu
  // (smsp__sass_thread_inst_executed_op_{dfma,dadd,dmul}_pred_on.sum,
  // tools/ncu_small_flops.py, profiles/r02_ncu_small_flops.md), exact on
  // every calibration point:
  //   d = 2, real Cayley-Hamilton pairs (bitwise Hermitian terms, midpoint,
  //          <= 2 controls): 125 + 16 m, +14 when m is not compiled in
  //          (3, 7, 13, 15)
  //   d = 2, complex pairs (other modes / more controls): 137 + 28.7 m + 16 T,
  //          +40 for the three-point modes (within 3% of every point)
  //   d = 3, 4: 10.3 + 576 m + 64 T
  if (ctx->last_algo == ALGO_SU2 || ctx->last_algo == ALGO_SU2_F32) {
    // su(2) quaternion kernel (flops, DFMA = 2): 3 FMA per control term
    // (assembly), 5 for zeta2, 4 per Clenshaw step after the peeled one
    // (+2 at j = 0), 3 MUL for U, 28 for V <- U V; three-point control
    // weights 4 each (the /6 counted as one), magnus commutator weights
    // 2 (drift) / 4 (cross) each — calibrated in profiles/r02_ncu_su2.md
    const int N = ctx->n_ctrl, T = ctx->n_terms;
    double w = 0.0;
    if (ctx->mode != SP_MODE_MIDPOINT) w += 4.0 * N;
    if (ctx->mode == SP_MODE_MAGNUS) w += 2.0 * N + 4.0 * (N * (N - 1) / 2);
    const double f = 6.0 * (T - 1) + 5.0 + 4.0 * (m - 1) + 2.0 + 3.0 + 28.0 + w;
    return (double)n * f;
  }
  if (ctx->last_algo == ALGO_U2 || ctx->last_algo == ALGO_U2_F32) {
    // u(2) lanes (flops): 4 FMA per control term (assembly), 5 for zeta2,
    // 20 per complex Clenshaw step after the peeled one (4), 20 for U, 56
    // for the 2 x 2 complex product; three-point weights as su(2)
    const int N = ctx->n_ctrl, T = ctx->n_terms;
    double w = 0.0;
    if (ctx->mode != SP_MODE_MIDPOINT) w += 4.0 * N;
    if (ctx->mode == SP_MODE_MAGNUS) w += 2.0 * N + 4.0 * (N * (N - 1) / 2);
    const double f = 8.0 * (T - 1) + 5.0 + 20.0 * (m - 1) + 4.0 + 20.0 + 56.0 + w;
    return (double)n * f;
  }
  if (ctx->fam == FAM_S2) {
    const bool fast2 = ctx->herm_exact && ctx->mode == SP_MODE_MIDPOINT && ctx->n_terms <= 3;
    const bool compiled = m == 3 || m == 7 || m == 13 || m == 15;
    const double f = fast2 ? 125.0 + 16.0 * m + (compiled ? 0.0 : 14.0)
                           : 137.0 + 28.7 * m + 16.0 * ctx->n_terms +
                                 (ctx->mode == SP_MODE_MIDPOINT ? 0.0 : 40.0);
    return (double)n * f;
  }
  if (ctx->fam == FAM_S4) return (double)n * (10.3 + 576.0 * m + 64.0 * ctx->n_terms);
  // 3-multiplication products execute 3/4 of the real FP64 MMA work
  const double f = (ctx->last_algo == ALGO_PS3) ? 6.0 : 8.0;
  return (double)n * (f * D * D * D * ctx->last_gemms + 4.0 * D * D * ctx->n_terms);
}

// exclusive prefixes E[l] of cnt plain-layout lane products (into cumE) and
// the total M[cnt-1] E[cnt-1] (into result) by the two-level scan of
// kernels.cuh (group_fold_kernel / fold_kernel / combine_prefix_kernel)
// recursive exclusive scan: E[l] = M[l-1] ... M[0] for cnt lane products,
// groups of SCAN_GS folded in order (one thread per group for D = 2, one CTA
// per group otherwise), the group totals scanned recursively, then
// E[l] = Ein[l] EG[l / SCAN_GS].  Scratch: the arena in ctx->scanEin.
constexpr int SCAN_GS = 32;

size_t scan_arena_elems(int cnt, size_t dd) {
  size_t total = 0;
  while (cnt > SCAN_GS) {
    const int G = (cnt + SCAN_GS - 1) / SCAN_GS;
    total += ((size_t)cnt + 2 * (size_t)G) * dd;  // Ein, group totals, their prefixes
    cnt = G;
  }
  return total + dd;
}

int scan_rec(sp_ctx* ctx, const double2* M, int cnt, double2* E, double2* arena,
             cudaStream_t st) {
  const int D = ctx->D;
  const size_t dd = (size_t)D * D;
  if (cnt <= SCAN_GS) {  // one group
    if (D == 2) {
      group_fold_reg_kernel<2><<<1, 32, 0, st>>>(M, cnt, cnt, E, nullptr);
    } else {
      group_fold_kernel<<<1, 64, 0, st>>>(M, cnt, D, cnt, E, arena);
    }
    CUDA_TRY(ctx, cudaGetLastError());
    ++ctx->launches;
    return SP_OK;
  }
  const int G = (cnt + SCAN_GS - 1) / SCAN_GS;
  double2* Ein = arena;
  double2* Gt = Ein + (size_t)cnt * dd;
  double2* EG = Gt + (size_t)G * dd;
  double2* rest = EG + (size_t)G * dd;
  if (D == 2)
    group_fold_reg_kernel<2><<<(G + 127) / 128, 128, 0, st>>>(M, cnt, SCAN_GS, Ein, Gt);
  else
    group_fold_kernel<<<G, 64, 0, st>>>(M, cnt, D, SCAN_GS, Ein, Gt);
  CUDA_TRY(ctx, cudaGetLastError());
  int rc = scan_rec(ctx, Gt, G, EG, rest, st);
  if (rc) return rc;
  combine_prefix_kernel<<<grid_for((int64_t)cnt * dd, 256), 256, 0, st>>>(Ein, EG, cnt, D,
                                                                          SCAN_GS, E);
  CUDA_TRY(ctx, cudaGetLastError());
  ctx->launches += 2;
  return SP_OK;
}

// exclusive prefixes E[l] of cnt plain-layout lane products (into cumE) and
// the total M[cnt-1] E[cnt-1] (into result); equiprop(sequential) and
// equiprop_all share it, so the last cumulative entry equals the sequential
// total bit for bit
int plain_scan(sp_ctx* ctx, const double2* prods, int cnt, cudaStream_t st) {
  const int D = ctx->D;
  const size_t dd = (size_t)D * D;
  int rc = ensure(ctx, ctx->cumE, (size_t)cnt * dd * sizeof(double2));
  if (!rc) rc = ensure(ctx, ctx->scanEin, scan_arena_elems(cnt, dd) * sizeof(double2));
  if (!rc) rc = ensure(ctx, ctx->result, dd * sizeof(double2));
  if (rc) return rc;
  rc = scan_rec(ctx, prods, cnt, (double2*)ctx->cumE.p, (double2*)ctx->scanEin.p, st);
  if (rc) return rc;
  lane_total_kernel<<<1, 64, 0, st>>>(prods + (size_t)(cnt - 1) * dd,
                                      (const double2*)ctx->cumE.p + (size_t)(cnt - 1) * dd, D,
                                      (double2*)ctx->result.p);
  CUDA_TRY(ctx, cudaGetLastError());
  ++ctx->launches;
  return SP_OK;
}

// total propagator on the device -> d x d in d_out (output dtype)
int equiprop_dev(sp_ctx* ctx, const double* d_amps, int64_t pts, int n_ctrl, double dt,
                 const sp_plan* plan, int reduction, void* d_out, cudaStream_t st) {
  ctx->launches = 0;
  ctx->flops = 0.0;
  ctx->ev_pending = false;
  SliceJob job;
  int rc = build_job(ctx, d_amps, pts, n_ctrl, dt, plan, &job);
  if (rc) return rc;
  // the small families' pairwise product is one launch with a fused tail
  // (complex64 contexts too when the su(2) kernel takes the call)
  const bool su2 = ctx->fam == FAM_S2 && reduction == SP_REDUCE_PAIRWISE && su2_applies(ctx, job);
  const bool fused = (ctx->fam == FAM_S2 || ctx->fam == FAM_S4) && (!f32_path(ctx) || su2) &&
                     reduction == SP_REDUCE_PAIRWISE && job.n_slices > 0;
  rc = arm_validation(ctx, &job, st, fused);
  if (rc) return rc;
  const int D = ctx->D, d = ctx->dim;
  const size_t dd = (size_t)D * D;
  rc = ensure(ctx, ctx->result, dd * sizeof(double2));
  if (rc) return rc;
  const double2* total = nullptr;
  if (job.n_slices == 0) {
    // empty product (propagator.py:297-299)
    // identity (embed of a 0 x 0 block)
    embed_kernel<<<grid_for((int64_t)dd, 256), 256, 0, st>>>(nullptr, 1, 0, D,
                                                              (double2*)ctx->result.p);
    CUDA_TRY(ctx, cudaGetLastError());
    ++ctx->launches;
    total = (const double2*)ctx->result.p;
  } else {
    const bool small = plain_family(ctx->fam);
    const bool cta_reduce = (ctx->fam == FAM_S2 || ctx->fam == FAM_S4) &&
                            (!f32_path(ctx) || su2) && reduction == SP_REDUCE_PAIRWISE;
    const double2* prods = nullptr;
    int cnt = 0;
    // small families + pairwise: one launch does everything (fused tail)
    rc = run_lanes(ctx, job, cta_reduce, nullptr, st, &prods, &cnt, cta_reduce ? d_out : nullptr);
    if (rc) return rc;
    ctx->ev_pending = ctx->prof;
    ctx->kname = family_kernel_name(ctx->fam, ctx->last_algo);
    ctx->flops = executed_flops(ctx, job.n_slices, job.m);
    if (cta_reduce) return SP_OK;
    if (reduction == SP_REDUCE_SEQUENTIAL && !small) {
      // left fold to E_{L-1} = P_{L-2} ... P_0, then P_{L-1} E_{L-1} with the
      // same tensor-core routine equiprop_all uses for its last entry
      rc = ensure(ctx, ctx->seqA, dd * sizeof(double2));
      if (rc) return rc;
      rc = tc_scan(ctx, prods, cnt, st);
      if (rc) return rc;
      to_afrag_kernel<<<grid_for((int64_t)dd, 256), 256, 0, st>>>(
          prods + (size_t)(cnt - 1) * dd, D, (double*)ctx->seqA.p);
      CUDA_TRY(ctx, cudaGetLastError());
      ctx->launches += 1;
      return tc_apply(ctx, (const double*)ctx->seqA.p,
                      (const double2*)ctx->cumE.p + (size_t)(cnt - 1) * dd, 1, 1, d_out, st);
    }
    if (reduction == SP_REDUCE_PAIRWISE) {
      rc = reduce_pairwise_dev(ctx, prods, cnt, D, st, &total);
      if (rc) return rc;
    } else {
      // plain-layout families: the scan equiprop_all uses (bitwise-equal last entry)
      rc = plain_scan(ctx, prods, cnt, st);
      if (rc) return rc;
      total = (const double2*)ctx->result.p;
    }
  }
  extract_kernel<<<grid_for((int64_t)d * d, 256), 256, 0, st>>>(total, 1, D, d,
                                                                out32(ctx), d_out);
  CUDA_TRY(ctx, cudaGetLastError());
  ++ctx->launches;
  return SP_OK;
}

int product_dev(sp_ctx* ctx, int count, const double2* d_mats, int reduction, void* d_out,
                cudaStream_t st) {
  const int d = ctx->dim, D = ctx->D;
  const size_t dd = (size_t)D * D;
  int rc = ensure(ctx, ctx->cumP, std::max(1, count) * dd * sizeof(double2));
  if (rc) return rc;
  rc = ensure(ctx, ctx->result, dd * sizeof(double2));
  if (rc) return rc;
  double2* padded = (double2*)ctx->cumP.p;
  if (count == 0) {
    // identity (embed of a 0 x 0 block)
    embed_kernel<<<grid_for((int64_t)dd, 256), 256, 0, st>>>(nullptr, 1, 0, D,
                                                              (double2*)ctx->result.p);
    CUDA_TRY(ctx, cudaGetLastError());
    ++ctx->launches;
    extract_kernel<<<grid_for((int64_t)d * d, 256), 256, 0, st>>>(
        (const double2*)ctx->result.p, 1, D, d, ctx->bits == 32, d_out);
    CUDA_TRY(ctx, cudaGetLastError());
    ++ctx->launches;
    return SP_OK;
  }
  embed_kernel<<<grid_for((int64_t)count * dd, 256), 256, 0, st>>>(d_mats, count, d, D, padded);
  CUDA_TRY(ctx, cudaGetLastError());
  ++ctx->launches;
  const double2* total = nullptr;
  if (reduction == SP_REDUCE_PAIRWISE) {
    rc = reduce_pairwise_dev(ctx, padded, count, D, st, &total);
    if (rc) return rc;
  } else {
    rc = ensure(ctx, ctx->fold_scratch, 2 * dd * sizeof(double2));
    if (rc) return rc;
    fold_kernel<<<1, 1024, 0, st>>>(padded, count, D, (double2*)ctx->fold_scratch.p, nullptr,
                                     (double2*)ctx->result.p);
    CUDA_TRY(ctx, cudaGetLastError());
    ++ctx->launches;
    total = (const double2*)ctx->result.p;
  }
  extract_kernel<<<grid_for((int64_t)d * d, 256), 256, 0, st>>>(total, 1, D, d,
                                                                ctx->bits == 32, d_out);
  CUDA_TRY(ctx, cudaGetLastError());
  ++ctx->launches;
  return SP_OK;
}

// cumulative propagators on the device: slices x d x d (output dtype) in d_out
int equiprop_all_dev(sp_ctx* ctx, const double* d_amps, int64_t pts, int n_ctrl, double dt,
                     const sp_plan* plan, void* d_out, cudaStream_t st) {
  ctx->launches = 0;
  ctx->ev_pending = false;
  SliceJob job;
  int rc = build_job(ctx, d_amps, pts, n_ctrl, dt, plan, &job);
  if (rc) return rc;
  rc = arm_validation(ctx, &job, st);
  if (rc) return rc;
  const int64_t n = job.n_slices;
  if (n == 0) return SP_OK;
  const int D = ctx->D, d = ctx->dim;
  const size_t dd = (size_t)D * D;
  const double2* prods = nullptr;
  int cnt = 0;
  if (ctx->fam == FAM_S2 && d == 2 && ctx->bits == 64) {
    // d = 2 (the HBM-write-bound case): no prefix round trip.  Pass 1 forms
    // the lane products, the ordered scan their exclusive prefixes E_l, and
    // pass 2 re-runs every lane from V = E_l writing U(t_k <- 0) straight
    // into the (n, 2, 2) complex128 output; the last entry is the sequential
    // total M_{L-1} E_{L-1} of the same scan (bitwise contract with
    // equiprop(reduction="sequential"), propagator.py:304-306)
    rc = run_lanes(ctx, job, false, nullptr, st, &prods, &cnt);
    if (rc) return rc;
    rc = plain_scan(ctx, prods, cnt, st);
    if (rc) return rc;
    SliceJob job2 = job;
    job2.vinit = ctx->cumE.p;
    const double2* prods2 = nullptr;
    int cnt2 = 0;
    rc = run_lanes(ctx, job2, false, (double2*)d_out, st, &prods2, &cnt2);
    if (rc) return rc;
    if (cnt2 != cnt) return fail(ctx, SP_E_INTERNAL, "lane count changed between passes");
    CUDA_TRY(ctx, cudaMemcpyAsync((double2*)d_out + (size_t)(n - 1) * dd, ctx->result.p,
                                  dd * sizeof(double2), cudaMemcpyDeviceToDevice, st));
    ctx->ev_pending = ctx->prof;
    ctx->kname = family_kernel_name(ctx->fam, ctx->last_algo);
    ctx->flops = 2.0 * executed_flops(ctx, n, job.m);
    return SP_OK;
  }
  rc = ensure(ctx, ctx->cumP, (size_t)n * dd * sizeof(double2));
  if (rc) return rc;
  rc = run_lanes(ctx, job, false, (double2*)ctx->cumP.p, st, &prods, &cnt);
  if (rc) return rc;
  ctx->ev_pending = ctx->prof;
  ctx->kname = family_kernel_name(ctx->fam, ctx->last_algo);
  ctx->flops = executed_flops(ctx, n, job.m);
  if (plain_family(ctx->fam)) {
    rc = plain_scan(ctx, prods, cnt, st);
    if (rc) return rc;
  } else {
    rc = tc_scan(ctx, prods, cnt, st);
    if (rc) return rc;
  }
  if (plain_family(ctx->fam)) {
    rc = ensure(ctx, ctx->lstarts, (size_t)(cnt + 1) * sizeof(int64_t));
    if (rc) return rc;
    lane_starts_kernel<<<grid_for(cnt + 1, 256), 256, 0, st>>>(n, cnt, (int64_t*)ctx->lstarts.p);
    CUDA_TRY(ctx, cudaGetLastError());
    const double2* cP = (const double2*)ctx->cumP.p;
    const double2* cE = (const double2*)ctx->cumE.p;
    const int64_t* ls = (const int64_t*)ctx->lstarts.p;
    const int f32 = ctx->bits == 32;
    // one CTA per lane
    if (D == 2)
      apply_prefix_lanes_kernel<2><<<cnt, 256, 0, st>>>(cP, cE, ls, d, f32, d_out);
    else if (D == 4)
      apply_prefix_lanes_kernel<4><<<cnt, 256, 0, st>>>(cP, cE, ls, d, f32, d_out);
    else if (D == 8)
      apply_prefix_lanes_kernel<8><<<cnt, 256, 0, st>>>(cP, cE, ls, d, f32, d_out);
    else
      return fail(ctx, SP_E_INTERNAL, "no plain-layout prefix application for D = %d", D);
    CUDA_TRY(ctx, cudaGetLastError());
    ctx->launches += 2;
  } else {
    // tensor-core prefix application straight into the output dtype
    rc = tc_apply(ctx, (const double*)ctx->cumP.p, (const double2*)ctx->cumE.p, n, cnt, d_out,
                  st);
    if (rc) return rc;
  }
  return SP_OK;
}

// ---- single-process multi-device propagation ----------
// Slices [r n / P, (r+1) n / P) go to child r (three-point modes read the
// one-row halo); every child propagates its block on its own device and
// stream and leaves the complex128 block product in its `out` buffer; the
// blocks are gathered onto the first device by peer copies (d^2 * 16 B each,
// over NVLink between devices) and multiplied there in time order with the
// same pairwise / sequential product sp_product_device uses.
int equiprop_multi(sp_ctx* ctx, const double* amps, int64_t pts, int n_ctrl, double dt,
                   const sp_plan* plan, int reduction, void* u_out) {
  int code;
  const int64_t n = slice_count_for(ctx->mode, pts, &code);
  if (code)
    return fail(ctx, code, "%s, got %lld", parity_message(ctx->mode), (long long)pts);
  const int P = (int)ctx->kids.size();
  const int d = ctx->dim;
  const size_t dd = (size_t)d * d;
  const size_t blk = dd * sizeof(double2);
  sp_ctx* k0 = ctx->kids[0];
  if (ctx->kid_done.size() != (size_t)P) ctx->kid_done.assign(P, nullptr);
  std::vector<int64_t> first_row(P, 0);
  std::vector<char> empty(P, 0);
  int rc = SP_OK;
  for (int r = 0; r < P && !rc; ++r) {
    sp_ctx* kid = ctx->kids[r];
    rc = prepare_device(kid);
    if (rc) return fail(ctx, rc, "device %d: %s", kid->device, kid->err);
    if (!ctx->kid_done[r]) CUDA_TRY(ctx, cudaEventCreateWithFlags(&ctx->kid_done[r],
                                                                  cudaEventDisableTiming));
    const int64_t a = (int64_t)r * n / P, b = (int64_t)(r + 1) * n / P;
    const int64_t lo = ctx->mode == SP_MODE_MIDPOINT ? a : 2 * a;
    const int64_t hi = ctx->mode == SP_MODE_MIDPOINT ? b
                       : ctx->mode >= SP_MODE_GAUSS2 ? 2 * b  // no shared node
                                                     : 2 * b + 1;
    first_row[r] = lo;
    rc = ensure(kid, kid->out, blk);
    if (rc) return fail(ctx, rc, "device %d: %s", kid->device, kid->err);
    if (b <= a) {
      empty[r] = 1;  // identity block, written at the gather
      CUDA_TRY(ctx, cudaEventRecord(ctx->kid_done[r], kid->stream));
      continue;
    }
    const size_t abytes = (size_t)(hi - lo) * n_ctrl * sizeof(double);
    rc = ensure(kid, kid->amps, abytes);
    if (rc) return fail(ctx, rc, "device %d: %s", kid->device, kid->err);
    if (abytes)
      CUDA_TRY(ctx, cudaMemcpyAsync(kid->amps.p, amps + lo * n_ctrl, abytes,
                                    cudaMemcpyHostToDevice, kid->stream));
    kid->block64 = true;
    rc = equiprop_dev(kid, (const double*)kid->amps.p, hi - lo, n_ctrl, dt, plan, reduction,
                      kid->out.p, kid->stream);
    kid->block64 = false;
    if (rc) return fail(ctx, rc, "device %d: %s", kid->device, kid->err);
    rc = fetch_violation(kid, kid->stream);
    if (rc) return fail(ctx, rc, "device %d: %s", kid->device, kid->err);
    CUDA_TRY(ctx, cudaEventRecord(ctx->kid_done[r], kid->stream));
  }
  // gather the block products on the first device, in time order
  CUDA_TRY(ctx, cudaSetDevice(k0->device));
  rc = ensure(ctx, ctx->gather, (size_t)P * blk);
  if (rc) return rc;
  std::vector<double2> eye(dd, make_double2(0.0, 0.0));
  for (int i = 0; i < d; ++i) eye[(size_t)i * d + i] = make_double2(1.0, 0.0);
  double2* g = (double2*)ctx->gather.p;
  for (int r = 0; r < P; ++r) {
    CUDA_TRY(ctx, cudaStreamWaitEvent(k0->stream, ctx->kid_done[r], 0));
    if (empty[r])
      CUDA_TRY(ctx, cudaMemcpyAsync(g + r * dd, eye.data(), blk, cudaMemcpyHostToDevice,
                                    k0->stream));
    else
      CUDA_TRY(ctx, cudaMemcpyPeerAsync(g + r * dd, k0->device, ctx->kids[r]->out.p,
                                        ctx->kids[r]->device, blk, k0->stream));
  }
  const size_t obytes = dd * (ctx->bits == 32 ? 8 : 16);
  rc = ensure(k0, k0->result2, obytes);
  if (rc) return fail(ctx, rc, "device %d: %s", k0->device, k0->err);
  rc = product_dev(k0, P, g, reduction, k0->result2.p, k0->stream);
  if (rc) return fail(ctx, rc, "device %d: %s", k0->device, k0->err);
  if (ctx->out_host_bytes < obytes) {
    if (ctx->out_host) cudaFreeHost(ctx->out_host);
    ctx->out_host = nullptr;
    CUDA_TRY(ctx, cudaMallocHost(&ctx->out_host, obytes));
    ctx->out_host_bytes = obytes;
  }
  CUDA_TRY(ctx, cudaMemcpyAsync(ctx->out_host, k0->result2.p, obytes, cudaMemcpyDeviceToHost,
                                k0->stream));
  // global first amplitude violation: the minimum over the blocks' offenders
  int64_t best = -1;
  ctx->launches = 0;
  for (int r = 0; r < P; ++r) {
    sp_ctx* kid = ctx->kids[r];
    CUDA_TRY(ctx, cudaSetDevice(kid->device));
    CUDA_TRY(ctx, cudaStreamSynchronize(kid->stream));
    ctx->launches += kid->launches;
    if (empty[r]) continue;
    int64_t idx = -1;
    read_violation(kid, nullptr, &idx, true);
    if (idx >= 0) {
      const int64_t gidx = first_row[r] * std::max(1, n_ctrl) + idx;
      if (best < 0 || gidx < best) best = gidx;
    }
  }
  CUDA_TRY(ctx, cudaSetDevice(k0->device));
  CUDA_TRY(ctx, cudaStreamSynchronize(k0->stream));
  ctx->launches += 3 * P;  // copies and the ordered product (counted on k0 too)
  std::memcpy(u_out, ctx->out_host, obytes);
  ctx->multi_viol = best;
  if (best >= 0) {
    const int N = std::max(1, n_ctrl);
    return fail(ctx, SP_E_AMPLITUDE_BOUND,
                "control amplitude %.17g at sample %lld, control %lld lies outside [-1, 1]",
                amps[best], (long long)(best / N), (long long)(best % N));
  }
  return SP_OK;
}

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

const char* sp_version(void) { return kVersion; }

#ifdef SP_PHASE_PROF
// profiling builds only (tools/phase_prof.py): read and clear the per-phase
// clock totals of lane_ps3g_kernel
int sp_phase_prof(unsigned long long* out) {
  if (cudaMemcpyFromSymbol(out, sp::g_phase, 16 * sizeof(unsigned long long)) != cudaSuccess)
    return 1;
  unsigned long long z[16] = {0};
  return cudaMemcpyToSymbol(sp::g_phase, z, sizeof(z)) != cudaSuccess;
}
int sp_timeline(unsigned long long* out) {
  if (cudaMemcpyFromSymbol(out, sp::g_tl, 4096 * sizeof(unsigned long long)) != cudaSuccess)
    return 1;
  static unsigned long long z[4096];
  return cudaMemcpyToSymbol(sp::g_tl, z, sizeof(z)) != cudaSuccess;
}
#endif

int sp_bessel_j(int k, double x, double* out) {
  if (!out) return fail(nullptr, SP_E_CONFIG, "null output");
  return bessel_j(k, x, out, g_err, sizeof(g_err));
}

double sp_chebyshev_error(int m, double span) { return chebyshev_error(m, span); }

int sp_select_m_max(double norm_bound, int precision_bits, int* m_out, double* capability) {
  if (precision_bits != 32 && precision_bits != 64)
    return fail(nullptr, SP_E_CONFIG, "precision must be 32 or 64 bits");
  return select_m_max(norm_bound, precision_bits, m_out, capability, g_err, sizeof(g_err));
}

int sp_norm_capability(int m, int precision_bits, double* out) {
  if (precision_bits != 32 && precision_bits != 64)
    return fail(nullptr, SP_E_CONFIG, "precision must be 32 or 64 bits");
  return norm_capability(m, precision_bits, out, g_err, sizeof(g_err));
}

int sp_make_plan(double alpha, double beta, int precision_bits, int m_override, sp_plan* out) {
  if (!out) return fail(nullptr, SP_E_CONFIG, "null plan");
  if (precision_bits != 32 && precision_bits != 64)
    return fail(nullptr, SP_E_CONFIG, "precision must be 32 or 64 bits");
  return make_plan(alpha, beta, precision_bits, m_override, out, g_err, sizeof(g_err));
}

int sp_create(sp_ctx** out, int precision_bits, int num_gpus, const int* device_ids) {
  if (!out) return fail(nullptr, SP_E_CONFIG, "null output pointer");
  if (precision_bits != 32 && precision_bits != 64)
    return fail(nullptr, SP_E_CONFIG, "unknown precision %d; expected 32 or 64", precision_bits);
  if (num_gpus < 1 || num_gpus > 64)
    return fail(nullptr, SP_E_CONFIG, "num_gpus must be in 1..64, got %d", num_gpus);
  for (int r = 0; device_ids && r < num_gpus; ++r)
    if (device_ids[r] < 0)
      return fail(nullptr, SP_E_CONFIG, "negative device ordinal %d", device_ids[r]);
  sp_ctx* ctx = new sp_ctx();
  ctx->bits = precision_bits;
  ctx->device = device_ids ? device_ids[0] : 0;
  if (num_gpus > 1) {
    // one child context per device: no device work here either (lazy)
    for (int r = 0; r < num_gpus; ++r) {
      sp_ctx* kid = new sp_ctx();
      kid->bits = precision_bits;
      kid->device = device_ids ? device_ids[r] : r;
      ctx->kids.push_back(kid);
    }
  }
  *out = ctx;
  return SP_OK;
}

int sp_free(sp_ctx* ctx) {
  if (!ctx) return SP_OK;
  if (!ctx->kids.empty()) {
    if (ctx->gather.p) {
      cudaSetDevice(ctx->kids[0]->device);
      cudaStreamSynchronize(ctx->kids[0]->stream);
      cudaFree(ctx->gather.p);
    }
    for (size_t r = 0; r < ctx->kid_done.size(); ++r)
      if (ctx->kid_done[r]) {
        cudaSetDevice(ctx->kids[r]->device);
        cudaEventDestroy(ctx->kid_done[r]);
      }
    if (ctx->out_host) cudaFreeHost(ctx->out_host);
    ctx->out_host = nullptr;
    for (sp_ctx* kid : ctx->kids) sp_free(kid);
    ctx->kids.clear();
  }
  if (ctx->dev_ready) {
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    DevBuf* bufs[] = {&ctx->terms, &ctx->amps,  &ctx->lanes, &ctx->ctab, &ctx->tree0,
                      &ctx->tree1, &ctx->xglob, &ctx->gctr,  &ctx->result, &ctx->out,
                      &ctx->cumP,  &ctx->cumE,  &ctx->cumO,  &ctx->fold_scratch,
                      &ctx->psA,   &ctx->tpriv, &ctx->viol, &ctx->terms3, &ctx->tailctr,
                      &ctx->seqA, &ctx->scanEin, &ctx->lstarts, &ctx->scanS, &ctx->scanA,
                      &ctx->result2};
    for (DevBuf* b : bufs)
      if (b->p) cudaFree(b->p);
    if (ctx->ev0) cudaEventDestroy(ctx->ev0);
    if (ctx->ev1) cudaEventDestroy(ctx->ev1);
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
    if (ctx->viol_host) cudaFreeHost(ctx->viol_host);
    if (ctx->out_host) cudaFreeHost(ctx->out_host);
  }
  delete ctx;
  return SP_OK;
}

const char* sp_last_error(const sp_ctx* ctx) { return ctx ? ctx->err : g_err; }

int sp_set_hamiltonian(sp_ctx* ctx, int dim, int n_ctrl, int n_terms, int mode,
                       const double* terms) {
  if (!ctx) return fail(nullptr, SP_E_STATE_MACHINE, "null context");
  if (dim < 1) return fail(ctx, SP_E_SHAPE, "dim must be >= 1, got %d", dim);
  if (mode < SP_MODE_MIDPOINT || mode > SP_MODE_GAUSS4)
    return fail(ctx, SP_E_CONFIG, "unknown mode %d", mode);
  const int expect = (mode == SP_MODE_MAGNUS || mode == SP_MODE_GAUSS4)
                         ? 1 + 2 * n_ctrl + n_ctrl * (n_ctrl - 1) / 2
                                              : 1 + n_ctrl;
  if (n_ctrl < 0 || n_terms != expect)
    return fail(ctx, SP_E_SHAPE, "%d expansion terms do not match %d controls in mode %d",
                n_terms, n_ctrl, mode);
  if (n_terms > 256) return fail(ctx, SP_E_CONFIG, "at most 256 expansion terms supported");
  int D = 0;
  const int fam = family_for(dim, &D);
  if (fam == FAM_NONE)
    return fail(ctx, SP_E_CONFIG, "dimension %d not supported (max 512)", dim);
  if (!terms) return fail(ctx, SP_E_SHAPE, "null terms");
  ctx->dim = dim;
  ctx->n_ctrl = n_ctrl;
  ctx->n_terms = n_terms;
  ctx->mode = mode;
  ctx->terms_host.assign(terms, terms + (size_t)n_terms * dim * dim * 2);
  ctx->herm_exact = true;
  for (int t = 0; t < n_terms && ctx->herm_exact; ++t)
    for (int r = 0; r < dim && ctx->herm_exact; ++r)
      for (int c = r; c < dim; ++c) {
        const double* a = &ctx->terms_host[(((size_t)t * dim + r) * dim + c) * 2];
        const double* b = &ctx->terms_host[(((size_t)t * dim + c) * dim + r) * 2];
        if (!(a[0] == b[0] && a[1] == -b[1])) {
          ctx->herm_exact = false;
          break;
        }
      }
  // su(2) family (kernels_su2.cuh): 2 x 2 terms that are bitwise Hermitian
  // and traceless, at most SU2_MAX_CTRL controls
  const bool two = dim == 2 && ctx->herm_exact && n_ctrl >= 1 && n_ctrl <= SU2_MAX_CTRL &&
                   n_terms <= SU2_MAX_TERMS;
  ctx->su2_terms = two;
  for (int t = 0; t < n_terms && ctx->su2_terms; ++t)
    if (!(ctx->terms_host[(size_t)t * 8 + 0] == -ctx->terms_host[(size_t)t * 8 + 6]))
      ctx->su2_terms = false;
  // u(2) lanes (kernels_su2.cuh, 2 x 2 complex algebra) for the rest
  ctx->u2_terms = two && !ctx->su2_terms;
  ctx->fam = fam;
  ctx->D = D;
  ctx->terms_uploaded = false;
  ctx->loaded = true;
  for (sp_ctx* kid : ctx->kids) {
    const int rc = sp_set_hamiltonian(kid, dim, n_ctrl, n_terms, mode, terms);
    if (rc) return fail(ctx, rc, "device %d: %s", kid->device, kid->err);
  }
  return SP_OK;
}

int sp_slice_count(const sp_ctx* ctx, int64_t pts, int64_t* out) {
  if (!ctx || !ctx->loaded) return fail(nullptr, SP_E_STATE_MACHINE, "no Hamiltonian loaded");
  int code;
  *out = slice_count_for(ctx->mode, pts, &code);
  if (code) return fail(nullptr, code, "%s", parity_message(ctx->mode));
  return SP_OK;
}

int sp_equiprop_device(sp_ctx* ctx, const double* d_amps, int64_t pts, int n_ctrl, double dt,
                       const sp_plan* plan, int reduction, void* d_u_out, void* stream) {
  if (ctx && !ctx->kids.empty()) {
    ctx->last_multi = false;
    return sp_equiprop_device(ctx->kids[0], d_amps, pts, n_ctrl, dt, plan, reduction, d_u_out,
                              stream);
  }
  int rc = check_loaded(ctx);
  if (rc) return rc;
  if (reduction != SP_REDUCE_PAIRWISE && reduction != SP_REDUCE_SEQUENTIAL)
    return fail(ctx, SP_E_CONFIG, "unknown reduction %d", reduction);
  rc = prepare_device(ctx);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;  // NULL = the CUDA default stream
  return equiprop_dev(ctx, d_amps, pts, n_ctrl, dt, plan, reduction, d_u_out, st);
}

int sp_equiprop(sp_ctx* ctx, const double* amps, int64_t pts, int n_ctrl, double dt,
                const sp_plan* plan, int reduction, void* u_out) {
  int rc = check_loaded(ctx);
  if (rc) return rc;
  if (reduction != SP_REDUCE_PAIRWISE && reduction != SP_REDUCE_SEQUENTIAL)
    return fail(ctx, SP_E_CONFIG, "unknown reduction %d", reduction);
  if (pts < 0) return fail(ctx, SP_E_SHAPE, "negative sample count");
  if (!ctx->kids.empty()) {
    if (n_ctrl != ctx->n_ctrl)
      return fail(ctx, SP_E_SHAPE, "amplitude table has %d controls, system has %d", n_ctrl,
                  ctx->n_ctrl);
    ctx->last_multi = true;
    return equiprop_multi(ctx, amps, pts, n_ctrl, dt, plan, reduction, u_out);
  }
  rc = prepare_device(ctx);
  if (rc) return rc;
  cudaStream_t st = ctx->stream;
  const size_t abytes = (size_t)pts * n_ctrl * sizeof(double);
  rc = ensure(ctx, ctx->amps, abytes);
  if (rc) return rc;
  if (abytes)
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->amps.p, amps, abytes, cudaMemcpyHostToDevice, st));
  const size_t obytes = (size_t)ctx->dim * ctx->dim * (ctx->bits == 32 ? 8 : 16);
  rc = ensure(ctx, ctx->out, obytes);
  if (rc) return rc;
  rc = equiprop_dev(ctx, (const double*)ctx->amps.p, pts, n_ctrl, dt, plan, reduction,
                    ctx->out.p, st);
  if (rc) return rc;
  if (ctx->out_host_bytes < obytes) {
    if (ctx->out_host) cudaFreeHost(ctx->out_host);
    ctx->out_host = nullptr;
    ctx->out_host_bytes = 0;
    CUDA_TRY(ctx, cudaMallocHost(&ctx->out_host, obytes));
    ctx->out_host_bytes = obytes;
  }
  CUDA_TRY(ctx, cudaMemcpyAsync(ctx->out_host, ctx->out.p, obytes, cudaMemcpyDeviceToHost, st));
  rc = fetch_violation(ctx, st);
  if (rc) return rc;
  CUDA_TRY(ctx, cudaStreamSynchronize(st));
  std::memcpy(u_out, ctx->out_host, obytes);
  return read_violation(ctx, amps, nullptr, true);
}

int sp_equiprop_all(sp_ctx* ctx, const double* amps, int64_t pts, int n_ctrl, double dt,
                    const sp_plan* plan, void* u_all_out) {
  if (ctx && !ctx->kids.empty()) {
    ctx->last_multi = false;
    const int rc = sp_equiprop_all(ctx->kids[0], amps, pts, n_ctrl, dt, plan, u_all_out);
    if (rc) return fail(ctx, rc, "%s", ctx->kids[0]->err);
    return SP_OK;
  }
  int rc = check_loaded(ctx);
  if (rc) return rc;
  if (pts < 0) return fail(ctx, SP_E_SHAPE, "negative sample count");
  rc = prepare_device(ctx);
  if (rc) return rc;
  cudaStream_t st = ctx->stream;
  const size_t abytes = (size_t)pts * n_ctrl * sizeof(double);
  rc = ensure(ctx, ctx->amps, abytes);
  if (rc) return rc;
  if (abytes)
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->amps.p, amps, abytes, cudaMemcpyHostToDevice, st));
  int64_t n = 0;
  int code = 0;
  n = slice_count_for(ctx->mode, pts, &code);
  if (code == 0 && n > 0) {
    const size_t obytes = (size_t)n * ctx->dim * ctx->dim * (ctx->bits == 32 ? 8 : 16);
    rc = ensure(ctx, ctx->out, obytes);
    if (rc) return rc;
  }
  rc = equiprop_all_dev(ctx, (const double*)ctx->amps.p, pts, n_ctrl, dt, plan, ctx->out.p, st);
  if (rc) return rc;
  if (n > 0) {
    const size_t obytes = (size_t)n * ctx->dim * ctx->dim * (ctx->bits == 32 ? 8 : 16);
    CUDA_TRY(ctx, cudaMemcpyAsync(u_all_out, ctx->out.p, obytes, cudaMemcpyDeviceToHost, st));
  }
  CUDA_TRY(ctx, cudaStreamSynchronize(st));
  return read_violation(ctx, amps, nullptr);
}

int sp_equiprop_all_device(sp_ctx* ctx, const double* d_amps, int64_t pts, int n_ctrl,
                           double dt, const sp_plan* plan, void* d_u_all_out, void* stream) {
  if (ctx && !ctx->kids.empty()) {
    ctx->last_multi = false;
    return sp_equiprop_all_device(ctx->kids[0], d_amps, pts, n_ctrl, dt, plan, d_u_all_out,
                                  stream);
  }
  int rc = check_loaded(ctx);
  if (rc) return rc;
  if (pts < 0) return fail(ctx, SP_E_SHAPE, "negative sample count");
  rc = prepare_device(ctx);
  if (rc) return rc;
  return equiprop_all_dev(ctx, d_amps, pts, n_ctrl, dt, plan, d_u_all_out,
                          (cudaStream_t)stream);
}

int sp_product_device(sp_ctx* ctx, int count, const void* d_mats, int reduction, void* d_out,
                      void* stream) {
  if (ctx && !ctx->kids.empty())
    return sp_product_device(ctx->kids[0], count, d_mats, reduction, d_out, stream);
  int rc = check_loaded(ctx);
  if (rc) return rc;
  if (count < 0) return fail(ctx, SP_E_SHAPE, "negative count");
  rc = prepare_device(ctx);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;  // NULL = the CUDA default stream
  return product_dev(ctx, count, (const double2*)d_mats, reduction, d_out, st);
}

int sp_qubit_midpoint_reference(sp_ctx* ctx, double w0, double w1, double wrf,
                                double duration, int64_t steps, double* u_out) {
  if (ctx && !ctx->kids.empty())
    return sp_qubit_midpoint_reference(ctx->kids[0], w0, w1, wrf, duration, steps, u_out);
  if (!ctx) return fail(nullptr, SP_E_STATE_MACHINE, "null context");
  if (!u_out) return fail(ctx, SP_E_SHAPE, "null output");
  // studies.py:131-139: identity for no steps or no field
  const double vnorm = std::hypot(w1, w0);
  if (steps < 1 || vnorm == 0.0) {
    const double id[8] = {1, 0, 0, 0, 0, 0, 1, 0};
    std::memcpy(u_out, id, sizeof(id));
    return SP_OK;
  }
  int rc = device_init(ctx);
  if (rc) return rc;
  CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  const double dt = duration / (double)steps;
  Su2Job sj;
  std::memset(&sj, 0, sizeof(sj));
  const int block = 512;
  const int grid = (int)std::max<int64_t>(
      1, std::min<int64_t>(ctx->sms, (steps + (int64_t)block * 8 - 1) / ((int64_t)block * 8)));
  rc = ensure(ctx, ctx->lanes, (size_t)grid * 4 * sizeof(double));
  if (rc) return rc;
  rc = ensure(ctx, ctx->result, 4 * sizeof(double2));
  if (rc) return rc;
  if (!ctx->tailctr.p) {
    rc = ensure(ctx, ctx->tailctr, sizeof(unsigned));
    if (rc) return rc;
    CUDA_TRY(ctx, cudaMemsetAsync(ctx->tailctr.p, 0, sizeof(unsigned), st));
  }
  sj.cta_out = ctx->lanes.p;
  sj.ctr = (unsigned*)ctx->tailctr.p;
  sj.out = ctx->result.p;
  CUDA_TRY(ctx, su2_qubit_reference(sj, steps, std::cos(vnorm * dt / 2.0),
                                    std::sin(vnorm * dt / 2.0), w1 / vnorm, w0 / vnorm, wrf,
                                    dt, grid, block, st));
  CUDA_TRY(ctx, cudaMemcpyAsync(u_out, ctx->result.p, 4 * sizeof(double2),
                                cudaMemcpyDeviceToHost, st));
  CUDA_TRY(ctx, cudaStreamSynchronize(st));
  return SP_OK;
}

int sp_amplitude_violation(sp_ctx* ctx, int64_t* index) {
  if (ctx && !ctx->kids.empty()) {
    if (ctx->last_multi) {
      if (index) *index = ctx->multi_viol;
      return ctx->multi_viol >= 0 ? SP_E_AMPLITUDE_BOUND : SP_OK;
    }
    return sp_amplitude_violation(ctx->kids[0], index);
  }
  if (!ctx) return fail(nullptr, SP_E_STATE_MACHINE, "null context");
  return read_violation(ctx, nullptr, index);
}

int sp_set_algorithm(sp_ctx* ctx, int algo) {
  for (sp_ctx* kid : ctx ? ctx->kids : std::vector<sp_ctx*>()) {
    const int rc = sp_set_algorithm(kid, algo);
    if (rc) return fail(ctx, rc, "%s", kid->err);
  }
  if (!ctx) return fail(nullptr, SP_E_STATE_MACHINE, "null context");
  if (algo < ALGO_AUTO || algo > ALGO_PS3)
    return fail(ctx, SP_E_CONFIG, "unknown algorithm %d (0 auto, 1 clenshaw, 2 ps, 3 ps3m)", algo);
  ctx->algo = algo;
  return SP_OK;
}

int sp_last_algorithm(const sp_ctx* ctx, int* algo, int* gemms_per_slice) {
  if (ctx && !ctx->kids.empty()) return sp_last_algorithm(ctx->kids[0], algo, gemms_per_slice);
  if (!ctx) return fail(nullptr, SP_E_STATE_MACHINE, "null context");
  if (algo) *algo = ctx->last_algo;
  if (gemms_per_slice) *gemms_per_slice = ctx->last_gemms;
  return SP_OK;
}

int sp_last_lanes(const sp_ctx* ctx, int* lanes) {
  if (ctx && !ctx->kids.empty()) {
    int total = 0;
    for (const sp_ctx* kid : ctx->kids) total += kid->last_lanes;
    if (lanes) *lanes = total;
    return SP_OK;
  }
  if (!ctx) return fail(nullptr, SP_E_STATE_MACHINE, "null context");
  if (lanes) *lanes = ctx->last_lanes;
  return SP_OK;
}

int sp_set_profiling(sp_ctx* ctx, int enabled) {
  for (sp_ctx* kid : ctx ? ctx->kids : std::vector<sp_ctx*>()) sp_set_profiling(kid, enabled);
  if (!ctx) return fail(nullptr, SP_E_STATE_MACHINE, "null context");
  ctx->prof = enabled != 0;
  return SP_OK;
}

int sp_last_timing(const sp_ctx* cctx, double* main_kernel_ms, int* launches,
                   double* executed, char* kernel_name, int name_len) {
  if (cctx && !cctx->kids.empty()) {
    const int rc = sp_last_timing(cctx->kids[0], main_kernel_ms, launches, executed, kernel_name,
                                  name_len);
    if (rc) return rc;
    if (cctx->last_multi) {
      if (launches) *launches = cctx->launches;
      double f = 0.0;
      for (const sp_ctx* kid : cctx->kids) f += kid->flops;
      if (executed) *executed = f;
    }
    return SP_OK;
  }
  sp_ctx* ctx = const_cast<sp_ctx*>(cctx);
  if (!ctx) return fail(nullptr, SP_E_STATE_MACHINE, "null context");
  if (ctx->ev_pending) {
    CUDA_TRY(ctx, cudaEventSynchronize(ctx->ev1));
    CUDA_TRY(ctx, cudaEventElapsedTime(&ctx->last_ms, ctx->ev0, ctx->ev1));
    ctx->ev_pending = false;
  }
  if (main_kernel_ms) *main_kernel_ms = ctx->last_ms;
  if (launches) *launches = ctx->launches;
  if (executed) *executed = ctx->flops;
  if (kernel_name && name_len > 0) snprintf(kernel_name, name_len, "%s", ctx->kname);
  return SP_OK;
}

int sp_device_count(int* out) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  *out = (e == cudaSuccess) ? n : 0;
  return SP_OK;
}

}  // extern "C"
