// Batched dense complex linear algebra on the device: the B200 counterpart
// of the reference's materialised batch layer (sliceprop/linalg.py:204-288,
// chebyshev.py:259-306), exposed for users who exponentiate or combine their
// own batches (expm_batch, build_exponent_batch, gemm_strided_batched).  The
// propagation hot path (equiprop) never uses these: it fuses all three
// stages into the lane kernels.
//
// Every kernel is templated on the real type R (double: complex128, FP64
// DFMA; float: complex64, FP32 FFMA), so a complex64 batch is computed in
// complex64 arithmetic as the reference does (linalg.py:270-287,
// chebyshev.py:293-303: terms, coefficients and series coefficients cast
// to the working dtype).
//
//   expand_kernel         out[k] = scale (T_0 + sum_i w[k,i] T_i)   HBM-write-bound
//   expm_fused_kernel     U[k] = p(X_k), X_k = (2/span)(G_k - c I), the whole
//                         Clenshaw recurrence on chip (d <= 64): one CTA holds
//                         X^T and the current iterate in smem, each thread a
//                         RT x RT block of D0 / D1 in registers
//   gemm_batched_kernel   C[k] = alpha A[k] B[k] + beta C[k] + gamma I
//                         (64 x 64 output tiles, 4 x 4 per thread, k-chunks
//                         of 16 staged in smem); the d > 64 Clenshaw steps
//   xprep_kernel          X = (2/span)(G - c I)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace sp {
namespace batch {

template <class R>
struct cplx {
  R x, y;
};

template <class R>
__device__ __forceinline__ cplx<R> cmk(R a, R b) {
  cplx<R> c;
  c.x = a;
  c.y = b;
  return c;
}

// c += a * b (complex), FMA order of a naive complex product
template <class R>
__device__ __forceinline__ void cfma(cplx<R>& c, const cplx<R>& a, const cplx<R>& b) {
  c.x = fma(a.x, b.x, c.x);
  c.x = fma(-a.y, b.y, c.x);
  c.y = fma(a.x, b.y, c.y);
  c.y = fma(a.y, b.x, c.y);
}

template <class R>
__device__ __forceinline__ cplx<R> cmul(const cplx<R>& a, const cplx<R>& b) {
  return cmk<R>(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// ---------------------------------------------------------------------------
// expansion: out[k, e] = scale * (T_0[e] + sum_{i>=1} w[k, i] T_i[e])
// terms: complex128 (T, d*d); w: float64 (count, T), column 0 == 1 (checked
// on the host, linalg.py:261-262).  Terms and weights are rounded to the
// working precision first, the drift is the broadcast column, the controls
// are accumulated in order and added, then the real scale multiplies
// (linalg.py:270-287).
// ---------------------------------------------------------------------------
template <class R>
__global__ void __launch_bounds__(256) expand_kernel(const double2* __restrict__ terms, int T,
                                                     int64_t dd,
                                                     const double* __restrict__ w,
                                                     int64_t count, double scale,
                                                     cplx<R>* __restrict__ out) {
  const int64_t total = count * dd;
  const R sc = (R)scale;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = idx / dd;
    const int64_t e = idx - k * dd;
    const double2 t0 = __ldg(&terms[e]);
    cplx<R> acc = cmk<R>((R)t0.x, (R)t0.y);
    if (T > 1) {
      cplx<R> ctl = cmk<R>((R)0, (R)0);
      const double* wk = w + k * T;
      for (int t = 1; t < T; ++t) {
        const R wt = (R)__ldg(&wk[t]);
        const double2 v = __ldg(&terms[(int64_t)t * dd + e]);
        ctl.x = fma(wt, (R)v.x, ctl.x);
        ctl.y = fma(wt, (R)v.y, ctl.y);
      }
      acc.x += ctl.x;
      acc.y += ctl.y;
    }
    acc.x *= sc;
    acc.y *= sc;
    out[idx] = acc;
  }
}

// ---------------------------------------------------------------------------
// fused Clenshaw exponential of small matrices (padded dim DP <= 64).
// Threads per matrix TPM = (DP / RT)^2; MPC matrices per CTA (RT = 1 only).
// Thread (rb, cb) owns rows rb + i (DP / RT), columns cb + j (DP / RT)
// (interleaved so that a warp's shared-memory reads are contiguous).
// smem per matrix: X^T (DP x DP) and the current iterate B (DP x DP).
// The recurrence is the reference's (chebyshev.py:294-303):
//   D1 <- 2 X D0 - D1 + a_k I;  D0 <- 2 X D1 - (k==1 ? 2 : 1) D0 + a_{k-1 or 0} I
// (the first product multiplies D0 = 0 and is skipped), U = phase D0.
// ---------------------------------------------------------------------------
struct ExpmParams {
  int d, DP, m;
  double xscale;   // 2 / span (0 when span == 0)
  double center;   // (alpha + beta) / 2
  double coef[2 * 26];
  double phase[2];
  int phase_one;
  int64_t count;
  int64_t stride_in, stride_out;  // complex elements between matrices
};

template <class R, int RT>
__global__ void __launch_bounds__(256) expm_fused_kernel(ExpmParams p,
                                                         const cplx<R>* __restrict__ g,
                                                         cplx<R>* __restrict__ u) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cplx<R>* sm = reinterpret_cast<cplx<R>*>(smem_raw);
  const int DP = p.DP, d = p.d;
  const int NB = DP / RT;            // row / column blocks
  const int TPM = NB * NB;           // threads per matrix
  const int MPC = blockDim.x / TPM;  // matrices per CTA
  const int local = threadIdx.x / TPM;
  const int t = threadIdx.x - local * TPM;
  const bool active = local < MPC;
  const int rb = t / NB, cb = t - rb * NB;
  const int64_t mat = (int64_t)blockIdx.x * MPC + local;
  const bool live = active && mat < p.count;
  const int DD = DP * DP;
  cplx<R>* xt = sm + (size_t)(active ? local : 0) * 2 * DD;  // X^T
  cplx<R>* bb = xt + DD;                                        // iterate

  // X^T = ((2/span)(G - c I))^T, zero padded, in the working precision
  // (reference: copy, diagonal shift, then *= real(2/span))
  const R xs = (R)p.xscale;
  const R cen = (R)p.center;
  if (active) {
    for (int e = t; e < DD; e += TPM) {
      const int i = e / DP, j = e - (e / DP) * DP;  // X[i][j]
      cplx<R> v = cmk<R>((R)0, (R)0);
      if (live && i < d && j < d) {
        v = g[mat * p.stride_in + (int64_t)i * d + j];
        if (i == j) v.x -= cen;
        v.x *= xs;
        v.y *= xs;
      }
      xt[j * DP + i] = v;  // transposed
    }
  }
  cplx<R> d0[RT][RT], d1[RT][RT];
#pragma unroll
  for (int a = 0; a < RT; ++a)
#pragma unroll
    for (int b = 0; b < RT; ++b) {
      d0[a][b] = cmk<R>((R)0, (R)0);
      d1[a][b] = cmk<R>((R)0, (R)0);
    }
  auto coef = [&](int k) { return cmk<R>((R)p.coef[2 * k], (R)p.coef[2 * k + 1]); };
  // acc = X B over the thread's block (B in smem)
  auto product = [&](cplx<R> (&acc)[RT][RT]) {
#pragma unroll
    for (int a = 0; a < RT; ++a)
#pragma unroll
      for (int b = 0; b < RT; ++b) acc[a][b] = cmk<R>((R)0, (R)0);
    for (int k = 0; k < DP; ++k) {
      cplx<R> xa[RT], bv[RT];
#pragma unroll
      for (int a = 0; a < RT; ++a) xa[a] = xt[k * DP + rb + a * NB];
#pragma unroll
      for (int b = 0; b < RT; ++b) bv[b] = bb[k * DP + cb + b * NB];
#pragma unroll
      for (int a = 0; a < RT; ++a)
#pragma unroll
        for (int b = 0; b < RT; ++b) cfma(acc[a][b], xa[a], bv[b]);
    }
  };
  auto publish = [&](cplx<R> (&v)[RT][RT]) {
    __syncthreads();
    if (active) {
#pragma unroll
      for (int a = 0; a < RT; ++a)
#pragma unroll
        for (int b = 0; b < RT; ++b) bb[(rb + a * NB) * DP + cb + b * NB] = v[a][b];
    }
    __syncthreads();
  };
  bool first = true;
  for (int k = p.m; k >= 1; k -= 2) {
    // D1 <- 2 X D0 - D1 + a_k I
    cplx<R> acc[RT][RT];
    if (first) {
#pragma unroll
      for (int a = 0; a < RT; ++a)
#pragma unroll
        for (int b = 0; b < RT; ++b) acc[a][b] = cmk<R>((R)0, (R)0);
      __syncthreads();  // X^T complete
    } else {
      product(acc);
    }
    first = false;
    const cplx<R> ak = coef(k);
#pragma unroll
    for (int a = 0; a < RT; ++a)
#pragma unroll
      for (int b = 0; b < RT; ++b) {
        cplx<R> v = cmk<R>((R)2 * acc[a][b].x - d1[a][b].x, (R)2 * acc[a][b].y - d1[a][b].y);
        if (rb + a * NB == cb + b * NB) {
          v.x += ak.x;
          v.y += ak.y;
        }
        d1[a][b] = v;
      }
    publish(d1);
    // D0 <- 2 X D1 - c D0 + a' I
    product(acc);
    const bool last = k == 1;
    const R c = last ? (R)2 : (R)1;
    const cplx<R> ap = coef(last ? 0 : k - 1);
#pragma unroll
    for (int a = 0; a < RT; ++a)
#pragma unroll
      for (int b = 0; b < RT; ++b) {
        cplx<R> v = cmk<R>((R)2 * acc[a][b].x - c * d0[a][b].x,
                           (R)2 * acc[a][b].y - c * d0[a][b].y);
        if (rb + a * NB == cb + b * NB) {
          v.x += ap.x;
          v.y += ap.y;
        }
        d0[a][b] = v;
      }
    if (!last) publish(d0);
  }
  if (!live) return;
  const cplx<R> ph = cmk<R>((R)p.phase[0], (R)p.phase[1]);
#pragma unroll
  for (int a = 0; a < RT; ++a)
#pragma unroll
    for (int b = 0; b < RT; ++b) {
      const int i = rb + a * NB, j = cb + b * NB;
      if (i < d && j < d) {
        cplx<R> v = d0[a][b];
        if (!p.phase_one) v = cmul(v, ph);
        u[mat * p.stride_out + (int64_t)i * d + j] = v;
      }
    }
}

// ---------------------------------------------------------------------------
// general batched complex GEMM with a fused epilogue:
//   C[k] = alpha A[k] B[k] + beta Cin[k] + gamma I       (Cin may equal C)
// 64 x 64 output tile per CTA (256 threads, 4 x 4 complex per thread,
// interleaved rows ty + 16 i / columns tx + 16 j), K in chunks of 16 staged
// through shared memory (A transposed).  beta == 0 never reads Cin
// (linalg.py:214-219).
// ---------------------------------------------------------------------------
struct GemmParams {
  int d;
  int64_t count;
  int64_t sa, sb, sc, scin;  // strides (complex elements)
  double alpha[2], beta[2], gamma[2];
  int beta_zero;
};

template <class R>
__global__ void __launch_bounds__(256) gemm_batched_kernel(GemmParams p,
                                                           const cplx<R>* __restrict__ A,
                                                           const cplx<R>* __restrict__ B,
                                                           const cplx<R>* Cin, cplx<R>* C) {
  constexpr int TM = 64, TK = 16;
  __shared__ cplx<R> As[TK][TM];
  __shared__ cplx<R> Bs[TK][TM];
  const int d = p.d;
  const int tiles = (d + TM - 1) / TM;
  const int64_t mat = blockIdx.x / (tiles * tiles);
  const int tile = blockIdx.x - (int)(mat * tiles * tiles);
  const int tr = (tile / tiles) * TM, tc = (tile % tiles) * TM;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const cplx<R>* a = A + mat * p.sa;
  const cplx<R>* b = B + mat * p.sb;
  cplx<R> acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = cmk<R>((R)0, (R)0);
  for (int k0 = 0; k0 < d; k0 += TK) {
    // A tile rows tr..tr+63, cols k0..k0+15 -> As[kk][row]; B rows k0.., cols tc..
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int e = threadIdx.x + q * 256;  // 0..1023
      const int ar = e >> 4, ak = e & 15;
      const int gr = tr + ar, gk = k0 + ak;
      As[ak][ar] = (gr < d && gk < d) ? a[(int64_t)gr * d + gk] : cmk<R>((R)0, (R)0);
      const int bk = e >> 6, bc = e & 63;
      const int hk = k0 + bk, hc = tc + bc;
      Bs[bk][bc] = (hk < d && hc < d) ? b[(int64_t)hk * d + hc] : cmk<R>((R)0, (R)0);
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < TK; ++kk) {
      cplx<R> av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) cfma(acc[i][j], av[i], bv[j]);
    }
    __syncthreads();
  }
  const cplx<R> al = cmk<R>((R)p.alpha[0], (R)p.alpha[1]);
  const cplx<R> be = cmk<R>((R)p.beta[0], (R)p.beta[1]);
  const cplx<R> ga = cmk<R>((R)p.gamma[0], (R)p.gamma[1]);
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = tr + ty + 16 * i, c = tc + tx + 16 * j;
      if (r >= d || c >= d) continue;
      cplx<R> v = cmul(al, acc[i][j]);
      if (!p.beta_zero) {
        const cplx<R> old = Cin[mat * p.scin + (int64_t)r * d + c];
        const cplx<R> bo = cmul(be, old);
        v.x += bo.x;
        v.y += bo.y;
      }
      if (r == c) {
        v.x += ga.x;
        v.y += ga.y;
      }
      C[mat * p.sc + (int64_t)r * d + c] = v;
    }
}

// X = (2/span)(G - c I) (compact output), or 0 when span == 0
template <class R>
__global__ void xprep_kernel(const cplx<R>* __restrict__ g, int64_t stride_in, int d,
                             int64_t count, double xscale, double center,
                             cplx<R>* __restrict__ x) {
  const int64_t dd = (int64_t)d * d, total = count * dd;
  const R xs = (R)xscale, cen = (R)center;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = idx / dd, e = idx - k * dd;
    cplx<R> v = g[k * stride_in + e];
    if (e / d == e % d) v.x -= cen;
    v.x *= xs;
    v.y *= xs;
    x[idx] = v;
  }
}

// out[k] = phase * in[k] (strided output)
template <class R>
__global__ void phase_copy_kernel(const cplx<R>* __restrict__ in, int d, int64_t count,
                                  double ph_re, double ph_im, int phase_one,
                                  cplx<R>* __restrict__ out, int64_t stride_out) {
  const int64_t dd = (int64_t)d * d, total = count * dd;
  const cplx<R> ph = cmk<R>((R)ph_re, (R)ph_im);
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = idx / dd, e = idx - k * dd;
    cplx<R> v = in[idx];
    if (!phase_one) v = cmul(v, ph);
    out[k * stride_out + e] = v;
  }
}

// ---- state propagation (apply, propagator.py:105-118) ----------------------
// out[k] = U psi_k: one thread per output entry, psi_k = row k of the
// (count, d) state batch
template <class R>
__global__ void __launch_bounds__(256) apply_vec_kernel(int d, int64_t count,
                                                        const cplx<R>* __restrict__ U,
                                                        const cplx<R>* __restrict__ psi,
                                                        cplx<R>* __restrict__ out) {
  const int64_t total = count * d;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = e / d;
    const int i = (int)(e % d);
    const cplx<R>* u = U + (size_t)i * d;
    const cplx<R>* v = psi + (size_t)k * d;
    R re = 0, im = 0;
    for (int j = 0; j < d; ++j) {
      re = fma(u[j].x, v[j].x, re);
      re = fma(-u[j].y, v[j].y, re);
      im = fma(u[j].x, v[j].y, im);
      im = fma(u[j].y, v[j].x, im);
    }
    out[e] = cmk<R>(re, im);
  }
}

// out = U^+ (conjugate transpose)
template <class R>
__global__ void adjoint_kernel(int d, const cplx<R>* __restrict__ U, cplx<R>* __restrict__ out) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < d * d; e += gridDim.x * blockDim.x) {
    const int i = e / d, j = e % d;
    const cplx<R> v = U[(size_t)j * d + i];
    out[e] = cmk<R>(v.x, -v.y);
  }
}

}  // namespace batch
}  // namespace sp
