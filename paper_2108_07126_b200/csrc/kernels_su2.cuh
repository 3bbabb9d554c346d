// Family SU2: d = 2 systems whose expansion terms are all bitwise Hermitian
// and traceless (the paper's driven qubit, any su(2) drive), symmetric plan.
//
// Why a separate family.  With Z = 2X = Z' traceless Hermitian (Z'^2 =
// zeta2 I, zeta2 = dz^2 + |zc|^2 real) and the alternating plan coefficients
// a_k = (-i)^k J_k(beta) (chebyshev.py:213-214; exact zeros in the other
// component, checked on the host), the reference's Clenshaw recurrence
// (chebyshev.py:298-303) on coefficient pairs b_j = A_j I + B_j Z' keeps A_j
// purely real / imaginary by the parity of j and B_j by the parity of j + 1,
// so it runs on ONE real number per pair entry:
//     A_j = c_j + zeta2 B_{j+1} - beta_j A_{j+2},   B_j = A_{j+1} - beta_j B_{j+2}
// (c_j = the nonzero component of a_j, beta_0 = 2, else 1), and
//     U = A_0 I + i b_0 Z' = [[p, q], [-conj(q), conj(p)]],
//     p = (A_0, b_0 dz),  q = (-b_0 Im zc, b_0 Re zc)      (Z'01 = zc)
// — the same U, entry for entry, as lane_small_kernel<2,1>'s real pair path
// (the dropped terms are exact zeros there).  Such matrices form the
// quaternion algebra: closed under products, so every running product
// V = U_k ... U_0 is [[v0, v1], [-conj(v1), conj(v0)]] and is carried as
// (v0, v1): 4 doubles, 16 FP64 operations per product instead of 32, and the
// row-0 entries are computed with exactly the reference's entry formula
// (row 0 of U times V, same operand order).
//
// Per slice (midpoint, N controls, m compiled in): 3N FMA of assembly, 3 for
// zeta2, ~2(m-1) for Clenshaw, 3 MUL for U, 16 for V <- U V: ~35 FP64
// instructions at the qubit's N = 2, m = 3 — below the 16 B amplitude row's
// share of HBM bandwidth, so a call streams the table at HBM speed.
//
// Structure: one CTA per SM (up to 1024 threads), each thread a lane of
// contiguous slices whose amplitude rows stream DS slices ahead through a
// per-thread cp.async ring in shared memory (~192 KB in flight per SM); ordered warp-shuffle products (later lanes on the
// left), the CTA's warp products by warp 0, then the last CTA to arrive
// (one acq_rel ticket) multiplies the <= 148 CTA products in time order and
// writes the d x d result: the whole equiprop is one launch.
// Amplitude bounds (|c| <= 1, NaN) are accumulated into a predicate; a lane
// that saw an offender rescans its own rows for the first one (row-major)
// and records it in the epoch slot (SliceJob::viol) — no branch per slice.
//
// u(2) systems (complex128 d = 2 terms with a trace part: Z = z0 I + Z')
// run on the same lanes with the algebra as a template parameter (QuatAlg /
// U2Alg): complex Clenshaw pairs (lane_small_kernel<2,1>'s d = 2 sequence)
// for two slices in lockstep, 2 x 2 complex running products (32 FP64
// operations), the same ordered CTA tree and fused tail.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "internal.h"

namespace sp {

template <class R>
struct QuatT {  // [[a, b], [-conj(b), conj(a)]]
  R ar, ai, br, bi;
};
using Quat = QuatT<double>;

// tools only: %globaltimer at phase k, min / max over the CTAs (thread 0)
__device__ __forceinline__ void su2_mark(const Su2Job& job, int k) {
  if (job.prof != nullptr && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMin(job.prof + 2 * k, t);
    atomicMax(job.prof + 2 * k + 1, t);
  }
}

template <class R = double>
__device__ __forceinline__ QuatT<R> quat_identity() {
  return QuatT<R>{R(1), R(0), R(0), R(0)};
}

// P Q (P later in time, on the left): row 0 of the 2 x 2 complex product
// with Q10 = -conj(Q.b), Q11 = conj(Q.a), summed in mat_mul's order
template <class R>
__device__ __forceinline__ QuatT<R> quat_mul(const QuatT<R>& P, const QuatT<R>& Q) {
  QuatT<R> Rs;
  R re = P.ar * Q.ar;
  re = fma(-P.ai, Q.ai, re);
  re = fma(P.br, -Q.br, re);
  re = fma(-P.bi, Q.bi, re);
  R im = P.ar * Q.ai;
  im = fma(P.ai, Q.ar, im);
  im = fma(P.br, Q.bi, im);
  im = fma(P.bi, -Q.br, im);
  Rs.ar = re;
  Rs.ai = im;
  re = P.ar * Q.br;
  re = fma(-P.ai, Q.bi, re);
  re = fma(P.br, Q.ar, re);
  re = fma(-P.bi, -Q.ai, re);
  im = P.ar * Q.bi;
  im = fma(P.ai, Q.br, im);
  im = fma(P.br, -Q.ai, im);
  im = fma(P.bi, Q.ar, im);
  Rs.br = re;
  Rs.bi = im;
  return Rs;
}

template <class R>
__device__ __forceinline__ QuatT<R> quat_shfl_down(const QuatT<R>& q, int k) {
  return QuatT<R>{__shfl_down_sync(0xffffffffu, q.ar, k), __shfl_down_sync(0xffffffffu, q.ai, k),
              __shfl_down_sync(0xffffffffu, q.br, k), __shfl_down_sync(0xffffffffu, q.bi, k)};
}

// lane 0 ends with M_{31} ... M_1 M_0 (later lanes on the left)
template <class R>
__device__ __forceinline__ void quat_warp_product(QuatT<R>& q) {
#pragma unroll
  for (int k = 1; k < 32; k <<= 1) q = quat_mul(quat_shfl_down(q, k), q);
}
// the same over the first `width` lanes only (lanes >= width hold identity):
// log2(width) levels
template <class R>
__device__ __forceinline__ void quat_warp_product(QuatT<R>& q, int width) {
  for (int k = 1; k < width; k <<= 1) q = quat_mul(quat_shfl_down(q, k), q);
}

// lane mode: the running product's initial value and per-slice output
template <class R>
__device__ __forceinline__ QuatT<R> su2_vinit(const Su2Job& job, int64_t lane) {
  if (job.vinit == nullptr) return quat_identity<R>();
  const double2* e = reinterpret_cast<const double2*>(job.vinit) + 4 * lane;
  const double2 a = e[0], b = e[1];  // row 0: (a, b); row 1 is (-conj b, conj a)
  return QuatT<R>{(R)a.x, (R)a.y, (R)b.x, (R)b.y};
}
template <class R>
__device__ __forceinline__ void su2_store(void* base, int64_t idx, const QuatT<R>& q) {
  // two 256-bit stores (sm_100 STG.256) per 64-byte 2 x 2 complex128 matrix
  double* o = reinterpret_cast<double*>(base) + 8 * idx;
  if (reinterpret_cast<uintptr_t>(o) & 31u) {  // caller's buffer not 32-byte aligned
    double2* q2 = reinterpret_cast<double2*>(o);
    q2[0] = make_double2(q.ar, q.ai);
    q2[1] = make_double2(q.br, q.bi);
    q2[2] = make_double2(-(double)q.br, q.bi);
    q2[3] = make_double2(q.ar, -(double)q.ai);
    return;
  }
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(o), "d"((double)q.ar),
               "d"((double)q.ai), "d"((double)q.br), "d"((double)q.bi)
               : "memory");
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(o + 4), "d"(-(double)q.br),
               "d"((double)q.bi), "d"((double)q.ar), "d"(-(double)q.ai)
               : "memory");
}

// ---------------------------------------------------------------------------
// u(2) systems (terms with a trace part, lane_u2 kernels): the slice
// propagators are general 2 x 2 complex matrices (no quaternion closure), the
// running products too: 8 values, 32 FP64 operations per product.
// ---------------------------------------------------------------------------
template <class R>
struct M2T {  // row-major: m[0..1] U00, m[2..3] U01, m[4..5] U10, m[6..7] U11 (re, im)
  R m[8];
};

// P Q (P later in time, on the left), in lane_small_kernel's summation order
template <class R>
__device__ __forceinline__ M2T<R> m2_mul(const M2T<R>& P, const M2T<R>& Q) {
  M2T<R> o;
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const R* p0 = &P.m[4 * r];
      const R* p1 = &P.m[4 * r + 2];
      const R* q0 = &Q.m[2 * c];
      const R* q1 = &Q.m[4 + 2 * c];
      R re = p0[0] * q0[0];
      re = fma(-p0[1], q0[1], re);
      re = fma(p1[0], q1[0], re);
      re = fma(-p1[1], q1[1], re);
      R im = p0[0] * q0[1];
      im = fma(p0[1], q0[0], im);
      im = fma(p1[0], q1[1], im);
      im = fma(p1[1], q1[0], im);
      o.m[4 * r + 2 * c] = re;
      o.m[4 * r + 2 * c + 1] = im;
    }
  return o;
}

// |v| <= 1 fails (also for NaN): accumulated without a branch
__device__ __forceinline__ bool amp_bad(double v) { return !(fabs(v) <= 1.0); }

template <int MODE, int NCC, class R = double, bool U2 = false>
struct Su2Shape {
  // doubles read per slice: midpoint one row; three-point the rows 2s+1, 2s+2
  // (row 2s is the previous slice's last row)
  static constexpr int K = MODE == SP_MODE_MIDPOINT ? NCC : 2 * NCC;
  static constexpr bool VEC = (NCC % 2) == 0;  // 16-byte rows (host-checked alignment)
  static constexpr int UNIT = VEC ? 16 : 8;    // bytes per cp.async
  static constexpr int CP = K * 8 / UNIT;      // cp.async per slice
  // threads per CTA: 1024 (64 registers) except the three-point forms, whose
  // float64 weights need more registers (with >= 3 controls, or next to the
  // float32 working set of complex64 contexts), and the u(2) forms (complex
  // Clenshaw pairs, 2 x 2 complex products: 128 registers)
  static constexpr bool F32 = sizeof(R) == 4;
  static constexpr int TPB = U2 ? (MODE != SP_MODE_MIDPOINT && NCC >= 3 ? 256 : 512)
                             : MODE == SP_MODE_MIDPOINT ? 1024
                             : NCC >= 3 ? (F32 ? 256 : 512)
                                        : (F32 ? 512 : 1024);
  // shared-memory ring: DS slices per thread in flight (<= 192 KB per CTA:
  // the bytes in flight an SM needs to stream HBM at speed)
  static constexpr int DS_RAW = (192 * 1024) / (TPB * K * 8);
  static constexpr int DS = DS_RAW < 2 ? 2 : (DS_RAW > 16 ? 16 : DS_RAW);
  static constexpr int SMEM_PER_THREAD = DS * K * 8;
};

__device__ __forceinline__ unsigned su2_smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
template <int UNIT>
__device__ __forceinline__ void su2_cp_async(void* dst, const void* src) {
  if constexpr (UNIT == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su2_smem_u32(dst)),
                 "l"(src)
                 : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(su2_smem_u32(dst)), "l"(src)
                 : "memory");
}
__device__ __forceinline__ void su2_cp_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void su2_cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// first offender of rows [r0, r1] (row-major index), ~0 if none
__device__ __noinline__ unsigned long long su2_first_bad(const double* amps, int64_t r0,
                                                         int64_t r1, int N) {
  for (int64_t r = r0; r <= r1; ++r)
    for (int c = 0; c < N; ++c)
      if (amp_bad(amps[r * N + c])) return (unsigned long long)(r * N + c);
  return ~0ull;
}

// Slice weights (hamiltonian.py:199-205, magnus.py:88-106) from the slice's
// amplitude samples `cur` (and, for the three-point modes, the carried row
// 2s in r1), and Z = sum_t w_t z_t (2X factor folded into the per-term
// components on the host): dz, zx, zy the traceless part, z0 (TR) the trace
// part.  (complex64 contexts: the float64 weights and the terms cast to the
// working precision, linalg.py:273-274, everything after in float32.)
template <class R, int MODE, int NCC, bool TR>
__device__ __forceinline__ void su2_weights(const Su2Job& job, const double* cur,
                                            double (&r1)[NCC], R& z0, R& dz, R& zx, R& zy) {
  constexpr int T = MODE == SP_MODE_MAGNUS ? 1 + 2 * NCC + NCC * (NCC - 1) / 2 : 1 + NCC;
  static_assert(T <= SU2_MAX_TERMS, "too many su(2) terms");
  z0 = TR ? (R)job.ta[0] : R(0);
  dz = (R)job.tz[0][0];
  zx = (R)job.tz[0][1];
  zy = (R)job.tz[0][2];
  auto add = [&](int t, double w64) {
    const R w = (R)w64;
    if constexpr (TR) z0 = fma(w, (R)job.ta[t], z0);
    dz = fma(w, (R)job.tz[t][0], dz);
    zx = fma(w, (R)job.tz[t][1], zx);
    zy = fma(w, (R)job.tz[t][2], zy);
  };
  if constexpr (MODE == SP_MODE_MIDPOINT) {
#pragma unroll
    for (int q = 0; q < NCC; ++q) add(1 + q, cur[q]);
  } else {
    const double* c2 = cur;        // row 2s + 1
    const double* c3 = cur + NCC;  // row 2s + 2
#pragma unroll
    for (int q = 0; q < NCC; ++q) add(1 + q, (r1[q] + 4.0 * c2[q] + c3[q]) / 6.0);
    if constexpr (MODE == SP_MODE_MAGNUS) {
#pragma unroll
      for (int q = 0; q < NCC; ++q) add(1 + NCC + q, job.dt6 * (c3[q] - r1[q]));
      int t = 1 + 2 * NCC;
#pragma unroll
      for (int a = 0; a < NCC; ++a)
#pragma unroll
        for (int b = a + 1; b < NCC; ++b) add(t++, job.dt6 * (r1[a] * c3[b] - c3[a] * r1[b]));
    }
#pragma unroll
    for (int q = 0; q < NCC; ++q) r1[q] = c3[q];
  }
}

// One su(2) slice's propagator: Z' = sum_t w_t tz_t, the real Clenshaw
// pairs, U = A I + i B Z'.
template <class R, int MODE, int NCC, int MC>
__device__ __forceinline__ QuatT<R> su2_u(const Su2Job& job, int m, const double* cur,
                                          double (&r1)[NCC]) {
  R z0, dz, zx, zy;
  su2_weights<R, MODE, NCC, false>(job, cur, r1, z0, dz, zx, zy);
  const R zeta2 = fma(dz, dz, fma(zx, zx, zy * zy));
  // ---- real Clenshaw pairs; the j = m - 1 step peeled (B_{m+1} = 0)
  R A = (R)job.cr[m - 1], B = (R)job.cr[m], oA = (R)job.cr[m], oB = R(0);
  constexpr int MU = MC > 0 ? MC : 1;
#pragma unroll MU
  for (int jj = m - 2; jj >= 0; --jj) {
    const R beta = (jj == 0) ? R(2) : R(1);
    const R nA = (R)job.cr[jj] + fma(zeta2, B, -beta * oA);
    const R nB = A - beta * oB;
    oA = A;
    oB = B;
    A = nA;
    B = nB;
  }
  return QuatT<R>{A, B * dz, -(B * zy), B * zx};
}

// u(2) slice propagators, K slices in lockstep (independent dependency
// chains for the in-order issue: one Clenshaw loop advances all K): Z = z0 I
// + Z' (Z'^2 = zeta2 I), the complex Clenshaw pairs b_j = a_j I + b_j' Z' of
// lane_small_kernel<2,1>'s d = 2 path (chebyshev.py:298-303 on the
// 2-dimensional algebra; first step peeled), U = a I + b Z' entry by entry.
template <class R, int MODE, int NCC, int MC, int K>
__device__ __forceinline__ void u2_u_multi(const Su2Job& job, int m, const double* const (&cur)[K],
                                           double (&r1)[NCC], M2T<R> (&U)[K]) {
  R z0[K], dz[K], zx[K], zy[K], zeta2[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    su2_weights<R, MODE, NCC, true>(job, cur[k], r1, z0[k], dz[k], zx[k], zy[k]);
    zeta2[k] = fma(dz[k], dz[k], fma(zx[k], zx[k], zy[k] * zy[k]));
  }
  auto cre = [&](int j) { return (R)job.cz[2 * j]; };
  auto cim = [&](int j) { return (R)job.cz[2 * j + 1]; };
  R car[K], cai[K], cbr[K], cbi[K], oar[K], oai[K], obr[K], obi[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    car[k] = cre(m);
    cai[k] = cim(m);
    cbr[k] = cbi[k] = oar[k] = oai[k] = obr[k] = obi[k] = R(0);
    if (m >= 1) {
      oar[k] = car[k];
      oai[k] = cai[k];
      cbr[k] = car[k];
      cbi[k] = cai[k];
      car[k] = cre(m - 1) + z0[k] * oar[k];
      cai[k] = cim(m - 1) + z0[k] * oai[k];
    }
  }
  constexpr int MU = MC > 0 ? MC : 1;
#pragma unroll MU
  for (int jj = m - 2; jj >= 0; --jj) {
    const R beta = (jj == 0) ? R(2) : R(1);
    const R ar = cre(jj), ai = cim(jj);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const R nar = ar + fma(z0[k], car[k], fma(zeta2[k], cbr[k], -beta * oar[k]));
      const R nai = ai + fma(z0[k], cai[k], fma(zeta2[k], cbi[k], -beta * oai[k]));
      const R nbr = car[k] + fma(z0[k], cbr[k], -beta * obr[k]);
      const R nbi = cai[k] + fma(z0[k], cbi[k], -beta * obi[k]);
      oar[k] = car[k];
      oai[k] = cai[k];
      obr[k] = cbr[k];
      obi[k] = cbi[k];
      car[k] = nar;
      cai[k] = nai;
      cbr[k] = nbr;
      cbi[k] = nbi;
    }
  }
#pragma unroll
  for (int k = 0; k < K; ++k) {
    U[k].m[0] = fma(cbr[k], dz[k], car[k]);
    U[k].m[1] = fma(cbi[k], dz[k], cai[k]);
    U[k].m[2] = cbr[k] * zx[k] - cbi[k] * zy[k];
    U[k].m[3] = cbr[k] * zy[k] + cbi[k] * zx[k];
    U[k].m[4] = cbr[k] * zx[k] + cbi[k] * zy[k];
    U[k].m[5] = cbi[k] * zx[k] - cbr[k] * zy[k];
    U[k].m[6] = fma(-cbr[k], dz[k], car[k]);
    U[k].m[7] = fma(-cbi[k], dz[k], cai[k]);
  }
}
template <class R, int MODE, int NCC, int MC>
__device__ __forceinline__ M2T<R> u2_u(const Su2Job& job, int m, const double* cur,
                                       double (&r1)[NCC]) {
  const double* const c[1] = {cur};
  M2T<R> U[1];
  u2_u_multi<R, MODE, NCC, MC, 1>(job, m, c, r1, U);
  return U[0];
}

// The two algebras behind one set of lane kernels: the element type, the
// product (later on the left), shuffles, the per-slice propagator, the
// complex128 2 x 2 stores / loads of lane mode, the CTA-product slots.
template <class R_>
struct QuatAlg {
  using R = R_;
  using E = QuatT<R>;
  static constexpr bool PAIRS = false;  // TMA round: all C propagators first (ILP)
  __device__ static E one() { return quat_identity<R>(); }
  __device__ static E mul(const E& a, const E& b) { return quat_mul(a, b); }
  __device__ static E shfl(const E& q, int k) { return quat_shfl_down(q, k); }
  template <int MODE, int NCC, int MC>
  __device__ static E slice(const Su2Job& job, int m, const double* cur, double (&r1)[NCC]) {
    return su2_u<R, MODE, NCC, MC>(job, m, cur, r1);
  }
  __device__ static void store(void* base, int64_t idx, const E& q) { su2_store(base, idx, q); }
  __device__ static E vinit(const Su2Job& job, int64_t lane) { return su2_vinit<R>(job, lane); }
  __device__ static void cta_put(void* p, int i, const E& q) { reinterpret_cast<E*>(p)[i] = q; }
  __device__ static E cta_get(const void* p, int i) {
    if constexpr (sizeof(R) == 8) {
      const double2* cp = reinterpret_cast<const double2*>(p);
      const double2 a = __ldcg(cp + 2 * i), b = __ldcg(cp + 2 * i + 1);
      return E{a.x, a.y, b.x, b.y};
    } else {
      const float4 a = __ldcg(reinterpret_cast<const float4*>(p) + i);
      return E{a.x, a.y, a.z, a.w};
    }
  }
  // [[a, b], [-conj(b), conj(a)]] row-major
  __device__ static void entries(const E& M, R (&e)[8]) {
    e[0] = M.ar; e[1] = M.ai; e[2] = M.br; e[3] = M.bi;
    e[4] = -M.br; e[5] = M.bi; e[6] = M.ar; e[7] = -M.ai;
  }
};

template <class R_>
struct U2Alg {
  using R = R_;
  using E = M2T<R>;
  static constexpr bool PAIRS = true;  // TMA round: propagators two at a time (registers)
  __device__ static E one() { return E{{R(1), R(0), R(0), R(0), R(0), R(0), R(1), R(0)}}; }
  __device__ static E mul(const E& a, const E& b) { return m2_mul(a, b); }
  __device__ static E shfl(const E& q, int k) {
    E o;
#pragma unroll
    for (int i = 0; i < 8; ++i) o.m[i] = __shfl_down_sync(0xffffffffu, q.m[i], k);
    return o;
  }
  template <int MODE, int NCC, int MC>
  __device__ static E slice(const Su2Job& job, int m, const double* cur, double (&r1)[NCC]) {
    return u2_u<R, MODE, NCC, MC>(job, m, cur, r1);
  }
  // two consecutive slices in lockstep (TMA rounds, cp.async ring pairs)
  template <int MODE, int NCC, int MC>
  __device__ static void slice2(const Su2Job& job, int m, const double* c0, const double* c1,
                                double (&r1)[NCC], E& u0, E& u1) {
    const double* const c[2] = {c0, c1};
    E U[2];
    u2_u_multi<R, MODE, NCC, MC, 2>(job, m, c, r1, U);
    u0 = U[0];
    u1 = U[1];
  }
  __device__ static void store(void* base, int64_t idx, const E& q) {
    double* o = reinterpret_cast<double*>(base) + 8 * idx;
    if (reinterpret_cast<uintptr_t>(o) & 31u) {
#pragma unroll
      for (int i = 0; i < 8; ++i) o[i] = (double)q.m[i];
      return;
    }
    asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(o), "d"((double)q.m[0]),
                 "d"((double)q.m[1]), "d"((double)q.m[2]), "d"((double)q.m[3])
                 : "memory");
    asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(o + 4), "d"((double)q.m[4]),
                 "d"((double)q.m[5]), "d"((double)q.m[6]), "d"((double)q.m[7])
                 : "memory");
  }
  __device__ static E vinit(const Su2Job& job, int64_t lane) {
    if (job.vinit == nullptr) return one();
    const double* e = reinterpret_cast<const double*>(job.vinit) + 8 * lane;
    E o;
#pragma unroll
    for (int i = 0; i < 8; ++i) o.m[i] = (R)e[i];
    return o;
  }
  __device__ static void cta_put(void* p, int i, const E& q) { reinterpret_cast<E*>(p)[i] = q; }
  __device__ static E cta_get(const void* p, int i) {
    E o;
    if constexpr (sizeof(R) == 8) {
      const double2* cp = reinterpret_cast<const double2*>(p) + 4 * i;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const double2 a = __ldcg(cp + k);
        o.m[2 * k] = a.x;
        o.m[2 * k + 1] = a.y;
      }
    } else {
      const float4* cp = reinterpret_cast<const float4*>(p) + 2 * i;
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const float4 a = __ldcg(cp + k);
        o.m[4 * k] = a.x;
        o.m[4 * k + 1] = a.y;
        o.m[4 * k + 2] = a.z;
        o.m[4 * k + 3] = a.w;
      }
    }
    return o;
  }
  __device__ static void entries(const E& M, R (&e)[8]) {
#pragma unroll
    for (int i = 0; i < 8; ++i) e[i] = M.m[i];
  }
};

template <class R, bool U2>
using Su2AlgT = typename std::conditional<U2, U2Alg<R>, QuatAlg<R>>::type;

// lane 0 ends with M_{31} ... M_1 M_0 (later lanes on the left); the width
// form over the first `width` lanes only (the others hold identity)
template <class A>
__device__ __forceinline__ void alg_warp_product(typename A::E& q) {
#pragma unroll
  for (int k = 1; k < 32; k <<= 1) q = A::mul(A::shfl(q, k), q);
}
template <class A>
__device__ __forceinline__ void alg_warp_product(typename A::E& q, int width) {
  for (int k = 1; k < width; k <<= 1) q = A::mul(A::shfl(q, k), q);
}

// After the lane loops: the lane's first amplitude offender (rare path; rows
// [r0, rl] of the table), the ordered CTA product, the arrival ticket and, in
// the last CTA, the ordered product of the CTA products and the d x d result.
template <class A, int NCC, bool PFX = false>
__device__ __forceinline__ void su2_finish(const Su2Job& job, typename A::E V, bool bad,
                                           int64_t r0, int64_t rl) {
  using R = typename A::R;
  using E = typename A::E;
  if (bad && job.viol) {
    const unsigned long long v = su2_first_bad(job.amps, r0, rl, NCC);
    // fused calls: the epoch slot (SliceJob::viol); multi-launch calls: slot 2
    unsigned long long* slot =
        job.viol_epoch ? job.viol + (__ldcg(job.viol + 3) & 1ull) : job.viol + 2;
    atomicMin(slot, v);
  }
  if (PFX && job.lane_out != nullptr) {  // lane mode: the lane product, no tree
    A::store(job.lane_out, (int64_t)blockIdx.x * blockDim.x + threadIdx.x, V);
    return;
  }
  // ---- ordered products: warps, then the CTA's warps (warp 0)
  __shared__ E wq[32];
  __shared__ bool last;
  const int ln = threadIdx.x & 31, wp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  auto cta_product = [&](E& q) {  // result in thread 0
    alg_warp_product<A>(q);
    if (ln == 0) wq[wp] = q;
    __syncthreads();
    if (wp == 0) {
      q = ln < nw ? wq[ln] : A::one();
      alg_warp_product<A>(q, nw);  // only the levels the nw warp products need
    }
    __syncthreads();
  };
  su2_mark(job, 2);
  cta_product(V);
  su2_mark(job, 3);
  if (threadIdx.x == 0) {
    A::cta_put(job.cta_out, blockIdx.x, V);
    unsigned old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;"
                 : "=r"(old)
                 : "l"(job.ctr)
                 : "memory");
    last = (old == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return;
  su2_mark(job, 4);
  // ---- fused tail: every thread folds a contiguous run of CTA products
  // (later on the left), then one CTA-wide ordered product
  const int G = (int)gridDim.x, per = (G + (int)blockDim.x - 1) / (int)blockDim.x;
  const int i0 = min(G, (int)threadIdx.x * per), i1 = min(G, i0 + per);
  E M = A::one();
  for (int i = i0; i < i1; ++i) M = A::mul(A::cta_get(job.cta_out, i), M);
  cta_product(M);
  if (threadIdx.x == 0) {
    // the 2 x 2 result, row-major, in the output dtype
    R e[8];
    A::entries(M, e);
    if (job.to_fp32) {
      float* o = reinterpret_cast<float*>(job.out);
#pragma unroll
      for (int i = 0; i < 8; ++i) o[i] = (float)e[i];
    } else {
      double* o = reinterpret_cast<double*>(job.out);
#pragma unroll
      for (int i = 0; i < 8; ++i) o[i] = (double)e[i];
    }
    su2_mark(job, 5);
    *job.ctr = 0;  // ready for the next launch
    if (job.viol) {  // rotate the violation slots (SliceJob::viol)
      const unsigned long long ep = __ldcg(job.viol + 3);
      job.viol[(ep + 1) & 1ull] = ~0ull;
      job.viol[2] = ~0ull;
      job.viol[3] = ep + 1;
    }
  }
}

// ---------------------------------------------------------------------------
// General form: every mode and control count.  Lane = contiguous slices
// [lane n / lanes, (lane + 1) n / lanes); the rows stream through a
// per-thread cp.async ring in shared memory.
// ---------------------------------------------------------------------------
template <int MODE, int NCC, int MC, class R = double, bool PFX = false, bool U2 = false>
__global__ void __launch_bounds__(Su2Shape<MODE, NCC, R, U2>::TPB, 1)
    lane_su2_kernel(const Su2Job job) {
  using S = Su2Shape<MODE, NCC, R, U2>;
  using A = Su2AlgT<R, U2>;
  constexpr int K = S::K, DS = S::DS, CP = S::CP, UNIT = S::UNIT;
  extern __shared__ __align__(16) unsigned char su2_ring[];
  const int m = MC > 0 ? MC : job.m;
  const int lane = blockIdx.x * blockDim.x + threadIdx.x;
  const int lanes = gridDim.x * blockDim.x;
  const int64_t s0 = (int64_t)lane * job.n_slices / lanes;
  const int64_t s1 = ((int64_t)lane + 1) * job.n_slices / lanes;
  const int cnt = (int)(s1 - s0);

  // PFX: lane mode (initial products, per-slice running products, lane
  // products instead of the fused tail)
  typename A::E V = PFX ? A::vinit(job, lane) : A::one();
  bool bad = false;
  // first unit of this lane: row s0 (midpoint) or rows 2 s0 + 1, 2 s0 + 2
  const unsigned char* unit0 = reinterpret_cast<const unsigned char*>(
      job.amps + (MODE == SP_MODE_MIDPOINT ? s0 * NCC : (2 * s0 + 1) * NCC));
  double r1[NCC];  // three-point: row 2s of the current slice
  if constexpr (MODE != SP_MODE_MIDPOINT) {
    if (cnt > 0) {
#pragma unroll
      for (int q = 0; q < NCC; ++q) {
        r1[q] = __ldg(job.amps + 2 * s0 * NCC + q);
        bad |= amp_bad(r1[q]);
      }
    }
  }
  // ring slot j, copy q of this thread: [slot][copy][thread] x UNIT bytes
  // (a warp's copies and reads are contiguous: no bank conflicts)
  const int nt = blockDim.x;
  auto slot_ptr = [&](int j, int q) {
    return su2_ring + ((size_t)(j * CP + q) * nt + threadIdx.x) * UNIT;
  };
  auto issue = [&](int k, int j) {  // unit k of the lane into slot j
    if (k < cnt) {
#pragma unroll
      for (int q = 0; q < CP; ++q)
        su2_cp_async<UNIT>(slot_ptr(j, q), unit0 + (size_t)k * K * 8 + q * UNIT);
    }
    su2_cp_commit();
  };
#pragma unroll
  for (int j = 0; j < DS - 1; ++j) issue(j, j);

  double prev[K];  // u(2): the held row of a slice pair
  bool held = false;
  for (int k0 = 0; k0 < cnt; k0 += DS) {
#pragma unroll
    for (int j = 0; j < DS; ++j) {
      if (k0 + j < cnt) {
        issue(k0 + j + DS - 1, (j + DS - 1) % DS);
        su2_cp_wait<DS - 1>();
        double cur[K];
#pragma unroll
        for (int q = 0; q < CP; ++q) {
          if constexpr (UNIT == 16) {
            const double2 t = *reinterpret_cast<const double2*>(slot_ptr(j, q));
            cur[2 * q] = t.x;
            cur[2 * q + 1] = t.y;
          } else {
            cur[q] = *reinterpret_cast<const double*>(slot_ptr(j, q));
          }
        }
#pragma unroll
        for (int q = 0; q < K; ++q) bad |= amp_bad(cur[q]);
        if constexpr (A::PAIRS) {
          // u(2): a slice's row is held until the next one arrives, then the
          // two Clenshaw recurrences run in lockstep (two dependency chains)
          if (!held) {
#pragma unroll
            for (int q = 0; q < K; ++q) prev[q] = cur[q];
            held = true;
          } else {
            typename A::E u0, u1;
            A::template slice2<MODE, NCC, MC>(job, m, prev, cur, r1, u0, u1);
            if (PFX && job.prefix_out != nullptr) {
              V = A::mul(u0, V);
              A::store(job.prefix_out, s0 + k0 + j - 1, V);
              V = A::mul(u1, V);
              A::store(job.prefix_out, s0 + k0 + j, V);
            } else {
              V = A::mul(A::mul(u1, u0), V);
            }
            held = false;
          }
        } else {
          V = A::mul(A::template slice<MODE, NCC, MC>(job, m, cur, r1), V);
          if (PFX && job.prefix_out != nullptr) A::store(job.prefix_out, s0 + k0 + j, V);
        }
      }
    }
  }
  if constexpr (A::PAIRS) {
    if (held) {  // odd slice count: the last one alone
      V = A::mul(A::template slice<MODE, NCC, MC>(job, m, prev, r1), V);
      if (PFX && job.prefix_out != nullptr) A::store(job.prefix_out, s1 - 1, V);
    }
  }
  su2_finish<A, NCC, PFX>(job, V, bad, MODE == SP_MODE_MIDPOINT ? s0 : 2 * s0,
                          MODE == SP_MODE_MIDPOINT ? s1 - 1 : 2 * s1);
}

// ---------------------------------------------------------------------------
// TMA form: midpoint, NCC in {2, 4} (the driven qubit).  Every lane owns L
// consecutive slices (the last used lane fewer); the table is a 2-D tensor
// [lane][L x NCC doubles] and one cp.async.bulk.tensor per warp and round
// brings the next C rows of the warp's 32 lanes (32 x C x NCC x 8 bytes,
// 128/64-byte swizzled so each thread's row reads are bank-conflict free)
// into the warp's ring of NST stages, completion on the stage's mbarrier.
// The partial last lane reads its rows from global memory directly.
// ---------------------------------------------------------------------------
template <int NCC, int C>
struct Su2Tma {
  static constexpr int ROWB = NCC * 8;       // bytes per amplitude row
  static constexpr int LROWB = C * ROWB;     // bytes per lane per round (64 or 128)
  static_assert(LROWB == 64 || LROWB == 128, "swizzle span");
  static_assert(C % 2 == 0, "rounds are taken in slice pairs");
  static constexpr int STAGE = 32 * LROWB;   // bytes per warp per stage
  static constexpr int TPB = LROWB == 128 ? 512 : 1024;
  static constexpr int NST = (192 * 1024) / ((TPB / 32) * STAGE);  // stages per warp
  static constexpr int SMEM = (TPB / 32) * NST * STAGE + 1024;     // + alignment slack
};

__device__ __forceinline__ void su2_mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su2_smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void su2_mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su2_smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void su2_mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(su2_smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void su2_tma_2d(void* dst, const void* tmap, int x, int y,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(su2_smem_u32(dst)),
      "l"(tmap), "r"(x), "r"(y), "r"(su2_smem_u32(bar))
      : "memory");
}

template <int NCC, int MC, int C, class R = double, bool PFX = false, bool U2 = false>
__global__ void __launch_bounds__(Su2Tma<NCC, C>::TPB, 1)
    lane_su2_tma_kernel(const Su2Job job, const __grid_constant__ CUtensorMap tmap,
                        const int64_t L) {
  using G = Su2Tma<NCC, C>;
  using A = Su2AlgT<R, U2>;
  using E = typename A::E;
  constexpr int NST = G::NST, STAGE = G::STAGE, LROWB = G::LROWB, ROWB = G::ROWB;
  extern __shared__ unsigned char su2_tma_raw[];
  __shared__ __align__(8) uint64_t bars[(G::TPB / 32) * NST];
  // 1024-byte aligned ring (the swizzle pattern follows absolute address
  // bits); offsets from the shared array keep every access in the shared
  // window (LDS, not generic loads)
  const unsigned raw_u32 = su2_smem_u32(su2_tma_raw);
  unsigned char* base = su2_tma_raw + (((raw_u32 + 1023u) & ~1023u) - raw_u32);
  const int m = MC > 0 ? MC : job.m;
  const int ln = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const int64_t lane = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t wlane0 = lane - ln;  // first lane of the warp
  const int64_t n = job.n_slices;
  const int64_t s0 = min(n, lane * L), s1 = min(n, s0 + L);
  const int cnt = (int)(s1 - s0);
  const int64_t full = n / L;          // lanes with exactly L slices (tensor rows)
  const bool direct = lane == full;    // the partial last lane: global loads
  // rounds the warp needs: its first lane has the most slices
  const int64_t wcnt = min(L, max((int64_t)0, n - wlane0 * L));
  const int rounds = (int)((wcnt + C - 1) / C);
  unsigned char* ring = base + (size_t)wp * NST * STAGE;
  uint64_t* wb = bars + wp * NST;
  const bool tma_warp = wlane0 < full;  // at least one tensor row in the box
  su2_mark(job, 0);
  if (ln == 0 && tma_warp) {
#pragma unroll
    for (int s = 0; s < NST; ++s) su2_mbar_init(wb + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
#pragma unroll
    for (int s = 0; s < NST; ++s)
      if (s < rounds) {
        su2_mbar_expect_tx(wb + s, STAGE);
        su2_tma_2d(ring + s * STAGE, &tmap, s * C * NCC, (int)wlane0, wb + s);
      }
  }
  __syncwarp();

  E V = PFX ? A::vinit(job, lane) : A::one();
  bool bad = false;
  double r1[NCC];
  const int sw = LROWB == 128 ? (ln & 7) : ((ln >> 1) & 3);  // swizzle of this lane's row
  for (int r = 0; r < rounds; ++r) {
    const int s = r % NST;
    if (tma_warp) su2_mbar_wait(wb + s, (unsigned)((r / NST) & 1));
    if (r == 0) su2_mark(job, 1);
    const unsigned row = su2_smem_u32(ring + s * STAGE) + ln * LROWB;
    auto smem_row = [&](int k, double (&cur)[NCC]) {
#pragma unroll
      for (int q = 0; q < NCC / 2; ++q) {
        const int chunk = (k * ROWB) / 16 + q;
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];"
                     : "=d"(cur[2 * q]), "=d"(cur[2 * q + 1])
                     : "r"(row + ((chunk ^ sw) << 4)));
      }
    };
    if (!direct && (r + 1) * C <= cnt) {
      // a whole round: the slice propagators are independent (ILP), the
      // running product takes them in adjacent pairs, later on the left —
      // all C first (quaternions) or two at a time (u(2): registers)
      auto u_of = [&](int k) {
        double cur[NCC];
        smem_row(k, cur);
#pragma unroll
        for (int q = 0; q < NCC; ++q) bad |= amp_bad(cur[q]);
        return A::template slice<SP_MODE_MIDPOINT, NCC, MC>(job, m, cur, r1);
      };
      if (PFX && job.prefix_out != nullptr) {  // every slice's running product is written
#pragma unroll
        for (int k = 0; k < C; ++k) {
          V = A::mul(u_of(k), V);
          A::store(job.prefix_out, s0 + r * C + k, V);
        }
      } else if constexpr (A::PAIRS) {
#pragma unroll
        for (int k = 0; k < C; k += 2) {
          double c0[NCC], c1[NCC];
          smem_row(k, c0);
          smem_row(k + 1, c1);
#pragma unroll
          for (int q = 0; q < NCC; ++q) bad |= amp_bad(c0[q]) | amp_bad(c1[q]);
          E u0, u1;
          A::template slice2<SP_MODE_MIDPOINT, NCC, MC>(job, m, c0, c1, r1, u0, u1);
          V = A::mul(A::mul(u1, u0), V);
        }
      } else {
        E U[C];
#pragma unroll
        for (int k = 0; k < C; ++k) U[k] = u_of(k);
#pragma unroll
        for (int k = 0; k < C; k += 2) V = A::mul(A::mul(U[k + 1], U[k]), V);
      }
    } else {
#pragma unroll
      for (int k = 0; k < C; ++k) {
        const int kk = r * C + k;
        if (kk < cnt) {
          double cur[NCC];
          if (!direct) {
            smem_row(k, cur);
          } else {
#pragma unroll
            for (int q = 0; q < NCC; ++q) cur[q] = __ldg(job.amps + (s0 + kk) * NCC + q);
          }
#pragma unroll
          for (int q = 0; q < NCC; ++q) bad |= amp_bad(cur[q]);
          V = A::mul(A::template slice<SP_MODE_MIDPOINT, NCC, MC>(job, m, cur, r1), V);
          if (PFX && job.prefix_out != nullptr) A::store(job.prefix_out, s0 + kk, V);
        }
      }
    }
    __syncwarp();
    if (ln == 0 && tma_warp && r + NST < rounds) {
      // every lane is done with stage s (syncwarp): refill it
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      su2_mbar_expect_tx(wb + s, STAGE);
      su2_tma_2d(ring + s * STAGE, &tmap, (r + NST) * C * NCC, (int)wlane0, wb + s);
    }
  }
  su2_finish<A, NCC, PFX>(job, V, bad, s0, s1 - 1);
}

}  // namespace sp

namespace sp {

// ---------------------------------------------------------------------------
// Analytic oracle on the device (studies.py:123-153, midpoint_reference): the
// driven qubit's midpoint-sliced propagator from EXACT per-slice SU(2)
// rotations exp(-i (vnorm dt / 2) n_k . sigma), n_k = (ax cos phi_k,
// ax sin phi_k, az), phi_k = wrf (k + 1/2) dt — no series, no amplitude
// table; the same lanes and ordered tail as the su(2) propagation.
// ---------------------------------------------------------------------------
struct QubitRef {
  int64_t steps;
  double c, s;      // cos / sin of vnorm dt / 2
  double ax, az;    // unit field axis in the rotating frame
  double wrf, dt;
};

__global__ void __launch_bounds__(512, 1) qubit_reference_kernel(const Su2Job job,
                                                                 const QubitRef q) {
  const int lane = blockIdx.x * blockDim.x + threadIdx.x;
  const int lanes = gridDim.x * blockDim.x;
  const int64_t s0 = (int64_t)lane * q.steps / lanes;
  const int64_t s1 = ((int64_t)lane + 1) * q.steps / lanes;
  Quat V = quat_identity();
  for (int64_t k = s0; k < s1; ++k) {
    const double t = ((double)k + 0.5) * q.dt;
    double sn, cs;
    sincos(q.wrf * t, &sn, &cs);
    const double nx = q.ax * cs, ny = q.ax * sn;
    // [[c - i s az, -i s (nx - i ny)], [-i s (nx + i ny), c + i s az]]
    V = quat_mul(Quat{q.c, -q.s * q.az, -q.s * ny, -q.s * nx}, V);
  }
  su2_finish<QuatAlg<double>, 1>(job, V, false, 0, 0);
}

}  // namespace sp
