// sm_100a kernels of the equiprop hot path.
//
// What the reference does in three materialised passes — expand every slice
// exponent (linalg.py:246-288), Chebyshev/Clenshaw-exponentiate the batch
// (chebyshev.py:259-306), fold the batch pairwise (propagator.py:68-102) —
// runs here as ONE streaming pass per "lane" (a contiguous run of slices):
//
//   for each slice s of the lane:
//     X_s = (2 scale / beta) (H0 + sum_t w_t(s) T_t)        assembled on chip
//     V   = p(X_s) V   by the reference's Clenshaw recurrence applied to
//           the running product V instead of I:
//           b_m = a_m V, b_{j} = a_j V + 2X b_{j+1} - (j==0 ? 2 : 1) b_{j+2}
//
// so p(X_s) (the slice propagator U_s) is never formed and nothing of size
// n*d^2 touches HBM.  The same m products per slice as the reference's
// m - 1 Clenshaw GEMMs + 1 reduction GEMM.  The lane products are then
// multiplied in time order (tree or left fold).
//
// Families
//   lane_small_kernel<D,TPL>  D in {2,4}: TPL threads per lane, each owning
//                             D/TPL columns of V; X in registers; DFMA.
//   lane_tc_kernel<Cfg>       D in {16..256}: FP64 tensor cores (DMMA,
//                             mma.sync m16n8k4 -> SASS DMMA.8x8x4).  A CTA
//                             (or a group of GPL CTAs) owns a lane; each CTA
//                             owns a WC-wide column block of V, because
//                             column j of p(X) V depends only on column j of
//                             V and on X — the Clenshaw recurrence needs no
//                             inter-CTA traffic except sharing X.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.h"

namespace sp {

#ifdef SP_PHASE_PROF
// per-phase SM clock totals of thread 0 of every CTA (tools/phase_prof.py;
// instrumented builds only)
__device__ unsigned long long g_phase[16];
// and per-CTA (start, end << 8 | smid) %globaltimer stamps of the first 2048 CTAs
__device__ unsigned long long g_tl[4096];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define PH_INIT long long ph_t = clock64(); unsigned long long ph_acc[10] = {0}; \
  const unsigned long long ph_g0 = gtimer();
#define PH(k) do { const long long t_ = clock64(); ph_acc[k] += t_ - ph_t; ph_t = t_; } while (0)
#define PH_DONE if (threadIdx.x == 0) { for (int k_ = 0; k_ < 10; ++k_) atomicAdd(&g_phase[k_], ph_acc[k_]); atomicAdd(&g_phase[15], 1ull); \
  if (blockIdx.x < 2048) { unsigned sm_; asm volatile("mov.u32 %0, %%smid;" : "=r"(sm_)); \
    g_tl[2 * blockIdx.x] = ph_g0; g_tl[2 * blockIdx.x + 1] = ((gtimer() - ph_g0) << 8) | (sm_ & 0xff); } }
#else
#define PH_INIT
#define PH(k) do {} while (0)
#define PH_DONE
#endif

// ---------------------------------------------------------------------------
// small helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ void dmma_16x8x4(double& c0, double& c1, double& c2, double& c3,
                                            double a0, double a1, double b) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
      "{%0,%1,%2,%3};\n"
      : "+d"(c0), "+d"(c1), "+d"(c2), "+d"(c3)
      : "d"(a0), "d"(a1), "d"(b));
}

__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// ---------------------------------------------------------------------------
// Tensor memory (TMEM) as a per-thread scratch extension of the register
// file: tcgen05.alloc/dealloc (warp-collective), 32x32b loads/stores (thread i
// of warp w owns TMEM lane 32*(w%4)+i).  The FP64 MMAs cannot use TMEM
// accumulators (tcgen05 has no f64 kind), but the 256 KB per SM holds the
// running product and the Chebyshev power blocks that would otherwise round
// trip through L2.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
// Ampere-style asynchronous 16-byte global -> shared copies (LDGSTS): many
// loads in flight per thread without holding registers
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem_dst)),
               "l"(gsrc)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}

__device__ __forceinline__ void tmem_alloc(uint32_t* slot, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(slot)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}
__device__ __forceinline__ void tmem_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tmem_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
// 4 complex doubles <-> 16 consecutive 32-bit columns of this thread's lane
__device__ __forceinline__ void tmem_st4(uint32_t taddr, const double* re, const double* im) {
  uint32_t w[16];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    w[4 * q + 0] = (uint32_t)__double2loint(re[q]);
    w[4 * q + 1] = (uint32_t)__double2hiint(re[q]);
    w[4 * q + 2] = (uint32_t)__double2loint(im[q]);
    w[4 * q + 3] = (uint32_t)__double2hiint(im[q]);
  }
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
      "%13,%14,%15,%16};" ::"r"(taddr),
      "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]),
      "r"(w[8]), "r"(w[9]), "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]), "r"(w[14]),
      "r"(w[15])
      : "memory");
}
// raw 16-column load; the values are valid only after tmem_wait_ld()
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&w)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15}, [%16];"
      : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]),
        "=r"(w[7]), "=r"(w[8]), "=r"(w[9]), "=r"(w[10]), "=r"(w[11]), "=r"(w[12]), "=r"(w[13]),
        "=r"(w[14]), "=r"(w[15])
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void tmem_unpack4(const uint32_t (&w)[16], double* re, double* im) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    re[q] = __hiloint2double((int)w[4 * q + 1], (int)w[4 * q + 0]);
    im[q] = __hiloint2double((int)w[4 * q + 3], (int)w[4 * q + 2]);
  }
}
// load NE complex doubles (NE % 4 == 0) from 4*NE consecutive columns
template <int NE>
__device__ __forceinline__ void tmem_load_block(uint32_t taddr, double (&re)[NE],
                                                double (&im)[NE]) {
  uint32_t w[NE / 4][16];
#pragma unroll
  for (int q = 0; q < NE / 4; ++q) tmem_ld16(taddr + 16 * q, w[q]);
  tmem_wait_ld();
#pragma unroll
  for (int q = 0; q < NE / 4; ++q) tmem_unpack4(w[q], &re[4 * q], &im[4 * q]);
}
template <int NE>
__device__ __forceinline__ void tmem_store_block(uint32_t taddr, const double (&re)[NE],
                                                 const double (&im)[NE]) {
#pragma unroll
  for (int q = 0; q < NE / 4; ++q) tmem_st4(taddr + 16 * q, &re[4 * q], &im[4 * q]);
  tmem_wait_st();
}

// Weight of expansion term t >= 1 for slice s (term 0 = drift, weight 1).
//   midpoint  hamiltonian.py:199-201        w = c_{s,t-1}
//   simpson   hamiltonian.py:202-205        w = (c1 + 4 c2 + c3) / 6
//   magnus    magnus.py:88-106, 134-139     controls: (c1+4c2+c3)/6,
//             i[H0,Hk]: (dt/6)(c3-c1),  i[Hk,Hk']: (dt/6)(c1_k c3_k' - c3_k c1_k')
//   (the reference divides the magnus columns by the 2dt scale; same values)
__device__ __forceinline__ void check_amp(const SliceJob& j, int64_t row, int col, double v) {
  // |c| <= 1 (false for NaN too); the first offender in row-major order wins
  if (!(fabs(v) <= 1.0) && j.viol) {
    unsigned long long* slot = j.viol + 2;
    if (j.viol_epoch) slot = j.viol + (__ldcg(j.viol + 3) & 1ull);
    atomicMin(slot, (unsigned long long)(row * j.n_ctrl + col));
  }
}

// end of a single-launch call (its last CTA, after every other CTA arrived):
// clear the slots the next call may use and advance the epoch (see SliceJob)
__device__ __forceinline__ void rotate_violation_slots(const SliceJob& j) {
  if (j.viol && j.viol_epoch) {
    const unsigned long long e = __ldcg(j.viol + 3);
    j.viol[(e + 1) & 1ull] = ~0ull;
    j.viol[2] = ~0ull;
    j.viol[3] = e + 1;
  }
}

// Every amplitude of the table is read by exactly one weight t in 1..N of
// some slice, so validating there covers the whole table in passing.
// pair (k, k') < N of cross-commutator column e (magnus.py:55-59 order)
__device__ __forceinline__ void cross_pair(int e, int N, int& k, int& kp) {
  k = 0;
  while (e >= N - 1 - k) {
    e -= N - 1 - k;
    ++k;
  }
  kp = k + 1 + e;
}

// Gauss-Legendre modes (extension): rows 2s (node a) and 2s + 1 (node b)
__device__ __forceinline__ double gauss_weight(const SliceJob& j, int64_t s, int t) {
  const int N = j.n_ctrl;
  const double* ra = j.amps + (2 * s) * N;
  const double* rb = ra + N;
  int e = t - 1;
  if (e < N) {
    check_amp(j, 2 * s, e, ra[e]);
    check_amp(j, 2 * s + 1, e, rb[e]);
    return 0.5 * (ra[e] + rb[e]);
  }
  e -= N;
  if (e < N) return j.gl * (rb[e] - ra[e]);
  int k, kp;
  cross_pair(e - N, N, k, kp);
  return j.gl * (ra[k] * rb[kp] - ra[kp] * rb[k]);
}

__device__ __forceinline__ double slice_weight(const SliceJob& j, int64_t s, int t) {
  const int N = j.n_ctrl;
  if (j.mode == SP_MODE_MIDPOINT) {
    const double v = j.amps[s * N + (t - 1)];
    check_amp(j, s, t - 1, v);
    return v;
  }
  if (j.mode >= SP_MODE_GAUSS2) return gauss_weight(j, s, t);
  const double* r1 = j.amps + (2 * s) * N;
  const double* r2 = r1 + N;
  const double* r3 = r2 + N;
  int e = t - 1;
  if (e < N) {
    check_amp(j, 2 * s, e, r1[e]);
    check_amp(j, 2 * s + 1, e, r2[e]);
    check_amp(j, 2 * s + 2, e, r3[e]);
    return (r1[e] + 4.0 * r2[e] + r3[e]) / 6.0;
  }
  e -= N;
  if (e < N) return (j.dt / 6.0) * (r3[e] - r1[e]);
  e -= N;
  int k = 0;
  while (e >= N - 1 - k) {
    e -= N - 1 - k;
    ++k;
  }
  const int kp = k + 1 + e;
  return (j.dt / 6.0) * (r1[k] * r3[kp] - r3[k] * r1[kp]);
}

// slice_weight split in two so that the amplitude loads of the next slice can
// be issued a slice ahead: weight_gather() reads the raw samples term t of
// slice s needs (at most 4), weight_combine() validates them and forms the
// weight with exactly slice_weight's arithmetic.
struct WRaw {
  double v[4];
};
__device__ __forceinline__ WRaw weight_gather(const SliceJob& j, int64_t s, int t) {
  WRaw w;
  const int N = j.n_ctrl;
  if (j.mode == SP_MODE_MIDPOINT) {
    w.v[0] = j.amps[s * N + (t - 1)];
    return w;
  }
  if (j.mode >= SP_MODE_GAUSS2) {
    const double* ra = j.amps + (2 * s) * N;
    const double* rb = ra + N;
    int e = t - 1;
    if (e >= N) e -= N;
    if (e < N) {
      w.v[0] = ra[e];
      w.v[1] = rb[e];
      return w;
    }
    int k, kp;
    cross_pair(e - N, N, k, kp);
    w.v[0] = ra[k];
    w.v[1] = rb[kp];
    w.v[2] = ra[kp];
    w.v[3] = rb[k];
    return w;
  }
  const double* r1 = j.amps + (2 * s) * N;
  const double* r2 = r1 + N;
  const double* r3 = r2 + N;
  int e = t - 1;
  if (e < N) {
    w.v[0] = r1[e];
    w.v[1] = r2[e];
    w.v[2] = r3[e];
    return w;
  }
  e -= N;
  if (e < N) {
    w.v[0] = r1[e];
    w.v[1] = r3[e];
    return w;
  }
  e -= N;
  int k = 0;
  while (e >= N - 1 - k) {
    e -= N - 1 - k;
    ++k;
  }
  const int kp = k + 1 + e;
  w.v[0] = r1[k];
  w.v[1] = r3[kp];
  w.v[2] = r3[k];
  w.v[3] = r1[kp];
  return w;
}
__device__ __forceinline__ double weight_combine(const SliceJob& j, int64_t s, int t,
                                                 const WRaw& w) {
  const int N = j.n_ctrl;
  if (j.mode == SP_MODE_MIDPOINT) {
    check_amp(j, s, t - 1, w.v[0]);
    return w.v[0];
  }
  if (j.mode >= SP_MODE_GAUSS2) {
    const int e = t - 1;
    if (e < N) {
      check_amp(j, 2 * s, e, w.v[0]);
      check_amp(j, 2 * s + 1, e, w.v[1]);
      return 0.5 * (w.v[0] + w.v[1]);
    }
    if (e < 2 * N) return j.gl * (w.v[1] - w.v[0]);
    return j.gl * (w.v[0] * w.v[1] - w.v[2] * w.v[3]);
  }
  int e = t - 1;
  if (e < N) {
    check_amp(j, 2 * s, e, w.v[0]);
    check_amp(j, 2 * s + 1, e, w.v[1]);
    check_amp(j, 2 * s + 2, e, w.v[2]);
    return (w.v[0] + 4.0 * w.v[1] + w.v[2]) / 6.0;
  }
  e -= N;
  if (e < N) return (j.dt / 6.0) * (w.v[1] - w.v[0]);
  return (j.dt / 6.0) * (w.v[0] * w.v[1] - w.v[2] * w.v[3]);
}

// The one complex dot product every ordered-product kernel uses (pair
// levels, left fold, prefix application): identical summation order
// everywhere keeps equiprop_all's last entry bitwise equal to the
// sequential reduction (reference property propagator.py:304-306, 310-316).
// (no __restrict__: the left fold reads matrices it wrote earlier in the
// same launch, so the non-coherent load path must not be used)
__device__ __forceinline__ double2 cdot(const double2* a_row, const double2* b, int ldb, int c,
                                        int D) {
  double re = 0.0, im = 0.0;
  for (int k = 0; k < D; ++k) {
    const double2 a = a_row[k];
    const double2 x = b[(size_t)k * ldb + c];
    re = fma(a.x, x.x, re);
    re = fma(-a.y, x.y, re);
    im = fma(a.x, x.y, im);
    im = fma(a.y, x.x, im);
  }
  return make_double2(re, im);
}

__device__ __forceinline__ void lane_range(int64_t n, int lanes, int lane, int64_t& s0,
                                           int64_t& s1) {
  s0 = (int64_t)lane * n / lanes;
  s1 = ((int64_t)lane + 1) * n / lanes;
}

// ---------------------------------------------------------------------------
// Family S: D in {2, 4}.  TPL threads per lane, CPT = D / TPL columns each.
// ---------------------------------------------------------------------------
// optional fused tail (pairwise reduction of the CTA products + output)
struct SmallTail {
  unsigned* ctr;  // zeroed before the launch; nullptr = no fused tail
  void* out;      // d x d result, complex128 or complex64
  int d;
  int to_fp32;
};

// C = A B for D x D complex matrices in registers
template <int D>
__device__ __forceinline__ void mat_mul(const double2 (&A)[D][D], const double2 (&B)[D][D],
                                        double2 (&C)[D][D]) {
#pragma unroll
  for (int r = 0; r < D; ++r)
#pragma unroll
    for (int c = 0; c < D; ++c) {
      double re = 0.0, im = 0.0;
#pragma unroll
      for (int k = 0; k < D; ++k) {
        re = fma(A[r][k].x, B[k][c].x, re);
        re = fma(-A[r][k].y, B[k][c].y, re);
        im = fma(A[r][k].x, B[k][c].y, im);
        im = fma(A[r][k].y, B[k][c].x, im);
      }
      C[r][c] = make_double2(re, im);
    }
}

// ordered product over the first `width` lanes of a warp: lane 0 ends with
// M_{width-1} ... M_1 M_0 (later lanes on the left)
template <int D>
__device__ __forceinline__ void warp_ordered_product(double2 (&M)[D][D], int width = 32) {
  for (int k = 1; k < width; k <<= 1) {
    double2 W[D][D], N[D][D];
#pragma unroll
    for (int r = 0; r < D; ++r)
#pragma unroll
      for (int c = 0; c < D; ++c)
        W[r][c] = make_double2(__shfl_down_sync(0xffffffffu, M[r][c].x, k),
                               __shfl_down_sync(0xffffffffu, M[r][c].y, k));
    mat_mul<D>(W, M, N);
#pragma unroll
    for (int r = 0; r < D; ++r)
#pragma unroll
      for (int c = 0; c < D; ++c) M[r][c] = N[r][c];
  }
}

// MC > 0: the series order m compiled in (the common orders 3, 7, 13, 15):
// the Clenshaw loop unrolls and the plan coefficients become constant-bank
// operands; 0 = runtime m
// ALT: the plan coefficients alternate real / imaginary (c_k = (-i)^k |c_k|,
// every symmetric equiprop plan: exact zeros, checked on the host), so each
// Clenshaw step of the d <= 4 general path needs one real-by-complex product
// per entry instead of a complex one (with MC the parity of every step is
// known at compile time)
template <int D, int TPL, int MC = 0, int NCC = 0, bool ALT = false>
// (register budget for 3 CTAs/SM at D = 2 and 2 at D = 4: the lane loop is
// latency bound and needs the resident warps)
__global__ void __launch_bounds__(256, D == 2 ? 3 : 2) lane_small_kernel(SliceJob job,
                                                         const double2* __restrict__ terms,
                                                         int lanes, double2* __restrict__ lane_out,
                                                         double2* cta_out,
                                                         double2* __restrict__ prefix_out,
                                                         SmallTail tail) {
  constexpr int CPT = D / TPL;
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = gtid / TPL;
  const int c0 = (gtid % TPL) * CPT;
  double2 V[D][CPT];
  const double2* vinit = static_cast<const double2*>(job.vinit);
#pragma unroll
  for (int r = 0; r < D; ++r)
#pragma unroll
    for (int cc = 0; cc < CPT; ++cc)
      V[r][cc] = (vinit != nullptr && lane < lanes)
                     ? vinit[(size_t)lane * D * D + r * D + c0 + cc]
                     : make_double2(r == c0 + cc ? 1.0 : 0.0, 0.0);

  int64_t s0 = 0, s1 = 0;
  if (lane < lanes) lane_range(job.n_slices, lanes, lane, s0, s1);
  const int T = job.n_terms;
  const int m = MC > 0 ? MC : job.m;
  constexpr int MUNR = MC > 0 ? MC : 1;
  const bool phase_one = job.phase[0] == 1.0 && job.phase[1] == 0.0;

  // the amplitude rows a few slices ahead are prefetched into L1 (no
  // registers held): the loop is otherwise bound by one memory round trip
  // per slice; a thread's slices are contiguous rows of the table
  // midpoint with <= RP controls (the driven qubit): the next slice's row is
  // loaded into registers a slice ahead instead
  const int64_t rows_per_slice = job.mode == SP_MODE_MIDPOINT ? 1 : 2;
  constexpr int RP = 4;
  const bool rowpf = D == 2 && job.mode == SP_MODE_MIDPOINT && job.n_ctrl <= RP;
  double nrow[RP];
  auto load_row = [&](int64_t sl) {
    const double* a = job.amps + sl * job.n_ctrl;
#pragma unroll
    for (int q = 0; q < RP; ++q)
      if (q < job.n_ctrl) nrow[q] = a[q];
  };
  if (rowpf && s0 < s1) load_row(s0);
  // D = 2, exactly Hermitian terms, <= 3 terms, midpoint (the driven qubit):
  // Z = 2X = z0 I + Z' with real z0, Z'00 = -Z'11 = dz real, Z'01 = conj(Z'10)
  // = zc, Z'^2 = zeta2 I with zeta2 = dz^2 + |zc|^2 real, so the Clenshaw
  // pairs below need real-by-complex products only; the per-term (z0, dz, zc)
  // contributions, with the 2X factor folded in, are formed once per thread
  const bool fast2 = D == 2 && job.herm_exact && rowpf && T <= 3;
  double tA[3] = {0.0, 0.0, 0.0}, tB[3] = {0.0, 0.0, 0.0};
  double2 tC[3] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0), make_double2(0.0, 0.0)};
  if (fast2) {
#pragma unroll
    for (int q = 0; q < 3; ++q)
      if (q < T) {
        const double2* H = terms + (size_t)q * D * D;
        tA[q] = job.xs * (0.5 * (H[0].x + H[D * D - 1].x));
        tB[q] = job.xs * (0.5 * (H[0].x - H[D * D - 1].x));
        tC[q] = make_double2(job.xs * H[1].x, job.xs * H[1].y);
      }
  }
  PH_INIT
  if constexpr (D == 2 && NCC > 0) {
    // the driven-qubit fast path with the control count compiled in: one
    // vector load per row (prefetched a slice ahead through a running
    // pointer), a 32-bit slice counter
    if (fast2 && job.n_ctrl == NCC) {
      auto ldrow = [&](const double* a, double (&rn)[NCC]) {
        if constexpr (NCC == 2) {
          const double2 v = *reinterpret_cast<const double2*>(a);
          rn[0] = v.x;
          rn[1] = v.y;
        } else {
#pragma unroll
          for (int q = 0; q < NCC; ++q) rn[q] = a[q];
        }
      };
      // U(slice s) from its amplitude row: the Clenshaw pairs (first step
      // peeled: b_{m+1} = b_{m+2} = 0 there, same values as the full step)
      auto slice_u = [&](const double (&rc)[NCC], int64_t s, double2 (&U)[2][2]) {
        double z0 = tA[0], dz = tB[0];
        double2 zc = tC[0];
#pragma unroll
        for (int q = 0; q < NCC; ++q) {
          const double w = rc[q];
          check_amp(job, s, q, w);
          z0 = fma(w, tA[q + 1], z0);
          dz = fma(w, tB[q + 1], dz);
          zc.x = fma(w, tC[q + 1].x, zc.x);
          zc.y = fma(w, tC[q + 1].y, zc.y);
        }
        const double zeta2 = fma(dz, dz, fma(zc.x, zc.x, zc.y * zc.y));
        double2 ca = make_double2(job.coef[2 * m], job.coef[2 * m + 1]);
        double2 cb = make_double2(0.0, 0.0), oa = cb, ob = cb;
        if (m >= 1) {
          const int jj = m - 1;
          oa = ca;
          cb = ca;
          ca = make_double2(job.coef[2 * jj] + z0 * oa.x, job.coef[2 * jj + 1] + z0 * oa.y);
        }
#pragma unroll MUNR
        for (int jj = m - 2; jj >= 0; --jj) {
          const double beta = (jj == 0) ? 2.0 : 1.0;
          const double2 na =
              make_double2(job.coef[2 * jj] + fma(z0, ca.x, fma(zeta2, cb.x, -beta * oa.x)),
                           job.coef[2 * jj + 1] + fma(z0, ca.y, fma(zeta2, cb.y, -beta * oa.y)));
          const double2 nb = make_double2(ca.x + fma(z0, cb.x, -beta * ob.x),
                                          ca.y + fma(z0, cb.y, -beta * ob.y));
          oa = ca;
          ob = cb;
          ca = na;
          cb = nb;
        }
        if (!phase_one) {
          const double pr = job.phase[0], pi = job.phase[1];
          ca = make_double2(pr * ca.x - pi * ca.y, pr * ca.y + pi * ca.x);
          cb = make_double2(pr * cb.x - pi * cb.y, pr * cb.y + pi * cb.x);
        }
        U[0][0] = make_double2(fma(cb.x, dz, ca.x), fma(cb.y, dz, ca.y));
        U[1][1] = make_double2(fma(-cb.x, dz, ca.x), fma(-cb.y, dz, ca.y));
        U[0][1] = make_double2(cb.x * zc.x - cb.y * zc.y, cb.x * zc.y + cb.y * zc.x);
        U[1][0] = make_double2(cb.x * zc.x + cb.y * zc.y, cb.y * zc.x - cb.x * zc.y);
      };
      // W <- U W (2 x 2 complex)
      auto left_mul = [&](const double2 (&U)[2][2], double2 (&W)[2][CPT]) {
        double2 nv[2][CPT];
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
          for (int cc = 0; cc < CPT; ++cc) {
            double re = U[r][0].x * W[0][cc].x;
            re = fma(-U[r][0].y, W[0][cc].y, re);
            re = fma(U[r][1].x, W[1][cc].x, re);
            re = fma(-U[r][1].y, W[1][cc].y, re);
            double im = U[r][0].x * W[0][cc].y;
            im = fma(U[r][0].y, W[0][cc].x, im);
            im = fma(U[r][1].x, W[1][cc].y, im);
            im = fma(U[r][1].y, W[1][cc].x, im);
            nv[r][cc] = make_double2(re, im);
          }
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
          for (int cc = 0; cc < CPT; ++cc) W[r][cc] = nv[r][cc];
      };
      const int cnt = (int)(s1 - s0);
      {
        const double* arow = job.amps + s0 * NCC;
        double rn[NCC];
        if (cnt > 0) ldrow(arow, rn);
        for (int k = 0; k < cnt; ++k) {
          double rc[NCC];
#pragma unroll
          for (int q = 0; q < NCC; ++q) rc[q] = rn[q];
          arow += NCC;
          if (k + 1 < cnt) ldrow(arow, rn);
          const int64_t s = s0 + k;
          double2 U[2][2];
          slice_u(rc, s, U);
          left_mul(U, V);
          if (prefix_out) {
            double2* o = prefix_out + (size_t)s * D * D;
#pragma unroll
            for (int r = 0; r < D; ++r)
#pragma unroll
              for (int cc = 0; cc < CPT; ++cc) o[r * D + c0 + cc] = V[r][cc];
          }
        }
      }
      s0 = s1;  // done: the general loop below has nothing left
    }
  }
  for (int64_t s = s0; s < s1; ++s) {
    double crow[RP];
#pragma unroll
    for (int q = 0; q < RP; ++q) crow[q] = nrow[q];
    if (rowpf) {
      if (s + 1 < s1) load_row(s + 1);
    } else if (s + 4 < s1) {
      asm volatile("prefetch.global.L1 [%0];" ::"l"(job.amps + (s + 4) * rows_per_slice *
                                                                   job.n_ctrl));
    }
    if constexpr (D == 2) {
      if (fast2) {
        double z0 = tA[0], dz = tB[0];
        double2 zc = tC[0];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          if (q + 1 >= T) break;
          const double w = crow[q];
          check_amp(job, s, q, w);
          z0 = fma(w, tA[q + 1], z0);
          dz = fma(w, tB[q + 1], dz);
          zc.x = fma(w, tC[q + 1].x, zc.x);
          zc.y = fma(w, tC[q + 1].y, zc.y);
        }
        const double zeta2 = fma(dz, dz, fma(zc.x, zc.x, zc.y * zc.y));
        double2 ca = make_double2(job.coef[2 * m], job.coef[2 * m + 1]);
        double2 cb = make_double2(0.0, 0.0), oa = cb, ob = cb;
#pragma unroll MUNR
        for (int jj = m - 1; jj >= 0; --jj) {
          const double beta = (jj == 0) ? 2.0 : 1.0;
          const double2 na =
              make_double2(job.coef[2 * jj] + fma(z0, ca.x, fma(zeta2, cb.x, -beta * oa.x)),
                           job.coef[2 * jj + 1] + fma(z0, ca.y, fma(zeta2, cb.y, -beta * oa.y)));
          const double2 nb = make_double2(ca.x + fma(z0, cb.x, -beta * ob.x),
                                          ca.y + fma(z0, cb.y, -beta * ob.y));
          oa = ca;
          ob = cb;
          ca = na;
          cb = nb;
        }
        if (!phase_one) {
          const double pr = job.phase[0], pi = job.phase[1];
          ca = make_double2(pr * ca.x - pi * ca.y, pr * ca.y + pi * ca.x);
          cb = make_double2(pr * cb.x - pi * cb.y, pr * cb.y + pi * cb.x);
        }
        double2 U[2][2];
        U[0][0] = make_double2(fma(cb.x, dz, ca.x), fma(cb.y, dz, ca.y));
        U[1][1] = make_double2(fma(-cb.x, dz, ca.x), fma(-cb.y, dz, ca.y));
        U[0][1] = make_double2(cb.x * zc.x - cb.y * zc.y, cb.x * zc.y + cb.y * zc.x);
        U[1][0] = make_double2(cb.x * zc.x + cb.y * zc.y, cb.y * zc.x - cb.x * zc.y);
        double2 nv[2][CPT];
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
          for (int cc = 0; cc < CPT; ++cc) {
            double re = U[r][0].x * V[0][cc].x;
            re = fma(-U[r][0].y, V[0][cc].y, re);
            re = fma(U[r][1].x, V[1][cc].x, re);
            re = fma(-U[r][1].y, V[1][cc].y, re);
            double im = U[r][0].x * V[0][cc].y;
            im = fma(U[r][0].y, V[0][cc].x, im);
            im = fma(U[r][1].x, V[1][cc].y, im);
            im = fma(U[r][1].y, V[1][cc].x, im);
            nv[r][cc] = make_double2(re, im);
          }
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
          for (int cc = 0; cc < CPT; ++cc) V[r][cc] = nv[r][cc];
        if (prefix_out) {
          double2* o = prefix_out + (size_t)s * D * D;
#pragma unroll
          for (int r = 0; r < D; ++r)
#pragma unroll
            for (int cc = 0; cc < CPT; ++cc) o[r * D + c0 + cc] = V[r][cc];
        }
        continue;
      }
    }
    // ---- assemble 2X in registers
    double2 X[D][D];
    if constexpr (D == 4 && TPL == 4) {
      // each of the lane's 4 threads assembles one row (its column index),
      // the rows are exchanged by shuffles within the 4-thread group (same
      // operations per entry as below)
      double2 xr[D];
      const int rr = c0;
#pragma unroll
      for (int c = 0; c < D; ++c) xr[c] = __ldg(&terms[rr * D + c]);
      for (int t = 1; t < T; ++t) {
        const double w = slice_weight(job, s, t);
        const double2* tt = terms + (size_t)t * D * D + rr * D;
#pragma unroll
        for (int c = 0; c < D; ++c) {
          const double2 h = __ldg(&tt[c]);
          xr[c].x = fma(w, h.x, xr[c].x);
          xr[c].y = fma(w, h.y, xr[c].y);
        }
      }
#pragma unroll
      for (int c = 0; c < D; ++c) {
        xr[c].x *= job.xs;
        xr[c].y *= job.xs;
      }
      const unsigned gm = 0xFu << (threadIdx.x & 28);
#pragma unroll
      for (int r = 0; r < D; ++r)
#pragma unroll
        for (int c = 0; c < D; ++c)
          X[r][c] = make_double2(__shfl_sync(gm, xr[c].x, r, 4), __shfl_sync(gm, xr[c].y, r, 4));
    } else {
#pragma unroll
    for (int r = 0; r < D; ++r)
#pragma unroll
      for (int c = 0; c < D; ++c) X[r][c] = __ldg(&terms[r * D + c]);
    auto add_term = [&](int t, double w) {
      const double2* tt = terms + (size_t)t * D * D;
#pragma unroll
      for (int r = 0; r < D; ++r)
#pragma unroll
        for (int c = 0; c < D; ++c) {
          const double2 h = __ldg(&tt[r * D + c]);
          X[r][c].x = fma(w, h.x, X[r][c].x);
          X[r][c].y = fma(w, h.y, X[r][c].y);
        }
    };
    if (rowpf) {
#pragma unroll
      for (int q = 0; q < RP; ++q) {
        if (q >= job.n_ctrl) break;
        check_amp(job, s, q, crow[q]);
        add_term(q + 1, crow[q]);
      }
    } else {
      for (int t = 1; t < T; ++t) add_term(t, slice_weight(job, s, t));
    }
#pragma unroll
    for (int r = 0; r < D; ++r)
#pragma unroll
      for (int c = 0; c < D; ++c) {
        X[r][c].x *= job.xs;
        X[r][c].y *= job.xs;
      }
    }
    if constexpr (D == 2) {
      // 2 x 2: every polynomial in Z = 2X lies in span{I, Z'}, Z' = Z - z0 I,
      // z0 = tr(Z)/2, Z'^2 = zeta2 I (Cayley-Hamilton, exact for any complex
      // 2 x 2), so the reference's matrix Clenshaw recurrence
      // (chebyshev.py:298-303) runs on coefficient pairs (a, b) = a I + b Z':
      // Z (a, b) = (z0 a + zeta2 b, a + z0 b).  Same polynomial, a quarter of
      // the work; U = a I + b Z' is formed once and applied to V.
      auto cmul = [](double2 x, double2 y) {
        return make_double2(fma(x.x, y.x, -x.y * y.y), fma(x.x, y.y, x.y * y.x));
      };
      const double2 z0 = make_double2(0.5 * (X[0][0].x + X[1][1].x),
                                      0.5 * (X[0][0].y + X[1][1].y));
      const double2 dz = make_double2(0.5 * (X[0][0].x - X[1][1].x),
                                      0.5 * (X[0][0].y - X[1][1].y));
      const double2 dd = cmul(dz, dz), od = cmul(X[0][1], X[1][0]);
      const double2 zeta2 = make_double2(dd.x + od.x, dd.y + od.y);
      double2 ca = make_double2(job.coef[2 * m], job.coef[2 * m + 1]);
      double2 cb = make_double2(0.0, 0.0), oa = cb, ob = cb;
#pragma unroll MUNR
      for (int jj = m - 1; jj >= 0; --jj) {
        const double beta = (jj == 0) ? 2.0 : 1.0;
        const double2 t1 = cmul(z0, ca), t2 = cmul(zeta2, cb), t3 = cmul(z0, cb);
        const double2 na = make_double2(job.coef[2 * jj] + t1.x + t2.x - beta * oa.x,
                                        job.coef[2 * jj + 1] + t1.y + t2.y - beta * oa.y);
        const double2 nb = make_double2(ca.x + t3.x - beta * ob.x, ca.y + t3.y - beta * ob.y);
        oa = ca;
        ob = cb;
        ca = na;
        cb = nb;
      }
      if (!phase_one) {
        const double2 ph = make_double2(job.phase[0], job.phase[1]);
        ca = cmul(ph, ca);
        cb = cmul(ph, cb);
      }
      const double2 bd = cmul(cb, dz);
      double2 U[2][2];
      U[0][0] = make_double2(ca.x + bd.x, ca.y + bd.y);
      U[1][1] = make_double2(ca.x - bd.x, ca.y - bd.y);
      U[0][1] = cmul(cb, X[0][1]);
      U[1][0] = cmul(cb, X[1][0]);
      double2 nv[2][CPT];
#pragma unroll
      for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int cc = 0; cc < CPT; ++cc) {
          double re = 0.0, im = 0.0;
#pragma unroll
          for (int k = 0; k < 2; ++k) {
            re = fma(U[r][k].x, V[k][cc].x, re);
            re = fma(-U[r][k].y, V[k][cc].y, re);
            im = fma(U[r][k].x, V[k][cc].y, im);
            im = fma(U[r][k].y, V[k][cc].x, im);
          }
          nv[r][cc] = make_double2(re, im);
        }
#pragma unroll
      for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int cc = 0; cc < CPT; ++cc) V[r][cc] = nv[r][cc];
    } else {
      // ---- Clenshaw applied to V (chebyshev.py:298-303 with I -> V)
      double2 cur[D][CPT], old[D][CPT];
      {
        const double ar = job.coef[2 * m], ai = job.coef[2 * m + 1];
  #pragma unroll
        for (int r = 0; r < D; ++r)
  #pragma unroll
          for (int cc = 0; cc < CPT; ++cc) {
            if (ALT && (m & 1))
              cur[r][cc] = make_double2(-ai * V[r][cc].y, ai * V[r][cc].x);
            else if (ALT)
              cur[r][cc] = make_double2(ar * V[r][cc].x, ar * V[r][cc].y);
            else
              cur[r][cc] = make_double2(ar * V[r][cc].x - ai * V[r][cc].y,
                                        ar * V[r][cc].y + ai * V[r][cc].x);
            old[r][cc] = make_double2(0.0, 0.0);
          }
      }
#pragma unroll MUNR
      for (int jj = m - 1; jj >= 0; --jj) {
        const double ar = job.coef[2 * jj], ai = job.coef[2 * jj + 1];
        const double beta = (jj == 0) ? 2.0 : 1.0;
        double2 nw[D][CPT];
  #pragma unroll
        for (int r = 0; r < D; ++r)
  #pragma unroll
          for (int cc = 0; cc < CPT; ++cc) {
            double re, im;
            if (ALT && (jj & 1)) {  // c_jj = i ai: same values, one product less
              re = fma(-ai, V[r][cc].y, -beta * old[r][cc].x);
              im = fma(ai, V[r][cc].x, -beta * old[r][cc].y);
            } else if (ALT) {  // c_jj = ar
              re = fma(ar, V[r][cc].x, -beta * old[r][cc].x);
              im = fma(ar, V[r][cc].y, -beta * old[r][cc].y);
            } else {
              re = fma(ar, V[r][cc].x, fma(-ai, V[r][cc].y, -beta * old[r][cc].x));
              im = fma(ar, V[r][cc].y, fma(ai, V[r][cc].x, -beta * old[r][cc].y));
            }
  #pragma unroll
            for (int k = 0; k < D; ++k) {
              re = fma(X[r][k].x, cur[k][cc].x, re);
              re = fma(-X[r][k].y, cur[k][cc].y, re);
              im = fma(X[r][k].x, cur[k][cc].y, im);
              im = fma(X[r][k].y, cur[k][cc].x, im);
            }
            nw[r][cc] = make_double2(re, im);
          }
  #pragma unroll
        for (int r = 0; r < D; ++r)
  #pragma unroll
          for (int cc = 0; cc < CPT; ++cc) {
            old[r][cc] = cur[r][cc];
            cur[r][cc] = nw[r][cc];
          }
      }
  #pragma unroll
      for (int r = 0; r < D; ++r)
  #pragma unroll
        for (int cc = 0; cc < CPT; ++cc) {
          if (phase_one) {
            V[r][cc] = cur[r][cc];
          } else {
            V[r][cc] = make_double2(job.phase[0] * cur[r][cc].x - job.phase[1] * cur[r][cc].y,
                                    job.phase[0] * cur[r][cc].y + job.phase[1] * cur[r][cc].x);
          }
        }
    }
    if (prefix_out) {
      double2* o = prefix_out + (size_t)s * D * D;
#pragma unroll
      for (int r = 0; r < D; ++r)
#pragma unroll
        for (int cc = 0; cc < CPT; ++cc) o[r * D + c0 + cc] = V[r][cc];
    }
  }

  if (cta_out == nullptr) {
    if (lane < lanes) {
      double2* o = lane_out + (size_t)lane * D * D;
#pragma unroll
      for (int r = 0; r < D; ++r)
#pragma unroll
        for (int cc = 0; cc < CPT; ++cc) o[r * D + c0 + cc] = V[r][cc];
    }
    return;
  }
  PH(0);
  if constexpr (TPL == 1) {
    // ---- one thread per lane (D = 2): ordered products by warp shuffles
    // (lane i takes V_{i+k} V_i, k = 1, 2, 4, ...; lanes without slices
    // hold I), then the CTA's 8 warp products by warp 0; the fused tail
    // reduces the CTA products the same way, 256 at a time
    __shared__ double2 wbuf[8][D * D];
    __shared__ bool last2;
    const int ln = threadIdx.x & 31, wp = threadIdx.x >> 5;
    auto load_id = [&](double2 (&M)[D][D]) {
#pragma unroll
      for (int r = 0; r < D; ++r)
#pragma unroll
        for (int c = 0; c < D; ++c) M[r][c] = make_double2(r == c ? 1.0 : 0.0, 0.0);
    };
    auto cta_product = [&](double2 (&M)[D][D]) {  // result in thread 0
      warp_ordered_product<D>(M);
      if (ln == 0)
#pragma unroll
        for (int r = 0; r < D; ++r)
#pragma unroll
          for (int c = 0; c < D; ++c) wbuf[wp][r * D + c] = M[r][c];
      __syncthreads();
      if (wp == 0) {
        if (ln < 8) {
#pragma unroll
          for (int r = 0; r < D; ++r)
#pragma unroll
            for (int c = 0; c < D; ++c) M[r][c] = wbuf[ln][r * D + c];
        } else {
          load_id(M);
        }
        warp_ordered_product<D>(M, 8);
      }
      __syncthreads();  // wbuf reusable
    };
    double2 M[D][D];
#pragma unroll
    for (int r = 0; r < D; ++r)
#pragma unroll
      for (int c = 0; c < D; ++c) M[r][c] = V[r][c];
    cta_product(M);
    PH(1);
    if (threadIdx.x == 0) {
      double2* o = cta_out + (size_t)blockIdx.x * D * D;
#pragma unroll
      for (int r = 0; r < D; ++r)
#pragma unroll
        for (int c = 0; c < D; ++c) o[r * D + c] = M[r][c];
      if (tail.ctr != nullptr) {
        // one acq_rel RMW: releases this thread's CTA product, acquires the
        // others' for the last arriver (the CTA barrier below extends it)
        unsigned old;
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;"
                     : "=r"(old)
                     : "l"(tail.ctr)
                     : "memory");
        last2 = (old == gridDim.x - 1);
      }
    }
    if (tail.ctr == nullptr) {
      PH_DONE
      return;
    }
    __syncthreads();
    PH(2);
    if (!last2) {
      PH_DONE
      return;
    }
    // every thread folds a contiguous run of CTA products (later on the
    // left), then one CTA-wide ordered product: a single pass for any grid
    {
      const int G = (int)gridDim.x, per = (G + 255) / 256;
      const int i0 = min(G, (int)threadIdx.x * per), i1 = min(G, i0 + per);
      load_id(M);
      for (int i = i0; i < i1; ++i) {
        double2 P[D][D], N[D][D];
#pragma unroll
        for (int r = 0; r < D; ++r)
#pragma unroll
          for (int c = 0; c < D; ++c) P[r][c] = __ldcg(&cta_out[(size_t)i * D * D + r * D + c]);
        mat_mul<D>(P, M, N);
#pragma unroll
        for (int r = 0; r < D; ++r)
#pragma unroll
          for (int c = 0; c < D; ++c) M[r][c] = N[r][c];
      }
      cta_product(M);
    }
    if (threadIdx.x == 0) {
      for (int e = 0; e < tail.d * tail.d; ++e) {
        const double2 v = M[e / tail.d][e % tail.d];
        if (tail.to_fp32)
          reinterpret_cast<float2*>(tail.out)[e] = make_float2((float)v.x, (float)v.y);
        else
          reinterpret_cast<double2*>(tail.out)[e] = v;
      }
      *tail.ctr = 0;  // ready for the next launch
      rotate_violation_slots(job);
    }
    PH(3);
    PH_DONE
    return;
  } else {
  // ---- in-CTA ordered pairwise tree over the CTA's consecutive lanes
  constexpr int LPB = 256 / TPL;  // lanes per block (blockDim = 256)
  __shared__ double2 buf[2][LPB * D * D];
  const int lb = threadIdx.x / TPL;
#pragma unroll
  for (int r = 0; r < D; ++r)
#pragma unroll
    for (int cc = 0; cc < CPT; ++cc) buf[0][lb * D * D + r * D + c0 + cc] = V[r][cc];
  __syncthreads();
  int cnt = LPB, src = 0;
  while (cnt > 1) {
    const int pairs = cnt >> 1;
    for (int e = threadIdx.x; e < pairs * D * D; e += blockDim.x) {
      const int p = e / (D * D), rc = e % (D * D), r = rc / D, c = rc % D;
      const double2* later = &buf[src][(2 * p + 1) * D * D];
      const double2* earlier = &buf[src][(2 * p) * D * D];
      buf[src ^ 1][p * D * D + rc] = cdot(later + r * D, earlier, D, c, D);
    }
    if (cnt & 1)
      for (int e = threadIdx.x; e < D * D; e += blockDim.x)
        buf[src ^ 1][pairs * D * D + e] = buf[src][(cnt - 1) * D * D + e];
    __syncthreads();
    cnt = pairs + (cnt & 1);
    src ^= 1;
  }
  PH(1);
  if (tail.ctr == nullptr) {
    for (int e = threadIdx.x; e < D * D; e += blockDim.x)
      cta_out[(size_t)blockIdx.x * D * D + e] = buf[src][e];
    PH_DONE
    return;
  }

  // ---- fused tail: the last CTA to finish multiplies the CTA products in
  // time order (chunks of LPB by the same smem tree, later chunks on the
  // left) and writes the d x d result — the whole equiprop in one launch.
  // One thread publishes the CTA product, fences and takes the ticket.
  __shared__ bool is_last;
  __shared__ double2 carry[D * D];
  if (threadIdx.x == 0) {
    for (int e = 0; e < D * D; ++e) cta_out[(size_t)blockIdx.x * D * D + e] = buf[src][e];
    __threadfence();
    is_last = (atomicAdd(tail.ctr, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  PH(2);
  if (!is_last) {
    PH_DONE
    return;
  }
  __threadfence();
  for (int e = threadIdx.x; e < D * D; e += blockDim.x)
    carry[e] = make_double2((e / D) == (e % D) ? 1.0 : 0.0, 0.0);
  for (int base = 0; base < (int)gridDim.x; base += LPB) {
    const int here = min(LPB, (int)gridDim.x - base);
    for (int e = threadIdx.x; e < here * D * D; e += blockDim.x)
      buf[0][e] = __ldcg(&cta_out[(size_t)base * D * D + e]);
    __syncthreads();
    int c2 = here, sr = 0;
    while (c2 > 1) {
      const int pairs = c2 >> 1;
      for (int e = threadIdx.x; e < pairs * D * D; e += blockDim.x) {
        const int p = e / (D * D), rc = e % (D * D), r = rc / D, c = rc % D;
        buf[sr ^ 1][p * D * D + rc] =
            cdot(&buf[sr][(2 * p + 1) * D * D + r * D], &buf[sr][(2 * p) * D * D], D, c, D);
      }
      if (c2 & 1)
        for (int e = threadIdx.x; e < D * D; e += blockDim.x)
          buf[sr ^ 1][pairs * D * D + e] = buf[sr][(c2 - 1) * D * D + e];
      __syncthreads();
      c2 = pairs + (c2 & 1);
      sr ^= 1;
    }
    // carry <- chunk product * carry
    for (int e = threadIdx.x; e < D * D; e += blockDim.x)
      buf[sr ^ 1][e] = cdot(&buf[sr][(e / D) * D], carry, D, e % D, D);
    __syncthreads();
    for (int e = threadIdx.x; e < D * D; e += blockDim.x) carry[e] = buf[sr ^ 1][e];
    __syncthreads();
  }
  for (int e = threadIdx.x; e < tail.d * tail.d; e += blockDim.x) {
    const double2 v = carry[(e / tail.d) * D + (e % tail.d)];
    if (tail.to_fp32)
      reinterpret_cast<float2*>(tail.out)[e] = make_float2((float)v.x, (float)v.y);
    else
      reinterpret_cast<double2*>(tail.out)[e] = v;
  }
  if (threadIdx.x == 0) {
    *tail.ctr = 0;  // ready for the next launch
    rotate_violation_slots(job);
  }
  PH(3);
  PH_DONE
  }
}

// ---------------------------------------------------------------------------
// Family TC: FP64 tensor cores.
// ---------------------------------------------------------------------------
// X fragment layout ("A-native"): for strip S (rows 16S..16S+15), k-block kb
// (cols 4kb..4kb+3), plane p (0 re, 1 im): 64 doubles; lane l holds
// {X[16S + g][4kb + t], X[16S + 8 + g][4kb + t]} at offset 2l, g = l>>2, t = l&3.
// B fragment layout (iterates, smem): for k-block kb, n-tile nt, plane p: 32
// doubles; lane l holds B[4kb + t][8nt + g].
template <int D_, int WC_, int MT_, int NT_, int WPL_, int LPC_, int GPL_, bool XS_>
struct TCCfg {
  static constexpr int D = D_, WC = WC_, MT = MT_, NT = NT_, WPL = WPL_, LPC = LPC_,
                       GPL = GPL_;
  static constexpr bool XS = XS_;
  static constexpr int S = D / 16;
  static constexpr int KB = D / 4;
  static constexpr int NTC = WC / 8;
  static constexpr int XDBL = 2 * D * D;
  static constexpr int BDBL = 2 * D * WC;
  static constexpr int WMAX = 256;  // max expansion terms
  static constexpr int THREADS = 32 * WPL * LPC;
  static constexpr int LANE_DBL = 2 * BDBL + (XS ? XDBL : 0) + WMAX;
  static constexpr size_t SMEM = (size_t)LANE_DBL * LPC * sizeof(double);
  static constexpr bool ASW = false;  // smem A operands swizzled (aswz)
  static_assert(D == WC * GPL, "column blocks must tile D");
  static_assert((S / MT) * (NTC / NT) == WPL, "warp tiling must cover the block");
  static_assert(GPL == 1 || LPC == 1, "groups own one lane per CTA");
};

// 256-bit global store (sm_100: STG.E.ENL2.256); p 32-byte aligned
__device__ __forceinline__ void st_global_v4(double* p, double a, double b, double c, double d) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a), "d"(b), "d"(c),
               "d"(d)
               : "memory");
}

// the same with an L2 cache-policy hint (createpolicy, e.g. evict_last for
// exchange buffers that are rewritten every slice and must stay L2-resident)
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void st_global_v4_hint(double* p, double a, double b, double c,
                                                  double d, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.f64 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "d"(a),
               "d"(b), "d"(c), "d"(d), "l"(pol)
               : "memory");
}

// swizzled shared-memory copy of the A-native layout (lane_ps_kernel): the
// 16-byte units of odd k blocks swap pairwise (bit 1 of the double offset),
// so a warp's 16-byte accumulator stores — rows g / g+8 of columns 2 t4,
// t4 = 0..3, spanning two k blocks — hit 8 distinct bank quads per phase;
// the fragment loads stay one unit per lane.  Valid for an even k-block count.
__host__ __device__ constexpr int aswz(int idx) { return idx ^ (((idx >> 7) & 1) << 1); }

__host__ __device__ constexpr int xfrag_index(int D, int r, int c, int plane) {
  // element (r, c) of a D x D matrix in the A-native layout
  return (((r >> 4) * (D >> 2) + (c >> 2)) * 2 + plane) * 64 + (((r & 7) << 2) | (c & 3)) * 2 +
         ((r >> 3) & 1);
}

// cumulative mode: per-slice in-lane prefixes are stored in the A-native
// 2-plane layout (2 D^2 doubles per slice) so that the prefix application
// (apply_prefix_tc_kernel) reads them as tensor-core A operands
__device__ __forceinline__ void store_prefix(double2* base, int D, int64_t slice, int r, int c,
                                             double re, double im) {
  double* o = reinterpret_cast<double*>(base) + (size_t)slice * 2 * D * D;
  o[xfrag_index(D, r, c, 0)] = re;
  o[xfrag_index(D, r, c, 1)] = im;
}

// B-native layout: per 4-row k block, 8-column n tile and plane, 32 doubles
// in mma.sync B-fragment order (lane n*4 + k), with bit 2 of the position
// flipped in its upper half (XOR swizzle: a warp's accumulator scatter —
// rows g, columns 2 t4 + par — then spans all 16 bank pairs of a block, 2
// wavefronts instead of 4; the fragment loads read position bswz(ln))
__host__ __device__ constexpr int bswz(int x) { return x ^ (((x >> 4) & 1) << 2); }

template <class C>
__device__ __forceinline__ int bfrag_index(int r, int n, int plane) {
  return (((r >> 2) * C::NTC + (n >> 3)) * 2 + plane) * 32 + bswz(((n & 7) << 2) + (r & 3));
}

template <class C>
__device__ __forceinline__ void lane_sync() {
  if constexpr (C::WPL == 1) {
    __syncwarp();
  } else if constexpr (C::LPC == 1) {
    __syncthreads();
  } else {
    const int lic = (threadIdx.x >> 5) / C::WPL;
    asm volatile("bar.sync %0, %1;" ::"r"(lic + 1), "r"(C::WPL * 32) : "memory");
  }
}

// Release / acquire at gpu scope, cumulative through the CTA barriers: the
// CTA's stores -> bar.sync -> red.release by thread 0 ... ld.acquire by the
// waiting CTA's thread 0 -> bar.sync -> its loads (no full fences).
__device__ __forceinline__ void red_release_gpu(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void group_barrier(unsigned* ctr, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    red_release_gpu(ctr, 1u);
    while (ld_acquire_gpu(ctr) < target) {
    }
  }
  __syncthreads();
}

// the same barrier split in two, so CTA-local work can run while the other
// CTAs of the group arrive: arrive after this CTA's stores, wait before
// reading theirs
__device__ __forceinline__ void group_arrive(unsigned* ctr) {
  __syncthreads();
  if (threadIdx.x == 0) red_release_gpu(ctr, 1u);
}
__device__ __forceinline__ void group_wait(unsigned* ctr, unsigned target) {
  if (threadIdx.x == 0) {
    while (ld_acquire_gpu(ctr) < target) {
    }
  }
  __syncthreads();
}

// lane_tc_kernel (the Clenshaw form) lives in kernels_tc.cuh

// ---------------------------------------------------------------------------
// ordered products of lane / block products
// ---------------------------------------------------------------------------
// one level of the reference's level-order fold (propagator.py:91-101):
// out[i] = in[2i+1] in[2i] (later on the left), odd last copied forward
__global__ void pair_level_kernel(const double2* __restrict__ in, int cnt, int D,
                                  double2* __restrict__ out) {
  const int pairs = cnt >> 1;
  const int64_t total = (int64_t)(pairs + (cnt & 1)) * D * D;
  const int64_t dd = (int64_t)D * D;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t pi = e / dd;
    const int rc = (int)(e % dd), r = rc / D, c = rc % D;
    if (pi < pairs)
      out[e] = cdot(in + (2 * pi + 1) * dd + (int64_t)r * D, in + 2 * pi * dd, D, c, D);
    else
      out[e] = in[(cnt - 1) * dd + rc];
  }
}

// single-CTA left fold: E[0] = I, E[l] = M[l-1] E[l-1] (exclusive prefixes,
// optional) and total = M[cnt-1] ... M[0] written to out.
__global__ void fold_kernel(const double2* __restrict__ mats, int cnt, int D,
                            double2* __restrict__ scratch, double2* __restrict__ prefixes,
                            double2* __restrict__ out) {
  const int dd = D * D;
  double2* acc[2] = {scratch, scratch + dd};
  for (int e = threadIdx.x; e < dd; e += blockDim.x) {
    const double2 id = make_double2((e / D) == (e % D) ? 1.0 : 0.0, 0.0);
    acc[0][e] = id;
    if (prefixes) prefixes[e] = id;
  }
  __syncthreads();
  int cur = 0;
  for (int l = 0; l < cnt; ++l) {
    const double2* Ml = mats + (size_t)l * dd;
    double2* dst = (l == cnt - 1) ? out : acc[cur ^ 1];
    for (int e = threadIdx.x; e < dd; e += blockDim.x) {
      const int r = e / D, c = e % D;
      dst[e] = cdot(Ml + (size_t)r * D, acc[cur], D, c, D);
    }
    __syncthreads();
    if (l == cnt - 1) break;
    cur ^= 1;
    if (prefixes)
      for (int e = threadIdx.x; e < dd; e += blockDim.x)
        prefixes[(size_t)(l + 1) * dd + e] = acc[cur][e];
  }
}

// Two-level exclusive scan of many lane products (plain-layout families,
// d <= 8, where thousands of lanes keep the lane pass busy):
//  group_fold_kernel: block b folds lanes [b GS, (b+1) GS) in order, writing
//    the in-group exclusive prefixes Ein[l] and the group total Gt[b];
//  fold_kernel over Gt gives the exclusive group prefixes EG[b];
//  combine_prefix_kernel: E[l] = Ein[l] EG[l / GS];
//  lane_total_kernel: total = M[L-1] E[L-1].
// The sequential reduction and equiprop_all share these steps, so the last
// cumulative entry P_last E[L-1] equals the sequential total bit for bit.
__global__ void group_fold_kernel(const double2* __restrict__ mats, int cnt, int D, int GS,
                                  double2* __restrict__ Ein, double2* __restrict__ Gt) {
  __shared__ double2 acc[2][64];
  const int dd = D * D, b = blockIdx.x;
  const int l0 = b * GS, l1 = min(cnt, l0 + GS);
  for (int e = threadIdx.x; e < dd; e += blockDim.x) {
    acc[0][e] = make_double2((e / D) == (e % D) ? 1.0 : 0.0, 0.0);
    Ein[(size_t)l0 * dd + e] = acc[0][e];
  }
  __syncthreads();
  int cur = 0;
  for (int l = l0; l < l1; ++l) {
    const double2* Ml = mats + (size_t)l * dd;
    for (int e = threadIdx.x; e < dd; e += blockDim.x)
      acc[cur ^ 1][e] = cdot(Ml + (size_t)(e / D) * D, acc[cur], D, e % D, D);
    __syncthreads();
    cur ^= 1;
    for (int e = threadIdx.x; e < dd; e += blockDim.x) {
      if (l + 1 < l1) Ein[(size_t)(l + 1) * dd + e] = acc[cur][e];
      else Gt[(size_t)b * dd + e] = acc[cur][e];
    }
  }
}

// the same group fold with one thread per group and the running product in
// registers (D <= 4: a short dependent chain per step, no barriers); the
// exclusive group prefixes use it too (one group spanning all totals)
template <int D>
__global__ void group_fold_reg_kernel(const double2* __restrict__ mats, int cnt, int GS,
                                      double2* __restrict__ Ein, double2* __restrict__ Gt) {
  constexpr int dd = D * D;
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  const int l0 = b * GS, l1 = min(cnt, l0 + GS);
  if (l0 >= cnt) return;
  double2 acc[D][D];
#pragma unroll
  for (int r = 0; r < D; ++r)
#pragma unroll
    for (int c = 0; c < D; ++c) acc[r][c] = make_double2(r == c ? 1.0 : 0.0, 0.0);
  // chunks of 8 lane products: all 8 loads in flight, then 8 dependent steps
  constexpr int CH = 8;
  for (int lb = l0; lb < l1; lb += CH) {
    double2 M[CH][D][D];
#pragma unroll
    for (int j = 0; j < CH; ++j)
      if (lb + j < l1) {
        const double2* Ml = mats + (size_t)(lb + j) * dd;
#pragma unroll
        for (int r = 0; r < D; ++r)
#pragma unroll
          for (int c = 0; c < D; ++c) M[j][r][c] = __ldcg(&Ml[r * D + c]);
      }
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      if (lb + j >= l1) break;
      double2* o = Ein + (size_t)(lb + j) * dd;
#pragma unroll
      for (int r = 0; r < D; ++r)
#pragma unroll
        for (int c = 0; c < D; ++c) o[r * D + c] = acc[r][c];
      // acc <- M acc, each entry with the cdot summation order
      double2 N[D][D];
#pragma unroll
      for (int r = 0; r < D; ++r)
#pragma unroll
        for (int c = 0; c < D; ++c) {
          double re = 0.0, im = 0.0;
#pragma unroll
          for (int k = 0; k < D; ++k) {
            re = fma(M[j][r][k].x, acc[k][c].x, re);
            re = fma(-M[j][r][k].y, acc[k][c].y, re);
            im = fma(M[j][r][k].x, acc[k][c].y, im);
            im = fma(M[j][r][k].y, acc[k][c].x, im);
          }
          N[r][c] = make_double2(re, im);
        }
#pragma unroll
      for (int r = 0; r < D; ++r)
#pragma unroll
        for (int c = 0; c < D; ++c) acc[r][c] = N[r][c];
    }
  }
  if (Gt != nullptr) {
#pragma unroll
    for (int r = 0; r < D; ++r)
#pragma unroll
      for (int c = 0; c < D; ++c) Gt[(size_t)b * dd + r * D + c] = acc[r][c];
  }
}

__global__ void combine_prefix_kernel(const double2* __restrict__ Ein,
                                      const double2* __restrict__ EG, int cnt, int D, int GS,
                                      double2* __restrict__ E) {
  const int64_t dd = (int64_t)D * D, total = (int64_t)cnt * dd;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t l = e / dd;
    const int rc = (int)(e % dd);
    E[e] = cdot(Ein + l * dd + (int64_t)(rc / D) * D, EG + (l / GS) * dd, D, rc % D, D);
  }
}

__global__ void lane_total_kernel(const double2* __restrict__ M, const double2* __restrict__ E,
                                  int D, double2* __restrict__ out) {
  const int dd = D * D;
  for (int e = threadIdx.x; e < dd; e += blockDim.x)
    out[e] = cdot(M + (e / D) * D, E, D, e % D, D);
}

// first slice of every lane under lane_range() (lanes + 1 entries)
__global__ void lane_starts_kernel(int64_t n, int lanes, int64_t* __restrict__ starts) {
  for (int l = blockIdx.x * blockDim.x + threadIdx.x; l <= lanes; l += gridDim.x * blockDim.x)
    starts[l] = (int64_t)l * n / lanes;
}

// cumulative products: out[s] = P[s] E[lane(s)] with P[s] the in-lane prefix,
// written straight into the (n, d, d) output in the output dtype
// (plain-layout families, D <= 8).
// The same product organised by lane: one CTA per lane; thread t owns
// output column c = t % D and keeps column c of E_lane in registers, and the
// CTA's 256 / D slice groups stream the lane's contiguous slices (the P_s
// rows are read once per slice group through L1, broadcast to the D threads
// of the slice; no per-element lane lookup).  Same summation order as cdot
// (k ascending, same fma pattern): the last entry stays bitwise equal to the
// sequential total.
template <int D>
__global__ void __launch_bounds__(256) apply_prefix_lanes_kernel(
    const double2* __restrict__ P, const double2* __restrict__ E,
    const int64_t* __restrict__ starts, int d, int to_fp32, void* __restrict__ out) {
  constexpr int dd = D * D, G = 256 / D;
  const int l = blockIdx.x;
  const int c = threadIdx.x % D, j = threadIdx.x / D;
  double2 ec[D];
#pragma unroll
  for (int k = 0; k < D; ++k) ec[k] = E[(int64_t)l * dd + k * D + c];
  const int64_t s1 = starts[l + 1];
  if (c >= d) return;
  for (int64_t s = starts[l] + j; s < s1; s += G) {
    const double2* ps = P + s * dd;
    const int64_t o = s * (int64_t)d * d + c;
#pragma unroll
    for (int r = 0; r < D; ++r) {
      if (r >= d) break;
      double re = 0.0, im = 0.0;
#pragma unroll
      for (int k = 0; k < D; ++k) {
        const double2 a = ps[r * D + k];
        re = fma(a.x, ec[k].x, re);
        re = fma(-a.y, ec[k].y, re);
        im = fma(a.x, ec[k].y, im);
        im = fma(a.y, ec[k].x, im);
      }
      if (to_fp32)
        reinterpret_cast<float2*>(out)[o + (int64_t)r * d] = make_float2((float)re, (float)im);
      else
        reinterpret_cast<double2*>(out)[o + (int64_t)r * d] = make_double2(re, im);
    }
  }
}

// pad a (cnt, d, d) complex128 batch to (cnt, D, D) by embedding in the
// top-left corner with an identity tail, and the reverse extraction
__global__ void embed_kernel(const double2* __restrict__ in, int cnt, int d, int D,
                             double2* __restrict__ out) {
  const int64_t total = (int64_t)cnt * D * D;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = e / ((int64_t)D * D);
    const int rc = (int)(e % ((int64_t)D * D)), r = rc / D, c = rc % D;
    out[e] = (r < d && c < d) ? in[k * d * d + r * d + c]
                              : make_double2(r == c ? 1.0 : 0.0, 0.0);
  }
}

__global__ void extract_kernel(const double2* __restrict__ in, int64_t cnt, int D, int d,
                               int to_fp32, void* __restrict__ out) {
  const int64_t total = cnt * d * d;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = e / ((int64_t)d * d);
    const int rc = (int)(e % ((int64_t)d * d)), r = rc / d, c = rc % d;
    const double2 v = in[k * D * D + (int64_t)r * D + c];
    if (to_fp32)
      reinterpret_cast<float2*>(out)[e] = make_float2((float)v.x, (float)v.y);
    else
      reinterpret_cast<double2*>(out)[e] = v;
  }
}

}  // namespace sp
