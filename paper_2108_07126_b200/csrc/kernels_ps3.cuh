// Paterson–Stockmeyer lane kernel with 3-multiplication complex products.
//
// Same evaluation as lane_ps_kernel (kernels_ps.cuh: powers, Clenshaw in
// y = T_s, V <- U V; same plan polynomial), but every complex tile product
// uses three real DMMAs instead of four:
//   P1 = Ar Br,  P2 = Ai Bi,  P3 = (Ar + Ai)(Br + Bi)
//   Re = P1 - P2,  Im = P3 - P1 - P2
// The sums Ar + Ai and Br + Bi are stored as a third plane of every operand
// (written once per operand, so the inner loop has no extra arithmetic), and
// the accumulator inits fold in as acc1 = init_re, acc2 = 0,
// acc3 = init_re + init_im.  25% fewer FP64 tensor-pipe instructions; the
// result is normwise as accurate as the 4-product form (Higham, "Stability of
// a method for multiplying complex matrices with three real matrix
// multiplications").
#pragma once
#include "kernels_ps.cuh"

namespace sp {

template <int D_, int WC_, int MT_, int NT_, int WPL_, int LPC_, int GPL_, bool XS_>
struct PS3Cfg {
  static constexpr int D = D_, WC = WC_, MT = MT_, NT = NT_, WPL = WPL_, LPC = LPC_, GPL = GPL_;
  static constexpr bool XS = XS_;
  static constexpr int S = D / 16, KB = D / 4, NTC = WC / 8;
  static constexpr int XDBL = 3 * D * D;   // A-native, 3 planes
  static constexpr int BDBL = 3 * D * WC;  // B-native, 3 planes
  static constexpr int WMAX = 256;
  static constexpr int THREADS = 32 * WPL * LPC;
  static constexpr int LANE_DBL = 2 * BDBL + (XS ? 2 * XDBL : 0) + WMAX;
  static constexpr size_t SMEM = (size_t)LANE_DBL * LPC * sizeof(double);
  // TMEM columns: per thread 4 blocks (P, T_1..T_3) of 4*NE 32-bit columns;
  // warps w and w+4 share a lane quarter, so column groups = ceil(warps/4)
  static constexpr int NE = MT * NT * 4;
  static constexpr int TMEM_NEED = 16 * NE * ((WPL * LPC + 3) / 4);
  static constexpr int TMEM_COLS = TMEM_NEED <= 32 ? 32 : TMEM_NEED <= 64 ? 64
                                   : TMEM_NEED <= 128 ? 128 : TMEM_NEED <= 256 ? 256 : 512;
  static_assert(TMEM_NEED <= 512, "TMEM budget");
  static_assert(D == WC * GPL, "column blocks must tile D");
  static_assert((S / MT) * (NTC / NT) == WPL, "warp tiling must cover the block");
  static_assert(GPL == 1 || LPC == 1, "groups own one lane per CTA");
};

// element (r, c), plane p (0 re, 1 im, 2 re+im) of the 3-plane A-native layout
__host__ __device__ constexpr int xfrag3_index(int D, int r, int c, int plane) {
  return (((r >> 4) * (D >> 2) + (c >> 2)) * 3 + plane) * 64 + (((r & 7) << 2) | (c & 3)) * 2 +
         ((r >> 3) & 1);
}

// 3-plane B-native layout (swizzled as bfrag_index, kernels.cuh)
template <class C>
__device__ __forceinline__ int bfrag3_index(int r, int n, int plane) {
  return (((r >> 2) * C::NTC + (n >> 3)) * 3 + plane) * 32 + bswz(((n & 7) << 2) + (r & 3));
}

template <class C, bool AG>
__device__ __forceinline__ void tile_mma3(const double* __restrict__ Ag, int a_off, int b_off,
                                          double (&a1)[C::MT * C::NT * 4],
                                          double (&a2)[C::MT * C::NT * 4],
                                          double (&a3)[C::MT * C::NT * 4], int ms0, int nt0,
                                          int ln) {
  extern __shared__ __align__(16) double smem[];
  constexpr int MT = C::MT, NT = C::NT, KB = C::KB;
  auto loadA = [&](int i, int kb, double2 (&v)[3]) {
    const int idx = (((ms0 + i) * KB + kb) * 3) * 64 + 2 * ln;
#pragma unroll
    for (int p = 0; p < 3; ++p) {
      if constexpr (AG)
        v[p] = __ldcg(reinterpret_cast<const double2*>(Ag + idx + 64 * p));
      else
        v[p] = *reinterpret_cast<const double2*>(&smem[a_off + idx + 64 * p]);
    }
  };
  double2 a[MT][3], nx[MT][3];
#pragma unroll
  for (int i = 0; i < MT; ++i) loadA(i, 0, a[i]);
#pragma unroll 2
  for (int kb = 0; kb < KB; ++kb) {
    if (kb + 1 < KB) {
#pragma unroll
      for (int i = 0; i < MT; ++i) loadA(i, kb + 1, nx[i]);
    }
    double b[NT][3];
#pragma unroll
    for (int jn = 0; jn < NT; ++jn) {
      const int bi = b_off + ((kb * C::NTC + nt0 + jn) * 3) * 32 + bswz(ln);
#pragma unroll
      for (int p = 0; p < 3; ++p) b[jn][p] = smem[bi + 32 * p];
    }
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
      for (int jn = 0; jn < NT; ++jn) {
        double* c1 = &a1[(i * NT + jn) * 4];
        double* c2 = &a2[(i * NT + jn) * 4];
        double* c3 = &a3[(i * NT + jn) * 4];
        dmma_16x8x4(c1[0], c1[1], c1[2], c1[3], a[i][0].x, a[i][0].y, b[jn][0]);
        dmma_16x8x4(c2[0], c2[1], c2[2], c2[3], a[i][1].x, a[i][1].y, b[jn][1]);
        dmma_16x8x4(c3[0], c3[1], c3[2], c3[3], a[i][2].x, a[i][2].y, b[jn][2]);
      }
    if (kb + 1 < KB) {
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int p = 0; p < 3; ++p) a[i][p] = nx[i][p];
    }
  }
}

template <class C>
__global__ void __launch_bounds__(C::THREADS, 1)
    lane_ps3_kernel(PSJob pj, const double* __restrict__ terms, int lanes,
                    double* __restrict__ gA, unsigned* __restrict__ gctr,
                    double2* __restrict__ tpriv, double2* __restrict__ lane_out,
                    double2* __restrict__ prefix_out) {
  constexpr int D = C::D, WC = C::WC, MT = C::MT, NT = C::NT, NE = MT * NT * 4;
  constexpr bool AG = !C::XS;
  const SliceJob& job = pj.base;
  extern __shared__ __align__(16) double smem[];
  const int warp = threadIdx.x >> 5, ln = threadIdx.x & 31;
  const int lic = warp / C::WPL;
  const int wil = warp % C::WPL;
  const int tid_l = threadIdx.x - lic * C::WPL * 32;
  constexpr int LT = C::WPL * 32;
  const int group = blockIdx.x / C::GPL;
  const int cb = blockIdx.x % C::GPL;
  const int lane = group * C::LPC + lic;
  const bool active = lane < lanes;

  const int lbase = lic * C::LANE_DBL;
  const int bofs0 = lbase, bofs1 = lbase + C::BDBL;
  const int ax_off = lbase + 2 * C::BDBL;  // XS: 2X, later U
  const int ay_off = ax_off + C::XDBL;     // XS: 2y
  const int w_off = lbase + 2 * C::BDBL + (C::XS ? 2 * C::XDBL : 0);
  double* gx = AG ? gA + (size_t)group * 3 * C::XDBL : nullptr;
  double* gy = AG ? gx + C::XDBL : nullptr;
  double* gu = AG ? gy + C::XDBL : nullptr;
  auto bo = [&](int which) { return which ? bofs1 : bofs0; };

  const int g = ln >> 2, t4 = ln & 3;
  const int ms0 = (wil % (C::S / MT)) * MT;
  const int nt0 = (wil / (C::S / MT)) * NT;
  const int col0 = cb * WC;
  const int s = pj.s, r = pj.r;
  auto row_of = [&](int idx) { return 16 * (ms0 + idx / (NT * 4)) + g + 8 * ((idx & 3) >> 1); };
  auto col_of = [&](int idx) { return 8 * (nt0 + (idx / 4) % NT) + 2 * t4 + (idx & 1); };

  // TMEM: per thread 4*NE columns for the running product P (block 0) and
  // for each power T_1..T_{s-1} (blocks 1..s-1, s <= 4)
  __shared__ uint32_t tmem_slot;
  if (warp == 0) tmem_alloc(&tmem_slot, C::TMEM_COLS);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tmem_base = tmem_slot;
  const uint32_t tmem_me =
      tmem_base + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * 16 * NE);
  auto tm = [&](int blk) { return tmem_me + (uint32_t)(blk * 4 * NE); };

  {
    double pr[NE], pi[NE];
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      pr[e] = (row_of(e) == col0 + col_of(e)) ? 1.0 : 0.0;
      pi[e] = 0.0;
    }
    tmem_store_block<NE>(tm(0), pr, pi);
  }
  (void)tpriv;
  int64_t s0 = 0, s1 = 0;
  if (active) lane_range(job.n_slices, lanes, lane, s0, s1);
  const int T = job.n_terms;
  const bool phase_one = job.phase[0] == 1.0 && job.phase[1] == 0.0;
  unsigned bar = 0;

  auto sync_all = [&]() {
    if constexpr (C::GPL > 1)
      group_barrier(gctr + group, (++bar) * C::GPL);
    else
      lane_sync<C>();
  };
  auto write_B = [&](int off, const double(&vr)[NE], const double(&vi)[NE], double f) {
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      const int rr = row_of(e), n = col_of(e);
      const double xr = f * vr[e], xi = f * vi[e];
      smem[off + bfrag3_index<C>(rr, n, 0)] = xr;
      smem[off + bfrag3_index<C>(rr, n, 1)] = xi;
      smem[off + bfrag3_index<C>(rr, n, 2)] = xr + xi;
    }
  };
  auto write_A = [&](double* gptr, int off, const double(&vr)[NE], const double(&vi)[NE],
                     double fr, double fi) {
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      const int rr = row_of(e), c = col0 + col_of(e);
      const double xr = fr * vr[e] - fi * vi[e], xi = fr * vi[e] + fi * vr[e];
      if constexpr (AG) {
        gptr[xfrag3_index(D, rr, c, 0)] = xr;
        gptr[xfrag3_index(D, rr, c, 1)] = xi;
        gptr[xfrag3_index(D, rr, c, 2)] = xr + xi;
      } else {
        smem[off + xfrag3_index(D, rr, c, 0)] = xr;
        smem[off + xfrag3_index(D, rr, c, 1)] = xi;
        smem[off + xfrag3_index(D, rr, c, 2)] = xr + xi;
      }
    }
  };
  auto load_Q = [&](int j, double(&qr)[NE], double(&qi)[NE]) {
    const double a0r = pj.alpha[2 * (j * s)], a0i = pj.alpha[2 * (j * s) + 1];
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      const bool diag = row_of(e) == col0 + col_of(e);
      qr[e] = diag ? a0r : 0.0;
      qi[e] = diag ? a0i : 0.0;
    }
    for (int i = 1; i < s; ++i) {
      const double ar = pj.alpha[2 * (j * s + i)], ai = pj.alpha[2 * (j * s + i) + 1];
      double tr[NE], ti[NE];
      tmem_load_block<NE>(tm(i), tr, ti);
      const int kind = alpha_kind(pj, j * s + i);
      if (kind == 1) {
#pragma unroll
        for (int e = 0; e < NE; ++e) {
          qr[e] = fma(ar, tr[e], qr[e]);
          qi[e] = fma(ar, ti[e], qi[e]);
        }
      } else if (kind == 2) {
#pragma unroll
        for (int e = 0; e < NE; ++e) {
          qr[e] = fma(-ai, ti[e], qr[e]);
          qi[e] = fma(ai, tr[e], qi[e]);
        }
      } else {
#pragma unroll
        for (int e = 0; e < NE; ++e) {
          qr[e] = fma(ar, tr[e], fma(-ai, ti[e], qr[e]));
          qi[e] = fma(ar, ti[e], fma(ai, tr[e], qi[e]));
        }
      }
    }
  };
  // complex GEMM step: (cr, ci) = (cr, ci) + A * B with the 3M split
  auto step = [&](const double* Ag, int a_off, int b_off, double(&cr)[NE], double(&ci)[NE]) {
    double a1[NE], a2[NE], a3[NE];
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      a1[e] = cr[e];
      a2[e] = 0.0;
      a3[e] = cr[e] + ci[e];
    }
    tile_mma3<C, AG>(Ag, a_off, b_off, a1, a2, a3, ms0, nt0, ln);
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      cr[e] = a1[e] - a2[e];
      ci[e] = (a3[e] - a1[e]) - a2[e];
    }
  };

  for (int64_t sl = s0; sl < s1; ++sl) {
    // ---- 1. weights, 2X assembly (3-plane A layout; terms carry the sum plane)
    for (int tt = tid_l; tt < T; tt += LT)
      smem[w_off + tt] = (tt == 0) ? job.xs : job.xs * slice_weight(job, sl, tt);
    lane_sync<C>();
    {
      int lo, hi, first, stride;
      if constexpr (C::XS) {
        lo = 0; hi = C::XDBL; first = tid_l; stride = LT;
      } else {
        lo = cb * (C::XDBL / C::GPL); hi = lo + C::XDBL / C::GPL;
        first = threadIdx.x; stride = C::THREADS;
      }
      for (int i = lo + 2 * first; i < hi; i += 2 * stride) {
        double2 h = __ldg(reinterpret_cast<const double2*>(terms + i));
        double xr = smem[w_off] * h.x, xi = smem[w_off] * h.y;
        for (int tt = 1; tt < T; ++tt) {
          h = __ldg(reinterpret_cast<const double2*>(terms + (size_t)tt * C::XDBL + i));
          xr = fma(smem[w_off + tt], h.x, xr);
          xi = fma(smem[w_off + tt], h.y, xi);
        }
        if constexpr (AG)
          *reinterpret_cast<double2*>(gx + i) = make_double2(xr, xi);
        else
          *reinterpret_cast<double2*>(&smem[ax_off + i]) = make_double2(xr, xi);
      }
    }
    sync_all();
    // ---- 2. T_1 = X column block
    double accR[NE], accI[NE];
    {
      double t1r[NE], t1i[NE];
#pragma unroll
      for (int e = 0; e < NE; ++e) {
        const int rr = row_of(e), c = col0 + col_of(e);
        const int i0 = xfrag3_index(D, rr, c, 0), i1 = xfrag3_index(D, rr, c, 1);
        t1r[e] = 0.5 * (AG ? __ldcg(gx + i0) : smem[ax_off + i0]);
        t1i[e] = 0.5 * (AG ? __ldcg(gx + i1) : smem[ax_off + i1]);
      }
      tmem_store_block<NE>(tm(1), t1r, t1i);
      write_B(bofs0, t1r, t1i, 1.0);
    }
    lane_sync<C>();
    // ---- 3. powers
    int pb = 0;
    for (int k = 2; k <= s; ++k) {
      if (k == 2) {
#pragma unroll
        for (int e = 0; e < NE; ++e) {
          accR[e] = (row_of(e) == col0 + col_of(e)) ? -1.0 : 0.0;
          accI[e] = 0.0;
        }
      } else {
        tmem_load_block<NE>(tm(k - 2), accR, accI);
#pragma unroll
        for (int e = 0; e < NE; ++e) {
          accR[e] = -accR[e];
          accI[e] = -accI[e];
        }
      }
      step(gx, ax_off, bo(pb), accR, accI);
      if (k < s) {
        write_B(bo(pb ^ 1), accR, accI, 1.0);
        tmem_store_block<NE>(tm(k), accR, accI);
        pb ^= 1;
        lane_sync<C>();
      } else {
        write_A(gy, ay_off, accR, accI, 2.0, 0.0);
      }
    }
    sync_all();
    // ---- 4. Clenshaw in y
    if (r == 1) {
      load_Q(0, accR, accI);
    } else {
      double qr[NE], qi[NE];
      load_Q(r - 1, qr, qi);
      int pc = 0;
      write_B(bo(pc), qr, qi, (r - 1 == 1) ? 0.5 : 1.0);
      lane_sync<C>();
      for (int j = r - 2; j >= 0; --j) {
        load_Q(j, accR, accI);
        if (j + 2 <= r - 1) {
          const int o = bo(pc ^ 1);
#pragma unroll
          for (int e = 0; e < NE; ++e) {
            const int rr = row_of(e), n = col_of(e);
            accR[e] -= smem[o + bfrag3_index<C>(rr, n, 0)];
            accI[e] -= smem[o + bfrag3_index<C>(rr, n, 1)];
          }
        }
        step(gy, ay_off, bo(pc), accR, accI);
        if (j >= 1) {
          write_B(bo(pc ^ 1), accR, accI, (j == 1) ? 0.5 : 1.0);
          pc ^= 1;
          lane_sync<C>();
        }
      }
    }
    write_A(gu, ax_off, accR, accI, phase_one ? 1.0 : job.phase[0],
            phase_one ? 0.0 : job.phase[1]);
    sync_all();
    // ---- 5. V <- U V   (P lives in TMEM between slices)
    tmem_load_block<NE>(tm(0), accR, accI);
    write_B(bofs0, accR, accI, 1.0);
    lane_sync<C>();
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      accR[e] = 0.0;
      accI[e] = 0.0;
    }
    step(gu, ax_off, bofs0, accR, accI);
    tmem_store_block<NE>(tm(0), accR, accI);
    if (prefix_out) {
#pragma unroll
      for (int e = 0; e < NE; ++e)
        store_prefix(prefix_out, D, sl, row_of(e), col0 + col_of(e), accR[e], accI[e]);
    }
    lane_sync<C>();
  }
  if (active) {
    double pr[NE], pi[NE];
    tmem_load_block<NE>(tm(0), pr, pi);
    double2* o = lane_out + (size_t)lane * D * D;
#pragma unroll
    for (int e = 0; e < NE; ++e)
      o[(size_t)row_of(e) * D + col0 + col_of(e)] = make_double2(pr[e], pi[e]);
  }
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  if (warp == 0) tmem_dealloc(tmem_base, C::TMEM_COLS);
}

}  // namespace sp
