// FP64 tensor-core tile product and the Clenshaw-form lane kernel.
//
// tile_mma is the one DMMA inner loop every tensor-core lane kernel uses:
// acc(own 16x8 tiles) += A * B over the full k range with A in the A-native
// fragment layout (global memory through L2, or shared memory) and B in the
// B-native layout in shared memory.  Shared operands are addressed by offsets
// into the dynamic smem array so every access compiles to LDS/STS.
#pragma once
#include "kernels.cuh"

namespace sp {

template <class C, bool AG>
__device__ __forceinline__ void tile_mma(const double* __restrict__ Ag, int a_off, int b_off,
                                         double (&accR)[C::MT * C::NT * 4],
                                         double (&accI)[C::MT * C::NT * 4], int ms0, int nt0,
                                         int ln) {
  extern __shared__ __align__(16) double smem[];
  constexpr int MT = C::MT, NT = C::NT, KB = C::KB;
  auto loadA = [&](int i, int kb, double2& re, double2& im) {
    const int idx = (((ms0 + i) * KB + kb) * 2) * 64 + 2 * ln;
    if constexpr (AG) {
      re = __ldcg(reinterpret_cast<const double2*>(Ag + idx));
      im = __ldcg(reinterpret_cast<const double2*>(Ag + idx + 64));
    } else {
      const int pi = C::ASW ? aswz(idx) : idx;
      re = *reinterpret_cast<const double2*>(&smem[a_off + pi]);
      im = *reinterpret_cast<const double2*>(&smem[a_off + pi + 64]);
    }
  };
  double2 aR[MT], aI[MT], nR[MT], nI[MT];
#pragma unroll
  for (int i = 0; i < MT; ++i) loadA(i, 0, aR[i], aI[i]);
#pragma unroll 2
  for (int kb = 0; kb < KB; ++kb) {
    if (kb + 1 < KB) {
#pragma unroll
      for (int i = 0; i < MT; ++i) loadA(i, kb + 1, nR[i], nI[i]);
    }
    double bR[NT], bI[NT];
#pragma unroll
    for (int jn = 0; jn < NT; ++jn) {
      const int bi = b_off + ((kb * C::NTC + nt0 + jn) * 2) * 32 + bswz(ln);
      bR[jn] = smem[bi];
      bI[jn] = smem[bi + 32];
    }
    // two passes: MMAs into the same accumulator are 2*MT*NT instructions
    // apart; the -B_im operand negation folds into the DMMA instruction
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
      for (int jn = 0; jn < NT; ++jn) {
        double* cr = &accR[(i * NT + jn) * 4];
        double* ci = &accI[(i * NT + jn) * 4];
        dmma_16x8x4(cr[0], cr[1], cr[2], cr[3], aR[i].x, aR[i].y, bR[jn]);
        dmma_16x8x4(ci[0], ci[1], ci[2], ci[3], aR[i].x, aR[i].y, bI[jn]);
      }
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
      for (int jn = 0; jn < NT; ++jn) {
        double* cr = &accR[(i * NT + jn) * 4];
        double* ci = &accI[(i * NT + jn) * 4];
        dmma_16x8x4(cr[0], cr[1], cr[2], cr[3], aI[i].x, aI[i].y, -bI[jn]);
        dmma_16x8x4(ci[0], ci[1], ci[2], ci[3], aI[i].x, aI[i].y, bR[jn]);
      }
    if (kb + 1 < KB) {
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        aR[i] = nR[i];
        aI[i] = nI[i];
      }
    }
  }
}

// tile_mma for one 16-row strip per warp (MT = 1) whose A fragments are
// already in registers (aR/aI[kb] = the lane's re/im pair of k block kb):
// 2X and 2y are the A operand of several GEMMs per slice
template <class C>
__device__ __forceinline__ void load_afrag_strip(int a_off, double2 (&aR)[C::KB],
                                                 double2 (&aI)[C::KB], int ms0, int ln) {
  extern __shared__ __align__(16) double smem[];
#pragma unroll
  for (int kb = 0; kb < C::KB; ++kb) {
    const int idx0 = ((ms0 * C::KB + kb) * 2) * 64 + 2 * ln;
    const int idx = C::ASW ? aswz(idx0) : idx0;
    aR[kb] = *reinterpret_cast<const double2*>(&smem[a_off + idx]);
    aI[kb] = *reinterpret_cast<const double2*>(&smem[a_off + idx + 64]);
  }
}

template <class C>
__device__ __forceinline__ void tile_mma_ra(const double2 (&aR)[C::KB],
                                            const double2 (&aI)[C::KB], int b_off,
                                            double (&accR)[C::NT * 4],
                                            double (&accI)[C::NT * 4], int nt0, int ln) {
  static_assert(C::MT == 1, "one strip per warp");
  extern __shared__ __align__(16) double smem[];
  constexpr int NT = C::NT, KB = C::KB;
#pragma unroll
  for (int kb = 0; kb < KB; ++kb) {
    double bR[NT], bI[NT];
#pragma unroll
    for (int jn = 0; jn < NT; ++jn) {
      const int bi = b_off + ((kb * C::NTC + nt0 + jn) * 2) * 32 + bswz(ln);
      bR[jn] = smem[bi];
      bI[jn] = smem[bi + 32];
    }
#pragma unroll
    for (int jn = 0; jn < NT; ++jn) {
      double* cr = &accR[jn * 4];
      double* ci = &accI[jn * 4];
      dmma_16x8x4(cr[0], cr[1], cr[2], cr[3], aR[kb].x, aR[kb].y, bR[jn]);
      dmma_16x8x4(ci[0], ci[1], ci[2], ci[3], aR[kb].x, aR[kb].y, bI[jn]);
    }
#pragma unroll
    for (int jn = 0; jn < NT; ++jn) {
      double* cr = &accR[jn * 4];
      double* ci = &accI[jn * 4];
      dmma_16x8x4(cr[0], cr[1], cr[2], cr[3], aI[kb].x, aI[kb].y, -bI[jn]);
      dmma_16x8x4(ci[0], ci[1], ci[2], ci[3], aI[kb].x, aI[kb].y, bR[jn]);
    }
  }
}

// Clenshaw form (the reference's recurrence applied to the running product):
// b_m = a_m V ; b_j = a_j V + 2X b_{j+1} - (j == 0 ? 2 : 1) b_{j+2} ; V = b_0.
// m GEMMs per slice; see kernels.cuh for the lane/group structure.
template <class C>
__global__ void __launch_bounds__(C::THREADS, 1)
    lane_tc_kernel(SliceJob job, const double* __restrict__ terms, int lanes,
                   double* __restrict__ xglob, unsigned* __restrict__ gctr,
                   double2* __restrict__ lane_out, double2* __restrict__ prefix_out) {
  constexpr int D = C::D, WC = C::WC, MT = C::MT, NT = C::NT, NE = MT * NT * 4;
  constexpr bool AG = !C::XS;
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
  const int x_off = lbase + 2 * C::BDBL;
  const int w_off = x_off + (C::XS ? C::XDBL : 0);
  auto bo = [&](int which) { return lbase + (which ? C::BDBL : 0); };

  const int g = ln >> 2, t4 = ln & 3;
  const int ms0 = (wil % (C::S / MT)) * MT;
  const int nt0 = (wil / (C::S / MT)) * NT;
  const int col0 = cb * WC;
  auto row_of = [&](int idx) { return 16 * (ms0 + idx / (NT * 4)) + g + 8 * ((idx & 3) >> 1); };
  auto col_of = [&](int idx) { return 8 * (nt0 + (idx / 4) % NT) + 2 * t4 + (idx & 1); };

  double Vr[NE], Vi[NE];
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    Vr[e] = (row_of(e) == col0 + col_of(e)) ? 1.0 : 0.0;
    Vi[e] = 0.0;
  }
  int64_t s0 = 0, s1 = 0;
  if (active) lane_range(job.n_slices, lanes, lane, s0, s1);
  const int T = job.n_terms, m = job.m;
  const bool phase_one = job.phase[0] == 1.0 && job.phase[1] == 0.0;
  int p = 0;  // buffer bo(p) holds the current iterate
  unsigned iter = 0;

  for (int64_t s = s0; s < s1; ++s, ++iter) {
    // ---- 1. expansion weights (scaled by 2*scale/beta)
    for (int tt = tid_l; tt < T; tt += LT)
      smem[w_off + tt] = (tt == 0) ? job.xs : job.xs * slice_weight(job, s, tt);
    lane_sync<C>();
    // ---- 2. assemble 2X in the A-native layout (smem, or this CTA's share
    //         of the group's double-buffered L2 copy)
    double* xg = AG ? xglob + ((size_t)group * 2 + (iter & 1)) * C::XDBL : nullptr;
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
          *reinterpret_cast<double2*>(xg + i) = make_double2(xr, xi);
        else
          *reinterpret_cast<double2*>(&smem[x_off + i]) = make_double2(xr, xi);
      }
    }
    // ---- 3. b_m = a_m V into the current buffer
    {
      const double ar = job.coef[2 * m], ai = job.coef[2 * m + 1];
      const int B = bo(p);
#pragma unroll
      for (int e = 0; e < NE; ++e) {
        const int rr = row_of(e), n = col_of(e);
        smem[B + bfrag_index<C>(rr, n, 0)] = ar * Vr[e] - ai * Vi[e];
        smem[B + bfrag_index<C>(rr, n, 1)] = ar * Vi[e] + ai * Vr[e];
      }
    }
    if constexpr (C::GPL > 1)
      group_barrier(gctr + group, (iter + 1) * C::GPL);
    else
      lane_sync<C>();

    // ---- 4. m Clenshaw steps: new = 2X cur - beta old + a_j V
    // (2X fragments in registers for the m GEMMs: measured -1..2% at m = 13
    // but +1.6% at m = 3, the orders this kernel runs under "auto"; off)
    constexpr bool RA = false;
    constexpr int KBR = RA ? C::KB : 1;
    double2 fR[KBR], fI[KBR];
    if constexpr (RA) load_afrag_strip<C>(x_off, fR, fI, ms0, ln);
    for (int jj = m - 1; jj >= 0; --jj) {
      const double ar = job.coef[2 * jj], ai = job.coef[2 * jj + 1];
      const int Bo = bo(p ^ 1);
      double accR[NE], accI[NE];
      const bool first = (jj == m - 1);
      const double beta = (jj == 0) ? 2.0 : 1.0;
#pragma unroll
      for (int e = 0; e < NE; ++e) {
        double orr = 0.0, oi = 0.0;
        if (!first) {
          const int rr = row_of(e), n = col_of(e);
          orr = smem[Bo + bfrag_index<C>(rr, n, 0)];
          oi = smem[Bo + bfrag_index<C>(rr, n, 1)];
        }
        accR[e] = fma(ar, Vr[e], fma(-ai, Vi[e], -beta * orr));
        accI[e] = fma(ar, Vi[e], fma(ai, Vr[e], -beta * oi));
      }
      if constexpr (RA)
        tile_mma_ra<C>(fR, fI, bo(p), accR, accI, nt0, ln);
      else
        tile_mma<C, AG>(xg, x_off, bo(p), accR, accI, ms0, nt0, ln);
      if (jj > 0) {
        // new iterate becomes "cur" for the next step (own positions only)
#pragma unroll
        for (int e = 0; e < NE; ++e) {
          const int rr = row_of(e), n = col_of(e);
          smem[Bo + bfrag_index<C>(rr, n, 0)] = accR[e];
          smem[Bo + bfrag_index<C>(rr, n, 1)] = accI[e];
        }
        p ^= 1;
        lane_sync<C>();
      } else {
#pragma unroll
        for (int e = 0; e < NE; ++e) {
          if (phase_one) {
            Vr[e] = accR[e];
            Vi[e] = accI[e];
          } else {
            Vr[e] = job.phase[0] * accR[e] - job.phase[1] * accI[e];
            Vi[e] = job.phase[0] * accI[e] + job.phase[1] * accR[e];
          }
        }
        // the next slice writes b_m into bo(p^1) (only own positions were
        // read there); flip so that it is the next slice's current buffer
        p ^= 1;
      }
    }
    if (prefix_out) {
#pragma unroll
      for (int e = 0; e < NE; ++e)
        store_prefix(prefix_out, D, s, row_of(e), col0 + col_of(e), Vr[e], Vi[e]);
    }
    // X (smem) and the weights are rewritten by the next slice
    if constexpr (C::GPL == 1) lane_sync<C>();
  }
  if (active) {
    double2* o = lane_out + (size_t)lane * D * D;
#pragma unroll
    for (int e = 0; e < NE; ++e)
      o[(size_t)row_of(e) * D + col0 + col_of(e)] = make_double2(Vr[e], Vi[e]);
  }
}

}  // namespace sp
