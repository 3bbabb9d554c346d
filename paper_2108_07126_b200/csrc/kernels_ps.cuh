// Paterson–Stockmeyer evaluation of the reference's Chebyshev polynomial on
// FP64 tensor cores (the north-star "expm kernel" variant, SURVEY.md §7.1
// item 7), same plan and same truncation as chebyshev.py:259-306.
//
// The plan's series  p(x) = a_0 + sum_{k>=1} 2 a_k T_k(x)  is regrouped in the
// Chebyshev basis as  p(x) = sum_{j<r} Q_j(x) T_j(y),  y = T_s(x),
// Q_j = sum_{i<s} alpha_{j,i} T_i(x)  (T_i T_js = (T_{js+i} + T_{|js-i|})/2;
// alpha from a triangular solve on the host, engine.cu ps_coefficients), and
// evaluated per slice as
//   powers   T_2..T_s      : T_k = 2X T_{k-1} - T_{k-2}            (s-1 GEMMs)
//   Clenshaw in y          : b_j = Q_j + 2y b_{j+1} - b_{j+2},
//                            U = Q_0 + y b_1 - b_2                  (r-1 GEMMs)
//   running product        : V <- U V                               (1 GEMM)
// i.e. s + r - 1 GEMMs per slice instead of the Clenshaw form's m (7 vs 13 at
// m = 13, 7 vs 15 at m = 15).  All operands are polynomials in X, so they
// commute and every GEMM is column-local: CTA j of a lane group computes
// column block j of each product from the full A operand (2X, 2y or U, shared
// through L2 or shared memory) and its own column blocks.
//
// Shared-memory operands are addressed by offsets into the dynamic smem
// array (not through pointer tables) so that every access compiles to
// LDS/STS rather than generic LD/ST.
#pragma once
#include "kernels_tc.cuh"

namespace sp {

constexpr int PS_MAXC = 40;  // max r*s coefficients
#ifndef SP_PS_GROUP_TCAP
#define SP_PS_GROUP_TCAP 0
#endif

// PS needs two A-operand buffers (2X / U, and 2y) when they live in smem,
// plus the private power blocks T_1..T_{s-1} (per thread, accumulator order):
// the first TSB of them in shared memory, as many as fit without lowering the
// CTA residency the registers allow (2 per SM for the smem-resident families,
// 1 for the group families); the rest in global memory (L2)
template <int D_, int WC_, int MT_, int NT_, int WPL_, int LPC_, int GPL_, bool XS_>
struct PSCfg : TCCfg<D_, WC_, MT_, NT_, WPL_, LPC_, GPL_, XS_> {
  using B = TCCfg<D_, WC_, MT_, NT_, WPL_, LPC_, GPL_, XS_>;
  static constexpr int NE = MT_ * NT_ * 4;
  static constexpr int TBLK = 2 * NE * WPL_ * 32;  // doubles of one power block (lane)
  static constexpr int BASE_DBL = 2 * B::BDBL + (XS_ ? 2 * B::XDBL : 0) + B::WMAX;
  static constexpr int CAP = XS_ ? 233472 / 2 - 1024 : SP_PS_GROUP_TCAP;  // bytes per CTA
  static constexpr int TSB = (BASE_DBL + 2 * TBLK) * LPC_ * 8 <= CAP   ? 2
                             : (BASE_DBL + TBLK) * LPC_ * 8 <= CAP ? 1
                                                                   : 0;
  static constexpr int LANE_DBL = BASE_DBL + TSB * TBLK;
  static constexpr size_t SMEM = (size_t)LANE_DBL * LPC_ * sizeof(double);
  static constexpr bool ASW = XS_;
  static_assert(!ASW || B::KB % 2 == 0, "aswz needs an even k-block count");
};

struct PSJob {
  SliceJob base;
  int s, r;
  double alpha[2 * PS_MAXC];  // alpha_{j,i} at (j*s + i), complex
  // alpha_{j,i} is exactly real for even j*s + i and imaginary for odd (the
  // plan's (-i)^k structure survives the regrouping): Q_j accumulates with
  // real-by-complex products
  int alt;
};

// 0: general complex alpha, 1: real, 2: imaginary (uniform per (j, i))
__device__ __forceinline__ int alpha_kind(const PSJob& pj, int q) {
  return pj.alt ? 1 + (q & 1) : 0;
}

// SC, RC > 0: the (s, r) split fixed at compile time (as lane_d8_kernel):
// the power / Clenshaw loops unroll and the power-block locations resolve
template <class C, int SC = 0, int RC = 0>
__global__ void __launch_bounds__(C::THREADS, 1)
    lane_ps_kernel(PSJob pj, const double* __restrict__ terms, int lanes,
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

  // smem offsets (doubles): B ping-pong, A buffers (XS), expansion weights
  const int lbase = lic * C::LANE_DBL;
  const int bofs0 = lbase, bofs1 = lbase + C::BDBL;
  const int ax_off = lbase + 2 * C::BDBL;           // XS: 2X, later U
  const int ay_off = ax_off + C::XDBL;              // XS: 2y
  const int w_off = lbase + 2 * C::BDBL + (C::XS ? 2 * C::XDBL : 0);
  const int t_off = w_off + C::WMAX;               // smem power blocks (TSB of them)
  // global A buffers (group families): 2X, 2y, U
  double* gx = AG ? gA + (size_t)group * 3 * C::XDBL : nullptr;
  double* gy = AG ? gx + C::XDBL : nullptr;
  double* gu = AG ? gy + C::XDBL : nullptr;
  auto bo = [&](int which) { return which ? bofs1 : bofs0; };

  const int g = ln >> 2, t4 = ln & 3;
  const int ms0 = (wil % (C::S / MT)) * MT;
  const int nt0 = (wil / (C::S / MT)) * NT;
  const int col0 = cb * WC;
  const int s = SC > 0 ? SC : pj.s, r = RC > 0 ? RC : pj.r;
  constexpr int UNR = SC > 0 ? 8 : 1;
  // private column blocks of T_1..T_{s-1}, acc-native, coalesced per thread:
  // blocks < TSB in shared memory, the rest in global memory
  auto tp_load = [&](int kk, int e) -> double2 {
    if (kk < C::TSB)
      return *reinterpret_cast<const double2*>(&smem[t_off + kk * C::TBLK + 2 * (e * LT + tid_l)]);
    return __ldcg(&tpriv[(((size_t)blockIdx.x * (s - 1) + kk) * NE + e) * C::THREADS +
                         threadIdx.x]);
  };
  auto tp_store = [&](int kk, int e, double2 v) {
    if (kk < C::TSB)
      *reinterpret_cast<double2*>(&smem[t_off + kk * C::TBLK + 2 * (e * LT + tid_l)]) = v;
    else
      tpriv[(((size_t)blockIdx.x * (s - 1) + kk) * NE + e) * C::THREADS + threadIdx.x] = v;
  };
  auto row_of = [&](int idx) { return 16 * (ms0 + idx / (NT * 4)) + g + 8 * ((idx & 3) >> 1); };
  auto col_of = [&](int idx) { return 8 * (nt0 + (idx / 4) % NT) + 2 * t4 + (idx & 1); };

  double Pr[NE], Pi[NE];
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    Pr[e] = (row_of(e) == col0 + col_of(e)) ? 1.0 : 0.0;
    Pi[e] = 0.0;
  }
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
      smem[off + bfrag_index<C>(rr, n, 0)] = f * vr[e];
      smem[off + bfrag_index<C>(rr, n, 1)] = f * vi[e];
    }
  };
  // A-native write of own positions: smem (XS) or global (group families).
  // A lane's (g, c), (g+8, c), (g, c+1), (g+8, c+1), c = 2 t4, are 4
  // consecutive doubles of one A block: two 16-byte stores per plane (smem,
  // swizzled: conflict-free) or one 32-byte store (global)
  auto write_A = [&](double* gptr, int off, const double(&vr)[NE], const double(&vi)[NE],
                     double fr, double fi) {
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
      for (int jn = 0; jn < NT; ++jn) {
        const int e0 = (i * NT + jn) * 4;
        double xr[4], xi[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          xr[q] = fr * vr[e0 + q] - fi * vi[e0 + q];
          xi[q] = fr * vi[e0 + q] + fi * vr[e0 + q];
        }
        const int c = col0 + 8 * (nt0 + jn) + 2 * t4;
        const int base = (((ms0 + i) * (D >> 2) + (c >> 2)) * 2) * 64 + (g * 4 + (c & 3)) * 2;
        if constexpr (AG) {
          st_global_v4(gptr + base, xr[0], xr[2], xr[1], xr[3]);
          st_global_v4(gptr + base + 64, xi[0], xi[2], xi[1], xi[3]);
        } else {
          *reinterpret_cast<double2*>(&smem[off + aswz(base)]) = make_double2(xr[0], xr[2]);
          *reinterpret_cast<double2*>(&smem[off + aswz(base + 2)]) = make_double2(xr[1], xr[3]);
          *reinterpret_cast<double2*>(&smem[off + aswz(base + 64)]) = make_double2(xi[0], xi[2]);
          *reinterpret_cast<double2*>(&smem[off + aswz(base + 66)]) = make_double2(xi[1], xi[3]);
        }
      }
  };
  // Q_j at own positions: alpha_{j,0} I + sum_{i>=1} alpha_{j,i} T_i
  auto load_Q = [&](int j, double(&qr)[NE], double(&qi)[NE]) {
    const double a0r = pj.alpha[2 * (j * s)], a0i = pj.alpha[2 * (j * s) + 1];
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      const bool diag = row_of(e) == col0 + col_of(e);
      qr[e] = diag ? a0r : 0.0;
      qi[e] = diag ? a0i : 0.0;
    }
#pragma unroll UNR
    for (int i = 1; i < s; ++i) {
      const double ar = pj.alpha[2 * (j * s + i)], ai = pj.alpha[2 * (j * s + i) + 1];
      const int kind = alpha_kind(pj, j * s + i);
      if (kind == 1) {
#pragma unroll
        for (int e = 0; e < NE; ++e) {
          const double2 tv = tp_load(i - 1, e);
          qr[e] = fma(ar, tv.x, qr[e]);
          qi[e] = fma(ar, tv.y, qi[e]);
        }
      } else if (kind == 2) {
#pragma unroll
        for (int e = 0; e < NE; ++e) {
          const double2 tv = tp_load(i - 1, e);
          qr[e] = fma(-ai, tv.y, qr[e]);
          qi[e] = fma(ai, tv.x, qi[e]);
        }
      } else {
#pragma unroll
        for (int e = 0; e < NE; ++e) {
          const double2 tv = tp_load(i - 1, e);
          qr[e] = fma(ar, tv.x, fma(-ai, tv.y, qr[e]));
          qi[e] = fma(ar, tv.y, fma(ai, tv.x, qi[e]));
        }
      }
    }
  };

  // raw samples of weight tid_l (>= 1) of the next slice, loaded a slice ahead
  // (smem-resident families; the group families are at the register limit)
  constexpr bool PFW = C::XS;
  WRaw wr{};
  if (PFW && s0 < s1 && tid_l >= 1 && tid_l < T) wr = weight_gather(job, s0, tid_l);
  PH_INIT
  for (int64_t sl = s0; sl < s1; ++sl) {
    // ---- 1. weights, 2X assembly (A layout)
    if (tid_l < T)
      smem[w_off + tid_l] = (tid_l == 0) ? job.xs
                            : job.xs * (PFW ? weight_combine(job, sl, tid_l, wr)
                                            : slice_weight(job, sl, tid_l));
    for (int tt = tid_l + LT; tt < T; tt += LT)
      smem[w_off + tt] = job.xs * slice_weight(job, sl, tt);
    if (PFW && sl + 1 < s1 && tid_l >= 1 && tid_l < T) wr = weight_gather(job, sl + 1, tid_l);
    lane_sync<C>();
    {
      // QB pairs x 2 terms of loads in flight per thread (L2-latency bound
      // otherwise); summation order as before: term 0, then 1..T-1
      constexpr int CH = C::XS ? C::XDBL : C::XDBL / C::GPL;  // doubles per lane / CTA
      constexpr int STR = C::XS ? LT : C::THREADS;
      constexpr int UPT = CH / (2 * STR);
      constexpr int QB = UPT < 4 ? UPT : 4;
      static_assert(CH % (2 * STR) == 0 && UPT % QB == 0, "assembly tiling");
      const int lo = C::XS ? 0 : cb * CH;
      const int first = C::XS ? tid_l : (int)threadIdx.x;
#pragma unroll 1
      for (int b = 0; b < UPT; b += QB) {
        int idx[QB];
        double2 x[QB];
        const double w0 = smem[w_off];
        auto term = [&](int t, int i) -> double2 {
          return __ldg(reinterpret_cast<const double2*>(terms + (size_t)t * C::XDBL + i));
        };
#pragma unroll
        for (int u = 0; u < QB; ++u) {
          idx[u] = lo + 2 * (first + (b + u) * STR);
          const double2 h = term(0, idx[u]);
          x[u] = make_double2(w0 * h.x, w0 * h.y);
        }
#pragma unroll 1
        for (int tt = 1; tt < T; tt += 2) {
          const bool two = tt + 1 < T;
          double2 h[2][QB];
#pragma unroll
          for (int k = 0; k < 2; ++k)
#pragma unroll
            for (int u = 0; u < QB; ++u)
              if (k == 0 || two) h[k][u] = term(tt + k, idx[u]);
#pragma unroll
          for (int k = 0; k < 2; ++k) {
            if (k == 1 && !two) break;
            const double w = smem[w_off + tt + k];
#pragma unroll
            for (int u = 0; u < QB; ++u) {
              x[u].x = fma(w, h[k][u].x, x[u].x);
              x[u].y = fma(w, h[k][u].y, x[u].y);
            }
          }
        }
#pragma unroll
        for (int u = 0; u < QB; ++u) {
          if constexpr (AG)
            *reinterpret_cast<double2*>(gx + idx[u]) = x[u];
          else
            *reinterpret_cast<double2*>(&smem[ax_off + aswz(idx[u])]) = x[u];
        }
      }
    }
    sync_all();
    PH(0);
    // ---- 2. T_1 = X column block (own positions), to B layout + private
    double accR[NE], accI[NE];
    {
      double t1r[NE], t1i[NE];
#pragma unroll
      for (int e = 0; e < NE; ++e) {
        const int rr = row_of(e), c = col0 + col_of(e);
        const int i0 = xfrag_index(D, rr, c, 0), i1 = xfrag_index(D, rr, c, 1);
        t1r[e] = 0.5 * (AG ? __ldcg(gx + i0) : smem[ax_off + aswz(i0)]);
        t1i[e] = 0.5 * (AG ? __ldcg(gx + i1) : smem[ax_off + aswz(i1)]);
        tp_store(0, e, make_double2(t1r[e], t1i[e]));
      }
      write_B(bofs0, t1r, t1i, 1.0);
    }
    lane_sync<C>();
    PH(1);
    // ---- 3. powers T_k = 2X T_{k-1} - T_{k-2}, k = 2..s
    // (smem-resident families, one strip per warp: 2X / 2y fragments in
    // registers across their GEMMs)
    // (measured: D16 -3.6%, D32 -2.2% at (s, r) = (3, 5); D32 +9% at (2, 4),
    // where one power GEMM does not pay for the registers)
    constexpr bool RA = C::MT == 1 && C::XS && !AG && (C::S == 1 || SC >= 3);
    constexpr int KBR = RA ? C::KB : 1;
    double2 fR[KBR], fI[KBR];
    if constexpr (RA) load_afrag_strip<C>(ax_off, fR, fI, ms0, ln);
    int pb = 0;
#pragma unroll UNR
    for (int k = 2; k <= s; ++k) {
      if (k == 2) {
#pragma unroll
        for (int e = 0; e < NE; ++e) {
          accR[e] = (row_of(e) == col0 + col_of(e)) ? -1.0 : 0.0;
          accI[e] = 0.0;
        }
      } else {
#pragma unroll
        for (int e = 0; e < NE; ++e) {
          const double2 tv = tp_load(k - 3, e);
          accR[e] = -tv.x;
          accI[e] = -tv.y;
        }
      }
      PH(8);
      if constexpr (RA)
        tile_mma_ra<C>(fR, fI, bo(pb), accR, accI, nt0, ln);
      else
        tile_mma<C, AG>(gx, ax_off, bo(pb), accR, accI, ms0, nt0, ln);
      PH(2);
      if (k < s) {
        write_B(bo(pb ^ 1), accR, accI, 1.0);
#pragma unroll
        for (int e = 0; e < NE; ++e) tp_store(k - 1, e, make_double2(accR[e], accI[e]));
        pb ^= 1;
        lane_sync<C>();
      } else {
        write_A(gy, ay_off, accR, accI, 2.0, 0.0);  // 2y = 2 T_s
      }
    }
    PH(8);
    sync_all();
    PH(3);
    if constexpr (RA) load_afrag_strip<C>(ay_off, fR, fI, ms0, ln);
    // ---- 4. Clenshaw in y = T_s with matrix coefficients Q_j
    if (r == 1) {
      load_Q(0, accR, accI);
    } else {
      double qr[NE], qi[NE];
      load_Q(r - 1, qr, qi);
      int pc = 0;
      write_B(bo(pc), qr, qi, (r - 1 == 1) ? 0.5 : 1.0);
      lane_sync<C>();
#pragma unroll UNR
      for (int j = r - 2; j >= 0; --j) {
        load_Q(j, accR, accI);
        if (j + 2 <= r - 1) {
          const int o = bo(pc ^ 1);
#pragma unroll
          for (int e = 0; e < NE; ++e) {
            const int rr = row_of(e), n = col_of(e);
            accR[e] -= smem[o + bfrag_index<C>(rr, n, 0)];
            accI[e] -= smem[o + bfrag_index<C>(rr, n, 1)];
          }
        }
        PH(9);
        if constexpr (RA)
          tile_mma_ra<C>(fR, fI, bo(pc), accR, accI, nt0, ln);
        else
          tile_mma<C, AG>(gy, ay_off, bo(pc), accR, accI, ms0, nt0, ln);
        PH(4);
        if (j >= 1) {
          write_B(bo(pc ^ 1), accR, accI, (j == 1) ? 0.5 : 1.0);
          pc ^= 1;
          lane_sync<C>();
        }
      }
    }
    PH(9);
    // U (times the plan phase, 1 for equiprop's symmetric plans) to A layout;
    // in smem it overwrites 2X, dead since the powers were formed
    write_A(gu, ax_off, accR, accI, phase_one ? 1.0 : job.phase[0],
            phase_one ? 0.0 : job.phase[1]);
    sync_all();
    PH(5);
    // ---- 5. V <- U V
    write_B(bofs0, Pr, Pi, 1.0);
    lane_sync<C>();
    PH(6);
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      accR[e] = 0.0;
      accI[e] = 0.0;
    }
    tile_mma<C, AG>(gu, ax_off, bofs0, accR, accI, ms0, nt0, ln);
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      Pr[e] = accR[e];
      Pi[e] = accI[e];
    }
    PH(7);
    if (prefix_out) {
#pragma unroll
      for (int e = 0; e < NE; ++e)
        store_prefix(prefix_out, D, sl, row_of(e), col0 + col_of(e), Pr[e], Pi[e]);
    }
    // smem A buffers (XS) and B buffers are rewritten by the next slice
    lane_sync<C>();
    PH(5);
  }
  PH_DONE
  if (active) {
    double2* o = lane_out + (size_t)lane * D * D;
#pragma unroll
    for (int e = 0; e < NE; ++e)
      o[(size_t)row_of(e) * D + col0 + col_of(e)] = make_double2(Pr[e], Pi[e]);
  }
}

}  // namespace sp
