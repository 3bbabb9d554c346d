// Family D8 (5 <= d <= 8): one warp per lane on the FP64 m8n8k4 tensor-core
// MMA (mma.sync .m8n8k4 .f64, SASS DMMA.8x8x4).  An 8 x 8 complex product is
// two k steps of 4 (4 real products each, or 3 with the 3-multiplication
// form), so an 8 x 8 system runs without the 8x flop padding of the D16
// family.  Every operand lives in the warp's shared-memory slot; the running
// product V, the power blocks T_i and the Clenshaw iterates live in
// registers at the thread's accumulator positions (row g = lane/4, columns
// 2 (lane%4) + {0, 1}).
//
// Same plan polynomial, same three series schemes as the larger families:
//   Clenshaw  (chebyshev.py:298-303 applied to V, as lane_small_kernel)
//   PS        (kernels_ps.cuh: powers, Clenshaw in y = T_s, V <- U V)
//   PS3       (PS with 3-multiplication complex products)
// Lane products and cumulative prefixes are written in the plain row-major
// layout of the small families, so the ordered tree / fold / prefix kernels
// are shared with them.
#pragma once
#include "kernels_ps.cuh"

namespace sp {

enum D8Alg { D8_CLENSHAW = 0, D8_PS = 1, D8_PS3 = 2 };

// doubles per warp: XA, YA, B0, B1 (np planes of 64) + 256 weights
__host__ __device__ constexpr int d8_slot(int np) { return 4 * 64 * np + 256; }
constexpr int D8_TSM = 16;              // expansion terms kept in shared memory (per CTA)
#ifndef SP_D8_TR
#define SP_D8_TR 4  // expansion terms kept in registers (lane entries)
#endif

// m8n8k4 fragment-native positions (0..63) of element (r, c)
__device__ __forceinline__ int d8_apos(int r, int c) { return (c >> 2) * 32 + ((r << 2) | (c & 3)); }
__device__ __forceinline__ int d8_bpos(int r, int c) { return (r >> 2) * 32 + ((c << 2) | (r & 3)); }

__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

// acc (own 2 complex entries) += A B for 8 x 8 complex A (A-native planes at
// A) and B (B-native planes at B); planes: re, im[, re + im]
template <bool M3>
__device__ __forceinline__ void d8_mma(const double* A, const double* B, double (&cr)[2],
                                       double (&ci)[2], int ln) {
  if constexpr (M3) {
    double a1[2] = {cr[0], cr[1]}, a2[2] = {0.0, 0.0};
    double a3[2] = {cr[0] + ci[0], cr[1] + ci[1]};
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      const int i = ks * 32 + ln;
      dmma_8x8x4(a1[0], a1[1], A[i], B[i]);
      dmma_8x8x4(a2[0], a2[1], A[64 + i], B[64 + i]);
      dmma_8x8x4(a3[0], a3[1], A[128 + i], B[128 + i]);
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      cr[j] = a1[j] - a2[j];
      ci[j] = (a3[j] - a1[j]) - a2[j];
    }
  } else {
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      const int i = ks * 32 + ln;
      const double ar = A[i], ai = A[64 + i], br = B[i], bi = B[64 + i];
      dmma_8x8x4(cr[0], cr[1], ar, br);
      dmma_8x8x4(ci[0], ci[1], ar, bi);
      dmma_8x8x4(cr[0], cr[1], -ai, bi);
      dmma_8x8x4(ci[0], ci[1], ai, br);
    }
  }
}

// the same with the A operand's fragments already in registers
// (af[ks][plane] = A[plane * 64 + ks * 32 + lane]): 2X and 2y are the A
// operand of several GEMMs of a slice
template <bool M3>
__device__ __forceinline__ void d8_mma_ra(const double (&af)[2][3], const double* B,
                                          double (&cr)[2], double (&ci)[2], int ln) {
  if constexpr (M3) {
    double a1[2] = {cr[0], cr[1]}, a2[2] = {0.0, 0.0};
    double a3[2] = {cr[0] + ci[0], cr[1] + ci[1]};
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      const int i = ks * 32 + ln;
      dmma_8x8x4(a1[0], a1[1], af[ks][0], B[i]);
      dmma_8x8x4(a2[0], a2[1], af[ks][1], B[64 + i]);
      dmma_8x8x4(a3[0], a3[1], af[ks][2], B[128 + i]);
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      cr[j] = a1[j] - a2[j];
      ci[j] = (a3[j] - a1[j]) - a2[j];
    }
  } else {
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      const int i = ks * 32 + ln;
      const double ar = af[ks][0], ai = af[ks][1], br = B[i], bi = B[64 + i];
      dmma_8x8x4(cr[0], cr[1], ar, br);
      dmma_8x8x4(ci[0], ci[1], ar, bi);
      dmma_8x8x4(cr[0], cr[1], -ai, bi);
      dmma_8x8x4(ci[0], ci[1], ai, br);
    }
  }
}

// SC, RC > 0: the Paterson-Stockmeyer split (s, r) fixed at compile time
// (m = 13 -> (3, 5), m = 15 -> (4, 4), m = 7 -> (2, 4)): every loop over the
// powers and the Clenshaw steps unrolls, so coefficient loads, buffer
// toggles and loop control become immediates; 0 = runtime (other orders)
template <int WPC, int ALG, int SC = 0, int RC = 0>
__global__ void __launch_bounds__(32 * WPC) lane_d8_kernel(PSJob pj,
                                                          const double2* __restrict__ terms,
                                                          int lanes,
                                                          double2* __restrict__ lane_out,
                                                          double2* __restrict__ prefix_out) {
  constexpr bool M3 = ALG == D8_PS3;
  constexpr int NP = M3 ? 3 : 2;  // operand planes
  // 2X / 2y fragments kept in registers across their GEMMs (measured: -4% at
  // (s, r) = (3, 5), +4% at (2, 4))
  constexpr bool RA = SC >= 3;
  extern __shared__ __align__(16) double smem[];
  const SliceJob& job = pj.base;
  const int warp = threadIdx.x >> 5, ln = threadIdx.x & 31;
  const int lane = blockIdx.x * WPC + warp;
  constexpr int PL = 64 * NP, SLOT = d8_slot(NP);
  double* XA = smem + warp * SLOT;  // 2X, later U (A-native)
  double* YA = XA + PL;             // 2y (A-native)
  auto Bb = [&](int i) { return XA + 2 * PL + PL * i; };  // B-native ping-pong
  double* W = XA + 4 * PL;          // weights
  double2* TS = reinterpret_cast<double2*>(smem + WPC * SLOT);  // terms (T <= D8_TSM)
  const int g = ln >> 2, c0 = 2 * (ln & 3);
  const int bp[2] = {d8_bpos(g, c0), d8_bpos(g, c0 + 1)};
  const int ap[2] = {d8_apos(g, c0), d8_apos(g, c0 + 1)};
  const bool dg[2] = {g == c0, g == c0 + 1};

  auto writeB = [&](double* B, const double(&vr)[2], const double(&vi)[2], double f) {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const double xr = f * vr[j], xi = f * vi[j];
      B[bp[j]] = xr;
      B[64 + bp[j]] = xi;
      if constexpr (M3) B[128 + bp[j]] = xr + xi;
    }
  };
  auto writeA = [&](double* A, const double(&vr)[2], const double(&vi)[2], double fr,
                    double fi) {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const double xr = fr * vr[j] - fi * vi[j], xi = fr * vi[j] + fi * vr[j];
      A[ap[j]] = xr;
      A[64 + ap[j]] = xi;
      if constexpr (M3) A[128 + ap[j]] = xr + xi;
    }
  };

  double Vr[2], Vi[2];
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    Vr[j] = dg[j] ? 1.0 : 0.0;
    Vi[j] = 0.0;
  }
  int64_t s0 = 0, s1 = 0;
  if (lane < lanes) lane_range(job.n_slices, lanes, lane, s0, s1);
  const int T = job.n_terms;
  const bool phase_one = job.phase[0] == 1.0 && job.phase[1] == 0.0;
  const int s = SC > 0 ? SC : pj.s, r = RC > 0 ? RC : pj.r, m = job.m;
  // the CTA's warps share one shared-memory copy of the expansion terms
  const bool tsm = T <= D8_TSM;
  if (tsm)
    for (int i = threadIdx.x; i < T * 64; i += blockDim.x) TS[i] = __ldg(&terms[i]);
  __syncthreads();
  const double2* tsrc = tsm ? TS : terms;
  // raw samples of weight ln (>= 1) of the next slice, loaded a slice ahead
  WRaw wr{};
  if (s0 < s1 && ln >= 1 && ln < T) wr = weight_gather(job, s0, ln);
  // up to TR terms: the lane's own entries of every term stay in registers
  // for the whole lane and the weights travel by shuffles (no shared-memory
  // round trip on the assembly's critical path)
  constexpr int TR = SP_D8_TR;
  const bool treg = T <= TR;
  double2 hreg[TR][2];
#pragma unroll
  for (int tt = 0; tt < TR; ++tt)
#pragma unroll
    for (int ks = 0; ks < 2; ++ks)
      hreg[tt][ks] = (treg && tt < T) ? tsrc[tt * 64 + ks * 32 + ln] : make_double2(0.0, 0.0);

  for (int64_t sl = s0; sl < s1; ++sl) {
    // ---- weights (xs folded in) and 2X (A-native, NP planes)
    double myw = 0.0;
    if (ln < T) myw = (ln == 0) ? job.xs : job.xs * weight_combine(job, sl, ln, wr);
    if (!treg) {
      if (ln < T) W[ln] = myw;
      for (int tt = ln + 32; tt < T; tt += 32) W[tt] = job.xs * slice_weight(job, sl, tt);
    }
    if (sl + 1 < s1 && ln >= 1 && ln < T) wr = weight_gather(job, sl + 1, ln);
    __syncwarp();
    double wv[TR];
#pragma unroll
    for (int tt = 0; tt < TR; ++tt) wv[tt] = __shfl_sync(0xffffffffu, myw, tt);
    double afx[2][3];  // this thread's fragments of 2X (it assembles exactly those)
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      const int i = ks * 32 + ln;
      double xr, xi;
      if (treg) {
        xr = wv[0] * hreg[0][ks].x;
        xi = wv[0] * hreg[0][ks].y;
#pragma unroll
        for (int tt = 1; tt < TR; ++tt) {
          if (tt >= T) break;
          xr = fma(wv[tt], hreg[tt][ks].x, xr);
          xi = fma(wv[tt], hreg[tt][ks].y, xi);
        }
      } else {
        double2 h = tsrc[i];
        xr = W[0] * h.x;
        xi = W[0] * h.y;
#pragma unroll 4
        for (int tt = 1; tt < T; ++tt) {
          h = tsrc[tt * 64 + i];
          xr = fma(W[tt], h.x, xr);
          xi = fma(W[tt], h.y, xi);
        }
      }
      XA[i] = xr;
      XA[64 + i] = xi;
      afx[ks][0] = xr;
      afx[ks][1] = xi;
      afx[ks][2] = xr + xi;
      if constexpr (NP == 3) XA[128 + i] = afx[ks][2];
    }
    __syncwarp();
    double accR[2], accI[2];
    if constexpr (ALG == D8_CLENSHAW) {
      // b_m = a_m V; b_j = a_j V + 2X b_{j+1} - (j = 0 ? 2 : 1) b_{j+2}
      double cr[2], ci[2], orr[2] = {0.0, 0.0}, oi[2] = {0.0, 0.0};
      {
        const double ar = job.coef[2 * m], ai = job.coef[2 * m + 1];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          cr[j] = ar * Vr[j] - ai * Vi[j];
          ci[j] = ar * Vi[j] + ai * Vr[j];
        }
      }
      int pb = 0;
      for (int jj = m - 1; jj >= 0; --jj) {
        const double ar = job.coef[2 * jj], ai = job.coef[2 * jj + 1];
        const double beta = (jj == 0) ? 2.0 : 1.0;
        writeB(Bb(pb), cr, ci, 1.0);
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          accR[j] = fma(ar, Vr[j], fma(-ai, Vi[j], -beta * orr[j]));
          accI[j] = fma(ar, Vi[j], fma(ai, Vr[j], -beta * oi[j]));
        }
        d8_mma<false>(XA, Bb(pb), accR, accI, ln);
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          orr[j] = cr[j];
          oi[j] = ci[j];
          cr[j] = accR[j];
          ci[j] = accI[j];
        }
        pb ^= 1;
      }
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        if (phase_one) {
          Vr[j] = cr[j];
          Vi[j] = ci[j];
        } else {
          Vr[j] = job.phase[0] * cr[j] - job.phase[1] * ci[j];
          Vi[j] = job.phase[0] * ci[j] + job.phase[1] * cr[j];
        }
      }
    } else {
      // ---- Paterson-Stockmeyer (kernels_ps.cuh), power blocks in registers
      double Tr[4][2], Ti[4][2];  // T_1 .. T_{s-1} (s <= 4)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        Tr[0][j] = 0.5 * XA[ap[j]];
        Ti[0][j] = 0.5 * XA[64 + ap[j]];
      }
      writeB(Bb(0), Tr[0], Ti[0], 1.0);
      __syncwarp();
      int pb = 0;
#pragma unroll
      for (int k = 2; k <= 4; ++k) {  // constant indices keep T_i in registers
        if (k > s) break;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          if (k == 2) {
            accR[j] = dg[j] ? -1.0 : 0.0;
            accI[j] = 0.0;
          } else {
            accR[j] = -Tr[k - 3][j];
            accI[j] = -Ti[k - 3][j];
          }
        }
        if constexpr (RA)
          d8_mma_ra<M3>(afx, Bb(pb), accR, accI, ln);
        else
          d8_mma<M3>(XA, Bb(pb), accR, accI, ln);
        if (k < s) {
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            Tr[k - 1][j] = accR[j];
            Ti[k - 1][j] = accI[j];
          }
          writeB(Bb(pb ^ 1), accR, accI, 1.0);
          pb ^= 1;
          __syncwarp();
        }
      }
      writeA(YA, accR, accI, 2.0, 0.0);  // 2y = 2 T_s
      __syncwarp();
      double afy[2][3] = {};
      if constexpr (RA) {
#pragma unroll
        for (int ks = 0; ks < 2; ++ks)
#pragma unroll
          for (int p = 0; p < NP; ++p) afy[ks][p] = YA[p * 64 + ks * 32 + ln];
      }
      auto loadQ = [&](int j, double(&qr)[2], double(&qi)[2]) {
        const double a0r = pj.alpha[2 * (j * s)], a0i = pj.alpha[2 * (j * s) + 1];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          qr[e] = dg[e] ? a0r : 0.0;
          qi[e] = dg[e] ? a0i : 0.0;
        }
#pragma unroll
        for (int i = 1; i < 4; ++i) {
          if (i >= s) break;
          const double ar = pj.alpha[2 * (j * s + i)], ai = pj.alpha[2 * (j * s + i) + 1];
          const int kind = alpha_kind(pj, j * s + i);
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            if (kind == 1) {
              qr[e] = fma(ar, Tr[i - 1][e], qr[e]);
              qi[e] = fma(ar, Ti[i - 1][e], qi[e]);
            } else if (kind == 2) {
              qr[e] = fma(-ai, Ti[i - 1][e], qr[e]);
              qi[e] = fma(ai, Tr[i - 1][e], qi[e]);
            } else {
              qr[e] = fma(ar, Tr[i - 1][e], fma(-ai, Ti[i - 1][e], qr[e]));
              qi[e] = fma(ar, Ti[i - 1][e], fma(ai, Tr[i - 1][e], qi[e]));
            }
          }
        }
      };
      // ---- Clenshaw in y with matrix coefficients Q_j (b_{j+1}, b_{j+2} in registers)
      if (r == 1) {
        loadQ(0, accR, accI);
      } else {
        double b1r[2], b1i[2], b2r[2] = {0.0, 0.0}, b2i[2] = {0.0, 0.0};
        loadQ(r - 1, b1r, b1i);
        int pc = 0;
        writeB(Bb(pc), b1r, b1i, (r - 1 == 1) ? 0.5 : 1.0);
        __syncwarp();
#pragma unroll
        for (int j = r - 2; j >= 0; --j) {
          loadQ(j, accR, accI);
          if (j + 2 <= r - 1) {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              accR[e] -= b2r[e];
              accI[e] -= b2i[e];
            }
          }
          if constexpr (RA)
            d8_mma_ra<M3>(afy, Bb(pc), accR, accI, ln);
          else
            d8_mma<M3>(YA, Bb(pc), accR, accI, ln);
          if (j >= 1) {
            writeB(Bb(pc ^ 1), accR, accI, (j == 1) ? 0.5 : 1.0);
            pc ^= 1;
            __syncwarp();
          }
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            b2r[e] = b1r[e];
            b2i[e] = b1i[e];
            b1r[e] = accR[e];
            b1i[e] = accI[e];
          }
        }
      }
      // U (times the plan phase) over 2X (dead since the powers), V <- U V
      __syncwarp();  // every thread is done reading the last B operand
      writeA(XA, accR, accI, phase_one ? 1.0 : job.phase[0], phase_one ? 0.0 : job.phase[1]);
      writeB(Bb(0), Vr, Vi, 1.0);
      __syncwarp();
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        accR[j] = 0.0;
        accI[j] = 0.0;
      }
      d8_mma<M3>(XA, Bb(0), accR, accI, ln);
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        Vr[j] = accR[j];
        Vi[j] = accI[j];
      }
    }
    if (prefix_out) {
      double2* o = prefix_out + (size_t)sl * 64;
#pragma unroll
      for (int j = 0; j < 2; ++j) o[g * 8 + c0 + j] = make_double2(Vr[j], Vi[j]);
    }
    __syncwarp();  // the next slice rewrites the slot
  }
  if (lane < lanes) {
    double2* o = lane_out + (size_t)lane * 64;
#pragma unroll
    for (int j = 0; j < 2; ++j) o[g * 8 + c0 + j] = make_double2(Vr[j], Vi[j]);
  }
}

}  // namespace sp
