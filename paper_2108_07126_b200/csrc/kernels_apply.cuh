// Cumulative propagators on tensor cores (equiprop_all).
//
// The lane kernels write every slice's in-lane prefix P_s = U_s ... U_{s0(l)}
// in the A-native 2-plane layout; the fold kernel forms the exclusive lane
// prefixes E_l = P_{lane l-1} ... P_{lane 0}; this kernel multiplies
// out[s] = P_s E_{lane(s)} with DMMA tiles and writes the d x d top-left block
// in the caller's dtype (fusing the extraction).  A CTA owns one column block
// of E (B layout, smem) and a contiguous run of slices, reloading E only when
// the run crosses into the next lane.  The same kernel forms the sequential
// total P_{L-1} E_{L-1}, which keeps equiprop_all's last entry bitwise equal
// to reduction="sequential" (reference property propagator.py:304-306).
#pragma once
#include "kernels_tc.cuh"

namespace sp {

__device__ __forceinline__ int64_t lane_of_slice(int64_t s, int64_t n, int lanes) {
  // largest l with l*n/lanes <= s  (inverse of lane_range)
  int64_t l = ((s + 1) * lanes - 1) / n;
  while (l > 0 && l * n / lanes > s) --l;
  while (l + 1 < lanes && (l + 1) * n / lanes <= s) ++l;
  return l;
}

template <class C>
__global__ void __launch_bounds__(C::THREADS)
    apply_prefix_tc_kernel(const double* __restrict__ P, const double2* __restrict__ E,
                           int64_t n, int lanes, int64_t spb, int d, int to_fp32,
                           void* __restrict__ out) {
  static_assert(C::LPC == 1, "one lane per CTA");
  constexpr int D = C::D, WC = C::WC, MT = C::MT, NT = C::NT, NE = MT * NT * 4;
  extern __shared__ __align__(16) double smem[];
  const int warp = threadIdx.x >> 5, ln = threadIdx.x & 31;
  const int g = ln >> 2, t4 = ln & 3;
  const int ms0 = (warp % (C::S / MT)) * MT;
  const int nt0 = (warp / (C::S / MT)) * NT;
  const int col0 = blockIdx.y * WC;
  auto row_of = [&](int idx) { return 16 * (ms0 + idx / (NT * 4)) + g + 8 * ((idx & 3) >> 1); };
  auto col_of = [&](int idx) { return 8 * (nt0 + (idx / 4) % NT) + 2 * t4 + (idx & 1); };

  const int64_t s0 = blockIdx.x * spb;
  const int64_t s1 = min(n, s0 + spb);
  int64_t cur = -1;
  for (int64_t s = s0; s < s1; ++s) {
    const int64_t l = lane_of_slice(s, n, lanes);
    if (l != cur) {
      __syncthreads();
      const double2* El = E + (size_t)l * D * D;
      for (int q = threadIdx.x; q < D * WC; q += C::THREADS) {
        const int k = q / WC, c = q % WC;
        const double2 v = El[(size_t)k * D + col0 + c];
        smem[bfrag_index<C>(k, c, 0)] = v.x;
        smem[bfrag_index<C>(k, c, 1)] = v.y;
      }
      __syncthreads();
      cur = l;
    }
    double accR[NE], accI[NE];
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      accR[e] = 0.0;
      accI[e] = 0.0;
    }
    tile_mma<C, true>(P + (size_t)s * 2 * D * D, 0, 0, accR, accI, ms0, nt0, ln);
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      const int r = row_of(e), c = col0 + col_of(e);
      if (r < d && c < d) {
        const size_t o = (size_t)s * d * d + (size_t)r * d + c;
        if (to_fp32)
          reinterpret_cast<float2*>(out)[o] = make_float2((float)accR[e], (float)accI[e]);
        else
          reinterpret_cast<double2*>(out)[o] = make_double2(accR[e], accI[e]);
      }
    }
  }
}

// row-major complex D x D -> A-native 2-plane layout (exact copy)
__global__ void to_afrag_kernel(const double2* __restrict__ in, int D, double* __restrict__ out) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < D * D; e += gridDim.x * blockDim.x) {
    const int r = e / D, c = e % D;
    out[xfrag_index(D, r, c, 0)] = in[e].x;
    out[xfrag_index(D, r, c, 1)] = in[e].y;
  }
}

}  // namespace sp
