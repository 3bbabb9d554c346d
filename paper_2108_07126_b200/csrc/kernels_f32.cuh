// complex64 contexts in complex64 arithmetic: the lane kernel of the plain
// families (d <= 8) on the FP32 pipe (FFMA, 2x the FP64 DFMA rate on B200).
//
// The reference's fp32 mode (sliceprop linalg.py:38-72, chebyshev.py:293,
// hamiltonian.py:186-207) computes everything in complex64: the expansion
// terms and the float64 weight table are cast to complex64, the exponent is
// G = scale (T_0 + sum_t w_t T_t) (drift broadcast, controls accumulated,
// real scale multiplied in float32), X = G * float(2 / span), and the
// Clenshaw recurrence runs in complex64 with the plan's coefficients cast to
// complex64.  This kernel follows that sequence per slice, on chip:
//
//   lane = D consecutive threads; thread c owns column c of the running
//   product V and of the Clenshaw iterates, both in registers
//   per slice:  X[:, c]  assembled in float32 -> the lane's smem X
//               U[:, c]  = p(X) e_c  by the reference's two-step Clenshaw
//                          recurrence (chebyshev.py:294-303), in float32
//               V[:, c] <- U V[:, c]  (U read back from the lane's smem)
//
// The lane products (and, for equiprop_all, the in-lane prefixes) are
// written in the shared plain D x D layout as complex128 (exact widening),
// so the ordered lane combination, the prefix scan and the output
// conversion are the plain families' (their lane combination runs in
// FP64: a lane holds n / lanes >= 16 slices, so the complex64 rounding of
// the lane loop dominates, as it does in the reference's fp32 fold).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.h"

namespace sp {

// weight of expansion term t >= 1 for slice s in float64 (the reference's
// table is float64, cast to complex64 afterwards); validates the samples
// when `val` (one thread per lane does)
__device__ __forceinline__ double f32_weight(const SliceJob& j, int64_t s, int t, bool val) {
  const int N = j.n_ctrl;
  if (j.mode == SP_MODE_MIDPOINT) {
    const double v = j.amps[s * N + (t - 1)];
    if (val) check_amp(j, s, t - 1, v);
    return v;
  }
  if (j.mode >= SP_MODE_GAUSS2) {  // Gauss-Legendre modes: rows 2s, 2s + 1
    const double* ra = j.amps + (2 * s) * N;
    const double* rb = ra + N;
    int e = t - 1;
    if (e < N) {
      if (val) {
        check_amp(j, 2 * s, e, ra[e]);
        check_amp(j, 2 * s + 1, e, rb[e]);
      }
      return 0.5 * (ra[e] + rb[e]);
    }
    e -= N;
    if (e < N) return j.gl * (rb[e] - ra[e]);
    int k, kp;
    cross_pair(e - N, N, k, kp);
    return j.gl * (ra[k] * rb[kp] - ra[kp] * rb[k]);
  }
  const double* r1 = j.amps + (2 * s) * N;
  const double* r2 = r1 + N;
  const double* r3 = r2 + N;
  int e = t - 1;
  if (e < N) {
    if (val) {
      check_amp(j, 2 * s, e, r1[e]);
      check_amp(j, 2 * s + 1, e, r2[e]);
      check_amp(j, 2 * s + 2, e, r3[e]);
    }
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

// c += a b in float32 (naive complex product with FMAs)
__device__ __forceinline__ void cfma32(float2& c, const float2 a, const float2 b) {
  c.x = fmaf(a.x, b.x, c.x);
  c.x = fmaf(-a.y, b.y, c.x);
  c.y = fmaf(a.x, b.y, c.y);
  c.y = fmaf(a.y, b.x, c.y);
}

constexpr int F32_THREADS = 256;

// dynamic smem: terms (T x D x D float2) + per lane X and U (2 x D x D float2)
template <int D>
constexpr size_t f32_smem_bytes(int n_terms) {
  return ((size_t)n_terms + (size_t)(F32_THREADS / D) * 2) * D * D * sizeof(float2);
}

template <int D>
__global__ void __launch_bounds__(F32_THREADS) lane_f32_kernel(SliceJob job,
                                                               const double2* __restrict__ terms,
                                                               int lanes,
                                                               double2* __restrict__ lane_out,
                                                               double2* __restrict__ prefix_out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int LPC = F32_THREADS / D;
  const int T = job.n_terms;
  float2* sterm = reinterpret_cast<float2*>(smem_raw);                 // T x D x D
  float2* slane = sterm + (size_t)T * D * D;                            // per lane X, U
  // terms cast to complex64 once per CTA (linalg.py:273-274); the device
  // copy is plain D x D for D <= 4 and in the m8n8k4 A-fragment order of the
  // D8 family (engine.cu upload_terms) for D = 8
  for (int e = threadIdx.x; e < T * D * D; e += blockDim.x) {
    const int t = e / (D * D), rc = e - t * D * D, r = rc / D, c = rc - r * D;
    const int src = D == 8 ? (c >> 2) * 32 + ((r << 2) | (c & 3)) : rc;
    const double2 v = terms[(size_t)t * D * D + src];
    sterm[e] = make_float2((float)v.x, (float)v.y);
  }
  __syncthreads();
  const int local = threadIdx.x / D;
  const int c = threadIdx.x % D;
  const int lane = blockIdx.x * LPC + local;
  float2* X = slane + (size_t)local * 2 * D * D;  // X[r * D + k]
  float2* U = X + D * D;                          // U[r * D + k]
  int64_t s0 = 0, s1 = 0;
  if (lane < lanes) lane_range(job.n_slices, lanes, lane, s0, s1);
  float2 V[D];
#pragma unroll
  for (int r = 0; r < D; ++r) V[r] = make_float2(r == c ? 1.0f : 0.0f, 0.0f);
  const float scale = (float)job.scale;
  const float xs = (float)job.xspan;
  const int m = job.m;
  const bool phase_one = job.phase[0] == 1.0 && job.phase[1] == 0.0;
  const float2 ph = make_float2((float)job.phase[0], (float)job.phase[1]);
  const bool val = c == 0;
  // lanes differ by at most one slice: the warp runs its longest lane's
  // count, the shorter lanes idle through the last iteration (the warp
  // barriers below need every thread)
  const int cnt = (int)(s1 - s0);
  const int wmax = __reduce_max_sync(0xffffffffu, cnt);
  for (int it = 0; it < wmax; ++it) {
    const bool act = it < cnt;
    const int64_t s = s0 + it;
    // X[:, c] = float(2 / span) * (scale * (T_0 + sum_t w_t T_t))[:, c]
    float2 g[D], ctl[D];
#pragma unroll
    for (int r = 0; r < D; ++r) {
      g[r] = sterm[r * D + c];
      ctl[r] = make_float2(0.0f, 0.0f);
    }
    for (int t = 1; t < (act ? T : 1); ++t) {
      const float w = (float)f32_weight(job, s, t, val);
      const float2* Ht = sterm + (size_t)t * D * D;
#pragma unroll
      for (int r = 0; r < D; ++r) {
        const float2 h = Ht[r * D + c];
        ctl[r].x = fmaf(w, h.x, ctl[r].x);
        ctl[r].y = fmaf(w, h.y, ctl[r].y);
      }
    }
    __syncwarp();  // the previous slice's readers of X / U are done
#pragma unroll
    for (int r = 0; r < D; ++r) {
      float2 v = make_float2((g[r].x + ctl[r].x) * scale, (g[r].y + ctl[r].y) * scale);
      v.x *= xs;
      v.y *= xs;
      X[r * D + c] = v;
    }
    __syncwarp();
    // U[:, c] = p(X) e_c: D1 <- 2 X D0 - D1 + a_k e_c; D0 <- 2 X D1 - cc D0 + a' e_c
    float2 d0[D], d1[D];
#pragma unroll
    for (int r = 0; r < D; ++r) d0[r] = d1[r] = make_float2(0.0f, 0.0f);
    bool first = true;
    for (int k = m; k >= 1; k -= 2) {
      const float2 ak = make_float2((float)job.coef[2 * k], (float)job.coef[2 * k + 1]);
      float2 acc[D];
#pragma unroll
      for (int r = 0; r < D; ++r) acc[r] = make_float2(0.0f, 0.0f);
      if (!first) {
#pragma unroll
        for (int q = 0; q < D; ++q) {
          const float2 b = d0[q];
#pragma unroll
          for (int r = 0; r < D; ++r) cfma32(acc[r], X[r * D + q], b);
        }
      }
      first = false;
#pragma unroll
      for (int r = 0; r < D; ++r) {
        float2 v = make_float2(-d1[r].x + 2.0f * acc[r].x, -d1[r].y + 2.0f * acc[r].y);
        if (r == c) {
          v.x += ak.x;
          v.y += ak.y;
        }
        d1[r] = v;
      }
      const bool last = k == 1;
      const float cc = last ? 2.0f : 1.0f;
      const int k2 = last ? 0 : k - 1;
      const float2 ap = make_float2((float)job.coef[2 * k2], (float)job.coef[2 * k2 + 1]);
#pragma unroll
      for (int r = 0; r < D; ++r) acc[r] = make_float2(0.0f, 0.0f);
#pragma unroll
      for (int q = 0; q < D; ++q) {
        const float2 b = d1[q];
#pragma unroll
        for (int r = 0; r < D; ++r) cfma32(acc[r], X[r * D + q], b);
      }
#pragma unroll
      for (int r = 0; r < D; ++r) {
        float2 v = make_float2(-cc * d0[r].x + 2.0f * acc[r].x, -cc * d0[r].y + 2.0f * acc[r].y);
        if (r == c) {
          v.x += ap.x;
          v.y += ap.y;
        }
        d0[r] = v;
      }
    }
#pragma unroll
    for (int r = 0; r < D; ++r) {
      float2 u = d0[r];
      if (!phase_one) u = make_float2(u.x * ph.x - u.y * ph.y, u.x * ph.y + u.y * ph.x);
      U[r * D + c] = u;
    }
    __syncwarp();
    // V[:, c] <- U V[:, c]
    float2 nv[D];
#pragma unroll
    for (int r = 0; r < D; ++r) nv[r] = make_float2(0.0f, 0.0f);
#pragma unroll
    for (int q = 0; q < D; ++q) {
      const float2 b = V[q];
#pragma unroll
      for (int r = 0; r < D; ++r) cfma32(nv[r], U[r * D + q], b);
    }
    if (!act) continue;
#pragma unroll
    for (int r = 0; r < D; ++r) V[r] = nv[r];
    if (prefix_out) {
      double2* o = prefix_out + (size_t)s * D * D;
#pragma unroll
      for (int r = 0; r < D; ++r) o[r * D + c] = make_double2(V[r].x, V[r].y);
    }
  }
  if (lane < lanes) {
    double2* o = lane_out + (size_t)lane * D * D;
#pragma unroll
    for (int r = 0; r < D; ++r) o[r * D + c] = make_double2(V[r].x, V[r].y);
  }
}

// D = 2 with one thread per lane: the same per-column arithmetic as
// lane_f32_kernel<2> (each column of U = p(X) e_c is computed by the
// identical operation sequence, so results are bitwise those of the two-
// thread form), with X, the Clenshaw iterates, U and V in registers — no
// shared-memory round trips or warp barriers per slice.  (Two slices in
// lockstep as well: the compiler contracts the iterate updates differently —
// no longer bitwise the two-thread form — and 1e7 slices ran 8 % slower.)
__global__ void __launch_bounds__(F32_THREADS, 2) lane_f32_reg2_kernel(SliceJob job,
                                                                    const double2* __restrict__ terms,
                                                                    int lanes,
                                                                    double2* __restrict__ lane_out,
                                                                    double2* __restrict__ prefix_out) {
  constexpr int D = 2;
  const int T = job.n_terms;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float2* sterm = reinterpret_cast<float2*>(smem_raw);  // T x 2 x 2, cast once per CTA
  for (int e = threadIdx.x; e < T * D * D; e += blockDim.x) {
    const double2 v = terms[e];
    sterm[e] = make_float2((float)v.x, (float)v.y);
  }
  __syncthreads();
  const int lane = blockIdx.x * blockDim.x + threadIdx.x;
  int64_t s0 = 0, s1 = 0;
  if (lane < lanes) lane_range(job.n_slices, lanes, lane, s0, s1);
  float2 V[D][D];  // V[r][c]
#pragma unroll
  for (int r = 0; r < D; ++r)
#pragma unroll
    for (int c = 0; c < D; ++c) V[r][c] = make_float2(r == c ? 1.0f : 0.0f, 0.0f);
  const float scale = (float)job.scale;
  const float xs = (float)job.xspan;
  const int m = job.m;
  const bool phase_one = job.phase[0] == 1.0 && job.phase[1] == 0.0;
  const float2 ph = make_float2((float)job.phase[0], (float)job.phase[1]);
  for (int64_t s = s0; s < s1; ++s) {
    // X = float(2 / span) * (scale * (T_0 + sum_t w_t T_t)), per column as
    // the two-thread form forms it
    float2 X[D][D];
    {
      float2 ctl[D][D];
#pragma unroll
      for (int r = 0; r < D; ++r)
#pragma unroll
        for (int c = 0; c < D; ++c) ctl[r][c] = make_float2(0.0f, 0.0f);
      for (int t = 1; t < T; ++t) {
        const float w = (float)f32_weight(job, s, t, true);
        const float2* Ht = sterm + (size_t)t * D * D;
#pragma unroll
        for (int r = 0; r < D; ++r)
#pragma unroll
          for (int c = 0; c < D; ++c) {
            const float2 h = Ht[r * D + c];
            ctl[r][c].x = fmaf(w, h.x, ctl[r][c].x);
            ctl[r][c].y = fmaf(w, h.y, ctl[r][c].y);
          }
      }
#pragma unroll
      for (int r = 0; r < D; ++r)
#pragma unroll
        for (int c = 0; c < D; ++c) {
          const float2 g = sterm[r * D + c];
          float2 v = make_float2((g.x + ctl[r][c].x) * scale, (g.y + ctl[r][c].y) * scale);
          v.x *= xs;
          v.y *= xs;
          X[r][c] = v;
        }
    }
    // U[:, c] = p(X) e_c for both columns, the two columns' Clenshaw
    // recurrences advanced in lockstep (two independent dependency chains;
    // each column's operation sequence is unchanged)
    float2 U[D][D];
    {
      float2 d0[D][D], d1[D][D];  // [column][row]
#pragma unroll
      for (int c = 0; c < D; ++c)
#pragma unroll
        for (int r = 0; r < D; ++r) d0[c][r] = d1[c][r] = make_float2(0.0f, 0.0f);
      bool first = true;
      for (int k = m; k >= 1; k -= 2) {
        const float2 ak = make_float2((float)job.coef[2 * k], (float)job.coef[2 * k + 1]);
        const bool last = k == 1;
        const float cc = last ? 2.0f : 1.0f;
        const int k2 = last ? 0 : k - 1;
        const float2 ap = make_float2((float)job.coef[2 * k2], (float)job.coef[2 * k2 + 1]);
#pragma unroll
        for (int c = 0; c < D; ++c) {
          float2 acc[D];
#pragma unroll
          for (int r = 0; r < D; ++r) acc[r] = make_float2(0.0f, 0.0f);
          if (!first) {
#pragma unroll
            for (int q = 0; q < D; ++q) {
              const float2 b = d0[c][q];
#pragma unroll
              for (int r = 0; r < D; ++r) cfma32(acc[r], X[r][q], b);
            }
          }
#pragma unroll
          for (int r = 0; r < D; ++r) {
            float2 v = make_float2(-d1[c][r].x + 2.0f * acc[r].x, -d1[c][r].y + 2.0f * acc[r].y);
            if (r == c) {
              v.x += ak.x;
              v.y += ak.y;
            }
            d1[c][r] = v;
          }
#pragma unroll
          for (int r = 0; r < D; ++r) acc[r] = make_float2(0.0f, 0.0f);
#pragma unroll
          for (int q = 0; q < D; ++q) {
            const float2 b = d1[c][q];
#pragma unroll
            for (int r = 0; r < D; ++r) cfma32(acc[r], X[r][q], b);
          }
#pragma unroll
          for (int r = 0; r < D; ++r) {
            float2 v = make_float2(-cc * d0[c][r].x + 2.0f * acc[r].x,
                                   -cc * d0[c][r].y + 2.0f * acc[r].y);
            if (r == c) {
              v.x += ap.x;
              v.y += ap.y;
            }
            d0[c][r] = v;
          }
        }
        first = false;
      }
#pragma unroll
      for (int c = 0; c < D; ++c)
#pragma unroll
        for (int r = 0; r < D; ++r) {
          float2 u = d0[c][r];
          if (!phase_one) u = make_float2(u.x * ph.x - u.y * ph.y, u.x * ph.y + u.y * ph.x);
          U[r][c] = u;
        }
    }
    // V[:, c] <- U V[:, c]
    float2 nv[D][D];
#pragma unroll
    for (int c = 0; c < D; ++c) {
#pragma unroll
      for (int r = 0; r < D; ++r) nv[r][c] = make_float2(0.0f, 0.0f);
#pragma unroll
      for (int q = 0; q < D; ++q) {
        const float2 b = V[q][c];
#pragma unroll
        for (int r = 0; r < D; ++r) cfma32(nv[r][c], U[r][q], b);
      }
    }
#pragma unroll
    for (int r = 0; r < D; ++r)
#pragma unroll
      for (int c = 0; c < D; ++c) V[r][c] = nv[r][c];
    if (prefix_out) {
      double2* o = prefix_out + (size_t)s * D * D;
#pragma unroll
      for (int r = 0; r < D; ++r)
#pragma unroll
        for (int c = 0; c < D; ++c) o[r * D + c] = make_double2(V[r][c].x, V[r][c].y);
    }
  }
  if (lane < lanes) {
    double2* o = lane_out + (size_t)lane * D * D;
#pragma unroll
    for (int r = 0; r < D; ++r)
#pragma unroll
      for (int c = 0; c < D; ++c) o[r * D + c] = make_double2(V[r][c].x, V[r][c].y);
  }
}

}  // namespace sp
