// Group-family (D >= 64, operands shared through L2) Paterson–Stockmeyer
// lane kernel with 3-multiplication complex products and TMEM-resident
// running product / power blocks — the production kernel for the C4 headline
// (d = 128).  Same arithmetic as lane_ps3_kernel (kernels_ps3.cuh); the
// slice loop is restructured to cut the non-MMA time per slice:
//
//  * column-block ownership of the shared operands: CTA j of a lane group
//    assembles and publishes COLUMN block j of 2X, 2y and U (the same blocks
//    its GEMMs produce), so T_1 = X[:, J] comes from its own shared memory;
//  * two group barriers per slice instead of three: the next slice's 2X is
//    assembled during the current slice's Clenshaw phase (its buffer is dead
//    once the powers are formed), so "U ready" and "next X ready" share one
//    barrier;
//  * the first A fragments of the next GEMM step are loaded during the last
//    k-block of the current one whenever that operand is already published;
//  * 2y and U are staged in shared memory in publication order and copied to
//    L2 with coalesced 16-byte stores.
//
// Per slice: 1 assembly, s-1 power GEMMs, r-1 Clenshaw GEMMs, 1 product GEMM,
// 2 group barriers.
#pragma once
#include "kernels_ps3.cuh"

namespace sp {


// tile_mma3 with cross-step prefetch: a holds the kb = 0 fragments on entry;
// on exit it holds the kb = 0 fragments of An (if An != nullptr)
template <class C>
__device__ __forceinline__ void tile_mma3_pf(const double* __restrict__ Ag,
                                             const double* __restrict__ An, int b_off,
                                             double2 (&a)[C::MT][3],
                                             double (&a1)[C::MT * C::NT * 4],
                                             double (&a2)[C::MT * C::NT * 4],
                                             double (&a3)[C::MT * C::NT * 4], int ms0, int nt0,
                                             int ln) {
  extern __shared__ __align__(16) double smem[];
  constexpr int MT = C::MT, NT = C::NT, KB = C::KB;
  auto loadA = [&](const double* A, int i, int kb, double2 (&v)[3]) {
    const int idx = (((ms0 + i) * KB + kb) * 3) * 64 + 2 * ln;
#pragma unroll
    for (int p = 0; p < 3; ++p) v[p] = __ldcg(reinterpret_cast<const double2*>(A + idx + 64 * p));
  };
  double2 nx[MT][3];
#pragma unroll 2
  for (int kb = 0; kb < KB; ++kb) {
    if (kb + 1 < KB) {
#pragma unroll
      for (int i = 0; i < MT; ++i) loadA(Ag, i, kb + 1, nx[i]);
    } else if (An != nullptr) {
#pragma unroll
      for (int i = 0; i < MT; ++i) loadA(An, i, 0, nx[i]);
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
    if (kb + 1 < KB || An != nullptr) {
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int p = 0; p < 3; ++p) a[i][p] = nx[i][p];
    }
  }
}

template <class C>
__global__ void __launch_bounds__(C::THREADS, 1)
    lane_ps3g_kernel(PSJob pj, const double* __restrict__ terms, int lanes,
                     double* __restrict__ gA, unsigned* __restrict__ gctr,
                     double2* __restrict__ tpriv, double2* __restrict__ lane_out,
                     double2* __restrict__ prefix_out) {
  // GPL == 1: a lane is one CTA owning every column (D = 64); its shared
  // operands still go through the L2 exchange buffer, and the group
  // barriers reduce to CTA barriers
  static_assert(C::LPC == 1 && !C::XS, "group configuration");
  constexpr int D = C::D, WC = C::WC, MT = C::MT, NT = C::NT, NE = MT * NT * 4;
  constexpr int KB = C::KB;
  constexpr int KBC = WC / 4;                 // k-blocks of one column block
  const SliceJob& job = pj.base;
  extern __shared__ __align__(16) double smem[];
  const int warp = threadIdx.x >> 5, ln = threadIdx.x & 31;
  const int group = blockIdx.x / C::GPL;
  const int cb = blockIdx.x % C::GPL;
  const int lane = group;
  const bool active = lane < lanes;

  const int bofs0 = 0, bofs1 = C::BDBL;
  const int w_off = 2 * C::BDBL;
  auto bo = [&](int which) { return which ? bofs1 : bofs0; };
  double* gx = gA + (size_t)group * 3 * C::XDBL;
  double* gy = gx + C::XDBL;
  double* gu = gy + C::XDBL;

  const int g = ln >> 2, t4 = ln & 3;
  const int ms0 = (warp % (C::S / MT)) * MT;
  const int nt0 = (warp / (C::S / MT)) * NT;
  const int col0 = cb * WC;
  const int s = pj.s, r = pj.r;
  auto row_of = [&](int idx) { return 16 * (ms0 + idx / (NT * 4)) + g + 8 * ((idx & 3) >> 1); };
  auto col_of = [&](int idx) { return 8 * (nt0 + (idx / 4) % NT) + 2 * t4 + (idx & 1); };

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
  auto gsync = [&]() {
    if constexpr (C::GPL > 1)
      group_barrier(gctr + group, (++bar) * C::GPL);
    else
      __syncthreads();
  };
  // split form: CTA-local work between the arrival and the wait
  auto garrive = [&]() {
    if constexpr (C::GPL > 1)
      group_arrive(gctr + group);
    else
      __syncthreads();
  };
  auto gwait = [&]() {
    if constexpr (C::GPL > 1)
      group_wait(gctr + group, (++bar) * C::GPL);
    else
      __syncthreads();
  };

  // weights of slice sl, then this CTA's column chunk of 2X (3-plane A
  // layout, L2) from the 2-plane terms, and T_1 = X[:, J] (B layout) into
  // smem at t1_off.  One unit = one lane's pair of A-fragment elements (rows
  // 16 strip + l/4 and +8, column 4 kbl + l%4); two terms of QB units are in
  // flight per thread (the loop is L2-latency bound otherwise).
  constexpr int UNITS = C::S * KBC * 32;
  constexpr int UPT = UNITS / C::THREADS;
  constexpr int QB = UPT < 4 ? UPT : (C::MT >= 4 ? 2 : 4);  // (D512: register budget)
  static_assert(UNITS % C::THREADS == 0 && UPT % QB == 0, "assembly tiling");
  constexpr size_t TD = (size_t)2 * D * D;  // doubles per 2-plane term
  // (s = 3: TMEM block 3 is free — the powers are T_1, T_2 — and holds the
  // scaled drift xs H0 of this thread's units for the whole call: the
  // per-slice assembly reads one term fewer from L2.  8 columns per unit.)
  static_assert(UPT * 8 == 4 * NE && QB % 2 == 0, "drift block in TMEM");
  const bool drift_tm = s == 3;
  auto unit_blk = [&](int unit) {
    return (unit / (KBC * 32)) * KB + cb * KBC + (unit / 32) % KBC;
  };
  if (drift_tm) {
#pragma unroll 1
    for (int b = 0; b < UPT; b += 2) {
      double re[4], im[4];
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const double* h = terms + (size_t)unit_blk(threadIdx.x + (b + v) * C::THREADS) * 128 +
                          2 * ln;
        const double2 hr = __ldg(reinterpret_cast<const double2*>(h));
        const double2 hi = __ldg(reinterpret_cast<const double2*>(h + 64));
        re[2 * v] = job.xs * hr.x;
        re[2 * v + 1] = job.xs * hr.y;
        im[2 * v] = job.xs * hi.x;
        im[2 * v + 1] = job.xs * hi.y;
      }
      tmem_st4(tm(3) + 8 * b, re, im);
    }
    tmem_wait_st();
  }
  auto assemble = [&](int64_t sl, int t1_off) {
    for (int tt = threadIdx.x; tt < T; tt += C::THREADS)
      smem[w_off + tt] = (tt == 0) ? job.xs : job.xs * slice_weight(job, sl, tt);
    __syncthreads();
#pragma unroll 1
    for (int b = 0; b < UPT; b += QB) {
      int blk[QB];
      double2 xr[QB], xi[QB];
#pragma unroll
      for (int u = 0; u < QB; ++u) blk[u] = unit_blk(threadIdx.x + (b + u) * C::THREADS);
      if (drift_tm) {  // xs H0 (the drift's weight is xs) from TMEM
        uint32_t w[QB / 2][16];
#pragma unroll
        for (int v = 0; v < QB / 2; ++v) tmem_ld16(tm(3) + 8 * (b + 2 * v), w[v]);
        tmem_wait_ld();
#pragma unroll
        for (int v = 0; v < QB / 2; ++v) {
          double re[4], im[4];
          tmem_unpack4(w[v], re, im);
          xr[2 * v] = make_double2(re[0], re[1]);
          xr[2 * v + 1] = make_double2(re[2], re[3]);
          xi[2 * v] = make_double2(im[0], im[1]);
          xi[2 * v + 1] = make_double2(im[2], im[3]);
        }
      } else {
        const double w = smem[w_off];
#pragma unroll
        for (int u = 0; u < QB; ++u) {
          const double* h = terms + (size_t)blk[u] * 128 + 2 * ln;
          const double2 hr = __ldg(reinterpret_cast<const double2*>(h));
          const double2 hi = __ldg(reinterpret_cast<const double2*>(h + 64));
          xr[u] = make_double2(w * hr.x, w * hr.y);
          xi[u] = make_double2(w * hi.x, w * hi.y);
        }
      }
#pragma unroll 1
      for (int tt = 1; tt < T; tt += 2) {
        const bool two = tt + 1 < T;
        double2 hr[2][QB], hi[2][QB];
#pragma unroll
        for (int k = 0; k < 2; ++k)
#pragma unroll
          for (int u = 0; u < QB; ++u) {
            if (k == 0 || two) {
              const double* h = terms + (size_t)(tt + k) * TD + (size_t)blk[u] * 128 + 2 * ln;
              hr[k][u] = __ldg(reinterpret_cast<const double2*>(h));
              hi[k][u] = __ldg(reinterpret_cast<const double2*>(h + 64));
            }
          }
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          if (k == 1 && !two) break;
          const double w = smem[w_off + tt + k];
#pragma unroll
          for (int u = 0; u < QB; ++u) {
            xr[u].x = fma(w, hr[k][u].x, xr[u].x);
            xr[u].y = fma(w, hr[k][u].y, xr[u].y);
            xi[u].x = fma(w, hi[k][u].x, xi[u].x);
            xi[u].y = fma(w, hi[k][u].y, xi[u].y);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < QB; ++u) {
        const int unit = threadIdx.x + (b + u) * C::THREADS;
        double* o = gx + (size_t)blk[u] * 192 + 2 * ln;
        *reinterpret_cast<double2*>(o) = xr[u];
        *reinterpret_cast<double2*>(o + 64) = xi[u];
        *reinterpret_cast<double2*>(o + 128) =
            make_double2(xr[u].x + xi[u].x, xr[u].y + xi[u].y);
        const int rw = 16 * (unit / (KBC * 32)) + (ln >> 2);
        const int n = 4 * ((unit / 32) % KBC) + (ln & 3);
        smem[t1_off + bfrag3_index<C>(rw, n, 0)] = 0.5 * xr[u].x;
        smem[t1_off + bfrag3_index<C>(rw, n, 1)] = 0.5 * xi[u].x;
        smem[t1_off + bfrag3_index<C>(rw, n, 2)] = 0.5 * (xr[u].x + xi[u].x);
        smem[t1_off + bfrag3_index<C>(rw + 8, n, 0)] = 0.5 * xr[u].y;
        smem[t1_off + bfrag3_index<C>(rw + 8, n, 1)] = 0.5 * xi[u].y;
        smem[t1_off + bfrag3_index<C>(rw + 8, n, 2)] = 0.5 * (xr[u].y + xi[u].y);
      }
    }
  };
  // own elements straight from the accumulator fragments into the 3-plane A
  // layout: a lane's (g, c), (g+8, c), (g, c+1), (g+8, c+1) for c = 2 t4
  // are 4 consecutive doubles of one A block (one full 32-byte sector), so
  // every store is a 256-bit st.global.v4.f64 and a warp instruction writes
  // two whole 512-byte blocks — no staging buffer, no CTA barrier
  auto publish = [&](double* dst, const double(&vr)[NE], const double(&vi)[NE], double fr,
                     double fi) {
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
        double* o = dst + ((((ms0 + i) * KB + (c >> 2)) * 3) * 64 + (g * 4 + (c & 3)) * 2);
        const uint64_t pol = l2_policy_evict_last();
        st_global_v4_hint(o, xr[0], xr[2], xr[1], xr[3], pol);
        st_global_v4_hint(o + 64, xi[0], xi[2], xi[1], xi[3], pol);
        st_global_v4_hint(o + 128, xr[0] + xi[0], xr[2] + xi[2], xr[1] + xi[1], xr[3] + xi[3],
                          pol);
      }
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
#pragma unroll
      for (int e = 0; e < NE; ++e) {
        qr[e] = fma(ar, tr[e], fma(-ai, ti[e], qr[e]));
        qi[e] = fma(ar, ti[e], fma(ai, tr[e], qi[e]));
      }
    }
  };
  double2 afr[MT][3];  // kb = 0 A fragments of the next GEMM step
  auto first_frags = [&](const double* A) {
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
      for (int p = 0; p < 3; ++p)
        afr[i][p] = __ldcg(reinterpret_cast<const double2*>(
            A + (((ms0 + i) * KB) * 3 + p) * 64 + 2 * ln));
  };
  auto step = [&](const double* Ag, const double* An, int b_off, double(&cr)[NE],
                  double(&ci)[NE]) {
    double a1[NE], a2[NE], a3[NE];
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      a1[e] = cr[e];
      a2[e] = 0.0;
      a3[e] = cr[e] + ci[e];
    }
    tile_mma3_pf<C>(Ag, An, b_off, afr, a1, a2, a3, ms0, nt0, ln);
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      cr[e] = a1[e] - a2[e];
      ci[e] = (a3[e] - a1[e]) - a2[e];
    }
  };

  PH_INIT
  int tb = 0;  // buffer holding this slice's T_1 (written by assemble)
  if (s0 < s1) {
    assemble(s0, bo(tb));
    gsync();
    first_frags(gx);
  }
  for (int64_t sl = s0; sl < s1; ++sl) {
    const bool more = sl + 1 < s1;
    double accR[NE], accI[NE];
    // ---- T_1 (own positions) from the B-layout copy written by assemble()
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      const int rr = row_of(e), n = col_of(e);
      accR[e] = smem[bo(tb) + bfrag3_index<C>(rr, n, 0)];
      accI[e] = smem[bo(tb) + bfrag3_index<C>(rr, n, 1)];
    }
    tmem_store_block<NE>(tm(1), accR, accI);
    PH(0);
    // ---- powers T_k = 2X T_{k-1} - T_{k-2}
    int pb = tb;
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
      step(gx, k < s ? gx : nullptr, bo(pb), accR, accI);
      if (k < s) {
        write_B(bo(pb ^ 1), accR, accI, 1.0);
        tmem_store_block<NE>(tm(k), accR, accI);
        pb ^= 1;
        __syncthreads();
      }
    }
    // 2y = 2 T_s
    PH(1);
    publish(gy, accR, accI, 2.0, 0.0);
    PH(2);
    // 2y published; the first Clenshaw B operand (own TMEM -> own smem) is
    // staged while the group's other CTAs arrive (the arrival's CTA barrier
    // also ends every warp's last power GEMM, which read bo(pb))
    garrive();
    int pc = 0;
    // Clenshaw step j's accumulator start Q_j - b_{j+2} (own positions: TMEM
    // and the owner's entries of bo(pc^1), which nobody writes before step
    // j's GEMM is over)
    auto clen_init = [&](int j) {
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
    };
    {
      double qr[NE], qi[NE];
      load_Q(r - 1, qr, qi);
      write_B(bo(pc), qr, qi, (r - 1 == 1) ? 0.5 : 1.0);
    }
    // EARLY (D128, measured +0.9 %; D256 -2 %): each Clenshaw step's start
    // is formed before the barrier that ends the previous step, so a warp's
    // wait for the slowest warp covers its TMEM / shared-memory round trips
    constexpr bool EARLY = C::D == 128;
    if (EARLY && r >= 2) clen_init(r - 2);  // (TMEM only) while the group arrives
    gwait();  // everybody's 2y published (and done reading 2X); b_{r-1} staged
    first_frags(gy);
    PH(3);
    // ---- Clenshaw in y
    for (int j = r - 2; j >= 0; --j) {
      if (!EARLY) clen_init(j);
      step(gy, j >= 1 ? gy : nullptr, bo(pc), accR, accI);
      if (j >= 1) {
        // b_j overwrites b_{j+2} at own positions only (read by the owner in
        // clen_init); every warp finished reading bo(pc^1) as the previous
        // step's B operand before the barrier that ended that step
        write_B(bo(pc ^ 1), accR, accI, (j == 1) ? 0.5 : 1.0);
        pc ^= 1;
        if (EARLY) clen_init(j - 1);  // b_{j+1}'s own entries: B operand still being read
        __syncthreads();
      }
    }
    PH(4);
    // U (times the plan phase), straight from the accumulators
    publish(gu, accR, accI, phase_one ? 1.0 : job.phase[0], phase_one ? 0.0 : job.phase[1]);
    // next slice's 2X (its buffer is dead since the powers phase) and T_1
    // into bo(pc^1) (b_2: assemble's barrier ends the owners' reads of it)
    PH(5);
    if (more) assemble(sl + 1, bo(pc ^ 1));
    tb = pc ^ 1;
    PH(6);
    garrive();  // U and the next 2X published
    // P (running product) into bo(pc) as the B operand of the product GEMM,
    // while the group arrives
    {
      double pr[NE], pi[NE];
      tmem_load_block<NE>(tm(0), pr, pi);
      write_B(bo(pc), pr, pi, 1.0);
    }
    gwait();  // everybody's U and next 2X published; P staged
    first_frags(gu);
    PH(7);
    // ---- V <- U V  (prefetches the next slice's first 2X fragments)
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      accR[e] = 0.0;
      accI[e] = 0.0;
    }
    step(gu, more ? gx : nullptr, bo(pc), accR, accI);
    tmem_store_block<NE>(tm(0), accR, accI);
    if (prefix_out) {
#pragma unroll
      for (int e = 0; e < NE; ++e)
        store_prefix(prefix_out, D, sl, row_of(e), col0 + col_of(e), accR[e], accI[e]);
    }
    __syncthreads();  // product GEMM done reading bo(pc)
    PH(8);
  }
  PH_DONE
  if (active) {
    double pr[NE], pi[NE];
    tmem_load_block<NE>(tm(0), pr, pi);
    double2* o = lane_out + (size_t)lane * D * D;
#pragma unroll
    for (int e = 0; e < NE; ++e)
      o[(size_t)row_of(e) * D + col0 + col_of(e)] = make_double2(pr[e], pi[e]);
  }
  // the exchange buffers are dead: once every CTA of the group is past its
  // last product GEMM, each drops the lines of its own column chunks from L2
  // (discard: no write-back to HBM, and the evict_last lines of this call do
  // not outlive it)
  if (s0 < s1) {
    gsync();
    constexpr int RUN = KBC * 3 * 64;  // doubles of one strip's column chunk
    for (int i = threadIdx.x; i < 3 * C::S * (RUN / 16); i += C::THREADS) {
      const int buf = i / (C::S * (RUN / 16)), rem = i % (C::S * (RUN / 16));
      const int strip = rem / (RUN / 16), line = rem % (RUN / 16);
      const double* a = gx + (size_t)buf * C::XDBL +
                        ((size_t)(strip * KB + cb * KBC) * 3) * 64 + 16 * line;
      asm volatile("discard.global.L2 [%0], 128;" ::"l"(a) : "memory");
    }
  }
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  if (warp == 0) tmem_dealloc(tmem_base, C::TMEM_COLS);
}

}  // namespace sp
