// Launchers of the su(2) family (kernels_su2.cuh), and of the same lanes on
// the 2 x 2 complex algebra for u(2) systems (terms with a trace part).
//   lane_su2_tma_kernel  midpoint, 2 or 4 controls (the driven qubit): TMA
//                        2-D tensor loads of the amplitude rows
//   lane_su2_kernel      every mode / control count: cp.async row ring
// Series orders 3, 5, 7 compiled in (the qubit's fine steps), 0 = runtime m.
// Environment (A/B timing only): SP_SU2_TMA=0 forces the cp.async form.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <set>
#include <utility>

#include "internal.h"
#include "kernels_su2.cuh"

namespace sp {
namespace {

struct Su2Kernel {
  const void* fn = nullptr;
  int smem = 0;       // dynamic shared memory bytes at max_block threads
  int max_block = 0;
  bool tma = false;
  int rows = 0;       // TMA: rows per lane per round (C)
};

template <int MODE, int NCC, class R, bool PFX, bool U2>
Su2Kernel su2_pick(int m) {
  using S = Su2Shape<MODE, NCC, R, U2>;
  Su2Kernel k;
  k.smem = S::SMEM_PER_THREAD * S::TPB;
  k.max_block = S::TPB;
  if constexpr (U2) {  // the random systems' fp64 midpoint order compiled in
    k.fn = m == 13 ? (const void*)lane_su2_kernel<MODE, NCC, 13, R, PFX, true>
                   : (const void*)lane_su2_kernel<MODE, NCC, 0, R, PFX, true>;
  } else {
    switch (m) {
      case 3: k.fn = (const void*)lane_su2_kernel<MODE, NCC, 3, R, PFX>; break;
      case 5: k.fn = (const void*)lane_su2_kernel<MODE, NCC, 5, R, PFX>; break;
      case 7: k.fn = (const void*)lane_su2_kernel<MODE, NCC, 7, R, PFX>; break;
      default: k.fn = (const void*)lane_su2_kernel<MODE, NCC, 0, R, PFX>;
    }
  }
  return k;
}

template <int NCC, int C, class R, bool PFX, bool U2>
Su2Kernel su2_pick_tma(int m) {
  using G = Su2Tma<NCC, C>;
  Su2Kernel k;
  k.smem = G::SMEM;
  k.max_block = G::TPB;
  k.tma = true;
  k.rows = C;
  if constexpr (U2) {  // the random systems' fp64 midpoint order compiled in
    k.fn = m == 13 ? (const void*)lane_su2_tma_kernel<NCC, 13, C, R, PFX, true>
                   : (const void*)lane_su2_tma_kernel<NCC, 0, C, R, PFX, true>;
  } else {
    switch (m) {
      case 3: k.fn = (const void*)lane_su2_tma_kernel<NCC, 3, C, R, PFX>; break;
      case 5: k.fn = (const void*)lane_su2_tma_kernel<NCC, 5, C, R, PFX>; break;
      case 7: k.fn = (const void*)lane_su2_tma_kernel<NCC, 7, C, R, PFX>; break;
      default: k.fn = (const void*)lane_su2_tma_kernel<NCC, 0, C, R, PFX>;
    }
  }
  return k;
}

template <int MODE, class R, bool PFX, bool U2>
Su2Kernel su2_pick_n(int n_ctrl, int m) {
  switch (n_ctrl) {
    case 1: return su2_pick<MODE, 1, R, PFX, U2>(m);
    case 2: return su2_pick<MODE, 2, R, PFX, U2>(m);
    case 3: return su2_pick<MODE, 3, R, PFX, U2>(m);
    case 4: return su2_pick<MODE, 4, R, PFX, U2>(m);
  }
  return {};
}

int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

template <class R, bool PFX, bool U2>
Su2Kernel su2_kernel_for_t(const Su2Job& job) {
  static const int use_tma = env_int("SP_SU2_TMA", 1);
  // 128-byte lane rows per round (measured: 64-byte rounds with 1024-thread
  // CTAs 1.4x slower at 1e7 slices)
  if (use_tma && job.mode == SP_MODE_MIDPOINT && (job.n_ctrl == 2 || job.n_ctrl == 4))
    return job.n_ctrl == 2 ? su2_pick_tma<2, 8, R, PFX, U2>(job.m)
                           : su2_pick_tma<4, 4, R, PFX, U2>(job.m);
  switch (job.mode) {
    case SP_MODE_MIDPOINT: return su2_pick_n<SP_MODE_MIDPOINT, R, PFX, U2>(job.n_ctrl, job.m);
    case SP_MODE_SIMPSON: return su2_pick_n<SP_MODE_SIMPSON, R, PFX, U2>(job.n_ctrl, job.m);
    case SP_MODE_MAGNUS: return su2_pick_n<SP_MODE_MAGNUS, R, PFX, U2>(job.n_ctrl, job.m);
  }
  return {};
}

// complex64 contexts: the same kernels in float32 arithmetic; lane mode
// (lane_out set: sequential reduction / equiprop_all) is complex128 only;
// u(2) systems (job.u2) on the 2 x 2 complex algebra: the TMA lanes only
// (engine.cu su2_applies routes the rest to lane_small_kernel<2,1>)
template <bool PFX>
Su2Kernel u2_kernel_for(const Su2Job& job) {  // complex128
  if (job.arith32) return {};
  return su2_kernel_for_t<double, PFX, true>(job);
}

Su2Kernel su2_kernel_for(const Su2Job& job) {
  if (job.u2) return job.lane_out ? u2_kernel_for<true>(job) : u2_kernel_for<false>(job);
  if (job.lane_out) return su2_kernel_for_t<double, true, false>(job);
  return job.arith32 ? su2_kernel_for_t<float, false, false>(job)
                     : su2_kernel_for_t<double, false, false>(job);
}

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

}  // namespace

cudaError_t su2_run(const Su2Job& job, int grid, int block, cudaStream_t st) {
  const Su2Kernel k = su2_kernel_for(job);
  if (!k.fn) return cudaErrorInvalidValue;
  // dynamic shared memory (opt-in above 48 KB, set once per kernel and
  // device: multi-device contexts launch on several devices)
  static std::mutex mu;
  static std::set<std::pair<int, const void*>> opted;
  {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> g(mu);
    if (!opted.count({dev, k.fn})) {
      e = cudaFuncSetAttribute(k.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, k.smem);
      if (e != cudaSuccess) return e;
      opted.insert({dev, k.fn});
    }
  }
  if (!k.tma) {
    void* args[] = {const_cast<Su2Job*>(&job)};
    return cudaLaunchKernel(k.fn, dim3(grid), dim3(block), args,
                            (size_t)k.smem / k.max_block * block, st);
  }
  // TMA form: L slices per lane, the table as the tensor [full lanes][L x N]
  const int64_t lanes = (int64_t)grid * block;
  int64_t L = std::max<int64_t>(1, (job.n_slices + lanes - 1) / lanes);
  const int64_t full = job.n_slices / L;
  PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
  if (!enc) return cudaErrorNotSupported;
  CUtensorMap tmap;
  const int N = job.n_ctrl;
  const cuuint64_t dims[2] = {(cuuint64_t)(L * N), (cuuint64_t)full};
  const cuuint64_t strides[1] = {(cuuint64_t)(L * N * 8)};
  const cuuint32_t box[2] = {(cuuint32_t)(k.rows * N), 32u};
  const cuuint32_t estr[2] = {1u, 1u};
  const bool sw128 = k.rows * N * 8 == 128;
  const CUresult r = enc(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2,
                         const_cast<double*>(job.amps), dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE,
                         sw128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
  void* args[] = {const_cast<Su2Job*>(&job), &tmap, &L};
  return cudaLaunchKernel(k.fn, dim3(grid), dim3(block), args, (size_t)k.smem, st);
}

int su2_max_block(const Su2Job& job) { return su2_kernel_for(job).max_block; }

cudaError_t su2_qubit_reference(const Su2Job& job, int64_t steps, double c, double s, double ax,
                                double az, double wrf, double dt, int grid, int block,
                                cudaStream_t st) {
  const QubitRef q{steps, c, s, ax, az, wrf, dt};
  qubit_reference_kernel<<<grid, block, 0, st>>>(job, q);
  return cudaGetLastError();
}

}  // namespace sp
