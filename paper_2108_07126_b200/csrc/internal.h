// Internal declarations shared by the host plan, the C ABI and the kernels.
#pragma once
#include <cstddef>
#include <cstdint>

#include "sliceprop_b200.h"

#include <cuda_runtime.h>

namespace sp {

int bessel_j(int k, double x, double* out, char* err, size_t errlen);
double chebyshev_error(int m, double span);
int norm_capability(int m, int bits, double* out, char* err, size_t errlen);
int select_m_max(double norm_bound, int bits, int* m_out, double* capability, char* err,
                 size_t errlen);
int make_plan(double alpha, double beta, int bits, int m_override, sp_plan* out, char* err,
              size_t errlen);
// record a context-free error (sp_last_error(NULL)) and return code
int set_error(int code, const char* fmt, ...);

// Everything one propagation needs on the device (all pointers device).
struct SliceJob {
  const double* amps;     // (pts, n_ctrl) float64
  int64_t pts;
  int n_ctrl;
  int n_terms;            // T = 1 + effective controls
  int mode;               // SP_MODE_*
  double dt;
  double xs;              // 2 * scale / beta  (0 when beta == 0): "2X" factor
  double scale;           // dt (midpoint) or 2 dt (three-point): the exponent scale
  double xspan;           // 2 / span (0 when span == 0): X = xspan * G
  double gl;              // sqrt(3) dt / 6: Gauss-Legendre commutator weight factor
  int m;                  // series order
  double coef[2 * (SP_MAX_ORDER + 1)];
  double phase[2];
  int64_t n_slices;
  // first out-of-range amplitude (row-major index), ULLONG_MAX if none:
  // validation fused into the weight computation (hamiltonian.py:145-153).
  // viol[0..2] are slots, viol[3] an epoch: multi-launch calls reset the
  // slots with a memset and record into slot 2; the single-launch (fused
  // tail) calls record into slot (epoch & 1) and their last CTA clears the
  // two other slots and advances the epoch, so no memset is needed in front
  // of the launch.  The host reads min(slots).
  unsigned long long* viol;
  int viol_epoch;
  // every expansion term is exactly (bitwise) Hermitian: the d <= 2 kernel
  // may then use real Cayley-Hamilton coefficients (lane_small_kernel<2,1>)
  int herm_exact;
  // the plan coefficients alternate exactly real / imaginary (ALT kernels)
  int coef_alt;
  // plain D x D per-lane initial running products (nullptr = identity): the
  // second pass of the d = 2 cumulative path (lane_small_kernel)
  const void* vinit;
};

// Family SU2 (kernels_su2.cuh): d = 2, every term bitwise Hermitian and
// traceless, symmetric plan with alternating coefficients, fp64, pairwise
// reduction fused into the one launch.
constexpr int SU2_MAX_TERMS = 16;
constexpr int SU2_MAX_CTRL = 4;
struct Su2Job {
  const double* amps;  // (pts, n_ctrl) float64, 16-byte aligned rows when n_ctrl is even
  int64_t n_slices;
  int n_ctrl;
  int mode;
  int m;
  double dt6;                       // dt / 6 (magnus commutator weights)
  double tz[SU2_MAX_TERMS][3];      // per term: 2X factor x ((H00 - H11) / 2, Re H01, Im H01)
  double cr[SP_MAX_ORDER + 1];      // nonzero component of a_k: Re (k even), Im (k odd)
  // u(2) systems (terms with a trace part): u2 = 1, the per-term trace part
  // 2X factor x (H00 + H11) / 2, and the full complex coefficients a_k
  int u2;
  double ta[SU2_MAX_TERMS];
  double cz[2 * (SP_MAX_ORDER + 1)];
  unsigned long long* viol;         // violation slots (epoch scheme of SliceJob), or null
  int viol_epoch;                   // 1: fused call (epoch slot), 0: slot 2
  unsigned* ctr;                    // arrival counter (zero between launches)
  void* cta_out;                    // gridDim x 8 doubles: CTA products
  void* out;                        // 2 x 2 result (complex128, or complex64 if to_fp32)
  int to_fp32;
  int arith32;                      // complex64 context: float32 arithmetic
  // phase timestamps (tools only, SP_SU2_PROF=1): [2k] = min, [2k+1] = max
  // over CTAs of %globaltimer at phase k; null = off
  unsigned long long* prof;
  // lane mode (sequential reductions, equiprop_all): no CTA tree / tail;
  // lane_out[lane] = the lane's 2 x 2 product (complex128), prefix_out[s] =
  // the running product after slice s, vinit[lane] = the lane's initial
  // product (null: identity); all complex128 2 x 2 row-major
  void* lane_out;
  void* prefix_out;
  const void* vinit;
};
// launch lane_su2_kernel (su2.cu); grid x block threads are the lanes
cudaError_t su2_run(const Su2Job& job, int grid, int block, cudaStream_t st);
// registers / max threads of the instance a job would launch (host tuning)
int su2_max_block(const Su2Job& job);
// the driven qubit's analytic midpoint reference (qubit_reference_kernel)
cudaError_t su2_qubit_reference(const Su2Job& job, int64_t steps, double c, double s, double ax,
                                double az, double wrf, double dt, int grid, int block,
                                cudaStream_t st);

}  // namespace sp
