// Internal declarations shared by the host plan, the C ABI and the kernels.
#pragma once
#include <cstddef>
#include <cstdint>

#include "sliceprop_b200.h"

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

}  // namespace sp
