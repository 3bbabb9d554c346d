// Host-side Chebyshev plan for the equiprop hot path (CPU code, no CUDA).
//
// Restates sliceprop/chebyshev.py:61-218 in C++ so that the C ABI is usable
// without Python.  The arithmetic follows the reference
// operation by operation: the Bessel recurrence runs in x86-64 80-bit
// long double exactly like numpy.longdouble, and the error estimate uses
// the same libm exp/pow as CPython's float ops, so every value is bit-for-bit
// identical to the reference (pinned by tests/test_plan.py against
// tests/golden/plan.npz).
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>

#include "sliceprop_b200.h"
#include "internal.h"

namespace sp {

static const double kMaxTrustedS = 1.0 / std::sqrt(2.0);  // chebyshev.py:56

// float(math.factorial(k)) with CPython's correctly rounded int->float
// conversion: exact multi-limb product, then round-half-even to 53 bits.
static double factorial_as_double(int k) {
  uint32_t limb[16] = {1};
  int n = 1;
  for (int f = 2; f <= k; ++f) {
    uint64_t carry = 0;
    for (int i = 0; i < n; ++i) {
      uint64_t v = (uint64_t)limb[i] * (uint64_t)f + carry;
      limb[i] = (uint32_t)v;
      carry = v >> 32;
    }
    if (carry) limb[n++] = (uint32_t)carry;
  }
  // bit length
  int top = n - 1;
  int bits = 32 * top;
  for (uint32_t t = limb[top]; t; t >>= 1) ++bits;
  if (bits <= 53) {
    double r = 0.0;
    for (int i = n - 1; i >= 0; --i) r = r * 4294967296.0 + (double)limb[i];
    return r;  // exact
  }
  auto bit = [&](int b) -> int { return (limb[b >> 5] >> (b & 31)) & 1u; };
  // mantissa = bits [bits-53, bits)
  uint64_t mant = 0;
  for (int b = bits - 1; b >= bits - 53; --b) mant = (mant << 1) | (uint64_t)bit(b);
  int guard = bit(bits - 54);
  int sticky = 0;
  for (int b = bits - 55; b >= 0 && !sticky; --b) sticky |= bit(b);
  if (guard && (sticky || (mant & 1ull))) ++mant;
  return std::ldexp((double)mant, bits - 53);
}

int bessel_j(int k, double x, double* out, char* err, size_t errlen) {
  if (k < 0 || k > 64) {
    snprintf(err, errlen, "order %d outside supported range 0..64", k);
    return SP_E_DOMAIN;
  }
  if (!(0.0 <= x && x <= 64.0)) {
    snprintf(err, errlen, "argument %g outside supported range 0..64.0", x);
    return SP_E_DOMAIN;
  }
  if (x == 0.0) {
    *out = (k == 0) ? 1.0 : 0.0;
    return SP_OK;
  }
  if (x < 1e-4) {  // series head, chebyshev.py:77-80
    double y = std::pow(0.5 * x, 2.0);
    double head = 1.0 - y / (double)(k + 1) + y * y / (2.0 * (double)(k + 1) * (double)(k + 2));
    *out = std::pow(0.5 * x, (double)k) / factorial_as_double(k) * head;
    return SP_OK;
  }
  int n_start = (int)std::ceil(x);
  if (k > n_start) n_start = k;
  n_start += 52;
  n_start += n_start % 2;
  typedef long double ld;
  const ld xl = (ld)x;
  ld jp = (ld)0.0;
  ld jc = (ld)1e-30;          // numpy.longdouble(1e-30): the double, widened
  ld acc = (ld)2.0 * jc;
  ld jk = (k == n_start) ? jc : (ld)0.0;
  const ld big = (ld)1e250;
  const ld tiny = (ld)1e-250;
  for (int n = n_start; n > 0; --n) {
    volatile ld q = (ld)(2 * n) / xl;  // keep the reference's rounding steps
    volatile ld prod = q * jc;
    ld next = prod - jp;
    jp = jc;
    jc = next;
    int m = n - 1;
    if (m == k) jk = jc;
    if (m > 0 && m % 2 == 0) acc += (ld)2.0 * jc;
    if (fabsl(jc) > big) {
      jp *= tiny;
      jc *= tiny;
      acc *= tiny;
      jk *= tiny;
    }
  }
  *out = (double)(jk / (acc + jc));
  return SP_OK;
}

double chebyshev_error(int m, double span) {
  double s = span / (4.0 * m + 4.0);
  return 4.0 * std::pow(std::exp(1.0 - s * s) * s, (double)(m + 1));
}

static double roundoff(int bits) { return bits == 32 ? std::ldexp(1.0, -24) : std::ldexp(1.0, -53); }

static bool on_grid(int m) { return m >= 3 && m <= SP_MAX_ORDER && (m % 2) == 1; }

int norm_capability(int m, int bits, double* out, char* err, size_t errlen) {
  if (!on_grid(m)) {
    snprintf(err, errlen, "order %d not in the supported grid (3, 5, ..., 25)", m);
    return SP_E_CONFIG;
  }
  const double target = roundoff(bits);
  double lo = 0.0, hi = (4.0 * m + 4.0) * kMaxTrustedS / 2.0;
  for (int it = 0; it < 200; ++it) {
    double mid = 0.5 * (lo + hi);
    if (chebyshev_error(m, 2.0 * mid) <= target)
      lo = mid;
    else
      hi = mid;
    if (hi - lo <= 1e-15 * hi) break;
  }
  *out = 0.5 * (lo + hi);
  return SP_OK;
}

int select_m_max(double norm_bound, int bits, int* m_out, double* capability, char* err,
                 size_t errlen) {
  if (norm_bound < 0) {
    snprintf(err, errlen, "norm bound must be >= 0, got %g", norm_bound);
    return SP_E_DOMAIN;
  }
  const double span = 2.0 * norm_bound;
  const double target = roundoff(bits);
  for (int m = 3; m <= SP_MAX_ORDER; m += 2) {
    if (span / (4.0 * m + 4.0) > kMaxTrustedS) continue;
    if (chebyshev_error(m, span) <= target) {
      *m_out = m;
      return SP_OK;
    }
  }
  double cap = 0.0;
  norm_capability(SP_MAX_ORDER, bits, &cap, err, errlen);
  if (capability) *capability = cap;
  snprintf(err, errlen,
           "exponent norm bound %.6g exceeds the order-25 capability %.3f for %s; "
           "shrink the time step",
           norm_bound, cap, bits == 32 ? "fp32" : "fp64");
  return SP_E_STEP_TOO_LARGE;
}

int make_plan(double alpha, double beta, int bits, int m_override, sp_plan* out, char* err,
              size_t errlen) {
  std::memset(out, 0, sizeof(*out));
  if (!(alpha <= beta)) {
    snprintf(err, errlen, "spectral bounds out of order: alpha=%g, beta=%g", alpha, beta);
    return SP_E_CONFIG;
  }
  const double span = beta - alpha;
  int m = m_override;
  if (m == 0) {
    double cap = 0.0;
    int rc = select_m_max(span / 2.0, bits, &m, &cap, err, errlen);
    if (rc != SP_OK) {
      out->capability = cap;
      out->norm_bound = span / 2.0;
      return rc;
    }
  } else {
    if (!on_grid(m)) {
      snprintf(err, errlen, "m_max override %d not an odd integer in 3..25", m);
      return SP_E_CONFIG;
    }
    double eps = chebyshev_error(m, span);
    if (span > 4.0 * m + 4.0 || eps >= 1.0) {
      double cap = 0.0;
      norm_capability(m, bits, &cap, err, errlen);
      out->capability = cap;
      out->norm_bound = span / 2.0;
      snprintf(err, errlen,
               "span %.6g is unusable at order %d (predicted error %.3g); shrink the time step",
               span, m, eps);
      return SP_E_STEP_TOO_LARGE;
    }
  }
  const double half = span / 2.0;
  out->alpha = alpha;
  out->beta = beta;
  out->m_max = m;
  for (int k = 0; k <= m; ++k) {
    double j = 0.0;
    int rc = bessel_j(k, half, &j, err, errlen);
    if (rc != SP_OK) return rc;
    // (-i)^k * J: exact unit factors (CPython's integer complex power)
    double re = 0.0, im = 0.0;
    switch (k & 3) {
      case 0: re = j; break;
      case 1: im = -j; break;
      case 2: re = -j; break;
      default: im = j; break;
    }
    out->coeffs[2 * k] = re;
    out->coeffs[2 * k + 1] = im;
  }
  const double theta = -0.5 * (alpha + beta);
  out->phase[0] = std::cos(theta);
  out->phase[1] = std::sin(theta);
  out->predicted_error = chebyshev_error(m, span);
  return SP_OK;
}

}  // namespace sp
