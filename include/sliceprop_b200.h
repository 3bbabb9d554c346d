/*
 * sliceprop_b200 — C ABI of the B200-native equiprop hot path.
 *
 * This is the drop-in boundary for the reference's propagation hot path
 * (sliceprop 0.1.0, /root/reference/pkg/src/sliceprop).  Every entry point
 * takes plain pointers and sizes; no torch or numpy types cross it.  The
 * reference has no C ABI of its own (it is pure Python/numpy), so each
 * function below cites the Python interface it replaces and the paper's
 * Parament_* C API it is modelled on.
 *
 * Conventions
 *   - complex matrices: row-major, interleaved (re, im) — numpy
 *     complex128 / complex64 memory layout (reference linalg.py:1-13);
 *   - amplitude tables: (pts, n_ctrl) float64 row-major, also in fp32 mode
 *     (reference hamiltonian.py:114-129);
 *   - time order: U = U[n-1] ... U[0], later slice on the left
 *     (reference propagator.py:68-80);
 *   - return value: 0 on success, else an SP_E_* code that maps 1:1 onto
 *     the reference ErrorCode strings (errors.py:27-36) plus SP_E_INTERNAL
 *     for CUDA failures (the reference CLI's exit code 4, cli.py:191-193);
 *     sp_last_error() returns the message.
 *   - a context is not thread-safe and not reentrant (PAPER.md:270,
 *     SPEC.md:416); independent contexts may coexist.
 */
#ifndef SLICEPROP_B200_H
#define SLICEPROP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* error codes: errors.py:27-36 (+ internal) */
enum {
  SP_OK = 0,
  SP_E_SHAPE = 1,            /* "shape"            */
  SP_E_HERMITICITY = 2,      /* "hermiticity"      */
  SP_E_AMPLITUDE_BOUND = 3,  /* "amplitude-bound"  */
  SP_E_SAMPLING_PARITY = 4,  /* "sampling-parity"  */
  SP_E_STEP_TOO_LARGE = 5,   /* "step-too-large"   */
  SP_E_STATE_MACHINE = 6,    /* "state-machine"    */
  SP_E_ALIASING = 7,         /* "aliasing"         */
  SP_E_DOMAIN = 8,           /* "domain"           */
  SP_E_CONFIG = 9,           /* "config"           */
  SP_E_INTERNAL = 10         /* CUDA / NCCL / no device */
};

/* slicing modes: propagator.py:175-201, hamiltonian.py:8-14, magnus.py:1-16 */
enum { SP_MODE_MIDPOINT = 0, SP_MODE_SIMPSON = 1, SP_MODE_MAGNUS = 2,
       /* extensions (north star; not in the reference): two samples per slice
        * of length 2 dt at the Gauss-Legendre nodes (k + 1/2 -+ sqrt(3)/6) 2 dt;
        * GAUSS2: terms [H0, H1..HN], weights (a + b)/2 (2nd order);
        * GAUSS4: the magnus effective terms, weights (a + b)/2,
        * (sqrt(3) dt / 6)(b - a), (sqrt(3) dt / 6)(a_k b_k' - a_k' b_k)
        * (4th-order Gauss-Legendre Magnus) */
       SP_MODE_GAUSS2 = 3, SP_MODE_GAUSS4 = 4 };

/* reductions: propagator.py:279-308 ("pairwise" | "sequential") */
enum { SP_REDUCE_PAIRWISE = 0, SP_REDUCE_SEQUENTIAL = 1 };

#define SP_MAX_ORDER 25

/* Chebyshev plan — replaces ChebyshevPlan / make_plan (chebyshev.py:155-218). */
typedef struct sp_plan {
  double alpha, beta;
  int m_max;
  double coeffs[2 * (SP_MAX_ORDER + 1)]; /* a_k = (-i)^k J_k(span/2), interleaved */
  double phase[2];                       /* e^{-i(alpha+beta)/2} */
  double predicted_error;
  double capability;                     /* filled on SP_E_STEP_TOO_LARGE */
  double norm_bound;                     /* filled on SP_E_STEP_TOO_LARGE */
} sp_plan;

typedef struct sp_ctx sp_ctx;

/* ---- host plan (CPU only; chebyshev.py:61-218) ------------------------ */
const char* sp_version(void);
/* J_k(x), 0<=k<=64, 0<=x<=64 (bessel_j, chebyshev.py:61-104) */
int sp_bessel_j(int k, double x, double* out);
/* 4 (e^{1-s^2} s)^{m+1}, s = span/(4m+4) (chebyshev_error, chebyshev.py:107-110) */
double sp_chebyshev_error(int m, double span);
/* smallest odd m in 3..25 (select_m_max, chebyshev.py:113-134);
 * on SP_E_STEP_TOO_LARGE *capability holds the order-25 capability */
int sp_select_m_max(double norm_bound, int precision_bits, int* m_out, double* capability);
/* norm_capability, chebyshev.py:137-152 */
int sp_norm_capability(int m, int precision_bits, double* out);
/* make_plan, chebyshev.py:185-218; m_override = 0 selects automatically */
int sp_make_plan(double alpha, double beta, int precision_bits, int m_override, sp_plan* out);

/* ---- context lifecycle (create / set_hamiltonian / close,
 *      propagator.py:132-216 and 334-355; Parament_create/_free) -------- */
/* no device work happens here: the GPU is touched lazily by the first
 * propagation, so contexts can be created and validated without a GPU.
 * num_gpus devices (device_ids[0..num_gpus-1], NULL = 0..num_gpus-1) in ONE
 * process (the paper's interactive use):
 * with num_gpus > 1, sp_equiprop time-shards the slices into contiguous
 * blocks, one per device (three-point modes read a one-row halo), gathers
 * the d x d block products on device_ids[0] by peer copies and multiplies
 * them in time order; the device-resident and cumulative entry points run
 * on device_ids[0].  A device may repeat (P blocks emulated on one GPU). */
int sp_create(sp_ctx** out, int precision_bits, int num_gpus, const int* device_ids);
int sp_free(sp_ctx* ctx);
const char* sp_last_error(const sp_ctx* ctx);   /* ctx may be NULL */
/* load the expansion terms [H0, effective controls...] (T x d x d complex128,
 * host).  For magnus the caller passes the effective system of
 * magnus.py:45-85 (controls, i[H0,Hk], i[Hk,Hk']).  Replaces
 * IntegratorContext.set_hamiltonian (propagator.py:175-201). */
int sp_set_hamiltonian(sp_ctx* ctx, int dim, int n_ctrl, int n_terms, int mode,
                       const double* terms);

/* ---- propagation (equiprop, propagator.py:238-308; Parament_equiprop) - */
/* host buffers: amps (pts x n_ctrl float64), u_out (d x d, complex128 for
 * fp64 contexts, complex64 for fp32).  plan comes from sp_make_plan on the
 * global bound (propagator.py:258-263).  Synchronous. */
int sp_equiprop(sp_ctx* ctx, const double* amps, int64_t pts, int n_ctrl, double dt,
                const sp_plan* plan, int reduction, void* u_out);
/* same, device-resident: d_amps and d_u_out are device pointers, stream a
 * cudaStream_t (NULL = the CUDA default stream); stream-ordered with the
 * caller's own work, asynchronous.  The caller owns amplitude validation. */
int sp_equiprop_device(sp_ctx* ctx, const double* d_amps, int64_t pts, int n_ctrl,
                       double dt, const sp_plan* plan, int reduction, void* d_u_out,
                       void* stream);
/* cumulative propagators U(t_k <- 0), k = 0..slices-1 (equiprop_all,
 * propagator.py:310-331).  u_all_out holds slices x d x d (host). */
int sp_equiprop_all(sp_ctx* ctx, const double* amps, int64_t pts, int n_ctrl, double dt,
                    const sp_plan* plan, void* u_all_out);
/* same, device-resident (d_u_all_out: slices x d x d on the device, output
 * dtype), stream-ordered and asynchronous; the caller owns amplitude
 * validation (sp_amplitude_violation).  HBM-write-bound path. */
int sp_equiprop_all_device(sp_ctx* ctx, const double* d_amps, int64_t pts, int n_ctrl,
                           double dt, const sp_plan* plan, void* d_u_all_out, void* stream);
/* ordered product mats[count-1] ... mats[0] of device-resident complex128
 * d x d matrices (the multi-GPU gather step; pairwise =
 * reduce_pairwise propagator.py:68-102, sequential = left fold) */
int sp_product_device(sp_ctx* ctx, int count, const void* d_mats, int reduction,
                      void* d_out, void* stream);
/* amplitude validation (|c| <= 1, NaN rejected; hamiltonian.py:145-174) is
 * fused into the lane kernels: sp_equiprop / sp_equiprop_all return
 * SP_E_AMPLITUDE_BOUND after the pass; for sp_equiprop_device call this
 * (it synchronises the propagation's stream).  *index = row-major index of
 * the first offending sample, or -1. */
int sp_amplitude_violation(sp_ctx* ctx, int64_t* index);
/* slice count for a table of pts samples in the loaded mode
 * (propagator.py:245-252); SP_E_SAMPLING_PARITY for even/short 3-point tables */
int sp_slice_count(const sp_ctx* ctx, int64_t pts, int64_t* out);

/* ---- device batch layer (context-free; device buffers, caller's stream,
 *      asynchronous).  For users who build / exponentiate / multiply their
 *      own batches, as the reference's materialised path does; equiprop
 *      never uses these (its three stages are fused in the lane kernels).
 *      Batches: compact or strided runs of d x d row-major interleaved
 *      complex matrices in the working dtype (complex128 for bits 64,
 *      complex64 for bits 32), computed in that dtype's arithmetic. ---- */
/* out[k] = scale (T_0 + sum_{i>=1} coeffs[k, i] T_i): terms complex128
 * (n_terms x d x d), coeffs float64 (count x n_terms, column 0 all ones),
 * out compact working dtype.  Replaces expand_linear_combination
 * (linalg.py:246-288) under build_exponent_batch (hamiltonian.py:186-207)
 * and build_magnus_exponent_batch (magnus.py:121-141). */
int sp_expand_batch_device(int precision_bits, int dim, int n_terms, const void* d_terms,
                           int64_t count, const double* d_coeffs, double scale, void* d_out,
                           void* stream);
/* U[k] = phase * p((2/span)(G[k] - center I)) with the plan's Chebyshev
 * polynomial (expm_batch, chebyshev.py:259-306).  dim <= 64: one fused
 * on-chip kernel (in place allowed); dim > 64: m+1 batched GEMM launches
 * through d_scratch (sp_expm_batch_scratch_bytes; may alias neither g nor u).
 * Strides in complex elements between consecutive matrices. */
size_t sp_expm_batch_scratch_bytes(int precision_bits, int dim, int64_t count);
int sp_expm_batch_device(int precision_bits, int dim, int64_t count, const void* d_g,
                         int64_t stride_in, const sp_plan* plan, void* d_u, int64_t stride_out,
                         void* d_scratch, void* stream);
/* C[k] = alpha A[k] B[k] + beta C[k] + gamma I; alpha/beta/gamma are
 * (re, im) pairs (NULL: 1, 0, 0); beta == 0 never reads C; C must not
 * overlap A or B (gemm_strided_batched + diagonal_add_batched,
 * linalg.py:204-237). */
int sp_gemm_batched_device(int precision_bits, int dim, int64_t count, const void* d_a,
                           int64_t stride_a, const void* d_b, int64_t stride_b,
                           const double* alpha, const double* beta, const double* gamma,
                           void* d_c, int64_t stride_c, void* stream);

/* state propagation (apply, propagator.py:105-118): out[k] = U psi_k
 * (kind 0: count x d vectors) or U rho_k U^+ (kind 1: count x d x d density
 * matrices, through d_scratch of sp_apply_batch_scratch_bytes), U and the
 * states device-resident in the working dtype. */
size_t sp_apply_batch_scratch_bytes(int precision_bits, int dim, int64_t count, int kind);
int sp_apply_batch_device(int precision_bits, int dim, const void* d_u, int64_t count, int kind,
                          const void* d_states, void* d_out, void* d_scratch, void* stream);

/* ---- analytic oracle on the device (studies.py:123-153) -----------------
 * The driven qubit H(t) = (w0/2) sz + (w1/2)(cos(wrf t) sx + sin(wrf t) sy)
 * propagated over steps midpoint slices of dt = duration / steps with EXACT
 * per-slice SU(2) rotations (midpoint_reference): no series, no amplitude
 * table.  u_out: 2 x 2 complex128 (host).  Identity for steps < 1 or no
 * field (studies.py:131-139).  ctx: any created context (device, stream). */
int sp_qubit_midpoint_reference(sp_ctx* ctx, double w0, double w1, double wrf,
                                double duration, int64_t steps, double* u_out);

/* ---- evaluation scheme of the slice series ------------------------------
 * 0 auto (Paterson-Stockmeyer in the Chebyshev basis whenever it needs fewer
 * GEMMs per slice than the reference's Clenshaw recurrence), 1 Clenshaw
 * (chebyshev.py:298-303 order of operations, applied to the running
 * product), 2 Paterson-Stockmeyer.  Same plan and same truncated polynomial
 * in every case; only the rounding differs. */
int sp_set_algorithm(sp_ctx* ctx, int algo);
int sp_last_algorithm(const sp_ctx* ctx, int* algo, int* gemms_per_slice);
/* number of lanes (contiguous runs of slices propagated by one warp / CTA /
 * CTA group) of the last lane pass: slices per lane = slice_count / lanes */
int sp_last_lanes(const sp_ctx* ctx, int* lanes);

/* ---- measurement hooks ------------------------------------------------ */
/* when enabled, the next propagations record CUDA events around the main
 * lane kernel; sp_last_timing returns its duration (ms), the number of
 * kernels launched by the last call and the executed FP64 flops */
int sp_set_profiling(sp_ctx* ctx, int enabled);
int sp_last_timing(const sp_ctx* ctx, double* main_kernel_ms, int* launches,
                   double* executed_flops, char* kernel_name, int name_len);
int sp_device_count(int* out);

#ifdef __cplusplus
}
#endif
#endif /* SLICEPROP_B200_H */
