/* nfftk.h -- C ABI of the B200-native NFFT library (libnfftk.so).
 *
 * Part 1 reproduces the reference interface symbol for symbol
 * (/root/reference/pkg/include/nfftk.h:22-59, generated from
 * pkg/src/nfftk/abi.py:24-93; semantics from pkg/src/nfftk/cabi.py:99-237).
 * Part 2 adds nfftk_* extensions for the GPU build: explicit window /
 * precision, device-pointer transforms on a caller stream, split adjoint
 * phases for multi-GPU reduction, phase timing and diagnostics.
 *
 * Complex buffers are interleaved (re, im) pairs: float64 for complex128
 * plans, float32 for complex64 plans (extension create only).  Handles are
 * opaque positive integers; a handle must not be used from two threads at
 * once.  Buffer pointers stay valid until nfftk_destroy.
 */
#ifndef NFFTK_H
#define NFFTK_H

#include <stdint.h>

#define NFFTK_ABI_VERSION "0.1.0"

#define NFFTK_ERR_HANDLE (-1)
#define NFFTK_ERR_SHAPE (-2)
#define NFFTK_ERR_DOMAIN (-3)
#define NFFTK_ERR_INTERNAL (-9)

/* f1 flag word -- the reference's own bit assignment (plan.py:31-43); the
 * reference header defines none of these, callers hard-coded them. */
#define NFFTK_PRE_PHI_HUT (1u << 0)
#define NFFTK_FG_PSI (1u << 1)
#define NFFTK_PRE_LIN_PSI (1u << 2)
#define NFFTK_PRE_FG_PSI (1u << 3)
#define NFFTK_PRE_PSI (1u << 4)
#define NFFTK_PRE_FULL_PSI (1u << 5)
#define NFFTK_MALLOC_X (1u << 6)
#define NFFTK_MALLOC_F_HAT (1u << 7)
#define NFFTK_MALLOC_F (1u << 8)
#define NFFTK_FFT_OUT_OF_PLACE (1u << 9)
#define NFFTK_FFTW_INIT (1u << 10)
#define NFFTK_NFFT_SORT_NODES (1u << 11)
#define NFFTK_NFFT_OMP_BLOCKWISE_ADJOINT (1u << 12)
/* f2 (accepted, ignored; plan.py:61-70) */
#define NFFTK_FFTW_MEASURE 0u
#define NFFTK_FFTW_DESTROY_INPUT (1u << 0)
#define NFFTK_FFTW_UNALIGNED (1u << 1)
#define NFFTK_FFTW_CONSERVE_MEMORY (1u << 2)
#define NFFTK_FFTW_EXHAUSTIVE (1u << 3)
#define NFFTK_FFTW_PRESERVE_INPUT (1u << 4)
#define NFFTK_FFTW_PATIENT (1u << 5)
#define NFFTK_FFTW_ESTIMATE (1u << 6)
#define NFFTK_FFTW_WISDOM_ONLY (1u << 21)

/* extension enums */
#define NFFTK_WINDOW_KAISER_BESSEL 0
#define NFFTK_WINDOW_GAUSSIAN 1
#define NFFTK_COMPLEX128 0
#define NFFTK_COMPLEX64 1
#define NFFTK_MODE_FOLLOW_FLAGS (-1)
#define NFFTK_MODE_DIRECT 0
#define NFFTK_MODE_TENSOR 1

#ifdef __cplusplus
extern "C" {
#endif

/* ===================== Part 1: reference interface ===================== */

/* semantic version of this ABI                       (ref nfftk.h:25, abi.py:21) */
const char * nfftk_abi_version(void);

/* new plan with default parameters; returns handle > 0 or negative error code
 *                                        (ref nfftk.h:28, cabi.py:99-109) */
int32_t nfftk_create(const int32_t * bandlimits, int32_t rank, int32_t node_count);

/* new plan with explicit grid, cutoff and flag words (ref nfftk.h:31, cabi.py:112-124) */
int32_t nfftk_create_advanced(const int32_t * bandlimits, int32_t rank, int32_t node_count, const int32_t * fft_lengths, int32_t cutoff, uint32_t flags, uint32_t fft_flags);

/* copy node_count*rank coordinates in [-1/2,1/2) and precompute
 *                                        (ref nfftk.h:34, cabi.py:127-146) */
int32_t nfftk_set_x(int32_t handle, const double * coords, int64_t len);

/* copy prod(bandlimits) complex coefficients, interleaved re/im (ref nfftk.h:37, cabi.py:163-168) */
int32_t nfftk_set_fhat(int32_t handle, const double * values, int64_t len);

/* copy node_count complex samples, interleaved re/im (ref nfftk.h:40, cabi.py:171-176) */
int32_t nfftk_set_f(int32_t handle, const double * values, int64_t len);

/* forward transform into the sample buffer (ref nfftk.h:43, cabi.py:179-191) */
int32_t nfftk_trafo(int32_t handle);

/* adjoint transform into the coefficient buffer (ref nfftk.h:46, cabi.py:194-206) */
int32_t nfftk_adjoint(int32_t handle);

/* pointer to the plan-owned sample buffer (2*node_count doubles); NULL if invalid
 *                                        (ref nfftk.h:49, cabi.py:209-212) */
const double * nfftk_get_f(int32_t handle);

/* pointer to the plan-owned coefficient buffer (2*prod(bandlimits) doubles); NULL if invalid
 *                                        (ref nfftk.h:52, cabi.py:215-218) */
const double * nfftk_get_fhat(int32_t handle);

/* error code of the last failing call    (ref nfftk.h:55, cabi.py:221-226) */
int32_t nfftk_last_error(int32_t handle);

/* message for the last failing call; valid until the next call on the handle
 *                                        (ref nfftk.h:58, abi.py:264-268) */
const char * nfftk_last_error_message(int32_t handle);

/* release the plan; exactly one per create (ref nfftk.h:61, cabi.py:229-237) */
int32_t nfftk_destroy(int32_t handle);

/* ======================== Part 2: B200 extensions ======================== */

const char * nfftk_ext_version(void);

/* Plan(N, M, n=None, m=None, f1=None, f2=None, window) of plan.py:138 with
 * optional fields: fft_lengths may be NULL (default n), has_* = 0 selects the
 * reference default.  window: NFFTK_WINDOW_*; precision: NFFTK_COMPLEX*. */
int32_t nfftk_create_ex(const int32_t * bandlimits, int32_t rank, int32_t node_count,
                        const int32_t * fft_lengths, int32_t has_cutoff, int32_t cutoff,
                        int32_t has_flags, uint32_t flags, int32_t has_fft_flags,
                        uint32_t fft_flags, int32_t window, int32_t precision);
/* error kind / message of the calling thread's last failed create (kinds mirror errors.py) */
int32_t nfftk_last_create_error_kind(void);
const char * nfftk_last_create_error_message(void);
/* fine-grained error kind of the handle's last failure (errors.py class) */
int32_t nfftk_last_error_kind(int32_t handle);

/* Plan.set_nodes (plan.py:210-233) without precompute; host or device coords */
int32_t nfftk_set_nodes(int32_t handle, const double * coords, int64_t len);
int32_t nfftk_set_nodes_device(int32_t handle, const double * coords_dev, int64_t len, void * stream);
/* Plan.precompute (plan.py:249-299) */
int32_t nfftk_precompute(int32_t handle);
int32_t nfftk_precompute_stream(int32_t handle, void * stream);
/* select the window-factor source before precompute: FOLLOW_FLAGS, DIRECT, TENSOR */
int32_t nfftk_set_psi_policy(int32_t handle, int32_t mode);

/* transforms on caller buffers: host pointers (synchronous) or device
 * pointers ordered on `stream` (cudaStream_t; NULL = legacy default stream) */
int32_t nfftk_trafo_host(int32_t handle, const void * fhat, void * f);
int32_t nfftk_adjoint_host(int32_t handle, const void * f, void * fhat);
int32_t nfftk_trafo_device(int32_t handle, const void * fhat_dev, void * f_dev, void * stream);
int32_t nfftk_adjoint_device(int32_t handle, const void * f_dev, void * fhat_dev, void * stream);
/* exact sums Plan.ndft / Plan.ndft_adjoint (transform.py:188-234), complex128
 * interleaved in and out, on the device (cuBLAS ZGEMM over the last dim) */
int32_t nfftk_ndft_host(int32_t handle, const double * fhat, double * f);
int32_t nfftk_ndft_adjoint_host(int32_t handle, const double * f, double * fhat);
int32_t nfftk_ndft_device(int32_t handle, const void * fhat_dev, void * f_dev, void * stream);
int32_t nfftk_ndft_adjoint_device(int32_t handle, const void * f_dev, void * fhat_dev, void * stream);
/* adjoint split for multi-GPU: spread into the plan grid, (caller reduces the
 * grid, e.g. NCCL all-reduce on a grid bound with nfftk_bind_grid), finish */
int32_t nfftk_spread_device(int32_t handle, const void * f_dev, void * stream);
int32_t nfftk_adjoint_finish_device(int32_t handle, void * fhat_dev, void * stream);
int32_t nfftk_bind_grid(int32_t handle, void * grid_dev, int64_t bytes);
/* B alone from the plan's dense n-grid (filled by the caller, e.g. a
 * distributed F into a bound grid): samples at the plan's nodes on `stream` */
int32_t nfftk_interp_device(int32_t handle, void * f_dev, void * stream);
/* the deconvolution column of dim: 1/(phi_hat_dim(k) * wscale) for
 * k = -N/2 .. N/2-1 (len = N_dim; transform.py:44-54) -- D / D^H of a
 * distributed F apply it with 1/|I_n| */
int32_t nfftk_deconv_cols(int32_t handle, int32_t dim, double * out, int64_t len);

/* introspection: out[0..count) = d, M, m, window, precision, f1, f2, has_nodes,
 * ready, factor mode, tiles, subproblems, sum of stencil widths, gridding
 * kernels (0 batch, 1 pipelined row-per-thread, 2 residue-owned spread),
 * nodes with a 2m+1 wide stencil (residue geometry), F / F^H (0 cuFFT on the
 * dense grid, 1 pruned two-/three-pass line FFTs with D, D^H and the ghost padding
 * fused in); count <= 16 */
int32_t nfftk_get_params(int32_t handle, int64_t * out, int32_t count);
int32_t nfftk_get_sizes(int32_t handle, int32_t * N, int32_t * n, int32_t * tile, int32_t count);
int32_t nfftk_get_window(int32_t handle, double * b, double * sigma, int32_t count);
int32_t nfftk_phi_hut(int32_t handle, int32_t dim, double * out, int64_t len);
int32_t nfftk_node_order(int32_t handle, int64_t * out, int64_t len);
int32_t nfftk_window_evals(int32_t handle, int64_t * last, int64_t * total);
/* PrecomputeTables contents in the reference layout (plan.py:109-121), built
 * on demand on the device and copied to host arrays: psi (M, d, 2m+1), len =
 * M*d*(2m+1); vals / idx (M, (2m+1)^d) and counts (M) of PRE_FULL_PSI when
 * vals is not NULL; lut (d, 2^14+1) and lut_steps (d) of PRE_LIN_PSI */
int32_t nfftk_psi_tables(int32_t handle, double * psi, double * vals, int64_t * idx, int64_t * counts,
                         int64_t len);
int32_t nfftk_lut_tables(int32_t handle, double * lut, double * steps, int64_t len);

/* instrumentation: per-phase CUDA-event timing and kernel launch counter */
int32_t nfftk_set_timing(int32_t handle, int32_t on);
int32_t nfftk_phase_times(int32_t handle, double * ms, int64_t * calls, int32_t count, int32_t reset);
uint64_t nfftk_launch_count(void);
/* FP64 / FP32 FMA throughput of this GPU (TFLOP/s), for roofline reporting */
int32_t nfftk_measure_fma_peaks(double * fp64_tflops, double * fp32_tflops);

/* the library's window math (window.py:38-181) for host-side callers:
 * shape parameter b_i, phi at offsets t, phi_hat at frequencies k (status
 * per entry: 0 ok, 1 the Kaiser-Bessel transform vanishes, 2 not positive),
 * the I0 series */
double nfftk_window_b(int32_t window, int32_t N_i, int32_t n_i, int32_t m);
int32_t nfftk_window_values(int32_t window, double n_i, int32_t m, double b_i, const double * t,
                            int64_t count, double * out);
int32_t nfftk_phi_hat_values(int32_t window, int32_t n_i, int32_t m, double b_i, const int32_t * k,
                             int64_t count, double * out, int32_t * status);
double nfftk_bessel_i0(double x);

/* leak counters (cabi.py:240-245) */
int32_t nfftk_live_handles(void);
int64_t nfftk_live_buffers(void);

#ifdef __cplusplus
}
#endif

#endif /* NFFTK_H */
