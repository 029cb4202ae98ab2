/*
 * kle_b200.h — C ABI of libkle_b200.so, the sm_100a implementation of the
 * KLE-CGC data-parallel hot path (arXiv 2510.26180; reference package
 * `pintuq`, /root/reference/pkg/src/pintuq).
 *
 * Conventions (all entry points):
 *  - every array argument is a DEVICE pointer owned by the caller; fp64
 *    throughout; sample-major C order exactly as the reference's per-sample
 *    arrays stacked over samples: a trajectory block is [M][N][nx]
 *    (CoarseTrajectory.states, pintuq/core.py:150-166), a tridiagonal
 *    operator is dia[M][nx], off[M][nx] (off[s][i] couples rows i and i+1;
 *    off[s][nx-1] is unused);
 *  - `stream` is a cudaStream_t passed as void*; all work is stream ordered,
 *    no implicit device synchronisation except where stated;
 *  - return 0 on success, else a KLE_ERR_* code; kle_last_error() returns a
 *    message for the calling thread's last failure. No exceptions cross the ABI;
 *  - no hidden device allocation: scratch/workspace is caller provided and
 *    sized by the matching *_bytes query;
 *  - library-owned state, all of it listed here: the thread-local error
 *    string; per (host thread, device) auxiliary streams/events and 16 pinned
 *    host bytes used by the multi-stream paths (kle_pcgc_solve_f64's sample
 *    pipelines, the large-block CGC), created on first use and freed by
 *    kle_release_resources(); per-device kernel-attribute flags (set once per
 *    device, atomically). Reentrant on distinct streams;
 *  - kle_pcgc_solve_f64 / kle_pcgc_solve_ref_f64 / kle_parareal_solve_f64 run
 *    the outer loop on the host: they read the active-sample count back every
 *    iteration and return after the work on `stream` has completed
 *    (synchronous, like the reference's pcgc_solve).
 *
 * The reference has no FFI for this path (it is pure numpy/scipy); each entry
 * point below names the reference function it replaces. INTEGRATION.md shows
 * the Python (ctypes) binding the reference package would add.
 */
#ifndef KLE_B200_H
#define KLE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KLE_ABI_VERSION 1

/* status codes */
#define KLE_OK 0
#define KLE_ERR_INVALID 1
#define KLE_ERR_CUDA 2
#define KLE_ERR_UNSUPPORTED 3
#define KLE_ERR_WORKSPACE 4

/* per-sample status words written by kle_pcgc_solve_f64 / kle_cgc_update_f64 */
#define KLE_SAMPLE_ACTIVE 0
#define KLE_SAMPLE_CONVERGED 1   /* increment <= tol            (pintuq/pcgc.py:345-348) */
#define KLE_SAMPLE_MAXITERS 2    /* MaxItersExceededError       (pintuq/pcgc.py:352-357) */
#define KLE_SAMPLE_NONFINITE 3   /* CoarseTrajectory.assert_finite (pintuq/core.py:179-181) */
#define KLE_SAMPLE_NEWTON 4      /* NonConvergenceError of the simplified Newton CGC (pintuq/pcgc.py:264-269) */

int kle_abi_version(void);
const char* kle_last_error(void);
/* Free the calling host thread's auxiliary streams/events/pinned bytes on the
 * current device (synchronises the device first). Safe to call at any time;
 * they are recreated on the next multi-stream call. */
int kle_release_resources(void);

/* Chunking of the register-resident tridiagonal solver for a given nx:
 * rows are padded to MR*P; the factor blob holds blob_doubles per sample. */
int kle_fine_layout(int nx, int* MR, int* P, int* blob_doubles);

/* LogNormalKL1D.linear_system (plugin contract pintuq/models.py:114-116):
 * a(m_j) = exp(sum_k kl_table[k][j] xi[s][k]) on the nx+1 midpoints,
 * dia = (a_j + a_{j+1}) inv_h2, off = -a_{j+1} inv_h2. xi is [M][d],
 * kl_table is [d][nx+1]. */
int kle_kl_tridiag_f64(const double* xi, int M, int d, const double* kl_table, int nx, double inv_h2,
                       double* dia, double* off, void* stream);

/* _linear_factor (pintuq/propagators.py:25-34): factor I + h*A for every
 * sample into the solver blob (size M * blob_doubles); g0 is the constant
 * source value (g(t) = g0 * ones). For 64 < nx <= 128 the blob also carries
 * the tables of the twisted two-lane sweep (kle_fine_tw.cu: twisted
 * factorisation, row scaling, steady state A x* = g0) and a per-sample flag
 * for samples without such a form (vanishing couplings, A without positive
 * pivots); kle_fgr_f64 sends flagged samples through the partitioned kernel.
 * For 128 < nx <= 512 it carries a second, (64, 8)-chunked blob with the
 * tables of the eight-lane scaled sweep (kle_fine_pw.cu), with the same flag
 * mechanism. Environment (read per call): KLE_FGR_TW=0 / KLE_FGR_PW=0 disable
 * those sweeps, KLE_FGR_SC=1 (set when factoring AND sweeping) selects the
 * scaled step of the partitioned kernel for 128 < nx <= 512. */
int kle_fine_factor_f64(const double* dia, const double* off, int M, int nx, double h, double g0,
                        double* blob, void* stream);

/* propagate_fine / propagate_coarse / fine_reference / coarse_sweep_init
 * (pintuq/propagators.py:121-176, pintuq/parareal.py:74-84):
 * out[s][q][g] = (J backward-Euler steps of size h)^(g+1) applied to
 * start[s][q], g = 0..nseg-1. start is [M][Q][nx], out is [M][Q][nseg][nx]. */
int kle_sweep_f64(const double* start, double* out, const double* blob, int M, int Q, int nx, int J,
                  int nseg, double h, double g0, void* stream);

/* Fused fine sweep + CGC right-hand side of one PCGC iteration
 * (pintuq/pcgc.py:321-330 fine sweeps; assemble_rhs_blocks :175-197;
 *  cgc_correct rhs :233-237):
 *   F_n   = F(from_n),  from = [u0, U_1..U_{N-1}]
 *   R_n   = scaling_n * ((I + dT A) F_n - prev_n),  prev = [alpha U_N, U_1..U_{N-1}]
 * which equals scaling_n * (dT (A b_n + g) + b_n) with b_n = F_n - G(prev_n).
 * F_given (optional) skips the sweep; F_out (optional) stores F. status
 * (optional) skips samples whose status word is not ACTIVE. */
int kle_fgr_f64(const double* U, const double* u0, const double* F_given, double* F_out, double* R,
                const double* fine_blob, const double* dia, const double* off, const double* scaling,
                const int32_t* status, int M, int N, int nx, int J, double dt, double dT, double g0,
                double alpha, void* stream);

/* Scratch for the three-step solve (per-CTA slabs). */
size_t kle_cgc_scratch_bytes(int M, int N, int nx);

/* Pivots of the shifted systems (lambda_f I + dT A), f = 0..N/2, for every
 * sample (factor_shifted, pintuq/pcgc.py:90-145; iteration invariant, so
 * computed once per batch). Layout [M][N/2+1][nx] complex. Returns 0 bytes /
 * KLE_ERR_UNSUPPORTED for shapes served by the on-the-fly path (N not a
 * power of two, N > 64, nx > 1024). */
size_t kle_shift_factor_bytes(int M, int N, int nx);
int kle_shift_factor_f64(const double* dia, const double* off, const double* lam, int M, int N, int nx, double dT,
                         double* sfac, void* stream);

/* three_step_solve (pintuq/pcgc.py:148-172) over M samples:
 *   u = diag(1/scaling) F (lambda I + dT A)^{-1} F* diag(scaling) r
 * r, u are [M][N][nx]; lam is [N] interleaved complex (re, im) =
 * build_alpha_circulant(N, alpha).eigenvalues (pintuq/pcgc.py:68-76),
 * scaling / inv_scaling its scaling and 1/scaling; imag[M] (optional) is
 * zeroed (every path here returns a real u via Hermitian completion; the
 * reference's max|Im u| diagnostic is kle_imag_residue_f64). sfac (optional, kle_shift_factor_f64)
 * selects the cluster kernel; without it the pivots are formed on the fly.
 * scratch: kle_cgc_scratch_bytes(M, N, nx) bytes (the cluster path needs
 * 16*M bytes of per-sample reduction slots; the call zeroes them). scaling
 * == NULL means r is already alpha-scaled. */
int kle_three_step_f64(const double* r, const double* scaling, const double* inv_scaling, const double* lam,
                       const double* dia, const double* off, const double* sfac, int M, int N, int nx, double dT,
                       double* u, double* imag, void* scratch, size_t scratch_bytes, void* stream);

/* max_imag_residue of three_step_solve (pintuq/pcgc.py:170-172, accumulated
 * per iteration at :340-342): the three-step solve done as the reference does
 * it — all N shifted systems solved independently, u = diag(1/scaling) F q
 * without Hermitian completion — and imag[s] = max(imag[s], max|Im u|) for
 * every sample with status == NULL or status[s] == KLE_SAMPLE_ACTIVE. r is
 * [M][N][nx]; load_scale == NULL means r is already alpha-scaled. A rounding-
 * level quantity that grows with cond(V) = alpha^{-(N-1)/N}; not bit-equal to
 * the reference's (different FFT). scratch: kle_imag_residue_scratch_bytes
 * (<= 256 MB). kle_pcgc_solve_f64 runs it every iteration when its imag
 * argument is non-NULL (and then uses one sample pipeline). */
size_t kle_imag_residue_scratch_bytes(int M, int N, int nx);
int kle_imag_residue_f64(const double* r, const double* load_scale, const double* inv_scaling, const double* lam,
                         const double* dia, const double* off, const int32_t* status, int M, int N, int nx,
                         double dT, double* imag, void* scratch, size_t scratch_bytes, void* stream);

/* CGC update of one PCGC iteration k (pintuq/pcgc.py:331-348): U <- three_step(R)
 * in place, increment = max|U_new - U| per sample, stop test against tol,
 * status/iters updated, inc_hist[s][k-1] recorded (imag[s]: the on-the-fly
 * path's Hermitian-completed residue, unused by the cluster/large paths), and
 * *active_count incremented once per still-active sample. R must already be
 * alpha-scaled (kle_fgr_f64 output). With sfac (cluster path) `scratch` holds
 * 16*M bytes of per-sample reduction slots that must be zero before the first
 * call; every call leaves them zero again. */
int kle_cgc_update_f64(const double* R, double* U, const double* inv_scaling, const double* lam,
                       const double* dia, const double* off, const double* sfac, int M, int N, int nx, double dT,
                       int k, int max_iters, double tol, int32_t* status, int32_t* iters, double* inc_hist,
                       double* imag, int32_t* active_count, void* scratch, size_t scratch_bytes,
                       void* stream);

/* Full outer loop of pcgc_solve (pintuq/pcgc.py:273-358) with
 * stop_on="increment" for M samples at once, each frozen at its own
 * iteration count. U: in = initial guess states [M][N][nx], out = final
 * states. status/iters [M], inc_hist [M][max_iters] (NaN-initialised by the
 * call), imag [M]. Synchronises the stream once per outer iteration (a
 * 4-byte read of the active-sample count). */
size_t kle_pcgc_workspace_bytes(int M, int N, int nx);
int kle_pcgc_solve_f64(double* U, const double* u0, const double* dia, const double* off,
                       const double* fine_blob, const double* scaling, const double* inv_scaling,
                       const double* lam, int M, int N, int nx, int J, double T, double alpha, double g0,
                       double tol, int max_iters, int32_t* status, int32_t* iters, double* inc_hist,
                       double* imag, void* workspace, size_t workspace_bytes, void* stream);

/* pcgc_solve with a reference trajectory (pintuq/pcgc.py:273-358 with
 * `reference=`): ref [M][N][nx] is the serial fine solution (fine_reference,
 * pintuq/propagators.py:160-176). Records err_hist [M][max_iters+1][N]
 * (_error_record, pintuq/parareal.py:87-91; k = 0 is the initial guess,
 * NaN-initialised) and max_err [M] (the last recorded max error); both
 * optional. stop_on_reference != 0 is stop_on="reference": a sample stops
 * at the first k whose max error is <= tol (k = 0 included, iters = 0);
 * otherwise the increment stops it as in kle_pcgc_solve_f64. */
int kle_pcgc_solve_ref_f64(double* U, const double* u0, const double* dia, const double* off,
                           const double* fine_blob, const double* scaling, const double* inv_scaling,
                           const double* lam, int M, int N, int nx, int J, double T, double alpha, double g0,
                           double tol, int max_iters, const double* ref, int stop_on_reference, int32_t* status,
                           int32_t* iters, double* inc_hist, double* err_hist, double* max_err, double* imag,
                           void* workspace, size_t workspace_bytes, void* stream);

/* One error record of the iterate U against ref (pintuq/parareal.py:87-91)
 * for the samples active at iteration k (status ACTIVE or iters == k; all at
 * k = 0), written to err_hist[s][k][:] ([M][max_iters+1][N], optional) and
 * max_err[s] (optional). With stop_on_reference, samples whose max error is
 * <= tol are marked CONVERGED with iters = k (active_count decremented for
 * k > 0; at k = 0 it counts the samples left active). Used by the batched
 * loops (1D and 2D). */
int kle_err_ref_f64(const double* U, const double* ref, int M, int N, int nx, int k, int max_iters, double tol,
                    int stop_on_reference, int32_t* status, int32_t* iters, int32_t* active_count, double* err_hist,
                    double* max_err, void* stream);

/* Mean-error aggregation of the experiment harness (pintuq/experiments.py:
 * 314-334) over the error records of a reference-tracked batch: a sample is
 * "good" when its records err_hist[s][0..iters[s]][:] ([M][max_iters+1][N],
 * as written by kle_pcgc_solve_ref_f64) are all finite; each good sample's
 * error vectors are padded with their last record to k_max + 1 rows and the
 * rows are summed over the good samples in id order. Writes good[M] (0/1),
 * counts[2] = (n_good, k_max) and sums[max_iters+1][N] for the rows 0..k_pad
 * (k_pad < 0: this batch's own k_max; a sharded caller passes the global
 * k_max), NaN past them. mean_vectors = sums / n_good (numpy's
 * stack.mean(axis=0), bit for bit); mean_max_error = their row-wise max. */
int kle_err_aggregate_f64(const double* err_hist, const int32_t* iters, int M, int N, int max_iters, int k_pad,
                          int32_t* good, int32_t* counts, double* sums, void* stream);

/* Classical parareal, the paper's comparison baseline (parareal_solve,
 * pintuq/parareal.py:100-191), for the tridiagonal models:
 *   U_n^{k+1} = G(U_{n-1}^{k+1}) + F(U_{n-1}^k) - G(U_{n-1}^k),  U_{-1} = u0,
 * G one backward-Euler step of dT (coarse_blob = kle_fine_factor_f64 with
 * h = dT), F J steps of dt (fine_blob). init: Gprev[s][n] = G(start_n) with
 * start = [u0, U_0 .. U_{N-2}] (:153-155). step: the sequential correction
 * of one outer iteration given F[s][n] = F(start_n) (:170-176), increment
 * and stop test (:181-190), per-sample status as kle_cgc_update_f64.
 * solve: the whole loop (ref / err_hist / max_err / stop_on_reference as
 * kle_pcgc_solve_ref_f64; ref may be NULL). nx <= 1024. */
int kle_parareal_init_f64(const double* U, const double* u0, const double* coarse_blob, int M, int N, int nx,
                          double dT, double g0, double* Gprev, void* stream);
int kle_parareal_step_f64(double* U, const double* u0, const double* F, double* Gprev, const double* coarse_blob,
                          int M, int N, int nx, double dT, double g0, int k, int max_iters, double tol,
                          int32_t* status, int32_t* iters, double* inc_hist, int32_t* active_count, void* stream);
size_t kle_parareal_workspace_bytes(int M, int N, int nx);
int kle_parareal_solve_f64(double* U, const double* u0, const double* dia, const double* off,
                           const double* fine_blob, const double* coarse_blob, int M, int N, int nx, int J, double T,
                           double g0, double tol, int max_iters, const double* ref, int stop_on_reference,
                           int32_t* status, int32_t* iters, double* inc_hist, double* err_hist, double* max_err,
                           void* workspace, size_t workspace_bytes, void* stream);

/* Nonlinear tridiagonal models (Burgers kind 0, Allen-Cahn kind 1): fused
 * backward-Euler sweeps with a damped Newton iteration per step, the
 * compiled kernels of the reference (pintuq/_kernels.pyx:100-163,
 * be_sweep_burgers / be_sweep_allencahn; propagators.py:82-99). For every
 * sample s and start q: out[s][q][g] = state after (g+1)*J steps of size h
 * from start[s][q]; p0[s] = nu (Burgers) or eps (Allen-Cahn); bc_lo/bc_hi the
 * Allen-Cahn boundary values. status[s][q] (optional) = 1-based index of the
 * first step whose Newton iteration missed newton_tol within max_newton
 * iterations (0 = success), as the reference's kernel status. */
size_t kle_newton_work_bytes(int M, int Q, int nx);
int kle_newton_sweep_f64(int kind, const double* start, double* out, const double* p0, int M, int Q, int nx, int J,
                         int nseg, double h, double dx, double bc_lo, double bc_hi, double newton_tol, int max_newton,
                         const int32_t* active, int32_t* status, void* work, size_t work_bytes, void* stream);

/* The parareal correction of subinterval n (pintuq/parareal.py:174-176) for
 * the samples with status ACTIVE (or all, status = NULL):
 * U[s][n] = (Gn[s] + F[s][n]) - Gprev[s][n]; Gprev[s][n] = Gn[s]. Used by the
 * nonlinear-model parareal loop, whose coarse steps are Newton sweeps. */
int kle_para_combine_f64(double* U, const double* Gn, const double* F, double* Gprev, const int32_t* status, int M,
                         int N, int nx, int n, void* stream);

/* cgc_correct for the nonlinear tridiagonal models (pintuq/pcgc.py:245-270):
 * the simplified Newton iteration with the averaged Jacobian, each inner step
 * a diagonalised three-step solve of (C_alpha (x) I - dT I (x) mean_jac),
 * until max|u_next - u_l| <= newton_tol (at most 150 inner steps; then the
 * sample's status becomes KLE_SAMPLE_NEWTON). One CTA per active sample:
 * U [M][N][nx] the previous iterate, b = F_end - G(prev) (assemble_rhs_blocks),
 * Uout the correction; inner[s] = inner iterations. N * nx <= ~9000. */
int kle_newton_cgc_f64(int kind, const double* U, const double* b, double* Uout, const double* p0, const double* lam,
                       const double* scaling, const double* inv_scaling, int M, int N, int nx, double dT, double dx,
                       double bc_lo, double bc_hi, double newton_tol, int32_t* status, int32_t* inner, void* stream);

/* forward_dft / inverse_dft (pintuq/pcgc.py:79-87): out[k][l] = sum_n in[n][l]
 * exp(sign 2 pi i n k / N) / sqrt(N) on [N][L] complex (interleaved re, im)
 * arrays; sign = +1 is F (x) I (np.fft.ifft, ortho), -1 is F* (x) I (np.fft.fft). */
int kle_block_dft_f64(const double* in, double* out, int N, int L, int sign, void* stream);

/* One shifted solver of factor_shifted (pintuq/pcgc.py:112-135):
 * (lam I - dT J) q = p for nrhs complex right-hand sides p [nrhs][nx], J =
 * tridiag(sub [nx-1] = J[i+1][i], dia [nx], sup [nx-1] = J[i][i+1]), real;
 * cwork [nrhs][nx] complex scratch; status [nrhs] = 1 on a zero pivot
 * (SingularShiftError). */
int kle_shifted_tridiag_solve_f64(const double* sub, const double* dia, const double* sup, double lam_re,
                                  double lam_im, double dT, const double* p, double* q, double* cwork, int nx,
                                  int nrhs, int32_t* status, void* stream);

/* Matrix-free Krylov 2D solvers (the alternative to the banded
 * factors above, selected by twod.DeviceOperator2D(solver="krylov")):
 * Jacobi-PCG for every backward-Euler step of (I + h A) (warm started from the
 * previous step) and Jacobi-COCG for the shifted systems (lambda_f I + dT A),
 * applied matrix-free from (dia, ex, ey), each to ||r||_2 <= rtol ||b||_2
 * (max_its iterations at most; *its, optional, accumulates the iteration
 * count). fgr: the fused fine sweeps + CGC right-hand side of
 * kle_2d_fgr_staged_f64 (F_given / F_out optional); sweep: out[s][q] = J
 * steps of size h from start[s][q] (nseg = 1); cgc: kle_2d_cgc_f64 with the
 * COCG solves (work: kle_2d_cgc_krylov_work_doubles, zeroed before the first
 * call). n <= 128. */
int kle_2d_fgr_krylov_f64(const double* U, const double* u0, const double* F_given, const double* dia,
                          const double* ex, const double* ey, const double* scaling, const int32_t* status, int M,
                          int N, int n, int J, double dt, double dT, double g0, double alpha, double rtol,
                          int max_its, double* R, double* F_out, long long* its, void* stream);
int kle_2d_sweep_krylov_f64(const double* start, const double* dia, const double* ex, const double* ey, int M, int Q,
                            int n, int J, double h, double g0, double rtol, int max_its, double* out, long long* its,
                            void* stream);
size_t kle_2d_cgc_krylov_work_doubles(int M, int N, int n);
int kle_2d_cgc_krylov_f64(const double* R, const double* load_scale, double* U, double* Uout, const double* dia,
                          const double* ex, const double* ey, const double* lam, const double* inv_scaling, int M,
                          int N, int n, int k, int max_iters, double tol, int32_t* status, int32_t* iters,
                          double* inc, double* inc_hist, int32_t* active_count, double dT, double rtol, int max_its,
                          double* work, size_t work_doubles, long long* its, void* stream);

/* gpc_basis_matrix (pintuq/surrogate.py:208-248) at the mapped points
 * (KLGpcSurrogate.map_parameters, ParameterMap.apply pintuq/models.py:39-45):
 * Psi[M][P] from raw xi[M][d]; family 0 = probabilists' Hermite
 * (norms[k] = 1/sqrt(k!)), 1 = Legendre (norms[k] = sqrt(2k+1));
 * maps = optional [d][3] (kind, lo, hi): kind 0 identity, 1 affine onto
 * [-1, 1], 2 cos(2 pi v); NULL = identity; midx[P][d] = gpc_multi_indices. */
int kle_gpc_basis_f64(const double* xi, int M, int d, int degree, int family, const double* maps,
                      const int32_t* midx, int P, const double* norms, double* Psi, void* stream);

/* surrogate_predict batched (pintuq/surrogate.py:321-333):
 * U0[M][L] = mean[L] + Psi[M][K] * C[K][L]  (FP64 tensor cores, DMMA). */
int kle_gpc_eval_f64(const double* Psi, int M, int K, const double* C, const double* mean, int L, double* U0,
                     void* stream);

/* Surrogate build on the device (pintuq/surrogate.py:144-184):
 * C[M][L] = bias[L] (optional) + A[M][K] * B, B = [K][L] row-major, or
 * B^T with B = [L][K] row-major when trans_b != 0 (the Gram matrix X X^T of
 * kl_build :153 and the projections X G^T of kl_coefficients :183), DMMA. */
int kle_gemm_f64(const double* A, const double* B, const double* bias, double* C, int M, int K, int L, int trans_b,
                 void* stream);
/* out[s][l] = X[s][l] - v[l]: snapshot fluctuations about the mean (:63). */
int kle_sub_row_f64(const double* X, const double* v, double* out, int M, int L, void* stream);

/* Moments (absent in the reference): out[l] = sum_s U[s][l]
 * (center == NULL) or sum_s (U[s][l] - center[l])^2. Deterministic order. */
size_t kle_col_sum_scratch_bytes(int M, int L);
int kle_col_sum_f64(const double* U, int M, int L, const double* center, double* out, void* scratch,
                    void* stream);

/* out = a*x + b*y (n elements). */
int kle_axpby_f64(const double* x, const double* y, double* out, double a, double b, size_t n, void* stream);


/* ===================== 2D 5-point path (BASELINE config 3) ==================
 * DOF order x fastest on an n x n interior grid (nx = n*n <= 127*127); the
 * operator is A = 5-point(dia, ex, ey): ex[i] = A[i][i+1], ey[i] = A[i][i+n]
 * (zero across the grid edge). Implicit solves are direct, like the
 * reference's SuperLU: banded L D L^T without pivoting, factored once per
 * solve and reused by every outer iteration. */

/* LinearModel.linear_system of the 2D KL plugin (pintuq/models.py:114-116;
 * models.LogNormalKL2D): xi[M][d] -> dia/ex/ey[M][n*n]. kl_table [d][(n+1)^2]. */
int kle_2d_kl5pt_f64(const double* xi, int M, int d, const double* kl_table, int n, double inv_h2, double* dia,
                     double* ex, double* ey, void* stream);

/* _linear_factor (pintuq/propagators.py:25-34) and factor_shifted
 * (pintuq/pcgc.py:137-145) for bandwidth n: B = L D L^T, L stored by columns,
 * Lt[i][t] = L(i+1+t, i), Dinv[i] = 1/D[i]. lam == NULL: B = shift*I + c*A,
 * real, one matrix per sample (Lt[M][nx][n], Dinv[M][nx]). lam != NULL (NF
 * interleaved complex shifts): B = lam_f*I + c*A, complex, M*NF matrices,
 * Lt[M*NF][nx][n] and Dinv[M*NF][nx] as interleaved complex. */
int kle_2d_factor_f64(const double* dia, const double* ex, const double* ey, int M, int n, const double* lam,
                      int NF, double shift, double c, double* Lt, double* Dinv, void* stream);

/* Scratch (doubles) of kle_2d_fgr_f64 / kle_2d_sweep_f64 for M samples of N
 * (or Q) right-hand sides. */
size_t kle_2d_fine_work_doubles(int M, int N, int n);

/* propagate_fine for all subintervals + assemble_rhs_blocks + the rhs of
 * cgc_correct (pintuq/propagators.py:121-145, pcgc.py:175-197, 233-237):
 * Rout[s][k] = scaling_k ((I + dT A) F_k - prev_k), F_k = J BE steps of dt from
 * U_{k-1} (u0 for k = 0), prev_0 = alpha U_{N-1}. Real factor of I + dt A.
 * F_given != NULL (stand-alone cgc_correct): no sweep, F_k = F_given[s][k]. */
int kle_2d_fgr_f64(const double* U, const double* u0, const double* F_given, const double* dia, const double* ex,
                   const double* ey, const double* Lt, const double* Dinv, const double* scaling,
                   const int32_t* active, int M, int N, int n, int J, double dt, double dT, double g0,
                   double alpha, double* work, size_t work_doubles, double* Rout, void* stream);

/* propagate_fine / propagate_coarse / fine_reference (pintuq/propagators.py
 * :121-176): out[s][q][g] = F^{(g+1)}(start[s][q]), segments of J steps of h. */
int kle_2d_sweep_f64(const double* start, const double* dia, const double* ex, const double* ey,
                     const double* Lt, const double* Dinv, int M, int Q, int n, int J,
                     int nseg, double h, double g0, double* work, size_t work_doubles, double* out, void* stream);

/* The real factor (Lt, Dinv from kle_2d_factor_f64) restaged for the TMA
 * sweeps: per sample, direction (forward, backward) and block of 8 rows, one
 * contiguous chunk of (n + 9) * 8 doubles holding the block's band
 * coefficients in the order the sweep reads them and D^{-1} of its rows.
 * Built once per solve; kle_2d_fgr_staged_f64 / kle_2d_sweep_staged_f64 stream
 * one chunk per block with cp.async.bulk (pintuq/propagators.py:25-39: the
 * factor is computed once and reused by every BE step, as SuperLU's is). */
size_t kle_2d_fine_stage_doubles(int M, int n);
int kle_2d_fine_stage_f64(const double* Lt, const double* Dinv, int M, int n, double* stage, void* stream);

/* kle_2d_fgr_f64 / kle_2d_sweep_f64 on the staged factor (same outputs, same
 * workspace size; one CTA per sample and 32 right-hand sides). */
int kle_2d_fgr_staged_f64(const double* U, const double* u0, const double* F_given, const double* dia,
                          const double* ex, const double* ey, const double* stage, const double* scaling,
                          const int32_t* active, int M, int N, int n, int J, double dt, double dT, double g0,
                          double alpha, double* work, size_t work_doubles, double* Rout, void* stream);
int kle_2d_sweep_staged_f64(const double* start, const double* stage, int M, int Q, int n, int J, int nseg,
                            double h, double g0, double* work, size_t work_doubles, double* out, void* stream);

/* Scratch (doubles) of kle_2d_cgc_f64. */
size_t kle_2d_cgc_work_doubles(int M, int N, int n);

/* three_step_solve (pintuq/pcgc.py:148-172) + the increment / stop test of
 * pcgc_solve (:335-348), N even: p = fft(r)/sqrt(N), q_f = B_f^{-1} p_f for
 * f <= N/2 (complex factors from kle_2d_factor_f64), u = Re ifft(q) sqrt(N)^-1
 * / scaling. R is alpha-scaled unless load_scale (stand-alone mode). With
 * status != NULL and Uout == NULL, U is updated in place and the per-sample
 * increment, status words, iteration counts and active count are written as
 * in kle_cgc_update_f64; otherwise u goes to Uout (imag residue is 0: the
 * Hermitian completion makes u real by construction). */
int kle_2d_cgc_f64(const double* R, const double* load_scale, double* U, double* Uout, const double* Lt,
                   const double* Dinv, const double* inv_scaling, int M, int N, int n, int k, int max_iters,
                   double tol, int32_t* status, int32_t* iters, double* inc, double* inc_hist,
                   int32_t* active_count, double* work, size_t work_doubles, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* KLE_B200_H */
