// Internal (C++) interfaces between the kernel translation units and the
// C-ABI layer (kle_capi.cu). Not exported.
#pragma once
#include <cuda_runtime.h>
#include <cstddef>
#include <atomic>
#include <cstdint>

namespace kle {

int set_error(int code, const char* msg);
int check_launch(const char* what);

// Kernel attributes (cudaFuncSetAttribute) are per device: the setup runs once
// per device this process touches (bit `dev` of the mask), its return codes are
// checked, and concurrent first calls from several host threads are benign
// (the attribute calls are idempotent).
struct PerDeviceOnce {
  std::atomic<unsigned long long> mask{0};
};
template <class F>
inline int once_per_device(PerDeviceOnce& once, const char* what, F&& setup) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev > 63) return set_error(2, what);
  const unsigned long long bit = 1ull << dev;
  if (once.mask.load(std::memory_order_acquire) & bit) return 0;
  const cudaError_t e = setup();
  if (e != cudaSuccess) {
    cudaGetLastError();
    return set_error(2, what);
  }
  once.mask.fetch_or(bit, std::memory_order_acq_rel);
  return 0;
}

// Stream-ordering helpers of the multi-stream paths (the PCGC sample pipelines
// in kle_capi.cu, the two sub-batch streams of the large-block CGC): created
// on first use per (host thread, current device), never device memory, freed
// by kle_release_resources() (include/kle_b200.h).
constexpr int kMaxPipes = 4;
struct AuxResources {
  cudaStream_t sf[kMaxPipes], sc[kMaxPipes];  // per pipeline: fine sweeps (low priority), CGC (high priority)
  cudaEvent_t done[kMaxPipes], fdone[kMaxPipes], ready;
  cudaStream_t cgcl[2];                       // large-block CGC sub-batch streams
  cudaEvent_t cgcl_ev[3];
  int32_t* h_count;                           // pinned [kMaxPipes]
};
AuxResources* aux_resources();  // nullptr (and the error string set) on failure

struct FineLayoutRT {
  int MR, P, R, pipe, doubles;
  int W = 0;     // > 0: multi-warp system (kle_fine_mw.cu), P = 32 * W
  int kind = 0;  // 0: factors in registers (kle_fine.cu); 1: factors in shared memory (kle_fine_sf.cu)
};
FineLayoutRT fine_layout(int nx);

struct FgrArgs {
  const double* U;        // [M][N][nx] current iterate (U_1..U_N)
  const double* u0;       // [nx] initial state (shared by all samples)
  const double* F_given;  // optional [M][N][nx]: skip the sweep, use these F ends
  double* F_out;          // optional [M][N][nx]: also store the F ends
  double* Rout;           // [M][N][nx] scaled CGC right-hand sides
  const double* ffac;     // fine factor blobs [M][doubles]
  const double* dia;      // [M][nx]
  const double* off;      // [M][nx] (entry nx-1 unused)
  const double* scaling;  // [N] alpha^(n/N)
  const int32_t* active;  // [M] sample status (0 = active) or null
  int M, N, nx, J;
  double dt, dT, g0, alpha;
  int tw_fallback = 0;    // 1: only the samples whose blob carries a nonzero flag at flag_off (the samples the
                          // twisted / scaled / eight-lane kernel skipped)
  int flag_off = 0;       // offset (doubles) of that flag in a sample's blob
  int tw_none_flagged = 0;  // the caller counted the flags (tw_count_flagged): no fallback launch needed
};

struct PararealArgs {
  double* U;              // [M][N][nx] in: U^k, out: U^{k+1} (mode 1); read-only in mode 0
  const double* u0;       // [nx]
  const double* F;        // [M][N][nx] fine ends F(U_n^k) (mode 1)
  double* Gprev;          // [M][N][nx] G(U_n^k): written (mode 0) / read and replaced (mode 1)
  const double* gfac;     // coarse factor blobs [M][doubles] of I + dT A
  int32_t* status;        // optional [M]
  int32_t* iters;         // optional [M]
  double* inc_hist;       // optional [M][max_iters]
  int32_t* active_count;  // optional
  int M, N, nx, k, max_iters, mode;
  double dT, g0, tol;
};
int parareal_run(FineLayoutRT lay, const PararealArgs& a, cudaStream_t st);

struct NewtonArgs {
  const double* start;    // [M][Q][nx]
  double* out;            // [M][Q][nseg][nx]
  const double* p0;       // [M] nu (Burgers) or eps (Allen-Cahn)
  const int32_t* active;  // optional [M]
  int32_t* status;        // optional [M][Q]: first failing step (1-based), 0 = ok
  int M, Q, nx, J, nseg, kind, max_newton;
  double h, dx, bc_lo, bc_hi, newton_tol;
};
size_t newton_work_doubles(int M, int Q, int nx);
struct NewtonCgcArgs {
  const double* U;            // [M][N][nx] U^k
  const double* b;            // [M][N][nx] F - G(prev)
  double* Uout;               // [M][N][nx] U^{k+1}
  const double* p0;           // [M]
  const double* lam;          // [2N]
  const double* scaling;      // [N]
  const double* inv_scaling;  // [N]
  int32_t* status;            // optional [M]: skip non-active, NEWTON on failure
  int32_t* inner;             // optional [M]: simplified-Newton iterations
  int M, N, nx, kind;
  double dT, dx, bc_lo, bc_hi, newton_tol;
};
int newton_cgc(const NewtonCgcArgs& a, cudaStream_t st);
int newton_sweep(const NewtonArgs& a, double* work, cudaStream_t st);
int para_combine(double* U, const double* Gn, const double* F, double* Gp, const int32_t* status, int M, int N,
                 int nx, int n, cudaStream_t st);

struct SweepArgs {
  const double* start;  // [M][Q][nx]
  double* out;          // [M][Q][nseg][nx]
  const double* fac;    // blobs [M][doubles] for step h
  int M, Q, nx, J, nseg;
  double h, g0;
};

int sf_blob_doubles(int MR, int P);
int sf_factor(FineLayoutRT lay, const double* dia, const double* off, double* blob, int M, int nx, double h,
              double g0, cudaStream_t st);
int sf_fgr(FineLayoutRT lay, const FgrArgs& a, cudaStream_t st);
int sf_sweep(FineLayoutRT lay, const SweepArgs& a, cudaStream_t st);
// twisted two-lane sweep for 64 < nx <= 128 (kle_fine_tw.cu); tables in the (16, 8) blob's spare part
bool tw_supported(const FineLayoutRT& lay, int nx);
bool sc_supported(const FineLayoutRT& lay);  // scaled partitioned sweep (be_steps_sc), P = 32 layouts
int sc_flag_offset(const FineLayoutRT& lay);
// eight-lane scaled sweep for 128 < nx <= 512 (kle_fine_pw.cu): 64 rows of one right-hand side per lane,
// coefficients from shared memory; tables = a (64, 8) blob behind the (16, 32) blob
bool pw_supported(const FineLayoutRT& lay, int nx);
int pw_flag_offset();
int pw_fgr(const FgrArgs& a, cudaStream_t st);
int tw_factor(const double* dia, const double* off, double* blob, int M, int nx, double h, double g0,
              cudaStream_t st);
int tw_fgr(const FgrArgs& a, cudaStream_t st);
// samples whose blob carries a nonzero "no scaled form" flag at blob[s * stride + off] (stride 0: the twisted tables)
int tw_count_flagged(const double* blob, int M, int stride, int off, int32_t* count, cudaStream_t st);
int mw_warps(int nx);
int mw_blob_doubles(int nx);
int mw_factor(const double* dia, const double* off, double* blob, int M, int nx, double h, cudaStream_t st);
int mw_fgr(const FgrArgs& a, cudaStream_t st);
int mw_sweep(const SweepArgs& a, cudaStream_t st);

int fine_factor(FineLayoutRT lay, const double* dia, const double* off, double* blob, int M, int nx,
                double h, double g0, cudaStream_t st);
int fine_fgr(FineLayoutRT lay, const FgrArgs& a, cudaStream_t st);
int fine_sweep(FineLayoutRT lay, const SweepArgs& a, cudaStream_t st);

struct CgcArgs {
  const double* R;          // [M][N][nx] right-hand sides (already alpha-scaled unless load_scale)
  const double* load_scale; // optional [N]: multiply R rows on load (stand-alone three-step)
  double* U;                // [M][N][nx] in: U^k (for the increment), out: U^{k+1} (fused mode)
  double* Uout;             // optional separate output (stand-alone mode); then U may be null
  const double* dia;        // [M][nx]
  const double* off;        // [M][nx]
  const double* lam;        // [2*N] interleaved (re, im) eigenvalues of C_alpha
  const double* inv_scaling;// [N] 1/alpha^(n/N)
  double* scratch;          // per-CTA slabs
  size_t scratch_doubles_per_cta;
  int32_t* status;          // optional [M] sample status (fused mode)
  int32_t* iters;           // optional [M]
  double* inc;              // optional [M] increment of this iteration
  double* inc_hist;         // optional [M][max_iters]
  double* imag;             // optional [M] running max imaginary residue
  int32_t* active_count;    // optional device counter of still-active samples
  unsigned long long* red_slots;  // cluster path: [M][2] (max bits, arrival ticket), zero-initialised once
  int full;                 // 1: imaginary-residue diagnostic (all N frequencies, no Hermitian
                            // completion; writes only imag, never U / status)
  int M, N, nx, k, max_iters;
  double dT, tol;
};

bool cgc_cluster_supported(int N, int nx);
size_t shift_factor_doubles(int M, int N, int nx);
int shift_factor(const double* dia, const double* off, const double* lam, int M, int N, int nx, double dT,
                 double* sfac, cudaStream_t st);
int cgc_cluster_run(const CgcArgs& a, const double* sfac, cudaStream_t st);
// small blocks (power-of-two N <= 16, nx <= 128): one CTA per sample, register FFTs (kle_cgc_row.cu);
// cgc_cluster_run dispatches to it
bool cgc_row_supported(int N, int nx);
int cgc_row_run(const CgcArgs& a, const double* sfac, cudaStream_t st);

int cgc_grid(int M, int N, int nx);
size_t cgc_scratch_doubles_per_cta(int N, int nx);
int cgc_run(const CgcArgs& a, cudaStream_t st);
size_t imag_residue_scratch_bytes(int M, int N, int nx);
int imag_residue_run(const CgcArgs& a, cudaStream_t st);
// large blocks (power-of-two N <= 1024, any nx): streaming FFT / solve / FFT kernels
bool cgc_large_supported(int N, int nx);
size_t cgc_large_scratch_bytes(int M, int N, int nx);
int cgc_large_run(const CgcArgs& a, cudaStream_t st);

int kl_tridiag(const double* xi, int M, int d, const double* table, int nx, double inv_h2, double* dia,
               double* off, cudaStream_t st);

int gpc_basis(const double* xi, int M, int d, int degree, int family, const double* maps, const int32_t* midx, int P,
              const double* norms, double* Psi, cudaStream_t st);
int gemm_bias(const double* A, const double* B, const double* bias, double* C, int M, int K, int L,
              cudaStream_t st, bool trans_b = false);
int sub_row(const double* X, const double* v, double* out, int M, int L, cudaStream_t st);

int col_sum(const double* U, int M, int L, const double* center, double* out, double* partial,
            cudaStream_t st);
size_t col_sum_partial_doubles(int M, int L);

int err_ref(const double* U, const double* ref, int M, int N, int nx, int k, int max_iters, double tol, int stop_ref,
            int32_t* status, int32_t* iters, int32_t* active_count, double* err_hist, double* max_err,
            cudaStream_t st);

int block_dft(const double* in, double* out, int N, int L, int sign, cudaStream_t st);
int shifted_tridiag(const double* sub, const double* dia, const double* sup, double lre, double lim, double dT,
                    const double* p, double* q, double* cwork, int nx, int nrhs, int32_t* status, cudaStream_t st);

int axpby(const double* x, const double* y, double* out, double a, double b, size_t n, cudaStream_t st);

int err_aggregate(const double* err, const int32_t* iters, int M, int N, int max_iters, int k_pad, int32_t* good,
                  int32_t* counts, double* sums, cudaStream_t st);

// Fused PCGC iteration for small blocks (kle_iter_small.cu): fine sweeps,
// CGC right-hand side and three-step solve of one sample per CTA.
struct IterSmallArgs {
  double* U;                // [M][N][nx] in: U^k, out: U^{k+1}
  const double* R;          // CGC-only variant: [M][N][nx] alpha-scaled right-hand sides (fgr_kernel)
  const double* u0;         // [nx]
  const double* ffac;       // fine factor blobs (layout 16 x 8) [M][doubles]
  const double* dia;        // [M][nx]
  const double* off;        // [M][nx]
  const double* sfac;       // shift pivots [M][N/2+1][nx] complex
  const double* scaling;    // [N]
  const double* inv_scaling;// [N]
  int32_t* status;          // [M]
  int32_t* iters;           // [M]
  double* inc_hist;         // optional [M][max_iters]
  int32_t* active_count;    // optional
  int M, N, nx, J, k, max_iters;
  double dt, dT, g0, alpha, tol;
};
bool iter_small_supported(int N, int nx);
int iter_small_run(const IterSmallArgs& a, cudaStream_t st);
bool cgc_small_supported(int N, int nx);
int cgc_small_run(const IterSmallArgs& a, cudaStream_t st);

// Matrix-free Krylov 2D solvers (kle_2d_krylov.cu).
struct Kry2dArgs {
  const double* start;      // start_from_u: the iterate U [M][Q][nx] (system q starts at u0 / U_{q-1},
                            // and prev rows of the CGC rhs come from it); else starts [M][Q][nx]
  const double* u0;         // [nx]
  const double* F_given;    // optional [M][Q][nx]: skip the sweeps, rhs epilogue from these F ends
  const double* dia;        // [M][nx]
  const double* ex;         // [M][nx]
  const double* ey;         // [M][nx]
  const double* scaling;    // [Q] (rhs epilogue)
  const int32_t* status;    // optional [M]
  double* F_out;            // optional [M][Q][nx]
  double* R;                // optional [M][Q][nx]: scaling_q ((I + dT A) F_q - prev_q)
  long long* its;           // optional: total CG iterations (atomic)
  int M, Q, n, J, max_its, start_from_u;
  double h, dT, g0, alpha, rtol;
};
int kry2d_fine(const Kry2dArgs& a, cudaStream_t st);
struct Cplx;
int kry2d_shift_solve(Cplx* P, const double* dia, const double* ex, const double* ey, const double* lam,
                      const int32_t* status, int M, int NF, int n, double dT, double rtol, int max_its, Cplx* work,
                      long long* its, cudaStream_t st);

}  // namespace kle
