// extern "C" boundary of libkle_b200.so (declared in include/kle_b200.h).
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>

#include "../../include/kle_b200.h"
#include "kle_common.cuh"
#include "kle_internal.h"

namespace kle {

static thread_local std::string g_err;

int set_error(int code, const char* msg) {
  g_err = msg ? msg : "";
  return code;
}

int check_launch(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    std::string m = std::string(what) + ": " + cudaGetErrorString(e);
    return set_error(KLE_ERR_CUDA, m.c_str());
  }
  return KLE_OK;
}

static inline size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

}  // namespace kle

using namespace kle;

#define KLE_STREAM(s) (reinterpret_cast<cudaStream_t>(s))
#define KLE_TRY(expr)            \
  do {                           \
    const int _rc = (expr);      \
    if (_rc != KLE_OK) return _rc; \
  } while (0)

namespace kle {

static thread_local AuxResources* g_aux[64] = {};

static void aux_destroy(AuxResources* r) {
  for (int p = 0; p < kMaxPipes; ++p) {
    if (r->sf[p]) cudaStreamDestroy(r->sf[p]);
    if (r->sc[p]) cudaStreamDestroy(r->sc[p]);
    if (r->done[p]) cudaEventDestroy(r->done[p]);
    if (r->fdone[p]) cudaEventDestroy(r->fdone[p]);
  }
  if (r->ready) cudaEventDestroy(r->ready);
  for (int q = 0; q < 2; ++q)
    if (r->cgcl[q]) cudaStreamDestroy(r->cgcl[q]);
  for (int q = 0; q < 3; ++q)
    if (r->cgcl_ev[q]) cudaEventDestroy(r->cgcl_ev[q]);
  if (r->h_count) cudaFreeHost(r->h_count);
  delete r;
}

AuxResources* aux_resources() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) {
    set_error(KLE_ERR_CUDA, "aux_resources: no current device");
    return nullptr;
  }
  if (g_aux[dev]) return g_aux[dev];
  auto* r = new AuxResources{};
  int lo = 0, hi = 0;
  bool ok = cudaDeviceGetStreamPriorityRange(&lo, &hi) == cudaSuccess;
  for (int p = 0; p < kMaxPipes && ok; ++p) {
    ok = ok && cudaStreamCreateWithPriority(&r->sf[p], cudaStreamNonBlocking, lo) == cudaSuccess;
    ok = ok && cudaStreamCreateWithPriority(&r->sc[p], cudaStreamNonBlocking, hi) == cudaSuccess;
    ok = ok && cudaEventCreateWithFlags(&r->done[p], cudaEventDisableTiming) == cudaSuccess;
    ok = ok && cudaEventCreateWithFlags(&r->fdone[p], cudaEventDisableTiming) == cudaSuccess;
  }
  ok = ok && cudaEventCreateWithFlags(&r->ready, cudaEventDisableTiming) == cudaSuccess;
  for (int q = 0; q < 2 && ok; ++q) ok = cudaStreamCreateWithFlags(&r->cgcl[q], cudaStreamNonBlocking) == cudaSuccess;
  for (int q = 0; q < 3 && ok; ++q) ok = cudaEventCreateWithFlags(&r->cgcl_ev[q], cudaEventDisableTiming) == cudaSuccess;
  ok = ok && cudaHostAlloc(&r->h_count, (kMaxPipes + 1) * sizeof(int32_t), cudaHostAllocDefault) == cudaSuccess;
  if (!ok) {
    cudaGetLastError();
    aux_destroy(r);
    set_error(KLE_ERR_CUDA, "aux_resources: stream/event/pinned-buffer creation failed");
    return nullptr;
  }
  g_aux[dev] = r;
  return r;
}

}  // namespace kle

extern "C" {

int kle_abi_version(void) { return KLE_ABI_VERSION; }

const char* kle_last_error(void) { return g_err.c_str(); }

int kle_fine_layout(int nx, int* MR, int* P, int* blob_doubles) {
  const FineLayoutRT l = fine_layout(nx);
  if (l.MR == 0) return set_error(KLE_ERR_UNSUPPORTED, "nx exceeds the largest supported fine layout (4096)");
  if (MR) *MR = l.MR;
  if (P) *P = l.P;
  if (blob_doubles) *blob_doubles = l.doubles;
  return KLE_OK;
}

int kle_kl_tridiag_f64(const double* xi, int M, int d, const double* kl_table, int nx, double inv_h2,
                       double* dia, double* off, void* stream) {
  if (M < 0 || d < 1 || nx < 1) return set_error(KLE_ERR_INVALID, "kl_tridiag: bad dims");
  return kl_tridiag(xi, M, d, kl_table, nx, inv_h2, dia, off, KLE_STREAM(stream));
}

int kle_fine_factor_f64(const double* dia, const double* off, int M, int nx, double h, double g0,
                        double* blob, void* stream) {
  if (M < 0 || nx < 1 || !(h > 0)) return set_error(KLE_ERR_INVALID, "fine_factor: bad arguments");
  if (M == 0) return KLE_OK;
  const FineLayoutRT l = fine_layout(nx);
  if (l.MR == 0) return set_error(KLE_ERR_UNSUPPORTED, "fine_factor: nx too large");
  return fine_factor(l, dia, off, blob, M, nx, h, g0, KLE_STREAM(stream));
}

int kle_sweep_f64(const double* start, double* out, const double* blob, int M, int Q, int nx, int J,
                  int nseg, double h, double g0, void* stream) {
  if (M < 0 || Q < 0 || nx < 1 || J < 1 || nseg < 1) return set_error(KLE_ERR_INVALID, "sweep: bad dims");
  if (M == 0 || Q == 0) return KLE_OK;
  const FineLayoutRT l = fine_layout(nx);
  if (l.MR == 0) return set_error(KLE_ERR_UNSUPPORTED, "sweep: nx too large");
  SweepArgs a{start, out, blob, M, Q, nx, J, nseg, h, g0};
  return fine_sweep(l, a, KLE_STREAM(stream));
}

int kle_fgr_f64(const double* U, const double* u0, const double* F_given, double* F_out, double* R,
                const double* fine_blob, const double* dia, const double* off, const double* scaling,
                const int32_t* status, int M, int N, int nx, int J, double dt, double dT, double g0,
                double alpha, void* stream) {
  if (M < 0 || N < 1 || nx < 1 || J < 1) return set_error(KLE_ERR_INVALID, "fgr: bad dims");
  if (M == 0) return KLE_OK;
  const FineLayoutRT l = fine_layout(nx);
  if (l.MR == 0) return set_error(KLE_ERR_UNSUPPORTED, "fgr: nx too large");
  if (!R && (F_given || !F_out || l.W || l.kind))
    return set_error(KLE_ERR_UNSUPPORTED, "fgr: F ends only (R = NULL) needs F_out and a register layout");
  FgrArgs a{U, u0, F_given, F_out, R, fine_blob, dia, off, scaling, status, M, N, nx, J, dt, dT, g0, alpha};
  return fine_fgr(l, a, KLE_STREAM(stream));
}

size_t kle_cgc_scratch_bytes(int M, int N, int nx) {
  if (M <= 0 || N <= 0 || nx <= 0) return 0;
  const size_t slab = (size_t)cgc_grid(M, N, nx) * cgc_scratch_doubles_per_cta(N, nx) * sizeof(double);
  const size_t slots = (size_t)M * 2 * sizeof(unsigned long long);
  size_t b = slab > slots ? slab : slots;
  if (cgc_large_supported(N, nx)) {
    const size_t l = cgc_large_scratch_bytes(M, N, nx);
    if (l > b) b = l;
  }
  return b;
}

size_t kle_shift_factor_bytes(int M, int N, int nx) {
  if (M <= 0 || N <= 0 || nx <= 0 || !cgc_cluster_supported(N, nx)) return 0;
  return shift_factor_doubles(M, N, nx) * sizeof(double);
}

int kle_shift_factor_f64(const double* dia, const double* off, const double* lam, int M, int N, int nx, double dT,
                         double* sfac, void* stream) {
  if (M < 0 || N < 1 || nx < 1) return set_error(KLE_ERR_INVALID, "shift_factor: bad dims");
  if (!cgc_cluster_supported(N, nx)) return set_error(KLE_ERR_UNSUPPORTED, "shift_factor: shape uses the on-the-fly path");
  return shift_factor(dia, off, lam, M, N, nx, dT, sfac, KLE_STREAM(stream));
}

int kle_three_step_f64(const double* r, const double* scaling, const double* inv_scaling, const double* lam,
                       const double* dia, const double* off, const double* sfac, int M, int N, int nx, double dT,
                       double* u, double* imag, void* scratch, size_t scratch_bytes, void* stream) {
  if (M < 0 || N < 1 || nx < 1) return set_error(KLE_ERR_INVALID, "three_step: bad dims");
  if (M == 0) return KLE_OK;
  if (scratch_bytes < (sfac ? (size_t)M * 16 : kle_cgc_scratch_bytes(M, N, nx)))
    return set_error(KLE_ERR_WORKSPACE, "three_step: scratch too small");
  if (imag) cudaMemsetAsync(imag, 0, sizeof(double) * M, KLE_STREAM(stream));
  CgcArgs a{};
  a.R = r;
  a.load_scale = scaling;
  a.U = nullptr;
  a.Uout = u;
  a.dia = dia;
  a.off = off;
  a.lam = lam;
  a.inv_scaling = inv_scaling;
  a.scratch = static_cast<double*>(scratch);
  a.scratch_doubles_per_cta = cgc_scratch_doubles_per_cta(N, nx);
  a.imag = nullptr;  // zeroed above: u is real by Hermitian completion (diagnostic: kle_imag_residue_f64)
  a.M = M;
  a.N = N;
  a.nx = nx;
  a.k = 1;
  a.max_iters = 1;
  a.dT = dT;
  a.tol = 0.0;
  if (sfac) {
    a.red_slots = static_cast<unsigned long long*>(scratch);
    cudaMemsetAsync(scratch, 0, (size_t)M * 16, KLE_STREAM(stream));
    return cgc_cluster_run(a, sfac, KLE_STREAM(stream));
  }
  return cgc_run(a, KLE_STREAM(stream));
}

int kle_cgc_update_f64(const double* R, double* U, const double* inv_scaling, const double* lam,
                       const double* dia, const double* off, const double* sfac, int M, int N, int nx, double dT,
                       int k, int max_iters, double tol, int32_t* status, int32_t* iters, double* inc_hist,
                       double* imag, int32_t* active_count, void* scratch, size_t scratch_bytes,
                       void* stream) {
  if (M < 0 || N < 1 || nx < 1 || k < 1 || max_iters < k) return set_error(KLE_ERR_INVALID, "cgc_update: bad arguments");
  if (M == 0) return KLE_OK;
  if (scratch_bytes < (sfac ? (size_t)M * 16 : kle_cgc_scratch_bytes(M, N, nx)))
    return set_error(KLE_ERR_WORKSPACE, "cgc_update: scratch too small");
  CgcArgs a{};
  a.R = R;
  a.U = U;
  a.dia = dia;
  a.off = off;
  a.lam = lam;
  a.inv_scaling = inv_scaling;
  a.scratch = static_cast<double*>(scratch);
  a.scratch_doubles_per_cta = cgc_scratch_doubles_per_cta(N, nx);
  a.status = status;
  a.iters = iters;
  a.inc_hist = inc_hist;
  a.imag = imag;
  a.active_count = active_count;
  a.M = M;
  a.N = N;
  a.nx = nx;
  a.k = k;
  a.max_iters = max_iters;
  a.dT = dT;
  a.tol = tol;
  if (sfac && !imag && cgc_small_supported(N, nx)) {  // N <= 16, nx <= 128: one CTA per sample (kle_iter_small.cu)
    IterSmallArgs ia{U, R, nullptr, nullptr, dia, off, sfac, nullptr, inv_scaling, status, iters, inc_hist,
                     active_count, M, N, nx, 1, k, max_iters, 0.0, dT, 0.0, 0.0, tol};
    return cgc_small_run(ia, KLE_STREAM(stream));
  }
  if (sfac) {
    // the slots return to zero after every launch (last CTA resets the max; the
    // ticket counts modulo the cluster size), so callers zero them once
    a.red_slots = static_cast<unsigned long long*>(scratch);
    return cgc_cluster_run(a, sfac, KLE_STREAM(stream));
  }
  return cgc_run(a, KLE_STREAM(stream));
}

size_t kle_imag_residue_scratch_bytes(int M, int N, int nx) { return imag_residue_scratch_bytes(M, N, nx); }

int kle_imag_residue_f64(const double* R, const double* load_scale, const double* inv_scaling, const double* lam,
                         const double* dia, const double* off, const int32_t* status, int M, int N, int nx,
                         double dT, double* imag, void* scratch, size_t scratch_bytes, void* stream) {
  if (M < 0 || N < 1 || nx < 1 || !imag) return set_error(KLE_ERR_INVALID, "imag_residue: bad arguments");
  if (M == 0) return KLE_OK;
  if (scratch_bytes < imag_residue_scratch_bytes(M, N, nx))
    return set_error(KLE_ERR_WORKSPACE, "imag_residue: scratch too small");
  CgcArgs a{};
  a.R = R;
  a.load_scale = load_scale;
  a.dia = dia;
  a.off = off;
  a.lam = lam;
  a.inv_scaling = inv_scaling;
  a.scratch = static_cast<double*>(scratch);
  a.status = const_cast<int32_t*>(status);
  a.imag = imag;
  a.M = M;
  a.N = N;
  a.nx = nx;
  a.k = 1;
  a.max_iters = 1;
  a.dT = dT;
  return imag_residue_run(a, KLE_STREAM(stream));
}

static size_t pcgc_scratch_part(int M, int N, int nx) {
  return cgc_cluster_supported(N, nx) ? align256(kle_shift_factor_bytes(M, N, nx)) + align256((size_t)M * 16)
                                      : kle_cgc_scratch_bytes(M, N, nx);
}

size_t kle_pcgc_workspace_bytes(int M, int N, int nx) {
  if (M <= 0 || N <= 0 || nx <= 0) return 0;
  return align256((size_t)M * N * nx * sizeof(double)) + align256(pcgc_scratch_part(M, N, nx)) + 256 +
         align256(imag_residue_scratch_bytes(M, N, nx));
}


int kle_release_resources(void) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return set_error(KLE_ERR_CUDA, "release: no device");
  if (AuxResources* r = g_aux[dev]) {
    if (cudaDeviceSynchronize() != cudaSuccess) return set_error(KLE_ERR_CUDA, "release: device synchronize failed");
    g_aux[dev] = nullptr;
    aux_destroy(r);
  }
  return KLE_OK;
}

static int pcgc_loop(double* U, const double* u0, const double* dia, const double* off, const double* fine_blob,
                     const double* scaling, const double* inv_scaling, const double* lam, int M, int N, int nx, int J,
                     double T, double alpha, double g0, double tol, int max_iters, int32_t* status, int32_t* iters,
                     double* inc_hist, double* imag, const double* ref, int stop_ref, double* err_hist,
                     double* max_err, void* workspace, size_t workspace_bytes, void* stream) {
  if (M < 0 || N < 1 || nx < 1 || J < 1 || max_iters < 1 || !(T > 0) || !(alpha > 0 && alpha < 1))
    return set_error(KLE_ERR_INVALID, "pcgc_solve: bad arguments");
  if (M == 0) return KLE_OK;
  if (workspace_bytes < kle_pcgc_workspace_bytes(M, N, nx))
    return set_error(KLE_ERR_WORKSPACE, "pcgc_solve: workspace too small");
  cudaStream_t st = KLE_STREAM(stream);
  char* ws = static_cast<char*>(workspace);
  double* R = reinterpret_cast<double*>(ws);
  ws += align256((size_t)M * N * nx * sizeof(double));
  const bool clustered = cgc_cluster_supported(N, nx);
  const size_t scratch_bytes = pcgc_scratch_part(M, N, nx);
  void* scratch = ws;
  ws += align256(scratch_bytes);
  int32_t* counter = reinterpret_cast<int32_t*>(ws);
  ws += 256;
  void* imag_scratch = ws;  // the max_imag_residue diagnostic (only when imag is requested)
  const size_t imag_scratch_bytes = imag_residue_scratch_bytes(M, N, nx);
  double* sfac = clustered ? static_cast<double*>(scratch) : nullptr;
  void* cgc_scratch = clustered ? static_cast<void*>(static_cast<char*>(scratch) + align256(kle_shift_factor_bytes(M, N, nx)))
                                : scratch;
  const size_t cgc_scratch_bytes = clustered ? (size_t)M * 16 : scratch_bytes;

  const double dT = T / N, dt = dT / J;
  if (clustered) {
    KLE_TRY(shift_factor(dia, off, lam, M, N, nx, dT, sfac, st));
    cudaMemsetAsync(cgc_scratch, 0, (size_t)M * 16, st);
  }
  cudaMemsetAsync(status, 0, sizeof(int32_t) * M, st);
  cudaMemsetAsync(iters, 0, sizeof(int32_t) * M, st);
  if (inc_hist) cudaMemsetAsync(inc_hist, 0xFF, sizeof(double) * (size_t)M * max_iters, st);
  if (imag) cudaMemsetAsync(imag, 0, sizeof(double) * M, st);
  if (err_hist) cudaMemsetAsync(err_hist, 0xFF, sizeof(double) * (size_t)M * (max_iters + 1) * N, st);
  KLE_TRY(check_launch("pcgc_solve: init"));
  if (ref)  // record k = 0 (the initial guess) and, for stop_on="reference", its stop test
    KLE_TRY(err_ref(U, ref, M, N, nx, 0, max_iters, tol, stop_ref, status, iters, nullptr, err_hist, max_err, st));
  // with stop_on="reference" the increment never stops a sample (tol < 0); err_ref_kernel does
  const double cgc_tol = (ref && stop_ref) ? -1.0 : tol;
  // Sample pipelines: the batch is split into `pipes` contiguous halves, each
  // running its own outer loop on its own stream, started half an iteration
  // apart, so the FP64-bound fine sweeps of one half share the SMs with the
  // latency-bound CGC of the other. Results do not depend on the split (every
  // sample's arithmetic is the same; only the launch grouping changes).
  int pipes = (M >= 8192 && clustered) ? 2 : 1;
  // small blocks (configs 1 / 4): the twisted fine sweep and the row-FFT CGC each fill the GPU, nothing
  // overlaps, and one pipeline measures 449.5 against 460.6 ms per 1M-sample solve
  if (cgc_row_supported(N, nx) && tw_supported(fine_layout(nx), nx)) pipes = 1;
  if (const char* e = getenv("KLE_PCGC_PIPES")) {
    pipes = clustered ? atoi(e) : 1;
    pipes = pipes < 1 ? 1 : (pipes > kMaxPipes ? kMaxPipes : pipes);
    if (pipes > M) pipes = M > 0 ? M : 1;
  }
  if (imag) pipes = 1;  // the diagnostic's scratch serves one pipeline
  // small blocks (configs 1 / 4): fused iteration kernel, unless the imag
  // diagnostic (which reads the CGC right-hand side R from global) is on
  const bool fused = clustered && !imag && iter_small_supported(N, nx);
  const FineLayoutRT lay = fine_layout(nx);
  struct Pipe {
    int m0, M, k;
    bool live;
    cudaStream_t st, sc;  // fine sweeps (low priority), CGC (high priority)
    cudaEvent_t done, fdone;
    int32_t* count_d;
  };
  Pipe pp[kMaxPipes];
  // streams, events and the pinned counters are created once per host thread
  // and device and reused: driver resource calls inside a solve serialise with
  // other driver clients (e.g. an nvidia-smi poll) and cost more than a short
  // solve
  AuxResources* res = aux_resources();
  if (!res) return KLE_ERR_CUDA;
  int32_t* h_count = res->h_count;
  // twisted / scaled fine sweeps (kle_fine_tw.cu, be_steps_sc): count the samples the table kernel flagged as having no scaled
  // form, so that the partitioned kernel is launched after each sweep only when there are any (one
  // stream synchronisation per solve instead of an empty 1M-CTA launch per sweep)
  int tw_none_flagged = 0;
  const bool pw = pw_supported(lay, nx), sc = !pw && sc_supported(lay);
  if (!fused && (pw || sc || tw_supported(lay, nx))) {
    cudaMemsetAsync(counter + 8, 0, sizeof(int32_t), st);
    const int foff = pw ? pw_flag_offset() : (sc ? sc_flag_offset(lay) : 0);
    KLE_TRY(tw_count_flagged(fine_blob, M, (pw || sc) ? lay.doubles : 0, foff, counter + 8, st));
    cudaMemcpyAsync(&h_count[kMaxPipes], counter + 8, sizeof(int32_t), cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return set_error(KLE_ERR_CUDA, "pcgc_solve: flag count");
    tw_none_flagged = h_count[kMaxPipes] == 0;
  }
  cudaEvent_t ready = res->ready;
  cudaEventRecord(ready, st);
  for (int p = 0; p < pipes; ++p) {
    pp[p].m0 = (int)((long long)M * p / pipes);
    pp[p].M = (int)((long long)M * (p + 1) / pipes) - pp[p].m0;
    pp[p].k = 0;
    pp[p].live = pp[p].M > 0;
    pp[p].count_d = counter + p;
    h_count[p] = pp[p].M;
    if (pipes == 1) {
      pp[p].st = pp[p].sc = st;
    } else {
      pp[p].st = res->sf[p];
      pp[p].sc = res->sc[p];
      cudaStreamWaitEvent(pp[p].st, ready, 0);
    }
    pp[p].done = res->done[p];
    pp[p].fdone = res->fdone[p];
  }
  auto enqueue = [&](Pipe& q) -> int {
    const int k = ++q.k;
    const size_t o = (size_t)q.m0;
    double* Uq = U + o * N * nx;
    const double* dq = dia + o * nx;
    const double* eq = off + o * nx;
    int32_t* sq = status + o;
    if (fused) {  // the whole iteration in one kernel (kle_iter_small.cu)
      cudaMemsetAsync(q.count_d, 0, sizeof(int32_t), q.st);
      IterSmallArgs ia{Uq, nullptr, u0, fine_blob + o * lay.doubles, dq, eq, sfac + o * shift_factor_doubles(1, N, nx), scaling,
                       inv_scaling, sq, iters + o, inc_hist ? inc_hist + o * max_iters : nullptr, q.count_d,
                       q.M, N, nx, J, k, max_iters, dt, dT, g0, alpha, cgc_tol};
      KLE_TRY(iter_small_run(ia, q.st));
      if (q.sc != q.st) {  // the pipeline's bookkeeping (count read-back, reference errors) runs on sc
        cudaEventRecord(q.fdone, q.st);
        cudaStreamWaitEvent(q.sc, q.fdone, 0);
      }
    } else {
    {
      FgrArgs fa{Uq, u0, nullptr, nullptr, R + o * N * nx, fine_blob + o * lay.doubles, dq, eq, scaling, sq,
                 q.M, N, nx, J, dt, dT, g0, alpha};
      fa.tw_none_flagged = tw_none_flagged;
      KLE_TRY(fine_fgr(lay, fa, q.st));
    }
    if (q.sc != q.st) {
      cudaEventRecord(q.fdone, q.st);
      cudaStreamWaitEvent(q.sc, q.fdone, 0);
    }
    cudaMemsetAsync(q.count_d, 0, sizeof(int32_t), q.sc);
    if (imag)  // max_imag_residue (pintuq/pcgc.py:170-172, 340-342) of this iteration's three-step solve
      KLE_TRY(kle_imag_residue_f64(R + o * N * nx, nullptr, inv_scaling, lam, dq, eq, sq, q.M, N, nx, dT, imag + o,
                                   imag_scratch, imag_scratch_bytes, q.sc));
    const double* sf = clustered ? sfac + o * (shift_factor_doubles(1, N, nx)) : nullptr;
    void* cs = clustered ? static_cast<void*>(static_cast<char*>(cgc_scratch) + o * 16) : cgc_scratch;
    KLE_TRY(kle_cgc_update_f64(R + o * N * nx, Uq, inv_scaling, lam, dq, eq, sf, q.M, N, nx, dT, k, max_iters,
                               cgc_tol, sq, iters + o, inc_hist ? inc_hist + o * max_iters : nullptr,
                               nullptr, q.count_d, cs,
                               clustered ? (size_t)q.M * 16 : cgc_scratch_bytes, q.sc));
    }
    if (ref)
      KLE_TRY(err_ref(Uq, ref + o * N * nx, q.M, N, nx, k, max_iters, tol, stop_ref, sq, iters + o, q.count_d,
                      err_hist ? err_hist + o * (size_t)(max_iters + 1) * N : nullptr, max_err ? max_err + o : nullptr,
                      q.sc));
    cudaMemcpyAsync(&h_count[&q - pp], q.count_d, sizeof(int32_t), cudaMemcpyDeviceToHost, q.sc);
    cudaEventRecord(q.done, q.sc);
    if (q.sc != q.st) cudaStreamWaitEvent(q.st, q.done, 0);
    return KLE_OK;
  };
  int rc = KLE_OK;
  for (int p = 0; p < pipes && rc == KLE_OK; ++p) {
    if (!pp[p].live) continue;
    rc = enqueue(pp[p]);
    if (p + 1 < pipes)  // each part starts after the previous part's first fine sweep
      cudaStreamWaitEvent(pp[p + 1].st, pp[p].fdone, 0);
  }
  for (bool any = true; any && rc == KLE_OK;) {
    any = false;
    for (int p = 0; p < pipes && rc == KLE_OK; ++p) {
      Pipe& q = pp[p];
      if (!q.live) continue;
      const cudaError_t e = cudaEventSynchronize(q.done);
      if (e != cudaSuccess) {
        rc = set_error(KLE_ERR_CUDA, cudaGetErrorString(e));
        break;
      }
      if (h_count[p] == 0 || q.k >= max_iters) {
        q.live = false;
        continue;
      }
      any = true;
      rc = enqueue(q);
    }
  }
  if (pipes > 1) {  // join: later work on `st` sees every part
    for (int p = 0; p < pipes; ++p) {
      cudaEventRecord(pp[p].done, pp[p].sc);
      cudaStreamWaitEvent(st, pp[p].done, 0);
    }
  }
  cudaStreamSynchronize(st);
  return rc;
}

int kle_pcgc_solve_f64(double* U, const double* u0, const double* dia, const double* off,
                       const double* fine_blob, const double* scaling, const double* inv_scaling,
                       const double* lam, int M, int N, int nx, int J, double T, double alpha, double g0,
                       double tol, int max_iters, int32_t* status, int32_t* iters, double* inc_hist,
                       double* imag, void* workspace, size_t workspace_bytes, void* stream) {
  return pcgc_loop(U, u0, dia, off, fine_blob, scaling, inv_scaling, lam, M, N, nx, J, T, alpha, g0, tol, max_iters,
                   status, iters, inc_hist, imag, nullptr, 0, nullptr, nullptr, workspace, workspace_bytes, stream);
}

int kle_pcgc_solve_ref_f64(double* U, const double* u0, const double* dia, const double* off,
                           const double* fine_blob, const double* scaling, const double* inv_scaling,
                           const double* lam, int M, int N, int nx, int J, double T, double alpha, double g0,
                           double tol, int max_iters, const double* ref, int stop_on_reference, int32_t* status,
                           int32_t* iters, double* inc_hist, double* err_hist, double* max_err, double* imag,
                           void* workspace, size_t workspace_bytes, void* stream) {
  if (!ref) return set_error(KLE_ERR_INVALID, "pcgc_solve_ref: reference trajectory required");
  return pcgc_loop(U, u0, dia, off, fine_blob, scaling, inv_scaling, lam, M, N, nx, J, T, alpha, g0, tol, max_iters,
                   status, iters, inc_hist, imag, ref, stop_on_reference, err_hist, max_err, workspace,
                   workspace_bytes, stream);
}

int kle_err_ref_f64(const double* U, const double* ref, int M, int N, int nx, int k, int max_iters, double tol,
                    int stop_on_reference, int32_t* status, int32_t* iters, int32_t* active_count, double* err_hist,
                    double* max_err, void* stream) {
  if (M < 0 || N < 1 || nx < 1 || k < 0 || max_iters < k) return set_error(KLE_ERR_INVALID, "err_ref: bad arguments");
  if (!status || !iters) return set_error(KLE_ERR_INVALID, "err_ref: status and iters are required");
  return err_ref(U, ref, M, N, nx, k, max_iters, tol, stop_on_reference, status, iters, active_count, err_hist,
                 max_err, KLE_STREAM(stream));
}

int kle_err_aggregate_f64(const double* err_hist, const int32_t* iters, int M, int N, int max_iters, int k_pad,
                          int32_t* good, int32_t* counts, double* sums, void* stream) {
  if (M < 0 || N < 1 || max_iters < 0 || k_pad > max_iters || !err_hist || !iters || !good || !counts || !sums)
    return set_error(KLE_ERR_INVALID, "err_aggregate: bad arguments");
  return err_aggregate(err_hist, iters, M, N, max_iters, k_pad, good, counts, sums, KLE_STREAM(stream));
}

// ---- classical parareal (pintuq/parareal.py:100-191) ------------------------
int kle_parareal_init_f64(const double* U, const double* u0, const double* coarse_blob, int M, int N, int nx,
                          double dT, double g0, double* Gprev, void* stream) {
  if (M < 0 || N < 1 || nx < 1 || !(dT > 0)) return set_error(KLE_ERR_INVALID, "parareal_init: bad arguments");
  PararealArgs a{};
  a.U = const_cast<double*>(U);
  a.u0 = u0;
  a.Gprev = Gprev;
  a.gfac = coarse_blob;
  a.M = M;
  a.N = N;
  a.nx = nx;
  a.mode = 0;
  a.dT = dT;
  a.g0 = g0;
  return parareal_run(fine_layout(nx), a, KLE_STREAM(stream));
}

int kle_parareal_step_f64(double* U, const double* u0, const double* F, double* Gprev, const double* coarse_blob,
                          int M, int N, int nx, double dT, double g0, int k, int max_iters, double tol,
                          int32_t* status, int32_t* iters, double* inc_hist, int32_t* active_count, void* stream) {
  if (M < 0 || N < 1 || nx < 1 || k < 1 || max_iters < k || !(dT > 0))
    return set_error(KLE_ERR_INVALID, "parareal_step: bad arguments");
  PararealArgs a{U, u0, F, Gprev, coarse_blob, status, iters, inc_hist, active_count, M, N, nx, k, max_iters, 1,
                 dT, g0, tol};
  return parareal_run(fine_layout(nx), a, KLE_STREAM(stream));
}

size_t kle_parareal_workspace_bytes(int M, int N, int nx) {
  if (M <= 0 || N <= 0 || nx <= 0) return 0;
  return 2 * align256((size_t)M * N * nx * sizeof(double)) + 256;
}

int kle_parareal_solve_f64(double* U, const double* u0, const double* dia, const double* off,
                           const double* fine_blob, const double* coarse_blob, int M, int N, int nx, int J, double T,
                           double g0, double tol, int max_iters, const double* ref, int stop_on_reference,
                           int32_t* status, int32_t* iters, double* inc_hist, double* err_hist, double* max_err,
                           void* workspace, size_t workspace_bytes, void* stream) {
  if (M < 0 || N < 1 || nx < 1 || J < 1 || max_iters < 1 || !(T > 0))
    return set_error(KLE_ERR_INVALID, "parareal_solve: bad arguments");
  if (M == 0) return KLE_OK;
  if (workspace_bytes < kle_parareal_workspace_bytes(M, N, nx))
    return set_error(KLE_ERR_WORKSPACE, "parareal_solve: workspace too small");
  const FineLayoutRT lay = fine_layout(nx);
  if (lay.W != 0 || lay.kind != 0) return set_error(KLE_ERR_UNSUPPORTED, "parareal_solve: nx > 1024");
  cudaStream_t st = KLE_STREAM(stream);
  char* ws = static_cast<char*>(workspace);
  double* F = reinterpret_cast<double*>(ws);
  ws += align256((size_t)M * N * nx * sizeof(double));
  double* G = reinterpret_cast<double*>(ws);
  ws += align256((size_t)M * N * nx * sizeof(double));
  int32_t* counter = reinterpret_cast<int32_t*>(ws);
  const double dT = T / N, dt = dT / J;
  cudaMemsetAsync(status, 0, sizeof(int32_t) * M, st);
  cudaMemsetAsync(iters, 0, sizeof(int32_t) * M, st);
  if (inc_hist) cudaMemsetAsync(inc_hist, 0xFF, sizeof(double) * (size_t)M * max_iters, st);
  if (err_hist) cudaMemsetAsync(err_hist, 0xFF, sizeof(double) * (size_t)M * (max_iters + 1) * N, st);
  KLE_TRY(check_launch("parareal_solve: init"));
  if (ref) KLE_TRY(err_ref(U, ref, M, N, nx, 0, max_iters, tol, stop_on_reference, status, iters, nullptr, err_hist,
                           max_err, st));
  const double step_tol = (ref && stop_on_reference) ? -1.0 : tol;
  KLE_TRY(kle_parareal_init_f64(U, u0, coarse_blob, M, N, nx, dT, g0, G, stream));
  int32_t h_count = M;
  for (int k = 1; k <= max_iters && h_count > 0; ++k) {
    FgrArgs fa{U, u0, nullptr, F, nullptr, fine_blob, dia, off, nullptr, status, M, N, nx, J, dt, dT, g0, 0.0};
    KLE_TRY(fine_fgr(lay, fa, st));
    cudaMemsetAsync(counter, 0, sizeof(int32_t), st);
    KLE_TRY(kle_parareal_step_f64(U, u0, F, G, coarse_blob, M, N, nx, dT, g0, k, max_iters, step_tol, status, iters,
                                  inc_hist, counter, stream));
    if (ref) KLE_TRY(err_ref(U, ref, M, N, nx, k, max_iters, tol, stop_on_reference, status, iters, counter,
                             err_hist, max_err, st));
    cudaMemcpyAsync(&h_count, counter, sizeof(int32_t), cudaMemcpyDeviceToHost, st);
    const cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return set_error(KLE_ERR_CUDA, cudaGetErrorString(e));
  }
  return KLE_OK;
}

// ---- nonlinear models: fused Newton backward-Euler sweeps (pintuq/_kernels.pyx) ----
size_t kle_newton_work_bytes(int M, int Q, int nx) {
  if (M <= 0 || Q <= 0 || nx <= 0) return 0;
  return newton_work_doubles(M, Q, nx) * sizeof(double);
}

int kle_newton_sweep_f64(int kind, const double* start, double* out, const double* p0, int M, int Q, int nx, int J,
                         int nseg, double h, double dx, double bc_lo, double bc_hi, double newton_tol, int max_newton,
                         const int32_t* active, int32_t* status, void* work, size_t work_bytes, void* stream) {
  if (kind < 0 || kind > 1 || M < 0 || Q < 0 || nx < 1 || J < 1 || nseg < 1 || max_newton < 0 || !(h > 0) ||
      !(dx > 0))
    return set_error(KLE_ERR_INVALID, "newton_sweep: bad arguments");
  if (M == 0 || Q == 0) return KLE_OK;
  if (work_bytes < kle_newton_work_bytes(M, Q, nx)) return set_error(KLE_ERR_WORKSPACE, "newton_sweep: work too small");
  NewtonArgs a{start, out, p0, active, status, M, Q, nx, J, nseg, kind, max_newton, h, dx, bc_lo, bc_hi, newton_tol};
  return newton_sweep(a, static_cast<double*>(work), KLE_STREAM(stream));
}

int kle_para_combine_f64(double* U, const double* Gn, const double* F, double* Gprev, const int32_t* status, int M,
                         int N, int nx, int n, void* stream) {
  if (M < 0 || N < 1 || nx < 1 || n < 0 || n >= N) return set_error(KLE_ERR_INVALID, "para_combine: bad arguments");
  return para_combine(U, Gn, F, Gprev, status, M, N, nx, n, KLE_STREAM(stream));
}

int kle_newton_cgc_f64(int kind, const double* U, const double* b, double* Uout, const double* p0, const double* lam,
                       const double* scaling, const double* inv_scaling, int M, int N, int nx, double dT, double dx,
                       double bc_lo, double bc_hi, double newton_tol, int32_t* status, int32_t* inner, void* stream) {
  if (kind < 0 || kind > 1 || M < 0 || N < 1 || nx < 1 || !(dT > 0) || !(dx > 0))
    return set_error(KLE_ERR_INVALID, "newton_cgc: bad arguments");
  NewtonCgcArgs a{U, b, Uout, p0, lam, scaling, inv_scaling, status, inner, M, N, nx, kind, dT, dx, bc_lo, bc_hi,
                  newton_tol};
  return newton_cgc(a, KLE_STREAM(stream));
}

int kle_block_dft_f64(const double* in, double* out, int N, int L, int sign, void* stream) {
  if (N < 1 || L < 0 || (sign != 1 && sign != -1)) return set_error(KLE_ERR_INVALID, "block_dft: bad arguments");
  return block_dft(in, out, N, L, sign, KLE_STREAM(stream));
}

int kle_shifted_tridiag_solve_f64(const double* sub, const double* dia, const double* sup, double lam_re,
                                  double lam_im, double dT, const double* p, double* q, double* cwork, int nx,
                                  int nrhs, int32_t* status, void* stream) {
  if (nx < 1 || nrhs < 0) return set_error(KLE_ERR_INVALID, "shifted_tridiag: bad arguments");
  return shifted_tridiag(sub, dia, sup, lam_re, lam_im, dT, p, q, cwork, nx, nrhs, status, KLE_STREAM(stream));
}

int kle_gpc_basis_f64(const double* xi, int M, int d, int degree, int family, const double* maps,
                      const int32_t* midx, int P, const double* norms, double* Psi, void* stream) {
  if (M < 0 || d < 1 || P < 1) return set_error(KLE_ERR_INVALID, "gpc_basis: bad dims");
  return gpc_basis(xi, M, d, degree, family, maps, midx, P, norms, Psi, KLE_STREAM(stream));
}

int kle_gpc_eval_f64(const double* Psi, int M, int K, const double* C, const double* mean, int L, double* U0,
                     void* stream) {
  if (M < 0 || K < 1 || L < 1) return set_error(KLE_ERR_INVALID, "gpc_eval: bad dims");
  return gemm_bias(Psi, C, mean, U0, M, K, L, KLE_STREAM(stream));
}

int kle_gemm_f64(const double* A, const double* B, const double* bias, double* C, int M, int K, int L, int trans_b,
                 void* stream) {
  if (M < 0 || K < 1 || L < 0) return set_error(KLE_ERR_INVALID, "gemm: bad dims");
  return gemm_bias(A, B, bias, C, M, K, L, KLE_STREAM(stream), trans_b != 0);
}

int kle_sub_row_f64(const double* X, const double* v, double* out, int M, int L, void* stream) {
  if (M < 0 || L < 0) return set_error(KLE_ERR_INVALID, "sub_row: bad dims");
  return sub_row(X, v, out, M, L, KLE_STREAM(stream));
}

size_t kle_col_sum_scratch_bytes(int M, int L) {
  if (L <= 0) return 0;
  return col_sum_partial_doubles(M, L) * sizeof(double);
}

int kle_col_sum_f64(const double* U, int M, int L, const double* center, double* out, void* scratch,
                    void* stream) {
  if (M < 0 || L < 0) return set_error(KLE_ERR_INVALID, "col_sum: bad dims");
  return col_sum(U, M, L, center, out, static_cast<double*>(scratch), KLE_STREAM(stream));
}

int kle_axpby_f64(const double* x, const double* y, double* out, double a, double b, size_t n, void* stream) {
  return axpby(x, y, out, a, b, n, KLE_STREAM(stream));
}

}  // extern "C"
