// Classical parareal (the paper's comparison baseline) for the linear
// tridiagonal models: the sequential-in-n predictor-corrector update
//
//   U_{n+1}^{k+1} = G(U_n^{k+1}) + F(U_n^k) - G(U_n^k),   U_0 = u0,
//
// of pintuq/parareal.py:100-191 (parareal_solve; coarse G = one backward-Euler
// step of dT, propagators.py:148-157). The fine ends F(U_n^k) come from the
// fused fine kernel (fgr_kernel with F_out, no CGC right-hand side); this file
// holds the sequential coarse correction, one P-lane group per sample, the
// coarse LDL^T factor of I + dT A in registers (the same partitioned solver
// as the fine sweep, J = 1).
//
//   mode 0 (init):    G_prev[n] = G(start_n), start = [u0, U_0 .. U_{N-2}]
//                     (parareal.py:153-155, the "old" coarse values)
//   mode 1 (correct): the sequential sweep above, increment max|U_new - U|
//                     (:181), stop test (:187-190) with per-sample freezing.
// HBM per (n, i) and iteration: read F, G_prev, U; write U, G_prev (40 B).
#include "kle_fine.cuh"
#include "kle_internal.h"

namespace kle {

template <int MR, int P>
__global__ void __launch_bounds__(128) parareal_kernel(PararealArgs a) {
  using L = FineLayout<MR, P>;
  constexpr int SLOTS = 32 / P;
  const int lane = threadIdx.x & 31, k = lane % P, slot = lane / P;
  const int s = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * SLOTS + slot;
  const bool live = s < a.M && (a.mode == 0 || !a.status || a.status[s] == KLE_SAMPLE_ACTIVE);
  // the whole warp takes part in the shuffles of the solver; dead slots run on zeros
  if (__all_sync(KLE_FULL_MASK, !live)) return;
  const int nx = a.nx, N = a.N;
  LaneFactors<MR, P> fac;
  const int sl = live ? s : 0;
  fac.load(a.gfac + (size_t)sl * L::DOUBLES, k, nx);
  const double hg = a.dT * a.g0;
  const size_t sb = (size_t)sl * N * nx;
  double prev[MR];  // current start row of the sweep (U_n^{k+1}; u0 for n = 0)
#pragma unroll
  for (int j = 0; j < MR; ++j) {
    const int row = k * MR + j;
    prev[j] = (live && row < nx) ? a.u0[row] : 0.0;
  }
  double incmax = 0.0;
  for (int n = 0; n < N; ++n) {
    double x[1][MR];
#pragma unroll
    for (int j = 0; j < MR; ++j) x[0][j] = (k * MR + j < nx) ? prev[j] + hg : 0.0;
    be_steps<MR, P, 1>(x, fac, k, 1, hg);
    const size_t o = sb + (size_t)n * nx;
#pragma unroll
    for (int j = 0; j < MR; ++j) {
      const int row = k * MR + j;
      const bool in = live && row < nx;
      const double g = x[0][j] - hg;
      if (a.mode == 0) {
        if (in) a.Gprev[o + row] = g;
        prev[j] = in ? a.U[o + row] : 0.0;  // start of subinterval n + 1 is U_n
      } else {
        double u = 0.0;
        if (in) {
          u = g + a.F[o + row] - a.Gprev[o + row];
          const double d = fabs(u - a.U[o + row]);
          incmax = nanmax(incmax, d);
          a.U[o + row] = u;
          a.Gprev[o + row] = g;
        }
        prev[j] = u;
      }
    }
  }
  if (a.mode == 0) return;
#pragma unroll
  for (int d = 1; d < P; d <<= 1) incmax = nanmax(incmax, __shfl_xor_sync(KLE_FULL_MASK, incmax, d, P));
  if (!live || k != 0) return;
  if (a.inc_hist) a.inc_hist[(size_t)s * a.max_iters + (a.k - 1)] = incmax;
  if (!a.status) return;
  int st = KLE_SAMPLE_ACTIVE;
  if (incmax <= a.tol) st = KLE_SAMPLE_CONVERGED;
  else if (!isfinite(incmax)) st = KLE_SAMPLE_NONFINITE;
  else if (a.k >= a.max_iters) st = KLE_SAMPLE_MAXITERS;
  if (st != KLE_SAMPLE_ACTIVE) {
    a.status[s] = st;
    if (a.iters) a.iters[s] = a.k;
  } else if (a.active_count) {
    atomicAdd(a.active_count, 1);
  }
}

template <int MR, int P>
static int launch_parareal(const PararealArgs& a, cudaStream_t st) {
  constexpr int SLOTS = 32 / P;
  const int warps = (a.M + SLOTS - 1) / SLOTS;
  const int blocks = (warps + 3) / 4;
  parareal_kernel<MR, P><<<blocks, 128, 0, st>>>(a);
  return check_launch("parareal_kernel");
}

int parareal_run(FineLayoutRT lay, const PararealArgs& a, cudaStream_t st) {
  if (a.M <= 0) return KLE_OK;
  if (lay.W != 0 || lay.kind != 0) return set_error(KLE_ERR_UNSUPPORTED, "parareal: nx needs a register layout (<= 1024)");
  if (lay.MR == 1 && lay.P == 16) return launch_parareal<1, 16>(a, st);
  if (lay.MR == 2 && lay.P == 16) return launch_parareal<2, 16>(a, st);
  if (lay.MR == 4 && lay.P == 16) return launch_parareal<4, 16>(a, st);
  if (lay.MR == 8 && lay.P == 16) return launch_parareal<8, 16>(a, st);
  if (lay.MR == 16 && lay.P == 8) return launch_parareal<16, 8>(a, st);
  if (lay.MR == 16 && lay.P == 32) return launch_parareal<16, 32>(a, st);
  if (lay.MR == 32 && lay.P == 32) return launch_parareal<32, 32>(a, st);
  return set_error(KLE_ERR_UNSUPPORTED, "parareal: fine layout");
}

}  // namespace kle
