// Eight-lane scaled fine sweep for 128 < nx <= 512 (config 2).
//
// Reference counterparts: propagate_fine (pintuq/propagators.py:121-145, J x splu.solve) and the
// right-hand side of cgc_correct (pintuq/pcgc.py:175-197, 233-237), as kle_fine.cu.
//
// The partitioned register kernel (kle_fine.cu: 32 lanes x 16 rows x 3 right-hand sides, factors in
// registers) spends its time in the two 5-round carry scans per step, which 16 rows of work per lane cannot
// hide (ncu: FP64 pipe 55%, the scans hold 27% of the stall samples). This kernel takes the twisted
// kernel's layout instead (kle_fine_tw.cu): each lane keeps H = 64 rows of ONE right-hand side in
// registers, so a system is 8 lanes, the scans shrink to 3 rounds and are amortised over four times the
// rows; the factor rows, shared by every subinterval of a sample, come from shared memory. The step is the
// scaled partitioned step of kle_fine.cuh (be_steps_sc): steady-state shift e = x - x*, chunk-local row
// scaling e = t w, so per row and step
//   yl_j = w_j + yl_{j-1}            (DADD; two independent chains per lane)
//   z_j  = (yl_j + C) inv_j          (DADD, DMUL; C = rho_k Y_{k-1} from the forward scan)
//   wl_j = z_j + kk_j wl_{j+1}       (DFMA)
//   w_j  = wl_j + sg_j X             (DFMA; X from the backward scan)
// with three coefficient doubles per row (inv, kk, sg) read as 16-byte broadcast loads.
//
// The tables are written by fine_factor_kernel<64, 8> behind the (16, 32) blob (FineLayout::PW_OFF), packed
// in this kernel's shared-memory order (kle_fine.cuh: kPw*): {1/beta, l^2}, sg, {x*, 1/t}, {t, dia}, off, the
// scan multipliers and the per-sample flag for samples without a scaled form, which this kernel skips and
// the partitioned kernel processes (FgrArgs::tw_fallback).
#include <algorithm>
#include <cstdlib>

#include "kle_common.cuh"
namespace kle {
#define FGR_T(i) \
  do {           \
  } while (0)
}
#include "kle_fine.cuh"
#include "kle_internal.h"

#ifndef KLE_FINE_LAZY
#define KLE_FINE_LAZY 0
#endif

namespace kle {

namespace {
constexpr int PW_H = 64, PW_P = 8;
using PwL = FineLayout<PW_H, PW_P>;
using PwOuter = FineLayout<16, 32>;
constexpr int PW_NC = 16;                  // subintervals per CTA (4 warps x 4 systems)
// staging pitch: chunk pitch 65 and 4 (mod 16) doubles per subinterval, so that the 16 lanes of a half-warp
// (4 chunks x 4 systems) hit 16 distinct banks
constexpr int PW_LD = PW_P * (PW_H + 1) + 12;
constexpr int PW_TAB = PW_H * PW_P;        // one [j][k] table
// shared memory (doubles): the tables, all read with 16-byte loads (a broadcast 8-byte load costs as many
// shared-memory wavefronts as a 16-byte one: 13.2 -> 8 ms per 8,192-sample c2 launch), then the staging rows:
//   T0 [j][k]   = {inv, kk}          T1 [j/2][k] = {sg_j, sg_{j+1}}      (step loop)
//   T2 [j][k]   = {x*, 1/t}          T3 [j][k]   = {t, dia}              T4 [j/2][k] = {off[row-1]} pairs
constexpr int PW_T0 = 0, PW_T1 = 2 * PW_TAB, PW_T2 = 3 * PW_TAB, PW_T3 = 5 * PW_TAB, PW_T4 = 7 * PW_TAB;
constexpr int PW_SMEM_DOUBLES = 8 * PW_TAB + (PW_NC + 1) * PW_LD;

__device__ __forceinline__ double2 lds_v2(unsigned addr) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr));
  return v;
}

__device__ __forceinline__ void cp_async8(unsigned sa, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void sts_f64(unsigned addr, double v) {
  asm volatile("st.shared.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
}
}  // namespace

__global__ void __launch_bounds__(128, 2) fgr_pw_kernel(FgrArgs a) {
  constexpr int H = PW_H, P = PW_P, LD = PW_LD, TAB = PW_TAB;
  const int s = blockIdx.x;
  if (a.active && a.active[s] != KLE_SAMPLE_ACTIVE) return;
  const double* bl = a.ffac + (size_t)s * PwOuter::DOUBLES + PwOuter::PW_OFF;  // the sample's (64, 8) blob
  if (bl[kPwFlag] != 0.0) return;  // no scaled form: the partitioned kernel takes it
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  // lane = 8 (k / 2) + 2 slot + (k & 1): a quarter-warp holds two chunks of all four systems, so that a 16-byte
  // coefficient load touches two distinct entries per quarter-warp (as in the twisted kernel, 2 shared-memory
  // wavefronts) instead of eight (4 wavefronts: ncu, 6.8 wavefronts per warp-row with lane = 8 slot + k)
  const int slot = (lane >> 1) & 3, k = ((lane >> 3) << 1) | (lane & 1);
  auto lane_of = [&](int kk_) { return ((kk_ >> 1) << 3) | (slot << 1) | (kk_ & 1); };
  int su[PwL::LOGP + 1], sd[PwL::LOGP + 1];  // source lanes of the scans: k - 2^t, k - 1; k + 2^t, k + 1
#pragma unroll
  for (int t = 0; t < PwL::LOGP; ++t) {
    su[t] = lane_of(max(k - (1 << t), 0));
    sd[t] = lane_of(min(k + (1 << t), PW_P - 1));
  }
  su[PwL::LOGP] = lane_of(max(k - 1, 0));
  sd[PwL::LOGP] = lane_of(min(k + 1, PW_P - 1));
  const int nx = a.nx, N = a.N;
  const size_t sbase = (size_t)s * N * nx;
  const int n0 = blockIdx.y * PW_NC;
  const int q = w * 4 + slot;  // subinterval slot of this lane's system
  const int n = n0 + q;
  const bool valid = n < N;
  const int nreal = min(H, max(0, nx - k * H));  // real rows of this lane's chunk

  extern __shared__ __align__(16) double sm[];
  double* st = sm + 8 * TAB;  // [17][LD] staging rows, chunk pitch 65; row 16: U_{N-1} (prev of n = 0)
  const unsigned st_s = (unsigned)__cvta_generic_to_shared(st);

  // start rows (coalesced 8-byte copies)
  for (int ln = 0; ln < PW_NC; ++ln) {
    const int nn = n0 + ln;
    if (nn >= N) break;
    const double* src = (nn == 0) ? a.u0 : a.U + sbase + (size_t)(nn - 1) * nx;
    for (int r = tid; r < nx; r += 128) cp_async8(st_s + (unsigned)((ln * LD + r + (r >> 6)) * sizeof(double)), src + r);
  }
  asm volatile("cp.async.commit_group;\n" ::);
  if (n0 == 0) {
    const double* src = a.U + sbase + (size_t)(N - 1) * nx;
    for (int r = tid; r < nx; r += 128) cp_async8(st_s + (unsigned)((PW_NC * LD + r + (r >> 6)) * sizeof(double)), src + r);
  }
  asm volatile("cp.async.commit_group;\n" ::);
  // the tables, packed by fine_factor_kernel<64, 8> in this kernel's shared-memory order (16-byte copies)
  {
    const unsigned tb0 = (unsigned)__cvta_generic_to_shared(sm);
#pragma unroll
    for (int i = 0; i < kPwTables / 2 / 128; ++i)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(tb0 + (unsigned)((tid + 128 * i) * 16)),
                   "l"(bl + (tid + 128 * i) * 2));
  }
  asm volatile("cp.async.commit_group;\n" ::);
  double af[PwL::LOGP], bb[PwL::LOGP];
#pragma unroll
  for (int t = 0; t < PwL::LOGP; ++t) {
    af[t] = bl[kPwAf + t * P + k];
    bb[t] = bl[kPwBb + t * P + k];
  }
  const double rho = bl[kPwRho + k];
  asm volatile("cp.async.wait_group 0;\n" ::);
  __syncthreads();

  // w = (x - x*) / t
  double x[H];
  const unsigned xs_ = st_s + (unsigned)((q * LD + k * (H + 1)) * sizeof(double));
  const unsigned tb = (unsigned)__cvta_generic_to_shared(sm) + (unsigned)(k * 16);
  constexpr unsigned RS = P * 16;  // bytes between consecutive table rows
#pragma unroll
  for (int j = 0; j < H; ++j) {
    const double v = lds_f64(xs_ + (unsigned)(j * sizeof(double)));
    const double2 c = lds_v2(tb + PW_T2 * 8 + j * RS);  // {x*, 1/t}
    x[j] = (valid && j < nreal) ? (v - c.x) * c.y : 0.0;
  }

#pragma unroll 1
  for (int step = 0; step < a.J; ++step) {
    // forward prefix sums, two independent chains
    double y0 = x[0], y1 = x[H / 2];
#pragma unroll
    for (int j = 1; j < H / 2; ++j) {
      y0 += x[j];
      x[j] = y0;
      y1 += x[H / 2 + j];
      x[H / 2 + j] = y1;
    }
    double Y = y0 + y1;
#pragma unroll
    for (int t = 0; t < PwL::LOGP; ++t) {
      const double o = __shfl_sync(KLE_FULL_MASK, Y, su[t]);
      Y = fma(af[t], o, Y);  // af = 0 for k < 2^t
    }
    const double C0 = rho * __shfl_sync(KLE_FULL_MASK, Y, su[PwL::LOGP]);  // rho_0 = 0
    const double C1 = C0 + y0;  // the second chain's rows also carry the first chain's total
    // scale + local backward
    double xn = 0.0;
#pragma unroll
    for (int j = H - 1; j >= 0; --j) {
      const double2 c = lds_v2(tb + PW_T0 * 8 + j * RS);  // {inv, kk}
      double z = (x[j] + (j >= H / 2 ? C1 : C0)) * c.x;
      if (j + 1 < H) z = fma(c.y, xn, z);
      x[j] = z;
      xn = z;
    }
    double X = xn;
#pragma unroll
    for (int t = 0; t < PwL::LOGP; ++t) {
      const double o = __shfl_sync(KLE_FULL_MASK, X, sd[t]);
      X = fma(bb[t], o, X);  // bb = 0 for k + 2^t >= P
    }
    X = __shfl_sync(KLE_FULL_MASK, X, sd[PwL::LOGP]);  // (sg = 0 in the last chunk)
#pragma unroll
    for (int jp = 0; jp < H / 2; ++jp) {
      const double2 g = lds_v2(tb + PW_T1 * 8 + jp * RS);
      x[2 * jp] = fma(g.x, X, x[2 * jp]);
      x[2 * jp + 1] = fma(g.y, X, x[2 * jp + 1]);
    }
  }

  // F = t w + x*, then rhs_n = scaling_n ((I + dT A) F_n - prev_n); the rhs rows replace the (consumed)
  // prev rows in st and the CTA stores them coalesced
  asm volatile("cp.async.wait_group 0;\n" ::);
  __syncthreads();
  {
    const double sc = valid ? a.scaling[n] : 0.0;
    const double pmul = (n == 0) ? a.alpha : 1.0;
    const unsigned ps = (n == 0) ? st_s + (unsigned)((PW_NC * LD + k * (H + 1)) * sizeof(double)) : xs_;
    double dd[2];  // dia of the current and the next row travel with t
    {
      const double2 c0 = lds_v2(tb + PW_T2 * 8), t0 = lds_v2(tb + PW_T3 * 8);
      x[0] = fma(t0.x, x[0], c0.x);
      dd[0] = t0.y;
    }
    // the conversion of row j + 1 (x[j + 1] = F_{j+1}, with its dia) runs one trip ahead of the matvec of row j
    const double2 el0 = lds_v2(tb + PW_T4 * 8);
    double em = el0.x;  // off[row - 1] of row 0 of this chunk
    // F of the last row of the previous chunk and the first row of the next chunk
    double f_last;
    {
      const double2 cl = lds_v2(tb + PW_T2 * 8 + (H - 1) * RS), tl = lds_v2(tb + PW_T3 * 8 + (H - 1) * RS);
      f_last = fma(tl.x, x[H - 1], cl.x);
    }
    const double left = __shfl_sync(KLE_FULL_MASK, f_last, su[PwL::LOGP]);
    const double right = __shfl_sync(KLE_FULL_MASK, x[0], sd[PwL::LOGP]);
    const double el_next0 = __shfl_sync(KLE_FULL_MASK, em, sd[PwL::LOGP]);  // off[row - 1] of the next chunk's row 0
    double xl = (k > 0) ? left : 0.0;
    double2 el = el0;
#pragma unroll
    for (int j = 0; j < H; ++j) {
      // F_{j+1} and dia_{j+1}
      double xp;
      if (j < H - 1) {
        const double2 c1 = lds_v2(tb + PW_T2 * 8 + (j + 1) * RS), t1 = lds_v2(tb + PW_T3 * 8 + (j + 1) * RS);
        x[j + 1] = fma(t1.x, x[j + 1], c1.x);
        dd[(j + 1) & 1] = t1.y;
        xp = x[j + 1];
      } else {
        xp = (k < P - 1) ? right : 0.0;
      }
      if ((j & 1) == 1 && j + 1 < H) el = lds_v2(tb + PW_T4 * 8 + ((j + 1) >> 1) * RS);
      // off[row] = off[(row + 1) - 1]: the next row's "em"
      const double ep = (j < H - 1) ? (((j + 1) & 1) ? el.y : el.x) : ((k < P - 1) ? el_next0 : 0.0);
      const double xc = x[j];
      const double Ax = fma(em, xl, fma(dd[j & 1], xc, ep * xp));
      const double prev = lds_f64(ps + (unsigned)(j * sizeof(double)));
      xl = xc;
      em = ep;
      x[j] = sc * (fma(a.dT, Ax, xc) - pmul * prev);
    }
  }
  __syncwarp();  // (a lane's prev rows are its own st positions, except row 16, which nobody writes)
#pragma unroll
  for (int j = 0; j < H; ++j) sts_f64(xs_ + (unsigned)(j * sizeof(double)), x[j]);
  __syncthreads();
  for (int ln = 0; ln < PW_NC; ++ln) {
    const int nn = n0 + ln;
    if (nn >= N) break;
    double* out = a.Rout + sbase + (size_t)nn * nx;
    const double* rs = st + ln * LD;
    for (int r = tid; r < nx; r += 128) out[r] = rs[r + (r >> 6)];
  }
}

bool pw_supported(const FineLayoutRT& lay, int nx) {
  if (KLE_FINE_LAZY || lay.W || lay.kind || lay.MR != 16 || lay.P != 32) return false;
  if (nx <= 128 || nx > PW_H * PW_P) return false;
  const char* e = getenv("KLE_FGR_PW");  // read per call (A/B in one process); KLE_FGR_PW=0: partitioned kernel
  return !(e && *e == '0');
}

int pw_flag_offset() { return PwOuter::PW_OFF + kPwFlag; }

int pw_fgr(const FgrArgs& a, cudaStream_t st) {
  constexpr size_t smem = sizeof(double) * (size_t)PW_SMEM_DOUBLES;
  static PerDeviceOnce attr_once;
  if (int rc = once_per_device(attr_once, "kle_fine_pw: cudaFuncSetAttribute", [&] {
        cudaError_t e = cudaFuncSetAttribute(fgr_pw_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        return cudaFuncSetAttribute(fgr_pw_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
      }))
    return rc;
  dim3 grid(a.M, (a.N + PW_NC - 1) / PW_NC);
  fgr_pw_kernel<<<grid, 128, smem, st>>>(a);
  return check_launch("fgr_pw_kernel");
}

}  // namespace kle
