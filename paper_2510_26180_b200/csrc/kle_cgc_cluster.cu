// Cluster-resident diagonalised CGC (three-step solve), one thread-block
// cluster per sample.
//
// Reference: three_step_solve pintuq/pcgc.py:148-172, factor_shifted :90-145,
// the increment / stop test of pcgc_solve :335-348.
//
// The sample's N x nx block is split into CL row blocks of RB = 16*MR rows,
// one CTA each (CL <= 8, a portable cluster). Per CTA:
//   1. R[:, rows] -> shared-memory tile, radix-2 FFT along the time axis
//      (p = F* scaling r, norm "ortho"); only f = 0..N/2 is solved
//      (real input: q_{N-f} = conj(q_f)).
//   2. For every frequency f, a 16-lane group owns the CTA's RB rows
//      (MR per lane, in registers) and runs the complex LDL^T solve of
//      (lambda_f I + dT A) with pivots 1/beta precomputed once per batch
//      (shift_factor_kernel: the factorisation is iteration invariant).
//      The two linear recurrences are stitched by a 16-lane affine scan
//      (shuffles) and across the cluster's CTAs through distributed shared
//      memory (each CTA publishes its block composite; consumers compose the
//      composites of the blocks before/after them).
//   3. Hermitian completion, inverse FFT, u = Re(.)/scaling, increment and
//      imaginary-residue max-reductions (block, then cluster via DSMEM), the
//      per-sample stop test.
// HBM traffic per outer iteration and (n, i): R 8 B + U 8 B read, U 8 B
// written, pivots 16 (N/2+1)/N B read.
#include <cooperative_groups.h>

#include "kle_common.cuh"
#include "kle_internal.h"

namespace cg = cooperative_groups;

namespace kle {

constexpr int CL_LANES = 16;

__device__ __forceinline__ Cplx cfma(Cplx a, Cplx b, Cplx c) {  // a*b + c
  return {fma(a.re, b.re, fma(-a.im, b.im, c.re)), fma(a.re, b.im, fma(a.im, b.re, c.im))};
}
__device__ __forceinline__ Cplx cneg_mul(Cplx a, Cplx b) {  // -(a*b)
  return {fma(-a.re, b.re, a.im * b.im), fma(-a.re, b.im, -a.im * b.re)};
}
__device__ __forceinline__ Cplx shfl_up_c(Cplx v, int d) {
  return {__shfl_up_sync(KLE_FULL_MASK, v.re, d, CL_LANES), __shfl_up_sync(KLE_FULL_MASK, v.im, d, CL_LANES)};
}
__device__ __forceinline__ Cplx shfl_down_c(Cplx v, int d) {
  return {__shfl_down_sync(KLE_FULL_MASK, v.re, d, CL_LANES), __shfl_down_sync(KLE_FULL_MASK, v.im, d, CL_LANES)};
}

// In-place radix-2 DIT over a [N][TC] tile (rows in bit-reversed order).
__device__ void fft_tile_nt(Cplx* t, const Cplx* tw, int N, int TC, bool inverse) {
  for (int len = 2; len <= N; len <<= 1) {
    const int half = len >> 1, step = N / len;
    const int nbf = (N >> 1) * TC;
    for (int b = threadIdx.x; b < nbf; b += blockDim.x) {
      const int c = b % TC, bf = b / TC;
      const int g = bf / half, j = bf - g * half;
      const int i0 = g * len + j, i1 = i0 + half;
      Cplx w = tw[j * step];
      if (inverse) w.im = -w.im;
      const Cplx x0 = t[i0 * TC + c];
      const Cplx x1 = t[i1 * TC + c];
      const Cplx v = {fma(x1.re, w.re, -x1.im * w.im), fma(x1.re, w.im, x1.im * w.re)};
      t[i0 * TC + c] = {x0.re + v.re, x0.im + v.im};
      t[i1 * TC + c] = {x0.re - v.re, x0.im - v.im};
    }
    __syncthreads();
  }
}

// pivots 1/beta_i of (lambda_f I + dT A), f = 0..N/2, layout [s][f][i]
__global__ void shift_factor_kernel(const double* __restrict__ dia, const double* __restrict__ off,
                                    const double* __restrict__ lam, int M, int NF, int nx, double dT,
                                    double* __restrict__ sfac) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= (long long)M * NF) return;
  const int s = (int)(t / NF), f = (int)(t - (long long)s * NF);
  const double* d = dia + (size_t)s * nx;
  const double* e = off + (size_t)s * nx;
  Cplx* out = reinterpret_cast<Cplx*>(sfac) + ((size_t)s * NF + f) * nx;
  const Cplx lm = {lam[2 * f], lam[2 * f + 1]};
  Cplx ib = {0.0, 0.0};
  for (int i = 0; i < nx; ++i) {
    Cplx beta = {fma(dT, d[i], lm.re), lm.im};
    if (i > 0) {
      const double E = dT * e[i - 1];
      beta.re = fma(-E * E, ib.re, beta.re);
      beta.im = fma(-E * E, ib.im, beta.im);
    }
    ib = crcp(beta);
    out[i] = ib;
  }
}

template <int MR>
__global__ void __launch_bounds__(576, 1) cgc_cluster_kernel(CgcArgs a, const double* __restrict__ sfac_d,
                                                              int log2N) {
  constexpr int RB = CL_LANES * MR;
  cg::cluster_group cluster = cg::this_cluster();
  const int CL = (int)cluster.num_blocks();
  const int c = (int)cluster.block_rank();
  const int s = blockIdx.x / CL;
  const int N = a.N, nx = a.nx, NF = N / 2 + 1;
  if (a.status && a.status[s] != KLE_SAMPLE_ACTIVE) return;  // uniform over the cluster

  extern __shared__ double smem[];
  Cplx* tile = reinterpret_cast<Cplx*>(smem);  // [N][RB]
  Cplx* tw = tile + N * RB;                    // [N]
  Cplx* fwd = tw + N;                          // [NF][2]: (A, B) block composite
  Cplx* bwd = fwd + 2 * NF;                    // [NF][2]: (S, T)
  double* red = reinterpret_cast<double*>(bwd + 2 * NF);  // [34]

  const int tid = threadIdx.x;
  for (int j = tid; j < N; j += blockDim.x) {
    double sn, cs;
    sincospi(-2.0 * (double)j / (double)N, &sn, &cs);
    tw[j] = {cs, sn};
  }
  const size_t sb = (size_t)s * N * nx;
  const int row0 = c * RB;
  // ---- phase 1: tile load (bit-reversed rows) + forward FFT --------------
  for (int idx = tid; idx < N * RB; idx += blockDim.x) {
    const int n = idx / RB, col = idx - n * RB, row = row0 + col;
    double v = 0.0;
    if (row < nx) {
      v = a.R[sb + (size_t)n * nx + row];
      if (a.load_scale) v *= a.load_scale[n];
    }
    const int pos = log2N > 0 ? (int)(__brev((unsigned)n) >> (32 - log2N)) : 0;
    tile[pos * RB + col] = {v, 0.0};
  }
  __syncthreads();
  fft_tile_nt(tile, tw, N, RB, false);

  // ---- phase 2: shifted solves ---------------------------------------------
  const int fsys = tid / CL_LANES, k = tid % CL_LANES;
  const bool valid = fsys < NF;
  const int f = valid ? fsys : NF - 1;
  const double rsN = 1.0 / sqrt((double)N);
  const Cplx* ib_s = reinterpret_cast<const Cplx*>(sfac_d) + ((size_t)s * NF + f) * nx;
  const double* ee = a.off + (size_t)s * nx;
  const int r0 = row0 + k * MR;

  Cplx y[MR], l[MR], ib[MR];
  // l_r = dT off_{r-1} / beta_{r-1} (0 for r = 0 and pad rows)
  Cplx ibprev = {0.0, 0.0};
  if (r0 > 0 && r0 - 1 < nx) ibprev = ib_s[r0 - 1];
#pragma unroll
  for (int j = 0; j < MR; ++j) {
    const int r = r0 + j;
    const Cplx p = tile[f * RB + k * MR + j];
    y[j] = {p.re * rsN, p.im * rsN};
    ib[j] = (r < nx) ? ib_s[r] : Cplx{1.0, 0.0};
    double E = 0.0;
    if (r > 0 && r < nx) E = a.dT * ee[r - 1];
    const Cplx ip = (j == 0) ? ibprev : ib[j - 1];
    l[j] = {E * ip.re, E * ip.im};
  }
  // forward, lane local: yl_j = p_j - l_j yl_{j-1}; composite (A = prod(-l), B = yl_end)
  Cplx A = {1.0, 0.0};
#pragma unroll
  for (int j = 0; j < MR; ++j) {
    if (j > 0) y[j] = cfma({-l[j].re, -l[j].im}, y[j - 1], y[j]);
    A = cneg_mul(l[j], A);
  }
  Cplx B = y[MR - 1];
#pragma unroll
  for (int d = 1; d < CL_LANES; d <<= 1) {
    const Cplx Ao = shfl_up_c(A, d), Bo = shfl_up_c(B, d);
    if (k >= d) {
      B = cfma(A, Bo, B);
      A = cmul(A, Ao);
    }
  }
  Cplx Ae = shfl_up_c(A, 1), Be = shfl_up_c(B, 1);
  if (k == 0) {
    Ae = {1.0, 0.0};
    Be = {0.0, 0.0};
  }
  if (valid && k == CL_LANES - 1) {
    fwd[2 * f] = A;
    fwd[2 * f + 1] = B;
  }
  cluster.sync();
  Cplx Yc = {0.0, 0.0};
  for (int q = 0; q < c; ++q) {
    const Cplx* rf = cluster.map_shared_rank(fwd, q);
    Yc = cfma(rf[2 * f], Yc, rf[2 * f + 1]);
  }
  const Cplx Cin = cfma(Ae, Yc, Be);
  // stitch + scale: y_j += pi_j Cin, z_j = y_j / beta_j
  {
    Cplx pi = {1.0, 0.0};
#pragma unroll
    for (int j = 0; j < MR; ++j) {
      pi = cneg_mul(l[j], pi);
      y[j] = cmul(cfma(pi, Cin, y[j]), ib[j]);
    }
  }
  // backward, lane local: xl_j = z_j - l_{j+1} xl_{j+1}
  Cplx lnext;
  {
    const int r = r0 + MR - 1;
    double E = 0.0;
    if (r + 1 < nx) E = a.dT * ee[r];
    lnext = {E * ib[MR - 1].re, E * ib[MR - 1].im};
  }
  Cplx S = {1.0, 0.0};
#pragma unroll
  for (int j = MR - 1; j >= 0; --j) {
    const Cplx ln = (j == MR - 1) ? lnext : l[j + 1];
    if (j < MR - 1) y[j] = cfma({-ln.re, -ln.im}, y[j + 1], y[j]);
    S = cneg_mul(ln, S);
  }
  Cplx T = y[0];
#pragma unroll
  for (int d = 1; d < CL_LANES; d <<= 1) {
    const Cplx So = shfl_down_c(S, d), To = shfl_down_c(T, d);
    if (k + d < CL_LANES) {
      T = cfma(S, To, T);
      S = cmul(S, So);
    }
  }
  Cplx Se = shfl_down_c(S, 1), Te = shfl_down_c(T, 1);
  if (k == CL_LANES - 1) {
    Se = {1.0, 0.0};
    Te = {0.0, 0.0};
  }
  if (valid && k == 0) {
    bwd[2 * f] = S;
    bwd[2 * f + 1] = T;
  }
  cluster.sync();
  Cplx Xc = {0.0, 0.0};
  for (int q = CL - 1; q > c; --q) {
    const Cplx* rb = cluster.map_shared_rank(bwd, q);
    Xc = cfma(rb[2 * f], Xc, rb[2 * f + 1]);
  }
  const Cplx Xin = cfma(Se, Xc, Te);
  {
    Cplx sg = {1.0, 0.0};
#pragma unroll
    for (int j = MR - 1; j >= 0; --j) {
      const Cplx ln = (j == MR - 1) ? lnext : l[j + 1];
      sg = cneg_mul(ln, sg);
      y[j] = cfma(sg, Xin, y[j]);
    }
  }
  // ---- phase 3: Hermitian completion, inverse FFT, update ----------------
  if (valid) {
    const int pf = log2N > 0 ? (int)(__brev((unsigned)f) >> (32 - log2N)) : 0;
    const int nf = N - f;
    const int pn = (f > 0 && nf > f) ? (int)(__brev((unsigned)nf) >> (32 - log2N)) : -1;
#pragma unroll
    for (int j = 0; j < MR; ++j) {
      tile[pf * RB + k * MR + j] = y[j];
      if (pn >= 0) tile[pn * RB + k * MR + j] = {y[j].re, -y[j].im};
    }
  }
  __syncthreads();
  fft_tile_nt(tile, tw, N, RB, true);
  double incmax = 0.0, immax = 0.0;
  for (int idx = tid; idx < N * RB; idx += blockDim.x) {
    const int n = idx / RB, col = idx - n * RB, row = row0 + col;
    if (row >= nx) continue;
    const Cplx v = tile[n * RB + col];
    const double isc = a.inv_scaling[n];
    const double u = (v.re * rsN) * isc;
    const double ui = (v.im * rsN) * isc;
    const size_t g = sb + (size_t)n * nx + row;
    if (a.Uout) {
      if (a.U) incmax = nanmax(incmax, fabs(u - a.U[g]));
      a.Uout[g] = u;
    } else {
      incmax = nanmax(incmax, fabs(u - a.U[g]));
      a.U[g] = u;
    }
    immax = nanmax(immax, fabs(ui));
  }
  // block then cluster reductions
  incmax = warp_max(incmax);
  immax = warp_max(immax);
  const int lane = tid & 31, w = tid >> 5, nw = (blockDim.x + 31) >> 5;
  if (lane == 0) red[w] = incmax;
  __syncthreads();
  if (tid == 0) {
    double r1 = 0.0;
    for (int i = 0; i < nw; ++i) r1 = nanmax(r1, red[i]);
    red[32] = r1;
  }
  __syncthreads();
  if (lane == 0) red[w] = immax;
  __syncthreads();
  if (tid == 0) {
    double r2 = 0.0;
    for (int i = 0; i < nw; ++i) r2 = nanmax(r2, red[i]);
    red[33] = r2;
  }
  cluster.sync();
  if (c == 0 && tid == 0) {
    double inc = red[32], im = red[33];
    for (int q = 1; q < CL; ++q) {
      const double* rr = cluster.map_shared_rank(red, q);
      inc = nanmax(inc, rr[32]);
      im = nanmax(im, rr[33]);
    }
    if (a.inc) a.inc[s] = inc;
    if (a.inc_hist) a.inc_hist[(size_t)s * a.max_iters + (a.k - 1)] = inc;
    if (a.imag) a.imag[s] = nanmax(a.imag[s], im);
    if (a.status) {
      int st = KLE_SAMPLE_ACTIVE;
      if (inc <= a.tol) st = KLE_SAMPLE_CONVERGED;
      else if (!isfinite(inc)) st = KLE_SAMPLE_NONFINITE;
      else if (a.k >= a.max_iters) st = KLE_SAMPLE_MAXITERS;
      if (st != KLE_SAMPLE_ACTIVE) {
        a.status[s] = st;
        if (a.iters) a.iters[s] = a.k;
      } else if (a.active_count) {
        atomicAdd(a.active_count, 1);
      }
    }
  }
  cluster.sync();  // keep every CTA's shared memory alive until rank 0 has read it
}

// ---------------------------------------------------------------------------
static bool cluster_shape(int N, int nx, int* MR, int* CL) {
  if (N < 2 || N > 64 || (N & (N - 1))) return false;  // <= 33 systems x 16 lanes <= 576 threads
  int mr = (nx <= 128 || nx > 512) ? 8 : 4;
  const int rb = CL_LANES * mr;
  const int cl = (nx + rb - 1) / rb;
  if (cl > 8) return false;
  *MR = mr;
  *CL = cl;
  return true;
}

bool cgc_cluster_supported(int N, int nx) {
  int mr, cl;
  return cluster_shape(N, nx, &mr, &cl);
}

size_t shift_factor_doubles(int M, int N, int nx) { return 2 * (size_t)M * (N / 2 + 1) * nx; }

int shift_factor(const double* dia, const double* off, const double* lam, int M, int N, int nx, double dT,
                 double* sfac, cudaStream_t st) {
  const int NF = N / 2 + 1;
  const long long nth = (long long)M * NF;
  if (nth == 0) return KLE_OK;
  shift_factor_kernel<<<(unsigned)((nth + 127) / 128), 128, 0, st>>>(dia, off, lam, M, NF, nx, dT, sfac);
  return check_launch("shift_factor_kernel");
}

template <int MR>
static int launch_cluster(const CgcArgs& a, const double* sfac, int CL, int log2N, cudaStream_t st) {
  constexpr int RB = CL_LANES * MR;
  const int NF = a.N / 2 + 1;
  const int nt = ((NF * CL_LANES + 31) / 32) * 32;
  const size_t smem = ((size_t)a.N * RB + a.N + 4 * NF) * sizeof(Cplx) + 34 * sizeof(double);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(cgc_cluster_kernel<MR>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(a.M * CL), 1, 1);
  cfg.blockDim = dim3((unsigned)nt, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = CL;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, cgc_cluster_kernel<MR>, a, sfac, log2N);
  if (e != cudaSuccess) return set_error(KLE_ERR_CUDA, cudaGetErrorString(e));
  return check_launch("cgc_cluster_kernel");
}

int cgc_cluster_run(const CgcArgs& a, const double* sfac, cudaStream_t st) {
  int MR, CL;
  if (!cluster_shape(a.N, a.nx, &MR, &CL)) return set_error(KLE_ERR_UNSUPPORTED, "cgc_cluster: shape");
  if (a.M <= 0) return KLE_OK;
  int log2N = 0;
  while ((1 << log2N) < a.N) ++log2N;
  return MR == 4 ? launch_cluster<4>(a, sfac, CL, log2N, st) : launch_cluster<8>(a, sfac, CL, log2N, st);
}

}  // namespace kle
