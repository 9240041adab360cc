// fm_small.cuh -- register-accumulating gain statistics and V_fm kernels for
// few channels (M <= 4: configs 0 and 2).
//
// At M <= 4 the staged, slice-parallel k_gain / k_vacc (fm_spatial.cuh) spend
// their time in per-chunk shared-memory staging and barriers around a few
// FMAs per frame (config 2: 2.1 / 2.3 TB/s of HBM). Here a CTA holds four
// bins, 64 threads (two warps) each; a thread walks frames t = ta + i,
// ta + i + 64, ... of its (bin, segment), keeping the whole per-bin sum set in
// registers -- 2NM gain sums (separate.py:217, _kernels.py:244-250) or the
// M x P complex V sums (_kernels.py:276-293) -- and each bin reduces once at
// the end: xor-shuffle trees within its warps, then its two warp partials in
// warp order (fixed order: bitwise reproducible).
// Outputs use the staged kernels' partial layouts, so the consumers (k_vacc's
// g MU, k_ip's V reduction) are unchanged.
//
// Measured on B200 at config 2: slower than the staged kernels
// (k_gain 1.18 vs 0.90 ms, k_vacc 1.34 vs 1.31 ms; unrolling the frame loop
// to overlap loads spills at 255 registers), so they are opt-in (FM_SMALL=1)
// and kept verified by tests/test_gpu_ipw.py.
#pragma once
#include "fm_common.cuh"
#include "fm_nmf.cuh"
#include "fm_spatial.cuh"

namespace fm {

constexpr int SMALL_BS = 256, SMALL_TPB = 64, SMALL_BPB = SMALL_BS / SMALL_TPB;

// per-bin fixed-order sum of NV per-thread values over the bin's two warps
// into out[bin][0..NV) (smem scratch red >= 8 * NV)
template <typename R, int NV>
__device__ __forceinline__ void bin_sum_fixed(R (&v)[NV], R* red, R* out) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    R x = v[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    v[i] = x;
  }
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) red[warp * NV + i] = v[i];
  }
  __syncthreads();
  constexpr int WPB = SMALL_TPB / 32;  // warps per bin
  for (int e = tid; e < SMALL_BPB * NV; e += SMALL_BS) {
    const int bl = e / NV, i = e % NV;
    R s = 0;
    for (int w = 0; w < WPB; ++w) s += red[(bl * WPB + w) * NV + i];
    out[e] = s;
  }
  __syncthreads();
}

// gain statistics, grid (nseg, ceil(F/4), B), block 256; writes GainArgs::part
template <typename R, int M>
__global__ void __launch_bounds__(SMALL_BS) k_gain_r(GainArgs<R> a) {
  pdl_entry();
  constexpr int NV = 2 * NMAX * M;  // [n][num M | den M]
  __shared__ __align__(16) R gs[SMALL_BPB][NMAX * M];
  __shared__ R red[(SMALL_BS / 32) * NV];
  __shared__ R out[SMALL_BPB * NV];
  const int seg = blockIdx.x, b = blockIdx.z, nseg = gridDim.x;
  const int tid = threadIdx.x, bl = tid / SMALL_TPB, ti = tid % SMALL_TPB;
  const int N = a.N, T = a.T, F = a.F;
  const int f = blockIdx.y * SMALL_BPB + bl;
  const bool fv = f < F;
  const size_t FT = (size_t)F * T;
  const int ta = seg * a.TR, tb = min(T, ta + a.TR);
  for (int e = ti; e < N * M; e += SMALL_TPB)
    gs[bl][e] = fv ? a.g[(size_t)b * N * F * M + (size_t)(e / M) * F * M + (size_t)f * M + (e % M)] : R(0);
  __syncthreads();
  const R fl = a.floorp[b];
  const R* lamb = a.lam + (size_t)b * N * FT + (size_t)(fv ? f : 0) * T;
  const R* xtb = a.xt + ((size_t)b * F + (fv ? f : 0)) * T * M;
  R acc[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) acc[i] = R(0);
  for (int t = ta + ti; fv && t < tb; t += SMALL_TPB) {
    R l[NMAX], xv[M], iy[M], y[M];
#pragma unroll
    for (int n = 0; n < NMAX; ++n) l[n] = n < N ? lamb[(size_t)n * FT + t] : R(0);
    RowIO<R, M>::load(xtb + (size_t)t * M, xv);
    model_power<R, M>(l, gs[bl], N, fl, iy, y);
#pragma unroll
    for (int m = 0; m < M; ++m) xv[m] *= iy[m] * iy[m];  // x~ / y^2
#pragma unroll
    for (int n = 0; n < NMAX; ++n) {
      if (n >= N) break;
#pragma unroll
      for (int m = 0; m < M; ++m) {
        acc[n * 2 * M + m] += l[n] * xv[m];
        acc[n * 2 * M + M + m] += l[n] * iy[m];
      }
    }
  }
  bin_sum_fixed<R, NV>(acc, red, out);
  for (int e = tid; e < SMALL_BPB * N * 2 * M; e += SMALL_BS) {
    const int bl2 = e / (N * 2 * M), i = e % (N * 2 * M), f2 = blockIdx.y * SMALL_BPB + bl2;
    if (f2 < F) a.part[(((size_t)b * F + f2) * nseg + seg) * N * 2 * M + i] = out[bl2 * NV + i];
  }
}

// g MU + V_fm = (1/T) sum_t x x^H / y_ftm, grid (nseg, ceil(F/4), B), block
// 256; writes VaccArgs::part (M x P complex per segment) and gnew (segment 0)
template <typename R, int M>
__global__ void __launch_bounds__(SMALL_BS) k_vacc_r(VaccArgs<R> a) {
  pdl_entry();
  using C = cplx<R>;
  constexpr int P = M * (M + 1) / 2, NV = 2 * M * P;  // [m][pair] (re, im)
  __shared__ __align__(16) R gs[SMALL_BPB][NMAX * M];
  __shared__ R red[(SMALL_BS / 32) * NV];
  __shared__ R out[SMALL_BPB * NV];
  const int seg = blockIdx.x, b = blockIdx.z, nseg = gridDim.x;
  const int tid = threadIdx.x, bl = tid / SMALL_TPB, ti = tid % SMALL_TPB;
  const int N = a.N, T = a.T, F = a.F;
  const int f = blockIdx.y * SMALL_BPB + bl;
  const bool fv = f < F;
  const size_t FT = (size_t)F * T;
  const int ta = seg * a.TR, tb = min(T, ta + a.TR);
  // finish the gain MU from the gain partials (fixed order), separate.py:218-220
  for (int e = ti; e < N * M; e += SMALL_TPB) {
    R gv = R(0);
    if (fv) {
      const int n = e / M, m = e % M;
      const R* gp = a.gpart + ((size_t)b * F + f) * a.gseg * N * 2 * M + n * 2 * M;
      R sn = 0, sd = 0;
      for (int q = 0; q < a.gseg; ++q) {
        sn += gp[(size_t)q * N * 2 * M + m];
        sd += gp[(size_t)q * N * 2 * M + M + m];
      }
      const size_t gi = (size_t)b * N * F * M + (size_t)n * F * M + (size_t)f * M + m;
      gv = a.g[gi] * mu_factor(sn, sd);
      if (seg == 0) a.gnew[gi] = gv;
    }
    gs[bl][e] = gv;
  }
  __syncthreads();
  const R fl = a.floorp[b];
  const R* lamb = a.lam + (size_t)b * N * FT + (size_t)(fv ? f : 0) * T;
  const C* Xb = a.X + ((size_t)b * F + (fv ? f : 0)) * T * M;
  R acc[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) acc[i] = R(0);
  for (int t = ta + ti; fv && t < tb; t += SMALL_TPB) {
    R l[NMAX], iy[M], y[M];
    C xv[M];
#pragma unroll
    for (int n = 0; n < NMAX; ++n) l[n] = n < N ? lamb[(size_t)n * FT + t] : R(0);
    CRowIO<R, M>::load(Xb + (size_t)t * M, xv);
    model_power<R, M>(l, gs[bl], N, fl, iy, y);
    int p = 0;
#pragma unroll
    for (int i = 0; i < M; ++i) {
#pragma unroll
      for (int j = i; j < M; ++j, ++p) {
        const R pr = xv[i].x * xv[j].x + xv[i].y * xv[j].y;  // x_i conj(x_j)
        const R pi = xv[i].y * xv[j].x - xv[i].x * xv[j].y;
#pragma unroll
        for (int m = 0; m < M; ++m) {
          acc[(m * P + p) * 2] += iy[m] * pr;
          acc[(m * P + p) * 2 + 1] += iy[m] * pi;
        }
      }
    }
  }
  bin_sum_fixed<R, NV>(acc, red, out);
  for (int e = tid; e < SMALL_BPB * M * P; e += SMALL_BS) {
    const int bl2 = e / (M * P), i = e % (M * P), f2 = blockIdx.y * SMALL_BPB + bl2;
    if (f2 < F)
      reinterpret_cast<C*>(a.part)[(((size_t)b * F + f2) * nseg + seg) * M * P + i] =
          cmake<C>(out[bl2 * NV + 2 * i], out[bl2 * NV + 2 * i + 1]);
  }
}

}  // namespace fm
