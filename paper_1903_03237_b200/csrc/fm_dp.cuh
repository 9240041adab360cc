// fm_dp.cuh -- FastMNMF-DP (BASELINE config 4) device kernels.
//
// Source 0 is the deep prior lambda_0[f,t] = u_f v_t r[t,f], r = exp(dec(z)),
// dec: D -> H tanh -> H tanh -> F linear (sources.py:207-220 with the config-4
// decoder); sources 1.. are NMF noise (sources.py:223-271). Per outer
// iteration the latents take `steps` Adam steps on the FastMNMF NLL against the
// frozen rest-of-model power y_rest (the hook at separate.py:205-213), then the
// U, V, W, H multiplicative steps run with a statistics refresh before each
// (sources.py:251-267, separate.py:214-216).
#pragma once
#include "fm_common.cuh"
#include "fm_nmf.cuh"

namespace fm {

constexpr int DEC_HMAX = 128;  // max hidden width (config 4: 128)
constexpr int DEC_DMAX = 64;   // max latent width

// lambda_0[b, 0, f, t] = u[b, f] v[b, t] r[b, t, f]; grid (ceil(T/32), ceil(F/32), B), block (32, 8)
template <typename R>
__global__ void k_dp_lambda(const R* __restrict__ u, const R* __restrict__ v, const R* __restrict__ r,
                            R* __restrict__ lam, int N, int F, int T) {
  pdl_entry();
  __shared__ R tile[32][33];
  const int b = blockIdx.z, t0 = blockIdx.x * 32, f0 = blockIdx.y * 32;
  const R* rb = r + (size_t)b * T * F;
  for (int i = threadIdx.y; i < 32; i += 8) {  // read r[t][f], f contiguous
    const int t = t0 + i, f = f0 + threadIdx.x;
    tile[i][threadIdx.x] = (t < T && f < F) ? rb[(size_t)t * F + f] : R(0);
  }
  __syncthreads();
  R* lb = lam + (size_t)b * N * F * T;  // source 0
  for (int i = threadIdx.y; i < 32; i += 8) {  // write lam[f][t], t contiguous
    const int f = f0 + i, t = t0 + threadIdx.x;
    if (f < F && t < T) lb[(size_t)f * T + t] = u[(size_t)b * F + f] * v[(size_t)b * T + t] * tile[threadIdx.x][i];
  }
}

// U step (sources.py:258-261): u_f *= sqrt(sum_t v_t r_tf phi1_0 / max(sum_t v_t r_tf phi2_0, TINY))
// grid (F, B), block 256
template <typename R>
__global__ void __launch_bounds__(256) k_dp_umu(R* __restrict__ u, const R* __restrict__ v,
                                                const R* __restrict__ r, const R* __restrict__ phi,
                                                int N, int F, int T) {
  pdl_entry();
  __shared__ R red[2][8];
  const int f = blockIdx.x, b = blockIdx.y, tid = threadIdx.x;
  const size_t FT = (size_t)F * T;
  const R* p1 = phi + (size_t)b * 2 * N * FT + (size_t)f * T;
  const R* p2 = p1 + (size_t)N * FT;
  R sn = 0, sd = 0;
  for (int t = tid; t < T; t += 256) {
    const R w = v[(size_t)b * T + t] * r[((size_t)b * T + t) * F + f];
    sn += w * p1[t];
    sd += w * p2[t];
  }
  sn = warp_sum(sn);
  sd = warp_sum(sd);
  if ((tid & 31) == 0) {
    red[0][tid >> 5] = sn;
    red[1][tid >> 5] = sd;
  }
  __syncthreads();
  if (tid == 0) {
    R a = 0, c = 0;
    for (int w = 0; w < 8; ++w) {
      a += red[0][w];
      c += red[1][w];
    }
    u[(size_t)b * F + f] *= mu_factor(a, c);
  }
}

// V step (sources.py:262-265): v_t *= sqrt(sum_f u_f r_tf phi1_0 / max(..., TINY)).
// grid (ceil(T/32), VMU_FS, B), block (32, 8): lanes over t, warps stride the
// bins of this CTA's split (f = fs*FR + w, w + 8, ...); each split publishes
// its (num, den) per frame and the CTA completing a 32-frame tile adds the
// splits in order and applies the update (deterministic).
constexpr int VMU_FS = 8;

template <typename R>
__global__ void k_dp_vmu(const R* __restrict__ u, R* __restrict__ v, const R* __restrict__ r,
                         const R* __restrict__ phi, int N, int F, int T, R* __restrict__ part,
                         unsigned* __restrict__ cnt) {
  pdl_entry();
  __shared__ R red[2][8][33];
  __shared__ int last;
  const int b = blockIdx.z, fs = blockIdx.y, t = blockIdx.x * 32 + threadIdx.x, w = threadIdx.y;
  const int FR = (F + VMU_FS - 1) / VMU_FS, fa = fs * FR, fb = min(F, fa + FR);
  const size_t FT = (size_t)F * T;
  const R* p1 = phi + (size_t)b * 2 * N * FT;
  const R* p2 = p1 + (size_t)N * FT;
  R sn = 0, sd = 0;
  if (t < T) {
    for (int f = fa + w; f < fb; f += 8) {
      const R q = u[(size_t)b * F + f] * r[((size_t)b * T + t) * F + f];
      sn += q * p1[(size_t)f * T + t];
      sd += q * p2[(size_t)f * T + t];
    }
  }
  red[0][w][threadIdx.x] = sn;
  red[1][w][threadIdx.x] = sd;
  __syncthreads();
  if (w == 0 && t < T) {
    R a = 0, c = 0;
    for (int k = 0; k < 8; ++k) {
      a += red[0][k][threadIdx.x];
      c += red[1][k][threadIdx.x];
    }
    part[(((size_t)b * VMU_FS + fs) * 2) * T + t] = a;
    part[(((size_t)b * VMU_FS + fs) * 2 + 1) * T + t] = c;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0 && w == 0) {
    unsigned* c = cnt + (size_t)b * gridDim.x + blockIdx.x;
    last = atomicAdd(c, 1u) == (unsigned)(VMU_FS - 1);
    if (last) *c = 0u;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (w == 0 && t < T) {
    R a = 0, c = 0;
    for (int q = 0; q < VMU_FS; ++q) {
      a += __ldcg(part + (((size_t)b * VMU_FS + q) * 2) * T + t);
      c += __ldcg(part + (((size_t)b * VMU_FS + q) * 2 + 1) * T + t);
    }
    v[(size_t)b * T + t] *= mu_factor(a, c);
  }
}

// absorb c[0] of the gain normalisation into u (sources.py:269-271); grid (ceil(F/256), B)

}  // namespace fm
