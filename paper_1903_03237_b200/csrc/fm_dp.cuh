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

namespace fm {

// ---------------------------------------------------------------------------
// Small SIMT GEMM with a fused epilogue, for the decoder MLP (per mixture b):
//   C[r, c] = epi( sum_k A[r, k] * B'(k, c) + bias[c] )
// B' = B^T (B stored (Ncol, K)) when BT, else B (stored (K, Ncol)).
// epilogue: 0 none, 1 tanh, 2 exp, 3 multiply by (1 - aux[r,c]^2) (tanh').
// grid (ceil(Ncol/64), ceil(Rows/64), batch), block 256, 4x4 per thread.
// A, C, aux are batched with strides sA, sC; B and bias are shared.
// ---------------------------------------------------------------------------
template <typename R, bool BT, int EPI>
__global__ void __launch_bounds__(256) k_mlp_gemm(const R* __restrict__ A, const R* __restrict__ Bm,
                                                  const R* __restrict__ bias, const R* __restrict__ aux,
                                                  R* __restrict__ Cm, int Rows, int Ncol, int K,
                                                  long long sA, long long sC) {
  pdl_entry();
  __shared__ R As[16][64 + 4];
  __shared__ R Bs[16][64 + 4];
  const int b = blockIdx.z;
  const R* Ab = A + (size_t)b * sA;
  R* Cb = Cm + (size_t)b * sC;
  const R* Xb = aux ? aux + (size_t)b * sC : nullptr;
  const int r0 = blockIdx.y * 64, c0 = blockIdx.x * 64;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  R acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0;
  for (int k0 = 0; k0 < K; k0 += 16) {
    for (int e = threadIdx.x; e < 64 * 16; e += 256) {
      const int rr = e / 16, kk = e % 16;  // A tile: rows x k (k contiguous)
      const int r = r0 + rr, k = k0 + kk;
      As[kk][rr] = (r < Rows && k < K) ? Ab[(size_t)r * K + k] : R(0);
      if (BT) {  // B stored (Ncol, K): element (c, k)
        const int cc = e / 16, c = c0 + cc;
        Bs[kk][cc] = (c < Ncol && k < K) ? Bm[(size_t)c * K + k] : R(0);
      } else {   // B stored (K, Ncol): element (k, c), c contiguous
        const int kb = e / 64, cb = e % 64, kq = k0 + kb, c = c0 + cb;
        Bs[kb][cb] = (kq < K && c < Ncol) ? Bm[(size_t)kq * Ncol + c] : R(0);
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      R a[4], h[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[k][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) h[j] = Bs[k][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] += a[i] * h[j];
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = r0 + ty * 4 + i;
    if (r >= Rows) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = c0 + tx * 4 + j;
      if (c >= Ncol) continue;
      R v = acc[i][j] + (bias ? bias[c] : R(0));
      if (EPI == 1) v = tanh(v);
      if (EPI == 2) v = exp(v);
      if (EPI == 3) {
        const R h = Xb[(size_t)r * Ncol + c];
        v = v * (R(1) - h * h);
      }
      Cb[(size_t)r * Ncol + c] = v;
    }
  }
}

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

// dL/do[t, f] of the NLL sum(x~/y + log y), y = max(lambda_0 g_0 + y_rest, TINY),
// y_rest = sum_{n>=1} lambda_n g_n (separate.py:207, metropolis_log_gamma_fast
// sources.py:292-304): dL/dlambda_0 = sum_m g_0 (1/y - x~/y^2), dlambda_0/do = lambda_0.
// grid (ceil(T/32), ceil(F/32), B), block (32, 8); lambda_0 read from lam.
template <typename R, int M>
__global__ void k_dp_grad(const R* __restrict__ lam, const R* __restrict__ xt, const R* __restrict__ g,
                          R* __restrict__ go, int N, int F, int T) {
  pdl_entry();
  __shared__ R tile[32][33];
  const int b = blockIdx.z, t0 = blockIdx.x * 32, f0 = blockIdx.y * 32;
  const size_t FT = (size_t)F * T;
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int f = f0 + i, t = t0 + threadIdx.x;
    R val = 0;
    if (f < F && t < T) {
      const R* lb = lam + (size_t)b * N * FT + (size_t)f * T + t;
      const R l0 = lb[0];
      R x[M];
      RowIO<R, M>::load(xt + (((size_t)b * F + f) * T + t) * M, x);
      R acc = 0;
#pragma unroll
      for (int m = 0; m < M; ++m) {
        R rest = 0;
        for (int n = 1; n < N; ++n) rest += lb[(size_t)n * FT] * g[(((size_t)b * N + n) * F + f) * M + m];
        const R g0 = g[((size_t)b * N * F + f) * M + m];
        R y = l0 * g0 + rest;
        y = y > RT<R>::tiny() ? y : RT<R>::tiny();
        const R iy = R(1) / y;
        acc += g0 * (iy - x[m] * iy * iy);
      }
      val = acc * l0;
    }
    tile[i][threadIdx.x] = val;
  }
  __syncthreads();
  R* gb = go + (size_t)b * T * F;
  for (int i = threadIdx.y; i < 32; i += 8) {  // write go[t][f], f contiguous
    const int t = t0 + i, f = f0 + threadIdx.x;
    if (t < T && f < F) gb[(size_t)t * F + f] = tile[threadIdx.x][i];
  }
}

// Adam on z (bias-corrected); m, v2 and the step counter persist across
// outer iterations. One thread per latent entry.
template <typename R>
__global__ void k_adam(R* __restrict__ z, const R* __restrict__ gz, R* __restrict__ m, R* __restrict__ v2,
                       unsigned* __restrict__ step, long long n, float lr, float b1, float b2, float eps) {
  pdl_entry();
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned t = *step + 1u;  // this step's index (counter advanced by k_dp_tick)
  if (i < n) {
    const R g = gz[i];
    const R mi = R(b1) * m[i] + R(1 - b1) * g;
    const R vi = R(b2) * v2[i] + R(1 - b2) * g * g;
    m[i] = mi;
    v2[i] = vi;
    const R mh = mi / (R(1) - (R)pow((double)b1, (double)t));
    const R vh = vi / (R(1) - (R)pow((double)b2, (double)t));
    z[i] -= R(lr) * mh / (sqrt_r(vh) + R(eps));
  }
}

static __global__ void k_dp_tick(unsigned* step) {
  pdl_entry();
  *step += 1u;
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

// V step (sources.py:262-265): v_t *= sqrt(sum_f u_f r_tf phi1_0 / max(..., TINY))
// grid (ceil(T/32), B), block (32, 8): lanes over t, warps stride f
template <typename R>
__global__ void k_dp_vmu(const R* __restrict__ u, R* __restrict__ v, const R* __restrict__ r,
                         const R* __restrict__ phi, int N, int F, int T) {
  pdl_entry();
  __shared__ R red[2][8][33];
  const int b = blockIdx.y, t = blockIdx.x * 32 + threadIdx.x, w = threadIdx.y;
  const size_t FT = (size_t)F * T;
  const R* p1 = phi + (size_t)b * 2 * N * FT;
  const R* p2 = p1 + (size_t)N * FT;
  R sn = 0, sd = 0;
  if (t < T) {
    for (int f = w; f < F; f += 8) {
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
    v[(size_t)b * T + t] *= mu_factor(a, c);
  }
}

// absorb c[0] of the gain normalisation into u (sources.py:269-271); grid (ceil(F/256), B)
template <typename R>
__global__ void k_dp_absorb(R* __restrict__ u, const R* __restrict__ cs, int F) {
  pdl_entry();
  const int f = blockIdx.x * blockDim.x + threadIdx.x, b = blockIdx.y;
  if (f < F) u[(size_t)b * F + f] *= cs[((size_t)b * F + f) * NMAX + 0];
}

}  // namespace fm
