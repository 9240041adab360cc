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

// ---------------------------------------------------------------------------
// Small SIMT GEMM with a fused epilogue, for the decoder MLP (per mixture b):
//   C[r, c] = epi( sum_k A[r, k] * B'(k, c) + bias[c] )
// B' = B^T (B stored (Ncol, K)) when BT, else B (stored (K, Ncol)).
// epilogue: 0 none, 1 tanh, 2 exp, 3 multiply by (1 - aux[r,c]^2) (tanh').
// grid (ceil(Ncol/64), ceil(Rows/64), batch), block 256, 4x4 per thread.
// A, C, aux are batched with strides sA, sC; B and bias are shared.
// ---------------------------------------------------------------------------
// Adam update fused into the last backward GEMM (EPI 4): the GEMM output is
// dL/dz; z, m, v2 are updated in place. Step index t = iter * steps + s + 1
// from the device iteration counter (no host round trip inside a graph).
template <typename R> struct AdamEpi {
  R* z;
  R* m;
  R* v2;
  const unsigned* iter;
  int s, steps;
  float lr, b1, b2, eps;
};

template <typename R, bool BT, int EPI, int TM, int TN>
__global__ void __launch_bounds__(256) k_mlp_gemm(const R* __restrict__ A, const R* __restrict__ Bm,
                                                  const R* __restrict__ bias, const R* __restrict__ aux,
                                                  R* __restrict__ Cm, int Rows, int Ncol, int K,
                                                  long long sA, long long sC, AdamEpi<R> ad) {
  pdl_entry();
  constexpr int KC = 16, IM = TM / 16, IN = TN / 16;  // thread tile IM x IN
  __shared__ R As[KC][TM + 4];
  __shared__ R Bs[KC][TN + 4];
  const int b = blockIdx.z;
  const R* Ab = A + (size_t)b * sA;
  R* Cb = Cm + (size_t)b * sC;
  const R* Xb = aux ? aux + (size_t)b * sC : nullptr;
  const int r0 = blockIdx.y * TM, c0 = blockIdx.x * TN;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  R acc[IM][IN];
#pragma unroll
  for (int i = 0; i < IM; ++i)
#pragma unroll
    for (int j = 0; j < IN; ++j) acc[i][j] = 0;
  for (int k0 = 0; k0 < K; k0 += KC) {
    for (int e = threadIdx.x; e < TM * KC; e += 256) {
      const int rr = e / KC, kk = e % KC;  // A tile: rows x k (k contiguous)
      const int r = r0 + rr, k = k0 + kk;
      As[kk][rr] = (r < Rows && k < K) ? Ab[(size_t)r * K + k] : R(0);
    }
    for (int e = threadIdx.x; e < TN * KC; e += 256) {
      if (BT) {  // B stored (Ncol, K): element (c, k)
        const int cc = e / KC, kk = e % KC, c = c0 + cc, k = k0 + kk;
        Bs[kk][cc] = (c < Ncol && k < K) ? Bm[(size_t)c * K + k] : R(0);
      } else {   // B stored (K, Ncol): element (k, c), c contiguous
        const int kb = e / TN, cb = e % TN, kq = k0 + kb, c = c0 + cb;
        Bs[kb][cb] = (kq < K && c < Ncol) ? Bm[(size_t)kq * Ncol + c] : R(0);
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < KC; ++k) {
      R a[IM], h[IN];
#pragma unroll
      for (int i = 0; i < IM; ++i) a[i] = As[k][ty * IM + i];
#pragma unroll
      for (int j = 0; j < IN; ++j) h[j] = Bs[k][tx * IN + j];
#pragma unroll
      for (int i = 0; i < IM; ++i)
#pragma unroll
        for (int j = 0; j < IN; ++j) acc[i][j] += a[i] * h[j];
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < IM; ++i) {
    const int r = r0 + ty * IM + i;
    if (r >= Rows) continue;
#pragma unroll
    for (int j = 0; j < IN; ++j) {
      const int c = c0 + tx * IN + j;
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

// ---------------------------------------------------------------------------
// Fused decoder layers for the latent loop (one CTA per 32 frames of one
// mixture; 256 threads; the hidden width Hd <= 256 lives in shared memory):
//   k_dec_fwd12 : h1 = tanh(W1 z + b1), h2 = tanh(W2 h1 + b2)
//   k_dec_bwd21 : d1 = (W2^T d2) (1 - h1^2), g = W1^T d1, Adam(z, g)
// Output layer (F wide) and its backward use the tiled k_mlp_gemm.
// ---------------------------------------------------------------------------
constexpr int DEC_RT = 16;     // frames per CTA
constexpr int DEC_HMAX = 128;  // max hidden width (config 4: 128)
constexpr int DEC_DMAX = 64;   // max latent width

template <typename R>
__global__ void __launch_bounds__(256) k_dec_fwd12(const R* __restrict__ z, const R* __restrict__ W1,
                                                   const R* __restrict__ b1, const R* __restrict__ W2,
                                                   const R* __restrict__ b2, R* __restrict__ h1,
                                                   R* __restrict__ h2, int T, int D, int Hd) {
  pdl_entry();
  __shared__ R zs[DEC_RT][DEC_DMAX + 1];
  __shared__ R hs[DEC_RT][DEC_HMAX + 1];
  const int b = blockIdx.y, t0 = blockIdx.x * DEC_RT, tid = threadIdx.x;
  const R* zb = z + ((size_t)b * T + t0) * D;
  for (int e = tid; e < DEC_RT * D; e += 256) {
    const int r = e / D, c = e % D;
    zs[r][c] = (t0 + r < T) ? zb[(size_t)r * D + c] : R(0);
  }
  __syncthreads();
  // layer 1: thread = hidden unit j (strided), all 32 rows
  for (int j = tid; j < Hd; j += 256) {
    R acc[DEC_RT];
#pragma unroll
    for (int r = 0; r < DEC_RT; ++r) acc[r] = b1[j];
    for (int k = 0; k < D; ++k) {
      const R w = W1[(size_t)j * D + k];
#pragma unroll
      for (int r = 0; r < DEC_RT; ++r) acc[r] += w * zs[r][k];
    }
#pragma unroll
    for (int r = 0; r < DEC_RT; ++r) hs[r][j] = tanh(acc[r]);
  }
  __syncthreads();
  R* h1b = h1 + ((size_t)b * T + t0) * Hd;
  for (int e = tid; e < DEC_RT * Hd; e += 256) {
    const int r = e / Hd, c = e % Hd;
    if (t0 + r < T) h1b[(size_t)r * Hd + c] = hs[r][c];
  }
  // layer 2
  R* h2b = h2 + ((size_t)b * T + t0) * Hd;
  for (int j = tid; j < Hd; j += 256) {
    R acc[DEC_RT];
#pragma unroll
    for (int r = 0; r < DEC_RT; ++r) acc[r] = b2[j];
    for (int k = 0; k < Hd; ++k) {
      const R w = W2[(size_t)j * Hd + k];
#pragma unroll
      for (int r = 0; r < DEC_RT; ++r) acc[r] += w * hs[r][k];
    }
#pragma unroll
    for (int r = 0; r < DEC_RT; ++r)
      if (t0 + r < T) h2b[(size_t)r * Hd + j] = tanh(acc[r]);
  }
}

template <typename R>
__global__ void __launch_bounds__(256) k_dec_bwd21(const R* __restrict__ d2, const R* __restrict__ h1,
                                                   const R* __restrict__ W1, const R* __restrict__ W2,
                                                   int T, int D, int Hd, AdamEpi<R> ad) {
  pdl_entry();
  __shared__ R ds[DEC_RT][DEC_HMAX + 1];
  __shared__ R d1s[DEC_RT][DEC_HMAX + 1];
  const int b = blockIdx.y, t0 = blockIdx.x * DEC_RT, tid = threadIdx.x;
  const R* d2b = d2 + ((size_t)b * T + t0) * Hd;
  const R* h1b = h1 + ((size_t)b * T + t0) * Hd;
  for (int e = tid; e < DEC_RT * Hd; e += 256) {
    const int r = e / Hd, c = e % Hd;
    ds[r][c] = (t0 + r < T) ? d2b[(size_t)r * Hd + c] : R(0);
  }
  __syncthreads();
  // d1[r][j] = (sum_k d2[r][k] W2[k][j]) (1 - h1[r][j]^2)
  for (int j = tid; j < Hd; j += 256) {
    R acc[DEC_RT];
#pragma unroll
    for (int r = 0; r < DEC_RT; ++r) acc[r] = 0;
    for (int k = 0; k < Hd; ++k) {
      const R w = W2[(size_t)k * Hd + j];
#pragma unroll
      for (int r = 0; r < DEC_RT; ++r) acc[r] += ds[r][k] * w;
    }
#pragma unroll
    for (int r = 0; r < DEC_RT; ++r) {
      const R h = (t0 + r < T) ? h1b[(size_t)r * Hd + j] : R(0);
      d1s[r][j] = acc[r] * (R(1) - h * h);
    }
  }
  __syncthreads();
  // gz[r][c] = sum_k d1[r][k] W1[k][c], then Adam on z[r][c]
  const double tstep = (double)(*ad.iter) * ad.steps + ad.s + 1;
  const R c1 = (R)(1.0 - pow((double)ad.b1, tstep)), c2 = (R)(1.0 - pow((double)ad.b2, tstep));
  for (int e = tid; e < DEC_RT * D; e += 256) {
    const int r = e / D, c = e % D;
    if (t0 + r >= T) continue;
    R gsum = 0;
    for (int k = 0; k < Hd; ++k) gsum += d1s[r][k] * W1[(size_t)k * D + c];
    const size_t i = ((size_t)b * T + t0 + r) * D + c;
    const R mi = R(ad.b1) * ad.m[i] + R(1 - ad.b1) * gsum;
    const R vi = R(ad.b2) * ad.v2[i] + R(1 - ad.b2) * gsum * gsum;
    ad.m[i] = mi;
    ad.v2[i] = vi;
    ad.z[i] -= R(ad.lr) * (mi / c1) / (sqrt_r(vi / c2) + R(ad.eps));
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
__global__ void k_dp_grad(const R* __restrict__ u, const R* __restrict__ v, const R* __restrict__ r,
                          const R* __restrict__ lam, const R* __restrict__ xt, const R* __restrict__ g,
                          R* __restrict__ go, int N, int F, int T) {
  pdl_entry();
  __shared__ R tile[32][33];
  __shared__ __align__(16) R gs[32][NMAX * M];  // g[n][f][m] of this tile's 32 bins
  const int b = blockIdx.z, t0 = blockIdx.x * 32, f0 = blockIdx.y * 32;
  const size_t FT = (size_t)F * T;
  const int tid = threadIdx.y * 32 + threadIdx.x;
  const R* rb = r + (size_t)b * T * F;
  for (int i = threadIdx.y; i < 32; i += 8) {  // r[t][f] tile, f contiguous
    const int t = t0 + i, f = f0 + threadIdx.x;
    tile[i][threadIdx.x] = (t < T && f < F) ? rb[(size_t)t * F + f] : R(0);
  }
  for (int e = tid; e < 32 * N * M; e += 256) {
    const int fl = e / (N * M), q = e % (N * M), n = q / M, m = q % M, f = f0 + fl;
    gs[fl][q] = f < F ? g[(((size_t)b * N + n) * F + f) * M + m] : R(0);
  }
  __syncthreads();
  R val[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int i = threadIdx.y + 8 * q;
    const int f = f0 + i, t = t0 + threadIdx.x;
    val[q] = 0;
    if (f < F && t < T) {
      const R l0 = u[(size_t)b * F + f] * v[(size_t)b * T + t] * tile[threadIdx.x][i];
      const R* lb = lam + (size_t)b * N * FT + (size_t)f * T + t;
      R ln[NMAX];
#pragma unroll
      for (int n = 1; n < NMAX; ++n) {
        ln[n] = R(0);
        if (n >= N) break;
        ln[n] = lb[(size_t)n * FT];
      }
      R x[M];
      RowIO<R, M>::load(xt + (((size_t)b * F + f) * T + t) * M, x);
      R acc = 0;
#pragma unroll
      for (int m = 0; m < M; ++m) {
        R rest = 0;
#pragma unroll
        for (int n = 1; n < NMAX; ++n) {
          if (n >= N) break;
          rest += ln[n] * gs[i][n * M + m];
        }
        const R g0 = gs[i][m];
        R y = l0 * g0 + rest;
        y = y > RT<R>::tiny() ? y : RT<R>::tiny();
        const R iy = rcp_r(y);
        acc += g0 * (iy - x[m] * iy * iy);
      }
      val[q] = acc * l0;
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < 4; ++q) tile[threadIdx.y + 8 * q][threadIdx.x] = val[q];
  __syncthreads();
  R* gb = go + (size_t)b * T * F;
  for (int i = threadIdx.y; i < 32; i += 8) {  // write go[t][f], f contiguous
    const int t = t0 + i, f = f0 + threadIdx.x;
    if (t < T && f < F) gb[(size_t)t * F + f] = tile[threadIdx.x][i];
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
