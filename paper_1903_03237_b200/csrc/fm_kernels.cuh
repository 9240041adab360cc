// fm_kernels.cuh -- hand-written sm_100a kernels of the FastMNMF iteration.
//
// One FastMNMF iteration (_DiagLoop.iterate, separate.py:201-234; paths are
// relative to /root/reference/pkg/src/fastsep) is executed as seven launches
// over device-resident state:
//
//   k_wstats   W statistics phi H^T + W MU (sources.py:191-194), from the phi
//              of the previous statistics pass
//   k_lambda   lambda = W H  (sources.py:184-187)
//   k_phi      second statistics pass (separate.py:215)
//   k_hstats   H statistics W^T phi + H MU (sources.py:195-198)
//   k_lambda   lambda = W H with the new H
//   k_front    gain stats + g MU, V_fm, IP rows, normalisations (fm_spatial.cuh)
//   k_back     projection + the NEXT iteration's first statistics pass
//
// Layout (row-major, batch-major): X (B,F,T,M) complex, xt (B,F,T,M),
// Q (B,F,M,M) complex, g (B,N,F,M), W (B,N,F,K), H (B,N,K,T),
// lam (B,N,F,T), phi (B,2,N,F,T).
#pragma once
#include "fm_common.cuh"
#include "fm_linalg.cuh"
#include "fm_nmf.cuh"
#include "fm_spatial.cuh"

namespace fm {

// ---------------------------------------------------------------------------
// lambda = W H per (b, n): (F x K) (K x T). SIMT register-blocked tile:
// 64 f x 64 t per CTA, 4 x 4 outputs per thread, K staged 32 at a time.
// ---------------------------------------------------------------------------
template <typename R>
__global__ void __launch_bounds__(256) k_lambda(const R* __restrict__ W, const R* __restrict__ H,
                                                R* __restrict__ lam, int F, int T, int K, int N,
                                                int n0) {
  pdl_entry();
  __shared__ __align__(16) R Ws[32][64 + 4];
  __shared__ __align__(16) R Hs[32][64 + 4];
  const int bn = blockIdx.z;  // (b, NMF source); NMF sources are lambda sources n0..N-1
  const int Nn = N - n0;
  const int t0 = blockIdx.x * 64, f0 = blockIdx.y * 64;
  const R* Wb = W + (size_t)bn * F * K;
  const R* Hb = H + (size_t)bn * K * T;
  R* Lb = lam + ((size_t)(bn / Nn) * N + n0 + bn % Nn) * F * T;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  // 16-B vector paths need 4-element alignment of rows (fp32 only)
  const bool vec = sizeof(R) == 4 && (K % 4) == 0 && (T % 4) == 0;
  R acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0;
  for (int k0 = 0; k0 < K; k0 += 32) {
    const int kc = min(32, K - k0);
    if (vec) {
      const int kq = kc / 4;  // float4 per W row segment
      for (int e = threadIdx.x; e < 64 * kq; e += 256) {
        const int fl = e / kq, q = e % kq, f = f0 + fl;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (f < F) v = *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(Wb) + (size_t)f * K + k0 + 4 * q);
        Ws[4 * q][fl] = v.x; Ws[4 * q + 1][fl] = v.y; Ws[4 * q + 2][fl] = v.z; Ws[4 * q + 3][fl] = v.w;
      }
      for (int e = threadIdx.x; e < kc * 16; e += 256) {
        const int kh = e / 16, q = e % 16, t = t0 + 4 * q;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (t < T) v = *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(Hb) + (size_t)(k0 + kh) * T + t);
        *reinterpret_cast<float4*>(&Hs[kh][4 * q]) = v;
      }
    } else {
      for (int e = threadIdx.x; e < 64 * kc; e += 256) {
        const int fl = e / kc, kl = e % kc, f = f0 + fl;
        Ws[kl][fl] = f < F ? Wb[(size_t)f * K + k0 + kl] : R(0);
      }
      for (int e = threadIdx.x; e < kc * 64; e += 256) {
        const int kh = e / 64, th = e % 64, t = t0 + th;
        Hs[kh][th] = t < T ? Hb[(size_t)(k0 + kh) * T + t] : R(0);
      }
    }
    __syncthreads();
    for (int k = 0; k < kc; ++k) {
      R a[4], h[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = Ws[k][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) h[j] = Hs[k][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] += a[i] * h[j];
    }
    __syncthreads();
  }
  const int tb = t0 + tx * 4;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int f = f0 + ty * 4 + i;
    if (f >= F) continue;
    R* o = Lb + (size_t)f * T + tb;
    if (vec && tb + 3 < T) {
      *reinterpret_cast<float4*>(reinterpret_cast<float*>(o)) =
          make_float4((float)acc[i][0], (float)acc[i][1], (float)acc[i][2], (float)acc[i][3]);
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (tb + j < T) o[j] = acc[i][j];
    }
  }
}

// ---------------------------------------------------------------------------
// H MU (sources.py:195-198) from the F-chunk partials, fixed summation order.
// mode 0: H *= mu(sum_c part); mode 1: hout = sum_c part (sharded phase 0);
// mode 2: H *= mu(hin) (sharded phase 1, after the all-reduce).
// ---------------------------------------------------------------------------
template <typename R>
__global__ void __launch_bounds__(256) k_hupdate(const R* __restrict__ part, R* __restrict__ H,
                                                 R* __restrict__ hbuf, int FC, long long NKT,
                                                 long long total, int mode) {
  pdl_entry();
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const long long b = i / NKT, r = i % NKT;
  R num = 0, den = 0;
  if (mode == 2) {
    num = hbuf[(b * 2) * NKT + r];
    den = hbuf[(b * 2 + 1) * NKT + r];
  } else {
    const R* pb = part + (b * FC * 2) * NKT + r;
    for (int c = 0; c < FC; ++c) {
      num += pb[(size_t)(2 * c) * NKT];
      den += pb[(size_t)(2 * c + 1) * NKT];
    }
  }
  if (mode == 1) {
    hbuf[(b * 2) * NKT + r] = num;
    hbuf[(b * 2 + 1) * NKT + r] = den;
  } else {
    H[i] = H[i] * mu_factor(num, den);
  }
}

}  // namespace fm
