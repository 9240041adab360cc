// fm_lambda_tc.cuh -- lambda = W H (sources.py:184-187) on the tensor cores
// for large complex64 problems with K a multiple of 8 up to 32 (config 3).
//
// Per (mixture, source): D[t][f] = sum_k A[t][k] B[f][k] with A[t][k] =
// H[k][t] (frames on the 128 accumulator lanes: a thread owns a frame, reads
// its column of H coalesced, splits it into TF32 hi / lo and stores both to
// its TMEM lane once per CTA) and B[f][k] = W[f][k] for a tile of 32 bins
// (K-major rows exactly as W lies in memory; hi rows then lo rows in shared
// memory). Per 8-column k-step: D[:, 0:64] (+)= A_hi [B_hi | B_lo] (N = 64)
// and D[:, 0:32] += A_lo B_hi (N = 32) -- 3xTF32, fp32 accumulation in TMEM.
// After the commit every thread reads its lane, adds the two halves and
// writes lambda[f][t] for the tile's 32 bins: a warp's stores are 128
// contiguous bytes. A CTA keeps its 128-frame tile and walks a group of bin
// tiles. grid (ceil(T/128), bin groups, B * sources), block 128, 128 TMEM
// columns (4 CTAs per SM).
#pragma once
#include "fm_vacc_tc.cuh"

namespace fm {

constexpr int LTC_FT = 32;  // bins per MMA tile

static __global__ void __launch_bounds__(128, 4)
k_lambda_tc(const float* __restrict__ W, const float* __restrict__ H, float* __restrict__ lam, int F,
            int T, int K, int N, int n0, int FPG) {
  pdl_entry();
  __shared__ __align__(128) unsigned char Bs[64 * 128];  // rows 0..31 hi, 32..63 lo; 8 k-quads per row
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int bn = blockIdx.z, Nn = N - n0;
  const int t0 = blockIdx.x * 128;
  const int fa = blockIdx.y * FPG, fb = min(F, fa + FPG);
  const int tid = threadIdx.x, warp = tid >> 5;
  const float* Wb = W + (size_t)bn * F * K;
  const float* Hb = H + (size_t)bn * K * T;
  float* Lb = lam + ((size_t)(bn / Nn) * N + n0 + bn % Nn) * F * T;
  const int KS = K >> 3;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (unsigned)__cvta_generic_to_shared(&tmem_base)),
                 "r"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    mbar_init(&mbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  const uint32_t tl = tmem + ((uint32_t)(warp * 32) << 16);
  const int t = t0 + tid;
  {  // A: this frame's column of H, hi / lo, K padded to 32 with zeros
    float ah[32], al[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      const float v = (k < K && t < T) ? Hb[(size_t)k * T + t] : 0.f;
      ah[k] = tf32_rna(v);
      al[k] = v - ah[k];
    }
    tmem_st_row<32>(tl + 0, ah);
    tmem_st_row<32>(tl + 32, al);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  const uint64_t dB = umma_desc((unsigned)__cvta_generic_to_shared(Bs), 128, 8 * 128);
  constexpr uint32_t IDESC64 = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(64 >> 3) << 17) |
                               ((uint32_t)(128 >> 4) << 24);
  constexpr uint32_t IDESC32 = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(32 >> 3) << 17) |
                               ((uint32_t)(128 >> 4) << 24);
  unsigned u = 0;
#pragma unroll 1
  for (int f0 = fa; f0 < fb; f0 += LTC_FT, ++u) {
    // B: W rows of the tile's bins (zeros beyond F and beyond K)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int e = tid + 128 * j, fl = e >> 5, k = e & 31;
      const float v = (f0 + fl < fb && k < K) ? Wb[(size_t)(f0 + fl) * K + k] : 0.f;
      const float hi = tf32_rna(v);
      const uint32_t o = (uint32_t)(((fl >> 3) * 8 + (k >> 2)) * 128 + (fl & 7) * 16 + (k & 3) * 4);
      *reinterpret_cast<float*>(Bs + o) = hi;
      *reinterpret_cast<float*>(Bs + o + 4096) = v - hi;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();  // B written, every lane's previous accumulator read done
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      for (int ks = 0; ks < KS; ++ks) {
        const uint64_t db = dB + (uint64_t)(ks * 16);
        umma_tf32_ts(tmem + 64, tmem + (uint32_t)(ks * 8), db, IDESC64, ks > 0 ? 1u : 0u);
        umma_tf32_ts(tmem + 64, tmem + (uint32_t)(32 + ks * 8), db, IDESC32, 1u);
      }
      umma_commit(&mbar);
    }
    mbar_wait(&mbar, u & 1u);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    float* lp = Lb + (size_t)f0 * T + t;
#pragma unroll
    for (int hf = 0; hf < 2; ++hf) {
      float d0[16], d1[16];
      tmem_ld16(tl + 64 + hf * 16, d0);
      tmem_ld16(tl + 96 + hf * 16, d1);
      if (t < T) {
#pragma unroll
        for (int i = 0; i < 16; ++i)
          if (f0 + hf * 16 + i < fb) lp[(size_t)(hf * 16 + i) * T] = d0[i] + d1[i];
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128));
}

}  // namespace fm
