// fm_back_tc.cuh -- the projection x~ = |Q x|^2 (separate.py:230,
// _kernels.py:204-217) on the tensor cores for complex64 with M > 8, fused
// with the next iteration's statistics pass exactly as k_back does it
// (data term, phi; separate.py:214-216, _kernels.py:226-250).
//
// Per bin, y(t) = Q x(t) over a tile of 128 frames is one real GEMM
//   D[t][j] = sum_k A[t][k] B[j][k],  k = 2c + (re|im) of channel c,
//                                     j = 2i + (re|im) of output row i,
// A[t][:] the frame's channel row exactly as it lies in memory, B the real
// 2M x 2M form of Q ([Qr -Qi; Qi Qr], rows interleaved). A thread owns a
// frame: it splits its row into TF32 hi / lo, stores both to its TMEM lane
// (tcgen05.st), one thread issues per 8-column k-step
//   D[:, 0:64] (+)= A_hi [B_hi | B_lo]   (N = 64)
//   D[:, 0:32]  += A_lo B_hi             (N = 32)
// (3xTF32: fp32-class products, fp32 accumulation in TMEM), and after the
// commit every thread reads its lane's 64 accumulator columns, forms
// x~_i = re^2 + im^2 and runs the statistics of its frame. At M = 16 the SIMT
// k_back spends 256 shared loads and 512 packed FMAs per frame on the
// projection; here it is 96 ALU operations per frame and 8 small MMAs per
// 128 frames. A CTA walks a segment of TR frames (a multiple of k_back's 256-frame
// tiles, whose data-term partial layout it keeps) of one bin, the next tile's
// loads in flight while the MMAs of the current one run. grid (nseg, F, B),
// block 128, 128 TMEM columns per CTA (4 CTAs per SM).
#pragma once
#include "fm_vacc_tc.cuh"

namespace fm {

template <int M>
__global__ void __launch_bounds__(128, 4) k_back_tc(BackArgs<float> a, int TR, int ntile) {
  pdl_entry();
  using C = float2;
  constexpr int KS = (2 * M + 7) / 8;  // 8-column k-steps
  __shared__ __align__(128) unsigned char Bq[64 * 128];  // rows 0..31 B_hi, 32..63 B_lo; K-major cores
  __shared__ __align__(16) float gs[NMAX * M];
  __shared__ float cs[NMAX];
  __shared__ double dred[4];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int seg = blockIdx.x, f = blockIdx.y, b = blockIdx.z;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int N = a.N, T = a.T, F = a.F;
  const size_t FT = (size_t)F * T;
  // B: real form of Q_f, element (j = 2i + pj, k = 2c + pk)
  const C* Qf = a.Q + ((size_t)b * F + f) * M * M;
  for (int e = tid; e < 32 * 32; e += 128) {
    const int j = e >> 5, k = e & 31;
    const int i = j >> 1, pj = j & 1, c = k >> 1, pk = k & 1;
    float v = 0.f;
    if (i < M && c < M) {
      const C q = Qf[i * M + c];
      v = pj == 0 ? (pk == 0 ? q.x : -q.y) : (pk == 0 ? q.y : q.x);
    }
    const float hi = tf32_rna(v);
    const uint32_t o = (uint32_t)(((j >> 3) * 8 + (k >> 2)) * 128 + (j & 7) * 16 + (k & 3) * 4);
    *reinterpret_cast<float*>(Bq + o) = hi;
    *reinterpret_cast<float*>(Bq + o + 4 * 1024) = v - hi;  // row 32 + j: four 8-row groups on
  }
  for (int e = tid; e < N * M; e += 128)
    gs[e] = a.g[(size_t)b * N * F * M + (size_t)(e / M) * F * M + (size_t)f * M + (e % M)];
  if (tid < NMAX) cs[tid] = a.cs ? a.cs[((size_t)b * F + f) * NMAX + tid] : 1.f;
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
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // B is read by the MMA (async proxy)
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  const uint32_t tl = tmem + ((uint32_t)(warp * 32) << 16);  // this thread's lane (= its frame)
  const uint64_t dB = umma_desc((unsigned)__cvta_generic_to_shared(Bq), 128, 8 * 128);
  constexpr uint32_t IDESC64 = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(64 >> 3) << 17) |
                               ((uint32_t)(128 >> 4) << 24);
  constexpr uint32_t IDESC32 = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(32 >> 3) << 17) |
                               ((uint32_t)(128 >> 4) << 24);
  const float fl = a.floorp[b];
  double ll = 0.0;
  const int t_begin = seg * TR, t_end = min(T, t_begin + TR);
  C xv[M];
  float ln[NMAX];
  auto fetch = [&](int t) {  // frame t's channel row and source powers (zeros beyond the segment)
#pragma unroll
    for (int m = 0; m < M; ++m) xv[m] = make_float2(0.f, 0.f);
#pragma unroll
    for (int n = 0; n < NMAX; ++n) ln[n] = 0.f;
    if (t < t_end) {
      CRowIO<float, M>::load(a.X + (((size_t)b * F + f) * T + t) * M, xv);
      const float* lb = a.lam + (size_t)b * N * FT + (size_t)f * T + t;
#pragma unroll
      for (int n = 0; n < NMAX; ++n) {
        if (n >= N) break;
        ln[n] = lb[(size_t)n * FT];
      }
    }
  };
  fetch(t_begin + tid);
  unsigned u = 0;
#pragma unroll 1
  for (int t0 = t_begin; t0 < t_end; t0 += 128, ++u) {
    const int t = t0 + tid;
    const bool tv = t < t_end;
    float l[NMAX];
#pragma unroll
    for (int n = 0; n < NMAX; ++n) l[n] = ln[n] * cs[n];
    {
      float ah[32], al[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        const float v = k < 2 * M ? ((k & 1) ? xv[k >> 1].y : xv[k >> 1].x) : 0.f;
        ah[k] = tf32_rna(v);
        al[k] = v - ah[k];
      }
      tmem_st_row<32>(tl + 0, ah);
      tmem_st_row<32>(tl + 32, al);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        const uint64_t db = dB + (uint64_t)(ks * 16);
        umma_tf32_ts(tmem + 64, tmem + (uint32_t)(ks * 8), db, IDESC64, ks > 0 ? 1u : 0u);
        umma_tf32_ts(tmem + 64, tmem + (uint32_t)(32 + ks * 8), db, IDESC32, 1u);
      }
      umma_commit(&mbar);
    }
    fetch(t + 128);  // the next tile's loads fly while the MMAs run
    mbar_wait(&mbar, u & 1u);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    float xtv[M];
    {
      float d0[16], d1[16];
      tmem_ld16(tl + 64, d0);
      tmem_ld16(tl + 96, d1);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (i >= M) break;
        const float re = d0[2 * i] + d1[2 * i], im = d0[2 * i + 1] + d1[2 * i + 1];
        xtv[i] = re * re + im * im;
      }
      if constexpr (M > 8) {
        tmem_ld16(tl + 80, d0);
        tmem_ld16(tl + 112, d1);
#pragma unroll
        for (int i = 8; i < M; ++i) {
          const float re = d0[2 * (i - 8)] + d1[2 * (i - 8)], im = d0[2 * (i - 8) + 1] + d1[2 * (i - 8) + 1];
          xtv[i] = re * re + im * im;
        }
      }
    }
    // the accumulator and operand columns are free again once every lane has read them
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    if (tv) {
      RowIO<float, M>::store(a.xt + (((size_t)b * F + f) * T + t) * M, xtv);
      float iy[M], y[M];
      model_power<float, M>(l, gs, N, fl, iy, y);
      float llt = 0;
#pragma unroll
      for (int m = 0; m < M; ++m) llt += -xtv[m] * iy[m] - log_fast(y[m]);
      ll += (double)llt;
      phi_point<float, M>(xtv, iy, gs, N, a.phi + (size_t)b * 2 * N * FT, FT, (size_t)f * T + t);
    }
  }
  ll = warp_sum(ll);
  if (lane == 0) dred[warp] = ll;
  __syncthreads();
  // data-term partials keep k_back's (B, F, ntile) layout of 256-frame slots: this
  // segment's sum in its first slot, zeros in its others
  const int slot0 = t_begin / 256, slot1 = min(ntile, (t_begin + TR + 255) / 256);
  for (int sl = slot0 + tid; sl < slot1; sl += 128)
    a.ll_part[((size_t)b * F + f) * ntile + sl] =
        sl == slot0 ? (dred[0] + dred[1]) + (dred[2] + dred[3]) : 0.0;
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128));
}

}  // namespace fm
