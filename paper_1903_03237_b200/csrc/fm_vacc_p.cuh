// fm_vacc_p.cuh -- k_vacc_p: the pair-per-thread V_fm accumulation of k_vacc
// (fm_spatial.cuh; separate.py:218-222, _kernels.py:276-293) as persistent
// CTAs for complex64, M = 5..8 (config 1).
//
// k_vacc runs one CTA per (bin, 512-frame segment): at config 1 that is 1026
// CTAs on 444 resident slots (2.31 waves, the last 31% full), and every CTA
// pays its own prologue (gain partials -> g MU, first X / lambda fetch), two
// barriers per 256-frame chunk and a slice reduction. Here the (bin, TB-frame
// chunk) items are dealt out in contiguous runs to a fixed grid of resident
// CTAs (item q of B*F*nseg goes to CTA q*G/items), and inside a CTA the
// chunks are software-pipelined over a double-buffered stage:
//   iteration j:  A(j+1)  frame-per-thread: 1/y and x of chunk j+1 from the
//                         registers fetched one iteration earlier -> stage
//                         (j+1)&1; then the global fetch of chunk j+2
//                 G(j+2)  gains of chunk j+2's bin (g MU from the k_gain
//                         partials; a copy when the bin does not change)
//                 B(j)    pair-per-thread accumulation over stage j&1
//                 one __syncthreads
// The accumulators stay in registers across the chunks of a bin; a run of
// chunks [s0, s1] of one bin is reduced over the slices (fixed order) and
// written to partial slot s0, slots s0+1..s1 get zeros, so k_ip still sums
// nseg partials per bin in slot order (deterministic for a given grid).
#pragma once
#include "fm_spatial.cuh"

namespace fm {

template <int M, int TB> struct VpCfg {
  static constexpr int BS = 256, P = M * (M + 1) / 2, S2 = BS / P;
  static constexpr int MINB = TB >= 256 ? 3 : 4;
  static constexpr size_t stage_bytes = (size_t)TB * M * 12;  // [TB][M] 1/y | [TB][M] complex x
  static constexpr size_t o_red = 2 * stage_bytes;
  static constexpr size_t red_bytes = (size_t)S2 * M * P * 8;
  static constexpr size_t o_gs = o_red + red_bytes;
  static constexpr size_t SMEM = o_gs + 2 * NMAX * M * 4;
};

template <int M, int TB>
__global__ void __launch_bounds__(256, VpCfg<M, TB>::MINB)
    k_vacc_p(VaccArgs<float> a, int nseg, int items) {
  pdl_entry();
  using C = float2;
  using Cf = VpCfg<M, TB>;
  constexpr int P = Cf::P, S2 = Cf::S2;
  extern __shared__ __align__(16) unsigned char smp[];
  __shared__ int pairs[2 * P];
  float* gsb = reinterpret_cast<float*>(smp + Cf::o_gs);  // [2][NMAX * M]
  C* red = reinterpret_cast<C*>(smp + Cf::o_red);
  const int tid = threadIdx.x;
  const int N = a.N, T = a.T, F = a.F;
  const size_t FT = (size_t)F * T;
  // 32-bit item arithmetic throughout (the host keeps items < 2^31): 64-bit
  // divisions per item cost as many instructions as the pair loop itself
  const int q0 = (int)((long long)items * blockIdx.x / gridDim.x);
  const int q1 = (int)((long long)items * (blockIdx.x + 1) / gridDim.x);
  if (q0 >= q1) return;
  if (tid < P) {
    int i = 0, r = tid;
    while (r >= M - i) {
      r -= M - i;
      ++i;
    }
    pairs[2 * tid] = i;
    pairs[2 * tid + 1] = i + r;
  }
  // gains of item q's bin into gs buffer `buf`: the g MU finished from the
  // k_gain partials in segment order (as k_vacc), or a copy of the previous
  // item's when the bin is the same; the bin's first chunk writes gnew
  auto gains = [&](int q, int bf, int seg, int buf) {
    float* gd = gsb + buf * (NMAX * M);
    if (q > q0 && seg > 0) {  // the previous item is the same bin's
      const float* gsrc = gsb + (buf ^ 1) * (NMAX * M);
      for (int e = tid; e < N * M; e += 256) gd[e] = gsrc[e];
      return;
    }
    if (tid >= N * M) return;
    const int b = bf / F, f = bf - b * F;
    for (int e = tid; e < N * M; e += 256) {
      const int n = e / M, m = e % M;
      const float* gp = a.gpart + (size_t)bf * a.gseg * N * 2 * M + n * 2 * M;
      float sn = 0, sd = 0;
      for (int s = 0; s < a.gseg; ++s) {
        sn += gp[(size_t)s * N * 2 * M + m];
        sd += gp[(size_t)s * N * 2 * M + M + m];
      }
      const size_t gi = (size_t)b * N * F * M + (size_t)n * F * M + (size_t)f * M + m;
      const float gv = a.g[gi] * mu_factor(sn, sd);
      gd[e] = gv;
      if (seg == 0) a.gnew[gi] = gv;
    }
  };
  float lp[NMAX];
  C xp[M];
  auto fetch = [&](int bf, int seg) {  // tid < TB
    const int b = bf / F, f = bf - b * F;
    const int ta = seg * TB, tb = min(T, ta + TB);
    const int t = ta + tid;
    const int tc = t < tb ? t : tb - 1;
    const float* lamb = a.lam + (size_t)b * N * FT + (size_t)f * T;
#pragma unroll
    for (int n = 0; n < NMAX; ++n) {
      lp[n] = 0.f;
      if (n >= N) break;
      lp[n] = lamb[(size_t)n * FT + tc];
    }
    CRowIO<float, M>::load(a.X + ((size_t)bf * T + tc) * M, xp);
  };
  // phase A of item q (registers from fetch(q)) into stage `buf`
  auto stage_a = [&](int bf, int seg, int buf) {  // tid < TB
    const int ta = seg * TB, tb = min(T, ta + TB);
    const bool tv = ta + tid < tb;
    const float fl = a.floorp[(unsigned)bf / (unsigned)F];
    float* iys = reinterpret_cast<float*>(smp + buf * Cf::stage_bytes);
    C* Xc = reinterpret_cast<C*>(smp + buf * Cf::stage_bytes + (size_t)TB * M * 4);
    float l[NMAX];
    C xv[M];
#pragma unroll
    for (int n = 0; n < NMAX; ++n) l[n] = lp[n];
#pragma unroll
    for (int m = 0; m < M; ++m) xv[m] = tv ? xp[m] : make_float2(0.f, 0.f);
    float iy[M], y[M];
    model_power<float, M>(l, gsb + buf * (NMAX * M), N, fl, iy, y);
#pragma unroll
    for (int m = 0; m < M; ++m)
      if (!tv) iy[m] = 0.f;
    RowIO<float, M>::store(iys + tid * M, iy);
    CRowIO<float, M>::store(Xc + tid * M, xv);
  };
  // (bin, chunk) of items q, q + 1, q + 2, advanced incrementally
  int bf0 = q0 / nseg, sg0 = q0 - bf0 * nseg;
  auto next = [&](int& bf, int& sg, int bfp, int sgp) {
    sg = sgp + 1;
    bf = bfp;
    if (sg == nseg) {
      sg = 0;
      bf = bfp + 1;
    }
  };
  int bf1, sg1, bf2, sg2;
  next(bf1, sg1, bf0, sg0);
  next(bf2, sg2, bf1, sg1);
  // ---- prologue: gains of the first two items, chunk 0 staged, chunk 1 in flight
  gains(q0, bf0, sg0, 0);
  if (tid < TB) fetch(bf0, sg0);
  __syncthreads();
  if (q0 + 1 < q1) gains(q0 + 1, bf1, sg1, 1);
  if (tid < TB) {
    stage_a(bf0, sg0, 0);
    if (q0 + 1 < q1) fetch(bf1, sg1);
  }
  __syncthreads();
  const int p = tid % P, s2 = tid / P;
  const bool act = s2 < S2;
  const int pi = pairs[2 * p], pj = pairs[2 * p + 1];
  C v[M];
#pragma unroll
  for (int m = 0; m < M; ++m) v[m] = make_float2(0.f, 0.f);
  int run_s0 = sg0;
  for (int q = q0; q < q1; ++q) {
    const int j = (q - q0) & 1;
    if (q + 1 < q1 && tid < TB) {
      stage_a(bf1, sg1, j ^ 1);
      if (q + 2 < q1) fetch(bf2, sg2);
    }
    if (q + 2 < q1) gains(q + 2, bf2, sg2, j);
    if (act) {
      const float* iys = reinterpret_cast<const float*>(smp + j * Cf::stage_bytes);
      const C* Xc = reinterpret_cast<const C*>(smp + j * Cf::stage_bytes + (size_t)TB * M * 4);
      int tl = s2;
      for (; tl + S2 < TB; tl += 2 * S2) {
        const C xi0 = Xc[tl * M + pi], xj0 = Xc[tl * M + pj];
        const C xi1 = Xc[(tl + S2) * M + pi], xj1 = Xc[(tl + S2) * M + pj];
        float iy0[M], iy1[M];
        RowIO<float, M>::load(iys + tl * M, iy0);
        RowIO<float, M>::load(iys + (tl + S2) * M, iy1);
        C p0, p1;  // x_i conj(x_j)
        p0.x = xi0.x * xj0.x + xi0.y * xj0.y;
        p0.y = xi0.y * xj0.x - xi0.x * xj0.y;
        p1.x = xi1.x * xj1.x + xi1.y * xj1.y;
        p1.y = xi1.y * xj1.x - xi1.x * xj1.y;
#pragma unroll
        for (int m = 0; m < M; ++m) {
          v[m] = fma2(make_float2(iy0[m], iy0[m]), p0, v[m]);
          v[m] = fma2(make_float2(iy1[m], iy1[m]), p1, v[m]);
        }
      }
      if (tl < TB) {
        const C xi = Xc[tl * M + pi], xj = Xc[tl * M + pj];
        C pr;
        pr.x = xi.x * xj.x + xi.y * xj.y;
        pr.y = xi.y * xj.x - xi.x * xj.y;
        float iy[M];
        RowIO<float, M>::load(iys + tl * M, iy);
#pragma unroll
        for (int m = 0; m < M; ++m) v[m] = fma2(make_float2(iy[m], iy[m]), pr, v[m]);
      }
    }
    const int bf = bf0, seg = sg0;
    const bool last = (q + 1 == q1) || (bf1 != bf0);  // CTA-uniform
    if (last && act) {
#pragma unroll
      for (int m = 0; m < M; ++m) red[(s2 * M + m) * P + p] = v[m];
    }
    __syncthreads();
    if (last) {
      C* pb = reinterpret_cast<C*>(a.part) + ((size_t)bf * nseg + run_s0) * M * P;
      for (int e = tid; e < M * P; e += 256) {
        C acc = red[e];
        for (int s = 1; s < S2; ++s) {
          const C o = red[s * M * P + e];
          acc.x += o.x;
          acc.y += o.y;
        }
        pb[e] = acc;
        for (int z = 1; z <= seg - run_s0; ++z) pb[(size_t)z * M * P + e] = make_float2(0.f, 0.f);
      }
#pragma unroll
      for (int m = 0; m < M; ++m) v[m] = make_float2(0.f, 0.f);
      run_s0 = 0;
      __syncthreads();
    }
    bf0 = bf1; sg0 = sg1;
    bf1 = bf2; sg1 = sg2;
    next(bf2, sg2, bf1, sg1);
  }
}

}  // namespace fm
