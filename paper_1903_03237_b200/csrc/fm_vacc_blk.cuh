// fm_vacc_blk.cuh -- register-blocked SIMT accumulation of the IP weighted
// covariances V_fm = (1/T) sum_t x_ft x_ft^H / y_ftm (complex64 mode).
//
// Same contract as k_vacc (fm_spatial.cuh): finish the g MU from the k_gain
// partials (separate.py:218-220), then the per-(bin, frame-segment) partial
// sums of the Hermitian upper triangle for every m (separate.py:221-222,
// spatial.py:182, _kernels.py:276-293), consumed in fixed segment order by
// k_ip. Only the thread mapping differs.
//
// Mapping. The M x M Hermitian matrix (padded to even MP) is cut into 2x2
// blocks; the NB = (MP/2)(MP/2+1)/2 blocks on or above the diagonal cover the
// upper triangle. A thread owns one block for MH = M/MS weights m (MS = 2
// m-halves when M > 8): 4 x MH complex accumulators in registers. Per frame
// it reads its two 2-vectors x_I, x_J (two 16-B shared loads) and its MH
// weights 1/y (16-B loads), forms the 4 products x_i conj(x_j) and issues
// 4*MH packed FFMA2 -- 4 shared loads per 32 FFMA2 at M = 8, against 4 per 8
// in the pair-per-thread k_vacc. Threads of one frame slice are TPS = NB*MS;
// S = BS/TPS slices stride over each staged chunk of TB frames.
//
// Reduction. Slices meet in a fixed-order binary tree through shared memory
// (value chunks of CV floats so the slots fit in the staging area); slice 0
// ends with the segment totals in registers and writes them to the (M, P)
// partial layout. Deterministic: the summation order depends only on shapes.
#pragma once
#include "fm_spatial.cuh"

namespace fm {

// CTA size and staged-chunk frames (host-visible: make_plan sizes the segments)
// (measured at M = 8, c1: 128 threads 40.8 us, 160 threads 51 us, 256 threads 60 us)
__host__ __device__ constexpr int vb_threads(int M) { return M > 8 ? 512 : 128; }
__host__ __device__ constexpr int vb_chunk(int M) { return M > 8 ? 256 : 128; }

template <int M> struct VbCfg {
  static constexpr int MP = (M + 1) / 2 * 2;
  static constexpr int NBK = MP / 2;
  static constexpr int NB = NBK * (NBK + 1) / 2;
  static constexpr int MS = (M > 8) ? 2 : 1;
  static constexpr int MH = (M + MS - 1) / MS;
  static constexpr int IW = (MS * MH + 3) / 4 * 4;  // weight row stride (floats)
  static constexpr int TPS = NB * MS;
  static constexpr int BS = vb_threads(M);
  static constexpr int S = BS / TPS;
  static constexpr int TB = vb_chunk(M);  // frames per staged chunk
  static constexpr int P = M * (M + 1) / 2;
  static constexpr int NV = 8 * MH;  // floats accumulated per thread
  // raw double buffer (X rows padded to MP, lambda rows) + the weight rows
  static constexpr int XB = TB * MP * 8, LB = NMAX * TB * 4;
  static constexpr int STAGE = 2 * (XB + LB) + TB * IW * 4;
  static constexpr int SLOTS = S / 2 > 0 ? S / 2 : 1;
  // largest value chunk (divisor of NV) whose tree slots fit in the staging area
  static constexpr int cv_pick(int cv) {
    return (cv <= 2 || SLOTS * TPS * cv * 4 <= STAGE) ? cv : cv_pick(cv / 2);
  }
  static constexpr int CV = (NV % 8 == 0) ? cv_pick(NV) : NV;
  static constexpr int SMEM = STAGE;
  static_assert(NV % CV == 0, "value chunk");
  static_assert(SLOTS * TPS * CV * 4 <= STAGE || CV <= 2, "tree slots exceed staging");
};

// n consecutive floats from 16-B aligned shared memory
template <int n> __device__ __forceinline__ void lds_row(const float* p, float (&v)[n]) {
  if constexpr (n % 4 == 0) {
#pragma unroll
    for (int i = 0; i < n; i += 4) {
      const float4 q = *reinterpret_cast<const float4*>(p + i);
      v[i] = q.x; v[i + 1] = q.y; v[i + 2] = q.z; v[i + 3] = q.w;
    }
  } else if constexpr (n % 2 == 0) {
#pragma unroll
    for (int i = 0; i < n; i += 2) {
      const float2 q = *reinterpret_cast<const float2*>(p + i);
      v[i] = q.x; v[i + 1] = q.y;
    }
  } else {
#pragma unroll
    for (int i = 0; i < n; ++i) v[i] = p[i];
  }
}

template <int M>
__global__ void __launch_bounds__(VbCfg<M>::BS) k_vacc_blk(VaccArgs<float> a) {
  pdl_entry();
  using R = float;
  using C = float2;
  using Cf = VbCfg<M>;
  constexpr int BS = Cf::BS, TB = Cf::TB, P = Cf::P, S = Cf::S, TPS = Cf::TPS, MP = Cf::MP;
  constexpr int NB = Cf::NB, NBK = Cf::NBK, MH = Cf::MH, IW = Cf::IW, NV = Cf::NV, CV = Cf::CV;
  extern __shared__ __align__(16) unsigned char vb_smem[];
  // [2][TB][MP] X rows | [2][NMAX][TB] lambda | [TB][IW] weights 1/y
  C* Xraw = reinterpret_cast<C*>(vb_smem);
  R* Lraw = reinterpret_cast<R*>(vb_smem + 2 * Cf::XB);
  R* iys = reinterpret_cast<R*>(vb_smem + 2 * (Cf::XB + Cf::LB));
  __shared__ __align__(16) R gs[NMAX * M];
  const int seg = blockIdx.x, f = blockIdx.y, b = blockIdx.z, nseg = a.gseg;
  const int tid = threadIdx.x;
  const int N = a.N, T = a.T, F = a.F;
  const size_t FT = (size_t)F * T;
  const int ta = seg * a.TR, tb = min(T, ta + a.TR);
  const R fl = a.floorp[b];
  const R* lamb = a.lam + (size_t)b * N * FT + (size_t)f * T;
  const C* Xb = a.X + ((size_t)b * F + f) * T * M;
  if constexpr (MP != M) {  // odd M: the pad column stays zero (never copied into)
    for (int t = tid; t < 2 * TB; t += BS) Xraw[t * MP + M] = make_float2(0.f, 0.f);
  }
  // chunk c0 -> buffer q: cp.async of the X rows and lambda; frames past the
  // segment re-read the last valid frame (finite data, weight 0 below)
  auto stage = [&](int c0, int q) {
    C* xd = Xraw + q * TB * MP;
    if constexpr (M % 2 == 0) {
      for (int e = tid; e < TB * (M / 2); e += BS) {
        const int t = e / (M / 2), k = e % (M / 2);
        const int tc = min(c0 + t, tb - 1);
        cp_async16(xd + t * MP + 2 * k, Xb + (size_t)tc * M + 2 * k, true);
      }
    } else {
      for (int e = tid; e < TB * M; e += BS) {
        const int t = e / M, k = e % M;
        const int tc = min(c0 + t, tb - 1);
        cp_async8(xd + t * MP + k, Xb + (size_t)tc * M + k);
      }
    }
    R* ld = Lraw + q * NMAX * TB;
    for (int e = tid; e < N * TB; e += BS) {
      const int n = e / TB, t = e % TB;
      const int tc = min(c0 + t, tb - 1);
      cp_async4(ld + n * TB + t, lamb + (size_t)n * FT + tc);
    }
    cp_async_commit();
  };
  stage(ta, 0);
  // finish the gain MU from the k_gain segment partials (fixed order)
  for (int e = tid; e < N * M; e += BS) {
    const int n = e / M, m = e % M;
    const R* gp = a.gpart + ((size_t)b * F + f) * nseg * N * 2 * M + n * 2 * M;
    R sn = 0, sd = 0;
    for (int q = 0; q < nseg; ++q) {
      sn += gp[(size_t)q * N * 2 * M + m];
      sd += gp[(size_t)q * N * 2 * M + M + m];
    }
    const size_t gi = (size_t)b * N * F * M + (size_t)n * F * M + (size_t)f * M + m;
    const R gv = a.g[gi] * mu_factor(sn, sd);
    gs[e] = gv;
    if (blockIdx.x == 0) a.gnew[gi] = gv;
  }
  // thread -> (frame slice s, m-half h, 2x2 block (I, J))
  const int s = tid / TPS, r = tid % TPS;
  const int h = r / NB, bk = r % NB;
  int I = 0, J = bk;
  while (J >= NBK - I) {
    J -= NBK - I;
    ++I;
  }
  J += I;
  const bool act = s < S;
  float2 v[4][MH];
#pragma unroll
  for (int e = 0; e < 4; ++e)
#pragma unroll
    for (int m = 0; m < MH; ++m) v[e][m] = make_float2(0.f, 0.f);
  int q = 0;
  for (int c0 = ta; c0 < tb; c0 += TB, q ^= 1) {
    cp_async_wait<0>();
    __syncthreads();  // chunk c0 landed; every thread is done with the previous chunk
    if (c0 + TB < tb) stage(c0 + TB, q ^ 1);
    for (int t = tid; t < TB; t += BS) {
      R l[NMAX];
#pragma unroll
      for (int n = 0; n < NMAX; ++n) l[n] = (n < N) ? Lraw[q * NMAX * TB + n * TB + t] : R(0);
      R iy[M], y[M];
      model_power<R, M>(l, gs, N, fl, iy, y);
      const bool tv = c0 + t < tb;
      R* ir = iys + t * IW;
#pragma unroll
      for (int m = 0; m < IW; ++m) ir[m] = (m < M && tv) ? iy[m < M ? m : 0] : R(0);
    }
    __syncthreads();
    if (act) {
      const C* Xc = Xraw + q * TB * MP;
#pragma unroll 2
      for (int tl = s; tl < TB; tl += S) {
        const float4 xi = *reinterpret_cast<const float4*>(Xc + tl * MP + 2 * I);
        const float4 xj = *reinterpret_cast<const float4*>(Xc + tl * MP + 2 * J);
        R w[MH];
        lds_row<MH>(iys + tl * IW + h * MH, w);
        // x_i conj(x_j) for (i, j) in {2I, 2I+1} x {2J, 2J+1}, packed:
        // (a.x b.x + a.y b.y, a.y b.x - a.x b.y) = (a.x, a.y) b.x + (a.y, -a.x) b.y
        const float2 i0 = make_float2(xi.x, xi.y), i1 = make_float2(xi.z, xi.w);
        const float2 r0 = make_float2(xi.y, -xi.x), r1 = make_float2(xi.w, -xi.z);
        const float2 z = make_float2(0.f, 0.f);
        float2 p[4];
        p[0] = fma2(r0, make_float2(xj.y, xj.y), fma2(i0, make_float2(xj.x, xj.x), z));
        p[1] = fma2(r0, make_float2(xj.w, xj.w), fma2(i0, make_float2(xj.z, xj.z), z));
        p[2] = fma2(r1, make_float2(xj.y, xj.y), fma2(i1, make_float2(xj.x, xj.x), z));
        p[3] = fma2(r1, make_float2(xj.w, xj.w), fma2(i1, make_float2(xj.z, xj.z), z));
#pragma unroll
        for (int m = 0; m < MH; ++m) {
          const float2 wm = make_float2(w[m], w[m]);
#pragma unroll
          for (int e = 0; e < 4; ++e) v[e][m] = fma2(wm, p[e], v[e][m]);
        }
      }
    }
  }
  __syncthreads();
  // fixed-order tree over the slices, CV floats at a time (staging area reused)
  R* slot = reinterpret_cast<R*>(vb_smem);
#pragma unroll
  for (int c = 0; c < NV; c += CV) {
    for (int wdt = 1; wdt < S; wdt *= 2) {
      if (act && (s % (2 * wdt)) == wdt) {
        R* d = slot + ((size_t)(s / (2 * wdt)) * TPS + r) * CV;
#pragma unroll
        for (int k = 0; k < CV; ++k) {
          const int q = c + k, e = q / (2 * MH), m = (q / 2) % MH;
          d[k] = (q & 1) ? v[e][m].y : v[e][m].x;
        }
      }
      __syncthreads();
      if (act && (s % (2 * wdt)) == 0 && s + wdt < S) {
        const R* d = slot + ((size_t)(s / (2 * wdt)) * TPS + r) * CV;
#pragma unroll
        for (int k = 0; k < CV; ++k) {
          const int q = c + k, e = q / (2 * MH), m = (q / 2) % MH;
          if (q & 1) v[e][m].y += d[k]; else v[e][m].x += d[k];
        }
      }
      __syncthreads();
    }
  }
  if (s == 0) {
    C* pb = reinterpret_cast<C*>(a.part) + (((size_t)b * F + f) * gridDim.x + seg) * M * P;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int i = 2 * I + (e >> 1), j = 2 * J + (e & 1);
      if (i <= j && j < M) {
        const int pij = i * M - i * (i - 1) / 2 + (j - i);
#pragma unroll
        for (int m = 0; m < MH; ++m) {
          const int mm = h * MH + m;
          if (mm < M) pb[mm * P + pij] = v[e][m];
        }
      }
    }
  }
}

}  // namespace fm
