// fm_spatial.cuh -- the per-frequency part of the FastMNMF iteration.
//
// k_gain / k_vacc ((bin, frame-segment) CTAs): gain statistics + g MU
//   (separate.py:217-220; _kernels.py:244-250) and the weighted covariances
//   V_fm = (1/T) sum_t x x^H / y_ftm from the floored model power with the new
//   gains (separate.py:221-222, spatial.py:182, _kernels.py:276-293).
// k_ip (one small CTA per (f, b)): the iterative-projection row updates
//   (spatial.py:181-199), row normalisation (separate.py:223-229), log|det Q|
//   (separate.py:236-238) and the gain normalisation folded into W
//   (separate.py:231-233, spatial.py:244-249, sources.py:202-204).
//
//   IP formulation. The reference solves (Q V_m) q = e_m with LAPACK for each
//   row m. Here q = V_m^-1 (Q^-1 e_m): the M HPD inverses V_m^-1 are formed in
//   parallel (one warp each, Gauss-Jordan), Q^-1 once per iteration
//   (pivoted Gauss-Jordan, which also yields log|det Q|), and each row update
//   Q <- Q + e_m (r - Q_m) is applied to Q^-1 by Sherman-Morrison with
//   denominator r.u = sqrt(q^H u) = sqrt(norm); norm = q^H V q = q^H u. The
//   determinant lemma gives log|det Q| += log sqrt(norm) per row, minus
//   log(row norm) per normalised row. Same mathematics, identical to the
//   reference to ~1e-15 in fp64 (checked against its outputs in
//   tests/test_gpu_ops.py); the sequential part per row is one mat-vec.
//
// k_back (one CTA per (f, b)): projection x~ = |Q x|^2 (separate.py:230;
//   _kernels.py:339-350) fused with the NEXT iteration's first statistics
//   pass (separate.py:186-193; _kernels.py:226-243): log-likelihood data term
//   and phi1/phi2 (written for k_wupdate), plus the fixed-order last-block
//   reduction of the trace entry.
#pragma once
#include "fm_common.cuh"
#include "fm_linalg.cuh"
#include "fm_nmf.cuh"

namespace fm {

// packed FMA on (x, y) pairs: FFMA2 on sm_100a (fma.rn.f32x2), two FMAs otherwise
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
  unsigned long long ra = *reinterpret_cast<unsigned long long*>(&a);
  unsigned long long rb = *reinterpret_cast<unsigned long long*>(&b);
  unsigned long long rc = *reinterpret_cast<unsigned long long*>(&c);
  unsigned long long rd;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(rd) : "l"(ra), "l"(rb), "l"(rc));
  return *reinterpret_cast<float2*>(&rd);
}
__device__ __forceinline__ double2 fma2(double2 a, double2 b, double2 c) {
  return make_double2(fma(a.x, b.x, c.x), fma(a.y, b.y, c.y));
}

// ---------------------------------------------------------------------------
// k_gain and k_vacc split the (f, t) plane into (bin, frame-segment) CTAs --
// grid (ceil(T/TR), F, B) -- that stream their segment in TB-frame chunks
// (register prefetch of the next chunk) and write fixed-order partial T-sums
// per segment. The consumer reduces the segments in order (deterministic):
// k_vacc finishes the g MU from the gain partials, k_ip finishes V_f.
// ---------------------------------------------------------------------------
template <typename R> struct GainArgs {
  const R* xt;
  const R* lam;
  const R* g;
  const R* floorp;
  R* part;  // (B, F, nseg, N, 2M)
  int F, T, N, TR;
};

template <typename R, int M> struct GaCfg {
  static constexpr int TB = (sizeof(R) == 4) ? 256 : 128;  // frames per chunk (smem bound)
  // weights per accumulating thread: 4 (16-B shared loads of the staged rows)
  // when M % 4 == 0 and M >= 8, else 1 (measured: c3 M = 16 660 -> 490 us,
  // c1 M = 8 unchanged, c2 M = 4 917 -> 956 us with 4)
  static constexpr int MQ = (M % 4 == 0 && M >= 8) ? 4 : 1;
  // source pairs per accumulating thread (fp32, MQ = 4, even N): 2x the slices
  static constexpr bool PAIRS = sizeof(R) == 4 && MQ == 4;
  static constexpr int RED = (PAIRS ? 1024 : 512) * MQ;  // >= slices x N x M x 2 partial sums
  // staged row stride: fp32 rows of M = 8 floats are padded by 4 (an odd
  // number of 16-byte words) so the frame-per-thread 16-byte stores
  // do not collide; the lambda rows by 8 so the (source, slice) loads of a
  // warp fall into distinct banks
  static constexpr int RS = M + ((sizeof(R) == 4 && M == 8) ? 4 : 0);
  static constexpr int LS = TB + ((sizeof(R) == 4 && M <= 8) ? 8 : 1);
  static constexpr bool ALIAS = RED <= 2 * TB * RS;  // reduction reuses the staged rows
};

// gain statistics (separate.py:217; _kernels.py:244-250)
template <typename R, int M>
__global__ void __launch_bounds__(256) k_gain(GainArgs<R> a) {
  pdl_entry();
  using Cf = GaCfg<R, M>;
  constexpr int TB = Cf::TB, MQ = Cf::MQ, RS = Cf::RS, LS = Cf::LS;
  __shared__ __align__(16) R lams[NMAX * LS];
  __shared__ __align__(16) R stage[2 * TB * RS];  // [TB][M] 1/y | [TB][M] x~/y^2
  __shared__ __align__(16) R gs[NMAX * M];
  __shared__ __align__(16) R redx[Cf::ALIAS ? 1 : Cf::RED];
  R* iys = stage;
  R* xrs = stage + TB * RS;
  R* redb = Cf::ALIAS ? stage : redx;
  const int seg = blockIdx.x, f = blockIdx.y, b = blockIdx.z, nseg = gridDim.x;
  const int tid = threadIdx.x;
  const int N = a.N, T = a.T, F = a.F;
  const size_t FT = (size_t)F * T;
  const int ta = seg * a.TR, tb = min(T, ta + a.TR);
  const R fl = a.floorp[b];
  const R* lamb = a.lam + (size_t)b * N * FT + (size_t)f * T;
  const R* xtb = a.xt + ((size_t)b * F + f) * T * M;
  R lp[NMAX], xp[M];
  auto fetch = [&](int c0) {
    const int t = c0 + tid;
    const int tc = t < tb ? t : tb - 1;
#pragma unroll
    for (int n = 0; n < NMAX; ++n) {
      lp[n] = R(0);
      if (n >= N) break;
      lp[n] = lamb[(size_t)n * FT + tc];
    }
    RowIO<R, M>::load(xtb + (size_t)tc * M, xp);
  };
  // M <= 8: the first chunk is in flight before the gains are staged (one
  // round trip, not two); M = 16 keeps the fetch behind them (c3: the 24
  // prefetched values held across the staging cost more than they save)
  if (M <= 8 && tid < TB) fetch(ta);
  for (int e = tid; e < N * M; e += 256)
    gs[e] = a.g[(size_t)b * N * F * M + (size_t)(e / M) * F * M + (size_t)f * M + (e % M)];
  if (M > 8 && tid < TB) fetch(ta);
  // accumulate mapping: thread = (NP sources from n1, MQ consecutive
  // channels, slice); with MQ = 4 and N even a thread takes a source pair, so
  // one pair of 16-B loads of x~/y^2 and 1/y feeds 16 FMAs (c3: the loop was
  // shared-memory bound, 90% of the pipe)
  constexpr int Q = M / MQ;
  // (only when enough items remain that the slice reduction stays short:
  // c3 k_gain 489 -> 418 us; c1, 4 pair items, 18.4 -> 20.5 us, so not there)
  const int NP = (Cf::PAIRS && (N % 2) == 0 && (N / 2) * Q >= 8) ? 2 : 1;
  const int E = (N / NP) * Q, S = 256 / E;
  const int e1 = tid % E, s1 = tid / E;
  const int n1 = (e1 / Q) * NP, m0 = (e1 % Q) * MQ;
  R num[2][MQ], den[2][MQ];
#pragma unroll
  for (int k = 0; k < MQ; ++k) num[0][k] = den[0][k] = num[1][k] = den[1][k] = R(0);
  __syncthreads();
  for (int c0 = ta; c0 < tb; c0 += TB) {
    if (tid < TB) {
      const bool tv = c0 + tid < tb;
      R l[NMAX], x[M];
#pragma unroll
      for (int n = 0; n < NMAX; ++n) l[n] = tv ? lp[n] : R(0);
#pragma unroll
      for (int m = 0; m < M; ++m) x[m] = xp[m];
      if (c0 + TB < tb) fetch(c0 + TB);
      R iy[M], y[M], xr[M];
      model_power<R, M>(l, gs, N, fl, iy, y);
#pragma unroll
      for (int m = 0; m < M; ++m) {
        if (!tv) iy[m] = R(0);
        xr[m] = x[m] * iy[m] * iy[m];
      }
      RowIO<R, M>::store(iys + tid * RS, iy);
      RowIO<R, M>::store(xrs + tid * RS, xr);
#pragma unroll
      for (int n = 0; n < NMAX; ++n) {
        if (n >= N) break;
        lams[n * LS + tid] = l[n];
      }
    }
    __syncthreads();
    if (s1 < S) {
      if (NP == 2) {
        for (int tl = s1; tl < TB; tl += S) {
          const R lv0 = lams[n1 * LS + tl], lv1 = lams[(n1 + 1) * LS + tl];
          R xv[MQ], iv[MQ];
          if constexpr (MQ == 4) {
            lds4(xrs + tl * RS + m0, xv);
            lds4(iys + tl * RS + m0, iv);
          } else {
            xv[0] = xrs[tl * RS + m0];
            iv[0] = iys[tl * RS + m0];
          }
#pragma unroll
          for (int k = 0; k < MQ; ++k) {
            num[0][k] += lv0 * xv[k];
            den[0][k] += lv0 * iv[k];
            num[1][k] += lv1 * xv[k];
            den[1][k] += lv1 * iv[k];
          }
        }
      } else {
        for (int tl = s1; tl < TB; tl += S) {
          const R lv = lams[n1 * LS + tl];
          R xv[MQ], iv[MQ];
          if constexpr (MQ == 4) {
            lds4(xrs + tl * RS + m0, xv);
            lds4(iys + tl * RS + m0, iv);
          } else {
            xv[0] = xrs[tl * RS + m0];
            iv[0] = iys[tl * RS + m0];
          }
#pragma unroll
          for (int k = 0; k < MQ; ++k) {
            num[0][k] += lv * xv[k];
            den[0][k] += lv * iv[k];
          }
        }
      }
    }
    __syncthreads();
  }
  // fixed-order slice sums: partial (slice, n, m) pairs, then one thread per (n, m)
  if (s1 < S) {
    for (int pp = 0; pp < NP; ++pp) {
#pragma unroll
      for (int k = 0; k < MQ; ++k) {
        const int en = (n1 + pp) * M + m0 + k;
        redb[(s1 * N * M + en) * 2] = num[pp][k];
        redb[(s1 * N * M + en) * 2 + 1] = den[pp][k];
      }
    }
  }
  __syncthreads();
  if (tid < N * M) {
    R vn = 0, vd = 0;
    for (int q = 0; q < S; ++q) {
      vn += redb[(q * N * M + tid) * 2];
      vd += redb[(q * N * M + tid) * 2 + 1];
    }
    const int nn = tid / M, mm = tid % M;
    R* pb = a.part + (((size_t)b * F + f) * nseg + seg) * N * 2 * M;
    pb[nn * 2 * M + mm] = vn;
    pb[nn * 2 * M + M + mm] = vd;
  }
}

template <typename R, int M> struct VaCfg {
  static constexpr int BS = (M <= 8) ? 256 : 512;
  static constexpr int P = M * (M + 1) / 2;
  static constexpr int S2 = BS / P;
  // staged row strides (elements). fp32 with M % 4 == 0 pads the 1/y row to
  // M + 4 floats and the x row to M + 2 complex: 3 and 5 (odd) 16-byte words,
  // so the frame-per-thread 16-byte stores of phase A are conflict-free
  // (unpadded 32- / 64-byte rows: 8 and 16 wavefronts per store instead of 4,
  // a quarter of the kernel's shared-memory wavefronts at config 1)
  static constexpr bool PAD = sizeof(R) == 4 && M % 4 == 0;
  static constexpr int IYS = M + (PAD ? 4 : 0), XCS = M + (PAD ? 2 : 0);
  // frames per chunk: the staged (x, 1/y) rows must fit ~36 KB of static smem
  static constexpr int ROWB = (IYS + 2 * XCS) * (int)sizeof(R);
  static constexpr int TB = (256 * ROWB <= 36864) ? 256 : (128 * ROWB <= 36864) ? 128 : 64;
  static constexpr int STAGEB = TB * ROWB;
  // fp32, M = 6..8: cap registers for 3 CTAs (24 warps) per SM -- the pair loop is
  // shared-load latency bound, not issue bound
  static constexpr int MINB = (sizeof(R) == 4 && M >= 6 && M <= 8) ? 3 : 1;
  static constexpr bool ONEPASS = S2 * M * P * (int)(2 * sizeof(R)) <= STAGEB;
};

template <typename R> struct VaccArgs {
  const cplx<R>* X;
  const R* lam;
  const R* g;      // gains before this iteration's MU
  const R* gpart;  // k_gain partials (B, F, nseg, N, 2M)
  const R* floorp;
  R* gnew;         // (B, N, F, M) gains after the MU (written by segment 0)
  R* part;         // (B, F, nseg, M, P) complex partial V sums
  int F, T, N, TR;
  int gseg;        // k_gain segments per bin (k_vacc_blk's own segmentation may differ)
  int dbg;         // timing experiments only (k_vacc_tc), bits: 1 skip MMAs, 2 skip operand builds, 4 one MMA of three
};

// g MU (separate.py:218-220) + V_fm = (1/T) sum_t x x^H / y_ftm with y from
// the updated gains (separate.py:221-222; spatial.py:182; _kernels.py:276-293)
template <typename R, int M>
__global__ void __launch_bounds__(VaCfg<R, M>::BS, VaCfg<R, M>::MINB) k_vacc(VaccArgs<R> a) {
  pdl_entry();
  using C = cplx<R>;
  using Cf = VaCfg<R, M>;
  constexpr int BS = Cf::BS, TB = Cf::TB, P = Cf::P, S2 = Cf::S2, IYS = Cf::IYS, XCS = Cf::XCS;
  constexpr int BUFB = (Cf::STAGEB > M * P * (int)sizeof(C)) ? Cf::STAGEB : M * P * (int)sizeof(C);
  __shared__ __align__(16) unsigned char buf[BUFB];
  R* iys = reinterpret_cast<R*>(buf);
  C* Xc = reinterpret_cast<C*>(buf + TB * IYS * sizeof(R));
  __shared__ __align__(16) R gs[NMAX * M];
  __shared__ int pairs[2 * P];
  const int seg = blockIdx.x, f = blockIdx.y, b = blockIdx.z, nseg = gridDim.x;
  const int tid = threadIdx.x;
  const int N = a.N, T = a.T, F = a.F;
  const size_t FT = (size_t)F * T;
  const int ta = seg * a.TR, tb = min(T, ta + a.TR);
  const R fl = a.floorp[b];
  const R* lamb = a.lam + (size_t)b * N * FT + (size_t)f * T;
  const C* Xb = a.X + ((size_t)b * F + f) * T * M;
  R lp[NMAX];
  C xp[M];
  auto fetch = [&](int c0) {
    const int t = c0 + tid;
    const int tc = t < tb ? t : tb - 1;
#pragma unroll
    for (int n = 0; n < NMAX; ++n) {
      lp[n] = R(0);
      if (n >= N) break;
      lp[n] = lamb[(size_t)n * FT + tc];
    }
    CRowIO<R, M>::load(Xb + (size_t)tc * M, xp);
  };
  if (tid < TB) fetch(ta);  // in flight while the gains are finished (one round trip, not two)
  // finish the gain MU from the k_gain segment partials (fixed order)
  for (int e = tid; e < N * M; e += BS) {
    const int n = e / M, m = e % M;
    const R* gp = a.gpart + ((size_t)b * F + f) * a.gseg * N * 2 * M + n * 2 * M;
    R sn = 0, sd = 0;
    for (int q = 0; q < a.gseg; ++q) {
      sn += gp[(size_t)q * N * 2 * M + m];
      sd += gp[(size_t)q * N * 2 * M + M + m];
    }
    const size_t gi = (size_t)b * N * F * M + (size_t)n * F * M + (size_t)f * M + m;
    const R gv = a.g[gi] * mu_factor(sn, sd);
    gs[e] = gv;
    if (seg == 0) a.gnew[gi] = gv;
  }
  if (tid < P) {
    int i = 0, r = tid;
    while (r >= M - i) {
      r -= M - i;
      ++i;
    }
    pairs[2 * tid] = i;
    pairs[2 * tid + 1] = i + r;
  }
  __syncthreads();
  const int p = tid % P, s2 = tid / P;
  const bool act = s2 < S2;
  const int pi = pairs[2 * p], pj = pairs[2 * p + 1];
  C v[M];
#pragma unroll
  for (int m = 0; m < M; ++m) v[m] = cmake<C>(0.0, 0.0);
  constexpr bool PACKW = sizeof(R) == 4 && M % 4 == 0;
  float2 ar[PACKW ? M / 2 : 1], ai[PACKW ? M / 2 : 1];
#pragma unroll
  for (int h = 0; h < (PACKW ? M / 2 : 1); ++h) ar[h] = ai[h] = make_float2(0.f, 0.f);
  for (int c0 = ta; c0 < tb; c0 += TB) {
    if (tid < TB) {
      const bool tv = c0 + tid < tb;
      R l[NMAX];
      C xv[M];
#pragma unroll
      for (int n = 0; n < NMAX; ++n) l[n] = lp[n];
#pragma unroll
      for (int m = 0; m < M; ++m) xv[m] = tv ? xp[m] : cmake<C>(0.0, 0.0);
      if (c0 + TB < tb) fetch(c0 + TB);
      R iy[M], y[M];
      model_power<R, M>(l, gs, N, fl, iy, y);
#pragma unroll
      for (int m = 0; m < M; ++m)
        if (!tv) iy[m] = R(0);
      RowIO<R, M>::store(iys + tid * IYS, iy);
      CRowIO<R, M>::store(Xc + tid * XCS, xv);
    }
    __syncthreads();
    if constexpr (PACKW) {
      // fp32, M % 4 == 0: the accumulators pack two WEIGHTS per FFMA2
      // (re and im parts apart), so the 1/y pairs are the 16-B shared loads'
      // own register pairs and only (p.x, p.x), (p.y, p.y) are formed per
      // frame -- the (1/y, 1/y) operand of the re/im packing costs a MOV per
      // FFMA2; two frames per trip, their FFMA2 groups not interleaved
      if (act) {
        auto frame = [&](const C xi, const C xj, const float (&iy)[M]) {
          const float px = xi.x * xj.x + xi.y * xj.y;  // x_i conj(x_j)
          const float py = xi.y * xj.x - xi.x * xj.y;
          const float2 pxx = make_float2(px, px), pyy = make_float2(py, py);
#pragma unroll
          for (int h = 0; h < M / 2; ++h) {
            const float2 w = make_float2(iy[2 * h], iy[2 * h + 1]);
            ar[h] = fma2(w, pxx, ar[h]);
            ai[h] = fma2(w, pyy, ai[h]);
          }
        };
        int tl = s2;
        for (; tl + S2 < TB; tl += 2 * S2) {
          const C xi0 = Xc[tl * XCS + pi], xj0 = Xc[tl * XCS + pj];
          const C xi1 = Xc[(tl + S2) * XCS + pi], xj1 = Xc[(tl + S2) * XCS + pj];
          float iy0[M], iy1[M];
          RowIO<float, M>::load(reinterpret_cast<const float*>(iys) + tl * IYS, iy0);
          RowIO<float, M>::load(reinterpret_cast<const float*>(iys) + (tl + S2) * IYS, iy1);
          frame(xi0, xj0, iy0);
          frame(xi1, xj1, iy1);
        }
        if (tl < TB) {
          const C xi = Xc[tl * XCS + pi], xj = Xc[tl * XCS + pj];
          float iy[M];
          RowIO<float, M>::load(reinterpret_cast<const float*>(iys) + tl * IYS, iy);
          frame(xi, xj, iy);
        }
      }
    } else
    if (act) {
      int tl = s2;
      for (; tl + S2 < TB; tl += 2 * S2) {
        const C xi0 = Xc[tl * XCS + pi], xj0 = Xc[tl * XCS + pj];
        const C xi1 = Xc[(tl + S2) * XCS + pi], xj1 = Xc[(tl + S2) * XCS + pj];
        R iy0[M], iy1[M];
        RowIO<R, M>::load(iys + tl * IYS, iy0);
        RowIO<R, M>::load(iys + (tl + S2) * IYS, iy1);
        C p0, p1;  // x_i conj(x_j)
        p0.x = xi0.x * xj0.x + xi0.y * xj0.y;
        p0.y = xi0.y * xj0.x - xi0.x * xj0.y;
        p1.x = xi1.x * xj1.x + xi1.y * xj1.y;
        p1.y = xi1.y * xj1.x - xi1.x * xj1.y;
#pragma unroll
        for (int m = 0; m < M; ++m) {
          v[m] = fma2(cmake<C>(iy0[m], iy0[m]), p0, v[m]);
          v[m] = fma2(cmake<C>(iy1[m], iy1[m]), p1, v[m]);
        }
      }
      if (tl < TB) {
        const C xi = Xc[tl * XCS + pi], xj = Xc[tl * XCS + pj];
        C pr;
        pr.x = xi.x * xj.x + xi.y * xj.y;
        pr.y = xi.y * xj.x - xi.x * xj.y;
        R iy[M];
        RowIO<R, M>::load(iys + tl * IYS, iy);
#pragma unroll
        for (int m = 0; m < M; ++m) v[m] = fma2(cmake<C>(iy[m], iy[m]), pr, v[m]);
      }
    }
    __syncthreads();
  }
  if constexpr (PACKW) {
#pragma unroll
    for (int h = 0; h < M / 2; ++h) {
      v[2 * h] = cmake<C>(ar[h].x, ai[h].x);
      v[2 * h + 1] = cmake<C>(ar[h].y, ai[h].y);
    }
  }
  // fixed-order slice reduction (staging area reused), then the segment partial
  C* red = reinterpret_cast<C*>(buf);
  C* pb = reinterpret_cast<C*>(a.part) + (((size_t)b * F + f) * nseg + seg) * M * P;
  if constexpr (Cf::ONEPASS) {
    if (act) {
#pragma unroll
      for (int m = 0; m < M; ++m) red[(s2 * M + m) * P + p] = v[m];
    }
    __syncthreads();
    for (int e = tid; e < M * P; e += BS) {
      C acc = red[e];
      for (int q = 1; q < S2; ++q) {
        const C o = red[q * M * P + e];
        acc.x += o.x;
        acc.y += o.y;
      }
      pb[e] = acc;
    }
  } else {
    for (int ss = 0; ss < S2; ++ss) {
      if (act && s2 == ss) {
#pragma unroll
        for (int m = 0; m < M; ++m) {
          C* d = red + m * P + p;
          if (ss == 0) {
            *d = v[m];
          } else {
            C o = *d;
            o.x += v[m].x;
            o.y += v[m].y;
            *d = o;
          }
        }
      }
      __syncthreads();
    }
    for (int e = tid; e < M * P; e += BS) pb[e] = red[e];
  }
}

// ---------------------------------------------------------------------------
// k_ip: iterative projection + normalisations, one small CTA per (f, b):
// warp 0 inverts [Q | I] (pivoted Gauss-Jordan; also log|det Q|) while warps
// 1.. invert the HPD V_fm in parallel; warp 0 then runs the M sequential row
// updates (one mat-vec each); all threads normalise and fold into W.
// ---------------------------------------------------------------------------
template <typename R> struct IpArgs {
  const cplx<R>* Vpart;  // (B, F, nseg, M, P) partial V sums from k_vacc
  int nseg, T;
  const R* gnew;         // (B, N, F, M) gains after the MU (k_vacc)
  cplx<R>* Q;
  R* g;
  R* W;
  const R* Wsrc;  // W before the absorb (== W: in place; else W = Wsrc c)
  R* cs_out;
  double* ld_part;
  const unsigned* iter;
  unsigned long long* status;
  R* u;    // deep-prior scale u (B, F) when n0 == 1 (absorbs c[0], sources.py:269-271)
  int n0;  // first NMF source (0, or 1 for FastMNMF-DP)
  int F, N, K;
  long long f_offset;
  int normalize, ip_sweeps;
  int B;  // mixtures (k_ip_w's flat (mixture, bin) grid)
};

template <int M> struct IpCfg {
  static constexpr int NW = (M < 8 ? M : 8) + 1;  // warp 0 + HPD-inversion warps
  static constexpr int BS = 32 * NW;
};

template <typename R, int M> struct IpSmem {
  static constexpr size_t al(size_t x) { return (x + 15) & ~size_t(15); }
  static constexpr size_t o_Vd = 0;
  static constexpr size_t o_Qd = o_Vd + al(sizeof(double2) * M * M * M);
  static constexpr size_t o_Ai = o_Qd + al(sizeof(double2) * M * M);
  static constexpr size_t o_vec = o_Ai + al(sizeof(double2) * M * 2 * M);
  static constexpr size_t o_gs = o_vec + al(sizeof(double2) * 3 * M);
  static constexpr size_t o_cs = o_gs + al(sizeof(R) * NMAX * M);
  static constexpr size_t o_rown = o_cs + al(sizeof(R) * NMAX);
  static constexpr size_t o_misc = o_rown + al(sizeof(double) * M);
  static constexpr size_t bytes = o_misc + al(sizeof(double) * 8 + sizeof(int) * (M + 8));
};

template <typename R, int M>
__global__ void __launch_bounds__(IpCfg<M>::BS) k_ip(IpArgs<R> a) {
  pdl_entry();
  using C = cplx<R>;
  using L = IpSmem<R, M>;
  // complex64 at M <= 8: the whole IP (Q inverse, V inverses, row updates,
  // normalisation) in fp32 -- the reference is fp64, but the fp32-accumulated
  // V already bounds the accuracy there (parity: profiles/parity_r2.json);
  // the log-determinant still accumulates in fp64. Otherwise fp64.
  constexpr bool F32 = sizeof(R) == 4 && M <= 8;
  using C2 = typename std::conditional<F32, float2, double2>::type;
  using Rc = typename std::conditional<F32, float, double>::type;
  constexpr int NW = IpCfg<M>::NW, BS = IpCfg<M>::BS;
  extern __shared__ __align__(16) unsigned char sm[];
  double2* Vd = reinterpret_cast<double2*>(sm + L::o_Vd);
  C2* Qd = reinterpret_cast<C2*>(sm + L::o_Qd);
  C2* Ai = reinterpret_cast<C2*>(sm + L::o_Ai);
  C2* ub = reinterpret_cast<C2*>(sm + L::o_vec);
  C2* qb = ub + M;
  C2* sk = qb + M;
  R* gs = reinterpret_cast<R*>(sm + L::o_gs);
  R* cs = reinterpret_cast<R*>(sm + L::o_cs);
  double* rown = reinterpret_cast<double*>(sm + L::o_rown);
  double* misc = reinterpret_cast<double*>(sm + L::o_misc);
  int* vfail = reinterpret_cast<int*>(misc + 8);
  int* flags = vfail + M;
  const int f = blockIdx.x, b = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int N = a.N, F = a.F, K = a.K;
  C* Qg = a.Q + ((size_t)b * F + f) * M * M;
  R* gg = a.g + (size_t)b * N * F * M + (size_t)f * M;
  R* Wg = a.W + (size_t)b * (N - a.n0) * F * K + (size_t)f * K;
  const R* Wsg = a.Wsrc + (size_t)b * (N - a.n0) * F * K + (size_t)f * K;
  const unsigned it = *a.iter;
  const long long fglob = a.f_offset + f;
  // Q and the updated gains go to registers before the V partials are summed
  // (their loads are in flight during that loop: one global round trip before
  // the first barrier, not two)
  constexpr bool PRE = M * M <= BS && NMAX * M <= BS;
  C qreg = cmake<C>(0.0, 0.0);
  R gnreg = R(0);
  if constexpr (PRE) {
    if (tid < M * M) qreg = Qg[tid];
    if (tid < N * M)
      gnreg = a.gnew[(size_t)b * N * F * M + (size_t)(tid / M) * F * M + (size_t)f * M + (tid % M)];
  }
  {  // V_f = (1/T) sum over the segment partials (fixed order, fp64), mirrored
    constexpr int P = M * (M + 1) / 2;
    const C* vp = a.Vpart + ((size_t)b * F + f) * a.nseg * M * P;
    const double invT = 1.0 / (double)a.T;
    for (int e = tid; e < M * P; e += BS) {
      double2 acc = make_double2(0.0, 0.0);
      for (int q = 0; q < a.nseg; ++q) {
        const C c = vp[(size_t)q * M * P + e];
        acc.x += (double)c.x;
        acc.y += (double)c.y;
      }
      const int m = e / P;
      int i = 0, r = e % P;
      while (r >= M - i) {
        r -= M - i;
        ++i;
      }
      const int j = i + r;
      const double2 d = make_double2(acc.x * invT, acc.y * invT);
      Vd[((size_t)m * M + i) * M + j] = d;
      if (i != j) Vd[((size_t)m * M + j) * M + i] = make_double2(d.x, -d.y);
    }
  }
  if constexpr (PRE) {
    if (tid < M * M) Qd[tid] = to_c2(qreg, C2());
    if (tid < N * M) gs[tid] = gnreg;
  } else {
    for (int e = tid; e < M * M; e += BS) Qd[e] = to_c2(Qg[e], C2());
    for (int e = tid; e < N * M; e += BS)
      gs[e] = a.gnew[(size_t)b * N * F * M + (size_t)(e / M) * F * M + (size_t)f * M + (e % M)];
  }
  if (tid < NMAX) cs[tid] = R(1);
  if (tid == 0) flags[0] = flags[1] = 0;
  __syncthreads();
  // ---- A3: iterative projection (spatial.py:181-199) -------------------------
  {
    if (warp == 0) {
      // [Q | I] -> Q^-1 and log|det Q|
      for (int e = lane; e < M * 2 * M; e += 32) {
        const int r = e / (2 * M), c = e % (2 * M);
        Ai[e] = c < M ? Qd[r * M + c] : to_c2(make_double2(c - M == r ? 1.0 : 0.0, 0.0), C2());
      }
      __syncwarp();
      double la = 0.0;
      const bool ok = warp_inv_pivot<M, C2, true>(Ai, lane, &la);
      if (lane == 0) {
        misc[0] = la;
        flags[0] = ok ? 0 : 1;
      }
    }
    for (int m = warp - 1; warp > 0 && m < M; m += NW - 1) {
      double2* Vm = Vd + (size_t)m * M * M;
      bool ok;
      if constexpr (sizeof(R) == 4 && M <= 8) {  // complex64: invert in fp32 in place
        constexpr int NE = (M * M + 31) / 32;
        float2 tv[NE];
#pragma unroll
        for (int r = 0; r < NE; ++r) {
          const int e = lane + 32 * r;
          if (e < M * M) tv[r] = make_float2((float)Vm[e].x, (float)Vm[e].y);
        }
        __syncwarp();
        float2* Vf = reinterpret_cast<float2*>(Vm);
#pragma unroll
        for (int r = 0; r < NE; ++r) {
          const int e = lane + 32 * r;
          if (e < M * M) Vf[e] = tv[r];
        }
        __syncwarp();
        ok = warp_inv_hpd_f32<M>(Vf, lane);  // stays fp32 in place (the F32 row updates read it)
        if (!ok) {
          // an fp32 pivot that is not positive (ill-conditioned V_m): rebuild
          // V_m in fp64 from the partials and retry before the reference's
          // error is raised
          constexpr int P = M * (M + 1) / 2;
          const C* vp = a.Vpart + ((size_t)b * F + f) * a.nseg * M * P + (size_t)m * P;
          for (int e = lane; e < P; e += 32) {
            double2 acc = make_double2(0.0, 0.0);
            for (int q = 0; q < a.nseg; ++q) {
              const C c = vp[(size_t)q * M * P + e];
              acc.x += (double)c.x;
              acc.y += (double)c.y;
            }
            int i = 0, r = e;
            while (r >= M - i) {
              r -= M - i;
              ++i;
            }
            const int j = i + r;
            const double2 d = make_double2(acc.x / (double)a.T, acc.y / (double)a.T);
            Vm[i * M + j] = d;
            if (i != j) Vm[j * M + i] = make_double2(d.x, -d.y);
          }
          __syncwarp();
          ok = warp_inv_hpd<M>(Vm, lane);
          if (ok) {  // fp64 inverse -> the fp32 layout the row updates read
#pragma unroll
            for (int r = 0; r < NE; ++r) {
              const int e = lane + 32 * r;
              if (e < M * M) tv[r] = make_float2((float)Vm[e].x, (float)Vm[e].y);
            }
            __syncwarp();
#pragma unroll
            for (int r = 0; r < NE; ++r) {
              const int e = lane + 32 * r;
              if (e < M * M) Vf[e] = tv[r];
            }
          }
          __syncwarp();
        }
      } else {
        ok = warp_inv_hpd<M>(Vm, lane);
      }
      if (lane == 0) vfail[m] = ok ? 0 : 1;
    }
    __syncthreads();
    if (warp == 0) {
      double ldet = misc[0], nprod = 1.0;
      int code = flags[0] ? 2 : 0, bad_m = 0;  // singular Q -> singular Q V at m = 0
      // lanes per row for the mat-vecs: largest power of two with M * GL <= 32
      constexpr int GL = M <= 1 ? 32 : M <= 2 ? 16 : M <= 4 ? 8 : M <= 8 ? 4 : M <= 16 ? 2 : 1;
      const int ri = lane / GL, sub = lane % GL;
      const bool rv = ri < M;
      for (int sw = 0; sw < a.ip_sweeps && code == 0; ++sw) {
        for (int m = 0; m < M; ++m) {
          if (vfail[m]) {
            code = 1;
            bad_m = m;
            break;
          }
          const C2* Vi = reinterpret_cast<const C2*>(Vd + (size_t)m * M * M);
          if (lane < M) ub[lane] = Ai[lane * 2 * M + M + m];  // u = Q^-1 e_m
          __syncwarp();
          // q = V_m^-1 u: GL lanes per row, strided partial dots + xor reduce
          C2 q = to_c2(make_double2(0.0, 0.0), C2());
          if (rv) {
#pragma unroll
            for (int j = sub; j < M; j += GL) q = cadd(q, cmul(Vi[ri * M + j], ub[j]));
          }
#pragma unroll
          for (int o = GL / 2; o > 0; o >>= 1) {
            q.x += __shfl_xor_sync(FM_FULL, q.x, o);
            q.y += __shfl_xor_sync(FM_FULL, q.y, o);
          }
          Rc part = Rc(0);
          if (rv && sub == 0) {
            const C2 u = ub[ri];
            part = q.x * u.x + q.y * u.y;  // Re(conj(q_i) u_i)
          }
          const Rc nrm = warp_sum(part);  // = q^H V q  (spatial.py:193)
          if (!(nrm > Rc(0)) || !isfinite(nrm)) {
            code = 1;
            bad_m = m;
            break;
          }
          const Rc isn = drsqrt(nrm);  // 1 / sqrt(norm)
          if (rv && sub == 0) {  // new row r = conj(q / sqrt(norm))  (spatial.py:199)
            C2 r = q;
            r.x = q.x * isn;
            r.y = -(q.y * isn);
            qb[ri] = r;
            Qd[m * M + ri] = r;
          }
          __syncwarp();
          // s = (r Q^-1 - e_m^T) / sqrt(norm), column ri per lane group
          C2 sv = to_c2(make_double2(0.0, 0.0), C2());
          if (rv) {
#pragma unroll
            for (int j = sub; j < M; j += GL) sv = cadd(sv, cmul(qb[j], Ai[j * 2 * M + M + ri]));
          }
#pragma unroll
          for (int o = GL / 2; o > 0; o >>= 1) {
            sv.x += __shfl_xor_sync(FM_FULL, sv.x, o);
            sv.y += __shfl_xor_sync(FM_FULL, sv.y, o);
          }
          if (rv && sub == 0) {
            if (ri == m) sv.x -= Rc(1);
            sv.x *= isn;
            sv.y *= isn;
            sk[ri] = sv;
          }
          __syncwarp();
          for (int e = lane; e < M * M; e += 32) {  // Q^-1 -= u s / sqrt(norm)
            const int i = e / M, k = e % M;
            C2* d = Ai + i * 2 * M + M + k;
            *d = csub(*d, cmul(ub[i], sk[k]));
          }
          nprod *= (double)nrm;  // log|det Q| += log sqrt(norm) (determinant lemma)
          if (nprod > 1e150 || nprod < 1e-150) {
            ldet += 0.5 * log(nprod);
            nprod = 1.0;
          }
          __syncwarp();
        }
      }
      if (lane == 0) {
        if (code) {
          report_status(a.status, it, bad_m, fglob, code);
          flags[1] = 1;
        }
        misc[1] = ldet + 0.5 * log(nprod);
      }
    }
    __syncthreads();
  }

  // ---- A4: row normalisation, gain normalisation + absorb ---------------------
  if (a.normalize) {
    if (tid < M) {
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < M; ++j) {
        const C2 q = Qd[tid * M + j];
        s += (double)q.x * q.x + (double)q.y * q.y;
      }
      rown[tid] = sqrt(s);
    }
    __syncthreads();
    for (int e = tid; e < M * M; e += BS) {
      const Rc r = (Rc)rown[e / M];
      C2 v = Qd[e];
      v.x = v.x / r;
      v.y = v.y / r;
      Qd[e] = v;
    }
    for (int e = tid; e < N * M; e += BS) {
      const double r = rown[e % M];
      gs[e] = (R)((double)gs[e] / (r * r));
    }
    if (tid == 0) {  // sum_m log ||row m||: one log per range-guarded product
      double s = 0.0, pr = 1.0;
      for (int m = 0; m < M; ++m) {
        pr *= rown[m];
        if (pr > 1e150 || pr < 1e-150) {
          s += log(pr);
          pr = 1.0;
        }
      }
      misc[1] -= s + log(pr);
    }
    __syncthreads();
    if (tid < N) {
      R s = 0;
#pragma unroll
      for (int m = 0; m < M; ++m) s += gs[tid * M + m];
      s = s > RT<R>::tiny() ? s : RT<R>::tiny();
      const R scl = R(M) / s;
#pragma unroll
      for (int m = 0; m < M; ++m) gs[tid * M + m] = gs[tid * M + m] * scl;
      cs[tid] = s / R(M);
    }
    __syncthreads();
    const int Nn = N - a.n0;
    for (int e = tid; e < Nn * K; e += BS) {
      const int n = e / K, k = e % K;
      const size_t wi = (size_t)n * F * K + k;
      Wg[wi] = Wsg[wi] * cs[a.n0 + n];  // sources.py:202-204
    }
    if (a.n0 && tid == 0) a.u[(size_t)b * F + f] *= cs[0];
  } else if (Wsg != Wg) {  // no absorb: the state W is the W-stepped one
    for (int e = tid; e < (N - a.n0) * K; e += BS) {
      const size_t wi = (size_t)(e / K) * F * K + e % K;
      Wg[wi] = Wsg[wi];
    }
  }
  for (int e = tid; e < M * M; e += BS) Qg[e] = cmake<C>(Qd[e].x, Qd[e].y);
  for (int e = tid; e < N * M; e += BS) gg[(size_t)(e / M) * F * M + (e % M)] = gs[e];
  if (tid < NMAX) a.cs_out[((size_t)b * F + f) * NMAX + tid] = cs[tid];
  if (tid == 0) a.ld_part[(size_t)b * F + f] = misc[1];
}


// ---------------------------------------------------------------------------
template <typename R> struct BackArgs {
  const cplx<R>* X;
  R* xt;
  const cplx<R>* Q;
  const R* g;
  const R* lam;
  const R* cs;  // (B, F, NMAX) or null (factor 1)
  R* phi;
  const R* floorp;
  double* ll_part;
  const double* ld_part;
  double* trace;
  unsigned* counter;
  unsigned* iter;
  int B, F, T, N;
  int record;
};

// One t per thread; grid (ceil(T/256), F, B): the (f, t) plane is tiled
// flat so every SM streams many small tiles (no per-bin serial loop).
// ll_part is (B, F, tiles) and reduced in fixed order by the last tile.
// 3 CTAs per SM (<= 85 registers) up to M = 8; 2 above, where the 16-channel
// rows would otherwise spill
// points (frames) per thread of k_back: 2 for M <= 4 and long recordings,
// whose CTAs otherwise spend half their life at the staging barrier with too
// few bytes in flight (c2: 52% barrier stalls, 44% of DRAM bandwidth; k_back
// 1.57 -> 1.34 ms); 1 otherwise (c0, T = 128: 8.2 -> 9.7 us with 2)
inline int back_ppt(long long M, long long T) { return (M <= 4 && T >= 512) ? 2 : 1; }

template <typename R, int M, int PPT>
__global__ void __launch_bounds__(256, (M > 8 ? 2 : (M == 8 && sizeof(R) == 4 ? 4 : 3))) k_back(BackArgs<R> a) {
  pdl_entry();
  using C = cplx<R>;
  __shared__ __align__(16) C Qr[M * M];
  __shared__ __align__(16) R gs[NMAX * M];
  __shared__ R cs[NMAX];
  __shared__ double dred[8];
  const int tile = blockIdx.x, f = blockIdx.y, b = blockIdx.z;
  const int ntile = gridDim.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int N = a.N, T = a.T, F = a.F;
  const size_t FT = (size_t)F * T;
  // Q, g and c go to registers first and to shared memory only after the
  // frame loads below are in flight: one global round trip before the barrier
  // instead of two (M * M <= 256 and N * M <= 256: one element per thread)
  C qreg = cmake<C>(0.0, 0.0);
  R greg = R(0), creg = R(1);
  if (tid < M * M) qreg = a.Q[((size_t)b * F + f) * M * M + tid];
  if (tid < N * M)
    greg = a.g[(size_t)b * N * F * M + (size_t)(tid / M) * F * M + (size_t)f * M + (tid % M)];
  if (tid < NMAX && a.cs) creg = a.cs[((size_t)b * F + f) * NMAX + tid];
  double ll = 0.0;
  C xv[PPT][M];
  R l[PPT][NMAX];
#pragma unroll
  for (int u = 0; u < PPT; ++u) {  // every point's loads issued before the barrier
    const int t = tile * 256 * PPT + u * 256 + tid;
    if (t < T) {
      CRowIO<R, M>::load(a.X + (((size_t)b * F + f) * T + t) * M, xv[u]);
      const R* lb = a.lam + (size_t)b * N * FT + (size_t)f * T + t;
#pragma unroll
      for (int n = 0; n < NMAX; ++n) {
        l[u][n] = R(0);
        if (n >= N) break;
        l[u][n] = lb[(size_t)n * FT];
      }
    }
  }
  if (tid < M * M) Qr[tid] = qreg;
  if (tid < N * M) gs[tid] = greg;
  if (tid < NMAX) cs[tid] = creg;
  __syncthreads();
  const R fl = a.floorp[b];
#pragma unroll
  for (int u = 0; u < PPT; ++u) {
    const int t = tile * 256 * PPT + u * 256 + tid;
    if (t >= T) continue;
#pragma unroll
    for (int n = 0; n < NMAX; ++n) l[u][n] *= cs[n];
    R xtv[M];
#pragma unroll
    for (int i = 0; i < M; ++i) {
      C s = cmake<C>(0.0, 0.0);
#pragma unroll
      for (int j = 0; j < M; ++j) {
        const C q = Qr[i * M + j];
        s = fma2(cmake<C>(q.x, q.x), xv[u][j], s);
        s = fma2(cmake<C>(-q.y, q.y), cmake<C>(xv[u][j].y, xv[u][j].x), s);
      }
      xtv[i] = s.x * s.x + s.y * s.y;
    }
    RowIO<R, M>::store(a.xt + (((size_t)b * F + f) * T + t) * M, xtv);
    R iy[M], y[M];
    model_power<R, M>(l[u], gs, N, fl, iy, y);
    R llt = 0;
#pragma unroll
    for (int m = 0; m < M; ++m) llt += -xtv[m] * iy[m] - log_fast(y[m]);
    ll += (double)llt;
    phi_point<R, M>(xtv, iy, gs, N, a.phi + (size_t)b * 2 * N * FT, FT, (size_t)f * T + t);
  }
  ll = warp_sum(ll);
  if (lane == 0) dred[warp] = ll;
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
    for (int w = 0; w < 8; ++w) s += dred[w];
    a.ll_part[((size_t)b * F + f) * ntile + tile] = s;
  }
}

// trace entry of the state after this iteration (separate.py:313-318, :321):
// sum of the data-term partials (B, np1, np2) + 2T sum_f log|det Q_f|, one CTA
// per mixture, fixed-order strided + tree reduction (deterministic).
static __global__ void __launch_bounds__(256) k_trace(const double* __restrict__ ll_part,
                                               const double* __restrict__ ld_part,
                                               double* __restrict__ trace, unsigned* iter, int B,
                                               int np1, int np2, int F, int T) {
  pdl_entry();
  __shared__ double r1[8], r2[8];
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const size_t n1 = (size_t)np1 * np2;  // data-term partials per mixture
  const double* p1 = ll_part + (size_t)b * n1;
  const double* p2 = ld_part + (size_t)b * F;
  double s1 = 0.0, s2 = 0.0;
  for (size_t e = tid; e < n1; e += 256) s1 += p1[e];
  for (int e = tid; e < F; e += 256) s2 += p2[e];
  s1 = warp_sum(s1);
  s2 = warp_sum(s2);
  if (lane == 0) {
    r1[warp] = s1;
    r2[warp] = s2;
  }
  __syncthreads();
  if (tid == 0) {
    double a1 = 0.0, a2 = 0.0;
    for (int w = 0; w < 8; ++w) {
      a1 += r1[w];
      a2 += r2[w];
    }
    const unsigned it = *iter;
    if (trace) trace[(size_t)it * B + b] = a1 + 2.0 * (double)T * a2;
    if (gridDim.x == 1) *iter = it + 1u;  // single mixture: advance here
  }
}

static __global__ void k_iter_advance(unsigned* iter) {
  pdl_entry(); *iter += 1u; }

}  // namespace fm
