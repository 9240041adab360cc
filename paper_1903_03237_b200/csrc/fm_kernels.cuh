// fm_kernels.cuh -- hand-written sm_100a kernels of the FastMNMF iteration.
//
// One FastMNMF iteration (_DiagLoop.iterate, separate.py:201-234; paths are
// relative to /root/reference/pkg/src/fastsep) is executed as five launches
// over device-resident state:
//
//   k_wupdate   W MU  (sources.py:191-194) from phi of the previous pass
//   k_hstats    2nd statistics pass (separate.py:215) fused with the H-stat
//               contraction sum_f W phi (sources.py:196-197), per-F-chunk partials
//   k_hupdate   H MU  (sources.py:195-198): fixed-order sum of the partials
//   k_lambda    lambda = W H  (sources.py:184-187)
//   k_spatial   per-frequency rest: gain stats + g MU (separate.py:217-220),
//               V_fm (spatial.py:182 / _kernels.py:276-293) from the floored
//               model power (separate.py:221), IP row updates (spatial.py:183-199),
//               row and gain normalisation (separate.py:223-233), log|det Q|
//               (separate.py:236-238), projection (separate.py:230) and the
//               NEXT iteration's first statistics pass (separate.py:186-193:
//               log-likelihood data term + phi), written for k_wupdate.
//
// Layout (row-major, batch-major): X (B,F,T,M) complex, xt (B,F,T,M),
// Q (B,F,M,M) complex, g (B,N,F,M), W (B,N,F,K), H (B,N,K,T),
// lam (B,N,F,T), phi (B,2,N,F,T).
#pragma once
#include "fm_common.cuh"
#include "fm_linalg.cuh"

namespace fm {

constexpr int NMAX = 8;  // sources per mixture supported by the fused kernels

// ---------------------------------------------------------------------------
// lambda = W H per (b, n): (F x K) (K x T). SIMT register-blocked tile:
// 64 f x 64 t per CTA, 4 x 4 outputs per thread, K staged 32 at a time.
// ---------------------------------------------------------------------------
template <typename R>
__global__ void __launch_bounds__(256) k_lambda(const R* __restrict__ W, const R* __restrict__ H,
                                                R* __restrict__ lam, int F, int T, int K) {
  __shared__ R Ws[32][64 + 4];
  __shared__ R Hs[32][64 + 4];
  const int bn = blockIdx.z;
  const int t0 = blockIdx.x * 64, f0 = blockIdx.y * 64;
  const R* Wb = W + (size_t)bn * F * K;
  const R* Hb = H + (size_t)bn * K * T;
  R* Lb = lam + (size_t)bn * F * T;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  R acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0;
  for (int k0 = 0; k0 < K; k0 += 32) {
    const int kc = min(32, K - k0);
    for (int e = threadIdx.x; e < 64 * 32; e += 256) {
      // W tile: 64 f rows x 32 k (k contiguous in memory) -> Ws[k][f]
      const int fl = e / 32, kl = e % 32;
      const int f = f0 + fl, k = k0 + kl;
      Ws[kl][fl] = (f < F && kl < kc) ? Wb[(size_t)f * K + k] : R(0);
      // H tile: 32 k rows x 64 t (t contiguous) -> Hs[k][t]
      const int kh = e / 64, th = e % 64;
      const int t = t0 + th;
      Hs[kh][th] = (kh < kc && t < T) ? Hb[(size_t)(k0 + kh) * T + t] : R(0);
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
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int f = f0 + ty * 4 + i;
    if (f >= F) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int t = t0 + tx * 4 + j;
      if (t < T) Lb[(size_t)f * T + t] = acc[i][j];
    }
  }
}

// ---------------------------------------------------------------------------
// W MU (sources.py:191-194): num = phi1 H^T, den = phi2 H^T (sum over T),
// W *= sqrt(num / max(den, TINY)). One warp per (b, n, f); lanes stride T.
// grid (ceil(F/8), N, B), block 256.
// ---------------------------------------------------------------------------
template <typename R, int KB>
__global__ void __launch_bounds__(256) k_wupdate(const R* __restrict__ phi, const R* __restrict__ H,
                                                 R* __restrict__ W, int N, int F, int T, int K) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int f = blockIdx.x * 8 + warp;
  const int n = blockIdx.y, b = blockIdx.z;
  if (f >= F) return;
  const size_t FT = (size_t)F * T;
  const R* p1 = phi + ((size_t)b * 2 * N + n) * FT + (size_t)f * T;
  const R* p2 = p1 + (size_t)N * FT;
  const R* Hn = H + ((size_t)b * N + n) * K * T;
  R num[KB], den[KB];
#pragma unroll
  for (int k = 0; k < KB; ++k) num[k] = den[k] = 0;
  for (int t = lane; t < T; t += 32) {
    const R a1 = p1[t], a2 = p2[t];
#pragma unroll
    for (int k = 0; k < KB; ++k) {
      if (k < K) {
        const R h = __ldg(Hn + (size_t)k * T + t);
        num[k] += a1 * h;
        den[k] += a2 * h;
      }
    }
  }
  R* Wr = W + (((size_t)b * N + n) * F + f) * K;
#pragma unroll
  for (int k = 0; k < KB; ++k) {
    if (k < K) {
      const R sn = warp_sum(num[k]), sd = warp_sum(den[k]);
      if (lane == (k & 31)) Wr[k] = Wr[k] * mu_factor(sn, sd);
    }
  }
}

// ---------------------------------------------------------------------------
// Second statistics pass of the iteration (separate.py:215 after the W step)
// fused with the H-statistic contraction (sources.py:196-197):
//   lam' = W' H, y = max(sum_n lam' g, floor), phi1 = sum_m g x~/y^2,
//   phi2 = sum_m g/y, numH[n,k,t] += W'[n,f,k] phi1, denH += W' phi2
// over the F-chunk of this CTA. Thread = (t, n); warps of one t-group share
// lambda through shared memory. Partials: part (B, FC, 2, N, K, T).
// grid (ceil(T/(32 G)), FC, B), block 32 N G.
// ---------------------------------------------------------------------------
template <typename R, int KB>
__global__ void __launch_bounds__(256) k_hstats(const R* __restrict__ W, const R* __restrict__ H,
                                                const R* __restrict__ g, const R* __restrict__ xt,
                                                const R* __restrict__ floorp, R* __restrict__ part,
                                                int N, int F, int T, int M, int K, int FCH, int G) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  R* Ws = reinterpret_cast<R*>(smem_raw);  // [FCH][N][K]
  R* gs = Ws + (size_t)FCH * N * K;        // [FCH][N][M]
  R* ls = gs + (size_t)FCH * N * M;        // [2][G][N][32]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int n = w % N, grp = w / N;
  const int b = blockIdx.z, chunk = blockIdx.y, FC = gridDim.y;
  const int f0 = chunk * FCH, f1 = min(F, f0 + FCH), nf = f1 - f0;
  const int t = blockIdx.x * 32 * G + grp * 32 + lane;
  const bool tv = t < T;
  const R fl = floorp[b];
  // stage the W rows and g rows of this F-chunk
  for (int e = threadIdx.x; e < nf * N * K; e += blockDim.x) {
    const int fi = e / (N * K), r = e % (N * K), nn = r / K, k = r % K;
    Ws[e] = W[(((size_t)b * N + nn) * F + f0 + fi) * K + k];
  }
  for (int e = threadIdx.x; e < nf * N * M; e += blockDim.x) {
    const int fi = e / (N * M), r = e % (N * M), nn = r / M, m = r % M;
    gs[e] = g[(((size_t)b * N + nn) * F + f0 + fi) * M + m];
  }
  R hreg[KB], an[KB], ad[KB];
  const R* Hn = H + ((size_t)b * N + n) * K * T;
#pragma unroll
  for (int k = 0; k < KB; ++k) {
    hreg[k] = (k < K && tv) ? Hn[(size_t)k * T + t] : R(0);
    an[k] = ad[k] = 0;
  }
  __syncthreads();
  const R* xtb = xt + (size_t)b * F * T * M;
  for (int fi = 0; fi < nf; ++fi) {
    const R* wr = Ws + ((size_t)fi * N + n) * K;
    R l = 0;
#pragma unroll
    for (int k = 0; k < KB; ++k)
      if (k < K) l += wr[k] * hreg[k];
    R* lsb = ls + (size_t)(fi & 1) * G * N * 32 + (size_t)grp * N * 32;
    lsb[n * 32 + lane] = l;
    const R* xr = xtb + ((size_t)(f0 + fi) * T + (tv ? t : 0)) * M;
    __syncthreads();
    const R* gf = gs + (size_t)fi * N * M;
    R p1 = 0, p2 = 0;
    for (int m = 0; m < M; ++m) {
      R acc = 0;
      for (int nn = 0; nn < N; ++nn) acc += lsb[nn * 32 + lane] * gf[nn * M + m];
      const R y = floor_max(acc, fl);
      const R iy = R(1) / y;
      const R gm = gf[n * M + m];
      p1 += gm * xr[m] * iy * iy;
      p2 += gm * iy;
    }
    if (!tv) p1 = p2 = 0;
#pragma unroll
    for (int k = 0; k < KB; ++k) {
      if (k < K) {
        an[k] += wr[k] * p1;
        ad[k] += wr[k] * p2;
      }
    }
  }
  if (tv) {
    const size_t NKT = (size_t)N * K * T;
    R* pb = part + (((size_t)b * FC + chunk) * 2) * NKT + (size_t)n * K * T + t;
#pragma unroll
    for (int k = 0; k < KB; ++k) {
      if (k < K) {
        pb[(size_t)k * T] = an[k];
        pb[NKT + (size_t)k * T] = ad[k];
      }
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

// ---------------------------------------------------------------------------
// Per-frequency kernel. See the file header. grid (F, B).
// ---------------------------------------------------------------------------
template <int M> struct SpCfg {
  static constexpr int BS = (M <= 8) ? 256 : 512;
  static constexpr int TC = (M <= 8) ? 256 : 128;
  static constexpr int P = M * (M + 1) / 2;
  static constexpr int S2 = BS / P;
};

template <typename R> struct SpArgs {
  const cplx<R>* X;
  R* xt;
  cplx<R>* Q;
  R* g;
  R* W;
  const R* lam;
  R* phi;
  const R* floorp;
  double* ll_part;   // (B, F)
  double* ld_part;   // (B, F)
  double* trace;     // (iters, B)
  unsigned* counter; // arrival counter (last-block reduction)
  unsigned* iter;    // iteration counter
  unsigned long long* status;
  int B, F, T, M, N, K;
  long long f_offset;
  int normalize, ip_sweeps, tail_only, record;
};

template <typename R, int M>
__host__ __device__ inline size_t spatial_smem_bytes() {
  using C = cplx<R>;
  constexpr int TC = SpCfg<M>::TC, BS = SpCfg<M>::BS, P = SpCfg<M>::P;
  size_t s = 0;
  auto al = [](size_t x) { return (x + 15) & ~size_t(15); };
  s += al(sizeof(double2) * M * M);        // Qd
  s += al(sizeof(double2) * M * (M + 1));  // A
  s += al(sizeof(double2) * M);            // xs
  s += al(sizeof(C) * M * M);              // Qr
  s += al(sizeof(R) * NMAX * M);           // gs
  s += al(sizeof(R) * NMAX);               // cs
  s += al(sizeof(double) * M);             // row norms
  s += al(sizeof(int) * 2 * P);            // pair table
  s += al(sizeof(R) * (BS / 32) * 2 * M);  // redw
  s += al(sizeof(C) * M * M * M);          // Vs
  s += al(sizeof(R) * NMAX * (TC + 1));    // lam chunk
  s += al(sizeof(R) * TC * M);             // iy
  s += al(sizeof(R) * TC * M);             // xr
  s += al(sizeof(C) * TC * M);             // Xc
  s += al(sizeof(double) * 40);            // reductions + flags
  return s;
}

template <typename R, int M>
__global__ void __launch_bounds__(SpCfg<M>::BS) k_spatial(SpArgs<R> a) {
  using C = cplx<R>;
  constexpr int BS = SpCfg<M>::BS, TC = SpCfg<M>::TC, P = SpCfg<M>::P, S2 = SpCfg<M>::S2;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned char* sp = smem_raw;
  auto take = [&](size_t bytes) {
    unsigned char* p = sp;
    sp += (bytes + 15) & ~size_t(15);
    return p;
  };
  double2* Qd = reinterpret_cast<double2*>(take(sizeof(double2) * M * M));
  double2* Am = reinterpret_cast<double2*>(take(sizeof(double2) * M * (M + 1)));
  double2* xs = reinterpret_cast<double2*>(take(sizeof(double2) * M));
  C* Qr = reinterpret_cast<C*>(take(sizeof(C) * M * M));
  R* gs = reinterpret_cast<R*>(take(sizeof(R) * NMAX * M));
  R* cs = reinterpret_cast<R*>(take(sizeof(R) * NMAX));
  double* rown = reinterpret_cast<double*>(take(sizeof(double) * M));
  int* pairs = reinterpret_cast<int*>(take(sizeof(int) * 2 * P));
  R* redw = reinterpret_cast<R*>(take(sizeof(R) * (BS / 32) * 2 * M));
  C* Vs = reinterpret_cast<C*>(take(sizeof(C) * M * M * M));
  R* lamc = reinterpret_cast<R*>(take(sizeof(R) * NMAX * (TC + 1)));
  R* iys = reinterpret_cast<R*>(take(sizeof(R) * TC * M));
  R* xrs = reinterpret_cast<R*>(take(sizeof(R) * TC * M));
  C* Xc = reinterpret_cast<C*>(take(sizeof(C) * TC * M));
  double* dred = reinterpret_cast<double*>(take(sizeof(double) * 40));
  int* flags = reinterpret_cast<int*>(dred + 36);

  const int f = blockIdx.x, b = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int N = a.N, T = a.T, F = a.F, K = a.K;
  const size_t FT = (size_t)F * T;
  const C* X = a.X + ((size_t)b * F + f) * T * M;
  R* xt = a.xt + ((size_t)b * F + f) * T * M;
  const R* lam = a.lam + (size_t)b * N * FT + (size_t)f * T;
  R* phi = a.phi + (size_t)b * 2 * N * FT + (size_t)f * T;
  C* Qg = a.Q + ((size_t)b * F + f) * M * M;
  R* gg = a.g + (size_t)b * N * F * M + (size_t)f * M;
  R* Wg = a.W + (size_t)b * N * F * K + (size_t)f * K;
  const R fl = a.floorp[b];
  const unsigned it = *a.iter;
  const long long fglob = a.f_offset + f;

  for (int e = tid; e < N * M; e += BS) gs[e] = gg[(size_t)(e / M) * F * M + (e % M)];
  for (int e = tid; e < M * M; e += BS) {
    const C q = Qg[e];
    Qd[e] = to_d2(q);
    Qr[e] = q;
  }
  if (tid < NMAX) cs[tid] = R(1);
  if (tid == 0) {
    int p = 0;
    for (int i = 0; i < M; ++i)
      for (int j = i; j < M; ++j) {
        pairs[2 * p] = i;
        pairs[2 * p + 1] = j;
        ++p;
      }
    flags[0] = 0;
  }
  __syncthreads();
  double ldet = 0.0;

  if (!a.tail_only) {
    // ---- A1: gain statistics + g MU (separate.py:217-220; _kernels.py:244-250)
    {
      const int WPN = (BS / 32) / N;  // warps per source
      const int n1 = warp / WPN, sub = warp % WPN;
      const bool act = n1 < N;
      const int S1 = WPN * 32, s1 = sub * 32 + lane;
      R num[M], den[M];
#pragma unroll
      for (int m = 0; m < M; ++m) num[m] = den[m] = 0;
      for (int t0 = 0; t0 < T; t0 += TC) {
        for (int tl = tid; tl < TC; tl += BS) {
          const int t = t0 + tl;
          if (t < T) {
            R l[NMAX];
#pragma unroll
            for (int n = 0; n < NMAX; ++n) {
              l[n] = (n < N) ? lam[(size_t)n * FT + t] : R(0);
              if (n < N) lamc[n * (TC + 1) + tl] = l[n];
            }
            R x[M];
            RowIO<R, M>::load(xt + (size_t)t * M, x);
#pragma unroll
            for (int m = 0; m < M; ++m) {
              R acc = 0;
#pragma unroll
              for (int n = 0; n < NMAX; ++n)
                if (n < N) acc += l[n] * gs[n * M + m];
              const R y = floor_max(acc, fl);
              const R iy = R(1) / y;
              iys[tl * M + m] = iy;
              xrs[tl * M + m] = x[m] * iy * iy;
            }
          } else {
            for (int n = 0; n < N; ++n) lamc[n * (TC + 1) + tl] = 0;
#pragma unroll
            for (int m = 0; m < M; ++m) iys[tl * M + m] = xrs[tl * M + m] = 0;
          }
        }
        __syncthreads();
        if (act) {
          for (int tl = s1; tl < TC; tl += S1) {
            const R l = lamc[n1 * (TC + 1) + tl];
#pragma unroll
            for (int m = 0; m < M; ++m) {
              num[m] += l * xrs[tl * M + m];
              den[m] += l * iys[tl * M + m];
            }
          }
        }
        __syncthreads();
      }
#pragma unroll
      for (int m = 0; m < M; ++m) {
        num[m] = warp_sum(num[m]);
        den[m] = warp_sum(den[m]);
      }
      if (act && lane == 0) {
#pragma unroll
        for (int m = 0; m < M; ++m) {
          redw[warp * 2 * M + m] = num[m];
          redw[warp * 2 * M + M + m] = den[m];
        }
      }
      __syncthreads();
      for (int e = tid; e < N * M; e += BS) {
        const int n = e / M, m = e % M;
        R sn = 0, sd = 0;
        for (int s = 0; s < WPN; ++s) {
          sn += redw[(n * WPN + s) * 2 * M + m];
          sd += redw[(n * WPN + s) * 2 * M + M + m];
        }
        gs[e] = gs[e] * mu_factor(sn, sd);
      }
      __syncthreads();
    }
    // ---- A2: V_fm = (1/T) sum_t x x^H / y_ftm with y = mix_power(lam, g)
    //      (separate.py:221-222 -> spatial.py:182 -> _kernels.py:276-293)
    {
      const int p = tid % P, s2 = tid / P;
      const bool act = s2 < S2;
      const int pi = pairs[2 * p], pj = pairs[2 * p + 1];
      R vr[M], vi[M];
#pragma unroll
      for (int m = 0; m < M; ++m) vr[m] = vi[m] = 0;
      for (int t0 = 0; t0 < T; t0 += TC) {
        for (int tl = tid; tl < TC; tl += BS) {
          const int t = t0 + tl;
          if (t < T) {
            R l[NMAX];
#pragma unroll
            for (int n = 0; n < NMAX; ++n) l[n] = (n < N) ? lam[(size_t)n * FT + t] : R(0);
#pragma unroll
            for (int m = 0; m < M; ++m) {
              R acc = 0;
#pragma unroll
              for (int n = 0; n < NMAX; ++n)
                if (n < N) acc += l[n] * gs[n * M + m];
              iys[tl * M + m] = R(1) / floor_max(acc, fl);
            }
            C xv[M];
            CRowIO<R, M>::load(X + (size_t)t * M, xv);
            CRowIO<R, M>::store(Xc + tl * M, xv);
          } else {
#pragma unroll
            for (int m = 0; m < M; ++m) {
              iys[tl * M + m] = 0;
              Xc[tl * M + m] = cmake<C>(0.0, 0.0);
            }
          }
        }
        __syncthreads();
        if (act) {
          for (int tl = s2; tl < TC; tl += S2) {
            const C xi = Xc[tl * M + pi], xj = Xc[tl * M + pj];
            const R pr = xi.x * xj.x + xi.y * xj.y;  // x_i conj(x_j)
            const R pm = xi.y * xj.x - xi.x * xj.y;
#pragma unroll
            for (int m = 0; m < M; ++m) {
              const R w = iys[tl * M + m];
              vr[m] += w * pr;
              vi[m] += w * pm;
            }
          }
        }
        __syncthreads();
      }
      // fixed-order reduction over the S2 slices
      for (int ss = 0; ss < S2; ++ss) {
        if (act && s2 == ss) {
#pragma unroll
          for (int m = 0; m < M; ++m) {
            C* v = Vs + ((size_t)m * M + pi) * M + pj;
            if (ss == 0) {
              *v = cmake<C>(vr[m], vi[m]);
            } else {
              C o = *v;
              o.x += vr[m];
              o.y += vi[m];
              *v = o;
            }
          }
        }
        __syncthreads();
      }
      const R invT = R(1) / R(T);
      for (int e = tid; e < M * P; e += BS) {
        const int m = e / P, pp = e % P;
        const int i = pairs[2 * pp], j = pairs[2 * pp + 1];
        C v = Vs[((size_t)m * M + i) * M + j];
        v.x *= invT;
        v.y *= invT;
        Vs[((size_t)m * M + i) * M + j] = v;
        if (i != j) Vs[((size_t)m * M + j) * M + i] = cmake<C>(v.x, -v.y);
      }
      __syncthreads();
    }
    // ---- A3: IP row updates (spatial.py:181-199), warp 0, fp64
    if (warp == 0) {
      int bad_m = 0;
      const int code = warp_ip_update<M>(Qd, Vs, Am, xs, a.ip_sweeps, lane, &bad_m);
      if (code != 0 && lane == 0) {
        report_status(a.status, it, bad_m, fglob, code);
        flags[0] = 1;
      }
    }
    __syncthreads();
    // ---- A4: row normalisation (separate.py:223-229)
    if (a.normalize) {
      if (tid < M) {
        double s = 0.0;
        for (int j = 0; j < M; ++j) {
          const double2 q = Qd[tid * M + j];
          s += q.x * q.x + q.y * q.y;
        }
        rown[tid] = sqrt(s);
      }
      __syncthreads();
      for (int e = tid; e < M * M; e += BS) {
        const double r = rown[e / M];
        Qd[e] = make_double2(Qd[e].x / r, Qd[e].y / r);
      }
      for (int e = tid; e < N * M; e += BS) {
        const double r = rown[e % M];
        gs[e] = (R)((double)gs[e] / (r * r));
      }
      __syncthreads();
    }
    // log|det Q_f| (separate.py:236-238) on the final Q of this iteration
    if (warp == 0) {
      for (int e = lane; e < M * M; e += 32) Am[(e / M) * (M + 1) + (e % M)] = Qd[e];
      __syncwarp();
      double la = 0.0;
      warp_lu<M>(Am, M + 1, M, lane, &la);
      if (lane == 0) dred[33] = la;
    }
    // gain normalisation + absorb into W (spatial.py:244-249, sources.py:202-204)
    if (a.normalize && tid < N) {
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
    ldet = dred[33];
    if (a.normalize) {
      for (int e = tid; e < N * K; e += BS) {
        const int n = e / K, k = e % K;
        R* wp = Wg + (size_t)n * F * K + k;
        *wp = *wp * cs[n];
      }
    }
    for (int e = tid; e < M * M; e += BS) {
      const C q = cmake<C>(Qd[e].x, Qd[e].y);
      Qr[e] = q;
      Qg[e] = q;
    }
    for (int e = tid; e < N * M; e += BS) gg[(size_t)(e / M) * F * M + (e % M)] = gs[e];
    __syncthreads();
  }

  // ---- A5: projection (separate.py:230; _kernels.py:339-350) and the next
  //      statistics pass (separate.py:186-193; _kernels.py:226-243)
  double ll = 0.0;
  for (int t = tid; t < T; t += BS) {
    C xv[M];
    CRowIO<R, M>::load(X + (size_t)t * M, xv);
    R xtv[M];
#pragma unroll
    for (int i = 0; i < M; ++i) {
      R sr = 0, si = 0;
#pragma unroll
      for (int j = 0; j < M; ++j) {
        const C q = Qr[i * M + j];
        sr += q.x * xv[j].x - q.y * xv[j].y;
        si += q.x * xv[j].y + q.y * xv[j].x;
      }
      xtv[i] = sr * sr + si * si;
    }
    RowIO<R, M>::store(xt + (size_t)t * M, xtv);
    R l[NMAX];
#pragma unroll
    for (int n = 0; n < NMAX; ++n) l[n] = (n < N) ? lam[(size_t)n * FT + t] * cs[n] : R(0);
    R iy[M];
    R llt = 0;
#pragma unroll
    for (int m = 0; m < M; ++m) {
      R acc = 0;
#pragma unroll
      for (int n = 0; n < NMAX; ++n)
        if (n < N) acc += l[n] * gs[n * M + m];
      const R y = floor_max(acc, fl);
      iy[m] = R(1) / y;
      llt += -xtv[m] * iy[m] - log_r(y);
    }
    ll += (double)llt;
    for (int n = 0; n < N; ++n) {
      R p1 = 0, p2 = 0;
#pragma unroll
      for (int m = 0; m < M; ++m) {
        const R gm = gs[n * M + m];
        p1 += gm * xtv[m] * iy[m] * iy[m];
        p2 += gm * iy[m];
      }
      phi[(size_t)n * FT + t] = p1;
      phi[(size_t)(N + n) * FT + t] = p2;
    }
  }
  // block reduction of the data term (fp64)
  ll = warp_sum(ll);
  if (lane == 0) dred[warp] = ll;
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
    for (int w = 0; w < BS / 32; ++w) s += dred[w];
    a.ll_part[(size_t)b * F + f] = s;
    a.ld_part[(size_t)b * F + f] = ldet;
  }
  if (a.record) {
    __shared__ int is_last;
    if (tid == 0) {
      __threadfence();
      const unsigned prev = atomicAdd(a.counter, 1u);
      is_last = (prev == gridDim.x * gridDim.y - 1);
    }
    __syncthreads();
    if (is_last) {
      __threadfence();
      for (int bb = tid; bb < a.B; bb += BS) {
        double s1 = 0.0, s2 = 0.0;
        for (int ff = 0; ff < F; ++ff) {
          s1 += __ldcg(a.ll_part + (size_t)bb * F + ff);
          s2 += __ldcg(a.ld_part + (size_t)bb * F + ff);
        }
        a.trace[(size_t)it * a.B + bb] = s1 + 2.0 * (double)T * s2;
      }
      if (tid == 0) {
        *a.counter = 0u;
        *a.iter = it + 1u;
      }
    }
  }
}

}  // namespace fm
