// fm_spatial.cuh -- the per-frequency part of the FastMNMF iteration.
//
// k_front (one CTA per (f, b)): gain statistics + g MU (separate.py:217-220;
//   _kernels.py:244-250), the weighted covariances V_fm = (1/T) sum_t x x^H /
//   y_ftm from the floored model power with the new gains (separate.py:221-222,
//   spatial.py:182, _kernels.py:276-293), the iterative-projection row updates
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

template <int M> struct FrCfg {
  static constexpr int BS = (M <= 8) ? 256 : 512;
  static constexpr int TC = 256;
  static constexpr int P = M * (M + 1) / 2;
  static constexpr int S2 = BS / P;
};

template <typename R> struct FrontArgs {
  const cplx<R>* X;
  const R* xt;
  cplx<R>* Q;
  R* g;
  R* W;
  const R* lam;
  const R* floorp;
  double2* V;       // (B, F, M, M, M) weighted covariances for k_ip
  int F, T, N, K;
  long long* timing;  // optional (F, 8) clock64 stamps per phase (profiling builds/tools)
};

template <typename R, int M> struct FrontSmem {
  using C = cplx<R>;
  static constexpr int BS = FrCfg<M>::BS, TC = FrCfg<M>::TC, P = FrCfg<M>::P;
  static constexpr size_t al(size_t x) { return (x + 15) & ~size_t(15); }
  // control region
  static constexpr size_t o_gs = 0;
  static constexpr size_t o_cs = o_gs + al(sizeof(R) * NMAX * M);
  static constexpr size_t o_rown = o_cs + al(sizeof(R) * NMAX);
  static constexpr size_t o_pairs = o_rown + al(sizeof(double) * M);
  static constexpr size_t o_redw = o_pairs + al(sizeof(int) * 2 * P);
  static constexpr size_t o_misc = o_redw + al(sizeof(R) * (BS / 32) * 2 * M);
  static constexpr size_t o_Qd = o_misc + al(sizeof(double) * 8 + sizeof(int) * (M + 8));
  static constexpr size_t o_Ai = o_Qd + al(sizeof(double2) * M * M);
  static constexpr size_t o_vec = o_Ai + al(sizeof(double2) * M * 2 * M);
  static constexpr size_t o_union = o_vec + al(sizeof(double2) * 3 * M);
  // streaming buffers (phases A1/A2) ...
  static constexpr size_t s_lam = 0;
  static constexpr size_t s_iy = s_lam + al(sizeof(R) * NMAX * (TC + 1));
  static constexpr size_t s_xr = s_iy + al(sizeof(R) * TC * M);
  static constexpr size_t s_X = s_xr + al(sizeof(R) * TC * M);
  static constexpr size_t s_end = s_X + al(sizeof(C) * TC * M);
  // ... overlaid by V (fp64) once streaming is done
  static constexpr size_t v_end = al(sizeof(double2) * M * M * M);
  static constexpr size_t bytes = o_union + (s_end > v_end ? s_end : v_end);
};

template <typename R, int M>
__global__ void __launch_bounds__(FrCfg<M>::BS, (M <= 8 ? 2 : 1)) k_front(FrontArgs<R> a) {
  using C = cplx<R>;
  using L = FrontSmem<R, M>;
  constexpr int BS = FrCfg<M>::BS, TC = FrCfg<M>::TC, P = FrCfg<M>::P, S2 = FrCfg<M>::S2;
  constexpr int NW = BS / 32;
  extern __shared__ __align__(16) unsigned char sm[];
  R* gs = reinterpret_cast<R*>(sm + L::o_gs);
  int* pairs = reinterpret_cast<int*>(sm + L::o_pairs);
  R* redw = reinterpret_cast<R*>(sm + L::o_redw);
  unsigned char* un = sm + L::o_union;
  R* lamc = reinterpret_cast<R*>(un + L::s_lam);
  R* iys = reinterpret_cast<R*>(un + L::s_iy);
  R* xrs = reinterpret_cast<R*>(un + L::s_xr);
  C* Xc = reinterpret_cast<C*>(un + L::s_X);
  double2* Vd = reinterpret_cast<double2*>(un);

  const int f = blockIdx.x, b = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int N = a.N, T = a.T, F = a.F, K = a.K;
  const size_t FT = (size_t)F * T;
  const C* X = a.X + ((size_t)b * F + f) * T * M;
  const R* xt = a.xt + ((size_t)b * F + f) * T * M;
  const R* lam = a.lam + (size_t)b * N * FT + (size_t)f * T;
  R* gg = a.g + (size_t)b * N * F * M + (size_t)f * M;
  const R fl = a.floorp[b];
  long long* tstamp = (a.timing && b == 0) ? a.timing + (size_t)f * 8 : nullptr;
#define FM_STAMP(i) \
  if (tstamp && tid == 0) tstamp[i] = clock64();
  FM_STAMP(0);

  for (int e = tid; e < N * M; e += BS) gs[e] = gg[(size_t)(e / M) * F * M + (e % M)];
  if (tid == 0) {
    int p = 0;
    for (int i = 0; i < M; ++i)
      for (int j = i; j < M; ++j) {
        pairs[2 * p] = i;
        pairs[2 * p + 1] = j;
        ++p;
      }
  }
  __syncthreads();

  // ---- A1: gain statistics + g MU ------------------------------------------
  {
    const int WPN = NW / N;  // warps per source
    const int n1 = warp / WPN, sub = warp % WPN;
    const bool act = n1 < N;
    const int S1 = WPN * 32, s1 = sub * 32 + lane;
    R num[M], den[M];
#pragma unroll
    for (int m = 0; m < M; ++m) num[m] = den[m] = 0;
    // register prefetch of the next chunk's lambda and x~ (one t per thread)
    R lp[NMAX], xp[M];
    auto fetchA1 = [&](int t0) {
      const int t = t0 + tid;
      const int tc = t < T ? t : T - 1;
#pragma unroll
      for (int n = 0; n < NMAX; ++n) {
        lp[n] = R(0);
        if (n >= N) break;
        lp[n] = lam[(size_t)n * FT + tc];
      }
      RowIO<R, M>::load(xt + (size_t)tc * M, xp);
    };
    if (tid < TC) fetchA1(0);
    for (int t0 = 0; t0 < T; t0 += TC) {
      if (tid < TC) {
        const int tl = tid, t = t0 + tl;
        R l[NMAX], x[M];
#pragma unroll
        for (int n = 0; n < NMAX; ++n) l[n] = t < T ? lp[n] : R(0);
#pragma unroll
        for (int m = 0; m < M; ++m) x[m] = xp[m];
        if (t0 + TC < T) fetchA1(t0 + TC);
#pragma unroll
        for (int n = 0; n < NMAX; ++n) {
          if (n >= N) break;
          lamc[n * (TC + 1) + tl] = l[n];
        }
        R iy[M], y[M], xr[M];
        model_power<R, M>(l, gs, N, fl, iy, y);
#pragma unroll
        for (int m = 0; m < M; ++m) {
          if (t >= T) iy[m] = R(0);
          xr[m] = x[m] * iy[m] * iy[m];
        }
        RowIO<R, M>::store(iys + tl * M, iy);
        RowIO<R, M>::store(xrs + tl * M, xr);
      }
      __syncthreads();
      if (act) {
        for (int tl = s1; tl < TC; tl += S1) {
          const R l = lamc[n1 * (TC + 1) + tl];
          R iy[M], xr[M];
          RowIO<R, M>::load(iys + tl * M, iy);
          RowIO<R, M>::load(xrs + tl * M, xr);
#pragma unroll
          for (int m = 0; m < M; ++m) {
            num[m] += l * xr[m];
            den[m] += l * iy[m];
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

  FM_STAMP(1);
  // ---- A2: V_fm accumulation ------------------------------------------------
  {
    const int p = tid % P, s2 = tid / P;
    const bool act = s2 < S2;
    const int pi = pairs[2 * p], pj = pairs[2 * p + 1];
    C v[M];  // (re, im) of V[m][pi][pj]
#pragma unroll
    for (int m = 0; m < M; ++m) v[m] = cmake<C>(0.0, 0.0);
    R lp[NMAX];
    C xp[M];
    auto fetchA2 = [&](int t0) {
      const int t = t0 + tid;
      const int tc = t < T ? t : T - 1;
#pragma unroll
      for (int n = 0; n < NMAX; ++n) {
        lp[n] = R(0);
        if (n >= N) break;
        lp[n] = lam[(size_t)n * FT + tc];
      }
      CRowIO<R, M>::load(X + (size_t)tc * M, xp);
    };
    if (tid < TC) fetchA2(0);
    for (int t0 = 0; t0 < T; t0 += TC) {
      if (tid < TC) {
        const int tl = tid, t = t0 + tl;
        R l[NMAX];
        C xv[M];
#pragma unroll
        for (int n = 0; n < NMAX; ++n) l[n] = lp[n];
#pragma unroll
        for (int m = 0; m < M; ++m) xv[m] = t < T ? xp[m] : cmake<C>(0.0, 0.0);
        if (t0 + TC < T) fetchA2(t0 + TC);
        R iy[M], y[M];
        model_power<R, M>(l, gs, N, fl, iy, y);
#pragma unroll
        for (int m = 0; m < M; ++m)
          if (t >= T) iy[m] = R(0);
        RowIO<R, M>::store(iys + tl * M, iy);
        CRowIO<R, M>::store(Xc + tl * M, xv);
      }
      __syncthreads();
      if (act) {
        // two t per trip: both rows' loads are in flight before the FMAs
        int tl = s2;
        for (; tl + S2 < TC; tl += 2 * S2) {
          const C xi0 = Xc[tl * M + pi], xj0 = Xc[tl * M + pj];
          const C xi1 = Xc[(tl + S2) * M + pi], xj1 = Xc[(tl + S2) * M + pj];
          R iy0[M], iy1[M];
          RowIO<R, M>::load(iys + tl * M, iy0);
          RowIO<R, M>::load(iys + (tl + S2) * M, iy1);
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
        if (tl < TC) {
          const C xi = Xc[tl * M + pi], xj = Xc[tl * M + pj];
          C pr;
          pr.x = xi.x * xj.x + xi.y * xj.y;
          pr.y = xi.y * xj.x - xi.x * xj.y;
          R iy[M];
          RowIO<R, M>::load(iys + tl * M, iy);
#pragma unroll
          for (int m = 0; m < M; ++m) v[m] = fma2(cmake<C>(iy[m], iy[m]), pr, v[m]);
        }
      }
      __syncthreads();
    }
    // fixed-order reduction over the S2 slices into Vd (fp64), then 1/T + mirror
    for (int ss = 0; ss < S2; ++ss) {
      if (act && s2 == ss) {
#pragma unroll
        for (int m = 0; m < M; ++m) {
          double2* d = Vd + ((size_t)m * M + pi) * M + pj;
          if (ss == 0) *d = to_d2(v[m]);
          else *d = cadd(*d, to_d2(v[m]));
        }
      }
      __syncthreads();
    }
    const double invT = 1.0 / (double)T;
    for (int e = tid; e < M * P; e += BS) {
      const int m = e / P, pp = e % P;
      const int i = pairs[2 * pp], j = pairs[2 * pp + 1];
      double2 d = Vd[((size_t)m * M + i) * M + j];
      d = make_double2(d.x * invT, d.y * invT);
      Vd[((size_t)m * M + i) * M + j] = d;
      if (i != j) Vd[((size_t)m * M + j) * M + i] = make_double2(d.x, -d.y);
    }
    __syncthreads();
  }

  // publish the updated gains and V_f (fp64) for k_ip
  {
    double2* Vg = a.V + ((size_t)b * F + f) * M * M * M;
    for (int e = tid; e < M * M * M; e += BS) Vg[e] = Vd[e];
    for (int e = tid; e < N * M; e += BS) gg[(size_t)(e / M) * F * M + (e % M)] = gs[e];
  }
  FM_STAMP(2);
#undef FM_STAMP
}

// ---------------------------------------------------------------------------
// k_ip: iterative projection + normalisations, one small CTA per (f, b):
// warp 0 inverts [Q | I] (pivoted Gauss-Jordan; also log|det Q|) while warps
// 1.. invert the HPD V_fm in parallel; warp 0 then runs the M sequential row
// updates (one mat-vec each); all threads normalise and fold into W.
// ---------------------------------------------------------------------------
template <typename R> struct IpArgs {
  const double2* V;  // (B, F, M, M, M) from k_front
  cplx<R>* Q;
  R* g;
  R* W;
  R* cs_out;
  double* ld_part;
  const unsigned* iter;
  unsigned long long* status;
  int F, N, K;
  long long f_offset;
  int normalize, ip_sweeps;
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
  using C = cplx<R>;
  using L = IpSmem<R, M>;
  constexpr int NW = IpCfg<M>::NW, BS = IpCfg<M>::BS;
  extern __shared__ __align__(16) unsigned char sm[];
  double2* Vd = reinterpret_cast<double2*>(sm + L::o_Vd);
  double2* Qd = reinterpret_cast<double2*>(sm + L::o_Qd);
  double2* Ai = reinterpret_cast<double2*>(sm + L::o_Ai);
  double2* ub = reinterpret_cast<double2*>(sm + L::o_vec);
  double2* qb = ub + M;
  double2* sk = qb + M;
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
  R* Wg = a.W + (size_t)b * N * F * K + (size_t)f * K;
  const unsigned it = *a.iter;
  const long long fglob = a.f_offset + f;
  const double2* Vg = a.V + ((size_t)b * F + f) * M * M * M;
  for (int e = tid; e < M * M * M; e += BS) Vd[e] = Vg[e];
  for (int e = tid; e < M * M; e += BS) Qd[e] = to_d2(Qg[e]);
  for (int e = tid; e < N * M; e += BS) gs[e] = gg[(size_t)(e / M) * F * M + (e % M)];
  if (tid < NMAX) cs[tid] = R(1);
  if (tid == 0) flags[0] = flags[1] = 0;
  __syncthreads();
  // ---- A3: iterative projection (spatial.py:181-199) -------------------------
  {
    if (warp == 0) {
      // [Q | I] -> Q^-1 and log|det Q|
      for (int e = lane; e < M * 2 * M; e += 32) {
        const int r = e / (2 * M), c = e % (2 * M);
        Ai[e] = c < M ? Qd[r * M + c] : make_double2(c - M == r ? 1.0 : 0.0, 0.0);
      }
      __syncwarp();
      double la = 0.0;
      const bool ok = warp_inv_pivot<M>(Ai, lane, &la);
      if (lane == 0) {
        misc[0] = la;
        flags[0] = ok ? 0 : 1;
      }
    }
    for (int m = warp - 1; warp > 0 && m < M; m += NW - 1) {
      const bool ok = warp_inv_hpd<M>(Vd + (size_t)m * M * M, lane);
      if (lane == 0) vfail[m] = ok ? 0 : 1;
    }
    __syncthreads();
    if (warp == 0) {
      double ldet = misc[0], nprod = 1.0;
      int code = flags[0] ? 2 : 0, bad_m = 0;  // singular Q -> singular Q V at m = 0
      for (int sw = 0; sw < a.ip_sweeps && code == 0; ++sw) {
        for (int m = 0; m < M; ++m) {
          if (vfail[m]) {
            code = 1;
            bad_m = m;
            break;
          }
          const double2* Vi = Vd + (size_t)m * M * M;
          if (lane < M) ub[lane] = Ai[lane * 2 * M + M + m];  // u = Q^-1 e_m
          __syncwarp();
          double2 q = make_double2(0.0, 0.0);
          double part = 0.0;
          if (lane < M) {
#pragma unroll
            for (int j = 0; j < M; ++j) q = cadd(q, cmul(Vi[lane * M + j], ub[j]));
            const double2 u = ub[lane];
            part = q.x * u.x + q.y * u.y;  // Re(conj(q_i) u_i)
          }
          const double nrm = warp_sum(part);  // = q^H V q  (spatial.py:193)
          if (!(nrm > 0.0) || !isfinite(nrm)) {
            code = 1;
            bad_m = m;
            break;
          }
          const double isn = rsqrt(nrm);  // 1 / sqrt(norm)
          if (lane < M) {  // new row r = conj(q / sqrt(norm))  (spatial.py:199)
            const double2 r = make_double2(q.x * isn, -(q.y * isn));
            qb[lane] = r;
            Qd[m * M + lane] = r;
          }
          __syncwarp();
          if (lane < M) {  // s = (r Q^-1 - e_m^T) / sqrt(norm)
            double2 s = make_double2(0.0, 0.0);
#pragma unroll
            for (int j = 0; j < M; ++j) s = cadd(s, cmul(qb[j], Ai[j * 2 * M + M + lane]));
            if (lane == m) s.x -= 1.0;
            sk[lane] = make_double2(s.x * isn, s.y * isn);
          }
          __syncwarp();
          for (int e = lane; e < M * M; e += 32) {  // Q^-1 -= u s / sqrt(norm)
            const int i = e / M, k = e % M;
            double2* d = Ai + i * 2 * M + M + k;
            *d = csub(*d, cmul(ub[i], sk[k]));
          }
          nprod *= nrm;  // log|det Q| += log sqrt(norm) (determinant lemma)
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
    if (tid == 0) {
      double s = 0.0;
      for (int m = 0; m < M; ++m) s += log(rown[m]);
      misc[1] -= s;
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
    for (int e = tid; e < N * K; e += BS) {
      const int n = e / K, k = e % K;
      R* wp = Wg + (size_t)n * F * K + k;
      *wp = *wp * cs[n];
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

template <typename R, int M>
__global__ void __launch_bounds__(256, 2) k_back(BackArgs<R> a) {
  using C = cplx<R>;
  __shared__ C Qr[M * M];
  __shared__ __align__(16) R gs[NMAX * M];
  __shared__ R cs[NMAX];
  __shared__ double dred[8];
  __shared__ int is_last;
  const int f = blockIdx.x, b = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int N = a.N, T = a.T, F = a.F;
  const size_t FT = (size_t)F * T;
  const C* X = a.X + ((size_t)b * F + f) * T * M;
  R* xt = a.xt + ((size_t)b * F + f) * T * M;
  const R* lam = a.lam + (size_t)b * N * FT + (size_t)f * T;
  R* phi = a.phi + (size_t)b * 2 * N * FT + (size_t)f * T;
  const R fl = a.floorp[b];
  for (int e = tid; e < M * M; e += 256) Qr[e] = a.Q[((size_t)b * F + f) * M * M + e];
  for (int e = tid; e < N * M; e += 256)
    gs[e] = a.g[(size_t)b * N * F * M + (size_t)(e / M) * F * M + (size_t)f * M + (e % M)];
  if (tid < NMAX) cs[tid] = a.cs ? a.cs[((size_t)b * F + f) * NMAX + tid] : R(1);
  __syncthreads();
  double ll = 0.0;
  // register prefetch of the next step's x row and lambda values
  C xp[M];
  R lp[NMAX];
  auto fetch = [&](int t) {
    CRowIO<R, M>::load(X + (size_t)t * M, xp);
#pragma unroll
    for (int n = 0; n < NMAX; ++n) {
      lp[n] = R(0);
      if (n >= N) break;
      lp[n] = lam[(size_t)n * FT + t];
    }
  };
  if (tid < T) fetch(tid);
  for (int t = tid; t < T; t += 256) {
    // compiler barrier: re-read the (broadcast) shared-memory parameters each
    // step instead of hoisting M*M + N*M of them into registers
    asm volatile("" ::: "memory");
    C xv[M];
    R l[NMAX];
#pragma unroll
    for (int m = 0; m < M; ++m) xv[m] = xp[m];
#pragma unroll
    for (int n = 0; n < NMAX; ++n) l[n] = lp[n] * cs[n];
    if (t + 256 < T) fetch(t + 256);
    R xtv[M];
#pragma unroll
    for (int i = 0; i < M; ++i) {
      C s = cmake<C>(0.0, 0.0);
#pragma unroll
      for (int j = 0; j < M; ++j) {
        const C q = Qr[i * M + j];
        s = fma2(cmake<C>(q.x, q.x), xv[j], s);
        s = fma2(cmake<C>(-q.y, q.y), cmake<C>(xv[j].y, xv[j].x), s);
      }
      xtv[i] = s.x * s.x + s.y * s.y;
    }
    RowIO<R, M>::store(xt + (size_t)t * M, xtv);
    R iy[M], y[M];
    model_power<R, M>(l, gs, N, fl, iy, y);
    R llt = 0;
#pragma unroll
    for (int m = 0; m < M; ++m) llt += -xtv[m] * iy[m] - log_fast(y[m]);
    ll += (double)llt;
    phi_point<R, M>(xtv, iy, gs, N, phi, FT, (size_t)t);
  }
  ll = warp_sum(ll);
  if (lane == 0) dred[warp] = ll;
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
    for (int w = 0; w < 8; ++w) s += dred[w];
    a.ll_part[(size_t)b * F + f] = s;
  }
  if (a.record) {
    if (tid == 0) {
      __threadfence();
      const unsigned prev = atomicAdd(a.counter, 1u);
      is_last = (prev == gridDim.x * gridDim.y - 1);
    }
    __syncthreads();
    if (is_last) {
      __threadfence();
      const unsigned it = *a.iter;
      for (int bb = tid; bb < a.B; bb += 256) {
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
