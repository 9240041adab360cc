// fm_fullrank.cuh -- the full-rank MNMF comparator on the device (SURVEY
// §8(f) 4): the slow model the paper's speed-up is measured against
// (PAPER.md:650-653), method="mnmf" (separate.py:83-107, 128-172).
//
//   k_fr_bin   per (f, t): Y = sum_n lam G + ridge I, Cholesky (log|Y| on the
//              fly), z = Y^-1 x, Yi = L^-H L^-1, trace x^H z, and per source
//              phi1 = z^H G z, phi2 = tr(G Yi)  (_kernels.py:62-163)
//   k_fr_ab    A_nf = sum_t lam z z^H, B_nf = sum_t lam Yi (upper triangle,
//              sequential over t as the numba loop, mirrored)
//   k_fr_scm   per (n, f): G <- B^-1/2 (B^1/2 G A G B^1/2)^1/2 B^-1/2, the
//              symmetrisations, eigenvalue clamps and breakdown check of
//              update_scm / hermitian_sqrt_pair / clamp_psd (spatial.py:145-
//              169, linalg.py:85-109), then normalize_trace (spatial.py:252-
//              257): warp-level cyclic complex Jacobi (fm_linalg.cuh)
//   k_fr_wiener  lam G Y^-1 x with the partition defect redistributed by
//              power share (separate.py:83-107)
// All per-bin linear algebra is fp64 (storage in the run's precision).
// Status word: code 1 = negative spectrum in the SCM update at (n, f)
// (NumericalBreakdownError), code 2 = non-positive-definite mixture
// covariance at (f, t) (singular Y); key = t << 44 | n << 24 | f << 2 | code.
#pragma once
#include "fm_common.cuh"
#include "fm_linalg.cuh"

namespace fm {

constexpr int FR_MMAX = 8;

template <typename R, int M>
__global__ void __launch_bounds__(128) k_fr_bin(const cplx<R>* __restrict__ X, const cplx<R>* __restrict__ G,
                                                const R* __restrict__ lam, double ridge, int N, int F,
                                                int T, int want_phi, R* __restrict__ phi,
                                                cplx<R>* __restrict__ Zs, cplx<R>* __restrict__ Yis,
                                                double* __restrict__ llp) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (long long)F * T) return;
  const int f = (int)(e / T), t = (int)(e % T);
  double2 L[M][M], Li[M][M], z[M];
  // Y (lower triangle) = sum_n lam G + ridge I
#pragma unroll
  for (int i = 0; i < M; ++i)
#pragma unroll
    for (int j = 0; j <= i; ++j) {
      double2 acc = make_double2(0.0, 0.0);
      for (int n = 0; n < N; ++n) {
        const double l = (double)lam[((size_t)n * F + f) * T + t];
        const cplx<R> g = G[(((size_t)n * F + f) * M + i) * M + j];
        acc.x += l * (double)g.x;
        acc.y += l * (double)g.y;
      }
      L[i][j] = acc;
    }
#pragma unroll
  for (int i = 0; i < M; ++i) L[i][i].x += ridge;
  // Cholesky Y = L L^H, log|Y| on the fly
  double logdet = 0.0;  // (a non-PD Y gives NaN, as the numba loop does)
#pragma unroll
  for (int i = 0; i < M; ++i) {
#pragma unroll
    for (int j = 0; j <= i; ++j) {
      double2 s = L[i][j];
#pragma unroll
      for (int k = 0; k < j; ++k) s = csub(s, cmulc(L[i][k], L[j][k]));
      if (i == j) {
        const double d = sqrt(s.x);
        L[i][i] = make_double2(d, 0.0);
        logdet += 2.0 * log(d);
      } else {
        L[i][j] = make_double2(s.x / L[j][j].x, s.y / L[j][j].x);
      }
    }
  }
  // z = Y^-1 x: forward then backward substitution
#pragma unroll
  for (int i = 0; i < M; ++i) {
    const cplx<R> xv = X[((size_t)f * T + t) * M + i];
    double2 s = make_double2((double)xv.x, (double)xv.y);
#pragma unroll
    for (int k = 0; k < i; ++k) s = csub(s, cmul(L[i][k], z[k]));
    z[i] = make_double2(s.x / L[i][i].x, s.y / L[i][i].x);
  }
#pragma unroll
  for (int i = M - 1; i >= 0; --i) {
    double2 s = z[i];
#pragma unroll
    for (int k = i + 1; k < M; ++k) s = csub(s, cmul(make_double2(L[k][i].x, -L[k][i].y), z[k]));
    z[i] = make_double2(s.x / L[i][i].x, s.y / L[i][i].x);
  }
  // Li = L^-1 (lower), Yi = Li^H Li
#pragma unroll
  for (int i = 0; i < M; ++i) {
    Li[i][i] = make_double2(1.0 / L[i][i].x, 0.0);
#pragma unroll
    for (int j = 0; j < i; ++j) {
      double2 s = make_double2(0.0, 0.0);
#pragma unroll
      for (int k = j; k < i; ++k) s = cadd(s, cmul(L[i][k], Li[k][j]));
      Li[i][j] = make_double2(-s.x / L[i][i].x, -s.y / L[i][i].x);
    }
  }
  double2 Yi[M][M];
#pragma unroll
  for (int i = 0; i < M; ++i)
#pragma unroll
    for (int j = 0; j <= i; ++j) {
      double2 s = make_double2(0.0, 0.0);
#pragma unroll
      for (int k = i; k < M; ++k) s = cadd(s, cmul(make_double2(Li[k][i].x, -Li[k][i].y), Li[k][j]));
      Yi[i][j] = s;
      Yi[j][i] = make_double2(s.x, -s.y);
    }
  double tr = 0.0;
#pragma unroll
  for (int i = 0; i < M; ++i) {
    const cplx<R> xv = X[((size_t)f * T + t) * M + i];
    tr += (double)xv.x * z[i].x + (double)xv.y * z[i].y;  // Re(conj(x) z)
  }
  llp[e] = -tr - logdet;
  if (want_phi) {
    const size_t FT = (size_t)F * T;
    for (int n = 0; n < N; ++n) {
      double p1 = 0.0, p2 = 0.0;
#pragma unroll
      for (int i = 0; i < M; ++i) {
        double2 gz = make_double2(0.0, 0.0);
#pragma unroll
        for (int j = 0; j < M; ++j) {
          const cplx<R> gv = G[(((size_t)n * F + f) * M + i) * M + j];
          const double2 g = make_double2((double)gv.x, (double)gv.y);
          gz = cadd(gz, cmul(g, z[j]));
          p2 += cmul(g, Yi[j][i]).x;
        }
        p1 += z[i].x * gz.x + z[i].y * gz.y;  // Re(conj(z_i) gz)
      }
      phi[(size_t)n * FT + (size_t)f * T + t] = (R)p1;
      phi[(size_t)(N + n) * FT + (size_t)f * T + t] = (R)p2;
    }
  }
  if (Zs) {
#pragma unroll
    for (int i = 0; i < M; ++i) Zs[(size_t)e * M + i] = cmake<cplx<R>>(z[i].x, z[i].y);
#pragma unroll
    for (int i = 0; i < M; ++i)
#pragma unroll
      for (int j = 0; j < M; ++j)
        Yis[((size_t)e * M + i) * M + j] = cmake<cplx<R>>(Yi[i][j].x, Yi[i][j].y);
  }
}

// A, B (N, F, M, M): thread per (n, f, i <= j), sequential over t; fp64 sums
template <typename R, int M>
__global__ void k_fr_ab(const R* __restrict__ lam, const cplx<R>* __restrict__ Zs,
                        const cplx<R>* __restrict__ Yis, int N, int F, int T, cplx<R>* __restrict__ A,
                        cplx<R>* __restrict__ B) {
  constexpr int P = M * (M + 1) / 2;
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (long long)N * F * P) return;
  const int n = (int)(e / ((long long)F * P)), f = (int)((e / P) % F);
  int i = 0, r = (int)(e % P);
  while (r >= M - i) {
    r -= M - i;
    ++i;
  }
  const int j = i + r;
  double2 a = make_double2(0.0, 0.0), b = make_double2(0.0, 0.0);
  for (int t = 0; t < T; ++t) {
    const double l = (double)lam[((size_t)n * F + f) * T + t];
    const size_t ft = (size_t)f * T + t;
    const cplx<R> zi = Zs[ft * M + i], zj = Zs[ft * M + j];
    const cplx<R> y = Yis[(ft * M + i) * M + j];
    const double2 zz = cmulc(make_double2(zi.x, zi.y), make_double2(zj.x, zj.y));  // z_i conj(z_j)
    a.x += l * zz.x;
    a.y += l * zz.y;
    b.x += l * (double)y.x;
    b.y += l * (double)y.y;
  }
  const size_t o = ((size_t)n * F + f) * M * M;
  A[o + i * M + j] = cmake<cplx<R>>(a.x, a.y);
  B[o + i * M + j] = cmake<cplx<R>>(b.x, b.y);
  if (i != j) {
    A[o + j * M + i] = cmake<cplx<R>>(a.x, -a.y);
    B[o + j * M + i] = cmake<cplx<R>>(b.x, -b.y);
  }
}

// fixed-order sum of n doubles (one CTA): strided per-thread sums + tree
static __global__ void __launch_bounds__(256) k_sum_fixed(const double* __restrict__ v, long long n,
                                                   double* __restrict__ out) {
  __shared__ double red[256];
  double s = 0.0;
  for (long long e = threadIdx.x; e < n; e += 256) s += v[e];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = red[0];
}

// ---- the SCM update (one warp per (n, f)) ------------------------------------
template <int M>
__device__ void wmatmul(const double2* Am, const double2* Bm, double2* Cm, int lane, bool conjB = false) {
  for (int e = lane; e < M * M; e += 32) {
    const int i = e / M, j = e % M;
    double2 s = make_double2(0.0, 0.0);
    for (int k = 0; k < M; ++k) {
      double2 bv = Bm[k * M + j];
      s = cadd(s, cmul(Am[i * M + k], bv));
    }
    Cm[e] = s;
  }
  __syncwarp();
}

template <int M>
__device__ void wsym(double2* Am, int lane) {  // 0.5 (A + A^H)
  double2 v[2];
  for (int e = lane, q = 0; e < M * M; e += 32, ++q) {
    const int i = e / M, j = e % M;
    const double2 a = Am[i * M + j], b = Am[j * M + i];
    v[q] = make_double2(0.5 * (a.x + b.x), 0.5 * (a.y - b.y));
  }
  __syncwarp();
  for (int e = lane, q = 0; e < M * M; e += 32, ++q) Am[e] = v[q];
  __syncwarp();
}

// out = V diag(d) V^H
template <int M>
__device__ void wrecon(const double2* V, const double* d, double2* out, int lane) {
  for (int e = lane; e < M * M; e += 32) {
    const int i = e / M, j = e % M;
    double2 s = make_double2(0.0, 0.0);
    for (int k = 0; k < M; ++k) {
      const double2 a = V[i * M + k], b = V[j * M + k];
      const double2 p = cmulc(a, b);  // V_ik conj(V_jk)
      s.x += d[k] * p.x;
      s.y += d[k] * p.y;
    }
    out[e] = s;
  }
  __syncwarp();
}

// grid (F, N), block 32
template <typename R, int M>
__global__ void __launch_bounds__(32) k_fr_scm(cplx<R>* __restrict__ G, const cplx<R>* __restrict__ A,
                                               const cplx<R>* __restrict__ B, int F, int normalize,
                                               R* __restrict__ cout, unsigned long long* __restrict__ status) {
  __shared__ double2 Bm[M * M], Gm[M * M], Am[M * M], V[M * M], S1[M * M], S2[M * M], T1[M * M];
  __shared__ double w[M], d1[M], d2[M];
  const int f = blockIdx.x, n = blockIdx.y, lane = threadIdx.x;
  const size_t o = ((size_t)n * F + f) * M * M;
  for (int e = lane; e < M * M; e += 32) {
    Bm[e] = make_double2((double)B[o + e].x, (double)B[o + e].y);
    Gm[e] = make_double2((double)G[o + e].x, (double)G[o + e].y);
    Am[e] = make_double2((double)A[o + e].x, (double)A[o + e].y);
  }
  __syncwarp();
  // hermitian_sqrt_pair(B) (linalg.py:97-109)
  wsym<M>(Bm, lane);
  warp_jacobi_eigh<M>(Bm, V, lane);
  if (lane == 0) {
    double top = -INFINITY;
    for (int k = 0; k < M; ++k) top = fmax(top, Bm[k * M + k].x);
    top = fmax(top, DBL_MIN);
    for (int k = 0; k < M; ++k) {
      const double wk = fmax(Bm[k * M + k].x, 1e-12 * top);
      d1[k] = sqrt(wk);
      d2[k] = 1.0 / sqrt(wk);
    }
  }
  __syncwarp();
  wrecon<M>(V, d1, S1, lane);  // B^1/2
  wrecon<M>(V, d2, S2, lane);  // B^-1/2
  // C = Bs G A G Bs (spatial.py:154), symmetrised
  wmatmul<M>(S1, Gm, T1, lane);
  wmatmul<M>(T1, Am, Bm, lane);
  wmatmul<M>(Bm, Gm, T1, lane);
  wmatmul<M>(T1, S1, Bm, lane);
  wsym<M>(Bm, lane);
  warp_jacobi_eigh<M>(Bm, V, lane);
  if (lane == 0) {
    double top = -INFINITY;
    for (int k = 0; k < M; ++k) top = fmax(top, Bm[k * M + k].x);
    top = fmax(top, 0.0);
    bool bad = false;
    for (int k = 0; k < M; ++k) {
      const double wk = Bm[k * M + k].x;
      if (wk < -1e-8 * top) bad = true;  // BREAKDOWN_TOL (spatial.py:33, :160-167)
      d1[k] = sqrt(fmax(wk, 0.0));
    }
    if (bad) report_status(status, 0u, n, f, 1);
  }
  __syncwarp();
  wrecon<M>(V, d1, T1, lane);          // C^1/2
  wmatmul<M>(S2, T1, Bm, lane);        // Bis Cs
  wmatmul<M>(Bm, S2, T1, lane);        // Bis Cs Bis
  // clamp_psd (linalg.py:85-94)
  wsym<M>(T1, lane);
  warp_jacobi_eigh<M>(T1, V, lane);
  if (lane == 0) {
    double top = -INFINITY;
    for (int k = 0; k < M; ++k) top = fmax(top, T1[k * M + k].x);
    top = fmax(top, 0.0);
    for (int k = 0; k < M; ++k) w[k] = fmax(T1[k * M + k].x, 1e-12 * top);
  }
  __syncwarp();
  wrecon<M>(V, w, Gm, lane);
  double scl = 1.0;
  if (normalize) {  // normalize_trace (spatial.py:252-257)
    double tr = 0.0;
    for (int k = 0; k < M; ++k) tr += Gm[k * M + k].x;
    tr = fmax(tr, DBL_MIN);
    scl = (double)M / tr;
    if (lane == 0) cout[(size_t)n * F + f] = (R)(tr / (double)M);
  }
  for (int e = lane; e < M * M; e += 32) G[o + e] = cmake<cplx<R>>(Gm[e].x * scl, Gm[e].y * scl);
}

// images (N, F, T, M) = lam G Y^-1 x + share * defect (separate.py:83-107); thread per (f, t)
template <typename R, int M>
__global__ void __launch_bounds__(128) k_fr_wiener(const R* __restrict__ lam, const cplx<R>* __restrict__ G,
                                                   const cplx<R>* __restrict__ X, double ridge, int N,
                                                   int F, int T, cplx<R>* __restrict__ out,
                                                   unsigned long long* __restrict__ status) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (long long)F * T) return;
  const int f = (int)(e / T), t = (int)(e % T);
  double2 L[M][M], z[M], xv[M];
#pragma unroll
  for (int i = 0; i < M; ++i)
#pragma unroll
    for (int j = 0; j <= i; ++j) {
      double2 acc = make_double2(0.0, 0.0);
      for (int n = 0; n < N; ++n) {
        const double l = (double)lam[((size_t)n * F + f) * T + t];
        const cplx<R> g = G[(((size_t)n * F + f) * M + i) * M + j];
        acc.x += l * (double)g.x;
        acc.y += l * (double)g.y;
      }
      L[i][j] = acc;
    }
#pragma unroll
  for (int i = 0; i < M; ++i) L[i][i].x += ridge;
  bool ok = true;
#pragma unroll
  for (int i = 0; i < M; ++i)
#pragma unroll
    for (int j = 0; j <= i; ++j) {
      double2 s = L[i][j];
#pragma unroll
      for (int k = 0; k < j; ++k) s = csub(s, cmulc(L[i][k], L[j][k]));
      if (i == j) {
        if (!(s.x > 0.0)) ok = false;
        L[i][i] = make_double2(sqrt(s.x > 0.0 ? s.x : 1.0), 0.0);
      } else {
        L[i][j] = make_double2(s.x / L[j][j].x, s.y / L[j][j].x);
      }
    }
  if (!ok) report_status(status, (unsigned)t, 0, f, 2);
#pragma unroll
  for (int i = 0; i < M; ++i) {
    const cplx<R> x0 = X[((size_t)f * T + t) * M + i];
    xv[i] = make_double2((double)x0.x, (double)x0.y);
    double2 s = xv[i];
#pragma unroll
    for (int k = 0; k < i; ++k) s = csub(s, cmul(L[i][k], z[k]));
    z[i] = make_double2(s.x / L[i][i].x, s.y / L[i][i].x);
  }
#pragma unroll
  for (int i = M - 1; i >= 0; --i) {
    double2 s = z[i];
#pragma unroll
    for (int k = i + 1; k < M; ++k) s = csub(s, cmul(make_double2(L[k][i].x, -L[k][i].y), z[k]));
    z[i] = make_double2(s.x / L[i][i].x, s.y / L[i][i].x);
  }
  double total = 0.0;
  for (int n = 0; n < N; ++n) total += (double)lam[((size_t)n * F + f) * T + t];
  double2 sum[M];
#pragma unroll
  for (int i = 0; i < M; ++i) sum[i] = make_double2(0.0, 0.0);
  const size_t FTM = (size_t)F * T * M;
  for (int n = 0; n < N; ++n) {
    const double l = (double)lam[((size_t)n * F + f) * T + t];
#pragma unroll
    for (int i = 0; i < M; ++i) {
      double2 s = make_double2(0.0, 0.0);
#pragma unroll
      for (int j = 0; j < M; ++j) {
        const cplx<R> gv = G[(((size_t)n * F + f) * M + i) * M + j];
        s = cadd(s, cmul(make_double2((double)gv.x, (double)gv.y), z[j]));
      }
      s = make_double2(l * s.x, l * s.y);
      sum[i] = cadd(sum[i], s);
      out[(size_t)n * FTM + ((size_t)f * T + t) * M + i] = cmake<cplx<R>>(s.x, s.y);
    }
  }
  for (int n = 0; n < N; ++n) {
    const double l = (double)lam[((size_t)n * F + f) * T + t];
    const double share = total > 0.0 ? l / total : 1.0 / (double)N;
#pragma unroll
    for (int i = 0; i < M; ++i) {
      const size_t oi = (size_t)n * FTM + ((size_t)f * T + t) * M + i;
      const cplx<R> im = out[oi];
      const double dx = xv[i].x - sum[i].x, dy = xv[i].y - sum[i].y;
      out[oi] = cmake<cplx<R>>((double)im.x + share * dx, (double)im.y + share * dy);
    }
  }
}

}  // namespace fm

namespace fm {

// NMF MU steps of the comparator from the full-rank phi (sources.py:191-198):
// W step: thread per (n, f, k), sum over t; H step: thread per (n, k, t), sum over f
template <typename R>
__global__ void k_fr_nmf_mu(const R* __restrict__ phi, R* __restrict__ W, R* __restrict__ H, int N,
                            int F, int T, int K, int step) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t FT = (size_t)F * T;
  if (step == 0) {
    if (e >= (long long)N * F * K) return;
    const int n = (int)(e / ((long long)F * K)), f = (int)((e / K) % F), k = (int)(e % K);
    double a = 0.0, c = 0.0;
    for (int t = 0; t < T; ++t) {
      const double h = (double)H[((size_t)n * K + k) * T + t];
      a += (double)phi[(size_t)n * FT + (size_t)f * T + t] * h;
      c += (double)phi[(size_t)(N + n) * FT + (size_t)f * T + t] * h;
    }
    W[e] = (R)((double)W[e] * sqrt(a / fmax(c, DBL_MIN)));
  } else {
    if (e >= (long long)N * K * T) return;
    const int n = (int)(e / ((long long)K * T)), k = (int)((e / T) % K), t = (int)(e % T);
    double a = 0.0, c = 0.0;
    for (int f = 0; f < F; ++f) {
      const double w = (double)W[((size_t)n * F + f) * K + k];
      a += w * (double)phi[(size_t)n * FT + (size_t)f * T + t];
      c += w * (double)phi[(size_t)(N + n) * FT + (size_t)f * T + t];
    }
    H[e] = (R)((double)H[e] * sqrt(a / fmax(c, DBL_MIN)));
  }
}

// W_nfk *= c_nf (absorb_scale, sources.py:202-204)
template <typename R>
__global__ void k_fr_absorb(R* __restrict__ W, const R* __restrict__ c, long long NF, int K) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= NF * K) return;
  W[e] = W[e] * c[e / K];
}

// G_nf = Q_f^-1 Diag(g_nf) Q_f^-H (reconstruct_scm, spatial.py:211-223); thread per f
template <typename R, int M>
__global__ void k_fr_reconstruct(const cplx<R>* __restrict__ Q, const R* __restrict__ g, int N, int F,
                                 cplx<R>* __restrict__ G, unsigned long long* __restrict__ status) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= F) return;
  double2 A[M][2 * M];
#pragma unroll
  for (int i = 0; i < M; ++i)
#pragma unroll
    for (int j = 0; j < 2 * M; ++j) {
      if (j < M) {
        const cplx<R> q = Q[((size_t)f * M + i) * M + j];
        A[i][j] = make_double2((double)q.x, (double)q.y);
      } else {
        A[i][j] = make_double2(j - M == i ? 1.0 : 0.0, 0.0);
      }
    }
  // Gauss-Jordan with partial pivoting on [Q | I]
  for (int c = 0; c < M; ++c) {
    int piv = c;
    double best = cabs1(A[c][c]);
    for (int r = c + 1; r < M; ++r)
      if (cabs1(A[r][c]) > best) { best = cabs1(A[r][c]); piv = r; }
    if (!(best > 0.0)) { report_status(status, 0u, 0, f, 3); return; }
    if (piv != c)
      for (int j = 0; j < 2 * M; ++j) { const double2 tmp = A[c][j]; A[c][j] = A[piv][j]; A[piv][j] = tmp; }
    const double2 inv = cdiv(make_double2(1.0, 0.0), A[c][c]);
    for (int j = 0; j < 2 * M; ++j) A[c][j] = cmul(A[c][j], inv);
    for (int r = 0; r < M; ++r) {
      if (r == c) continue;
      const double2 fct = A[r][c];
      for (int j = 0; j < 2 * M; ++j) A[r][j] = csub(A[r][j], cmul(fct, A[c][j]));
    }
  }
  for (int n = 0; n < N; ++n)
#pragma unroll
    for (int i = 0; i < M; ++i)
#pragma unroll
      for (int k = 0; k < M; ++k) {
        double2 s = make_double2(0.0, 0.0);
#pragma unroll
        for (int j = 0; j < M; ++j) {
          const double gj = (double)g[((size_t)n * F + f) * M + j];
          const double2 p = cmulc(A[i][M + j], A[k][M + j]);  // Qi_ij conj(Qi_kj)
          s.x += gj * p.x;
          s.y += gj * p.y;
        }
        G[(((size_t)n * F + f) * M + i) * M + k] = cmake<cplx<R>>(s.x, s.y);
      }
}

}  // namespace fm
