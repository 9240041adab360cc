// fm_ops.cuh -- per-op kernels behind the _kernels.py-seam entry points of
// fastmnmf.h (fm_fast_stats, fm_mix_power, fm_ip_weights, fm_project_power,
// fm_update_diagonalizer, fm_logdet, fm_wiener_fast) and the observation
// prologue of run(). Single-mixture layouts as in the reference (no batch).
#pragma once
#include "fm_common.cuh"
#include "fm_linalg.cuh"

namespace fm {

// _kernels.fast_stats (_kernels.py:208-251). grid F, block 256.
// phi1/phi2 (N,F,T) written if non-null; gnum/gden (N,F,M) if non-null;
// ll_part[f] = sum_{t,m} (-x~/y - log y).
template <typename R, int M>
__global__ void __launch_bounds__(256) k_fast_stats(const R* __restrict__ xt, const R* __restrict__ g,
                                                    const R* __restrict__ lam, R fl, int N, int F,
                                                    int T, R* phi1, R* phi2, R* gnum, R* gden,
                                                    double* ll_part) {
  __shared__ double red[8];
  __shared__ R gsh[8 * 16 * 2];
  const int f = blockIdx.x, tid = threadIdx.x;
  const size_t FT = (size_t)F * T;
  R* gsm = gsh;  // N*M <= 8*16
  for (int e = tid; e < N * M; e += 256) gsm[e] = g[(size_t)(e / M) * F * M + (size_t)f * M + e % M];
  __syncthreads();
  double ll = 0.0;
  for (int t = tid; t < T; t += 256) {
    R x[M], y[M];
    RowIO<R, M>::load(xt + ((size_t)f * T + t) * M, x);
    R llt = 0;
#pragma unroll
    for (int m = 0; m < M; ++m) {
      R acc = 0;
      for (int n = 0; n < N; ++n) acc += lam[n * FT + (size_t)f * T + t] * gsm[n * M + m];
      y[m] = floor_max(acc, fl);
      llt += -x[m] / y[m] - log_r(y[m]);
    }
    ll += (double)llt;
    if (phi1) {
      for (int n = 0; n < N; ++n) {
        R p1 = 0, p2 = 0;
#pragma unroll
        for (int m = 0; m < M; ++m) {
          const R iy = R(1) / y[m];
          p1 += gsm[n * M + m] * x[m] * iy * iy;
          p2 += gsm[n * M + m] * iy;
        }
        phi1[n * FT + (size_t)f * T + t] = p1;
        phi2[n * FT + (size_t)f * T + t] = p2;
      }
    }
  }
  ll = warp_sum(ll);
  if ((tid & 31) == 0) red[tid >> 5] = ll;
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
    for (int w = 0; w < 8; ++w) s += red[w];
    ll_part[f] = s;
  }
  if (gnum) {
    // thread = (n, m) entry, sequential over t (fixed order)
    for (int e = tid; e < N * M; e += 256) {
      const int n = e / M, m = e % M;
      R sn = 0, sd = 0;
      for (int t = 0; t < T; ++t) {
        R acc = 0;
        for (int nn = 0; nn < N; ++nn) acc += lam[nn * FT + (size_t)f * T + t] * gsm[nn * M + m];
        const R y = floor_max(acc, fl);
        const R iy = R(1) / y;
        const R la = lam[n * FT + (size_t)f * T + t];
        sn += la * xt[((size_t)f * T + t) * M + m] * iy * iy;
        sd += la * iy;
      }
      gnum[(size_t)n * F * M + (size_t)f * M + m] = sn;
      gden[(size_t)n * F * M + (size_t)f * M + m] = sd;
    }
  }
}

// _kernels.mix_power (_kernels.py:310-322): one thread per (f, t).
template <typename R>
__global__ void k_mix_power(const R* __restrict__ lam, const R* __restrict__ g, R fl, int N, int F,
                            int T, int M, R* __restrict__ y) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)F * T) return;
  const long long f = i / T;
  const size_t FT = (size_t)F * T;
  for (int m = 0; m < M; ++m) {
    R acc = 0;
    for (int n = 0; n < N; ++n) acc += lam[n * FT + i] * g[((size_t)n * F + f) * M + m];
    y[i * M + m] = floor_max(acc, fl);
  }
}

// _kernels.ip_weights (_kernels.py:276-293): V (F,M,M,M). grid F, block 256;
// thread = (pair i<=j, slice), fixed-order slice reduction through smem.
template <typename R, int M>
__global__ void __launch_bounds__(256) k_ip_weights(const cplx<R>* __restrict__ X,
                                                    const R* __restrict__ y, int T,
                                                    cplx<R>* __restrict__ V) {
  using C = cplx<R>;
  constexpr int P = M * (M + 1) / 2;
  constexpr int S = 256 / P;
  __shared__ int pr[2 * P];
  const int f = blockIdx.x, tid = threadIdx.x;
  if (tid == 0) {
    int p = 0;
    for (int i = 0; i < M; ++i)
      for (int j = i; j < M; ++j) {
        pr[2 * p] = i;
        pr[2 * p + 1] = j;
        ++p;
      }
  }
  __syncthreads();
  const int p = tid % P, s = tid / P;
  const bool act = s < S;
  const int i = pr[2 * p], j = pr[2 * p + 1];
  R vr[M], vi[M];
#pragma unroll
  for (int m = 0; m < M; ++m) vr[m] = vi[m] = 0;
  const C* Xf = X + (size_t)f * T * M;
  const R* yf = y + (size_t)f * T * M;
  if (act) {
    for (int t = s; t < T; t += S) {
      const C xi = Xf[(size_t)t * M + i], xj = Xf[(size_t)t * M + j];
      const R a = xi.x * xj.x + xi.y * xj.y, bq = xi.y * xj.x - xi.x * xj.y;
#pragma unroll
      for (int m = 0; m < M; ++m) {
        const R w = R(1) / yf[(size_t)t * M + m];
        vr[m] += w * a;
        vi[m] += w * bq;
      }
    }
  }
  C* Vf = V + (size_t)f * M * M * M;
  for (int ss = 0; ss < S; ++ss) {
    if (act && s == ss) {
#pragma unroll
      for (int m = 0; m < M; ++m) {
        C* v = Vf + ((size_t)m * M + i) * M + j;
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
  for (int e = tid; e < M * P; e += 256) {
    const int m = e / P, pp = e % P;
    const int ii = pr[2 * pp], jj = pr[2 * pp + 1];
    C v = Vf[((size_t)m * M + ii) * M + jj];
    v.x *= invT;
    v.y *= invT;
    Vf[((size_t)m * M + ii) * M + jj] = v;
    if (ii != jj) Vf[((size_t)m * M + jj) * M + ii] = cmake<C>(v.x, -v.y);
  }
}

// _kernels.project_power (_kernels.py:339-350): thread per (f, t).
template <typename R, int M>
__global__ void k_project(const cplx<R>* __restrict__ Q, const cplx<R>* __restrict__ X, int F,
                          int T, R* __restrict__ xt) {
  using C = cplx<R>;
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)F * T) return;
  const long long f = i / T;
  const C* Qf = Q + f * M * M;
  C xv[M];
  CRowIO<R, M>::load(X + i * M, xv);
  R o[M];
#pragma unroll
  for (int r = 0; r < M; ++r) {
    R sr = 0, si = 0;
#pragma unroll
    for (int j = 0; j < M; ++j) {
      const C q = Qf[r * M + j];
      sr += q.x * xv[j].x - q.y * xv[j].y;
      si += q.x * xv[j].y + q.y * xv[j].x;
    }
    o[r] = sr * sr + si * si;
  }
  RowIO<R, M>::store(xt + i * M, o);
}

// IP rows from a precomputed V (spatial.py:183-199): one warp per bin.
template <typename R, int M>
__global__ void __launch_bounds__(32) k_ipsolve(cplx<R>* Q, const cplx<R>* __restrict__ V,
                                                int sweeps, unsigned long long* status) {
  using C = cplx<R>;
  __shared__ double2 Qd[M * M];
  __shared__ double2 A[M * (M + 1)];
  __shared__ double2 x[M];
  const int f = blockIdx.x, lane = threadIdx.x;
  C* Qf = Q + (size_t)f * M * M;
  for (int e = lane; e < M * M; e += 32) Qd[e] = to_d2(Qf[e]);
  __syncwarp();
  int bad_m = 0;
  const int code = warp_ip_update<M>(Qd, V + (size_t)f * M * M * M, A, x, sweeps, lane, &bad_m);
  if (code != 0) {
    if (lane == 0) report_status(status, 0, bad_m, f, code);
    return;
  }
  for (int e = lane; e < M * M; e += 32) Qf[e] = cmake<C>(Qd[e].x, Qd[e].y);
}

// slogdet(Q)[1] per bin.
template <typename R, int M>
__global__ void __launch_bounds__(32) k_logdet(const cplx<R>* __restrict__ Q, double* out) {
  __shared__ double2 A[M * (M + 1)];
  const int f = blockIdx.x, lane = threadIdx.x;
  for (int e = lane; e < M * M; e += 32) A[(e / M) * (M + 1) + e % M] = to_d2(Q[(size_t)f * M * M + e]);
  __syncwarp();
  double la = 0.0;
  warp_lu<M>(A, M + 1, M, lane, &la);
  if (lane == 0) out[f] = la;
}

// separate.wiener_fast (separate.py:110-125). grid F, block 256:
// warp 0 inverts Q_f (LU against I, as numpy.linalg.inv), then thread per t.
template <typename R, int M>
__global__ void __launch_bounds__(256) k_wiener(const R* __restrict__ lam, const cplx<R>* __restrict__ Q,
                                                const R* __restrict__ g, const cplx<R>* __restrict__ X,
                                                int N, int F, int T, cplx<R>* __restrict__ out,
                                                unsigned long long* status) {
  using C = cplx<R>;
  __shared__ double2 A[M * (2 * M)];
  __shared__ C Qi[M * M];
  __shared__ C Qs[M * M];
  __shared__ R gs[8 * M];
  __shared__ int bad;
  const int f = blockIdx.x, tid = threadIdx.x, lane = tid & 31;
  const C* Qf = Q + (size_t)f * M * M;
  for (int e = tid; e < M * M; e += 256) Qs[e] = Qf[e];
  for (int e = tid; e < N * M; e += 256) gs[e] = g[((size_t)(e / M) * F + f) * M + e % M];
  if (tid < 32) {
    constexpr int LD = 2 * M;
    for (int e = lane; e < M * M; e += 32) {
      const int r = e / M, c = e % M;
      A[r * LD + c] = to_d2(Qf[e]);
      A[r * LD + M + c] = make_double2(r == c ? 1.0 : 0.0, 0.0);
    }
    __syncwarp();
    const bool ok = warp_lu<M>(A, LD, 2 * M, lane, nullptr);
    if (ok) warp_backsubM<M>(A, LD, lane);
    if (lane == 0) {
      bad = ok ? 0 : 1;
      if (!ok) report_status(status, 0, 0, f, 3);
    }
    __syncwarp();
    for (int e = lane; e < M * M; e += 32) {
      const double2 v = A[(e / M) * LD + M + e % M];
      Qi[e] = cmake<C>(v.x, v.y);
    }
  }
  __syncthreads();
  if (bad) return;
  const size_t FT = (size_t)F * T;
  for (int t = tid; t < T; t += 256) {
    C xv[M];
    CRowIO<R, M>::load(X + ((size_t)f * T + t) * M, xv);
    C qx[M];
#pragma unroll
    for (int r = 0; r < M; ++r) {
      R sr = 0, si = 0;
#pragma unroll
      for (int j = 0; j < M; ++j) {
        const C q = Qs[r * M + j];
        sr += q.x * xv[j].x - q.y * xv[j].y;
        si += q.x * xv[j].y + q.y * xv[j].x;
      }
      qx[r] = cmake<C>(sr, si);
    }
    R den[M];
#pragma unroll
    for (int m = 0; m < M; ++m) den[m] = 0;
    for (int n = 0; n < N; ++n) {
      const R l = lam[n * FT + (size_t)f * T + t];
#pragma unroll
      for (int m = 0; m < M; ++m) den[m] += l * gs[n * M + m];
    }
    for (int n = 0; n < N; ++n) {
      const R l = lam[n * FT + (size_t)f * T + t];
      C z[M];
#pragma unroll
      for (int m = 0; m < M; ++m) {
        const R gain = den[m] > R(0) ? (l * gs[n * M + m]) / den[m] : R(1) / R(N);
        z[m] = cmake<C>(gain * qx[m].x, gain * qx[m].y);
      }
      C o[M];
#pragma unroll
      for (int r = 0; r < M; ++r) {
        R sr = 0, si = 0;
#pragma unroll
        for (int j = 0; j < M; ++j) {
          const C q = Qi[r * M + j];
          sr += q.x * z[j].x - q.y * z[j].y;
          si += q.x * z[j].y + q.y * z[j].x;
        }
        o[r] = cmake<C>(sr, si);
      }
      CRowIO<R, M>::store(out + ((size_t)n * FT + (size_t)f * T + t) * M, o);
    }
  }
}

// separate.wiener_fast in two launches (the single-CTA-per-bin k_wiener
// above hoists Q and Q^-1 into 254 registers: 12% occupancy, c1 176 us).
// k_qinv: one warp per bin inverts Q_f (LU against I, numpy.linalg.inv,
// separate.py:122) into Qi; a singular bin sets its flag and the status.
template <typename R, int M>
__global__ void __launch_bounds__(128) k_qinv(const cplx<R>* __restrict__ Q, int F, cplx<R>* __restrict__ Qi,
                                              int* __restrict__ bad, unsigned long long* status) {
  using C = cplx<R>;
  constexpr int LD = 2 * M;
  __shared__ double2 As[4][M * LD];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int f = blockIdx.x * 4 + warp;
  if (f >= F) return;
  double2* A = As[warp];
  const C* Qf = Q + (size_t)f * M * M;
  for (int e = lane; e < M * M; e += 32) {
    const int r = e / M, c = e % M;
    A[r * LD + c] = to_d2(Qf[e]);
    A[r * LD + M + c] = make_double2(r == c ? 1.0 : 0.0, 0.0);
  }
  __syncwarp();
  const bool ok = warp_lu<M>(A, LD, 2 * M, lane, nullptr);
  if (ok) warp_backsubM<M>(A, LD, lane);
  __syncwarp();
  if (lane == 0) {
    bad[f] = ok ? 0 : 1;
    if (!ok) report_status(status, 0, 0, f, 3);
  }
  for (int e = lane; e < M * M; e += 32) {
    const double2 v = A[(e / M) * LD + M + e % M];
    Qi[(size_t)f * M * M + e] = cmake<C>(v.x, v.y);
  }
}

// k_wiener_t: one frame per thread, grid (ceil(T/128), F), block 128; Q, Q^-1
// and the gains of the bin in shared memory; image_n = Q^-1 (gain_n . Q x),
// gain_n = lam_n g_n / sum_n' lam_n' g_n' (1/N where the sum is 0).
template <typename R, int M>
__global__ void __launch_bounds__(128, 4) k_wiener_t(const R* __restrict__ lam, const cplx<R>* __restrict__ Q,
                                                     const cplx<R>* __restrict__ Qi, const int* __restrict__ bad,
                                                     const R* __restrict__ g, const cplx<R>* __restrict__ X,
                                                     int N, int F, int T, cplx<R>* __restrict__ out) {
  using C = cplx<R>;
  __shared__ __align__(16) C Qs[M * M];
  __shared__ __align__(16) C Qis[M * M];
  __shared__ R gs[8 * M];
  const int f = blockIdx.y, tid = threadIdx.x;
  if (bad[f]) return;
  for (int e = tid; e < M * M; e += 128) {
    Qs[e] = Q[(size_t)f * M * M + e];
    Qis[e] = Qi[(size_t)f * M * M + e];
  }
  for (int e = tid; e < N * M; e += 128) gs[e] = g[((size_t)(e / M) * F + f) * M + e % M];
  __syncthreads();
  const int t = blockIdx.x * 128 + tid;
  if (t >= T) return;
  const size_t FT = (size_t)F * T;
  C xv[M];
  CRowIO<R, M>::load(X + ((size_t)f * T + t) * M, xv);
  C qx[M];
#pragma unroll
  for (int r = 0; r < M; ++r) {
    R sr = 0, si = 0;
#pragma unroll
    for (int j = 0; j < M; ++j) {
      const C q = Qs[r * M + j];
      sr += q.x * xv[j].x - q.y * xv[j].y;
      si += q.x * xv[j].y + q.y * xv[j].x;
    }
    qx[r] = cmake<C>(sr, si);
  }
  R den[M];
#pragma unroll
  for (int m = 0; m < M; ++m) den[m] = 0;
  for (int n = 0; n < N; ++n) {
    const R l = lam[n * FT + (size_t)f * T + t];
#pragma unroll
    for (int m = 0; m < M; ++m) den[m] += l * gs[n * M + m];
  }
  for (int n = 0; n < N; ++n) {
    const R l = lam[n * FT + (size_t)f * T + t];
    C z[M];
#pragma unroll
    for (int m = 0; m < M; ++m) {
      const R gain = den[m] > R(0) ? (l * gs[n * M + m]) / den[m] : R(1) / R(N);
      z[m] = cmake<C>(gain * qx[m].x, gain * qx[m].y);
    }
    C o[M];
#pragma unroll
    for (int r = 0; r < M; ++r) {
      R sr = 0, si = 0;
#pragma unroll
      for (int j = 0; j < M; ++j) {
        const C q = Qis[r * M + j];
        sr += q.x * z[j].x - q.y * z[j].y;
        si += q.x * z[j].y + q.y * z[j].x;
      }
      o[r] = cmake<C>(sr, si);
    }
    CRowIO<R, M>::store(out + ((size_t)n * FT + (size_t)f * T + t) * M, o);
  }
}

// sum |X|^2 and max |X|^2 per mixture: partials (B, nblk) of fp64.
template <typename R>
__global__ void __launch_bounds__(256) k_obs_stats(const cplx<R>* __restrict__ X, long long n_per_b,
                                                   double* psum, double* pmax) {
  __shared__ double rs[8], rm[8];
  const int b = blockIdx.y, tid = threadIdx.x;
  const cplx<R>* Xb = X + (size_t)b * n_per_b;
  double s = 0.0, mx = 0.0;
  for (long long i = (long long)blockIdx.x * 256 + tid; i < n_per_b; i += (long long)gridDim.x * 256) {
    const double re = Xb[i].x, im = Xb[i].y;
    const double a = re * re + im * im;
    s += a;
    mx = a > mx ? a : mx;
  }
  s = warp_sum(s);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((tid & 31) == 0) {
    rs[tid >> 5] = s;
    rm[tid >> 5] = mx;
  }
  __syncthreads();
  if (tid == 0) {
    double a = 0.0, m = 0.0;
    for (int w = 0; w < 8; ++w) {
      a += rs[w];
      m = fmax(m, rm[w]);
    }
    psum[(size_t)b * gridDim.x + blockIdx.x] = a;
    pmax[(size_t)b * gridDim.x + blockIdx.x] = m;
  }
}

// X /= scale[b]  (separate.py:293, computed in fp64 and rounded once).
template <typename R>
__global__ void k_scale(cplx<R>* X, long long n_per_b, const double* scale, int B) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_per_b * B) return;
  const double s = scale[i / n_per_b];
  cplx<R> v = X[i];
  v.x = (R)((double)v.x / s);
  v.y = (R)((double)v.y / s);
  X[i] = v;
}

}  // namespace fm
