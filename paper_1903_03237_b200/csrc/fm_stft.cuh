// fm_stft.cuh -- multichannel STFT / iSTFT on the device:
// the reference's front/back end (stft.py:27-91): periodic Hann window,
// reflect padding by L/2, frames every `hop` samples (zero tail to a whole
// frame), rfft -> (F, T, M); inverse: irfft per frame, window, overlap-add
// divided by the summed squared window (max with TINY), de-padded, trimmed.
//
// FFT: iterative radix-2 decimation in time in shared memory, one CTA per
// (frame, channel group); the group's channels share the twiddle table
// exp(-2 pi i k / L), k < L/2 (computed with sincospi in the working
// precision). Real input runs as a complex transform with zero imaginary
// part; bins 0..L/2 are written with the channel index innermost, so the
// (F, T, M) output rows of a group are contiguous. The inverse builds the
// Hermitian spectrum (imaginary parts of bins 0 and L/2 dropped, as numpy's
// c2r does), transforms with conjugate twiddles and scales by 1/L.
// Overlap-add is a gather (each output sample sums its <= ceil(L/hop)
// frames in increasing frame order, like the reference loop): deterministic,
// no atomics.
#pragma once
#include "fm_common.cuh"

namespace fm {

constexpr int STFT_THREADS = 512;

__host__ __device__ inline long long stft_frames(long long n, long long L, long long hop) {
  const long long padded = n + 2 * (L / 2);
  return 1 + (padded - L + hop - 1) / hop;  // 1 + ceil((padded - L) / hop)
}

template <typename R> __device__ __forceinline__ void sincospi_r(R x, R* s, R* c);
template <> __device__ __forceinline__ void sincospi_r<float>(float x, float* s, float* c) {
  sincospif(x, s, c);
}
template <> __device__ __forceinline__ void sincospi_r<double>(double x, double* s, double* c) {
  sincospi(x, s, c);
}

// in-place radix-2 DIT on G length-L rows (bit-reversed input order), sign -1
// forward / +1 inverse; tw[k] = exp(-2 pi i k / L)
template <typename R>
__device__ void fft_rows(cplx<R>* s, const cplx<R>* tw, int L, int logL, int G, bool inverse) {
  using C = cplx<R>;
  for (int lg = 1; lg <= logL; ++lg) {
    const int len = 1 << lg, half = len >> 1, stride = L >> lg;
    for (int e = threadIdx.x; e < G * (L >> 1); e += blockDim.x) {
      const int g = e / (L >> 1), j = e % (L >> 1);
      const int k = j & (half - 1), i0 = ((j >> (lg - 1)) << lg) + k, i1 = i0 + half;
      C w = tw[k * stride];
      if (inverse) w.y = -w.y;
      C* row = s + (size_t)g * L;
      const C a = row[i0], bv = row[i1];
      C b;
      b.x = bv.x * w.x - bv.y * w.y;
      b.y = bv.x * w.y + bv.y * w.x;
      row[i0] = cmake<C>(a.x + b.x, a.y + b.y);
      row[i1] = cmake<C>(a.x - b.x, a.y - b.y);
    }
    __syncthreads();
  }
}

template <typename R> __device__ __forceinline__ R hann_r(int i, int L) {
  // 0.5 - 0.5 cos(2 pi i / L)  (stft.py:15-17)
  R s, c;
  sincospi_r<R>(R(2) * (R)i / (R)L, &s, &c);
  return R(0.5) - R(0.5) * c;
}

template <typename R>
__device__ void fill_twiddles(cplx<R>* tw, int L) {
  for (int k = threadIdx.x; k < L / 2; k += blockDim.x) {
    R s, c;
    sincospi_r<R>(-R(2) * (R)k / (R)L, &s, &c);
    tw[k] = cmake<cplx<R>>(c, s);
  }
}

// grid (T, ceil(M / G)); smem (G * L + L/2) complex
template <typename R>
__global__ void __launch_bounds__(STFT_THREADS) k_stft(const R* __restrict__ wave, cplx<R>* __restrict__ spec,
                                                       long long n, int M, int L, int logL, int hop,
                                                       int T, int G) {
  using C = cplx<R>;
  extern __shared__ __align__(16) unsigned char st_smem[];
  C* tw = reinterpret_cast<C*>(st_smem);
  C* s = tw + L / 2;
  const int t = blockIdx.x, m0 = blockIdx.y * G, g_n = min(G, M - m0);
  const int pad = L / 2;
  fill_twiddles<R>(tw, L);
  for (int e = threadIdx.x; e < g_n * L; e += blockDim.x) {
    const int i = e / g_n, g = e % g_n;  // channel innermost: coalesced waveform rows
    const long long p = (long long)t * hop + i;  // position in the padded signal
    long long q = p - pad;
    R x = R(0);
    if (p < n + 2 * pad) {  // reflect padding (numpy mode="reflect", edge not repeated)
      if (q < 0) q = -q;
      if (q >= n) q = 2 * (n - 1) - q;
      x = wave[q * M + m0 + g];
    }  // else: the zero tail up to a whole frame
    const unsigned r = __brev((unsigned)i) >> (32 - logL);
    s[(size_t)g * L + r] = cmake<C>(x * hann_r<R>(i, L), R(0));
  }
  __syncthreads();
  fft_rows<R>(s, tw, L, logL, g_n, false);
  const int F = L / 2 + 1;
  for (int e = threadIdx.x; e < F * g_n; e += blockDim.x) {
    const int f = e / g_n, g = e % g_n;
    spec[((size_t)f * T + t) * M + m0 + g] = s[(size_t)g * L + f];
  }
}

// inverse transform + window: frames (T, L, M) real; grid (T, ceil(M / G))
template <typename R>
__global__ void __launch_bounds__(STFT_THREADS) k_istft_frames(const cplx<R>* __restrict__ spec,
                                                               R* __restrict__ frames, int M, int L,
                                                               int logL, int T, int G) {
  using C = cplx<R>;
  extern __shared__ __align__(16) unsigned char st_smem[];
  C* tw = reinterpret_cast<C*>(st_smem);
  C* s = tw + L / 2;
  const int t = blockIdx.x, m0 = blockIdx.y * G, g_n = min(G, M - m0);
  const int h = L / 2;
  fill_twiddles<R>(tw, L);
  for (int e = threadIdx.x; e < g_n * L; e += blockDim.x) {
    const int k = e / g_n, g = e % g_n;
    C v;
    if (k <= h) {
      v = spec[((size_t)k * T + t) * M + m0 + g];
      if (k == 0 || k == h) v.y = R(0);  // c2r ignores these imaginary parts
    } else {
      const C c = spec[((size_t)(L - k) * T + t) * M + m0 + g];
      v = cmake<C>(c.x, -c.y);
    }
    const unsigned r = __brev((unsigned)k) >> (32 - logL);
    s[(size_t)g * L + r] = v;
  }
  __syncthreads();
  fft_rows<R>(s, tw, L, logL, g_n, true);
  const R inv = R(1) / (R)L;
  for (int e = threadIdx.x; e < g_n * L; e += blockDim.x) {
    const int i = e / g_n, g = e % g_n;
    frames[((size_t)t * L + i) * M + m0 + g] = s[(size_t)g * L + i].x * inv * hann_r<R>(i, L);
  }
}

// overlap-add gather: out (len, M) = sum_t frames[t][j - t hop] / max(sum_t w^2, TINY),
// j = sample + L/2 (de-padded); grid-stride over len * M
template <typename R>
__global__ void k_ola(const R* __restrict__ frames, R* __restrict__ out, long long len, int M, int L,
                      int hop, int T) {
  const long long total = len * M;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / M;
    const int m = (int)(e % M);
    const long long j = i + L / 2;
    long long t1 = j / hop;  // last frame starting at or before j
    if (t1 > T - 1) t1 = T - 1;
    long long t0 = (j - L) / hop + 1;  // first frame with t hop + L > j
    if (j - L < 0) t0 = 0;
    R acc = 0, nrm = 0;
    for (long long t = t0; t <= t1; ++t) {
      const int o = (int)(j - t * hop);
      const R w = hann_r<R>(o, L);
      acc += frames[((size_t)t * L + o) * M + m];
      nrm += w * w;
    }
    out[e] = acc / (nrm > RT<R>::tiny() ? nrm : RT<R>::tiny());
  }
}

}  // namespace fm
