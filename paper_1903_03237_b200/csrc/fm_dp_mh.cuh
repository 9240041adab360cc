// fm_dp_mh.cuh -- the reference's FastMNMF-DP latent update: the Metropolis
// random walk of update_latents_fast (sources.py:307-339, driver _run_chain
// :307-322, ratio metropolis_log_gamma_fast :292-304), hooked at
// separate.py:205-213, with either decoder (the reference's ToyDecoder,
// sources.py:52-80, or the config-4 exp-MLP). SURVEY §8(f) item 2.
//
// Every frame's chain is independent (frame t's latent reaches only r[t, :],
// and the ratio of frame t only involves frame t), so one CTA owns FPB frames
// and runs all `steps` proposals on chip:
//   z' = z + std * n_s            (n_s: caller-filled numpy draws or Philox)
//   r' = dec(z')                  hidden layer(s) in shared memory, output
//                                 rows streamed from L2, each row reused by
//                                 the CTA's FPB frames
//   log gamma_t = - sum_fm x~ (1/y' - 1/y) - sum_fm log(y'/y),
//                 y = max(lambda g_0 + y_rest, TINY), y_rest = sum_{n>=1}
//                 lambda_n g_n (mix_power without floor, separate.py:207)
//   accept iff log(u_s) <= log gamma_t: z, r (and lambda_old) take z', r'.
// The two sums are block-reduced in a fixed order (deterministic). x~ and
// y_rest of the CTA's frames are staged once in shared memory when they fit.
// steps = 0 is the decoder refresh r = dec(z) alone (prologue).
#pragma once
#include "fm_common.cuh"
#include "fm_nmf.cuh"

namespace fm {

template <typename R> struct MhArgs {
  const R *W1, *b1;  // (Hd, D), (Hd)
  const R *W2, *b2;  // (Hd, Hd), (Hd): exp-MLP second hidden layer
  const R *WoT, *bo; // (Hd, F) transposed output layer (W3^T, written by the prologue), (F)
  const R *u, *v;    // (B, F), (B, T)
  R *z, *r;          // (B, T, D), (B, T, F)
  const R* lam;      // (B, N, F, T)
  const R* g;        // (B, N, F, M)
  const R* xt;       // (B, F, T, M)
  const R* noise;    // (steps, B, T, D) or null (Philox)
  const R* unif;     // (steps, B, T) or null
  const unsigned* iter;
  unsigned long long seed;
  double stdv;
  int steps, kind, D, Hd, N, F, T, M, B, fpb, cache;
};

// Philox-4x32-10 (Salmon et al., SC'11): counter c, key k -> 4 x 32 random bits
__device__ __forceinline__ uint4 philox4x32(uint4 c, uint2 k) {
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    const unsigned long long p0 = (unsigned long long)0xD2511F53u * c.x;
    const unsigned long long p1 = (unsigned long long)0xCD9E8D57u * c.z;
    const unsigned h0 = (unsigned)(p0 >> 32), l0 = (unsigned)p0;
    const unsigned h1 = (unsigned)(p1 >> 32), l1 = (unsigned)p1;
    c = make_uint4(h1 ^ c.y ^ k.x, l1, h0 ^ c.w ^ k.y, l0);
    k.x += 0x9E3779B9u;
    k.y += 0xBB67AE85u;
  }
  return c;
}
// uniform in (0, 1] from 32 bits (never 0: log-safe)
__device__ __forceinline__ double u01(unsigned x) { return ((double)x + 1.0) * 2.3283064365386963e-10; }

template <typename R> __device__ __forceinline__ R softplus_r(R x) {
  // log1p(exp(-|x|)) + max(x, 0)  (sources.py:31-35)
  return log1p(exp(-fabs(x))) + (x > R(0) ? x : R(0));
}

template <typename R>
__global__ void __launch_bounds__(256) k_dp_mh(MhArgs<R> a) {
  pdl_entry();
  extern __shared__ __align__(16) unsigned char mh_smem[];
  const int FPB = a.fpb, D = a.D, Hd = a.Hd, F = a.F, T = a.T, M = a.M, N = a.N;
  const int b = blockIdx.y, t0 = blockIdx.x * FPB, tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int nfr = min(FPB, T - t0);
  R* zc = reinterpret_cast<R*>(mh_smem);          // [FPB][D] current z
  R* zn = zc + FPB * D;                           // [FPB][D] proposal
  R* h1 = zn + FPB * D;                           // [FPB][Hd]
  R* h2 = h1 + FPB * Hd;                          // [FPB][Hd]
  R* rc = h2 + FPB * Hd;                          // [FPB][F] current r
  R* rn = rc + FPB * F;                           // [FPB][F] proposal r
  R* red = rn + FPB * F;                          // [8 warps][FPB][2]
  R* lg = red + 8 * FPB * 2;                      // [FPB] log gamma
  R* xs = lg + FPB;                               // [FPB][F][M] x~ (cache)
  R* ys = xs + (size_t)FPB * F * M;               // [FPB][F][M] y_rest (cache)
  const size_t FT = (size_t)F * T;
  const R* ub = a.u + (size_t)b * F;
  const R* g0 = a.g + (size_t)b * N * F * M;      // source 0 gains (F, M)
  const unsigned it = a.iter ? *a.iter : 0u;
  const uint2 key = make_uint2((unsigned)a.seed, (unsigned)(a.seed >> 32));
  for (int e = tid; e < nfr * D; e += 256) zc[e] = a.z[((size_t)b * T + t0) * D + e];
  auto yrest = [&](int fr, int f, int m) -> R {  // mix_power(lam[1:], g[1:]) (floor 0)
    R acc = 0;
    for (int n = 1; n < N; ++n)
      acc += a.lam[((size_t)b * N + n) * FT + (size_t)f * T + t0 + fr] *
             a.g[(((size_t)b * N + n) * F + f) * M + m];
    return acc;
  };
  if (a.steps > 0) {
    for (int e = tid; e < nfr * F; e += 256) rc[e] = a.r[((size_t)b * T + t0) * F + e];
    if (a.cache) {
      for (int e = tid; e < nfr * F * M; e += 256) {
        const int fr = e / (F * M), f = (e / M) % F, m = e % M;
        xs[e] = a.xt[(((size_t)b * F + f) * T + t0 + fr) * M + m];
        ys[e] = yrest(fr, f, m);
      }
    }
  }
  __syncthreads();

  // r_out[fr][f] = dec(zin[fr]) for the CTA's frames
  auto decode = [&](const R* zin, R* rout) {
    for (int e = tid; e < nfr * Hd; e += 256) {
      const int fr = e / Hd, j = e % Hd;
      R acc = a.b1[j];
      for (int d = 0; d < D; ++d) acc += a.W1[(size_t)j * D + d] * zin[fr * D + d];
      h1[fr * Hd + j] = tanh(acc);
    }
    __syncthreads();
    const R* hl = h1;
    if (a.kind == 0) {  // exp-MLP: second hidden layer
      for (int e = tid; e < nfr * Hd; e += 256) {
        const int fr = e / Hd, j = e % Hd;
        R acc = a.b2[j];
        for (int k = 0; k < Hd; ++k) acc += a.W2[(size_t)j * Hd + k] * h1[fr * Hd + k];
        h2[fr * Hd + j] = tanh(acc);
      }
      __syncthreads();
      hl = h2;
    }
    for (int f = tid; f < F; f += 256) {
      R acc[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[q] = a.bo[f];
      for (int j = 0; j < Hd; ++j) {
        const R w = a.WoT[(size_t)j * F + f];  // coalesced across the f threads
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (q < nfr) acc[q] += w * hl[q * Hd + j];
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (q >= nfr) break;
        R o;
        if (a.kind == 0) {
          o = exp(acc[q]);
        } else {  // ToyDecoder: max(softplus(.), OUTPUT_FLOOR) (sources.py:61, :70-73)
          o = softplus_r(acc[q]);
          o = o > R(1e-8) ? o : R(1e-8);
        }
        rout[q * F + f] = o;
      }
    }
    __syncthreads();
  };

  if (a.steps == 0) {  // refresh r = dec(z)
    decode(zc, rn);
    for (int e = tid; e < nfr * F; e += 256) a.r[((size_t)b * T + t0) * F + e] = rn[e];
    return;
  }
  const R tiny = RT<R>::tiny();
  for (int s = 0; s < a.steps; ++s) {
    // proposal z' = z + std * n  (sources.py:315)
    for (int e = tid; e < nfr * D; e += 256) {
      const int fr = e / D, d = e % D;
      const int t = t0 + fr;
      R nv;
      if (a.noise) {
        nv = a.noise[(((size_t)s * a.B + b) * T + t) * D + d];
      } else {  // Box-Muller on a Philox pair
        const uint4 q = philox4x32(make_uint4((unsigned)(d >> 1), (unsigned)t, (unsigned)b,
                                              it * (unsigned)a.steps + (unsigned)s), key);
        const double rr = sqrt(-2.0 * log(u01(q.x))), th = 6.283185307179586 * u01(q.y);
        nv = (R)((d & 1) ? rr * sin(th) : rr * cos(th));
      }
      zn[e] = zc[e] + (R)a.stdv * nv;
    }
    __syncthreads();
    decode(zn, rn);
    // log gamma per frame: two fixed-order block sums (sources.py:298-304)
    R s1[4] = {0, 0, 0, 0}, s2[4] = {0, 0, 0, 0};
    for (int f = tid; f < F; f += 256) {
      const R uf = ub[f];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (q >= nfr) break;
        const R vt = a.v[(size_t)b * T + t0 + q];
        const R ln = uf * (vt * rn[q * F + f]), lo = uf * (vt * rc[q * F + f]);
        for (int m = 0; m < M; ++m) {
          const R gm = g0[(size_t)f * M + m];
          const R yr = a.cache ? ys[((size_t)q * F + f) * M + m] : yrest(q, f, m);
          const R x = a.cache ? xs[((size_t)q * F + f) * M + m]
                              : a.xt[(((size_t)b * F + f) * T + t0 + q) * M + m];
          R yn = ln * gm + yr, yo = lo * gm + yr;
          yn = yn > tiny ? yn : tiny;
          yo = yo > tiny ? yo : tiny;
          if constexpr (sizeof(R) == 8) {  // the reference's expression order
            s1[q] += x * (R(1) / yn - R(1) / yo);
            s2[q] += log(yn / yo);
          } else {  // complex64 mode: MUFU reciprocals / log (<= 2 ulp)
            const R iyn = rcp_r(yn), iyo = rcp_r(yo);
            s1[q] += x * (iyn - iyo);
            s2[q] += log_fast(yn * iyo);
          }
        }
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      s1[q] = warp_sum(s1[q]);
      s2[q] = warp_sum(s2[q]);
      if (lane == 0 && q < nfr) {
        red[(warp * FPB + q) * 2] = s1[q];
        red[(warp * FPB + q) * 2 + 1] = s2[q];
      }
    }
    __syncthreads();
    if (tid < nfr) {
      R t1 = 0, t2 = 0;
      for (int w = 0; w < 8; ++w) {
        t1 += red[(w * FPB + tid) * 2];
        t2 += red[(w * FPB + tid) * 2 + 1];
      }
      const R lgam = -t1 - t2;
      const int t = t0 + tid;
      double uu;
      if (a.unif) {
        uu = (double)a.unif[((size_t)s * a.B + b) * T + t];
      } else {
        uu = u01(philox4x32(make_uint4(0xFFFFFFFFu, (unsigned)t, (unsigned)b,
                                       it * (unsigned)a.steps + (unsigned)s), key).x);
      }
      // np.log(rng.uniform(size=T)) <= log_gamma  (sources.py:318)
      lg[tid] = (log((R)uu) <= lgam) ? R(1) : R(0);
    }
    __syncthreads();
    for (int e = tid; e < nfr * D; e += 256)
      if (lg[e / D] != R(0)) zc[e] = zn[e];
    for (int e = tid; e < nfr * F; e += 256)
      if (lg[e / F] != R(0)) rc[e] = rn[e];
    __syncthreads();
  }
  for (int e = tid; e < nfr * D; e += 256) a.z[((size_t)b * T + t0) * D + e] = zc[e];
  for (int e = tid; e < nfr * F; e += 256) a.r[((size_t)b * T + t0) * F + e] = rc[e];
}

// W3 (F, Hd) -> W3^T (Hd, F); grid (ceil(F/32), ceil(Hd/32)), block (32, 8)
template <typename R>
__global__ void k_transpose_fh(const R* __restrict__ W, R* __restrict__ Wt, int F, int Hd) {
  __shared__ R tile[32][33];
  const int f0 = blockIdx.x * 32, j0 = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int f = f0 + i, j = j0 + threadIdx.x;
    tile[i][threadIdx.x] = (f < F && j < Hd) ? W[(size_t)f * Hd + j] : R(0);
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int j = j0 + i, f = f0 + threadIdx.x;
    if (f < F && j < Hd) Wt[(size_t)j * F + f] = tile[threadIdx.x][i];
  }
}

// shared-memory bytes of k_dp_mh for FPB frames (cache: x~ and y_rest staged)
inline size_t mh_smem_bytes(size_t rs, int fpb, int D, int Hd, int F, int M, bool cache) {
  size_t n = (size_t)fpb * (2 * D + 2 * Hd + 2 * F + 1) + 8 * fpb * 2;
  if (cache) n += (size_t)2 * fpb * F * M;
  return n * rs;
}

}  // namespace fm
