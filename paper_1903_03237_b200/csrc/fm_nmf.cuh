// fm_nmf.cuh -- the NMF source-model part of the FastMNMF iteration as
// register-blocked SIMT contractions (sources.py:167-204).
//
//   k_wstats  num/den_W = phi{1,2} H^T  (sum over T; sources.py:192-193),
//             split over T across CTAs; the last CTA of each F-tile reduces
//             the partials in fixed order and applies the W MU
//             (sources.py:194).
//   k_phi     statistics pass (separate.py:186-193; _kernels.py:226-243):
//             phi1 = sum_m g x~/y^2, phi2 = sum_m g/y from lambda, x~, g.
//   k_hstats  num/den_H = W^T phi{1,2}  (sum over F; sources.py:196-197),
//             split over F across CTAs; the last CTA of each T-tile reduces
//             in fixed order and applies the H MU (sources.py:198) -- or,
//             frequency-sharded, writes the sums for the NCCL all-reduce.
//
// Both contractions stage their operands in shared memory with the
// reduction index contiguous, and every thread owns a 4 x 4 (x2: numerator
// and denominator) output block: 3 LDS.128 per 32 FMA.
#pragma once
#include "fm_common.cuh"

namespace fm {

__device__ __forceinline__ void lds4(const float* p, float (&v)[4]) {
  const float4 q = *reinterpret_cast<const float4*>(p);
  v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
}
__device__ __forceinline__ void lds4(const double* p, double (&v)[4]) {
  const double2 a = *reinterpret_cast<const double2*>(p);
  const double2 b = *reinterpret_cast<const double2*>(p + 2);
  v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
}

// cp.async (LDGSTS) 16-byte copies with zero-fill, for double-buffered staging
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  const int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int NPEND> __device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(NPEND));
}

// ---------------------------------------------------------------------------
// W statistics + W MU (sources.py:191-194). One CTA owns FT bins of one
// (b, n) and reduces over all of T itself (no split, no partials): operands
// stream through a cp.async double buffer in TCH-frame chunks; thread tile
// 4 f x 4 k (x2: num, den); slices of the CTA take interleaved frame quads
// and are summed in one fixed-order pass at the end.
// grid (ceil(F/FT), B*N), block 256.
// ---------------------------------------------------------------------------
template <typename R, int KB, int FT> struct WsCfg {
  static constexpr int TCH = sizeof(R) == 4 ? 128 : 64;  // frames per staged chunk
  static constexpr int LD = TCH + 4;                     // padded row
  static constexpr int NTH = (FT / 4) * (KB / 4);        // threads per slice
  static constexpr int S = 256 / NTH;                    // slices per CTA
  static constexpr int STAGE = (2 * FT + KB) * LD;       // staged operands (elements)
  static constexpr int RED = S * 2 * FT * KB;            // one-pass slice reduction
  static constexpr size_t bytes = sizeof(R) * (2 * STAGE > RED ? 2 * STAGE : RED);
};

template <typename R, int KB, int FT>
__global__ void __launch_bounds__(256) k_wstats(const R* __restrict__ phi, const R* __restrict__ H,
                                                R* __restrict__ W, int N, int F, int T, int K,
                                                int n0) {
  pdl_entry();
  using Cf = WsCfg<R, KB, FT>;
  constexpr int TCH = Cf::TCH, LD = Cf::LD, NTH = Cf::NTH, S = Cf::S;
  constexpr int FG = FT / 4, KG = KB / 4;
  extern __shared__ __align__(16) unsigned char smraw[];
  R* stage0 = reinterpret_cast<R*>(smraw);
  const int bn = blockIdx.y, f0 = blockIdx.x * FT;
  const int tid = threadIdx.x;
  const int slot = tid % NTH, s = tid / NTH;
  const int fg = slot % FG, kg = slot / FG;
  const size_t FTs = (size_t)F * T;
  const int b = bn / (N - n0), n = n0 + bn % (N - n0);  // W/H hold the NMF sources n0..N-1
  const R* P1 = phi + ((size_t)b * 2 * N + n) * FTs;
  const R* P2 = P1 + (size_t)N * FTs;
  const R* Hn = H + (size_t)bn * K * T;
  const bool async = sizeof(R) == 4 && (T % 4) == 0;
  auto stage = [&](int st) { return stage0 + st * Cf::STAGE; };
  auto load = [&](int st, int t0) {
    R* p1s = stage(st);
    R* p2s = p1s + FT * LD;
    R* hs = p2s + FT * LD;
    if (async) {
      constexpr int Q = TCH / 4;
      for (int e = tid; e < FT * Q; e += 256) {
        const int fl = e / Q, q = e % Q, f = f0 + fl, t = t0 + 4 * q;
        const bool v = f < F && t < T;
        const size_t off = v ? (size_t)f * T + t : 0;
        cp_async16(p1s + fl * LD + 4 * q, P1 + off, v);
        cp_async16(p2s + fl * LD + 4 * q, P2 + off, v);
      }
      for (int e = tid; e < KB * Q; e += 256) {
        const int kl = e / Q, q = e % Q, t = t0 + 4 * q;
        const bool v = kl < K && t < T;
        cp_async16(hs + kl * LD + 4 * q, Hn + (v ? (size_t)kl * T + t : 0), v);
      }
    } else {
      for (int e = tid; e < FT * TCH; e += 256) {
        const int fl = e / TCH, tl = e % TCH, f = f0 + fl, t = t0 + tl;
        const bool v = f < F && t < T;
        p1s[fl * LD + tl] = v ? P1[(size_t)f * T + t] : R(0);
        p2s[fl * LD + tl] = v ? P2[(size_t)f * T + t] : R(0);
      }
      for (int e = tid; e < KB * TCH; e += 256) {
        const int kl = e / TCH, tl = e % TCH, t = t0 + tl;
        hs[kl * LD + tl] = (kl < K && t < T) ? Hn[(size_t)kl * T + t] : R(0);
      }
    }
    cp_async_commit();
  };
  R a1[4][4], a2[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) a1[i][j] = a2[i][j] = 0;
  int st = 0;
  load(0, 0);
  for (int t0 = 0; t0 < T; t0 += TCH, st ^= 1) {
    if (t0 + TCH < T) {
      load(st ^ 1, t0 + TCH);  // next chunk in flight during this one
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const R* p1s = stage(st);
    const R* p2s = p1s + FT * LD;
    const R* hs = p2s + FT * LD;
    for (int tq = s * 4; tq < TCH; tq += 4 * S) {
      R x1[4][4], x2[4][4], h[4][4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        lds4(p1s + (fg + FG * i) * LD + tq, x1[i]);
        lds4(p2s + (fg + FG * i) * LD + tq, x2[i]);
        lds4(hs + (kg + KG * i) * LD + tq, h[i]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            a1[i][j] += x1[i][u] * h[j][u];
            a2[i][j] += x2[i][u] * h[j][u];
          }
    }
    __syncthreads();
  }
  // one-pass fixed-order reduction over the S slices
  R* red = stage0;  // [S][2][FT][KB]
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int idx = (fg + FG * i) * KB + kg + KG * j;
      red[(s * 2) * FT * KB + idx] = a1[i][j];
      red[(s * 2 + 1) * FT * KB + idx] = a2[i][j];
    }
  __syncthreads();
  R* Wn = W + (size_t)bn * F * K;
  for (int e = tid; e < FT * KB; e += 256) {
    const int fl = e / KB, k = e % KB, f = f0 + fl;
    if (f < F && k < K) {
      R sn = 0, sd = 0;
      for (int q = 0; q < S; ++q) {
        sn += red[(q * 2) * FT * KB + e];
        sd += red[(q * 2 + 1) * FT * KB + e];
      }
      Wn[(size_t)f * K + k] *= mu_factor(sn, sd);  // sources.py:194
    }
  }
}

// ---------------------------------------------------------------------------
// H statistics + H MU (sources.py:195-198). One CTA owns TT frames of one
// (b, n) and reduces over all local F itself; W rows and phi rows stream
// through a cp.async double buffer in FCH-bin chunks; thread tile 4 k x 4 t
// (x2). mode 0 applies the MU; mode 1 writes the (num, den) sums to hout
// (B, 2, N, K, T) for the cross-shard all-reduce. When T-tiles alone leave
// SMs idle the bins split FS ways (grid z): each CTA publishes its partial
// sums and the last one of the tile adds them in split order.
// grid (ceil(T/TT), B*N, FS), block 256.
// ---------------------------------------------------------------------------
template <typename R, int KB, int TT> struct HsCfg {
  static constexpr int FCH = sizeof(R) == 4 ? 32 : 16;   // bins per staged chunk
  static constexpr int NTH = (KB / 4) * (TT / 4);        // threads per slice
  static constexpr int S = 256 / NTH;                    // slices (over bins)
  static constexpr int LDW = KB + 4, LDP = TT + 4;
  static constexpr int STAGE = FCH * LDW + 2 * FCH * LDP;
  static constexpr int RED = S * 2 * KB * TT;
  static constexpr size_t bytes = sizeof(R) * (2 * STAGE > RED ? 2 * STAGE : RED);
};

template <typename R, int KB, int TT>
__global__ void __launch_bounds__(256) k_hstats(const R* __restrict__ phi, const R* __restrict__ W,
                                                R* __restrict__ H, R* __restrict__ hout, int N,
                                                int F, int T, int K, int mode, int n0, int frange,
                                                R* __restrict__ part, unsigned* __restrict__ cnt) {
  pdl_entry();
  using Cf = HsCfg<R, KB, TT>;
  constexpr int FCH = Cf::FCH, NTH = Cf::NTH, S = Cf::S, LDW = Cf::LDW, LDP = Cf::LDP;
  constexpr int TG = TT / 4;
  extern __shared__ __align__(16) unsigned char smraw[];
  R* stage0 = reinterpret_cast<R*>(smraw);
  const int bn = blockIdx.y, t0 = blockIdx.x * TT;
  const int tid = threadIdx.x;
  const int slot = tid % NTH, s = tid / NTH;
  const int tg = slot % TG, kg = slot / TG;
  const size_t FTs = (size_t)F * T;
  const int Nn = N - n0;
  const int b = bn / Nn, nl = bn % Nn, n = n0 + nl;
  const R* P1 = phi + ((size_t)b * 2 * N + n) * FTs;
  const R* P2 = P1 + (size_t)N * FTs;
  const R* Wn = W + (size_t)bn * F * K;
  const bool async = sizeof(R) == 4 && (T % 4) == 0;
  const bool asyncw = sizeof(R) == 4 && (K % 4) == 0 && (LDW % 4) == 0 && (KB % 4) == 0 &&
                      (reinterpret_cast<uintptr_t>(W) & 15) == 0;
  auto stage = [&](int st) { return stage0 + st * Cf::STAGE; };
  auto load = [&](int st, int c0) {
    R* ws = stage(st);
    R* p1s = ws + FCH * LDW;
    R* p2s = p1s + FCH * LDP;
    if (asyncw) {
      // W rows by 16-byte cp.async like the phi tiles: the plain load -> store
      // staging made every thread wait out a global round trip per chunk
      // (a third of the kernel's stall samples at config 1)
      constexpr int QW = KB / 4;
      for (int e = tid; e < FCH * QW; e += 256) {
        const int fl = e / QW, q = e % QW, f = c0 + fl;
        const bool v = f < F && 4 * q < K;
        cp_async16(ws + fl * LDW + 4 * q, Wn + (v ? (size_t)f * K + 4 * q : 0), v);
      }
    } else {
      for (int e = tid; e < FCH * KB; e += 256) {
        const int fl = e / KB, k = e % KB, f = c0 + fl;
        ws[fl * LDW + k] = (f < F && k < K) ? Wn[(size_t)f * K + k] : R(0);
      }
    }
    if (async) {
      constexpr int Q = TT / 4;
      for (int e = tid; e < FCH * Q; e += 256) {
        const int fl = e / Q, q = e % Q, f = c0 + fl, t = t0 + 4 * q;
        const bool v = f < F && t < T;
        const size_t off = v ? (size_t)f * T + t : 0;
        cp_async16(p1s + fl * LDP + 4 * q, P1 + off, v);
        cp_async16(p2s + fl * LDP + 4 * q, P2 + off, v);
      }
    } else {
      for (int e = tid; e < FCH * TT; e += 256) {
        const int fl = e / TT, tl = e % TT, f = c0 + fl, t = t0 + tl;
        const bool v = f < F && t < T;
        p1s[fl * LDP + tl] = v ? P1[(size_t)f * T + t] : R(0);
        p2s[fl * LDP + tl] = v ? P2[(size_t)f * T + t] : R(0);
      }
    }
    cp_async_commit();
  };
  R a1[4][4], a2[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) a1[i][j] = a2[i][j] = 0;
  int st = 0;
  const int fbeg = blockIdx.z * frange, fend = min(F, fbeg + frange);  // this CTA's bin range
  load(0, fbeg);
  for (int c0 = fbeg; c0 < fend; c0 += FCH, st ^= 1) {
    if (c0 + FCH < fend) {
      load(st ^ 1, c0 + FCH);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const R* ws = stage(st);
    const R* p1s = ws + FCH * LDW;
    const R* p2s = p1s + FCH * LDP;
    const int fe = min(FCH, fend - c0);
    for (int fl = s; fl < fe; fl += S) {
      R w[4], x1[4], x2[4];
      lds4(ws + fl * LDW + kg * 4, w);
      lds4(p1s + fl * LDP + tg * 4, x1);
      lds4(p2s + fl * LDP + tg * 4, x2);
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          a1[i][j] += w[i] * x1[j];
          a2[i][j] += w[i] * x2[j];
        }
    }
    __syncthreads();
  }
  R* red = stage0;  // [S][2][KB][TT]
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int idx = (kg * 4 + i) * TT + tg * 4 + j;
      red[(s * 2) * KB * TT + idx] = a1[i][j];
      red[(s * 2 + 1) * KB * TT + idx] = a2[i][j];
    }
  __syncthreads();
  R* Hn = H + (size_t)bn * K * T;
  const int FS = gridDim.z;
  R* pt = part + ((size_t)(bn * gridDim.x + blockIdx.x) * FS) * 2 * KB * TT;  // [FS][2][KB][TT]
  if (FS > 1) {
    // bin-split: publish this CTA's sums; the last CTA of the T-tile adds the
    // FS partials in split order (deterministic) and finishes the update
    for (int e = tid; e < KB * TT; e += 256) {
      R sn = 0, sd = 0;
      for (int q = 0; q < S; ++q) {
        sn += red[(q * 2) * KB * TT + e];
        sd += red[(q * 2 + 1) * KB * TT + e];
      }
      pt[((size_t)blockIdx.z * 2) * KB * TT + e] = sn;
      pt[((size_t)blockIdx.z * 2 + 1) * KB * TT + e] = sd;
    }
    __threadfence();
    __syncthreads();
    __shared__ unsigned last;
    if (tid == 0) last = atomicAdd(cnt + bn * gridDim.x + blockIdx.x, 1u) == (unsigned)FS - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    if (tid == 0) cnt[bn * gridDim.x + blockIdx.x] = 0;  // re-armed for the next launch
  }
  for (int e = tid; e < KB * TT; e += 256) {
    const int k = e / TT, tl = e % TT, t = t0 + tl;
    if (k < K && t < T) {
      R sn = 0, sd = 0;
      if (FS > 1) {
        for (int z = 0; z < FS; ++z) {
          sn += __ldcg(pt + ((size_t)z * 2) * KB * TT + e);
          sd += __ldcg(pt + ((size_t)z * 2 + 1) * KB * TT + e);
        }
      } else {
        for (int q = 0; q < S; ++q) {
          sn += red[(q * 2) * KB * TT + e];
          sd += red[(q * 2 + 1) * KB * TT + e];
        }
      }
      if (mode == 0) {
        Hn[(size_t)k * T + t] *= mu_factor(sn, sd);  // sources.py:198
      } else {
        const size_t NKT = (size_t)Nn * K * T;
        hout[(size_t)b * 2 * NKT + (size_t)nl * K * T + (size_t)k * T + t] = sn;
        hout[(size_t)b * 2 * NKT + NKT + (size_t)nl * K * T + (size_t)k * T + t] = sd;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Statistics pass at one (f, t): phi1[n] = sum_m g x~/y^2, phi2[n] = sum_m g/y,
// and the data term sum_m (-x~/y - log y)  (_kernels.py:226-243).
// Loops over sources exit early (uniform branch) instead of predicating.
// ---------------------------------------------------------------------------
// 1/y: MUFU.RCP (rcp.approx, <= 1 ulp) in fp32 -- the IEEE __frcp_rn sequence
// with its slow path cost ~50 instructions per call in the streaming loops
__device__ __forceinline__ float rcp_r(float y) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(y));
  return r;
}
__device__ __forceinline__ double rcp_r(double y) { return 1.0 / y; }

template <typename R, int M>
__device__ __forceinline__ void model_power(const R (&l)[NMAX], const R* gs, int N, R fl,
                                            R (&iy)[M], R (&y)[M]) {
#pragma unroll
  for (int m = 0; m < M; ++m) y[m] = 0;
#pragma unroll
  for (int n = 0; n < NMAX; ++n) {
    if (n >= N) break;
    R g[M];
    RowIO<R, M>::load(gs + n * M, g);
#pragma unroll
    for (int m = 0; m < M; ++m) y[m] += l[n] * g[m];
  }
#pragma unroll
  for (int m = 0; m < M; ++m) {
    y[m] = floor_max(y[m], fl);
    iy[m] = rcp_r(y[m]);
  }
}

template <typename R, int M>
__device__ __forceinline__ void phi_point(const R (&xtv)[M], const R (&iy)[M], const R* gs, int N,
                                          R* phi, size_t FT, size_t off) {
  R r[M];
#pragma unroll
  for (int m = 0; m < M; ++m) r[m] = xtv[m] * iy[m] * iy[m];
#pragma unroll
  for (int n = 0; n < NMAX; ++n) {
    if (n >= N) break;
    R g[M];
    RowIO<R, M>::load(gs + n * M, g);
    R p1 = 0, p2 = 0;
#pragma unroll
    for (int m = 0; m < M; ++m) {
      p1 += g[m] * r[m];
      p2 += g[m] * iy[m];
    }
    phi[(size_t)n * FT + off] = p1;
    phi[(size_t)(N + n) * FT + off] = p2;
  }
}

// refresh after the W step (separate.py:215): grid (ceil(T/256), F, B), block 256
template <typename R, int M>
__global__ void __launch_bounds__(256) k_phi(const R* __restrict__ lam, const R* __restrict__ xt,
                                             const R* __restrict__ g, const R* __restrict__ floorp,
                                             R* __restrict__ phi, int N, int F, int T) {
  pdl_entry();
  __shared__ __align__(16) R gs[NMAX * M];
  const int f = blockIdx.y, b = blockIdx.z, tid = threadIdx.x;
  const int t = blockIdx.x * 256 + tid;
  const size_t FT = (size_t)F * T;
  // M <= 8: the frame's own loads go out before the gains are staged, so a CTA
  // waits for one global round trip, not two (gains -> barrier -> lambda, x~;
  // c1 k_phi). At M = 16 the values held across the barrier cost more than the
  // round trip (c3: 248 -> 256 us), so the loads stay behind it there.
  if constexpr (M <= 8) {
    const int tc = t < T ? t : T - 1;
    const R fl = floorp[b];
    const R* lb = lam + (size_t)b * N * FT + (size_t)f * T + tc;
    R l[NMAX];
#pragma unroll
    for (int n = 0; n < NMAX; ++n) l[n] = n < N ? lb[(size_t)n * FT] : R(0);
    R xtv[M], iy[M], y[M];
    RowIO<R, M>::load(xt + (((size_t)b * F + f) * T + tc) * M, xtv);
    for (int e = tid; e < N * M; e += 256)
      gs[e] = g[(size_t)b * N * F * M + (size_t)(e / M) * F * M + (size_t)f * M + (e % M)];
    __syncthreads();
    if (t >= T) return;
    model_power<R, M>(l, gs, N, fl, iy, y);
    phi_point<R, M>(xtv, iy, gs, N, phi + (size_t)b * 2 * N * FT, FT, (size_t)f * T + t);
  } else {
    for (int e = tid; e < N * M; e += 256)
      gs[e] = g[(size_t)b * N * F * M + (size_t)(e / M) * F * M + (size_t)f * M + (e % M)];
    __syncthreads();
    if (t >= T) return;
    const R fl = floorp[b];
    const R* lb = lam + (size_t)b * N * FT + (size_t)f * T + t;
    R l[NMAX];
#pragma unroll
    for (int n = 0; n < NMAX; ++n) l[n] = n < N ? lb[(size_t)n * FT] : R(0);
    R xtv[M], iy[M], y[M];
    RowIO<R, M>::load(xt + (((size_t)b * F + f) * T + t) * M, xtv);
    model_power<R, M>(l, gs, N, fl, iy, y);
    phi_point<R, M>(xtv, iy, gs, N, phi + (size_t)b * 2 * N * FT, FT, (size_t)f * T + t);
  }
}

}  // namespace fm
