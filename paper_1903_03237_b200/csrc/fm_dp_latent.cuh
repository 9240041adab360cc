// fm_dp_latent.cuh -- the whole latent hook of FastMNMF-DP in ONE launch.
//
// The hook (separate.py:205-213 with the config-4 update) takes `steps` Adam
// steps on z against the frozen rest-of-model power, then refreshes
// r = exp(dec(z)). Frame t's latent z_t only reaches r[t, :], and its
// gradient only involves frame t, so every frame's Adam trajectory is
// independent: one CTA owns FR = 4 frames of one mixture and runs all steps,
// forward and backward, with activations, Adam moments and the output-layer
// gradient on chip. The decoder weights stream from L2 through an S-stage
// cp.async pipeline (S = 2..4, as shared memory allows) in CH-row chunks; the output layer W3 is read ONCE per step:
// each W3 chunk gives o[t, f-chunk] (forward), the NLL gradient dL/do for
// those bins, and the chunk's contribution to W3^T dL/do (backward).
//
// Per step the chunk sequence is
//   A1: h1 = tanh(W1 z + b1)          (W1 rows, forward)
//   A2: h2 = tanh(W2 h1 + b2)         (W2 rows, forward)
//   O : o = W3 h2 + b3, r = exp(o), go = dL/do, d2 += W3^T go
//   C2: d1 += W2^T (d2 (1 - h2^2))
//   C1: gz += W1^T (d1 (1 - h1^2)); Adam(z, gz)
// and the final refresh runs A1, A2, O writing r to HBM.
//
// Work split inside a chunk (CH = 64 rows fp32, 32 fp64): warp w owns CH/8
// consecutive chunk rows, lane l owns the 4 columns of 16-byte segment(s)
// l (+32). A forward row product is a lane partial over the lane's columns,
// reduced across the warp by a 32- (16-) value butterfly that leaves lane l
// with output (row, frame) = (l/4, l%4) (fp64: ((l/2)/4, (l/2)%4)); the
// backward product reuses the same staged weights in registers
// (acc[col][frame] += coef[row][frame] * W[row][col]), so an O chunk needs no
// barrier between its forward, gradient and backward parts. Warp partials of
// the backward products meet once per layer in a fixed-order sum.
// grid (ceil(T/4), B), block 256.
#pragma once
#include <type_traits>

#include "fm_dp.cuh"
#include "fm_spatial.cuh"

namespace fm {

constexpr int LT_LDW = DEC_HMAX;      // row pitch of a staged chunk (elements)
constexpr int LT_FR = 4;              // frames per CTA

template <typename R> struct LatentArgs {
  const R *W1, *b1, *W2, *b2, *W3, *b3;  // decoder (W1 Hd x D, W2 Hd x Hd, W3 F x Hd)
  const R *u, *v;                        // (B, F), (B, T)
  R *z, *m, *v2;                         // (B, T, D) latents and Adam moments
  R* r;                                  // (B, T, F) decoder output exp(dec(z))
  const R* lam;                          // (B, N, F, T); sources >= 1 are the frozen noise
  const R* xt;                           // (B, F, T, M)
  const R* g;                            // (B, N, F, M)
  const unsigned* iter;                  // device iteration counter (Adam step index)
  int T, F, D, Hd, N, steps, stages;
  float lr, b1a, b2a, eps;
};

template <typename R, int M> struct LtCfg {
  static constexpr int FR = LT_FR;
  static constexpr int VEC = 16 / (int)sizeof(R);           // elements per 16-byte segment
  static constexpr int SPL = DEC_HMAX / VEC / 32;           // segments per lane
  static constexpr int NCL = SPL * VEC;                     // columns per lane (4)
  static constexpr bool XVEC = (M * sizeof(R)) % 16 == 0;   // x~ / g rows in 16-byte segments
  static constexpr int CH = sizeof(R) == 4 ? 64 : 32;       // weight rows per chunk
  static constexpr int NT = 256;                             // threads per CTA
  static constexpr int NW = NT / 32;                        // warps
  static constexpr int RPW = CH / NW;                       // chunk rows per warp (4)
  static constexpr int WB = CH * LT_LDW;                    // one weight buffer
  static constexpr int NV = RPW * FR;                       // forward outputs per warp
  static constexpr int QSH = NV == 8 ? 2 : NV == 16 ? 1 : 0; // lane -> output shift
  static_assert(NV == 8 || NV == 16 || NV == 32, "butterfly sizes");
  static_assert(NCL % 2 == 0, "column pairs");
  static_assert(NW * FR * DEC_HMAX <= WB, "layer-end partials fit a weight buffer");
};

// shared-memory carve (elements of R) for S pipeline stages and N sources;
// the layer-end warp partials [NW][FR][HMAX] reuse the consumed weight buffer
struct LtLayout {
  int S, stage;                 // stages, elements per stage
  int W, XS, LS, GS, US, BS;    // offsets inside a stage
  int ZT, H1, H2, D1, D2, AM, AV, B1, B2, VS, total;
};
template <typename R, int M> __host__ __device__ inline LtLayout lt_layout(int S, int N) {
  constexpr int FR = LT_FR, LT_CH = LtCfg<R, M>::CH;
  auto up4 = [](int x) { return (x + 3) / 4 * 4; };
  LtLayout L;
  L.S = S;
  L.W = 0;
  L.XS = L.W + LT_CH * LT_LDW;
  L.LS = L.XS + up4(LT_CH * FR * M);
  L.GS = L.LS + up4((N - 1) * LT_CH * FR);
  L.US = L.GS + up4(N * LT_CH * M);
  L.BS = L.US + LT_CH;
  L.stage = L.BS + LT_CH;
  L.ZT = S * L.stage;
  L.H1 = L.ZT + DEC_DMAX * FR;
  L.H2 = L.H1 + DEC_HMAX * FR;
  L.D1 = L.H2 + DEC_HMAX * FR;
  L.D2 = L.D1 + DEC_HMAX * FR;
  L.AM = L.D2 + DEC_HMAX * FR;
  L.AV = L.AM + FR * DEC_DMAX;
  L.B1 = L.AV + FR * DEC_DMAX;
  L.B2 = L.B1 + DEC_HMAX;
  L.VS = L.B2 + DEC_HMAX;
  L.total = up4(L.VS + FR);
  return L;
}

template <typename R> __device__ __forceinline__ void cp_async_el(R* s, const R* gp) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"(
                   (unsigned)__cvta_generic_to_shared(s)),
               "l"(gp), "n"((int)sizeof(R)));
}

enum { LT_A1 = 0, LT_A2 = 1, LT_O = 2, LT_C2 = 3, LT_C1 = 4, LT_END = 5 };

// chunk sequence: steps x [A1 A2 O C2 C1] then the refresh [A1 A2 O]
struct LtIt {
  int grp, idx, s;
  __device__ __forceinline__ int count(int nc1, int nc3) const { return grp == LT_O ? nc3 : nc1; }
  __device__ __forceinline__ bool last(int nc1, int nc3) const { return idx == count(nc1, nc3) - 1; }
  __device__ __forceinline__ void next(int nc1, int nc3, int steps) {
    if (++idx < count(nc1, nc3)) return;
    idx = 0;
    if (grp == LT_C1) { grp = LT_A1; ++s; }
    else if (grp == LT_O && s == steps) grp = LT_END;
    else ++grp;
  }
};

template <typename R, int VEC> __device__ __forceinline__ void lds_vec(const R* p, R* v) {
  if constexpr (VEC == 4) {
    const float4 q = *reinterpret_cast<const float4*>(p);
    v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
  } else {
    const double2 q = *reinterpret_cast<const double2*>(p);
    v[0] = q.x; v[1] = q.y;
  }
}

// one butterfly level: lanes with bit `MASK` set keep the upper half
template <int HALF, int MASK, typename R> __device__ __forceinline__ void lt_fold(R* v, int lane) {
  const bool hi = lane & MASK;
#pragma unroll
  for (int j = 0; j < HALF; ++j) {
    const R send = hi ? v[j] : v[j + HALF];
    const R keep = hi ? v[j + HALF] : v[j];
    v[j] = keep + __shfl_xor_sync(0xffffffffu, send, MASK);
  }
}
// warp sum of NV per-lane partials; lane l returns the total of output l >> (5 - log2 NV)
template <int NV, typename R> __device__ __forceinline__ R lt_reduce(R (&v)[NV], int lane) {
  if constexpr (NV >= 2) lt_fold<NV / 2, 16>(v, lane);
  if constexpr (NV >= 4) lt_fold<NV / 4, 8>(v, lane);
  if constexpr (NV >= 8) lt_fold<NV / 8, 4>(v, lane);
  if constexpr (NV >= 16) lt_fold<NV / 16, 2>(v, lane);
  if constexpr (NV >= 32) lt_fold<1, 1>(v, lane);
  R x = v[0];
  if constexpr (NV < 32) x += __shfl_xor_sync(0xffffffffu, x, 1);
  if constexpr (NV < 16) x += __shfl_xor_sync(0xffffffffu, x, 2);
  if constexpr (NV < 8) x += __shfl_xor_sync(0xffffffffu, x, 4);
  return x;
}

template <typename R, int M>
__global__ void __launch_bounds__(LtCfg<R, M>::NT) k_dp_latent(LatentArgs<R> a) {
  pdl_entry();
  using C = LtCfg<R, M>;
  constexpr int FR = C::FR, VEC = C::VEC, NCL = C::NCL, SPL = C::SPL;
  const LtLayout L = lt_layout<R, M>(a.stages, a.N);
  const int S = L.S;
  constexpr int LT_CH = C::CH, LT_RPW = C::RPW, LT_NT = C::NT, LT_NW = C::NW;
  using R2 = typename RT<R>::C;
  extern __shared__ __align__(16) unsigned char lt_raw[];
  R* sm = reinterpret_cast<R*>(lt_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int b = blockIdx.y, t0 = blockIdx.x * FR;
  const int T = a.T, F = a.F, D = a.D, Hd = a.Hd, N = a.N;
  const int nr = min(FR, T - t0);
  const int nc1 = (Hd + LT_CH - 1) / LT_CH, nc3 = (F + LT_CH - 1) / LT_CH;
  const size_t FT = (size_t)F * T;

  // latents, Adam moments, biases, v of this CTA's frames
  for (int e = tid; e < DEC_DMAX * FR; e += LT_NT) {
    const int d = e / FR, r = e % FR;
    const bool ok = d < D && r < nr;
    const size_t i = ((size_t)b * T + t0 + r) * D + d;
    sm[L.ZT + e] = ok ? a.z[i] : R(0);
    sm[L.AM + r * DEC_DMAX + d] = ok ? a.m[i] : R(0);
    sm[L.AV + r * DEC_DMAX + d] = ok ? a.v2[i] : R(0);
  }
  for (int j = tid; j < DEC_HMAX; j += LT_NT) {
    sm[L.B1 + j] = j < Hd ? a.b1[j] : R(0);
    sm[L.B2 + j] = j < Hd ? a.b2[j] : R(0);
  }
  if (tid < FR) sm[L.VS + tid] = tid < nr ? a.v[(size_t)b * T + t0 + tid] : R(0);

  // per-thread weight-staging maps for the two row widths (D and Hd)
  const int sgD = D / VEC, sgH = Hd / VEC;
  const int stD = LT_NT / sgD, stH = LT_NT / sgH;
  const int iD0 = tid < stD * sgD ? tid / sgD : LT_CH, sD = tid % sgD;
  const int iH0 = tid < stH * sgH ? tid / sgH : LT_CH, sH = tid % sgH;

  const unsigned sbase = (unsigned)__cvta_generic_to_shared(sm);
  auto load = [&](const LtIt& c, int buf) {
    const bool narrow = c.grp == LT_A1 || c.grp == LT_C1;
    const R* Wm = narrow ? a.W1 : c.grp == LT_O ? a.W3 : a.W2;
    const int rows = c.grp == LT_O ? F : Hd, K = narrow ? D : Hd;
    const int row0 = c.idx * LT_CH, nrow = min(LT_CH, rows - row0);
    const int i0 = narrow ? iD0 : iH0, sg = narrow ? sD : sH, st = narrow ? stD : stH;
    unsigned dst = sbase + (unsigned)((buf * L.stage + L.W + i0 * LT_LDW + sg * VEC) * sizeof(R));
    const R* src = Wm + ((size_t)row0 + i0) * K + sg * VEC;
    const unsigned dstep = (unsigned)(st * LT_LDW * sizeof(R));
    const size_t sstep = (size_t)st * K;
#pragma unroll 4
    for (int i = i0; i < nrow; i += st, dst += dstep, src += sstep)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src));
    if (c.grp != LT_O) return;
    const int f0 = row0;
    R* xs = sm + buf * L.stage + L.XS;
    if constexpr (C::XVEC) {
      constexpr int MS = M / VEC;
      for (int e = tid; e < LT_CH * FR * MS; e += LT_NT) {
        const int fl = e / (FR * MS), q = e % (FR * MS), r = q / MS, sgm = q % MS;
        if (fl < nrow && r < nr)
          cp_async16(xs + (fl * FR + r) * M + sgm * VEC,
                     a.xt + (((size_t)b * F + f0 + fl) * T + t0 + r) * M + sgm * VEC, true);
      }
    } else {
      for (int e = tid; e < LT_CH * FR * M; e += LT_NT) {
        const int fl = e / (FR * M), q = e % (FR * M), r = q / M;
        if (fl < nrow && r < nr)
          cp_async_el(xs + fl * FR * M + q, a.xt + (((size_t)b * F + f0 + fl) * T + t0) * M + q);
      }
    }
    R* ls = sm + buf * L.stage + L.LS;
    for (int e = tid; e < (N - 1) * LT_CH * FR; e += LT_NT) {
      const int n = e / (LT_CH * FR), q = e % (LT_CH * FR), fl = q / FR, r = q % FR;
      if (fl < nrow && r < nr)
        cp_async_el(ls + e, a.lam + ((size_t)b * N + n + 1) * FT + (size_t)(f0 + fl) * T + t0 + r);
    }
    R* gs = sm + buf * L.stage + L.GS;
    if constexpr (C::XVEC) {
      constexpr int GSG = LT_CH * M / VEC;
      for (int e = tid; e < N * GSG; e += LT_NT) {
        const int n = e / GSG, q = e % GSG;
        if (q * VEC < nrow * M)
          cp_async16(gs + n * LT_CH * M + q * VEC, a.g + (((size_t)b * N + n) * F + f0) * M + q * VEC,
                     true);
      }
    } else {
      for (int e = tid; e < N * LT_CH * M; e += LT_NT) {
        const int n = e / (LT_CH * M), q = e % (LT_CH * M);
        if (q < nrow * M) cp_async_el(gs + e, a.g + (((size_t)b * N + n) * F + f0) * M + q);
      }
    }
    if (tid < nrow) {
      cp_async_el(sm + buf * L.stage + L.US + tid, a.u + (size_t)b * F + f0 + tid);
      cp_async_el(sm + buf * L.stage + L.BS + tid, a.b3 + f0 + tid);
    }
  };

  // lane's columns: segment (lane + 32 j) of a staged row, j < SPL
  auto colof = [&](int c) { return (lane + 32 * (c / VEC)) * VEC + (c % VEC); };
  const int q = lane >> C::QSH, qi = q / FR, qr = q % FR;  // lane's output after the butterfly
  const bool qlead = (lane & ((1 << C::QSH) - 1)) == 0;       // one writer per output

  R2 acc[NCL / 2][FR];   // backward partials: (column pair, frame)
  R2 xin[NCL][FR / 2];   // forward input rows of the lane's k columns, per frame pair
#pragma unroll
  for (int c = 0; c < NCL / 2; ++c)
#pragma unroll
    for (int r = 0; r < FR; ++r) acc[c][r] = R2{0, 0};

  // S-stage cp.async pipeline: chunk gi lives in stage gi % S; loads run S-1 chunks ahead
  LtIt cur{LT_A1, 0, 0};
  LtIt ld = cur;
  for (int p = 0; p < S - 1; ++p) {
    if (ld.grp != LT_END) {
      load(ld, p);
      ld.next(nc1, nc3, a.steps);
    }
    cp_async_commit();
  }
  int buf = 0, bld = S - 1;  // stage of the current chunk / of the next load
  for (; cur.grp != LT_END; cur.next(nc1, nc3, a.steps), buf = buf + 1 == S ? 0 : buf + 1,
                            bld = bld + 1 == S ? 0 : bld + 1) {
    if (S == 2) cp_async_wait<0>();
    else if (S == 3) cp_async_wait<1>();
    else cp_async_wait<2>();
    __syncthreads();
    if (ld.grp != LT_END) {
      load(ld, bld);
      ld.next(nc1, nc3, a.steps);
    }
    cp_async_commit();
    R* Wc = sm + buf * L.stage + L.W;
    const bool refresh = cur.s == a.steps;
    const bool fwd = cur.grp <= LT_O;
    const int row0 = cur.idx * LT_CH;
    const int K = (cur.grp == LT_A1 || cur.grp == LT_C1) ? D : Hd;   // staged row width
    const int nrow = min(LT_CH, (cur.grp == LT_O ? F : Hd) - row0);

    // the warp's 4 staged rows, lane's columns (zero outside the chunk / row width)
    R w[LT_RPW][NCL];
#pragma unroll
    for (int i = 0; i < LT_RPW; ++i) {
      const int row = warp * LT_RPW + i;
#pragma unroll
      for (int j = 0; j < SPL; ++j) {
        const int seg = lane + 32 * j;
        if (row < nrow && seg * VEC < K) {
          lds_vec<R, VEC>(Wc + row * LT_LDW + seg * VEC, &w[i][j * VEC]);
        } else {
#pragma unroll
          for (int v = 0; v < VEC; ++v) w[i][j * VEC + v] = 0;
        }
      }
    }

    if (fwd) {
      if (cur.idx == 0) {  // the layer input, in registers for the whole layer
        const R* inT = sm + (cur.grp == LT_A1 ? L.ZT : cur.grp == LT_A2 ? L.H1 : L.H2);
#pragma unroll
        for (int c = 0; c < NCL; ++c) {
          const int k = colof(c);
#pragma unroll
          for (int h = 0; h < FR / 2; ++h)
            xin[c][h] = k < K ? reinterpret_cast<const R2*>(inT + k * FR)[h] : R2{0, 0};
        }
      }
      R pv[C::NV];
#pragma unroll
      for (int i = 0; i < LT_RPW; ++i) {
        R2 s2[FR / 2];
#pragma unroll
        for (int h = 0; h < FR / 2; ++h) s2[h] = R2{0, 0};
#pragma unroll
        for (int c = 0; c < NCL; ++c)
#pragma unroll
          for (int h = 0; h < FR / 2; ++h) s2[h] = fma2(R2{w[i][c], w[i][c]}, xin[c][h], s2[h]);
#pragma unroll
        for (int h = 0; h < FR / 2; ++h) {
          pv[i * FR + 2 * h] = s2[h].x;
          pv[i * FR + 2 * h + 1] = s2[h].y;
        }
      }
      const R o = lt_reduce<C::NV>(pv, lane);
      const int rl = warp * LT_RPW + qi, j = row0 + rl;  // chunk row, global row
      if (cur.grp == LT_A1) {
        if (qlead && j < Hd) sm[L.H1 + j * FR + qr] = tanh(o + sm[L.B1 + j]);
        continue;
      }
      if (cur.grp == LT_A2) {
        if (qlead && j < Hd) sm[L.H2 + j * FR + qr] = tanh(o + sm[L.B2 + j]);
        continue;
      }
      // output layer + NLL gradient dL/do of sum x~/y + log y (all copies of an output)
      const bool ok = j < F && qr < nr;
      R go = 0;
      if (ok) {
        const R rr = exp(o + sm[buf * L.stage + L.BS + rl]);
        if (refresh) {
          if (qlead) a.r[((size_t)b * T + t0 + qr) * F + j] = rr;
        } else {
          const R l0 = sm[buf * L.stage + L.US + rl] * sm[L.VS + qr] * rr;
          const R* xr = sm + buf * L.stage + L.XS + (rl * FR + qr) * M;
          const R* ls = sm + buf * L.stage + L.LS + rl * FR + qr;
          const R* gs = sm + buf * L.stage + L.GS + rl * M;
          R ln[NMAX];
#pragma unroll
          for (int n = 1; n < NMAX; ++n) {
            ln[n] = R(0);
            if (n >= N) break;
            ln[n] = ls[(n - 1) * LT_CH * FR];
          }
          R s = 0;
#pragma unroll
          for (int m = 0; m < M; ++m) {
            R rest = 0;
#pragma unroll
            for (int n = 1; n < NMAX; ++n) {
              if (n >= N) break;
              rest += ln[n] * gs[n * LT_CH * M + m];
            }
            const R g0 = gs[m];
            R y = l0 * g0 + rest;
            y = y > RT<R>::tiny() ? y : RT<R>::tiny();
            const R iy = rcp_r(y);
            s += g0 * (iy - xr[m] * iy * iy);
          }
          go = s * l0;
        }
      }
      if (refresh) continue;
      // backward part of the O chunk: acc[col][r] += go[row][r] W3[row][col]
#pragma unroll
      for (int qq = 0; qq < LT_RPW * FR; ++qq) {
        const R gq = __shfl_sync(0xffffffffu, go, qq << C::QSH);
        const int i = qq / FR, r = qq % FR;
#pragma unroll
        for (int c = 0; c < NCL / 2; ++c)
          acc[c][r] = fma2(R2{w[i][2 * c], w[i][2 * c + 1]}, R2{gq, gq}, acc[c][r]);
      }
    } else {
      // C2 / C1: acc[col][r] += coef[row][r] W[row][col]
      const R* coef = sm + (cur.grp == LT_C2 ? L.D2 : L.D1) + (row0 + warp * LT_RPW) * FR;
#pragma unroll
      for (int i = 0; i < LT_RPW; ++i) {
        R cf[FR];
#pragma unroll
        for (int h = 0; h < FR / 2; ++h) {
          const R2 t = reinterpret_cast<const R2*>(coef + i * FR)[h];
          cf[2 * h] = t.x;
          cf[2 * h + 1] = t.y;
        }
#pragma unroll
        for (int r = 0; r < FR; ++r)
#pragma unroll
          for (int c = 0; c < NCL / 2; ++c)
            acc[c][r] = fma2(R2{w[i][2 * c], w[i][2 * c + 1]}, R2{cf[r], cf[r]}, acc[c][r]);
      }
    }
    if (!cur.last(nc1, nc3)) continue;

    // layer end: warp partials -> the consumed weight buffer -> fixed-order sum
    const int ncol = cur.grp == LT_C1 ? D : Hd;
    __syncthreads();
    R* red = Wc;  // [NW][FR][HMAX]
#pragma unroll
    for (int c = 0; c < NCL / 2; ++c)
#pragma unroll
      for (int r = 0; r < FR; ++r) {
        const int col = colof(2 * c);
        red[(warp * FR + r) * DEC_HMAX + col] = acc[c][r].x;
        red[(warp * FR + r) * DEC_HMAX + col + 1] = acc[c][r].y;
        acc[c][r] = R2{0, 0};
      }
    __syncthreads();
    double c1 = 0, c2 = 0;
    if (cur.grp == LT_C1) {  // Adam step index iter * steps + s + 1
      const double tstep = (double)(*a.iter) * a.steps + cur.s + 1;
      c1 = 1.0 - pow((double)a.b1a, tstep);
      c2 = 1.0 - pow((double)a.b2a, tstep);
    }
    for (int e = tid; e < FR * DEC_HMAX; e += LT_NT) {
      const int r = e / DEC_HMAX, col = e % DEC_HMAX;
      if (col >= ncol) continue;
      R sum = 0;
#pragma unroll
      for (int ww = 0; ww < LT_NW; ++ww) sum += red[(ww * FR + r) * DEC_HMAX + col];
      const int i = col * FR + r;
      if (cur.grp == LT_O) {  // d2 = (W3^T go) (1 - h2^2)
        const R hv = sm[L.H2 + i];
        sm[L.D2 + i] = sum * (R(1) - hv * hv);
      } else if (cur.grp == LT_C2) {  // d1 = (W2^T d2) (1 - h1^2)
        const R hv = sm[L.H1 + i];
        sm[L.D1 + i] = sum * (R(1) - hv * hv);
      } else if (r < nr) {  // gz = W1^T d1; Adam on z
        R* mp = sm + L.AM + r * DEC_DMAX + col;
        R* vp = sm + L.AV + r * DEC_DMAX + col;
        const R mi = R(a.b1a) * *mp + R(1 - a.b1a) * sum;
        const R vi = R(a.b2a) * *vp + R(1 - a.b2a) * sum * sum;
        *mp = mi;
        *vp = vi;
        sm[L.ZT + i] -= R(a.lr) * (mi / (R)c1) / (sqrt_r(vi / (R)c2) + R(a.eps));
      }
    }
  }
  cp_async_wait<0>();
  __syncthreads();
  if (a.steps == 0) return;
  for (int e = tid; e < D * nr; e += LT_NT) {
    const int r = e / D, d = e - r * D;
    const size_t i = ((size_t)b * T + t0 + r) * D + d;
    a.z[i] = sm[L.ZT + d * FR + r];
    a.m[i] = sm[L.AM + r * DEC_DMAX + d];
    a.v2[i] = sm[L.AV + r * DEC_DMAX + d];
  }
}

}  // namespace fm
