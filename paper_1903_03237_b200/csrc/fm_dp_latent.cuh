// fm_dp_latent.cuh -- the whole latent hook of FastMNMF-DP in ONE launch.
//
// The hook (separate.py:205-213 with the config-4 update) takes `steps` Adam
// steps on z against the frozen rest-of-model power, then refreshes
// r = exp(dec(z)). Frame t's latent z_t only reaches r[t, :], and its
// gradient only involves frame t, so every frame's Adam trajectory is
// independent: one CTA owns RT frames of one mixture and runs all steps,
// forward and backward, with activations, Adam moments and the output-layer
// gradient on chip. The decoder weights stream from L2 through a cp.async
// double buffer in 32-row chunks (16-byte segments, XOR-swizzled by row so
// both the row-parallel forward and the column-parallel backward products
// read shared memory conflict-free); the output layer W3 is read ONCE per step:
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
// grid (ceil(T/RT), B), block 256.
#pragma once
#include "fm_dp.cuh"
#include "fm_spatial.cuh"

namespace fm {

constexpr int LT_NT = 256;             // threads per CTA
constexpr int LT_CH = 32;              // weight rows per chunk
constexpr int LT_LDW = DEC_HMAX;       // row pitch of a staged chunk (elements)
constexpr int LT_KQ = LT_NT / LT_CH;   // k-slices of the forward chunk product

template <typename R> struct LatentArgs {
  const R *W1, *b1, *W2, *b2, *W3, *b3;  // decoder (W1 Hd x D, W2 Hd x Hd, W3 F x Hd)
  const R *u, *v;                        // (B, F), (B, T)
  R *z, *m, *v2;                         // (B, T, D) latents and Adam moments
  R* r;                                  // (B, T, F) decoder output exp(dec(z))
  const R* lam;                          // (B, N, F, T); sources >= 1 are the frozen noise
  const R* xt;                           // (B, F, T, M)
  const R* g;                            // (B, N, F, M)
  const unsigned* iter;                  // device iteration counter (Adam step index)
  int T, F, D, Hd, N, steps;
  float lr, b1a, b2a, eps;
};

template <typename R, int M, int RT> struct LtCfg {
  static constexpr int VEC = 16 / (int)sizeof(R);           // elements per 16-byte segment
  static constexpr int SEGMAX = DEC_HMAX / VEC;             // segments per staged row
  static constexpr int NQ = LT_NT / SEGMAX;                 // backward: threads per column segment
  static constexpr int RP = 2;                              // backward: frames per thread
  static constexpr int NRP = RT / RP;                       // backward: frame groups
  static constexpr int NIQ = NQ / NRP;                      // backward: chunk-row slices
  static constexpr bool XVEC = (M * sizeof(R)) % 16 == 0;   // x~ / g rows in 16-byte segments
  static_assert(RT % RP == 0 && NQ % NRP == 0, "frame tiling");
  // shared-memory carve (elements of R)
  static constexpr int RED_A = LT_KQ * RT * LT_CH, RED_C = NIQ * RT * DEC_HMAX;
  static constexpr int W = 0;                                    // [2][LT_CH][LT_LDW] swizzled
  static constexpr int XS = W + 2 * LT_CH * LT_LDW;              // [2][LT_CH][RT][M]
  static constexpr int LS = XS + 2 * LT_CH * RT * M;             // [2][NMAX-1][LT_CH][RT]
  static constexpr int GS = LS + 2 * (NMAX - 1) * LT_CH * RT;    // [2][NMAX][LT_CH][M]
  static constexpr int US = GS + 2 * NMAX * LT_CH * M;           // [2][LT_CH]
  static constexpr int BS = US + 2 * LT_CH;                      // [2][LT_CH]
  static constexpr int ZT = BS + 2 * LT_CH;                      // [DMAX][RT]
  static constexpr int H1 = ZT + DEC_DMAX * RT;                  // [HMAX][RT]
  static constexpr int H2 = H1 + DEC_HMAX * RT;
  static constexpr int D1 = H2 + DEC_HMAX * RT;
  static constexpr int D2 = D1 + DEC_HMAX * RT;
  static constexpr int RED = D2 + DEC_HMAX * RT;                 // partial sums (both phases)
  static constexpr int GO = RED + (RED_A > RED_C ? RED_A : RED_C);  // [LT_CH][RT]
  static constexpr int AM = GO + LT_CH * RT;                     // [RT][DMAX]
  static constexpr int AV = AM + RT * DEC_DMAX;
  static constexpr int B1 = AV + RT * DEC_DMAX;                  // [HMAX]
  static constexpr int B2 = B1 + DEC_HMAX;
  static constexpr int VS = B2 + DEC_HMAX;                       // [RT]
  static constexpr int TOTAL = ((VS + RT) + 3) / 4 * 4;
};

template <typename R> __device__ __forceinline__ void cp_async_el(R* s, const R* gp) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"(
                   (unsigned)__cvta_generic_to_shared(s)),
               "l"(gp), "n"((int)sizeof(R)));
}

// swizzled position of element (row, k) in a staged chunk: 16-byte segment
// k / VEC lands at segment (k / VEC) ^ (row & 7)
template <int VEC> __device__ __forceinline__ int lt_swz(int row, int k) {
  return row * LT_LDW + ((((k / VEC) ^ (row & 7))) * VEC) + (k % VEC);
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

template <typename R, int VEC> __device__ __forceinline__ void lds_vec(const R* p, R (&v)[VEC]) {
  if constexpr (VEC == 4) {
    const float4 q = *reinterpret_cast<const float4*>(p);
    v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
  } else {
    const double2 q = *reinterpret_cast<const double2*>(p);
    v[0] = q.x; v[1] = q.y;
  }
}

template <typename R, int M, int RT>
__global__ void __launch_bounds__(LT_NT) k_dp_latent(LatentArgs<R> a) {
  pdl_entry();
  using C = LtCfg<R, M, RT>;
  constexpr int VEC = C::VEC;
  using R2 = typename std::conditional<sizeof(R) == 4, float2, double2>::type;
  extern __shared__ __align__(16) unsigned char lt_raw[];
  R* sm = reinterpret_cast<R*>(lt_raw);
  const int tid = threadIdx.x, b = blockIdx.y, t0 = blockIdx.x * RT;
  const int T = a.T, F = a.F, D = a.D, Hd = a.Hd, N = a.N;
  const int nr = min(RT, T - t0);
  const int nc1 = (Hd + LT_CH - 1) / LT_CH, nc3 = (F + LT_CH - 1) / LT_CH;
  const size_t FT = (size_t)F * T;

  // latents, Adam moments, biases, v of this CTA's frames
  for (int e = tid; e < DEC_DMAX * RT; e += LT_NT) {
    const int d = e / RT, r = e % RT;
    const bool ok = d < D && r < nr;
    const size_t i = ((size_t)b * T + t0 + r) * D + d;
    sm[C::ZT + e] = ok ? a.z[i] : R(0);
    sm[C::AM + r * DEC_DMAX + d] = ok ? a.m[i] : R(0);
    sm[C::AV + r * DEC_DMAX + d] = ok ? a.v2[i] : R(0);
  }
  for (int j = tid; j < DEC_HMAX; j += LT_NT) {
    sm[C::B1 + j] = j < Hd ? a.b1[j] : R(0);
    sm[C::B2 + j] = j < Hd ? a.b2[j] : R(0);
  }
  if (tid < RT) sm[C::VS + tid] = tid < nr ? a.v[(size_t)b * T + t0 + tid] : R(0);

  // per-thread weight-staging maps for the two row widths (D and Hd)
  const int sgD = D / VEC, sgH = Hd / VEC;
  const int stD = LT_NT / sgD, stH = LT_NT / sgH;
  const int iD0 = tid < stD * sgD ? tid / sgD : LT_CH, sD = tid % sgD;
  const int iH0 = tid < stH * sgH ? tid / sgH : LT_CH, sH = tid % sgH;

  auto load = [&](const LtIt& c, int buf) {
    const bool narrow = c.grp == LT_A1 || c.grp == LT_C1;
    const R* Wm = narrow ? a.W1 : c.grp == LT_O ? a.W3 : a.W2;
    const int rows = c.grp == LT_O ? F : Hd, K = narrow ? D : Hd;
    const int row0 = c.idx * LT_CH, nrow = min(LT_CH, rows - row0);
    R* Wc = sm + C::W + buf * LT_CH * LT_LDW;
    const R* Wg = Wm + (size_t)row0 * K;
    const int i0 = narrow ? iD0 : iH0, sg = narrow ? sD : sH, st = narrow ? stD : stH;
    for (int i = i0; i < nrow; i += st)
      cp_async16(Wc + i * LT_LDW + ((sg ^ (i & 7)) * VEC), Wg + (size_t)i * K + sg * VEC, true);
    if (c.grp != LT_O) return;
    const int f0 = row0;
    R* xs = sm + C::XS + buf * LT_CH * RT * M;
    if constexpr (C::XVEC) {
      constexpr int MS = M / VEC;
      for (int e = tid; e < LT_CH * RT * MS; e += LT_NT) {
        const int fl = e / (RT * MS), q = e % (RT * MS), r = q / MS, sgm = q % MS;
        if (fl < nrow && r < nr)
          cp_async16(xs + (fl * RT + r) * M + sgm * VEC,
                     a.xt + (((size_t)b * F + f0 + fl) * T + t0 + r) * M + sgm * VEC, true);
      }
    } else {
      for (int e = tid; e < LT_CH * RT * M; e += LT_NT) {
        const int fl = e / (RT * M), q = e % (RT * M), r = q / M;
        if (fl < nrow && r < nr)
          cp_async_el(xs + fl * RT * M + q, a.xt + (((size_t)b * F + f0 + fl) * T + t0) * M + q);
      }
    }
    R* ls = sm + C::LS + buf * (NMAX - 1) * LT_CH * RT;
    for (int e = tid; e < (N - 1) * LT_CH * RT; e += LT_NT) {
      const int n = e / (LT_CH * RT), q = e % (LT_CH * RT), fl = q / RT, r = q % RT;
      if (fl < nrow && r < nr)
        cp_async_el(ls + e, a.lam + ((size_t)b * N + n + 1) * FT + (size_t)(f0 + fl) * T + t0 + r);
    }
    R* gs = sm + C::GS + buf * NMAX * LT_CH * M;
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
      cp_async_el(sm + C::US + buf * LT_CH + tid, a.u + (size_t)b * F + f0 + tid);
      cp_async_el(sm + C::BS + buf * LT_CH + tid, a.b3 + f0 + tid);
    }
  };

  // backward-product thread map: column segment, frame pair, chunk-row slice
  const int cseg = tid % C::SEGMAX, cq = tid / C::SEGMAX;
  const int crp = cq % C::NRP, ciq = cq / C::NRP;
  R accC[VEC][C::RP];
#pragma unroll
  for (int v = 0; v < VEC; ++v)
#pragma unroll
    for (int h = 0; h < C::RP; ++h) accC[v][h] = 0;

  LtIt cur{LT_A1, 0, 0};
  if (a.steps == 0) cur.s = 0;
  LtIt nxt = cur;
  load(cur, 0);
  cp_async_commit();
  for (int gi = 0; cur.grp != LT_END; ++gi, cur = nxt) {
    cp_async_wait<0>();
    __syncthreads();
    nxt.next(nc1, nc3, a.steps);
    if (nxt.grp != LT_END) load(nxt, (gi + 1) & 1);
    cp_async_commit();
    const int buf = gi & 1;
    const R* Wc = sm + C::W + buf * LT_CH * LT_LDW;
    const bool refresh = cur.s == a.steps;
    const int row0 = cur.idx * LT_CH;

    if (cur.grp <= LT_O) {
      // forward chunk: out[r][row0 + row] = sum_k Wc[row][k] in[k][r]
      const int K = cur.grp == LT_A1 ? D : Hd;
      const R* inT = sm + (cur.grp == LT_A1 ? C::ZT : cur.grp == LT_A2 ? C::H1 : C::H2);
      const int row = tid & (LT_CH - 1), kq = tid / LT_CH;
      const int nsg = K / VEC, spq = (nsg + LT_KQ - 1) / LT_KQ;
      const int s0 = kq * spq, s1 = min(nsg, s0 + spq);
      R2 acc[RT / 2];
#pragma unroll
      for (int h = 0; h < RT / 2; ++h) acc[h] = R2{0, 0};
      const R* wrow = Wc + row * LT_LDW;
      for (int sg = s0; sg < s1; ++sg) {
        R w[VEC];
        lds_vec<R, VEC>(wrow + ((sg ^ (row & 7)) * VEC), w);
#pragma unroll
        for (int v = 0; v < VEC; ++v) {
          const R2* in2 = reinterpret_cast<const R2*>(inT + (sg * VEC + v) * RT);
#pragma unroll
          for (int h = 0; h < RT / 2; ++h) acc[h] = fma2(R2{w[v], w[v]}, in2[h], acc[h]);
        }
      }
#pragma unroll
      for (int h = 0; h < RT / 2; ++h) {
        sm[C::RED + (kq * RT + 2 * h) * LT_CH + row] = acc[h].x;
        sm[C::RED + (kq * RT + 2 * h + 1) * LT_CH + row] = acc[h].y;
      }
      __syncthreads();
      if (tid < RT * LT_CH) {
        const int r = tid / LT_CH, rw = tid & (LT_CH - 1);
        R o = 0;
#pragma unroll
        for (int q = 0; q < LT_KQ; ++q) o += sm[C::RED + (q * RT + r) * LT_CH + rw];
        const int j = row0 + rw;
        if (cur.grp == LT_A1) {
          if (j < Hd) sm[C::H1 + j * RT + r] = tanh(o + sm[C::B1 + j]);
        } else if (cur.grp == LT_A2) {
          if (j < Hd) sm[C::H2 + j * RT + r] = tanh(o + sm[C::B2 + j]);
        } else {
          // output layer + NLL gradient (dL/do of sum x~/y + log y)
          const bool ok = j < F && r < nr;
          R go = 0;
          if (ok) {
            const R rr = exp(o + sm[C::BS + buf * LT_CH + rw]);
            if (refresh) {
              a.r[((size_t)b * T + t0 + r) * F + j] = rr;
            } else {
              const R l0 = sm[C::US + buf * LT_CH + rw] * sm[C::VS + r] * rr;
              const R* xr = sm + C::XS + buf * LT_CH * RT * M + (rw * RT + r) * M;
              const R* ls = sm + C::LS + buf * (NMAX - 1) * LT_CH * RT + rw * RT + r;
              const R* gs = sm + C::GS + buf * NMAX * LT_CH * M + rw * M;
              R ln[NMAX];
#pragma unroll
              for (int n = 1; n < NMAX; ++n) {
                ln[n] = R(0);
                if (n >= N) break;
                ln[n] = ls[(n - 1) * LT_CH * RT];
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
                y = y > ::fm::RT<R>::tiny() ? y : ::fm::RT<R>::tiny();
                const R iy = rcp_r(y);
                s += g0 * (iy - xr[m] * iy * iy);
              }
              go = s * l0;
            }
          }
          sm[C::GO + rw * RT + r] = go;
        }
      }
      if (cur.grp != LT_O || refresh) continue;
      __syncthreads();
    }

    // backward chunk: acc[col][r] += sum_i coef[i][r] Wc[i][col] over this
    // thread's columns (one segment), frames (a pair) and chunk rows (a slice)
    const int ncol = cur.grp == LT_C1 ? D : Hd;
    const int nrow = min(LT_CH, (cur.grp == LT_O ? F : Hd) - row0);
    const R* coef = cur.grp == LT_O ? sm + C::GO : sm + (cur.grp == LT_C2 ? C::D2 : C::D1) + row0 * RT;
    if (cseg * VEC < ncol) {
      for (int i = ciq; i < nrow; i += C::NIQ) {
        R w[VEC];
        lds_vec<R, VEC>(Wc + i * LT_LDW + ((cseg ^ (i & 7)) * VEC), w);
        const R2 cf = *reinterpret_cast<const R2*>(coef + i * RT + crp * C::RP);
#pragma unroll
        for (int v = 0; v < VEC; ++v) {
          R2 t = R2{accC[v][0], accC[v][1]};
          t = fma2(R2{w[v], w[v]}, cf, t);
          accC[v][0] = t.x;
          accC[v][1] = t.y;
        }
      }
    }
    if (!cur.last(nc1, nc3)) continue;
    // group end: fixed-order sum over the chunk-row slices, then the epilogue
#pragma unroll
    for (int v = 0; v < VEC; ++v)
#pragma unroll
      for (int h = 0; h < C::RP; ++h) {
        sm[C::RED + (ciq * RT + crp * C::RP + h) * DEC_HMAX + cseg * VEC + v] = accC[v][h];
        accC[v][h] = 0;
      }
    __syncthreads();
    double c1 = 0, c2 = 0;
    if (cur.grp == LT_C1) {  // Adam step index iter * steps + s + 1
      const double tstep = (double)(*a.iter) * a.steps + cur.s + 1;
      c1 = 1.0 - pow((double)a.b1a, tstep);
      c2 = 1.0 - pow((double)a.b2a, tstep);
    }
    for (int e = tid; e < RT * DEC_HMAX; e += LT_NT) {
      const int r = e / DEC_HMAX, col = e % DEC_HMAX;
      if (col >= ncol) continue;
      R sum = 0;
#pragma unroll
      for (int q = 0; q < C::NIQ; ++q) sum += sm[C::RED + (q * RT + r) * DEC_HMAX + col];
      const int i = col * RT + r;
      if (cur.grp == LT_O) {  // d2 = (W3^T go) (1 - h2^2)
        const R hv = sm[C::H2 + i];
        sm[C::D2 + i] = sum * (R(1) - hv * hv);
      } else if (cur.grp == LT_C2) {  // d1 = (W2^T d2) (1 - h1^2)
        const R hv = sm[C::H1 + i];
        sm[C::D1 + i] = sum * (R(1) - hv * hv);
      } else if (r < nr) {  // gz = W1^T d1; Adam on z
        R* mp = sm + C::AM + r * DEC_DMAX + col;
        R* vp = sm + C::AV + r * DEC_DMAX + col;
        const R mi = R(a.b1a) * *mp + R(1 - a.b1a) * sum;
        const R vi = R(a.b2a) * *vp + R(1 - a.b2a) * sum * sum;
        *mp = mi;
        *vp = vi;
        sm[C::ZT + i] -= R(a.lr) * (mi / (R)c1) / (sqrt_r(vi / (R)c2) + R(a.eps));
      }
    }
  }
  cp_async_wait<0>();
  __syncthreads();
  if (a.steps == 0) return;
  for (int e = tid; e < D * nr; e += LT_NT) {
    const int r = e / D, d = e - r * D;
    const size_t i = ((size_t)b * T + t0 + r) * D + d;
    a.z[i] = sm[C::ZT + d * RT + r];
    a.m[i] = sm[C::AM + r * DEC_DMAX + d];
    a.v2[i] = sm[C::AV + r * DEC_DMAX + d];
  }
}

}  // namespace fm
