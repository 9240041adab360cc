// fm_fused.cuh -- the three statistics passes of the FastMNMF iteration with
// lambda = W H formed on chip and phi never written to HBM (SURVEY §8(a)
// A2-A7, A11, A13; _kernels.py:226-250, sources.py:184-198).
//
// All three share one tile shape: a warp owns one frequency bin and 32
// consecutive frames (lane <-> frame), a CTA owns FB bins (FB warps). The
// H columns of the CTA's frames are staged in shared memory as rows
// Hs[n][t][k] (k contiguous, row pitch KP = K4 + 4 so 16-B loads by 32
// consecutive frames are conflict-free) from Ht = H transposed (B, N, T, K4),
// a copy of H the passes keep in step with H; a lane forms
// lambda_n = W_f,n . H_n,t with 16-B loads from Hs and the warp-broadcast W
// row of its bin.
//
// Every global read of the frame loops is a cp.async issued S-1 chunks ahead
// into an S-deep ring (H columns, and each lane's x~ or X row), so the
// copies of later chunks stream while chunk c computes.
//
//   k_hpass  (H step, separate.py:214-216 with "H"): one 32-frame tile of H
//            per CTA, looping over its bin range; phi from lambda(W, H),
//            x~, g; num/den_H[n,k,t] = sum_f W phi accumulated per thread in
//            fixed bin order; bin splits reduced in split order by the last
//            CTA, which applies the MU (sources.py:198) to H and Ht, or
//            writes the sums for the cross-shard all-reduce.
//   k_gpass  (gain step, separate.py:217-220): (FB bins, frame segment) per
//            CTA; gain statistics sum_t lambda x~/y^2, sum_t lambda/y per
//            (n, f, m) as segment partials for the V kernel (which finishes
//            the g MU); lambda(W, H) of the updated H is also written once
//            for the V kernel.
//   k_bpass  (end of the iteration + the next one's first refresh,
//            separate.py:230, :186-193, :214-216 with "W"): projection
//            x~ = |Q x|^2 (written), the log-likelihood data term, phi from
//            the absorbed W, and num/den_W[n,f,k] = sum_t phi H; the last
//            CTA of each bin block reduces the segments in order and writes
//            Wn = W sqrt(num/den) -- the W of the coming iteration's H step.
//            The loop state W stays the post-absorb W the reference exposes.
//
// Template shape parameters: MP = channels padded to 4, 8 or 16 (runtime M
// guards; padded channels carry zero gains and are excluded from every
// sum); NN / KC = the source count and the padded basis count K4 when known
// at compile time (0 = runtime), so the benchmark shapes get fully unrolled
// source and basis loops and every other shape runs the generic build.
#pragma once
#include "fm_common.cuh"
#include "fm_nmf.cuh"

namespace fm {

constexpr int FTC = 32;  // frames per chunk = warp width

__host__ __device__ constexpr int k4_of(int K) { return (K + 3) & ~3; }
__host__ __device__ constexpr int kp_of(int K) { return k4_of(K) + 4; }
// smem row pitch (bytes) of a lane's staged row: 16-B aligned, an odd number
// of 16-B units so 16-B loads by 8 consecutive lanes hit distinct banks
__host__ __device__ constexpr int row_pitch(int bytes) {
  return (((bytes + 15) / 16) % 2 == 1) ? (bytes + 15) / 16 * 16 : (bytes + 15) / 16 * 16 + 16;
}
__host__ __device__ constexpr size_t al16(size_t b) { return (b + 15) & ~size_t(15); }

// ---- cp.async with zero fill (src-size 0 -> the destination is zeroed) ----
__device__ __forceinline__ void cpa4(void* s, const void* g, bool v) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(s);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(sa), "l"(g), "r"(v ? 4 : 0));
}
__device__ __forceinline__ void cpa8(void* s, const void* g, bool v) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(s);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(g), "r"(v ? 8 : 0));
}
__device__ __forceinline__ void cpa16(void* s, const void* g, bool v) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(s);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(g), "r"(v ? 16 : 0));
}
__device__ __forceinline__ void cp_async_wait_n(int n) {
  if (n >= 2) cp_async_wait<2>();
  else if (n == 1) cp_async_wait<1>();
  else cp_async_wait<0>();
}

// `bytes` bytes (a multiple of 4; both bases aligned to the largest
// power-of-two divisor of `bytes` up to 16), split into the widest pieces
__device__ __forceinline__ void row_async(unsigned char* dst, const unsigned char* src, int bytes,
                                          bool v, const unsigned char* safe) {
  const unsigned char* s = v ? src : safe;
  if ((bytes & 15) == 0) {
    for (int o = 0; o < bytes; o += 16) cpa16(dst + o, s + o, v);
  } else if ((bytes & 7) == 0) {
    for (int o = 0; o < bytes; o += 8) cpa8(dst + o, s + o, v);
  } else {
    for (int o = 0; o < bytes; o += 4) cpa4(dst + o, s + o, v);
  }
}

// Ht[b, n, t0 .. t0+31, 0 .. K4) -> Hs[(n * 32 + tl) * KP + k] in 16-B pieces
// (zero for t >= tend). Ht rows are K4 reals, zero beyond K.
template <typename R, int NN, int KC>
__device__ __forceinline__ void stage_h_async(R* __restrict__ Hs, const R* __restrict__ Htb, int Nrt,
                                              int K4rt, int T, int t0, int tend, int tid, int nthr) {
  const int N = NN ? NN : Nrt, K4 = KC ? KC : K4rt, KP = K4 + 4;
  constexpr int PE = 16 / (int)sizeof(R);  // reals per 16-B piece
  const int PR = K4 / PE;                  // pieces per row (K4 * rs is a multiple of 16)
  const int tot = N * FTC * PR;
  for (int e = tid; e < tot; e += nthr) {
    const int q = e % PR, r = e / PR, tl = r % FTC, n = r / FTC;
    const int t = t0 + tl;
    const bool v = t < tend;
    cpa16(Hs + (n * FTC + tl) * KP + q * PE, v ? Htb + ((size_t)n * T + t) * K4 + q * PE : Htb, v);
  }
}

// rows W[b, n, f0 + w, :] and g[b, n, f0 + w, :] of warp w's bin into
// Ws[(w * N + n) * KP + k] / gs[(w * N + n) * MP + m], zero outside the bin
// range and beyond K / M; lanes along the rows, 16-B pieces where aligned
template <typename R, int MP, int NN>
__device__ __forceinline__ void stage_wg_async(R* __restrict__ Ws, R* __restrict__ gs,
                                               const R* __restrict__ Wb, const R* __restrict__ gb,
                                               int Nrt, int F, int K, int M, int f0, int fend,
                                               int lane, int warp) {
  const int N = NN ? NN : Nrt;
  const int K4 = k4_of(K), KP = K4 + 4;
  const int f = f0 + warp;
  const bool fv = f < fend;
  constexpr int PE = 16 / (int)sizeof(R);
  if ((K * (int)sizeof(R)) % 16 == 0) {  // rows of whole 16-B pieces
    const int PR = K / PE;
    for (int e = lane; e < N * PR; e += 32) {
      const int n = e / PR, q = e % PR;
      cpa16(Ws + (warp * N + n) * KP + q * PE, fv ? Wb + ((size_t)n * F + f) * K + q * PE : Wb, fv);
    }
  } else {
    for (int e = lane; e < N * K4; e += 32) {
      const int n = e / K4, k = e % K4;
      const bool v = fv && k < K;
      if constexpr (sizeof(R) == 4) cpa4(Ws + (warp * N + n) * KP + k, v ? Wb + ((size_t)n * F + f) * K + k : Wb, v);
      else cpa8(Ws + (warp * N + n) * KP + k, v ? Wb + ((size_t)n * F + f) * K + k : Wb, v);
    }
  }
  if (M == MP && (M * (int)sizeof(R)) % 16 == 0) {
    constexpr int PR = MP / PE;
    for (int e = lane; e < N * PR; e += 32) {
      const int n = e / PR, q = e % PR;
      cpa16(gs + (warp * N + n) * MP + q * PE, fv ? gb + ((size_t)n * F + f) * M + q * PE : gb, fv);
    }
  } else {
    for (int e = lane; e < N * MP; e += 32) {
      const int n = e / MP, m = e % MP;
      const bool v = fv && m < M;
      if constexpr (sizeof(R) == 4) cpa4(gs + (warp * N + n) * MP + m, v ? gb + ((size_t)n * F + f) * M + m : gb, v);
      else cpa8(gs + (warp * N + n) * MP + m, v ? gb + ((size_t)n * F + f) * M + m : gb, v);
    }
  }
}

// lambda_n at one (bin, frame): W row (broadcast in the warp) . H row
template <typename R, int NN, int KC>
__device__ __forceinline__ void lam_point(const R* __restrict__ Wrow, const R* __restrict__ Hs, int tl,
                                          int Nrt, int K4rt, R (&l)[NMAX]) {
  const int N = NN ? NN : Nrt, K4 = KC ? KC : K4rt, KP = K4 + 4;
#pragma unroll
  for (int n = 0; n < NMAX; ++n) {
    l[n] = R(0);
    if (n >= N) break;
    const R* hr = Hs + (n * FTC + tl) * KP;
    const R* wr = Wrow + n * KP;
    R acc0 = 0, acc1 = 0;
    if constexpr (KC > 0) {
#pragma unroll
      for (int k = 0; k < KC; k += 4) {
        R h0[4], w0[4];
        lds4(hr + k, h0);
        lds4(wr + k, w0);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if ((k / 4) % 2 == 0) acc0 += w0[c] * h0[c];
          else acc1 += w0[c] * h0[c];
        }
      }
    } else {
      int k = 0;
      for (; k + 8 <= K4; k += 8) {
        R h0[4], w0[4], h1[4], w1[4];
        lds4(hr + k, h0);
        lds4(wr + k, w0);
        lds4(hr + k + 4, h1);
        lds4(wr + k + 4, w1);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          acc0 += w0[c] * h0[c];
          acc1 += w1[c] * h1[c];
        }
      }
      if (k < K4) {
        R h0[4], w0[4];
        lds4(hr + k, h0);
        lds4(wr + k, w0);
#pragma unroll
        for (int c = 0; c < 4; ++c) acc0 += w0[c] * h0[c];
      }
    }
    l[n] = acc0 + acc1;
  }
}

// y = max(sum_n lambda g, floor), iy = 1/y on the M live channels (0 on the
// padded ones and on invalid points)
template <typename R, int MP, int NN>
__device__ __forceinline__ void power_point(const R (&l)[NMAX], const R* __restrict__ gs, int Nrt, int M,
                                            R fl, bool valid, R (&y)[MP], R (&iy)[MP]) {
  const int N = NN ? NN : Nrt;
#pragma unroll
  for (int m = 0; m < MP; ++m) y[m] = 0;
#pragma unroll
  for (int n = 0; n < NMAX; ++n) {
    if (n >= N) break;
    R g[MP];
    RowIO<R, MP>::load(gs + n * MP, g);
#pragma unroll
    for (int m = 0; m < MP; ++m) y[m] += l[n] * g[m];
  }
#pragma unroll
  for (int m = 0; m < MP; ++m) {
    y[m] = floor_max(y[m], fl);
    iy[m] = (valid && m < M) ? rcp_r(y[m]) : R(0);
  }
}

// phi1_n = sum_m g x~ / y^2, phi2_n = sum_m g / y  (_kernels.py:236-243)
template <typename R, int MP>
__device__ __forceinline__ void phi_of(const R (&xr)[MP], const R (&iy)[MP], const R* __restrict__ gs,
                                       int n, R& p1, R& p2) {
  R g[MP];
  RowIO<R, MP>::load(gs + n * MP, g);
  p1 = 0;
  p2 = 0;
#pragma unroll
  for (int m = 0; m < MP; ++m) {
    p1 += g[m] * xr[m];
    p2 += g[m] * iy[m];
  }
}

// a lane's staged real row (M live values) into registers
template <typename R, int MP>
__device__ __forceinline__ void read_row(const R* __restrict__ p, int M, R (&v)[MP]) {
  if (M == MP) {
    RowIO<R, MP>::load(p, v);
  } else {
#pragma unroll
    for (int m = 0; m < MP; ++m) v[m] = m < M ? p[m] : R(0);
  }
}

// ---------------------------------------------------------------------------
// Ht maintenance: Ht[b, n, t, k] = H[b, n, k, t] (zero for K <= k < K4);
// mode 1 first applies the sharded H MU from the all-reduced sums
// hbuf (B, 2, N, K, T) (sources.py:198). grid over B * N * T * K4.
// ---------------------------------------------------------------------------
template <typename R>
__global__ void __launch_bounds__(256) k_hstore(R* __restrict__ H, R* __restrict__ Ht,
                                                const R* __restrict__ hbuf, int N, int K, int T,
                                                long long total, int mode) {
  pdl_entry();
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const int K4 = k4_of(K);
  const int k = (int)(i % K4);
  const long long r = i / K4;
  const int t = (int)(r % T);
  const long long bn = r / T;  // b * N + n
  R v = R(0);
  if (k < K) {
    const size_t hi = ((size_t)bn * K + k) * T + t;
    v = H[hi];
    if (mode == 1) {
      const size_t NKT = (size_t)N * K * T;
      const size_t b = (size_t)(bn / N), rel = hi - b * NKT;
      v *= mu_factor(hbuf[b * 2 * NKT + rel], hbuf[b * 2 * NKT + NKT + rel]);
      H[hi] = v;
    }
  }
  Ht[i] = v;
}

// ---------------------------------------------------------------------------
// lambda tile: lam_s[(n * FB + fl) * 32 + tl] = W[fl][n] . H[n][tl] for the
// CTA's FB bins x 32 frames. Warp w takes source n = w % N and bin group
// w / N (FB / N groups), so each H row a lane loads serves every bin of its
// group (the W rows are warp broadcasts).
// ---------------------------------------------------------------------------
template <typename R, int NN, int KC>
__device__ __forceinline__ void lam_tile(const R* __restrict__ Ws, const R* __restrict__ Hs,
                                         R* __restrict__ lam_s, int Nrt, int K4rt, int FB, int warp,
                                         int lane) {
  const int N = NN ? NN : Nrt, K4 = KC ? KC : K4rt, KP = K4 + 4;
  const int NBG = FB / N > 1 ? FB / N : 1;
  const int BPG = (FB + NBG - 1) / NBG;
  for (int as = warp; as < N * NBG; as += FB) {  // (source, bin group) assignments of this warp
    const int n = as % N, fb0 = (as / N) * BPG;
    const int nb = min(BPG, FB - fb0);
    R acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = R(0);
    const R* hr = Hs + (n * FTC + lane) * KP;
    const R* wr = Ws + (fb0 * N + n) * KP;
    auto quad = [&](int k) {
      R h[4];
      lds4(hr + k, h);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (j < nb) {
          R w[4];
          lds4(wr + j * N * KP + k, w);
#pragma unroll
          for (int c = 0; c < 4; ++c) acc[j] += w[c] * h[c];
        }
      }
    };
    if constexpr (KC > 0) {
#pragma unroll
      for (int k = 0; k < KC; k += 4) quad(k);
    } else {
      for (int k = 0; k < K4; k += 4) quad(k);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (j < nb) lam_s[(n * FB + fb0 + j) * FTC + lane] = acc[j];
  }
}

// ---------------------------------------------------------------------------
// k_hpass: H statistics + H MU. grid (ceil(T/32), B * NG, HS), block 32 * FB.
// Each CTA accumulates sources [ng * NS, ng * NS + NS) of its 32-frame tile:
// item j = tid + 256 i (i < IT) is (source nl, k-chunk ko of KCH = 8 or 4
// bases) at frame lane, so a warp's 32 lanes share one (nl, ko) and the W
// loads are broadcasts.
// ---------------------------------------------------------------------------
template <typename R> struct HpArgs {
  const R* xt;
  const R* W;   // Wn: W after this iteration's W step
  R* H;
  R* Ht;        // H transposed (B, N, T, K4), kept in step
  const R* g;
  const R* floorp;
  R* part;      // (tiles * B * NG, HS, 2, NS * K4, 32) split partials
  unsigned* cnt;
  R* hout;      // mode 1: (B, 2, N, K, T) sums
  int F, T, N, K, M;
  int mode;     // 0 apply the MU, 1 write the sums
  int HFR;      // bins per split (multiple of FB)
  int NS, NG;   // sources accumulated per CTA, source groups
  int S;        // cp.async pipeline stages (2..4)
};

__host__ __device__ constexpr int hp_kch(int K4) { return K4 % 8 == 0 ? 8 : 4; }

// shared-memory layout (bytes): Hs | S x (Ws | gs) | S x per-warp x~ rows |
// lambda tile | phi
struct HpLayout {
  size_t o_ws0, wg_stride, gs_off, o_rows0, rows_stride, o_lam, o_ph, total;
  int rowp;
  __host__ __device__ HpLayout(int rs, int N, int K, int M, int MP, int FB, int NS, int S) {
    o_ws0 = al16((size_t)rs * N * FTC * kp_of(K));
    gs_off = al16((size_t)rs * FB * N * kp_of(K));
    wg_stride = gs_off + al16((size_t)rs * FB * N * MP);
    rowp = row_pitch(rs * M);
    o_rows0 = o_ws0 + S * wg_stride;
    rows_stride = al16((size_t)FB * FTC * rowp);
    o_lam = o_rows0 + S * rows_stride;
    o_ph = o_lam + al16((size_t)rs * N * FB * FTC);
    total = o_ph + al16((size_t)rs * FB * 2 * NS * FTC);
  }
  __host__ __device__ size_t ws(int buf) const { return o_ws0 + buf * wg_stride; }
  __host__ __device__ size_t gs(int buf) const { return o_ws0 + buf * wg_stride + gs_off; }
  __host__ __device__ size_t rows(int buf) const { return o_rows0 + buf * rows_stride; }
};

template <typename R, int MP, int IT, int NN, int KC>
__global__ void __launch_bounds__(256) k_hpass(HpArgs<R> a) {
  pdl_entry();
  extern __shared__ __align__(16) unsigned char smraw[];
  const int FB = blockDim.x / FTC;
  const int N = NN ? NN : a.N, K = a.K, M = a.M, F = a.F, T = a.T, NS = a.NS;
  const int K4 = KC ? KC : k4_of(K), KP = K4 + 4;
  const int KCH = hp_kch(K4), KO = K4 / KCH;
  const int S = a.S;
  const HpLayout L((int)sizeof(R), N, K, M, MP, FB, NS, S);
  R* Hs = reinterpret_cast<R*>(smraw);
  R* lam_s = reinterpret_cast<R*>(smraw + L.o_lam);  // [N][FB][32]
  R* ph = reinterpret_cast<R*>(smraw + L.o_ph);      // [fl][2][NS][32]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int t0 = blockIdx.x * FTC;
  const int b = blockIdx.y / a.NG, ng = blockIdx.y % a.NG;
  const int nb = ng * NS, ns = min(NS, N - nb);
  const int fbeg = blockIdx.z * a.HFR, fend = min(F, fbeg + a.HFR);
  const R* Wb = a.W + (size_t)b * N * F * K;
  const R* gb = a.g + (size_t)b * N * F * M;
  const R* xtb = a.xt + (size_t)b * F * T * M;
  const int t = t0 + lane;
  const int rb = M * (int)sizeof(R);
  auto issue = [&](int f0, int buf) {
    stage_wg_async<R, MP, NN>(reinterpret_cast<R*>(smraw + L.ws(buf)), reinterpret_cast<R*>(smraw + L.gs(buf)),
                              Wb, gb, N, F, K, M, f0, fend, lane, warp);
    const int f = f0 + warp;
    const bool v = f < fend && t < T;
    row_async(smraw + L.rows(buf) + (size_t)(warp * FTC + lane) * L.rowp,
              reinterpret_cast<const unsigned char*>(xtb + ((size_t)(v ? f : 0) * T + (v ? t : 0)) * M),
              rb, v, reinterpret_cast<const unsigned char*>(xtb));
  };
  stage_h_async<R, NN, KC>(Hs, a.Ht + (size_t)b * N * T * K4, N, K4, T, t0, T, tid, blockDim.x);
  for (int st = 0; st < S - 1; ++st) {  // pipeline prologue: steps 0 .. S-2
    if (fbeg + st * FB < fend) issue(fbeg + st * FB, st);
    cp_async_commit();
  }
  const R fl = a.floorp[b];
  R a1[IT][8], a2[IT][8];
#pragma unroll
  for (int i = 0; i < IT; ++i)
#pragma unroll
    for (int c = 0; c < 8; ++c) a1[i][c] = a2[i][c] = R(0);
  // this thread's items (hoisted): W row offset (-1: none) and phi offset
  int iw[IT], ip1[IT];
#pragma unroll
  for (int i = 0; i < IT; ++i) {
    const int r = warp + FB * i;  // (nl, ko) index; lane = frame
    iw[i] = -1;
    ip1[i] = 0;
    if (r < ns * KO) {
      const int nl = r / KO, ko = r % KO;
      iw[i] = (nb + nl) * KP + ko * KCH;
      ip1[i] = nl * FTC + lane;
    }
  }
  int buf = 0;
  for (int f0 = fbeg; f0 < fend; f0 += FB, buf = (buf + 1 == S) ? 0 : buf + 1) {
    cp_async_wait_n(S - 2);
    __syncthreads();  // step data landed; every thread is done with the previous step
    if (f0 + (S - 1) * FB < fend) issue(f0 + (S - 1) * FB, buf == 0 ? S - 1 : buf - 1);
    cp_async_commit();
    const R* Ws = reinterpret_cast<const R*>(smraw + L.ws(buf));
    const R* gs = reinterpret_cast<const R*>(smraw + L.gs(buf));
    lam_tile<R, NN, KC>(Ws, Hs, lam_s, N, K4, FB, warp, lane);
    __syncthreads();
    {  // phi at (bin f0 + warp, frame t)
      const int f = f0 + warp;
      const bool v = f < fend && t < T;
      R l[NMAX];
#pragma unroll
      for (int n = 0; n < NMAX; ++n) l[n] = n < N ? lam_s[(n * FB + warp) * FTC + lane] : R(0);
      R xv[MP];
      read_row<R, MP>(reinterpret_cast<const R*>(smraw + L.rows(buf) + (size_t)(warp * FTC + lane) * L.rowp),
                      M, xv);
      R y[MP], iy[MP], xr[MP];
      const R* gw = gs + warp * N * MP;
      power_point<R, MP, NN>(l, gw, N, M, fl, v, y, iy);
#pragma unroll
      for (int m = 0; m < MP; ++m) xr[m] = xv[m] * iy[m] * iy[m];
      R* pw = ph + warp * 2 * NS * FTC;
#pragma unroll
      for (int nl = 0; nl < NMAX; ++nl) {
        if (nl >= ns) break;
        R p1, p2;
        phi_of<R, MP>(xr, iy, gw, nb + nl, p1, p2);
        pw[nl * FTC + lane] = p1;
        pw[(NS + nl) * FTC + lane] = p2;
      }
    }
    __syncthreads();
    for (int fl2 = 0; fl2 < FB; ++fl2) {  // fixed bin order
      const R* pw = ph + fl2 * 2 * NS * FTC;
      const R* wr = Ws + fl2 * N * KP;
#pragma unroll
      for (int i = 0; i < IT; ++i) {
        if (iw[i] >= 0) {
          const R p1 = pw[ip1[i]], p2 = pw[NS * FTC + ip1[i]];
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            if (q * 4 < KCH) {
              R w4[4];
              lds4(wr + iw[i] + q * 4, w4);
#pragma unroll
              for (int c = 0; c < 4; ++c) {
                a1[i][q * 4 + c] += w4[c] * p1;
                a2[i][q * 4 + c] += w4[c] * p2;
              }
            }
          }
        }
      }
    }
  }
  cp_async_wait<0>();
  const int HS = gridDim.z;
  const size_t tileid = ((size_t)blockIdx.x * gridDim.y + blockIdx.y);
  const size_t PSZ = (size_t)2 * NS * K4 * FTC;  // one split's partial
  R* pt = a.part + tileid * HS * PSZ;
  auto pidx = [&](int i, int c) {  // partial index of (item i, basis c of its chunk)
    const int r = warp + FB * i, nl = r / KO, ko = r % KO;
    return (size_t)(nl * K4 + ko * KCH + c) * FTC + lane;
  };
  if (HS > 1) {
#pragma unroll
    for (int i = 0; i < IT; ++i) {
      if (iw[i] >= 0) {
        for (int c = 0; c < KCH; ++c) {
          pt[(size_t)blockIdx.z * PSZ + pidx(i, c)] = a1[i][c];
          pt[(size_t)blockIdx.z * PSZ + (size_t)NS * K4 * FTC + pidx(i, c)] = a2[i][c];
        }
      }
    }
    __threadfence();
    __syncthreads();
    __shared__ unsigned last;
    if (tid == 0) last = atomicAdd(a.cnt + tileid, 1u) == (unsigned)HS - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    if (tid == 0) a.cnt[tileid] = 0;  // re-armed for the next launch
#pragma unroll
    for (int i = 0; i < IT; ++i) {
      if (iw[i] >= 0) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          if (c < KCH) {
            R sn = 0, sd = 0;
            for (int z = 0; z < HS; ++z) {  // split order
              sn += __ldcg(pt + (size_t)z * PSZ + pidx(i, c));
              sd += __ldcg(pt + (size_t)z * PSZ + (size_t)NS * K4 * FTC + pidx(i, c));
            }
            a1[i][c] = sn;
            a2[i][c] = sd;
          }
        }
      }
    }
  }
  if (t >= T) return;
#pragma unroll
  for (int i = 0; i < IT; ++i) {
    if (iw[i] < 0) continue;
    const int r = warp + FB * i, n = nb + r / KO, k0 = (r % KO) * KCH;
    if (a.mode == 0) {
      R hv[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        hv[c] = R(0);
        const int k = k0 + c;
        if (c < KCH && k < K) {
          const size_t hi = (((size_t)b * N + n) * K + k) * T + t;
          hv[c] = a.H[hi] * mu_factor(a1[i][c], a2[i][c]);  // sources.py:198
          a.H[hi] = hv[c];
        }
      }
      R* ht = a.Ht + (((size_t)b * N + n) * T + t) * K4 + k0;
#pragma unroll
      for (int c = 0; c < 8; ++c)
        if (c < KCH) ht[c] = hv[c];
    } else {
      const size_t NKT = (size_t)N * K * T;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int k = k0 + c;
        if (c < KCH && k < K) {
          const size_t hi = ((size_t)n * K + k) * T + t;
          a.hout[(size_t)b * 2 * NKT + hi] = a1[i][c];
          a.hout[(size_t)b * 2 * NKT + NKT + hi] = a2[i][c];
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Per-warp reduction layout of k_gpass: NI items (one per lane when NI <= 32,
// S = 32 / NI frame slices; else IT items per lane, S = 1).
// ---------------------------------------------------------------------------
struct WarpItems {
  int NI, S, item, slice;
  __device__ WarpItems(int ni, int lane) : NI(ni) {
    if (ni <= 32) {
      S = 32 / ni;
      item = lane % ni;
      slice = lane / ni;
      if (slice >= S) slice = -1;  // idle lane
    } else {
      S = 1;
      item = lane;
      slice = 0;
    }
  }
};

// ---------------------------------------------------------------------------
// k_gpass: gain statistics (+ lambda for the V kernel).
// grid (nseg, ceil(F/FB), B), block 32 * FB.
// ---------------------------------------------------------------------------
template <typename R> struct GpArgs {
  const R* xt;
  const R* W;   // Wn
  const R* Ht;  // H transposed, after this iteration's H MU
  const R* g;   // gains before the MU
  const R* floorp;
  R* lam;       // (B, N, F, T) out
  R* part;      // (B, F, nseg, N, 2M) segment partials (k_vacc finishes the MU)
  int F, T, N, K, M, TR;  // TR: frames per segment (multiple of 32)
  int S;                  // cp.async pipeline stages (2..4)
};

// shared-memory layout (bytes): S x Hs | Ws | gs | S x per-warp x~ rows |
// lambda tile | per warp: iy [32][MP + 4], xr [32][MP + 4], red [32][8]
struct GpLayout {
  size_t hs_stride, o_ws, o_gs, o_rows0, rows_stride, o_lam, o_warp, warp_bytes, total;
  int rowp;
  __host__ __device__ GpLayout(int rs, int N, int K, int M, int MP, int FB, int S) {
    hs_stride = al16((size_t)rs * N * FTC * kp_of(K));
    o_ws = S * hs_stride;
    o_gs = o_ws + al16((size_t)rs * FB * N * kp_of(K));
    o_rows0 = o_gs + al16((size_t)rs * FB * N * MP);
    rowp = row_pitch(rs * M);
    rows_stride = al16((size_t)FB * FTC * rowp);
    o_lam = o_rows0 + S * rows_stride;
    warp_bytes = al16((size_t)rs * (2 * FTC * (MP + 4) + 32 * 8));
    o_warp = o_lam + al16((size_t)rs * N * FB * FTC);
    total = o_warp + (size_t)FB * warp_bytes;
  }
  __host__ __device__ size_t hs(int buf) const { return buf * hs_stride; }
  __host__ __device__ size_t rows(int buf) const { return o_rows0 + buf * rows_stride; }
};

template <typename R, int MP, int NN, int KC>
__global__ void __launch_bounds__(256) k_gpass(GpArgs<R> a) {
  pdl_entry();
  extern __shared__ __align__(16) unsigned char smraw[];
  const int FB = blockDim.x / FTC;
  const int N = NN ? NN : a.N, K = a.K, M = a.M, F = a.F, T = a.T;
  const int K4 = KC ? KC : k4_of(K);
  constexpr int MQ = MP / 4, LDR = MP + 4;
  const int S = a.S;
  const GpLayout L((int)sizeof(R), N, K, M, MP, FB, S);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  R* Ws = reinterpret_cast<R*>(smraw + L.o_ws);
  R* gs = reinterpret_cast<R*>(smraw + L.o_gs);
  R* lam_s = reinterpret_cast<R*>(smraw + L.o_lam);  // [N][FB][32]
  R* iyw = reinterpret_cast<R*>(smraw + L.o_warp + (size_t)warp * L.warp_bytes);  // [32][LDR]
  R* xrw = iyw + FTC * LDR;      // [32][LDR]
  R* red = xrw + FTC * LDR;      // [32][8]
  const int seg = blockIdx.x, nseg = gridDim.x, b = blockIdx.z;
  const int f0 = blockIdx.y * FB, f = f0 + warp;
  const bool fv = f < F;
  const int ta = seg * a.TR, tb = min(T, ta + a.TR);
  const R* Htb = a.Ht + (size_t)b * N * T * K4;
  const R* xtb = a.xt + (size_t)b * F * T * M;
  const int rb = M * (int)sizeof(R);
  auto issue = [&](int t0, int buf) {
    stage_h_async<R, NN, KC>(reinterpret_cast<R*>(smraw + L.hs(buf)), Htb, N, K4, T, t0, tb, tid, blockDim.x);
    const int t = t0 + lane;
    const bool v = fv && t < tb;
    row_async(smraw + L.rows(buf) + (size_t)(warp * FTC + lane) * L.rowp,
              reinterpret_cast<const unsigned char*>(xtb + ((size_t)(v ? f : 0) * T + (v ? t : 0)) * M),
              rb, v, reinterpret_cast<const unsigned char*>(xtb));
  };
  stage_wg_async<R, MP, NN>(Ws, gs, a.W + (size_t)b * N * F * K, a.g + (size_t)b * N * F * M, N, F, K, M,
                            f0, F, lane, warp);
  for (int st = 0; st < S - 1; ++st) {  // pipeline prologue: chunks 0 .. S-2
    if (ta + st * FTC < tb) issue(ta + st * FTC, st);
    cp_async_commit();
  }
  const R fl = a.floorp[b];
  const WarpItems wi(N * MQ, lane);
  const int n1 = wi.item / MQ, mq = wi.item % MQ;
  R num[4] = {0, 0, 0, 0}, den[4] = {0, 0, 0, 0};
  const R* gw = gs + warp * N * MP;
  const R* lw = lam_s + warp * FTC;  // + n FB 32 + t
  const size_t FTs = (size_t)F * T;
  R* lamp = a.lam + (size_t)b * N * FTs + (size_t)(fv ? f : 0) * T + lane;  // + n FT + t0
  int buf = 0;
  for (int t0 = ta; t0 < tb; t0 += FTC, buf = (buf + 1 == S) ? 0 : buf + 1) {
    cp_async_wait_n(S - 2);
    __syncthreads();  // chunk landed; every thread is done with the chunk before
    if (t0 + (S - 1) * FTC < tb) issue(t0 + (S - 1) * FTC, buf == 0 ? S - 1 : buf - 1);
    cp_async_commit();
    const R* Hs = reinterpret_cast<const R*>(smraw + L.hs(buf));
    lam_tile<R, NN, KC>(Ws, Hs, lam_s, N, K4, FB, warp, lane);
    __syncthreads();
    const bool v = fv && t0 + lane < tb;
    R l[NMAX];
#pragma unroll
    for (int n = 0; n < NMAX; ++n) l[n] = n < N ? lw[n * FB * FTC + lane] : R(0);
    R xv[MP];
    read_row<R, MP>(reinterpret_cast<const R*>(smraw + L.rows(buf) + (size_t)(warp * FTC + lane) * L.rowp),
                    M, xv);
    R y[MP], iy[MP];
    power_point<R, MP, NN>(l, gw, N, M, fl, v, y, iy);
    if (v) {
#pragma unroll
      for (int n = 0; n < NMAX; ++n)
        if (n < N) lamp[(size_t)n * FTs + t0] = l[n];
    }
    R xr[MP];
#pragma unroll
    for (int m = 0; m < MP; ++m) xr[m] = xv[m] * iy[m] * iy[m];
    RowIO<R, MP>::store(iyw + lane * LDR, iy);  // iy = 0 on invalid frames
    RowIO<R, MP>::store(xrw + lane * LDR, xr);
    __syncwarp();
    if (wi.slice >= 0) {
      for (int tl = wi.slice; tl < FTC; tl += wi.S) {
        const R lv = lw[n1 * FB * FTC + tl];
        R xq[4], iq[4];
        lds4(xrw + tl * LDR + mq * 4, xq);
        lds4(iyw + tl * LDR + mq * 4, iq);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          num[c] += lv * xq[c];
          den[c] += lv * iq[c];
        }
      }
    }
  }
  cp_async_wait<0>();
  // slice sums in fixed order, then the segment partial of (n, f, m)
  if (wi.slice >= 0) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      red[lane * 8 + c] = num[c];
      red[lane * 8 + 4 + c] = den[c];
    }
  }
  __syncwarp();
  if (fv && lane < wi.NI) {
    R sn[4] = {0, 0, 0, 0}, sd[4] = {0, 0, 0, 0};
    for (int s = 0; s < wi.S; ++s) {
      const R* r = red + (s * wi.NI + lane) * 8;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        sn[c] += r[c];
        sd[c] += r[4 + c];
      }
    }
    R* pb = a.part + (((size_t)b * F + f) * nseg + seg) * N * 2 * M + n1 * 2 * M;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int m = mq * 4 + c;
      if (m < M) {
        pb[m] = sn[c];
        pb[M + m] = sd[c];
      }
    }
  }
}

// ---------------------------------------------------------------------------
// k_bpass: projection + data term + W statistics -> Wn.
// grid (nseg, ceil(F/FB), B), block 32 * FB.
// W statistics: CTA item j = (source n, bin pair fp, k-quad kq), NI =
// N (FB/2) KQ; threads tid = s NI + j take frames t = s, s + BS, ... of every
// chunk (BS = 256 / NI frame slices, or IT items per thread when NI > 256);
// one 16-B H load feeds two bins' numerators and denominators.
// ---------------------------------------------------------------------------
template <typename R> struct BpArgs {
  const cplx<R>* X;
  R* xt;
  const cplx<R>* Q;
  const R* g;     // gains after the normalisation
  const R* W;     // W after the absorb (the loop state)
  const R* Ht;    // H transposed
  const R* floorp;
  R* Wn;          // W of the next iteration's H step
  R* part;        // (B, F, nseg, 2, N, K4) W-statistic segment partials
  unsigned* cnt;  // (B, nfb) completion counters
  double* llp;    // (B, nfb, nseg) data-term partials
  int F, T, N, K, M, TR;
  int S;          // cp.async pipeline stages (2..4)
  int dbg;        // timing experiments only: bit 0 skip W statistics, 1 lambda, 2 projection, 3 phi
};

// shared-memory layout (bytes): S x Hs | Ws | gs | Qs | S x per-warp X rows |
// lambda tile | phi [FB][2][N][32] (the W-statistic slice reduction reuses
// the Hs ring after the frame loop)
struct BpLayout {
  size_t hs_stride, o_ws, o_gs, o_q, o_rows0, rows_stride, o_lam, o_ph, total;
  int rowp;
  __host__ __device__ BpLayout(int rs, int N, int K, int M, int MP, int FB, int S) {
    hs_stride = al16((size_t)rs * N * FTC * kp_of(K));
    const int NI = N * ((FB + 1) / 2) * (k4_of(K) / 4);  // W-statistic items
    size_t ring = S * hs_stride, red = (size_t)rs * (NI > 32 * FB ? NI : 32 * FB) * 16;
    o_ws = al16(ring > red ? ring : red);
    o_gs = o_ws + al16((size_t)rs * FB * N * kp_of(K));
    o_q = o_gs + al16((size_t)rs * FB * N * MP);
    o_rows0 = o_q + al16((size_t)2 * rs * FB * M * M);
    rowp = row_pitch(2 * rs * M);
    rows_stride = al16((size_t)FB * FTC * rowp);
    o_lam = o_rows0 + S * rows_stride;
    o_ph = o_lam + al16((size_t)rs * N * FB * FTC);
    total = o_ph + al16((size_t)rs * FB * 2 * N * FTC);
  }
  __host__ __device__ size_t hs(int buf) const { return buf * hs_stride; }
  __host__ __device__ size_t rows(int buf) const { return o_rows0 + buf * rows_stride; }
};

template <typename R, int MP, int IT, int NN, int KC>
__global__ void __launch_bounds__(256) k_bpass(BpArgs<R> a) {
  pdl_entry();
  using C = cplx<R>;
  extern __shared__ __align__(16) unsigned char smraw[];
  const int FB = blockDim.x / FTC, BSZ = blockDim.x;
  const int N = NN ? NN : a.N, K = a.K, M = a.M, F = a.F, T = a.T;
  const int K4 = KC ? KC : k4_of(K), KP = K4 + 4, KQ = K4 / 4;
  const int S = a.S;
  const BpLayout L((int)sizeof(R), N, K, M, MP, FB, S);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  R* Ws = reinterpret_cast<R*>(smraw + L.o_ws);
  R* gs = reinterpret_cast<R*>(smraw + L.o_gs);
  C* Qs = reinterpret_cast<C*>(smraw + L.o_q);
  R* lam_s = reinterpret_cast<R*>(smraw + L.o_lam);  // [N][FB][32]
  R* ph = reinterpret_cast<R*>(smraw + L.o_ph);      // [FB][2][N][32]
  __shared__ double dred[8];
  __shared__ unsigned last;
  const int seg = blockIdx.x, nseg = gridDim.x, b = blockIdx.z, fblk = blockIdx.y;
  const int f0 = fblk * FB, f = f0 + warp;
  const bool fv = f < F;
  const int ta = seg * a.TR, tb = min(T, ta + a.TR);
  const R* Htb = a.Ht + (size_t)b * N * T * K4;
  const R* Wb = a.W + (size_t)b * N * F * K;
  const C* Xb = a.X + (size_t)b * F * T * M;
  R* xtp = a.xt + ((size_t)b * F + (fv ? f : 0)) * T * M + (size_t)lane * M;  // + t0 M
  const int rb = M * (int)sizeof(C);
  auto issue = [&](int t0, int buf) {
    stage_h_async<R, NN, KC>(reinterpret_cast<R*>(smraw + L.hs(buf)), Htb, N, K4, T, t0, tb, tid, BSZ);
    const int t = t0 + lane;
    const bool v = fv && t < tb;
    row_async(smraw + L.rows(buf) + (size_t)(warp * FTC + lane) * L.rowp,
              reinterpret_cast<const unsigned char*>(Xb + ((size_t)(v ? f : 0) * T + (v ? t : 0)) * M),
              rb, v, reinterpret_cast<const unsigned char*>(Xb));
  };
  stage_wg_async<R, MP, NN>(Ws, gs, Wb, a.g + (size_t)b * N * F * M, N, F, K, M, f0, F, lane, warp);
  for (int e = tid; e < FB * M * M; e += BSZ) {
    const int fl = e / (M * M), ff = f0 + fl;
    Qs[e] = ff < F ? a.Q[((size_t)b * F + ff) * M * M + e % (M * M)] : cmake<C>(0.0, 0.0);
  }
  for (int st = 0; st < S - 1; ++st) {  // pipeline prologue: chunks 0 .. S-2
    if (ta + st * FTC < tb) issue(ta + st * FTC, st);
    cp_async_commit();
  }
  const R fl = a.floorp[b];
  // W-statistic items of this thread
  const int FP = (FB + 1) / 2, NI = N * FP * KQ;
  const int SL = NI <= BSZ ? BSZ / NI : 1;
  const int slice = NI <= BSZ ? tid / NI : 0;
  int jn[IT], jf[IT], jk[IT];  // source, first bin, k offset (jn = -1: none)
#pragma unroll
  for (int i = 0; i < IT; ++i) {
    const int j = NI <= BSZ ? (i == 0 ? tid % NI : NI) : tid + BSZ * i;
    const bool has = j < NI && slice < SL;
    jn[i] = has ? j / (FP * KQ) : -1;
    jf[i] = has ? 2 * ((j / KQ) % FP) : 0;
    jk[i] = has ? (j % KQ) * 4 : 0;
  }
  R acc[IT][16];  // [bin 0/1][num/den][4 k]
#pragma unroll
  for (int i = 0; i < IT; ++i)
#pragma unroll
    for (int c = 0; c < 16; ++c) acc[i][c] = R(0);
  double ll = 0.0;
  const R* gw = gs + warp * N * MP;
  const C* Qw = Qs + warp * M * M;
  int buf = 0;
  for (int t0 = ta; t0 < tb; t0 += FTC, buf = (buf + 1 == S) ? 0 : buf + 1) {
    cp_async_wait_n(S - 2);
    __syncthreads();
    if (t0 + (S - 1) * FTC < tb) issue(t0 + (S - 1) * FTC, buf == 0 ? S - 1 : buf - 1);
    cp_async_commit();
    const R* Hs = reinterpret_cast<const R*>(smraw + L.hs(buf));
    if (!(a.dbg & 2)) lam_tile<R, NN, KC>(Ws, Hs, lam_s, N, K4, FB, warp, lane);
    const bool v = fv && t0 + lane < tb;
    // projection x~_i = |q_i^H x|^2 (row i of Q = q_i^H; _kernels.py:339-350)
    C xv[MP];
    {
      const C* xs = reinterpret_cast<const C*>(smraw + L.rows(buf) + (size_t)(warp * FTC + lane) * L.rowp);
      if (M == MP) {
        CRowIO<R, MP>::load(xs, xv);
      } else {
#pragma unroll
        for (int m = 0; m < MP; ++m) xv[m] = m < M ? xs[m] : cmake<C>(0.0, 0.0);
      }
    }
    R xtv[MP];
#pragma unroll
    for (int i = 0; i < MP; ++i) {
      xtv[i] = R(0);
      if (a.dbg & 4) { xtv[i] = xv[i].x; continue; }
      if (i < M) {
        C s = cmake<C>(0.0, 0.0);
#pragma unroll
        for (int j = 0; j < MP; ++j) {
          if (j < M) {
            const C q = Qw[i * M + j];
            s = fma2(cmake<C>(q.x, q.x), xv[j], s);
            s = fma2(cmake<C>(-q.y, q.y), cmake<C>(xv[j].y, xv[j].x), s);
          }
        }
        xtv[i] = s.x * s.x + s.y * s.y;
      }
    }
    if (v) {
      R* xo = xtp + (size_t)t0 * M;
      if (M == MP) {
        RowIO<R, MP>::store(xo, xtv);
      } else {
#pragma unroll
        for (int m = 0; m < MP; ++m)
          if (m < M) xo[m] = xtv[m];
      }
    }
    __syncthreads();  // lambda tile complete
    R l[NMAX];
#pragma unroll
    for (int n = 0; n < NMAX; ++n) l[n] = n < N ? lam_s[(n * FB + warp) * FTC + lane] : R(0);
    R y[MP], iy[MP];
    power_point<R, MP, NN>(l, gw, N, M, fl, v, y, iy);
    if (v) {
      R llt = 0;
#pragma unroll
      for (int m = 0; m < MP; ++m)
        if (m < M) llt += -xtv[m] * iy[m] - log_fast(y[m]);
      ll += (double)llt;
    }
    R xr[MP];
#pragma unroll
    for (int m = 0; m < MP; ++m) xr[m] = xtv[m] * iy[m] * iy[m];
    R* pw = ph + warp * 2 * N * FTC;
#pragma unroll
    for (int n = 0; n < NMAX; ++n) {
      if (n >= N || (a.dbg & 8)) break;
      R p1, p2;
      phi_of<R, MP>(xr, iy, gw, n, p1, p2);  // 0 on invalid frames (iy = 0)
      pw[n * FTC + lane] = p1;
      pw[(N + n) * FTC + lane] = p2;
    }
    __syncthreads();  // phi of every bin
#pragma unroll
    for (int i = 0; i < IT; ++i) {
      if (jn[i] < 0 || (a.dbg & 1)) continue;
      const int n = jn[i];
      const R* h0 = Hs + n * FTC * KP + jk[i];
      const R* pa = ph + jf[i] * 2 * N * FTC + n * FTC;  // bin jf: phi1 at +0, phi2 at + N 32
      const R* pb = pa + 2 * N * FTC;                    // bin jf + 1
      for (int tl = slice; tl < FTC; tl += SL) {
        R h4[4];
        lds4(h0 + tl * KP, h4);
        const R a1 = pa[tl], a2 = pa[N * FTC + tl], b1 = pb[tl], b2 = pb[N * FTC + tl];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          acc[i][c] += a1 * h4[c];
          acc[i][4 + c] += a2 * h4[c];
          acc[i][8 + c] += b1 * h4[c];
          acc[i][12 + c] += b2 * h4[c];
        }
      }
    }
  }
  cp_async_wait<0>();
  // data-term partial of this CTA (fixed order: lanes, then warps)
  ll = warp_sum(ll);
  if (lane == 0) dred[warp] = ll;
  __syncthreads();  // also: every thread is past its last read of the Hs ring
  const int nfb = gridDim.y;
  if (tid == 0) {
    double s = 0.0;
    for (int w = 0; w < FB; ++w) s += dred[w];
    a.llp[((size_t)b * nfb + fblk) * nseg + seg] = s;
  }
  // W statistics: slice partials (in the Hs ring) summed in slice order ->
  // this segment's partial (bin, 2, N, K4)
  R* red = reinterpret_cast<R*>(smraw);  // [slice][item][16] or [thread][IT][16]
#pragma unroll
  for (int i = 0; i < IT; ++i) {
    if (jn[i] < 0) continue;
    const int j = NI <= BSZ ? tid % NI : tid + BSZ * i;
    const int row = NI <= BSZ ? slice * NI + j : j;
#pragma unroll
    for (int c = 0; c < 16; ++c) red[(size_t)row * 16 + c] = acc[i][c];
  }
  __syncthreads();
  const size_t PW = (size_t)2 * N * K4;  // one (bin, segment) partial
  for (int e = tid; e < NI * 16; e += BSZ) {
    const int j = e / 16, c = e % 16;
    R sum = 0;
    const int nsl = NI <= BSZ ? SL : 1;
    for (int s = 0; s < nsl; ++s) sum += red[(size_t)(s * NI + j) * 16 + c];
    const int n = j / (FP * KQ), fb = 2 * ((j / KQ) % FP) + c / 8, k = (j % KQ) * 4 + c % 4;
    const int nd = (c / 4) % 2;
    const int ff = f0 + fb;
    if (fb < FB && ff < F)
      a.part[(((size_t)b * F + ff) * nseg + seg) * PW + (size_t)nd * N * K4 + n * K4 + k] = sum;
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) last = atomicAdd(a.cnt + (size_t)b * nfb + fblk, 1u) == (unsigned)nseg - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (tid == 0) a.cnt[(size_t)b * nfb + fblk] = 0;  // re-armed
  // W MU for the FB bins of this block (sources.py:191-194), segments in order
  R* Wnb = a.Wn + (size_t)b * N * F * K;
  for (int e = tid; e < FB * N * K; e += BSZ) {
    const int k = e % K, r = e / K, n = r % N, fl2 = r / N, ff = f0 + fl2;
    if (ff >= F) continue;
    const R* pb = a.part + ((size_t)b * F + ff) * nseg * PW;
    R sn = 0, sd = 0;
    for (int s = 0; s < nseg; ++s) {
      sn += __ldcg(pb + (size_t)s * PW + n * K4 + k);
      sd += __ldcg(pb + (size_t)s * PW + (size_t)N * K4 + n * K4 + k);
    }
    Wnb[((size_t)n * F + ff) * K + k] = Ws[(fl2 * N + n) * KP + k] * mu_factor(sn, sd);
  }
}

}  // namespace fm
