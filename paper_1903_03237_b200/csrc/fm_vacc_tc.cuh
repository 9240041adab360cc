// fm_vacc_tc.cuh -- the V_fm accumulation on the 5th-generation tensor cores
// (complex64 path, _kernels.py:276-293, spatial.py:182).
//
// V_fm[i,k] = sum_t iy[t,m] x_i(t) conj(x_k(t)) is, per bin f, one small GEMM
//   D[j][m] = sum_t A[j][t] B[m][t]
// with A[j][t] the M*M real components of the Hermitian outer product
// x(t) x(t)^H (rows j < P = M(M+1)/2: Re of pair p = j in the k_vacc/k_ip pair
// order; rows j >= P: Im of the (j-P)-th off-diagonal pair) and B[m][t] =
// 1/y(t, m). The SIMT threads build A and B for a chunk of KC frames (the
// outer products are M-fold cheaper than the weighted accumulation they
// replace), one thread issues tcgen05.mma.kind::tf32 into a TMEM accumulator
// (128-lane tiles), and tcgen05.commit on a per-stage mbarrier hands the
// stage back. Precision: 3xTF32 (A_hi B_hi + A_hi B_lo + A_lo B_hi with
// hi = rna-rounded TF32, lo = residual), i.e. fp32-level products with fp32
// accumulation -- the same arithmetic class as the SIMT k_vacc.
//
// Shared-memory operand layout: UMMA K-major, no swizzle: 8-row x 16-byte
// core matrices, LBO = 128 B between the K-adjacent cores, SBO = (KC/4)*128 B
// between 8-row groups. The gain MU that k_vacc finishes is done identically.
// grid (nseg, F, B), block 256; fp32 only.
#pragma once
#include "fm_spatial.cuh"

namespace fm {

template <int M> struct VtcCfg {
  static constexpr int P = M * (M + 1) / 2;
  static constexpr int J = M * M;                  // real rows of A
  static constexpr int NTILE = (J + 127) / 128;    // 128-lane tiles (A and accumulator)
  static constexpr int NB = (M + 7) / 8 * 8;       // MMA N (weights per m, padded)
  static constexpr int KC = 16;                    // frames per chunk (KC/8 MMA k-steps)
  static constexpr int BS = 256;
  static constexpr int WG = 8 / (4 * NTILE);       // warp groups sharing a tile's rows (split frames)
  static constexpr int KW = KC / WG;               // frames per thread per chunk
  static constexpr int SBO = (KC / 4) * 128;       // B plane: bytes between 8-row core groups
  static constexpr int BBYTES = NB * KC * 4;       // one B plane (hi or lo)
  static constexpr int TBLK = M <= 8 ? 256 : 128;  // frames staged per block (x, 1/y)
  static constexpr int STAGE = 2 * BBYTES;
  static constexpr int XS = 2 * STAGE;             // x block (M x TBLK complex, padded rows)
  static constexpr int XLD = TBLK + 2;             // x row pitch (complex): rows land on distinct banks
  static constexpr int IYS = XS + XLD * M * 8;     // 1/y block (M x TBLK)
  static constexpr int SMEM = IYS + TBLK * M * 4;
  // TMEM columns: accumulator [0, NTILE*NB), then per stage, tile and plane (hi, lo) KC columns
  static constexpr int ACOL = 32;
  static constexpr int TCOLS_USED = ACOL + 2 * NTILE * 2 * KC;
  static constexpr int TCOLS = TCOLS_USED <= 128 ? 128 : TCOLS_USED <= 256 ? 256 : 512;
  static_assert(NTILE * NB <= ACOL, "accumulator columns");
  static_assert(WG >= 1 && KC % WG == 0, "warp groups");
};
__host__ __device__ constexpr int vtc_acol(int stage, int tile, int plane, int ntile, int kc) {
  return 32 + ((stage * ntile + tile) * 2 + plane) * kc;
}

// byte offset of element (row, k) in a K-major no-swizzle operand plane
template <int M> __device__ __forceinline__ uint32_t vtc_off(int row, int k) {
  return (uint32_t)((((row >> 3) * (VtcCfg<M>::KC / 4) + (k >> 2)) * 128) + ((row & 7) * 16) +
                    ((k & 3) * 4));
}

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
  return d;                // base offset 0, layout SWIZZLE_NONE
}

__device__ __forceinline__ float tf32_rna(float v) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
  return __uint_as_float(r);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)),
               "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}\n" ::"r"((unsigned)__cvta_generic_to_shared(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// A operand from tensor memory (rows = lanes, K along columns)
__device__ __forceinline__ void umma_tf32_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// registers -> TMEM: lane (warp quadrant) x NC consecutive columns
template <int NC> __device__ __forceinline__ void tmem_st_row(uint32_t taddr, const float (&v)[NC]);
template <> __device__ __forceinline__ void tmem_st_row<8>(uint32_t taddr, const float (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
               "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
               : "memory");
}
template <> __device__ __forceinline__ void tmem_st_row<16>(uint32_t taddr, const float (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]),
      "f"(v[9]), "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15])
      : "memory");
}
template <> __device__ __forceinline__ void tmem_st_row<32>(uint32_t taddr, const float (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]),
      "f"(v[9]), "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]), "f"(v[16]),
      "f"(v[17]), "f"(v[18]), "f"(v[19]), "f"(v[20]), "f"(v[21]), "f"(v[22]), "f"(v[23]), "f"(v[24]),
      "f"(v[25]), "f"(v[26]), "f"(v[27]), "f"(v[28]), "f"(v[29]), "f"(v[30]), "f"(v[31])
      : "memory");
}

template <int NB> __device__ __forceinline__ void tmem_ld_row(uint32_t taddr, float (&v)[NB]) {
  uint32_t r[NB];
  if constexpr (NB == 8) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                   "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
  } else {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, "
        "[%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
  }
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < NB; ++i) v[i] = __uint_as_float(r[i]);
}

template <int M>
__global__ void __launch_bounds__(256) k_vacc_tc(VaccArgs<float> a) {
  pdl_entry();
  using Cf = VtcCfg<M>;
  using C = float2;
  constexpr int P = Cf::P, J = Cf::J, NTILE = Cf::NTILE, NB = Cf::NB, KC = Cf::KC, BS = Cf::BS;
  constexpr int KW = Cf::KW;
  extern __shared__ __align__(1024) unsigned char smv[];
  __shared__ __align__(8) uint64_t mbar[2];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(16) float gs[NMAX * M];
  __shared__ unsigned char pairI[P], pairK[P];
  __shared__ short pairIm[P];  // A row of Im(pair), -1 on the diagonal
  const int seg = blockIdx.x, f = blockIdx.y, b = blockIdx.z, nseg = gridDim.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int N = a.N, T = a.T, F = a.F;
  const size_t FT = (size_t)F * T;
  const int ta = seg * a.TR, tb = min(T, ta + a.TR);

  // gain MU from the k_gain segment partials (fixed order; as k_vacc)
  for (int e = tid; e < N * M; e += BS) {
    const int n = e / M, m = e % M;
    const float* gp = a.gpart + ((size_t)b * F + f) * a.gseg * N * 2 * M + n * 2 * M;
    float sn = 0, sd = 0;
    for (int q = 0; q < a.gseg; ++q) {
      sn += gp[(size_t)q * N * 2 * M + m];
      sd += gp[(size_t)q * N * 2 * M + M + m];
    }
    const size_t gi = (size_t)b * N * F * M + (size_t)n * F * M + (size_t)f * M + m;
    const float gv = a.g[gi] * mu_factor(sn, sd);
    gs[e] = gv;
    if (seg == 0) a.gnew[gi] = gv;
  }
  // pair p = (i <= k) in the k_vacc / k_ip order; its Re is A row p, its Im
  // (off-diagonal pairs only) A row P + (index among the off-diagonal pairs)
  for (int p = tid; p < P; p += BS) {
    int i = 0, r = p;
    while (r >= M - i) {
      r -= M - i;
      ++i;
    }
    pairI[p] = (unsigned char)i;
    pairK[p] = (unsigned char)(i + r);
    pairIm[p] = r == 0 ? (short)-1 : (short)(P + p - i - 1);  // off-diagonals before p: p - (i + 1)
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (unsigned)__cvta_generic_to_shared(&tmem_base)),
                 "r"(Cf::TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  const uint32_t sbase = (unsigned)__cvta_generic_to_shared(smv);
  // operand descriptors of stage 0 (A hi plane, B hi plane); per-MMA offsets are
  // added to the 14-bit start-address field (16-byte units, no carry out: < 256 KB)
  const uint64_t dB = umma_desc(sbase, 128, Cf::SBO);
  // this thread's A row: tile (warp / 4 when two tiles), lane quadrant (warp % 4), frame group
  const int tile = NTILE == 2 ? warp >> 2 : 0, wg = NTILE == 2 ? 0 : warp >> 2;
  const int arow = tile * 128 + (warp & 3) * 32 + lane;  // A row j (rows >= J are padding)
  int ai = 0, ak = 0;
  {
    const int j = arow < J ? arow : 0;
    int p = j, q = j - P;
    if (j >= P) {  // Im of the q-th off-diagonal pair
      int i = 0, rem = q;
      while (rem >= M - 1 - i) {
        rem -= M - 1 - i;
        ++i;
      }
      ai = i;
      ak = i + 1 + rem;
    } else {
      int i = 0, rem = p;
      while (rem >= M - i) {
        rem -= M - i;
        ++i;
      }
      ai = i;
      ak = i + rem;
    }
  }
  constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(NB >> 3) << 17) |
                             ((uint32_t)(128 >> 4) << 24);

  const float fl = a.floorp[b];
  const float* lamb = a.lam + (size_t)b * N * FT + (size_t)f * T;
  const C* Xb = a.X + ((size_t)b * F + f) * T * M;
  float lp[NMAX];
  C xp[M];
  auto fetch = [&](int c0) {
    const int t = c0 + tid;
    const int tc = t < tb ? t : tb - 1;
#pragma unroll
    for (int n = 0; n < NMAX; ++n) {
      lp[n] = 0.f;
      if (n >= N) break;
      lp[n] = lamb[(size_t)n * FT + tc];
    }
    CRowIO<float, M>::load(Xb + (size_t)tc * M, xp);
  };
  // x and 1/y are staged TBLK frames at a time by all threads (one frame each,
  // the next block prefetched into registers); each block feeds TBLK/KC
  // tensor-core chunks through the two operand stages
  C* Xs = reinterpret_cast<C*>(smv + Cf::XS);
  float* Ys = reinterpret_cast<float*>(smv + Cf::IYS);
  constexpr int TBLK = Cf::TBLK;
  if (tid < TBLK) fetch(ta);
  int c = 0;  // chunk counter (stage = c & 1)
  for (int b0 = ta; b0 < tb; b0 += TBLK) {
    __syncthreads();  // previous block's x / 1/y consumed
    if (tid < TBLK) {
      const bool tv = b0 + tid < tb;
      float l[NMAX];
      C xv[M];
#pragma unroll
      for (int n = 0; n < NMAX; ++n) l[n] = lp[n];
#pragma unroll
      for (int m = 0; m < M; ++m) xv[m] = tv ? xp[m] : make_float2(0.f, 0.f);
      if (b0 + TBLK < tb) fetch(b0 + TBLK);
      float iy[M], y[M];
      model_power<float, M>(l, gs, N, fl, iy, y);
#pragma unroll
      for (int m = 0; m < M; ++m)
        if (!tv) iy[m] = 0.f;
#pragma unroll
      for (int m = 0; m < M; ++m) {  // [m][t]: 4 consecutive frames of one channel are 16/32 B
        Xs[m * Cf::XLD + tid] = xv[m];
        Ys[m * TBLK + tid] = iy[m];
      }
    }
    __syncthreads();
    const int nchb = min(TBLK, tb - b0 + KC - 1) / KC;
    for (int cb = 0; cb < nchb; ++cb, ++c) {
      const int s = c & 1;
      unsigned char* Bhi = smv + s * Cf::STAGE;
      unsigned char* Blo = Bhi + Cf::BBYTES;
      if (c >= 2) mbar_wait(&mbar[s], (unsigned)(((c >> 1) - 1) & 1));  // MMAs of chunk c-2 done
      const int k0 = cb * KC;  // chunk's first frame inside the block
      // B rows: 1/y of the chunk's frames, 4 frames per item (smem, UMMA K-major)
      for (int e = a.dbg == 2 ? BS : tid; e < M * (KC / 4); e += BS) {
        const int m = e / (KC / 4), kq = e % (KC / 4);
        const float4 v = *reinterpret_cast<const float4*>(Ys + m * TBLK + k0 + kq * 4);
        float4 h;
        h.x = tf32_rna(v.x); h.y = tf32_rna(v.y); h.z = tf32_rna(v.z); h.w = tf32_rna(v.w);
        const uint32_t o = vtc_off<M>(m, kq * 4);
        *reinterpret_cast<float4*>(Bhi + o) = h;
        *reinterpret_cast<float4*>(Blo + o) = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
      }
      // A rows -> TMEM: this thread's row (lane) for its KW frames, hi and lo planes
      if (a.dbg != 2) {
        const bool im = arow >= P;
        const C* xi = Xs + ai * Cf::XLD + k0 + wg * KW;
        const C* xk = Xs + ak * Cf::XLD + k0 + wg * KW;
        float hv[KW], lv[KW];
#pragma unroll
        for (int u = 0; u < KW; u += 2) {
          const float4 pi = *reinterpret_cast<const float4*>(xi + u);
          const float4 pk = *reinterpret_cast<const float4*>(xk + u);
          const float v0 = im ? (pi.y * pk.x - pi.x * pk.y) : (pi.x * pk.x + pi.y * pk.y);
          const float v1 = im ? (pi.w * pk.z - pi.z * pk.w) : (pi.z * pk.z + pi.w * pk.w);
          hv[u] = tf32_rna(v0);
          hv[u + 1] = tf32_rna(v1);
          lv[u] = v0 - hv[u];
          lv[u + 1] = v1 - hv[u + 1];
        }
        const uint32_t lanes = (uint32_t)((warp & 3) * 32) << 16;
        tmem_st_row<KW>(tmem + lanes + vtc_acol(s, tile, 0, NTILE, KC) + wg * KW, hv);
        tmem_st_row<KW>(tmem + lanes + vtc_acol(s, tile, 1, NTILE, KC) + wg * KW, lv);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncthreads();
      if (tid == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint64_t so = (uint64_t)((uint32_t)(s * Cf::STAGE) >> 4);  // stage offset (16-byte units)
#pragma unroll
        for (int ks = 0; ks < KC / 8; ++ks) {
          const uint64_t dbh = dB + so + ks * 16, dbl = dB + so + (Cf::BBYTES >> 4) + ks * 16;
#pragma unroll
          for (int tt = 0; tt < NTILE; ++tt) {
            const uint32_t tah = tmem + (uint32_t)(vtc_acol(s, tt, 0, NTILE, KC) + ks * 8);
            const uint32_t tal = tmem + (uint32_t)(vtc_acol(s, tt, 1, NTILE, KC) + ks * 8);
            const uint32_t td = tmem + (uint32_t)(tt * NB);
            if (a.dbg == 1) continue;
            umma_tf32_ts(td, tah, dbh, IDESC, (c > 0 || ks > 0) ? 1u : 0u);
            umma_tf32_ts(td, tah, dbl, IDESC, 1u);
            umma_tf32_ts(td, tal, dbh, IDESC, 1u);
          }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         (unsigned)__cvta_generic_to_shared(&mbar[s]))
                     : "memory");
      }
    }
  }
  const int nch = c;
  // the last commit covers every MMA of this CTA
  mbar_wait(&mbar[(nch - 1) & 1], (unsigned)(((nch - 1) >> 1) & 1));
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  C* pb = reinterpret_cast<C*>(a.part) + (((size_t)b * F + f) * nseg + seg) * M * P;
  if (warp < 4) {
#pragma unroll
    for (int tt = 0; tt < NTILE; ++tt) {
      float d[NB];
      tmem_ld_row<NB>(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(tt * NB), d);
      const int r = tt * 128 + warp * 32 + lane;
      if (r < J) {
        int p = r, part = 0;
        if (r >= P) {  // Im row: find the off-diagonal pair
          const int q = r - P;
          int i = 0, rem = q;
          while (rem >= M - 1 - i) {
            rem -= M - 1 - i;
            ++i;
          }
          p = q + i + 1;  // pairs before (i, i+1+rem): q off-diagonals + (i + 1) diagonals
          part = 1;
        }
        float* dst = reinterpret_cast<float*>(pb + p) + part;
        const bool diag = part == 0 && pairI[p] == pairK[p];
#pragma unroll
        for (int m = 0; m < M; ++m) {
          if (a.dbg) d[m] = diag ? 1.f : 0.f;  // timing experiments: a valid V
          dst[(size_t)m * P * 2] = d[m];
          if (diag) dst[(size_t)m * P * 2 + 1] = 0.f;
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(Cf::TCOLS));
}

}  // namespace fm
