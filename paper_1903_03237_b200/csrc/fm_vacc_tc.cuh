// fm_vacc_tc.cuh -- the V_fm accumulation on the 5th-generation tensor cores
// (complex64 path, even M >= 12, _kernels.py:276-293,
// spatial.py:182).
//
// V_fm[i,k] = sum_t iy[t,m] x_i(t) conj(x_k(t)) is, per bin f, one small GEMM
//   D[j][m] = sum_t A[j][t] B[m][t]
// with A[j][t] the M*M real components of the Hermitian outer product
// x(t) x(t)^H and B[m][t] = 1/y(t, m). Building A costs O(M^2) per frame, M
// times less than the weighted SIMT accumulation it replaces.
//
// Warp-specialised, mbarrier-pipelined, no CTA barrier in the frame loop:
//   loader warps (4)  X of a 128-frame block by one bulk async copy
//                     (cp.async.bulk, the block is contiguous in (B,F,T,M));
//                     1/y from lambda and the updated gains, rounded and split
//                     into TF32 hi / lo planes written straight into the UMMA
//                     K-major layout of the block (rows 0..15 hi, 16..31 lo)
//   producer warps (8) a thread owns accumulator lane L of BOTH 128-lane
//                     tiles: Re (tile 0) and Im (tile 1) of off-diagonal pair L
//                     (L < M(M-1)/2), or |x_d|^2 of two diagonal entries (lanes
//                     120..127); per 16-frame chunk it forms its products for 8
//                     frames from shared x rows, splits them hi / lo and
//                     stores them to TMEM (tcgen05.st) as the A operand
//   MMA warp (1 lane)  per chunk and tile, per 8-frame k-step:
//                     D[:, 0:32] += A_hi [B_hi | B_lo]  (one N = 32 MMA) and
//                     D[:, 0:16] += A_lo B_hi           (N = 16); tcgen05.commit hands
//                     the operand stage (and, per block, the block buffers) back
// Precision: 3xTF32 (A_hi B_hi + A_hi B_lo + A_lo B_hi, fp32 accumulation in
// TMEM; the accumulator's two halves are summed in the epilogue) -- fp32-class products,
// the same arithmetic class as the SIMT k_vacc. The gain MU that k_vacc
// finishes is done identically. grid (nseg, F, B), block 416; fp32 only.
#pragma once
#include "fm_spatial.cuh"

namespace fm {

template <int M> struct VtcCfg {
  // used for even M in 10..16 (Impl::vacc); instantiable for every M
  static constexpr int P = M * (M + 1) / 2;
  static constexpr int PO = M * (M - 1) / 2;       // off-diagonal pairs (<= 120): lanes [0, PO)
  static constexpr int DL = 120;                   // first diagonal lane (8 per tile)
  static constexpr int NB = 16;                    // weight rows per plane (m, zero-padded)
  static constexpr int KC = 16;                    // frames per chunk (two MMA k-steps)
  static constexpr int TBLK = 128;                 // frames per staged block
  static constexpr int NPROD = 8, NLOAD = 4;       // warps
  static constexpr int MMAW = NPROD;               // the MMA warp
  static constexpr int BS = (NPROD + 1 + NLOAD) * 32;
  static constexpr int XB = TBLK * M * 8;          // x block (frames x channels, complex)
  static constexpr int WB = 2 * NB * TBLK * 4;     // weight block: hi rows then lo rows
  static constexpr int SBO = (TBLK / 4) * 128;     // bytes between 8-row core groups
  static constexpr int OFF_W = 2 * XB;
  static constexpr int OFF_L = OFF_W + 2 * WB;     // loader warps' lambda rows (cp.async)
  static constexpr int SMEM = OFF_L + NLOAD * 2 * NMAX * 8 * 16;
  static constexpr int S = 2;                      // operand stages in TMEM (one per producer group)
  // TMEM columns: per tile 32 accumulator columns (A_hi B_hi + A_lo B_hi | A_hi B_lo);
  // then per stage, tile and plane KC columns
  static constexpr int DCOLS = 32, ACOL = 2 * DCOLS;
  static constexpr int TCOLS = 256;
  static_assert(ACOL + S * 2 * 2 * KC <= TCOLS, "tensor memory columns");
};
__host__ __device__ constexpr int vtc_acol(int stage, int tile, int plane) {
  return 64 + ((stage * 2 + tile) * 2 + plane) * 16;
}

// byte offset of element (row, k) in the block's K-major no-swizzle weight plane
template <int M> __device__ __forceinline__ uint32_t vtc_off(int row, int k) {
  return (uint32_t)((((row >> 3) * (VtcCfg<M>::TBLK / 4) + (k >> 2)) * 128) + ((row & 7) * 16) +
                    ((k & 3) * 4));
}

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
  return d;                // base offset 0, layout SWIZZLE_NONE
}

// Round to TF32 (10 mantissa bits), nearest with ties away from zero -- what
// cvt.rna.tf32.f32 returns for finite normal inputs -- with two integer
// operations: the conversion instruction issues at 16 lanes per clock per SM
// and was the limit of the operand build (8192 per 16-frame chunk).
__device__ __forceinline__ float tf32_rna(float v) {
  return __uint_as_float((__float_as_uint(v) + 0x1000u) & 0xFFFFE000u);
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

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((unsigned)__cvta_generic_to_shared(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                   (unsigned)__cvta_generic_to_shared(bar)),
               "r"(bytes)
               : "memory");
}
// global -> shared bulk async copy (TMA engine, no tensor map); completes on the mbarrier
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          (unsigned)__cvta_generic_to_shared(dst)),
      "l"(src), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(bar))
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   (unsigned)__cvta_generic_to_shared(bar))
               : "memory");
}
// 16 accumulator columns of this thread's lane, no wait
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, "
      "[%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

template <int M>
__global__ void __launch_bounds__(VtcCfg<M>::BS, 2) k_vacc_tc(VaccArgs<float> a) {
  pdl_entry();
  using Cf = VtcCfg<M>;
  using C = float2;
  constexpr int P = Cf::P, PO = Cf::PO, DL = Cf::DL, KC = Cf::KC, TBLK = Cf::TBLK, S = Cf::S;
  constexpr int BS = Cf::BS;
  extern __shared__ __align__(1024) unsigned char smv[];
  // mbarriers: block buffers full (x landed + weights written) / empty (producers and
  // MMAs done with them), operand stages full / empty, all MMAs done
  __shared__ __align__(8) uint64_t bfull[2], bempty[2], sfull[S], sempty[S], done;
  __shared__ uint32_t tmem_base;
  __shared__ __align__(16) float gs[NMAX * 16];  // updated gains, m padded to 16 with zeros
  const int seg = blockIdx.x, f = blockIdx.y, b = blockIdx.z, nseg = gridDim.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int N = a.N, T = a.T, F = a.F;
  const size_t FT = (size_t)F * T;
  const int ta = seg * a.TR, tb = min(T, ta + a.TR);
  const int nblk = (tb - ta + TBLK - 1) / TBLK;

  // gain MU from the k_gain segment partials (fixed order; as k_vacc)
  for (int e = tid; e < NMAX * 16; e += BS) {
    const int n = e >> 4, m = e & 15;
    float gv = 0.f;
    if (n < N && m < M) {
      const float* gp = a.gpart + ((size_t)b * F + f) * a.gseg * N * 2 * M + n * 2 * M;
      float sn = 0, sd = 0;
      for (int q = 0; q < a.gseg; ++q) {
        sn += gp[(size_t)q * N * 2 * M + m];
        sd += gp[(size_t)q * N * 2 * M + M + m];
      }
      const size_t gi = (size_t)b * N * F * M + (size_t)n * F * M + (size_t)f * M + m;
      gv = a.g[gi] * mu_factor(sn, sd);
      if (seg == 0) a.gnew[gi] = gv;
    }
    gs[e] = gv;
  }
  // x buffers start as zeros: the frames of a ragged last chunk beyond the copied
  // ones are read with zero weights and must hold finite values
  for (int e = tid; e < 2 * Cf::XB / 16; e += BS)
    reinterpret_cast<float4*>(smv)[e] = make_float4(0.f, 0.f, 0.f, 0.f);
  if (warp == Cf::MMAW) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (unsigned)__cvta_generic_to_shared(&tmem_base)),
                 "r"(Cf::TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bfull[i], Cf::NLOAD + 1);   // loader warps + the expect_tx arrive
      mbar_init(&bempty[i], Cf::NPROD + 1);  // producer warps + the MMA commit
    }
    for (int i = 0; i < S; ++i) {
      mbar_init(&sfull[i], Cf::NPROD / 2);
      mbar_init(&sempty[i], 1);
    }
    mbar_init(&done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // zero fill before the bulk copies
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;

  if (warp < Cf::NPROD) {
    // ---------------- producers: A rows -> TMEM ----------------
    // warps 0-3 build the even chunks in stage 0, warps 4-7 the odd chunks in stage 1:
    // one handshake per 16 frames x 2 rows per thread
    const int q = warp & 3, par = warp >> 2;  // lane quadrant, chunk parity (= stage)
    const int L = q * 32 + lane;
    int ai = 0, ak = 0;
    const bool isdiag = L >= DL;
    if (L < PO) {  // L-th off-diagonal pair (i < k), i-major
      int i = 0, rem = L;
      while (rem >= M - 1 - i) {
        rem -= M - 1 - i;
        ++i;
      }
      ai = i;
      ak = i + 1 + rem;
    } else if (isdiag) {  // |x_d|^2 for d = L - DL (tile 0) and d + 8 (tile 1)
      ai = L - DL < M ? L - DL : 0;
      ak = L - DL + 8 < M ? L - DL + 8 : 0;
    }
    const uint32_t tst = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)vtc_acol(par, 0, 0);
    int c = 0;
    for (int blk = 0; blk < nblk; ++blk) {
      const int bb = blk & 1;
      mbar_wait(&bfull[bb], (unsigned)((blk >> 1) & 1));
      const C* Xs = reinterpret_cast<const C*>(smv + bb * Cf::XB);
      const int nfr = min(TBLK, tb - ta - blk * TBLK);
      const int nchb = (nfr + KC - 1) / KC;
      for (int cb = 0; cb < nchb; ++cb, ++c) {
        if ((c & 1) != par) continue;
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const C* xr = Xs + (cb * KC + hh * 8) * M;
          float h0[8], l0[8], h1[8], l1[8];
          if (!(a.dbg & 2)) {
            if (q != 3) {  // warp-uniform: only the last lane quadrant holds diagonal lanes
#pragma unroll
              for (int u = 0; u < 8; ++u) {
                const C xi = xr[u * M + ai], xk = xr[u * M + ak];
                const float v0 = xi.x * xk.x + xi.y * xk.y;
                const float v1 = xi.y * xk.x - xi.x * xk.y;
                h0[u] = tf32_rna(v0);
                l0[u] = v0 - h0[u];
                h1[u] = tf32_rna(v1);
                l1[u] = v1 - h1[u];
              }
            } else {
#pragma unroll
              for (int u = 0; u < 8; ++u) {
                const C xi = xr[u * M + ai], xk = xr[u * M + ak];
                const float v0 = isdiag ? (xi.x * xi.x + xi.y * xi.y) : (xi.x * xk.x + xi.y * xk.y);
                const float v1 = isdiag ? (xk.x * xk.x + xk.y * xk.y) : (xi.y * xk.x - xi.x * xk.y);
                h0[u] = tf32_rna(v0);
                l0[u] = v0 - h0[u];
                h1[u] = tf32_rna(v1);
                l1[u] = v1 - h1[u];
              }
            }
          }
          if (hh == 0) {
            // the first products are ready before the stage is: the MMAs of chunk c-2 overlap them
            if (c >= 2) mbar_wait(&sempty[par], (unsigned)(((c >> 1) - 1) & 1));
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          }
          if (!(a.dbg & 2)) {
            tmem_st_row<8>(tst + 0 * KC + hh * 8, h0);
            tmem_st_row<8>(tst + 1 * KC + hh * 8, l0);
            tmem_st_row<8>(tst + 2 * KC + hh * 8, h1);
            tmem_st_row<8>(tst + 3 * KC + hh * 8, l1);
          }
        }
        if (!(a.dbg & 2)) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&sfull[par]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&bempty[bb]);  // this warp has read the block's x
    }
  } else if (warp == Cf::MMAW) {
    // ---------------- MMA issue: one lane ----------------
    if (lane == 0) {
      constexpr uint32_t IDESC32 = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(32 >> 3) << 17) |
                                   ((uint32_t)(128 >> 4) << 24);
      constexpr uint32_t IDESC16 = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(16 >> 3) << 17) |
                                   ((uint32_t)(128 >> 4) << 24);
      const uint32_t sbase = (unsigned)__cvta_generic_to_shared(smv);
      int c = 0;
      for (int blk = 0; blk < nblk; ++blk) {
        const int bb = blk & 1;
        mbar_wait(&bfull[bb], (unsigned)((blk >> 1) & 1));
        const uint64_t dB = umma_desc(sbase + Cf::OFF_W + bb * Cf::WB, 128, Cf::SBO);
        const int nfr = min(TBLK, tb - ta - blk * TBLK);
        const int nchb = (nfr + KC - 1) / KC;
        for (int cb = 0; cb < nchb; ++cb, ++c) {
          const int s = c & 1;
          mbar_wait(&sfull[s], (unsigned)((c >> 1) & 1));
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          if (!(a.dbg & 1)) {
#pragma unroll
            for (int ks = 0; ks < KC / 8; ++ks) {
              const uint64_t db = dB + (uint64_t)(cb * (KC / 4) * 8 + ks * 16);  // 16-byte units
#pragma unroll
              for (int tt = 0; tt < 2; ++tt) {
                const uint32_t acc = (c > 0 || ks > 0) ? 1u : 0u;
                umma_tf32_ts(tmem + (uint32_t)(tt * Cf::DCOLS), tmem + (uint32_t)(vtc_acol(s, tt, 0) + ks * 8),
                             db, IDESC32, acc);
                umma_tf32_ts(tmem + (uint32_t)(tt * Cf::DCOLS),
                             tmem + (uint32_t)(vtc_acol(s, tt, 1) + ks * 8), db, IDESC16, 1u);
              }
            }
          }
          umma_commit(&sempty[s]);
        }
        umma_commit(&bempty[bb]);  // the block's weight planes are free once these MMAs retire
      }
      umma_commit(&done);
    }
  } else {
    // ---------------- loaders: x by bulk copy, weights 1/y as TF32 hi / lo planes ----------------
    const int lw = warp - Cf::MMAW - 1;  // 0..3
    const int ml = lane & 7, tql = lane >> 3;
    const float fl = a.floorp[b];
    const float* lamb = a.lam + (size_t)b * N * FT + (size_t)f * T;
    const C* Xb = a.X + ((size_t)b * F + f) * T * M;
    const bool vec = (T & 3) == 0;
    // lambda of the next block: cp.async into this warp's private rows
    // Lw[buf][n][quad] (a warp covers 8 frame quads of a block), so no register
    // holds a prefetch and no other warp is involved
    float4* Lw = reinterpret_cast<float4*>(smv + Cf::OFF_L) + lw * 2 * NMAX * 8;
    auto fetch = [&](int blk) {
      float4* dstb = Lw + (blk & 1) * NMAX * 8;
      for (int e = lane; e < N * 8; e += 32) {
        const int n = e >> 3, qi = e & 7;
        const int t = ta + blk * TBLK + (((qi >> 2) * 4 + lw) * 4 + (qi & 3)) * 4;
        const float* lp = lamb + (size_t)n * FT + t;
        const unsigned dst = (unsigned)__cvta_generic_to_shared(dstb + e);
        if (vec) {
          const unsigned sz = t < tb ? 16u : 0u;
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst),
                       "l"(t < tb ? lp : lamb), "r"(sz)
                       : "memory");
        } else {
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const unsigned sz = t + u < tb ? 4u : 0u;
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst + 4 * u),
                         "l"(t + u < tb ? lp + u : lamb), "r"(sz)
                         : "memory");
          }
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    fetch(0);
    for (int blk = 0; blk < nblk; ++blk) {
      const int bb = blk & 1;
      if (blk + 1 < nblk) {
        fetch(blk + 1);
        asm volatile("cp.async.wait_group 1;" ::: "memory");
      } else {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
      }
      __syncwarp();
      if (blk >= 2) mbar_wait(&bempty[bb], (unsigned)(((blk >> 1) - 1) & 1));
      const int t0 = ta + blk * TBLK;
      const int nfr = min(TBLK, tb - t0);
      if (lw == 0 && lane == 0) {
        const unsigned bytes = (unsigned)(nfr * M * 8);
        mbar_arrive_expect_tx(&bfull[bb], bytes);
        bulk_g2s(smv + bb * Cf::XB, Xb + (size_t)t0 * M, bytes, &bfull[bb]);
      }
      unsigned char* Wp = smv + Cf::OFF_W + bb * Cf::WB;
      const float4* Lb = Lw + bb * NMAX * 8;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int kq = (j * 4 + lw) * 4 + tql;  // frame quad inside the block
        const int t = t0 + kq * 4;
#pragma unroll
        for (int mh = 0; mh < 2; ++mh) {
          const int m = mh * 8 + ml;
          float y0 = 0.f, y1 = 0.f, y2 = 0.f, y3 = 0.f;
#pragma unroll
          for (int n = 0; n < NMAX; ++n) {
            if (n >= N) break;
            const float gv = gs[n * 16 + m];
            const float4 l4 = Lb[n * 8 + j * 4 + tql];
            y0 += l4.x * gv;
            y1 += l4.y * gv;
            y2 += l4.z * gv;
            y3 += l4.w * gv;
          }
          float4 v;
          v.x = (m < M && t < tb) ? rcp_r(floor_max(y0, fl)) : 0.f;
          v.y = (m < M && t + 1 < tb) ? rcp_r(floor_max(y1, fl)) : 0.f;
          v.z = (m < M && t + 2 < tb) ? rcp_r(floor_max(y2, fl)) : 0.f;
          v.w = (m < M && t + 3 < tb) ? rcp_r(floor_max(y3, fl)) : 0.f;
          float4 hi;
          hi.x = tf32_rna(v.x); hi.y = tf32_rna(v.y); hi.z = tf32_rna(v.z); hi.w = tf32_rna(v.w);
          *reinterpret_cast<float4*>(Wp + vtc_off<M>(m, kq * 4)) = hi;
          *reinterpret_cast<float4*>(Wp + vtc_off<M>(16 + m, kq * 4)) =
              make_float4(v.x - hi.x, v.y - hi.y, v.z - hi.z, v.w - hi.w);
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&bfull[bb]);
    }
  }

  // ---------------- epilogue: accumulator halves -> the segment's partial V ----------------
  if (warp < Cf::NPROD) {
    mbar_wait(&done, 0u);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int q = warp & 3, tt = warp >> 2;  // warps 0-3 read tile 0 (Re), 4-7 tile 1 (Im)
    const int L = q * 32 + lane;
    const uint32_t base = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(tt * Cf::DCOLS);
    float d0[16], d1[16];
    tmem_ld16(base, d0);
    tmem_ld16(base + 16, d1);
    int p = -1, part = tt;
    if (L < PO) {
      int i = 0, rem = L;
      while (rem >= M - 1 - i) {
        rem -= M - 1 - i;
        ++i;
      }
      p = i * M - i * (i - 1) / 2 + 1 + rem;  // pairs before row i, then (k - i)
    } else if (L >= DL) {
      const int dd = L - DL + 8 * tt;
      if (dd < M) p = dd * M - dd * (dd - 1) / 2;
      part = 0;
    }
    if (p >= 0) {
      float* dst = reinterpret_cast<float*>(reinterpret_cast<C*>(a.part) +
                                            (((size_t)b * F + f) * nseg + seg) * M * P + p) + part;
      const bool diag = L >= DL;
#pragma unroll
      for (int m = 0; m < M; ++m) {
        float v = d0[m] + d1[m];
        if (a.dbg) v = diag ? 1.f : 0.f;  // timing experiments: a valid V
        dst[(size_t)m * P * 2] = v;
        if (diag) dst[(size_t)m * P * 2 + 1] = 0.f;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == Cf::MMAW)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(Cf::TCOLS));
}

}  // namespace fm
