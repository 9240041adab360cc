// fm_impl.cuh -- host-side launch logic, templated on the real type.
// Explicitly instantiated in fm_f32.cu / fm_f64.cu (parallel compilation);
// fm_api.cu holds the extern "C" boundary (include/fastmnmf.h).
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/fastmnmf.h"
#include "fm_kernels.cuh"
#include "fm_ops.cuh"
#include "fm_dp_latent.cuh"
#include "fm_dp_mh.cuh"
#include "fm_vacc_tc.cuh"
#include "fm_back_tc.cuh"
#include "fm_lambda_tc.cuh"
#include "fm_vacc_blk.cuh"
#include "fm_vacc_p.cuh"
#include "fm_init.cuh"
#include "fm_stft.cuh"
#include "fm_fullrank.cuh"
#include "fm_fused.cuh"
#include "fm_ipw.cuh"
#include "fm_small.cuh"

namespace fm {

void set_error(const char* fmt, ...);


#define FM_CHECK_LAUNCH(what)                                                   \
  do {                                                                          \
    cudaError_t e_ = cudaGetLastError();                                        \
    if (e_ != cudaSuccess) {                                                    \
      set_error("%s: %s", what, cudaGetErrorString(e_));                         \
      return FM_ECUDA;                                                          \
    }                                                                           \
  } while (0)

#define FM_CUDA(call)                                                           \
  do {                                                                          \
    cudaError_t e_ = (call);                                                    \
    if (e_ != cudaSuccess) {                                                    \
      set_error("%s: %s", #call, cudaGetErrorString(e_));                        \
      return FM_ECUDA;                                                          \
    }                                                                           \
  } while (0)

// M dispatch (M = 1..16), compile-time channel count for the per-bin kernels.
#define FM_DISPATCH_M(Mrt, ...)                                                \
  switch (Mrt) {                                                                \
    case 1: { constexpr int MM = 1; __VA_ARGS__; } break;                              \
    case 2: { constexpr int MM = 2; __VA_ARGS__; } break;                              \
    case 3: { constexpr int MM = 3; __VA_ARGS__; } break;                              \
    case 4: { constexpr int MM = 4; __VA_ARGS__; } break;                              \
    case 5: { constexpr int MM = 5; __VA_ARGS__; } break;                              \
    case 6: { constexpr int MM = 6; __VA_ARGS__; } break;                              \
    case 7: { constexpr int MM = 7; __VA_ARGS__; } break;                              \
    case 8: { constexpr int MM = 8; __VA_ARGS__; } break;                              \
    case 9: { constexpr int MM = 9; __VA_ARGS__; } break;                              \
    case 10: { constexpr int MM = 10; __VA_ARGS__; } break;                            \
    case 11: { constexpr int MM = 11; __VA_ARGS__; } break;                            \
    case 12: { constexpr int MM = 12; __VA_ARGS__; } break;                            \
    case 13: { constexpr int MM = 13; __VA_ARGS__; } break;                            \
    case 14: { constexpr int MM = 14; __VA_ARGS__; } break;                            \
    case 15: { constexpr int MM = 15; __VA_ARGS__; } break;                            \
    case 16: { constexpr int MM = 16; __VA_ARGS__; } break;                            \
    default: set_error("M=%d outside the supported 1..16", (int)(Mrt)); return FM_EINVAL; \
  }

#define FM_DISPATCH_KB(Krt, ...)                                               \
  if ((Krt) <= 4) { constexpr int KB = 4; __VA_ARGS__; }                               \
  else if ((Krt) <= 8) { constexpr int KB = 8; __VA_ARGS__; }                          \
  else if ((Krt) <= 16) { constexpr int KB = 16; __VA_ARGS__; }                        \
  else if ((Krt) <= 32) { constexpr int KB = 32; __VA_ARGS__; }                        \
  else if ((Krt) <= 64) { constexpr int KB = 64; __VA_ARGS__; }                        \
  else { set_error("K=%d outside the supported 1..64", (int)(Krt)); return FM_EINVAL; }

// padded channel count of the fused statistics passes (fm_fused.cuh)
#define FM_DISPATCH_MP(Mrt, ...)                                               \
  if ((Mrt) <= 4) { constexpr int MP = 4; __VA_ARGS__; }                               \
  else if ((Mrt) <= 8) { constexpr int MP = 8; __VA_ARGS__; }                          \
  else { constexpr int MP = 16; __VA_ARGS__; }

#define FM_DISPATCH_IT(ITrt, ...)                                              \
  if ((ITrt) <= 1) { constexpr int IT = 1; __VA_ARGS__; }                              \
  else if ((ITrt) <= 2) { constexpr int IT = 2; __VA_ARGS__; }                         \
  else if ((ITrt) <= 4) { constexpr int IT = 4; __VA_ARGS__; }                         \
  else { constexpr int IT = 8; __VA_ARGS__; }

// The device's default stream-ordered pool returns freed blocks to the OS at
// every synchronisation (release threshold 0), so a per-call
// cudaMallocAsync / cudaFreeAsync re-maps memory each time; keep it mapped.
inline void keep_pool_mapped() {
  static thread_local int done_dev = -1;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev == done_dev) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done_dev = dev;
}

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// Launch with programmatic stream serialisation (PDL): the kernel may begin
// launching while its predecessor drains; it waits in pdl_entry() before
// touching the predecessor's outputs. Works inside CUDA-graph capture.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// Workspace plan for the fused iteration.
struct Plan {
  int FT, TT;    // k_wstats bins per CTA, k_hstats frames per CTA
  int HS, HFR;   // k_hstats bin splits and bins per split
  int TR, nseg;  // k_gain (and k_vacc/k_vacc_tc) frames per CTA segment, segments per bin
  int VTR, vnseg;  // V accumulation segments (k_ip reduces vnseg partials per bin)
  int ntile;       // k_back frame tiles per bin (data-term partials per bin)
  size_t off_lam, off_phi, off_gpart, off_vpart, off_gnew, off_llp, off_ldp, off_cs, off_hpart;
  size_t off_vmu;  // FastMNMF-DP V-step split partials (B, VMU_FS, 2, T)
  // fused statistics passes (plain FastMNMF; fm_fused.cuh)
  int FB, nfb;            // bins per CTA, bin blocks
  int gTR, gseg;          // k_gpass frames per segment, segments
  int bTR, bseg, bIT;     // k_bpass frames per segment, segments, items per lane
  int hHS, hHFR, hNS, hNG, hIT, htl;  // k_hpass bin splits, bins per split, sources per
                                      // CTA, source groups, items per thread, T tiles
  size_t smem_g, smem_b, smem_h;
  int gS, bS, hS;  // cp.async pipeline stages of k_gpass, k_bpass, k_hpass
  size_t off_wn, off_wpart, off_hpart2, off_ht;
  size_t off_cnt, off_hcnt, off_vcnt, off_bcnt, off_hcnt2, total;
};

// complex64 V accumulation: 0 register-blocked SIMT (k_vacc_blk), 1
// pair-per-thread SIMT (k_vacc), 2 tensor cores (k_vacc_tc, even M in 10..16).
// FM_VACC=blk|simt|tc forces one for A/B runs; read at every launch (or graph
// capture) so tests can switch it within one process.
inline int vacc_mode(const fm_dims* d) {
  const bool tc_ok = d->M >= 10 && d->M % 2 == 0;
  const char* e = getenv("FM_VACC");
  if (e && strcmp(e, "simt") == 0) return 1;
  if (e && strcmp(e, "tc") == 0) return tc_ok ? 2 : 1;
  if (e && strcmp(e, "blk") == 0) return 0;
  const bool p_ok = d->dtype == FM_F32 && d->M >= 5 && d->M <= 8;
  if (e && strcmp(e, "p") == 0) return p_ok ? 3 : 1;
  // measured on B200: pair-per-thread wins at M = 4 (c2: 1.13 vs 1.89 ms) and
  // M = 8 (c1: 39.1 vs 40.8 us); at M = 16 (c3) the tensor cores (1.06 ms)
  // beat the blocked kernel (2.00 ms) and pair-per-thread (4.67 ms)
  if (d->M > 8) return tc_ok ? 2 : 0;
  return 1;
}

// k_vacc_p knobs (A/B runs): frames per chunk (128 | 256) and CTAs per SM
inline int vp_tb() {
  const char* e = getenv("FM_VP_TB");
  return (e && atoi(e) == 128) ? 128 : 256;
}
inline int vp_ctas_per_sm() {
  const char* e = getenv("FM_VP_CTAS");
  const int v = e ? atoi(e) : 0;
  return (v >= 1 && v <= 8) ? v : 0;
}

// complex64, M > 8: the projection on the tensor cores (k_back_tc);
// FM_BACK=simt forces the SIMT k_back (A/B runs, tests)
inline bool back_tc_mode() {
  const char* e = getenv("FM_BACK");
  return !(e && strcmp(e, "simt") == 0);
}

// lambda = W H on the tensor cores (k_lambda_tc): complex64, K a multiple of 8 up
// to 32, >= 2^24 lambda entries (config 3); FM_LAMBDA=simt|tc forces either
inline bool lambda_tc_mode(const fm_dims* d, int n0) {
  if (d->dtype != FM_F32 || d->K % 8 != 0 || d->K > 32) return false;
  const char* e = getenv("FM_LAMBDA");
  if (e && strcmp(e, "simt") == 0) return false;
  if (e && strcmp(e, "tc") == 0) return true;
  return d->B * (d->N - n0) * d->F * d->T >= (1LL << 24);
}
inline bool back_tc_forced() {  // FM_BACK=tc: also for M in 5..8 (A/B runs)
  const char* e = getenv("FM_BACK");
  return e && strcmp(e, "tc") == 0;
}

// FM_GSEG: segment-count tuning knob (A/B runs); read at every plan
inline int gseg_override() {
  const char* e = getenv("FM_GSEG");
  return e ? atoi(e) : 0;
}

// Schedule of the plain iteration (fastmnmf.h FM_SCHED_*):
//   split  ten launches, the register-tiled NMF contractions separate
//   fused  five statistics passes with on-chip lambda (FM_SCHEDULE=fused, §4a)
//   bin    k_hstats + the per-bin kernel k_binw + k_trace (fm_bin.cuh, §4c):
//          complex64, M <= 4, N in 2..4, K <= 8, H of a mixture in shared memory
// FM_SCHEDULE=split|fused|bin forces one (bin only where it is eligible); the
// default is bin for eligible shapes with >= FM_BIN_MIN_BINS (bin, mixture) pairs.
constexpr long long FM_BIN_MIN_BINS = 4096;  // measured: 8 mixtures x 513 bins already win (5177 vs 4309 it/s)
inline bool bin_eligible(const fm_dims* d) {
  if (d->dtype != FM_F32 || d->dp || d->M > 4 || d->N < 2 || d->N > 4 || d->K > 8) return false;
  const long long hs = d->N * 8LL * d->T * 4LL;  // staged H (KK = 8 rows per source)
  return hs + 8LL * 4096 <= 200LL * 1024;
}
inline int schedule_of(const fm_dims* d) {
  const char* e = getenv("FM_SCHEDULE");
  if (e && strcmp(e, "fused") == 0) return FM_SCHED_FUSED;
  if (e && strcmp(e, "split") == 0) return FM_SCHED_SPLIT;
  if (e && strcmp(e, "bin") == 0) return bin_eligible(d) ? FM_SCHED_BIN : FM_SCHED_SPLIT;
  // default: one warp per bin once the batch gives every SM a few CTAs of bins
  // (config 2 shape: 8 mixtures 5177 vs 4309 iterations/s, 64: 809 vs 637,
  // 256: 228 vs 163); the split schedule's (bin, frame-tile) CTAs otherwise
  if (bin_eligible(d) && d->B * d->F >= FM_BIN_MIN_BINS) return FM_SCHED_BIN;
  return FM_SCHED_SPLIT;
}
inline bool use_fused(const fm_dims* d) { return schedule_of(d) == FM_SCHED_FUSED; }
inline bool use_bin(const fm_dims* d) { return !d->dp && schedule_of(d) == FM_SCHED_BIN; }

// M <= 4: register-accumulating gain / V kernels (fm_small.cuh) with
// FM_SMALL=1 (measured slower than the staged ones at config 2; A/B runs)
inline bool small_m_mode() {
  const char* e = getenv("FM_SMALL");
  return e && strcmp(e, "1") == 0;
}

// IP kernel: one warp per bin (k_ip_w, M <= 8) for many bins, the multi-warp
// k_ip otherwise; FM_IP=w|cta forces one (A/B runs, tests)
inline bool ip_warp_mode(const fm_dims* d) {
  const char* e = getenv("FM_IP");
  if (e && strcmp(e, "w") == 0) return d->M <= 8;
  if (e && strcmp(e, "cta") == 0) return false;
  return d->M <= 8 && d->B * d->F >= 4 * 148 * 4;
}

// FM_PASS_CTAS / FM_PASS_S: work-split and pipeline-depth knobs of the fused
// statistics passes (A/B runs); read at every plan
inline int pass_ctas_override() {
  const char* e = getenv("FM_PASS_CTAS");
  return e ? atoi(e) : 0;
}
inline int pass_stages_override() {
  const char* e = getenv("FM_PASS_S");
  const int v = e ? atoi(e) : 0;
  return v < 2 ? 0 : v > 4 ? 4 : v;
}

// Everything outside fm_dims that changes which kernels an iteration
// launches: part of the CUDA-graph cache key (fm_api.cu run_common).
inline unsigned long long variant_key(const fm_dims* d) {
  const unsigned lo = (unsigned)vacc_mode(d) | ((unsigned)(gseg_override() & 0xff) << 4) |
         ((unsigned)(pass_ctas_override() & 0xfff) << 12) | ((unsigned)pass_stages_override() << 26) |
         ((unsigned)use_fused(d) << 31) | ((unsigned)ip_warp_mode(d) << 3) |
         ((unsigned)use_bin(d) << 30) |
         ((unsigned)small_m_mode() << 2) | ((unsigned)back_tc_mode() << 29) |
         ((unsigned)back_tc_forced() << 25) | ((unsigned)lambda_tc_mode(d, d->dp ? 1 : 0) << 24);
  // k_vacc_p knobs (chunk size, CTAs per SM) above the 32 selection bits
  return (unsigned long long)lo | ((unsigned long long)(vp_tb() == 128) << 32) |
         ((unsigned long long)vp_ctas_per_sm() << 33);
}

inline Plan make_plan(const fm_dims* d) {
  Plan p;
  const size_t rs = d->dtype == FM_F64 ? 8 : 4;
  const long long B = d->B, F = d->F, T = d->T, N = d->N, M = d->M;
  const long long target = 2 * 148;  // >= 2 CTAs per SM
  // largest tile that still gives ~2 CTAs per SM
  {  // k_back frame tiles per bin (data-term partials per bin)
    const long long fr = 256 * back_ppt(M, T);
    p.ntile = (int)((T + fr - 1) / fr);
  }
  p.FT = 32;
  while (p.FT > 8 && ((F + p.FT - 1) / p.FT) * B * N < target) p.FT /= 2;
  p.TT = 64;
  while (p.TT > 16 && ((T + p.TT - 1) / p.TT) * B * N < target) p.TT /= 2;
  // k_hstats bin splits: fill the SMs when T-tiles x sources are few (each
  // split keeps >= 64 bins, a multiple of the 32-bin staging chunk)
  const long long htiles = ((T + p.TT - 1) / p.TT) * B * N;
  long long hs = std::max<long long>(1, (target + htiles - 1) / htiles);
  hs = std::min<long long>(hs, std::max<long long>(1, F / 64));
  p.HFR = (int)((((F + hs - 1) / hs) + 31) / 32 * 32);
  p.HS = (int)((F + p.HFR - 1) / p.HFR);
  // k_gain / k_vacc: segments per bin so that bins x segments >= ~4 CTAs per SM,
  // each segment a multiple of 256 frames (the fp32 chunk; 64/128 divide it)
  long long segs = std::max<long long>(1, (4 * 148 + F * B - 1) / (F * B));
  const int seg_override = gseg_override();
  if (seg_override > 0) segs = seg_override;
  long long tr = (T + segs - 1) / segs;
  tr = ((tr + 255) / 256) * 256;
  p.TR = (int)std::min<long long>(tr, std::max<long long>(T, 1));
  if (p.TR < 256) p.TR = 256;
  p.nseg = (int)((T + p.TR - 1) / p.TR);
  const size_t gpart = (size_t)B * F * p.nseg * N * 2 * M;
  p.VTR = p.TR;
  p.vnseg = p.nseg;
  if (d->dtype == FM_F32 && vacc_mode(d) == 0) {
    // k_vacc_blk: long frame runs per thread amortise the slice tree; enough
    // (bin, segment) CTAs for ~3/4 of the resident slots (VbCfg: 128-thread
    // CTAs, 4 per SM, for M <= 8; one 512-thread CTA per SM above)
    const long long tbv = vb_chunk((int)M), slots = (M > 8 ? 1 : 4) * 148 * 3 / 4;
    const long long vs = std::max<long long>(1, (slots + F * B - 1) / (F * B));
    long long vtr = (T + vs - 1) / vs;
    vtr = std::max<long long>(tbv, (vtr + tbv - 1) / tbv * tbv);
    p.VTR = (int)vtr;
    p.vnseg = (int)((T + vtr - 1) / vtr);
  }
  if (d->dtype == FM_F32 && vacc_mode(d) == 2) {
    // k_vacc_tc: two CTAs per SM; segments of whole 128-frame blocks, at least
    // eight blocks each, until the (bin, segment) CTAs make ~6 waves
    const long long slots = 2 * 148, blocks = (T + 127) / 128;
    long long vs = std::max<long long>(1, (6 * slots + F * B - 1) / (F * B));
    vs = std::max<long long>(1, std::min(vs, blocks / 8));
    const long long vtr = (blocks + vs - 1) / vs * 128;
    p.VTR = (int)vtr;
    p.vnseg = (int)((T + vtr - 1) / vtr);
  }
  if (d->dtype == FM_F32 && vacc_mode(d) == 3) {  // k_vacc_p: one chunk per item
    p.VTR = vp_tb();
    p.vnseg = (int)((T + p.VTR - 1) / p.VTR);
  }
  const size_t vpart = (size_t)B * F * p.vnseg * M * (M * (M + 1) / 2) * 2;
  // ---- fused passes: bins per CTA (8 warps; fewer where fp64 rows overflow
  // shared memory), segments for >= ~3 CTAs per SM
  {
    const int K = (int)d->K, K4 = k4_of(K), KQ = K4 / 4;
    const int MPv = M <= 4 ? 4 : M <= 8 ? 8 : 16;
    p.FB = 8;
    // work split: enough CTAs that every SM holds several (FM_PASS_CTAS
    // overrides the target for A/B runs)
    const long long want = pass_ctas_override() > 0 ? pass_ctas_override() : 8 * 148;
    const long long chunks = (T + FTC - 1) / FTC;
    auto split = [&](int FB) {
      p.nfb = (int)((F + FB - 1) / FB);
      auto segs_for = [&](long long ctas, int& TRo, int& nsego) {
        long long sg = std::max<long long>(1, (want + ctas - 1) / ctas);
        sg = std::min(sg, chunks);
        const long long tr = (chunks + sg - 1) / sg * FTC;
        TRo = (int)tr;
        nsego = (int)((T + tr - 1) / tr);
      };
      segs_for((long long)p.nfb * B, p.gTR, p.gseg);
      segs_for((long long)p.nfb * B, p.bTR, p.bseg);
      p.htl = (int)chunks;
    };
    auto fit = [&](int FB, int& NS, int& NG, int& IT) {
      split(FB);
      // k_bpass: W-statistic items (source, bin pair, k-quad) per thread
      const long long NIb = N * ((FB + 1) / 2) * KQ;
      p.bIT = NIb <= 32 * FB ? 1 : (int)((NIb + 32 * FB - 1) / (32 * FB));
      p.bIT = p.bIT <= 1 ? 1 : p.bIT <= 2 ? 2 : 4;
      // k_hpass: (source, k chunk) items per thread, <= 4 (source groups beyond)
      const int KO = K4 / hp_kch(K4);
      NG = 1;
      NS = (int)N;
      IT = (NS * KO + FB - 1) / FB;
      while (IT > 4) {
        ++NG;
        NS = (int)((N + NG - 1) / NG);
        IT = (NS * KO + FB - 1) / FB;
      }
      IT = IT <= 1 ? 1 : IT <= 2 ? 2 : 4;
      const long long hct = chunks * B * NG;
      long long hs = std::max<long long>(1, (want + hct - 1) / hct);
      hs = std::min<long long>(hs, (F + FB - 1) / FB);
      p.hHFR = (int)(((F + hs - 1) / hs + FB - 1) / FB * FB);
      p.hHS = (int)((F + p.hHFR - 1) / p.hHFR);
      // cp.async stages: no deeper than the chunks (steps) a CTA walks, 2..4;
      // then the deepest that keeps >= 3 CTAs per SM (<= 72 KB), else 2, else 1
      auto pick = [&](auto total_of, int steps, int& S, size_t& bytes) {
        const int smax = (int)std::max<long long>(2, std::min<long long>(4, steps));
        const int so = pass_stages_override();
        for (size_t cap : {(size_t)72 * 1024, (size_t)112 * 1024, (size_t)200 * 1024}) {
          for (S = so ? so : smax; S >= 2; --S) {
            bytes = total_of(S);
            if (bytes <= cap) return true;
            if (so) break;
          }
        }
        S = 2;
        bytes = total_of(2);
        return false;
      };
      bool ok = pick([&](int S) { return GpLayout((int)rs, (int)N, K, (int)M, MPv, FB, S).total; },
                     p.gTR / FTC, p.gS, p.smem_g);
      ok = pick([&](int S) { return BpLayout((int)rs, (int)N, K, (int)M, MPv, FB, S).total; },
                p.bTR / FTC, p.bS, p.smem_b) && ok;
      ok = pick([&](int S) { return HpLayout((int)rs, (int)N, K, (int)M, MPv, FB, NS, S).total; },
                p.hHFR / FB, p.hS, p.smem_h) && ok;
      return ok;
    };
    while (p.FB > 1 && !fit(p.FB, p.hNS, p.hNG, p.hIT)) p.FB /= 2;
    fit(p.FB, p.hNS, p.hNG, p.hIT);
  }
  const size_t gpart_f = (size_t)B * F * p.gseg * N * 2 * M;
  size_t o = 0;
  p.off_lam = o; o = align256(o + (size_t)B * N * F * T * rs);
  p.off_phi = o; o = align256(o + (size_t)B * 2 * N * F * T * rs);
  p.off_gpart = o; o = align256(o + std::max<size_t>(gpart, gpart_f) * rs);
  p.off_vpart = o; o = align256(o + vpart * rs);
  p.off_gnew = o; o = align256(o + (size_t)B * N * F * M * rs);
  p.off_llp = o; o = align256(o + std::max<size_t>((size_t)B * F * p.ntile, (size_t)B * p.nfb * p.bseg) * 8);
  p.off_ldp = o; o = align256(o + (size_t)B * F * 8);
  p.off_cs = o; o = align256(o + (size_t)B * F * NMAX * rs);
  p.off_hpart = o; o = align256(o + (size_t)htiles * p.HS * 2 * 64 * 64 * rs);
  p.off_vmu = o; o = align256(o + (size_t)B * VMU_FS * 2 * T * rs);
  {
    const size_t K4 = (size_t)k4_of((int)d->K);
    p.off_wn = o; o = align256(o + (size_t)B * N * F * d->K * rs);
    p.off_ht = o; o = align256(o + (size_t)B * N * T * K4 * rs);
    p.off_wpart = o; o = align256(o + (size_t)B * F * p.bseg * 2 * N * K4 * rs);
    p.off_hpart2 = o;
    if (p.hHS > 1)
      o = align256(o + (size_t)p.htl * B * p.hNG * p.hHS * 2 * p.hNS * K4 * FTC * rs);
  }
  p.off_cnt = o; o = align256(o + 64);
  p.off_hcnt = o; o = align256(o + (size_t)htiles * 4);
  p.off_vcnt = o; o = align256(o + (size_t)B * ((T + 31) / 32) * 4);  // k_dp_vmu tile counters
  p.off_bcnt = o; o = align256(o + (size_t)B * p.nfb * 4);
  p.off_hcnt2 = o; o = align256(o + (size_t)p.htl * B * p.hNG * 4);
  p.total = o;
  return p;
}

#define FM_DISPATCH_TILE(X, NAME, ...)                                           \
  switch (X) {                                                                   \
    case 8: { constexpr int NAME = 8; __VA_ARGS__; } break;                     \
    case 16: { constexpr int NAME = 16; __VA_ARGS__; } break;                   \
    case 32: { constexpr int NAME = 32; __VA_ARGS__; } break;                   \
    case 64: { constexpr int NAME = 64; __VA_ARGS__; } break;                   \
    default: set_error("tile %d", (int)(X)); return FM_EINVAL;                  \
  }

int validate_dims(const fm_dims* d);

template <typename R> struct Impl {
  using C = cplx<R>;

  static int prologue(const fm_dims* d, const fm_state* s, cudaStream_t st, bool reset = true);
  static int iterate_phase(const fm_dims* d, const fm_state* s, int phase, void* hstat,
                           cudaStream_t st, cudaEvent_t* ev = nullptr);  // ev: 11 / 7 events
  static int iterate_split(const fm_dims* d, const fm_state* s, int phase, void* hstat,
                           cudaStream_t st, cudaEvent_t* ev);
  static int iterate_fused(const fm_dims* d, const fm_state* s, int phase, void* hstat,
                           cudaStream_t st, cudaEvent_t* ev);
  static int iterate_bin(const fm_dims* d, const fm_state* s, int phase, void* hstat,
                         cudaStream_t st, cudaEvent_t* ev);
  static int prologue_bin(const fm_dims* d, const fm_state* s, cudaStream_t st);
  static int binw(const fm_dims* d, const fm_state* s, cudaStream_t st);
  static int hstats(const fm_dims* d, const fm_state* s, const R* Wsrc, int mode, void* hstat,
                    cudaStream_t st);
  static int lambda(const fm_dims* d, const R* W, const R* H, R* lam, cudaStream_t st);
  static int gain(const fm_dims* d, const fm_state* s, cudaStream_t st);
  static int vacc(const fm_dims* d, const fm_state* s, cudaStream_t st);
  static int ip(const fm_dims* d, const fm_state* s, cudaStream_t st, R* u = nullptr);
  static int lambda_nmf(const fm_dims* d, const fm_state* s, cudaStream_t st);
  static int phi_pass(const fm_dims* d, const fm_state* s, cudaStream_t st);
  static int dp_latent(const fm_dims* d, const fm_state* s, const fm_dp* p, int steps, cudaStream_t st);
  static int dp_mh(const fm_dims* d, const fm_state* s, const fm_dp* p, int steps, cudaStream_t st);
  static int dp_lambda(const fm_dims* d, const fm_state* s, const fm_dp* p, cudaStream_t st);
  static int prologue_dp(const fm_dims* d, const fm_state* s, const fm_dp* p, cudaStream_t st);
  static int iterate_dp(const fm_dims* d, const fm_state* s, const fm_dp* p, cudaStream_t st,
                        cudaEvent_t* ev = nullptr);  // ev: DP_NEV events
  static int back(const fm_dims* d, const fm_state* s, int tail_only, int record, cudaStream_t st);
  static int hpass(const fm_dims* d, const fm_state* s, int mode, void* hout, cudaStream_t st);
  static int gpass(const fm_dims* d, const fm_state* s, cudaStream_t st);
  static int bpass(const fm_dims* d, const fm_state* s, cudaStream_t st);
  static int trace(const fm_dims* d, const fm_state* s, cudaStream_t st);
  static int hstore(const fm_dims* d, const fm_state* s, const void* hbuf, cudaStream_t st);

  static int fast_stats(int64_t F, int64_t T, int64_t M, int64_t N, const void* xt,
                        const void* g, const void* lam, double floor, int want_gain,
                        int want_phi, void* phi1, void* phi2, void* gnum, void* gden,
                        double* ll_host, cudaStream_t st);
  static int mix_power(int64_t N, int64_t F, int64_t T, int64_t M, const void* lam,
                       const void* g, double floor, void* y, cudaStream_t st);
  static int ip_weights(int64_t F, int64_t T, int64_t M, const void* X, const void* y, void* V,
                        cudaStream_t st);
  static int project(int64_t F, int64_t T, int64_t M, const void* Q, const void* X, void* xt,
                     cudaStream_t st);
  static int update_diagonalizer(int64_t F, int64_t T, int64_t M, void* Q, const void* X,
                                 const void* y, int sweeps, uint64_t* status, cudaStream_t st);
  static int logdet(int64_t F, int64_t M, const void* Q, double* out, cudaStream_t st);
  static int wiener(int64_t N, int64_t F, int64_t T, int64_t M, const void* lam, const void* Q,
                    const void* g, const void* X, void* out, uint64_t* status, cudaStream_t st);
  static int obs_stats(const fm_dims* d, const void* X, double* sumsq, double* maxsq,
                       cudaStream_t st);
  static int scale(const fm_dims* d, void* X, const double* scale_host, cudaStream_t st);
  static int spatial_init(const fm_dims* d, const void* X, void* Q, double* w, cudaStream_t st);
  static int stft(int64_t n, int64_t M, int64_t L, int64_t hop, const void* wave, void* spec,
                  cudaStream_t st);
  static int fr_stats(int64_t F, int64_t T, int64_t M, int64_t N, const void* X, const void* G,
                      const void* lam, double ridge, int want_ab, int want_phi, void* phi, void* A,
                      void* B, void* work, double* ll, cudaStream_t st);
  static int fr_scm(int64_t N, int64_t F, int64_t M, void* G, const void* A, const void* B,
                    int normalize, void* c, uint64_t* status, cudaStream_t st);
  static int fr_wiener(int64_t N, int64_t F, int64_t T, int64_t M, const void* lam, const void* G,
                       const void* X, double ridge, void* out, uint64_t* status, cudaStream_t st);
  static int fr_nmf_mu(int64_t N, int64_t F, int64_t T, int64_t K, const void* phi, void* W, void* H,
                       int step, cudaStream_t st);
  static int fr_absorb(int64_t N, int64_t F, int64_t K, void* W, const void* c, cudaStream_t st);
  static int fr_reconstruct(int64_t N, int64_t F, int64_t M, const void* Q, const void* g, void* G,
                            uint64_t* status, cudaStream_t st);
  static int istft(int64_t T, int64_t M, int64_t L, int64_t hop, int64_t length, const void* spec,
                   void* work, void* out, cudaStream_t st);
};

template <typename Kern>
inline int ensure_smem(Kern k, size_t bytes) {
  if (bytes + 4096 > 48 * 1024) {  // dynamic + static smem above the default 48 KB
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) {
      set_error("cudaFuncSetAttribute(%zu B smem): %s", bytes, cudaGetErrorString(e));
      return FM_ECUDA;
    }
  }
  return FM_OK;
}

template <typename R>
int Impl<R>::lambda(const fm_dims* d, const R* W, const R* H, R* lam, cudaStream_t st) {
  const int n0 = d->dp ? 1 : 0;
  if constexpr (sizeof(R) == 4) {
    if (lambda_tc_mode(d, n0)) {  // tensor cores: large problems, K in {8, 16, 24, 32}
      const long long tt = (d->T + 127) / 128, bn = d->B * (d->N - n0);
      long long fg = std::max<long long>(1, (6LL * 4 * 148 + tt * bn - 1) / (tt * bn));
      long long fpg = ((d->F + fg - 1) / fg + LTC_FT - 1) / LTC_FT * LTC_FT;
      fg = (d->F + fpg - 1) / fpg;
      launch_pdl(k_lambda_tc, dim3((unsigned)tt, (unsigned)fg, (unsigned)bn), dim3(128), 0, st, W, H,
                 lam, (int)d->F, (int)d->T, (int)d->K, (int)d->N, n0, (int)fpg);
      FM_CHECK_LAUNCH("k_lambda_tc");
      return FM_OK;
    }
  }
  dim3 grid((unsigned)((d->T + 63) / 64), (unsigned)((d->F + 63) / 64),
            (unsigned)(d->B * (d->N - n0)));
  launch_pdl(k_lambda<R>, grid, dim3(256), 0, st, W, H, lam, (int)d->F, (int)d->T, (int)d->K,
             (int)d->N, n0);
  FM_CHECK_LAUNCH("k_lambda");
  return FM_OK;
}

template <typename R>
int Impl<R>::gain(const fm_dims* d, const fm_state* s, cudaStream_t st) {
  const Plan p = make_plan(d);
  unsigned char* w = reinterpret_cast<unsigned char*>(s->work);
  GainArgs<R> a;
  a.xt = reinterpret_cast<const R*>(s->xt);
  a.lam = reinterpret_cast<const R*>(w + p.off_lam);
  a.g = reinterpret_cast<const R*>(s->g);
  a.floorp = reinterpret_cast<const R*>(s->floor);
  a.part = reinterpret_cast<R*>(w + p.off_gpart);
  a.F = (int)d->F; a.T = (int)d->T; a.N = (int)d->N; a.TR = p.TR;
  dim3 grid((unsigned)p.nseg, (unsigned)d->F, (unsigned)d->B);
  FM_DISPATCH_M(d->M, {
    if constexpr (MM <= 4) {  // register-accumulating, four bins per CTA (fm_small.cuh)
      if (small_m_mode()) {
        launch_pdl(k_gain_r<R, MM>, dim3((unsigned)p.nseg, (unsigned)((d->F + SMALL_BPB - 1) / SMALL_BPB),
                                         (unsigned)d->B),
                   dim3(SMALL_BS), 0, st, a);
        FM_CHECK_LAUNCH("k_gain_r");
        return FM_OK;
      }
    }
    launch_pdl(k_gain<R, MM>, grid, dim3(256), 0, st, a);
    FM_CHECK_LAUNCH("k_gain");
  });
  return FM_OK;
}

template <typename R>
int Impl<R>::vacc(const fm_dims* d, const fm_state* s, cudaStream_t st) {
  const Plan p = make_plan(d);
  unsigned char* w = reinterpret_cast<unsigned char*>(s->work);
  VaccArgs<R> a;
  a.X = reinterpret_cast<const C*>(s->X);
  a.lam = reinterpret_cast<const R*>(w + p.off_lam);
  a.g = reinterpret_cast<const R*>(s->g);
  a.gpart = reinterpret_cast<const R*>(w + p.off_gpart);
  a.floorp = reinterpret_cast<const R*>(s->floor);
  a.gnew = reinterpret_cast<R*>(w + p.off_gnew);
  a.part = reinterpret_cast<R*>(w + p.off_vpart);
  a.F = (int)d->F; a.T = (int)d->T; a.N = (int)d->N; a.TR = p.TR;
  a.gseg = (d->dp || !use_fused(d)) ? p.nseg : p.gseg;  // k_gain or k_gpass partials
  static const int dbg = [] { const char* e = getenv("FM_VTC_DBG"); return e ? atoi(e) : 0; }();
  a.dbg = dbg;
  dim3 grid((unsigned)p.nseg, (unsigned)d->F, (unsigned)d->B);
  const int mode = vacc_mode(d);
  FM_DISPATCH_M(d->M, {
    if constexpr (sizeof(R) == 4) {
      if constexpr (MM >= 10 && MM % 2 == 0) {
        if (mode == 2) {
          if (reinterpret_cast<uintptr_t>(s->X) & 15) {  // the bulk copies of X blocks
            set_error("k_vacc_tc: X must be 16-byte aligned");
            return FM_EINVAL;
          }
          const size_t smv = VtcCfg<MM>::SMEM;
          if (int rc = ensure_smem(k_vacc_tc<MM>, smv)) return rc;
          VaccArgs<float> at = *reinterpret_cast<VaccArgs<float>*>(&a);
          at.TR = p.VTR;
          launch_pdl(k_vacc_tc<MM>, dim3((unsigned)p.vnseg, (unsigned)d->F, (unsigned)d->B),
                     dim3(VtcCfg<MM>::BS), smv, st, at);
          FM_CHECK_LAUNCH("k_vacc_tc");
          return FM_OK;
        }
      }
      if constexpr (MM >= 5 && MM <= 8) {
        if (mode == 3) {
          VaccArgs<float> ap = *reinterpret_cast<VaccArgs<float>*>(&a);
          ap.TR = p.VTR;
          const long long items = (long long)d->B * d->F * p.vnseg;
          if (items >= (1ll << 31) || d->B * d->F >= (1ll << 31)) {
            set_error("k_vacc_p: too many (bin, chunk) items");
            return FM_EINVAL;
          }
          auto go = [&](auto kern, size_t smv, int minb) -> int {
            if (int rc = ensure_smem(kern, smv)) return rc;
            const int per_sm = vp_ctas_per_sm() ? vp_ctas_per_sm() : minb;
            const long long G = std::min<long long>(items, 148LL * per_sm);
            launch_pdl(kern, dim3((unsigned)G), dim3(256), smv, st, ap, p.vnseg, (int)items);
            return FM_OK;
          };
          int rc;
          if (p.VTR == 128) rc = go(k_vacc_p<MM, 128>, VpCfg<MM, 128>::SMEM, VpCfg<MM, 128>::MINB);
          else rc = go(k_vacc_p<MM, 256>, VpCfg<MM, 256>::SMEM, VpCfg<MM, 256>::MINB);
          if (rc) return rc;
          FM_CHECK_LAUNCH("k_vacc_p");
          return FM_OK;
        }
      }
      if (mode == 0) {
        const size_t smb = VbCfg<MM>::SMEM;
        if (int rc = ensure_smem(k_vacc_blk<MM>, smb)) return rc;
        VaccArgs<float> ab = *reinterpret_cast<VaccArgs<float>*>(&a);
        ab.TR = p.VTR;
        launch_pdl(k_vacc_blk<MM>, dim3((unsigned)p.vnseg, (unsigned)d->F, (unsigned)d->B),
                   dim3(VbCfg<MM>::BS), smb, st, ab);
        FM_CHECK_LAUNCH("k_vacc_blk");
        return FM_OK;
      }
    }
    if constexpr (MM <= 4) {  // register-accumulating, four bins per CTA (fm_small.cuh)
      if (small_m_mode()) {
        launch_pdl(k_vacc_r<R, MM>, dim3((unsigned)p.nseg, (unsigned)((d->F + SMALL_BPB - 1) / SMALL_BPB),
                                         (unsigned)d->B),
                   dim3(SMALL_BS), 0, st, a);
        FM_CHECK_LAUNCH("k_vacc_r");
        return FM_OK;
      }
    }
    launch_pdl(k_vacc<R, MM>, grid, dim3(VaCfg<R, MM>::BS), 0, st, a);
    FM_CHECK_LAUNCH("k_vacc");
  });
  return FM_OK;
}

template <typename R>
int Impl<R>::ip(const fm_dims* d, const fm_state* s, cudaStream_t st, R* u) {
  const Plan p = make_plan(d);
  unsigned char* w = reinterpret_cast<unsigned char*>(s->work);
  IpArgs<R> a;
  a.Vpart = reinterpret_cast<const C*>(w + p.off_vpart);
  a.nseg = p.vnseg;
  a.T = (int)d->T;
  a.gnew = reinterpret_cast<const R*>(w + p.off_gnew);
  a.Q = reinterpret_cast<C*>(s->Q);
  a.g = reinterpret_cast<R*>(s->g);
  a.W = reinterpret_cast<R*>(s->W);
  // plain FastMNMF: the W-stepped Wn (k_bpass) is absorbed into the state W
  a.Wsrc = (d->dp || !use_fused(d)) ? a.W : reinterpret_cast<const R*>(w + p.off_wn);
  a.cs_out = reinterpret_cast<R*>(w + p.off_cs);
  a.ld_part = reinterpret_cast<double*>(w + p.off_ldp);
  a.iter = reinterpret_cast<const unsigned*>(w + p.off_cnt) + 1;
  a.status = reinterpret_cast<unsigned long long*>(s->status);
  a.F = (int)d->F; a.N = (int)d->N; a.K = (int)d->K;
  a.n0 = d->dp ? 1 : 0;
  a.u = u;
  a.f_offset = d->f_offset;
  a.normalize = d->normalize;
  a.ip_sweeps = d->ip_sweeps;
  a.B = (int)d->B;
  dim3 grid((unsigned)d->F, (unsigned)d->B);
  FM_DISPATCH_M(d->M, {
    // many bins (batches): one warp per bin (fm_ipw.cuh) -- c2 k_ip 1.20 ->
    // 0.53 ms; few bins: the multi-warp k_ip, whose per-bin chain is shorter
    // (c1: 24.6 vs 36.9 us)
    if constexpr (MM <= 8) {
      if (ip_warp_mode(d)) {
        const size_t sm = IpwSmem<R, MM>::bytes * IPW_WARPS;
        if (int rc = ensure_smem(k_ip_w<R, MM>, sm)) return rc;
        const long long nb = d->B * d->F;
        launch_pdl(k_ip_w<R, MM>, dim3((unsigned)((nb + IPW_WARPS - 1) / IPW_WARPS)),
                   dim3(32 * IPW_WARPS), sm, st, a);
        FM_CHECK_LAUNCH("k_ip_w");
        return FM_OK;
      }
    }
    {
      const size_t sm = IpSmem<R, MM>::bytes;
      if (int rc = ensure_smem(k_ip<R, MM>, sm)) return rc;
      launch_pdl(k_ip<R, MM>, grid, dim3(IpCfg<MM>::BS), sm, st, a);
      FM_CHECK_LAUNCH("k_ip");
    }
  });
  return FM_OK;
}

template <typename R>
int Impl<R>::back(const fm_dims* d, const fm_state* s, int tail_only, int record,
                  cudaStream_t st) {
  const Plan p = make_plan(d);
  unsigned char* w = reinterpret_cast<unsigned char*>(s->work);
  BackArgs<R> a;
  a.X = reinterpret_cast<const C*>(s->X);
  a.xt = reinterpret_cast<R*>(s->xt);
  a.Q = reinterpret_cast<const C*>(s->Q);
  a.g = reinterpret_cast<const R*>(s->g);
  a.lam = reinterpret_cast<const R*>(w + p.off_lam);
  a.cs = tail_only ? nullptr : reinterpret_cast<const R*>(w + p.off_cs);
  a.phi = reinterpret_cast<R*>(w + p.off_phi);
  a.floorp = reinterpret_cast<const R*>(s->floor);
  a.ll_part = reinterpret_cast<double*>(w + p.off_llp);
  a.ld_part = reinterpret_cast<const double*>(w + p.off_ldp);
  a.trace = s->trace;
  a.counter = reinterpret_cast<unsigned*>(w + p.off_cnt);
  a.iter = a.counter + 1;
  a.B = (int)d->B; a.F = (int)d->F; a.T = (int)d->T; a.N = (int)d->N;
  a.record = record && s->trace != nullptr;
  FM_DISPATCH_M(d->M, {
    const int ppt = back_ppt(d->M, d->T);
    const dim3 grid((unsigned)((d->T + 256 * ppt - 1) / (256 * ppt)), (unsigned)d->F, (unsigned)d->B);
    if constexpr (MM <= 4) {
      if (ppt == 2) launch_pdl(k_back<R, MM, 2>, grid, dim3(256), 0, st, a);
      else launch_pdl(k_back<R, MM, 1>, grid, dim3(256), 0, st, a);
    } else {
      bool done = false;
      if constexpr (sizeof(R) == 4 && MM > 4) {
        if (back_tc_mode() && (MM > 8 || back_tc_forced())) {  // tensor-core projection; segments of whole 256-frame tiles
          const long long ctas = 6LL * 4 * 148, fb = (long long)d->F * d->B;
          long long ns = std::max<long long>(1, std::min<long long>(p.ntile, (ctas + fb - 1) / fb));
          const int TRb = (int)((p.ntile + ns - 1) / ns) * 256;
          const dim3 gridt((unsigned)((d->T + TRb - 1) / TRb), (unsigned)d->F, (unsigned)d->B);
          launch_pdl(k_back_tc<MM>, gridt, dim3(128), 0, st, a, TRb, p.ntile);
          done = true;
        }
      }
      if (!done) launch_pdl(k_back<R, MM, 1>, grid, dim3(256), 0, st, a);
    }
    FM_CHECK_LAUNCH("k_back");
  });
  return FM_OK;
}

// trace entry of the state after this iteration, then the device iteration
// counter (k_trace; a separate advance when B > 1)
template <typename R>
int Impl<R>::trace(const fm_dims* d, const fm_state* s, cudaStream_t st) {
  const Plan p = make_plan(d);
  unsigned char* w = reinterpret_cast<unsigned char*>(s->work);
  unsigned* itp = reinterpret_cast<unsigned*>(w + p.off_cnt) + 1;
  // data-term partials: (B, F, ntile) from k_back (deep prior), (B, nfb, bseg)
  // from k_bpass
  const bool fz = !d->dp && use_fused(d);
  const int np1 = fz ? p.nfb : (int)d->F, np2 = fz ? p.bseg : p.ntile;
  launch_pdl(k_trace, dim3((unsigned)d->B), dim3(256), 0, st,
             reinterpret_cast<const double*>(w + p.off_llp),
             reinterpret_cast<const double*>(w + p.off_ldp), s->trace, itp, (int)d->B, np1, np2,
             (int)d->F, (int)d->T);
  FM_CHECK_LAUNCH("k_trace");
  if (d->B > 1) {
    launch_pdl(k_iter_advance, dim3(1), dim3(1), 0, st, itp);
    FM_CHECK_LAUNCH("k_iter_advance");
  }
  return FM_OK;
}


template <typename R>
int Impl<R>::prologue(const fm_dims* d, const fm_state* s, cudaStream_t st, bool reset) {
  const Plan p = make_plan(d);
  unsigned char* w = reinterpret_cast<unsigned char*>(s->work);
  if (reset) FM_CUDA(cudaMemsetAsync(w + p.off_cnt, 0, p.total - p.off_cnt, st));
  if (use_bin(d)) return prologue_bin(d, s, st);
  if (!use_fused(d)) {  // split: lambda, then x~, data term and phi of the initial state
    if (int rc = lambda(d, reinterpret_cast<const R*>(s->W), reinterpret_cast<const R*>(s->H),
                        reinterpret_cast<R*>(w + p.off_lam), st))
      return rc;
    return back(d, s, /*tail_only=*/1, /*record=*/0, st);
  }
  // fused: Ht from H, then x~ of the initial Q, the data term of the initial
  // state and the first iteration's W step (separate.py:183, :186-193, :214-216)
  if (int rc = hstore(d, s, nullptr, st)) return rc;
  return bpass(d, s, st);
}

// The split schedule (ten launches; phi and lambda through HBM):
//   k_wstats  W step from the phi the previous k_back wrote  (separate.py:214-216 "W")
//   k_lambda, k_phi  refresh with the new W
//   k_hstats  H step                                        (separate.py:214-216 "H")
//   k_lambda  refresh with the new H
//   k_gain, k_vacc, k_ip  gains, V, IP, normalisations       (separate.py:217-233)
//   k_back    x~ = |Qx|^2, data term, phi for the next W step (separate.py:230; :186-193)
//   k_trace
template <typename R>
int Impl<R>::iterate_split(const fm_dims* d, const fm_state* s, int phase, void* hstat,
                           cudaStream_t st, cudaEvent_t* ev) {
#define FM_EV(i) \
  if (ev) FM_CUDA(cudaEventRecordWithFlags(ev[i], st, cudaEventRecordExternal));
  const Plan p = make_plan(d);
  unsigned char* w = reinterpret_cast<unsigned char*>(s->work);
  R* lam = reinterpret_cast<R*>(w + p.off_lam);
  R* phi = reinterpret_cast<R*>(w + p.off_phi);
  R* W = reinterpret_cast<R*>(s->W);
  R* H = reinterpret_cast<R*>(s->H);
  const int N = (int)d->N, F = (int)d->F, T = (int)d->T, K = (int)d->K;
  const int n0 = d->dp ? 1 : 0;
  const unsigned BN = (unsigned)(d->B * (d->N - n0));
  if (phase == 0 || phase == 2) {
    // W step (separate.py:214-216 with step "W"): statistics from the phi of the
    // previous pass, MU, then the refresh with the new W (lambda + phi)
    FM_EV(0);
    FM_DISPATCH_KB(K, {
      FM_DISPATCH_TILE(p.FT, FTT, {
        if constexpr (FTT <= 32) {
          const size_t smw = WsCfg<R, KB, FTT>::bytes;
          if (int rc = ensure_smem(k_wstats<R, KB, FTT>, smw)) return rc;
          launch_pdl(k_wstats<R, KB, FTT>, dim3((unsigned)((F + FTT - 1) / FTT), BN), dim3(256),
                     smw, st, phi, H, W, N, F, T, K, 0);
          FM_CHECK_LAUNCH("k_wstats");
        }
      });
    });
    FM_EV(1);
    if (int rc = lambda(d, W, H, lam, st)) return rc;
    FM_EV(2);
    FM_DISPATCH_M(d->M, {
      launch_pdl(k_phi<R, MM>, dim3((unsigned)((T + 255) / 256), (unsigned)F, (unsigned)d->B),
                 dim3(256), 0, st, lam, reinterpret_cast<const R*>(s->xt),
                 reinterpret_cast<const R*>(s->g), reinterpret_cast<const R*>(s->floor), phi, N, F,
                 T);
      FM_CHECK_LAUNCH("k_phi");
    });
    // H step (separate.py:214-216 with step "H")
    FM_EV(3);
    if (int rc = hstats(d, s, W, phase == 0 ? 1 : 0, hstat, st)) return rc;
  }
  if (phase == 0) return FM_OK;
  if (phase == 1) {
    const long long NKT = (long long)N * K * T, total = (long long)d->B * NKT;
    k_hupdate<R><<<(unsigned)((total + 255) / 256), 256, 0, st>>>(
        nullptr, H, reinterpret_cast<R*>(hstat), 1, NKT, total, 2);
    FM_CHECK_LAUNCH("k_hupdate");
  }
  FM_EV(4);
  if (int rc = lambda(d, W, H, lam, st)) return rc;  // refresh after the H step
  FM_EV(5);
  if (int rc = gain(d, s, st)) return rc;
  FM_EV(6);
  if (int rc = vacc(d, s, st)) return rc;
  FM_EV(7);
  if (int rc = ip(d, s, st)) return rc;
  FM_EV(8);
  if (int rc = back(d, s, /*tail_only=*/0, /*record=*/1, st)) return rc;
  FM_EV(9);
  if (int rc = trace(d, s, st)) return rc;  // trace entry, then the iteration counter
  FM_EV(10);
  return FM_OK;
#undef FM_EV
}

// H statistics + MU (mode 0) or the statistics for the all-reduce (mode 1)
// from the phi in the workspace and the W given (k_hstats, fm_nmf.cuh)
template <typename R>
int Impl<R>::hstats(const fm_dims* d, const fm_state* s, const R* Wsrc, int mode, void* hstat,
                    cudaStream_t st) {
  const Plan p = make_plan(d);
  unsigned char* w = reinterpret_cast<unsigned char*>(s->work);
  const R* phi = reinterpret_cast<const R*>(w + p.off_phi);
  R* H = reinterpret_cast<R*>(s->H);
  const int N = (int)d->N, F = (int)d->F, T = (int)d->T, K = (int)d->K;
  const unsigned BN = (unsigned)(d->B * (d->N - (d->dp ? 1 : 0)));
  FM_DISPATCH_KB(K, {
    FM_DISPATCH_TILE(p.TT, TTT, {
      if constexpr (TTT >= 16) {
        const size_t smh = HsCfg<R, KB, TTT>::bytes;
        if (int rc = ensure_smem(k_hstats<R, KB, TTT>, smh)) return rc;
        launch_pdl(k_hstats<R, KB, TTT>, dim3((unsigned)((T + TTT - 1) / TTT), BN, (unsigned)p.HS),
                   dim3(256), smh, st, phi, Wsrc, H, reinterpret_cast<R*>(hstat), N, F, T, K,
                   mode, 0, p.HFR, reinterpret_cast<R*>(w + p.off_hpart),
                   reinterpret_cast<unsigned*>(w + p.off_hcnt));
        FM_CHECK_LAUNCH("k_hstats");
      }
    });
  });
  return FM_OK;
}

// The per-bin schedule (fm_bin.cuh): the W step of the first iteration and
// the refresh after it run here (k_lambda, k_back, k_wstats on Wn, k_lambda,
// k_phi), leaving x~, Wn and phi; each iteration is then
//   k_hstats  H step from phi(Wn, H)                        (separate.py:214-216 "H")
//   k_binw    gains, V, IP, normalisations, W = Wn c, x~, data term, the
//             next W step -> Wn and its refresh -> phi      (separate.py:217-234,
//                                                           :186-193, :214-216 "W")
//   k_trace
// The state W stays the reference's (after the absorb); fm_refresh re-runs
// this prologue after a caller assigns state.
template <typename R>
int Impl<R>::prologue_bin(const fm_dims* d, const fm_state* s, cudaStream_t st) {
  const Plan p = make_plan(d);
  unsigned char* w = reinterpret_cast<unsigned char*>(s->work);
  R* lam = reinterpret_cast<R*>(w + p.off_lam);
  R* phi = reinterpret_cast<R*>(w + p.off_phi);
  R* Wn = reinterpret_cast<R*>(w + p.off_wn);
  const R* H = reinterpret_cast<const R*>(s->H);
  const int N = (int)d->N, F = (int)d->F, T = (int)d->T, K = (int)d->K;
  if (int rc = lambda(d, reinterpret_cast<const R*>(s->W), H, lam, st)) return rc;
  if (int rc = back(d, s, /*tail_only=*/1, /*record=*/0, st)) return rc;  // x~, data term, phi
  FM_CUDA(cudaMemcpyAsync(Wn, s->W, (size_t)d->B * N * F * K * sizeof(R), cudaMemcpyDeviceToDevice, st));
  FM_DISPATCH_KB(K, {
    FM_DISPATCH_TILE(p.FT, FTT, {
      if constexpr (FTT <= 32) {
        const size_t smw = WsCfg<R, KB, FTT>::bytes;
        if (int rc = ensure_smem(k_wstats<R, KB, FTT>, smw)) return rc;
        launch_pdl(k_wstats<R, KB, FTT>, dim3((unsigned)((F + FTT - 1) / FTT), (unsigned)(d->B * N)),
                   dim3(256), smw, st, phi, H, Wn, N, F, T, K, 0);
        FM_CHECK_LAUNCH("k_wstats");
      }
    });
  });
  if (int rc = lambda(d, Wn, H, lam, st)) return rc;
  FM_DISPATCH_M(d->M, {
    launch_pdl(k_phi<R, MM>, dim3((unsigned)((T + 255) / 256), (unsigned)F, (unsigned)d->B),
               dim3(256), 0, st, lam, reinterpret_cast<const R*>(s->xt),
               reinterpret_cast<const R*>(s->g), reinterpret_cast<const R*>(s->floor), phi, N, F, T);
    FM_CHECK_LAUNCH("k_phi");
  });
  return FM_OK;
}

template <typename R>
int Impl<R>::iterate_bin(const fm_dims* d, const fm_state* s, int phase, void* hstat,
                         cudaStream_t st, cudaEvent_t* ev) {
#define FM_EV(i) \
  if (ev) FM_CUDA(cudaEventRecordWithFlags(ev[i], st, cudaEventRecordExternal));
  const Plan p = make_plan(d);
  unsigned char* w = reinterpret_cast<unsigned char*>(s->work);
  R* H = reinterpret_cast<R*>(s->H);
  FM_EV(0);
  if (phase == 0 || phase == 2) {
    if (int rc = hstats(d, s, reinterpret_cast<const R*>(w + p.off_wn), phase == 0 ? 1 : 0, hstat, st))
      return rc;
  }
  if (phase == 0) return FM_OK;
  if (phase == 1) {
    const long long NKT = d->N * d->K * d->T, total = d->B * NKT;
    k_hupdate<R><<<(unsigned)((total + 255) / 256), 256, 0, st>>>(
        nullptr, H, reinterpret_cast<R*>(hstat), 1, NKT, total, 2);
    FM_CHECK_LAUNCH("k_hupdate");
  }
  FM_EV(1);
  if (int rc = binw(d, s, st)) return rc;
  FM_EV(2);
  if (int rc = trace(d, s, st)) return rc;
  FM_EV(3);
  return FM_OK;
#undef FM_EV
}

template <typename R>
int Impl<R>::iterate_phase(const fm_dims* d, const fm_state* s, int phase, void* hstat,
                           cudaStream_t st, cudaEvent_t* ev) {
  if (d->dp) { set_error("deep-prior dims: use fm_iterate_dp"); return FM_EINVAL; }
  if (use_bin(d)) return iterate_bin(d, s, phase, hstat, st, ev);
  return use_fused(d) ? iterate_fused(d, s, phase, hstat, st, ev)
                      : iterate_split(d, s, phase, hstat, st, ev);
}

template <typename R>
int Impl<R>::iterate_fused(const fm_dims* d, const fm_state* s, int phase, void* hstat,
                           cudaStream_t st, cudaEvent_t* ev) {
#define FM_EV(i) \
  if (ev) FM_CUDA(cudaEventRecordWithFlags(ev[i], st, cudaEventRecordExternal));
  // The plain FastMNMF iteration (separate.py:201-234) in five compute
  // launches; its W step already ran in the previous k_bpass (or the
  // prologue), leaving Wn:
  //   k_hpass   H step: phi from lambda(Wn, H), H MU        (separate.py:214-216)
  //   k_gpass   gain statistics from lambda(Wn, H_new)     (separate.py:217)
  //   k_vacc    g MU + V_fm                                 (separate.py:218-222)
  //   k_ip      IP rows, row/gain normalisation, W = Wn c   (separate.py:222-233)
  //   k_bpass   x~ = |Qx|^2, data term, next W step -> Wn   (separate.py:230; :186-193)
  //   k_trace   trace entry
  if (d->dp) { set_error("deep-prior dims: use fm_iterate_dp"); return FM_EINVAL; }
  FM_EV(0);
  if (phase == 0 || phase == 2) {
    if (int rc = hpass(d, s, phase == 0 ? 1 : 0, hstat, st)) return rc;
  }
  if (phase == 0) return FM_OK;
  if (phase == 1) {  // H MU from the all-reduced statistics, and Ht
    if (int rc = hstore(d, s, hstat, st)) return rc;
  }
  FM_EV(1);
  if (int rc = gpass(d, s, st)) return rc;
  FM_EV(2);
  if (int rc = vacc(d, s, st)) return rc;
  FM_EV(3);
  if (int rc = ip(d, s, st)) return rc;
  FM_EV(4);
  if (int rc = bpass(d, s, st)) return rc;
  FM_EV(5);
  if (int rc = trace(d, s, st)) return rc;
  FM_EV(6);
  return FM_OK;
#undef FM_EV
}

// ---------------------------------------------------------------------------
// FastMNMF-DP (config 4)
// ---------------------------------------------------------------------------
constexpr size_t LT_SMEM_MAX = 226 * 1024;  // opt-in dynamic limit less the static kernel smem

// The latent hook in one launch (fm_dp_latent.cuh): `steps` Adam steps and the
// refresh r = exp(dec(z)); steps = 0 is the refresh alone.
template <typename R>
int Impl<R>::dp_latent(const fm_dims* d, const fm_state* s, const fm_dp* p, int steps, cudaStream_t st) {
  const Plan pl = make_plan(d);
  unsigned char* w = reinterpret_cast<unsigned char*>(s->work);
  LatentArgs<R> a;
  a.W1 = reinterpret_cast<const R*>(p->W1);
  a.b1 = reinterpret_cast<const R*>(p->b1);
  a.W2 = reinterpret_cast<const R*>(p->W2);
  a.b2 = reinterpret_cast<const R*>(p->b2);
  a.W3 = reinterpret_cast<const R*>(p->W3);
  a.b3 = reinterpret_cast<const R*>(p->b3);
  a.u = reinterpret_cast<const R*>(p->u);
  a.v = reinterpret_cast<const R*>(p->v);
  a.z = reinterpret_cast<R*>(p->z);
  a.m = reinterpret_cast<R*>(p->adam_m);
  a.v2 = reinterpret_cast<R*>(p->adam_v);
  a.r = reinterpret_cast<R*>(p->r);
  a.lam = reinterpret_cast<const R*>(w + pl.off_lam);
  a.xt = reinterpret_cast<const R*>(s->xt);
  a.g = reinterpret_cast<const R*>(s->g);
  a.iter = reinterpret_cast<const unsigned*>(w + pl.off_cnt) + 1;
  a.T = (int)d->T;
  a.F = (int)d->F;
  a.D = (int)p->D;
  a.Hd = (int)p->Hd;
  a.N = (int)d->N;
  a.steps = steps;
  a.lr = p->lr;
  a.b1a = p->beta1;
  a.b2a = p->beta2;
  a.eps = p->eps;
  dim3 grid((unsigned)((d->T + LT_FR - 1) / LT_FR), (unsigned)d->B);
  FM_DISPATCH_M(d->M, {
    size_t sm = 0;
    static const int max_stages = [] {  // FM_LT_STAGES: pipeline-depth tuning knob (2..4)
      const char* e = getenv("FM_LT_STAGES");
      const int v = e ? atoi(e) : 3;
      return v < 2 ? 2 : v > 4 ? 4 : v;
    }();
    for (a.stages = max_stages; a.stages > 2; --a.stages) {  // deepest pipeline that fits
      sm = sizeof(R) * lt_layout<R, MM>(a.stages, a.N).total;
      if (sm <= LT_SMEM_MAX) break;
    }
    sm = sizeof(R) * lt_layout<R, MM>(a.stages, a.N).total;
    if (sm > LT_SMEM_MAX) {
      set_error("latent kernel needs %zu B shared memory (N=%d M=%d)", sm, a.N, (int)MM);
      return FM_EINVAL;
    }
    if (int rc = ensure_smem(k_dp_latent<R, MM>, sm)) return rc;
    launch_pdl(k_dp_latent<R, MM>, grid, dim3(LtCfg<R, MM>::NT), sm, st, a);
    FM_CHECK_LAUNCH("k_dp_latent");
  });
  return FM_OK;
}

// The reference's Metropolis latent chain (fm_dp_mh.cuh); steps = 0 is the
// decoder refresh r = dec(z) (any decoder kind).
template <typename R>
int Impl<R>::dp_mh(const fm_dims* d, const fm_state* s, const fm_dp* p, int steps, cudaStream_t st) {
  const Plan pl = make_plan(d);
  unsigned char* w = reinterpret_cast<unsigned char*>(s->work);
  MhArgs<R> a;
  a.W1 = reinterpret_cast<const R*>(p->W1);
  a.b1 = reinterpret_cast<const R*>(p->b1);
  a.W2 = reinterpret_cast<const R*>(p->W2);
  a.b2 = reinterpret_cast<const R*>(p->b2);
  a.WoT = reinterpret_cast<const R*>(reinterpret_cast<unsigned char*>(p->work) + 256);
  a.bo = reinterpret_cast<const R*>(p->b3);
  a.u = reinterpret_cast<const R*>(p->u);
  a.v = reinterpret_cast<const R*>(p->v);
  a.z = reinterpret_cast<R*>(p->z);
  a.r = reinterpret_cast<R*>(p->r);
  a.lam = reinterpret_cast<const R*>(w + pl.off_lam);
  a.g = reinterpret_cast<const R*>(s->g);
  a.xt = reinterpret_cast<const R*>(s->xt);
  a.noise = reinterpret_cast<const R*>(p->mh_noise);
  a.unif = reinterpret_cast<const R*>(p->mh_unif);
  a.iter = reinterpret_cast<const unsigned*>(w + pl.off_cnt) + 1;
  a.seed = p->mh_seed;
  a.stdv = p->mh_std;
  a.steps = steps;
  a.kind = p->decoder_kind;
  a.D = (int)p->D; a.Hd = (int)p->Hd;
  a.N = (int)d->N; a.F = (int)d->F; a.T = (int)d->T; a.M = (int)d->M; a.B = (int)d->B;
  // frames per CTA: 2, fewer while the staged x~ / y_rest do
  // not fit; without staging they are re-read from L2 every proposal
  const size_t rs = sizeof(R), cap = 200 * 1024;
  a.cache = 1;
  a.fpb = 2;  // 2 frames per 256-thread CTA: ~2 CTAs (16 warps) per SM at config 4
  while (a.fpb > 1 && mh_smem_bytes(rs, a.fpb, a.D, a.Hd, a.F, a.M, true) > cap) --a.fpb;
  if (mh_smem_bytes(rs, a.fpb, a.D, a.Hd, a.F, a.M, true) > cap) {
    a.cache = 0;
    a.fpb = 2;
  }
  if (steps == 0) a.cache = 0;
  const size_t sm = mh_smem_bytes(rs, a.fpb, a.D, a.Hd, a.F, a.M, a.cache != 0);
  if (sm > LT_SMEM_MAX) {
    set_error("Metropolis kernel needs %zu B shared memory (F=%d Hd=%d)", sm, a.F, a.Hd);
    return FM_EINVAL;
  }
  if (int rc = ensure_smem(k_dp_mh<R>, sm)) return rc;
  launch_pdl(k_dp_mh<R>, dim3((unsigned)((d->T + a.fpb - 1) / a.fpb), (unsigned)d->B), dim3(256), sm,
             st, a);
  FM_CHECK_LAUNCH("k_dp_mh");
  return FM_OK;
}

template <typename R>
int Impl<R>::dp_lambda(const fm_dims* d, const fm_state* s, const fm_dp* p, cudaStream_t st) {
  const Plan pl = make_plan(d);
  R* lam = reinterpret_cast<R*>(reinterpret_cast<unsigned char*>(s->work) + pl.off_lam);
  dim3 grid((unsigned)((d->T + 31) / 32), (unsigned)((d->F + 31) / 32), (unsigned)d->B);
  launch_pdl(k_dp_lambda<R>, grid, dim3(32, 8), 0, st, reinterpret_cast<const R*>(p->u),
             reinterpret_cast<const R*>(p->v), reinterpret_cast<const R*>(p->r), lam, (int)d->N,
             (int)d->F, (int)d->T);
  FM_CHECK_LAUNCH("k_dp_lambda");
  return FM_OK;
}

template <typename R>
int Impl<R>::lambda_nmf(const fm_dims* d, const fm_state* s, cudaStream_t st) {
  const Plan pl = make_plan(d);
  return lambda(d, reinterpret_cast<const R*>(s->W), reinterpret_cast<const R*>(s->H),
                reinterpret_cast<R*>(reinterpret_cast<unsigned char*>(s->work) + pl.off_lam), st);
}

template <typename R>
int Impl<R>::phi_pass(const fm_dims* d, const fm_state* s, cudaStream_t st) {
  const Plan pl = make_plan(d);
  unsigned char* w = reinterpret_cast<unsigned char*>(s->work);
  const int N = (int)d->N, F = (int)d->F, T = (int)d->T;
  FM_DISPATCH_M(d->M, {
    launch_pdl(k_phi<R, MM>, dim3((unsigned)((T + 255) / 256), (unsigned)F, (unsigned)d->B),
               dim3(256), 0, st, reinterpret_cast<const R*>(w + pl.off_lam),
               reinterpret_cast<const R*>(s->xt), reinterpret_cast<const R*>(s->g),
               reinterpret_cast<const R*>(s->floor), reinterpret_cast<R*>(w + pl.off_phi), N, F, T);
    FM_CHECK_LAUNCH("k_phi");
  });
  return FM_OK;
}

template <typename R>
int Impl<R>::prologue_dp(const fm_dims* d, const fm_state* s, const fm_dp* p, cudaStream_t st) {
  const Plan pl = make_plan(d);
  unsigned char* w = reinterpret_cast<unsigned char*>(s->work);
  FM_CUDA(cudaMemsetAsync(w + pl.off_cnt, 0, pl.total - pl.off_cnt, st));
  k_transpose_fh<R><<<dim3((unsigned)((d->F + 31) / 32), (unsigned)((p->Hd + 31) / 32)), dim3(32, 8), 0,
                      st>>>(reinterpret_cast<const R*>(p->W3),
                            reinterpret_cast<R*>(reinterpret_cast<unsigned char*>(p->work) + 256),
                            (int)d->F, (int)p->Hd);
  FM_CHECK_LAUNCH("k_transpose_fh");
  if (p->decoder_kind == FM_DEC_TOY) {
    if (int rc = dp_mh(d, s, p, 0, st)) return rc;
  } else {
    if (int rc = dp_latent(d, s, p, 0, st)) return rc;
  }
  if (int rc = dp_lambda(d, s, p, st)) return rc;
  if (int rc = lambda_nmf(d, s, st)) return rc;
  return back(d, s, /*tail_only=*/1, /*record=*/0, st);
}

template <typename R>
int Impl<R>::iterate_dp(const fm_dims* d, const fm_state* s, const fm_dp* p, cudaStream_t st,
                        cudaEvent_t* ev) {
  int nev = 0;  // external event-record nodes between launches (fm_iterate_dp_profiled)
#define FM_EVD() \
  if (ev) FM_CUDA(cudaEventRecordWithFlags(ev[nev++], st, cudaEventRecordExternal));
  const Plan pl = make_plan(d);
  unsigned char* w = reinterpret_cast<unsigned char*>(s->work);
  R* phi = reinterpret_cast<R*>(w + pl.off_phi);
  R* W = reinterpret_cast<R*>(s->W);
  R* H = reinterpret_cast<R*>(s->H);
  R* u = reinterpret_cast<R*>(p->u);
  R* v = reinterpret_cast<R*>(p->v);
  const R* r = reinterpret_cast<const R*>(p->r);
  const int N = (int)d->N, F = (int)d->F, T = (int)d->T, K = (int)d->K, B = (int)d->B;
  const unsigned BN = (unsigned)(d->B * (d->N - 1));
  // lambda of the state after the previous iteration (u absorbed c[0], W c[1:])
  FM_EVD();
  if (int rc = lambda_nmf(d, s, st)) return rc;
  FM_EVD();
  if (int rc = dp_lambda(d, s, p, st)) return rc;
  // latent hook (separate.py:205-213): Adam on z against the frozen y_rest,
  // then r = exp(dec(z)) -- one launch
  if (p->mh_steps > 0) {  // the reference's Metropolis chain (sources.py:307-339)
    FM_EVD();
    if (int rc = dp_mh(d, s, p, p->mh_steps, st)) return rc;
    FM_EVD();
    if (int rc = dp_lambda(d, s, p, st)) return rc;
  } else if (p->adam_steps > 0) {  // BASELINE config 4: Adam
    FM_EVD();
    if (int rc = dp_latent(d, s, p, p->adam_steps, st)) return rc;
    FM_EVD();
    if (int rc = dp_lambda(d, s, p, st)) return rc;
  }
  // U step (sources.py:258-261)
  FM_EVD();
  if (int rc = phi_pass(d, s, st)) return rc;
  FM_EVD();
  launch_pdl(k_dp_umu<R>, dim3((unsigned)F, (unsigned)B), dim3(256), 0, st, u, (const R*)v, r,
             (const R*)phi, N, F, T);
  FM_CHECK_LAUNCH("k_dp_umu");
  FM_EVD();
  if (int rc = dp_lambda(d, s, p, st)) return rc;
  // V step (sources.py:262-265)
  FM_EVD();
  if (int rc = phi_pass(d, s, st)) return rc;
  FM_EVD();
  launch_pdl(k_dp_vmu<R>, dim3((unsigned)((T + 31) / 32), (unsigned)VMU_FS, (unsigned)B), dim3(32, 8), 0,
             st, (const R*)u, v, r, (const R*)phi, N, F, T, reinterpret_cast<R*>(w + pl.off_vmu),
             reinterpret_cast<unsigned*>(w + pl.off_vcnt));
  FM_CHECK_LAUNCH("k_dp_vmu");
  FM_EVD();
  if (int rc = dp_lambda(d, s, p, st)) return rc;
  // W step (noise NMF, sources.py:253 -> 191-194)
  FM_EVD();
  if (int rc = phi_pass(d, s, st)) return rc;
  FM_EVD();
  FM_DISPATCH_KB(K, {
    FM_DISPATCH_TILE(pl.FT, FTT, {
      if constexpr (FTT <= 32) {
        const size_t smw = WsCfg<R, KB, FTT>::bytes;
        if (int rc = ensure_smem(k_wstats<R, KB, FTT>, smw)) return rc;
        launch_pdl(k_wstats<R, KB, FTT>, dim3((unsigned)((F + FTT - 1) / FTT), BN), dim3(256), smw,
                   st, (const R*)phi, (const R*)H, W, N, F, T, K, 1);
        FM_CHECK_LAUNCH("k_wstats");
      }
    });
  });
  // H step
  FM_EVD();
  if (int rc = lambda_nmf(d, s, st)) return rc;
  FM_EVD();
  if (int rc = phi_pass(d, s, st)) return rc;
  FM_EVD();
  FM_DISPATCH_KB(K, {
    FM_DISPATCH_TILE(pl.TT, TTT, {
      if constexpr (TTT >= 16) {
        const size_t smh = HsCfg<R, KB, TTT>::bytes;
        if (int rc = ensure_smem(k_hstats<R, KB, TTT>, smh)) return rc;
        launch_pdl(k_hstats<R, KB, TTT>, dim3((unsigned)((T + TTT - 1) / TTT), BN, (unsigned)pl.HS),
                   dim3(256), smh, st, (const R*)phi, (const R*)W, H, (R*)nullptr, N, F, T, K, 0, 1,
                   pl.HFR, reinterpret_cast<R*>(w + pl.off_hpart),
                   reinterpret_cast<unsigned*>(w + pl.off_hcnt));
        FM_CHECK_LAUNCH("k_hstats");
      }
    });
  });
  FM_EVD();
  if (int rc = lambda_nmf(d, s, st)) return rc;
  // spatial part as in the plain iteration; k_ip folds c[0] into u
  FM_EVD();
  if (int rc = gain(d, s, st)) return rc;
  FM_EVD();
  if (int rc = vacc(d, s, st)) return rc;
  FM_EVD();
  if (int rc = ip(d, s, st, u)) return rc;
  FM_EVD();
  if (int rc = back(d, s, /*tail_only=*/0, /*record=*/1, st)) return rc;
  FM_EVD();
  if (int rc = trace(d, s, st)) return rc;
  FM_EVD();
  return FM_OK;
#undef FM_EVD
}

// ---------------------------------------------------------------------------
// per-op entry points
// ---------------------------------------------------------------------------
template <typename R>
int Impl<R>::fast_stats(int64_t F, int64_t T, int64_t M, int64_t N, const void* xt,
                        const void* g, const void* lam, double floor, int want_gain,
                        int want_phi, void* phi1, void* phi2, void* gnum, void* gden,
                        double* ll_host, cudaStream_t st) {
  if (N > 8) { set_error("N=%lld outside 1..8", (long long)N); return FM_EINVAL; }
  double* llp = nullptr;
  FM_CUDA(cudaMallocAsync(&llp, sizeof(double) * std::max<int64_t>(F, 1), st));
  int rc = FM_OK;
  FM_DISPATCH_M(M, {
    k_fast_stats<R, MM><<<(unsigned)F, 256, 0, st>>>(
        reinterpret_cast<const R*>(xt), reinterpret_cast<const R*>(g),
        reinterpret_cast<const R*>(lam), (R)floor, (int)N, (int)F, (int)T,
        want_phi ? reinterpret_cast<R*>(phi1) : nullptr,
        want_phi ? reinterpret_cast<R*>(phi2) : nullptr,
        want_gain ? reinterpret_cast<R*>(gnum) : nullptr,
        want_gain ? reinterpret_cast<R*>(gden) : nullptr, llp);
  });
  if (cudaGetLastError() != cudaSuccess) rc = FM_ECUDA;
  std::vector<double> h((size_t)F);
  if (rc == FM_OK && F > 0) {
    FM_CUDA(cudaMemcpyAsync(h.data(), llp, sizeof(double) * F, cudaMemcpyDeviceToHost, st));
  }
  FM_CUDA(cudaFreeAsync(llp, st));
  FM_CUDA(cudaStreamSynchronize(st));
  if (rc != FM_OK) { set_error("k_fast_stats launch failed"); return rc; }
  double s = 0.0;
  for (int64_t f = 0; f < F; ++f) s += h[(size_t)f];
  if (ll_host) *ll_host = s;
  return FM_OK;
}

template <typename R>
int Impl<R>::mix_power(int64_t N, int64_t F, int64_t T, int64_t M, const void* lam, const void* g,
                       double floor, void* y, cudaStream_t st) {
  const long long n = (long long)F * T;
  if (n == 0) return FM_OK;
  k_mix_power<R><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(
      reinterpret_cast<const R*>(lam), reinterpret_cast<const R*>(g), (R)floor, (int)N, (int)F,
      (int)T, (int)M, reinterpret_cast<R*>(y));
  FM_CHECK_LAUNCH("k_mix_power");
  return FM_OK;
}

template <typename R>
int Impl<R>::ip_weights(int64_t F, int64_t T, int64_t M, const void* X, const void* y, void* V,
                        cudaStream_t st) {
  if (F == 0) return FM_OK;
  FM_DISPATCH_M(M, {
    k_ip_weights<R, MM><<<(unsigned)F, 256, 0, st>>>(reinterpret_cast<const C*>(X),
                                                      reinterpret_cast<const R*>(y), (int)T,
                                                      reinterpret_cast<C*>(V));
    FM_CHECK_LAUNCH("k_ip_weights");
  });
  return FM_OK;
}

template <typename R>
int Impl<R>::project(int64_t F, int64_t T, int64_t M, const void* Q, const void* X, void* xt,
                     cudaStream_t st) {
  const long long n = (long long)F * T;
  if (n == 0) return FM_OK;
  FM_DISPATCH_M(M, {
    k_project<R, MM><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(
        reinterpret_cast<const C*>(Q), reinterpret_cast<const C*>(X), (int)F, (int)T,
        reinterpret_cast<R*>(xt));
    FM_CHECK_LAUNCH("k_project");
  });
  return FM_OK;
}

template <typename R>
int Impl<R>::update_diagonalizer(int64_t F, int64_t T, int64_t M, void* Q, const void* X,
                                 const void* y, int sweeps, uint64_t* status, cudaStream_t st) {
  if (F == 0) return FM_OK;
  C* V = nullptr;
  FM_CUDA(cudaMallocAsync(&V, sizeof(C) * F * M * M * M, st));
  int rc = ip_weights(F, T, M, X, y, V, st);
  if (rc == FM_OK) {
    FM_DISPATCH_M(M, {
      k_ipsolve<R, MM><<<(unsigned)F, 32, 0, st>>>(reinterpret_cast<C*>(Q), V, sweeps,
                                                    reinterpret_cast<unsigned long long*>(status));
      FM_CHECK_LAUNCH("k_ipsolve");
    });
  }
  FM_CUDA(cudaFreeAsync(V, st));
  return rc;
}

template <typename R>
int Impl<R>::logdet(int64_t F, int64_t M, const void* Q, double* out, cudaStream_t st) {
  if (F == 0) return FM_OK;
  FM_DISPATCH_M(M, {
    k_logdet<R, MM><<<(unsigned)F, 32, 0, st>>>(reinterpret_cast<const C*>(Q), out);
    FM_CHECK_LAUNCH("k_logdet");
  });
  return FM_OK;
}

template <typename R>
int Impl<R>::wiener(int64_t N, int64_t F, int64_t T, int64_t M, const void* lam, const void* Q,
                    const void* g, const void* X, void* out, uint64_t* status, cudaStream_t st) {
  if (N > 8) { set_error("N=%lld outside 1..8", (long long)N); return FM_EINVAL; }
  if (F == 0) return FM_OK;
  // Q^-1 per bin (k_qinv), then one frame per thread (k_wiener_t); the
  // scratch comes from the device's stream-ordered pool (kept mapped: see
  // keep_pool_mapped)
  keep_pool_mapped();
  unsigned char* scratch = nullptr;
  const size_t qbytes = align256(sizeof(C) * (size_t)F * M * M);
  FM_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&scratch), qbytes + sizeof(int) * (size_t)F, st));
  C* Qi = reinterpret_cast<C*>(scratch);
  int* bad = reinterpret_cast<int*>(scratch + qbytes);
  int rc = FM_OK;
  FM_DISPATCH_M(M, {
    k_qinv<R, MM><<<(unsigned)((F + 3) / 4), 128, 0, st>>>(
        reinterpret_cast<const C*>(Q), (int)F, Qi, bad, reinterpret_cast<unsigned long long*>(status));
    k_wiener_t<R, MM><<<dim3((unsigned)((T + 127) / 128), (unsigned)F), 128, 0, st>>>(
        reinterpret_cast<const R*>(lam), reinterpret_cast<const C*>(Q), Qi, bad,
        reinterpret_cast<const R*>(g), reinterpret_cast<const C*>(X), (int)N, (int)F, (int)T,
        reinterpret_cast<C*>(out));
  });
  if (cudaGetLastError() != cudaSuccess) {
    set_error("k_qinv / k_wiener_t launch failed");
    rc = FM_ECUDA;
  }
  FM_CUDA(cudaFreeAsync(scratch, st));
  return rc;
}

// Small persistent device + pinned host scratch for the synchronous prologue
// helpers (observation statistics, scaling): a per-call cudaMallocAsync /
// cudaFreeAsync re-mapped pool memory on every run() (~10 ms per call).
struct HostSync {
  std::mutex mu;
  double* dev = nullptr;
  double* host = nullptr;
  size_t n = 0;
  int grow(size_t need) {
    if (need <= n) return FM_OK;
    if (dev) cudaFree(dev);
    if (host) cudaFreeHost(host);
    dev = nullptr;
    host = nullptr;
    n = 0;
    if (cudaMalloc(&dev, need * sizeof(double)) != cudaSuccess ||
        cudaMallocHost(&host, need * sizeof(double)) != cudaSuccess) {
      set_error("scratch allocation of %zu doubles failed", need);
      return FM_ECUDA;
    }
    n = need;
    return FM_OK;
  }
};
inline HostSync& host_sync() {
  static HostSync h;
  return h;
}

template <typename R>
int Impl<R>::obs_stats(const fm_dims* d, const void* X, double* sumsq, double* maxsq,
                       cudaStream_t st) {
  const long long per_b = d->F * d->T * d->M;
  const unsigned nblk = (unsigned)std::max<long long>(1, std::min<long long>(256, (per_b + 4095) / 4096));
  HostSync& hs = host_sync();
  std::lock_guard<std::mutex> lock(hs.mu);
  const size_t nv = (size_t)2 * nblk * d->B;
  if (int rc = hs.grow(nv)) return rc;
  double* buf = hs.dev;
  k_obs_stats<R><<<dim3(nblk, (unsigned)d->B), 256, 0, st>>>(reinterpret_cast<const C*>(X), per_b,
                                                             buf, buf + (size_t)nblk * d->B);
  FM_CHECK_LAUNCH("k_obs_stats");
  FM_CUDA(cudaMemcpyAsync(hs.host, buf, sizeof(double) * nv, cudaMemcpyDeviceToHost, st));
  FM_CUDA(cudaStreamSynchronize(st));
  const double* h = hs.host;
  for (long long b = 0; b < d->B; ++b) {
    double s = 0.0, m = 0.0;
    for (unsigned i = 0; i < nblk; ++i) {
      s += h[(size_t)b * nblk + i];
      m = std::max(m, h[(size_t)nblk * d->B + (size_t)b * nblk + i]);
    }
    if (sumsq) sumsq[b] = s;
    if (maxsq) maxsq[b] = m;
  }
  return FM_OK;
}

template <typename R>
int Impl<R>::scale(const fm_dims* d, void* X, const double* scale_host, cudaStream_t st) {
  const long long per_b = d->F * d->T * d->M;
  HostSync& hs = host_sync();
  std::lock_guard<std::mutex> lock(hs.mu);
  if (int rc = hs.grow((size_t)d->B)) return rc;
  double* sc = hs.dev;
  memcpy(hs.host, scale_host, sizeof(double) * d->B);
  FM_CUDA(cudaMemcpyAsync(sc, hs.host, sizeof(double) * d->B, cudaMemcpyHostToDevice, st));
  const long long n = per_b * d->B;
  k_scale<R><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(reinterpret_cast<C*>(X), per_b, sc, (int)d->B);
  FM_CHECK_LAUNCH("k_scale");
  FM_CUDA(cudaStreamSynchronize(st));
  return FM_OK;
}

template <typename R>
int Impl<R>::spatial_init(const fm_dims* d, const void* X, void* Q, double* w, cudaStream_t st) {
  InitArgs<R> a;
  a.X = reinterpret_cast<const C*>(X);
  a.Q = reinterpret_cast<C*>(Q);
  a.w = w;
  a.F = (int)d->F;
  a.T = (int)d->T;
  FM_DISPATCH_M(d->M, {
    k_spatial_init<R, MM><<<dim3((unsigned)d->F, (unsigned)d->B), 256, 0, st>>>(a);
    FM_CHECK_LAUNCH("k_spatial_init");
  });
  return FM_OK;
}

// ---- STFT / iSTFT (fm_stft.cuh) ----------------------------------------------
inline int stft_group(int64_t M, int64_t L, size_t csize) {
  // channels per CTA: their rows + twiddles within ~96 KB (2 CTAs per SM)
  const long long per = (long long)L * (long long)csize;
  long long g = std::max<long long>(1, (96 * 1024 - (long long)(L / 2) * (long long)csize) / per);
  return (int)std::min<long long>(g, M);
}

inline int stft_check(int64_t M, int64_t L, int64_t hop) {
  if (L < 2 || (L & (L - 1)) || L > (1 << 16) || hop < 1 || hop > L || M < 1) {
    set_error("stft sizes: window_length %lld (power of two, 2..65536), hop %lld, M %lld",
              (long long)L, (long long)hop, (long long)M);
    return FM_EINVAL;
  }
  return FM_OK;
}

template <typename R>
int Impl<R>::stft(int64_t n, int64_t M, int64_t L, int64_t hop, const void* wave, void* spec,
                  cudaStream_t st) {
  if (int rc = stft_check(M, L, hop)) return rc;
  if (n < L) {
    set_error("signal length %lld is shorter than one window (%lld)", (long long)n, (long long)L);
    return FM_EINVAL;
  }
  const long long T = stft_frames(n, L, hop);
  const int G = stft_group(M, L, sizeof(C));
  const size_t sm = ((size_t)G * L + L / 2) * sizeof(C);
  if (sm > LT_SMEM_MAX) { set_error("window_length %lld too large", (long long)L); return FM_EINVAL; }
  if (int rc = ensure_smem(k_stft<R>, sm)) return rc;
  int logL = 0;
  while ((1LL << logL) < L) ++logL;
  k_stft<R><<<dim3((unsigned)T, (unsigned)((M + G - 1) / G)), STFT_THREADS, sm, st>>>(
      reinterpret_cast<const R*>(wave), reinterpret_cast<C*>(spec), (long long)n, (int)M, (int)L, logL,
      (int)hop, (int)T, G);
  FM_CHECK_LAUNCH("k_stft");
  return FM_OK;
}

template <typename R>
int Impl<R>::istft(int64_t T, int64_t M, int64_t L, int64_t hop, int64_t length, const void* spec,
                   void* work, void* out, cudaStream_t st) {
  if (int rc = stft_check(M, L, hop)) return rc;
  if (T < 1 || length < 0 || length > (T - 1) * hop) {
    set_error("istft: length %lld outside 0..%lld", (long long)length, (long long)((T - 1) * hop));
    return FM_EINVAL;
  }
  const int G = stft_group(M, L, sizeof(C));
  const size_t sm = ((size_t)G * L + L / 2) * sizeof(C);
  if (sm > LT_SMEM_MAX) { set_error("window_length %lld too large", (long long)L); return FM_EINVAL; }
  if (int rc = ensure_smem(k_istft_frames<R>, sm)) return rc;
  int logL = 0;
  while ((1LL << logL) < L) ++logL;
  k_istft_frames<R><<<dim3((unsigned)T, (unsigned)((M + G - 1) / G)), STFT_THREADS, sm, st>>>(
      reinterpret_cast<const C*>(spec), reinterpret_cast<R*>(work), (int)M, (int)L, logL, (int)T, G);
  FM_CHECK_LAUNCH("k_istft_frames");
  if (length > 0) {
    const long long tot = length * M;
    const unsigned blocks = (unsigned)std::min<long long>((tot + 255) / 256, 148 * 16);
    k_ola<R><<<blocks, 256, 0, st>>>(reinterpret_cast<const R*>(work), reinterpret_cast<R*>(out),
                                     (long long)length, (int)M, (int)L, (int)hop, (int)T);
    FM_CHECK_LAUNCH("k_ola");
  }
  return FM_OK;
}

// ---- full-rank MNMF comparator (fm_fullrank.cuh) ----------------------------
#define FM_DISPATCH_M8(Mrt, ...)                                                       \
  switch (Mrt) {                                                                       \
    case 1: { constexpr int MM = 1; __VA_ARGS__; } break;                              \
    case 2: { constexpr int MM = 2; __VA_ARGS__; } break;                              \
    case 3: { constexpr int MM = 3; __VA_ARGS__; } break;                              \
    case 4: { constexpr int MM = 4; __VA_ARGS__; } break;                              \
    case 5: { constexpr int MM = 5; __VA_ARGS__; } break;                              \
    case 6: { constexpr int MM = 6; __VA_ARGS__; } break;                              \
    case 7: { constexpr int MM = 7; __VA_ARGS__; } break;                              \
    case 8: { constexpr int MM = 8; __VA_ARGS__; } break;                              \
    default: set_error("full-rank model: M=%d outside 1..8", (int)(Mrt)); return FM_EINVAL; \
  }

inline size_t fr_workspace(size_t rs, int64_t F, int64_t T, int64_t M) {
  const size_t ft = (size_t)F * T;
  return align256(ft * M * 2 * rs) + align256(ft * M * M * 2 * rs) + align256(ft * 8) + 256;
}

template <typename R>
int Impl<R>::fr_stats(int64_t F, int64_t T, int64_t M, int64_t N, const void* X, const void* G,
                      const void* lam, double ridge, int want_ab, int want_phi, void* phi, void* A,
                      void* B, void* work, double* ll, cudaStream_t st) {
  unsigned char* w = reinterpret_cast<unsigned char*>(work);
  const size_t ft = (size_t)F * T;
  C* Zs = reinterpret_cast<C*>(w);
  C* Yis = reinterpret_cast<C*>(w + align256(ft * M * sizeof(C)));
  double* llp = reinterpret_cast<double*>(w + align256(ft * M * sizeof(C)) + align256(ft * M * M * sizeof(C)));
  const unsigned nb = (unsigned)((ft + 127) / 128);
  FM_DISPATCH_M8(M, {
    k_fr_bin<R, MM><<<nb, 128, 0, st>>>(reinterpret_cast<const C*>(X), reinterpret_cast<const C*>(G),
                                        reinterpret_cast<const R*>(lam), ridge, (int)N, (int)F, (int)T,
                                        want_phi, reinterpret_cast<R*>(phi), want_ab ? Zs : nullptr,
                                        Yis, llp);
    FM_CHECK_LAUNCH("k_fr_bin");
    if (want_ab) {
      const long long nt = N * F * (MM * (MM + 1) / 2);
      k_fr_ab<R, MM><<<(unsigned)((nt + 127) / 128), 128, 0, st>>>(
          reinterpret_cast<const R*>(lam), Zs, Yis, (int)N, (int)F, (int)T, reinterpret_cast<C*>(A),
          reinterpret_cast<C*>(B));
      FM_CHECK_LAUNCH("k_fr_ab");
    }
  });
  if (ll) {
    k_sum_fixed<<<1, 256, 0, st>>>(llp, (long long)ft, ll);
    FM_CHECK_LAUNCH("k_sum_fixed");
  }
  return FM_OK;
}

template <typename R>
int Impl<R>::fr_scm(int64_t N, int64_t F, int64_t M, void* G, const void* A, const void* B,
                    int normalize, void* c, uint64_t* status, cudaStream_t st) {
  FM_DISPATCH_M8(M, {
    k_fr_scm<R, MM><<<dim3((unsigned)F, (unsigned)N), 32, 0, st>>>(
        reinterpret_cast<C*>(G), reinterpret_cast<const C*>(A), reinterpret_cast<const C*>(B), (int)F,
        normalize, reinterpret_cast<R*>(c), reinterpret_cast<unsigned long long*>(status));
    FM_CHECK_LAUNCH("k_fr_scm");
  });
  return FM_OK;
}

template <typename R>
int Impl<R>::fr_wiener(int64_t N, int64_t F, int64_t T, int64_t M, const void* lam, const void* G,
                       const void* X, double ridge, void* out, uint64_t* status, cudaStream_t st) {
  const size_t ft = (size_t)F * T;
  FM_DISPATCH_M8(M, {
    k_fr_wiener<R, MM><<<(unsigned)((ft + 127) / 128), 128, 0, st>>>(
        reinterpret_cast<const R*>(lam), reinterpret_cast<const C*>(G), reinterpret_cast<const C*>(X),
        ridge, (int)N, (int)F, (int)T, reinterpret_cast<C*>(out),
        reinterpret_cast<unsigned long long*>(status));
    FM_CHECK_LAUNCH("k_fr_wiener");
  });
  return FM_OK;
}

template <typename R>
int Impl<R>::fr_nmf_mu(int64_t N, int64_t F, int64_t T, int64_t K, const void* phi, void* W, void* H,
                       int step, cudaStream_t st) {
  const long long nt = step == 0 ? N * F * K : N * K * T;
  k_fr_nmf_mu<R><<<(unsigned)((nt + 255) / 256), 256, 0, st>>>(
      reinterpret_cast<const R*>(phi), reinterpret_cast<R*>(W), reinterpret_cast<R*>(H), (int)N, (int)F,
      (int)T, (int)K, step);
  FM_CHECK_LAUNCH("k_fr_nmf_mu");
  return FM_OK;
}

template <typename R>
int Impl<R>::fr_absorb(int64_t N, int64_t F, int64_t K, void* W, const void* c, cudaStream_t st) {
  const long long nt = N * F * K;
  k_fr_absorb<R><<<(unsigned)((nt + 255) / 256), 256, 0, st>>>(reinterpret_cast<R*>(W),
                                                               reinterpret_cast<const R*>(c), N * F, (int)K);
  FM_CHECK_LAUNCH("k_fr_absorb");
  return FM_OK;
}

template <typename R>
int Impl<R>::fr_reconstruct(int64_t N, int64_t F, int64_t M, const void* Q, const void* g, void* G,
                            uint64_t* status, cudaStream_t st) {
  FM_DISPATCH_M8(M, {
    k_fr_reconstruct<R, MM><<<(unsigned)((F + 63) / 64), 64, 0, st>>>(
        reinterpret_cast<const C*>(Q), reinterpret_cast<const R*>(g), (int)N, (int)F,
        reinterpret_cast<C*>(G), reinterpret_cast<unsigned long long*>(status));
    FM_CHECK_LAUNCH("k_fr_reconstruct");
  });
  return FM_OK;
}

}  // namespace fm
