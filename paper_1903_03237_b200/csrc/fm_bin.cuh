// fm_bin.cuh -- the per-bin schedule (complex64, M <= 4): every step of one
// FastMNMF iteration that is local to a frequency bin runs in ONE kernel,
// k_binw, one warp per (bin, mixture); only the H step, which sums over the
// bins (sources.py:195-198), stays a separate launch (k_hstats).
//
// Per bin, in the reference's order (separate.py:201-234), after the H step:
//   E  lambda = Wn H (refresh after the H step) and the gain statistics;
//      g MU                                          (separate.py:217-220)
//   V  V_fm = (1/T) sum_t x x^H / y_ftm               (separate.py:221-222)
//   IP row updates, row / gain normalisation, W = Wn c  (separate.py:222-233)
//   P  x~ = |Q x|^2, the data term of the new state, and the NEXT iteration's
//      W statistics sum_t phi H^T and W MU -> Wn     (separate.py:230, :186-193,
//                                                      :214-216 "W")
//   R  the refresh after that W step: phi (B, 2N, F, T) for the next k_hstats
//
// H of the mixture (N x K x T, zero-padded to KK rows per source) is staged
// once per CTA in shared memory and serves every bin of the CTA; a lane owns
// the frames t = lane + 32 j of its warp's bin, so a bin's X, x~ and H rows
// are read coalesced and nothing but x~ (read and written) and phi (written)
// goes through HBM besides the two reads of X. A bin's statistics are summed
// per lane and reduced across the warp by recursive halving (fixed order:
// deterministic). The IP is the warp-private ipw_core of k_ip_w.
#pragma once
#include "fm_ipw.cuh"
#include "fm_nmf.cuh"

namespace fm {

template <typename R> struct BinArgs {
  const cplx<R>* X;
  R* xt;
  cplx<R>* Q;
  R* g;
  R* W;        // state W (after the absorb), written
  R* Wn;       // W-stepped W: read (this iteration's), written (the next one's)
  const R* H;  // (B, N, K, T) after this iteration's H step
  const R* floorp;
  R* phi;           // (B, 2N, F, T) refresh after the next W step (k_hstats input)
  double* ll_part;  // (B, F, ntile): data term in tile 0, zeros elsewhere
  double* ld_part;  // (B, F)
  const unsigned* iter;
  unsigned long long* status;
  int B, F, T, N, K;
  long long f_offset;
  int normalize, ip_sweeps;
  int rounds;  // bins per warp (a CTA covers BW_WARPS * rounds bins of one mixture)
  int ntile;   // k_back's data-term tiles per bin (ll_part layout)
};

constexpr int BW_WARPS = 8;

constexpr int pad32(int n) { return (n + 31) / 32 * 32; }

template <int M, int NN, int KK> struct BwCfg {
  static constexpr int P = M * (M + 1) / 2;
  static constexpr int NV_V = pad32(2 * M * P), NV_G = pad32(2 * NN * M), NV_W = pad32(2 * NN * KK);
  static constexpr int NV = NV_V > NV_G ? (NV_V > NV_W ? NV_V : NV_W) : (NV_G > NV_W ? NV_G : NV_W);
  static constexpr size_t al(size_t x) { return (x + 15) & ~size_t(15); }
  // per-warp region: the IP core's layout, then the reduction scratch, Wn and Q
  static constexpr size_t o_red = al(IpwSmem<float, M>::bytes);
  static constexpr size_t o_wn = o_red + al(sizeof(float) * NV);
  static constexpr size_t o_qf = o_wn + al(sizeof(float) * NN * KK);
  static constexpr size_t warp_bytes = o_qf + al(sizeof(float2) * M * M);
  static size_t smem(int T) { return al(sizeof(float) * NN * KK * (size_t)T) + BW_WARPS * warp_bytes; }
};

// Sum NV values over the warp's 32 lanes by recursive halving: after the five
// exchange steps lane l holds the totals of values [l * NV/32, (l+1) * NV/32)
// in v[0 .. NV/32). NV must be a multiple of 32. ~NV shuffles instead of the
// butterfly's 5 NV.
template <int NV>
__device__ __forceinline__ void warp_reduce_halving(float (&v)[NV], int lane) {
#pragma unroll
  for (int s = 0; s < 5; ++s) {
    const int o = 16 >> s, L = NV >> (s + 1);
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < L; ++i) {
      const float lo = v[i], hi = v[i + L];
      const float send = up ? lo : hi;
      const float keep = up ? hi : lo;
      v[i] = keep + __shfl_xor_sync(FM_FULL, send, o);
    }
  }
}

// y_m = max(sum_n lambda_n g_nm, floor), iy = 1/y (model_power, fm_nmf.cuh)
template <int M, int NN>
__device__ __forceinline__ void bw_power(const float (&l)[NN], const float (&gr)[NN][M], float fl,
                                         float (&y)[M], float (&iy)[M]) {
#pragma unroll
  for (int m = 0; m < M; ++m) {
    float s = 0.f;
#pragma unroll
    for (int n = 0; n < NN; ++n) s += l[n] * gr[n][m];
    y[m] = floor_max(s, fl);
    iy[m] = rcp_r(y[m]);
  }
}

template <int M, int NN, int KK>
__global__ void __launch_bounds__(32 * BW_WARPS, 2) k_binw(BinArgs<float> a) {
  pdl_entry();
  using Cf = BwCfg<M, NN, KK>;
  using L = IpwSmem<float, M>;
  constexpr int P = Cf::P;
  extern __shared__ __align__(16) unsigned char smb[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int b = blockIdx.y;
  const int T = a.T, F = a.F, K = a.K;
  float* Hs = reinterpret_cast<float*>(smb);  // [NN][KK][T]
  {  // stage H of mixture b (rows k >= K zero)
    const float* Hb = a.H + (size_t)b * NN * K * T;
    const int tot = NN * KK * T;
    for (int e = threadIdx.x; e < tot; e += 32 * BW_WARPS) {
      const int t = e % T, nk = e / T, k = nk % KK, n = nk / KK;
      Hs[e] = k < K ? Hb[((size_t)n * K + k) * T + t] : 0.f;
    }
  }
  __syncthreads();  // the only CTA barrier: the warps' bins are independent below
  unsigned char* sm = smb + Cf::al(sizeof(float) * NN * KK * (size_t)T) + (size_t)warp * Cf::warp_bytes;
  float* red = reinterpret_cast<float*>(sm + Cf::o_red);
  float* wn = reinterpret_cast<float*>(sm + Cf::o_wn);
  float2* Qf = reinterpret_cast<float2*>(sm + Cf::o_qf);
  double2* Vd = reinterpret_cast<double2*>(sm + L::o_Vd);
  float2* Vi = reinterpret_cast<float2*>(sm + L::o_Vi);
  double2* Qd = reinterpret_cast<double2*>(sm + L::o_Qd);
  float* gs = reinterpret_cast<float*>(sm + L::o_gs);
  float* cs = reinterpret_cast<float*>(sm + L::o_cs);
  const float fl = a.floorp[b];
  const unsigned it = *a.iter;
  const size_t FT = (size_t)F * T;
  const double invT = 1.0 / (double)T;
  for (int r = 0; r < a.rounds; ++r) {
    const int f = (blockIdx.x * a.rounds + r) * BW_WARPS + warp;
    if (f >= F) break;  // warp-uniform
    const size_t bf = (size_t)b * F + f;
    const float2* Xb = a.X + bf * T * M;
    float* xtb = a.xt + bf * T * M;
    // ---- bin state: Wn (zero-padded to KK), g, Q ------------------------------
    for (int e = lane; e < NN * KK; e += 32) {
      const int n = e / KK, k = e % KK;
      wn[e] = k < K ? a.Wn[((size_t)b * NN + n) * F * K + (size_t)f * K + k] : 0.f;
    }
    for (int e = lane; e < NN * M; e += 32)
      gs[e] = a.g[((size_t)b * NN + e / M) * F * M + (size_t)f * M + (e % M)];
    for (int e = lane; e < M * M; e += 32) Qd[e] = to_d2(a.Q[bf * M * M + e]);
    __syncwarp();
    // the weights of the current lambda (Wn, then W = Wn c, then the next Wn)
    // and the gains stay in shared memory: broadcast 16-B loads per frame
    // keep the frame loops under 128 registers
    auto wload = [&](float (&wr)[NN][KK]) {
#pragma unroll
      for (int n = 0; n < NN; ++n)
#pragma unroll
        for (int k = 0; k < KK; k += 4) {
          const float4 v = *reinterpret_cast<const float4*>(wn + n * KK + k);
          wr[n][k] = v.x; wr[n][k + 1] = v.y; wr[n][k + 2] = v.z; wr[n][k + 3] = v.w;
        }
    };
    auto gload = [&](float (&gr)[NN][M]) {
#pragma unroll
      for (int n = 0; n < NN; ++n) RowIO<float, M>::load(gs + n * M, gr[n]);
    };
    // lambda_n(t) = sum_k w[n][k] H[n][k][t] (sources.py:184-187)
    auto lam_at = [&](int t, float (&l)[NN]) {
      float wr[NN][KK];
      wload(wr);
#pragma unroll
      for (int n = 0; n < NN; ++n) {
        float s = 0.f;
#pragma unroll
        for (int k = 0; k < KK; ++k) s += wr[n][k] * Hs[(n * KK + k) * T + t];
        l[n] = s;
      }
    };
    // ---- E: gain statistics from lambda(Wn, H) (separate.py:217) --------------
    {
      float acc[Cf::NV_G];
#pragma unroll
      for (int i = 0; i < Cf::NV_G; ++i) acc[i] = 0.f;
      for (int t = lane; t < T; t += 32) {
        float l[NN], xv[M], y[M], iy[M], gr[NN][M];
        RowIO<float, M>::load(xtb + (size_t)t * M, xv);
        lam_at(t, l);
        gload(gr);
        bw_power<M, NN>(l, gr, fl, y, iy);
#pragma unroll
        for (int m = 0; m < M; ++m) {
          const float xr = xv[m] * iy[m] * iy[m];
#pragma unroll
          for (int n = 0; n < NN; ++n) {
            acc[(n * M + m) * 2] += l[n] * xr;
            acc[(n * M + m) * 2 + 1] += l[n] * iy[m];
          }
        }
      }
      warp_reduce_halving<Cf::NV_G>(acc, lane);
      constexpr int J = Cf::NV_G / 32;
#pragma unroll
      for (int j = 0; j < J; ++j) red[lane * J + j] = acc[j];
      __syncwarp();
      if (lane < NN * M) gs[lane] = gs[lane] * mu_factor(red[2 * lane], red[2 * lane + 1]);  // :218-220
      __syncwarp();
    }
    // ---- V: V_fm = (1/T) sum_t x x^H / y_ftm with the new gains ---------------
    {
      float2 acc[M][P];
#pragma unroll
      for (int m = 0; m < M; ++m)
#pragma unroll
        for (int p = 0; p < P; ++p) acc[m][p] = make_float2(0.f, 0.f);
      for (int t = lane; t < T; t += 32) {
        float2 x[M];
        float l[NN], y[M], iy[M], gr[NN][M];
        CRowIO<float, M>::load(Xb + (size_t)t * M, x);
        lam_at(t, l);
        gload(gr);
        bw_power<M, NN>(l, gr, fl, y, iy);
        int p = 0;
#pragma unroll
        for (int i = 0; i < M; ++i) {
#pragma unroll
          for (int j = i; j < M; ++j, ++p) {
            float2 pr;  // x_i conj(x_j)
            pr.x = x[i].x * x[j].x + x[i].y * x[j].y;
            pr.y = x[i].y * x[j].x - x[i].x * x[j].y;
#pragma unroll
            for (int m = 0; m < M; ++m) acc[m][p] = fma2(make_float2(iy[m], iy[m]), pr, acc[m][p]);
          }
        }
      }
      float v[Cf::NV_V];
#pragma unroll
      for (int m = 0; m < M; ++m)
#pragma unroll
        for (int p = 0; p < P; ++p) {
          v[(m * P + p) * 2] = acc[m][p].x;
          v[(m * P + p) * 2 + 1] = acc[m][p].y;
        }
#pragma unroll
      for (int i = 2 * M * P; i < Cf::NV_V; ++i) v[i] = 0.f;
      warp_reduce_halving<Cf::NV_V>(v, lane);
      constexpr int J = Cf::NV_V / 32;
#pragma unroll
      for (int j = 0; j < J; ++j) red[lane * J + j] = v[j];
      __syncwarp();
      for (int e = lane; e < M * P; e += 32) {  // mirrored, fp64 (retries) and fp32
        const int m = e / P;
        int i = 0, rr = e % P;
        while (rr >= M - i) {
          rr -= M - i;
          ++i;
        }
        const int j = i + rr;
        const double2 d = make_double2((double)red[2 * e] * invT, (double)red[2 * e + 1] * invT);
        Vd[(m * M + i) * M + j] = d;
        Vi[(m * M + i) * M + j] = make_float2((float)d.x, (float)d.y);
        if (i != j) {
          Vd[(m * M + j) * M + i] = make_double2(d.x, -d.y);
          Vi[(m * M + j) * M + i] = make_float2((float)d.x, (float)-d.y);
        }
      }
      __syncwarp();
    }
    // ---- IP, row / gain normalisation (spatial.py:181-199, separate.py:223-233)
    double ldet = 0.0;
    int code = 0, bad_m = 0;
    ipw_core<float, M>(sm, lane, NN, a.ip_sweeps, a.normalize, [](int, double2*) {}, ldet, code,
                       bad_m);
    if (code && lane == 0) report_status(a.status, it, bad_m, a.f_offset + f, code);
    __syncwarp();
    // absorb (sources.py:202-204): the state W = Wn c; it is also the W the
    // next iteration's statistics start from
    for (int e = lane; e < NN * KK; e += 32) wn[e] *= cs[e / KK];
    __syncwarp();
    for (int e = lane; e < NN * K; e += 32) {
      const int n = e / K, k = e % K;
      a.W[((size_t)b * NN + n) * F * K + (size_t)f * K + k] = wn[n * KK + k];
    }
    for (int e = lane; e < M * M; e += 32) {
      const float2 q = make_float2((float)Qd[e].x, (float)Qd[e].y);
      Qf[e] = q;
      a.Q[bf * M * M + e] = q;
    }
    for (int e = lane; e < NN * M; e += 32)
      a.g[((size_t)b * NN + e / M) * F * M + (size_t)f * M + (e % M)] = gs[e];
    if (lane == 0) a.ld_part[bf] = ldet;
    __syncwarp();
    // ---- P: x~ = |Q x|^2 (_kernels.py:339-350) --------------------------------
    {
      float2 q[M][M];
#pragma unroll
      for (int i = 0; i < M; ++i)
#pragma unroll
        for (int j = 0; j < M; ++j) q[i][j] = Qf[i * M + j];
      for (int t = lane; t < T; t += 32) {
        float2 x[M];
        CRowIO<float, M>::load(Xb + (size_t)t * M, x);
        float xv[M];
#pragma unroll
        for (int i = 0; i < M; ++i) {
          float2 s = make_float2(0.f, 0.f);
#pragma unroll
          for (int j = 0; j < M; ++j) {
            s = fma2(make_float2(q[i][j].x, q[i][j].x), x[j], s);
            s = fma2(make_float2(-q[i][j].y, q[i][j].y), make_float2(x[j].y, x[j].x), s);
          }
          xv[i] = s.x * s.x + s.y * s.y;
        }
        RowIO<float, M>::store(xtb + (size_t)t * M, xv);
      }
    }
    // ---- S: data term of the new state and the W statistics of the next W
    // step, phi H^T (_kernels.py:226-243, sources.py:191-194) ------------------
    {
      float acc[Cf::NV_W];
#pragma unroll
      for (int i = 0; i < Cf::NV_W; ++i) acc[i] = 0.f;
      double ll = 0.0;
      for (int t = lane; t < T; t += 32) {
        float xv[M], gr[NN][M];
        RowIO<float, M>::load(xtb + (size_t)t * M, xv);  // this lane's own x~ row
        float h[NN][KK], l[NN], y[M], iy[M];
        {
          float wr[NN][KK];
          wload(wr);
#pragma unroll
          for (int n = 0; n < NN; ++n) {
            float s = 0.f;
#pragma unroll
            for (int k = 0; k < KK; ++k) {
              h[n][k] = Hs[(n * KK + k) * T + t];
              s += wr[n][k] * h[n][k];
            }
            l[n] = s;
          }
        }
        gload(gr);
        bw_power<M, NN>(l, gr, fl, y, iy);
        float llt = 0.f;
#pragma unroll
        for (int m = 0; m < M; ++m) llt += -xv[m] * iy[m] - log_fast(y[m]);
        ll += (double)llt;
        float rr[M];
#pragma unroll
        for (int m = 0; m < M; ++m) rr[m] = xv[m] * iy[m] * iy[m];
#pragma unroll
        for (int n = 0; n < NN; ++n) {
          float p1 = 0.f, p2 = 0.f;
#pragma unroll
          for (int m = 0; m < M; ++m) {
            p1 += gr[n][m] * rr[m];
            p2 += gr[n][m] * iy[m];
          }
#pragma unroll
          for (int k = 0; k < KK; ++k) {
            acc[(n * KK + k) * 2] += p1 * h[n][k];
            acc[(n * KK + k) * 2 + 1] += p2 * h[n][k];
          }
        }
      }
      ll = warp_sum(ll);
      for (int e = lane; e < a.ntile; e += 32) a.ll_part[bf * a.ntile + e] = e == 0 ? ll : 0.0;
      warp_reduce_halving<Cf::NV_W>(acc, lane);
      constexpr int J = Cf::NV_W / 32;
#pragma unroll
      for (int j = 0; j < J; ++j) red[lane * J + j] = acc[j];
      __syncwarp();
      // W MU of the next iteration (sources.py:191-194) on the absorbed W
      for (int e = lane; e < NN * KK; e += 32) wn[e] *= mu_factor(red[2 * e], red[2 * e + 1]);
      __syncwarp();
      for (int e = lane; e < NN * K; e += 32) {
        const int n = e / K, k = e % K;
        a.Wn[((size_t)b * NN + n) * F * K + (size_t)f * K + k] = wn[n * KK + k];
      }
    }
    // ---- R: phi after that W step (separate.py:215), for the next H step ------
    {
      float* phib = a.phi + (size_t)b * 2 * NN * FT + (size_t)f * T;
      for (int t = lane; t < T; t += 32) {
        float xv[M], l[NN], y[M], iy[M], gr[NN][M];
        RowIO<float, M>::load(xtb + (size_t)t * M, xv);  // this lane's own x~ row
        lam_at(t, l);
        gload(gr);
        bw_power<M, NN>(l, gr, fl, y, iy);
        float rr[M];
#pragma unroll
        for (int m = 0; m < M; ++m) rr[m] = xv[m] * iy[m] * iy[m];
#pragma unroll
        for (int n = 0; n < NN; ++n) {
          float p1 = 0.f, p2 = 0.f;
#pragma unroll
          for (int m = 0; m < M; ++m) {
            p1 += gr[n][m] * rr[m];
            p2 += gr[n][m] * iy[m];
          }
          phib[(size_t)n * FT + t] = p1;
          phib[(size_t)(NN + n) * FT + t] = p2;
        }
      }
    }
    __syncwarp();
  }
}

}  // namespace fm
