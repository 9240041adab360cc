// fm_fused_impl.cuh -- launch logic of the fused statistics passes
// (fm_fused.cuh), compiled in their own translation units (fm_fused_f32.cu,
// fm_fused_f64.cu) so the kernel instantiations build in parallel with the
// rest of the library.
#pragma once
#include <type_traits>

#include "fm_impl.cuh"

namespace fm {

template <int V> using ic = std::integral_constant<int, V>;

// Shapes with compile-time source / basis counts (fully unrolled loops): the
// BASELINE configs' (M pad, N, K4) -- c0 (4, 2, 8), c2 (4, 3, 8), c1 (8, 4, 16),
// c3 (16, 6, 32) -- at 8 bins per CTA. Everything else runs the generic build
// (NN = KC = 0) of the same kernels.
template <typename R, int MP, typename Fn>
inline int with_shape(int N, int K4, int FB, Fn&& fn) {
  if (FB == 8) {
    if constexpr (MP == 4) {
      if (N == 2 && K4 == 8) return fn(ic<2>{}, ic<8>{});
      if constexpr (sizeof(R) == 4) {
        if (N == 3 && K4 == 8) return fn(ic<3>{}, ic<8>{});
      }
    } else if constexpr (MP == 8 && sizeof(R) == 4) {
      if (N == 4 && K4 == 16) return fn(ic<4>{}, ic<16>{});
    } else if constexpr (MP == 16 && sizeof(R) == 4) {
      if (N == 6 && K4 == 32) return fn(ic<6>{}, ic<32>{});
    }
  }
  return fn(ic<0>{}, ic<0>{});
}

// items per thread of k_hpass (8 warps) / per lane of k_bpass for a
// compile-time (N, K4); 0 = take the plan's runtime value
constexpr int hp_it(int NN, int KC) { return NN ? (NN * (KC / hp_kch(KC)) + 7) / 8 : 0; }
constexpr int bp_it(int NN, int KC) {
  return NN ? (NN * 4 * (KC / 4) <= 256 ? 1 : (NN * 4 * (KC / 4) + 255) / 256) : 0;
}

template <typename R>
int Impl<R>::hstore(const fm_dims* d, const fm_state* s, const void* hbuf, cudaStream_t st) {
  const Plan p = make_plan(d);
  unsigned char* w = reinterpret_cast<unsigned char*>(s->work);
  const long long total = d->B * d->N * d->T * (long long)k4_of((int)d->K);
  launch_pdl(k_hstore<R>, dim3((unsigned)((total + 255) / 256)), dim3(256), 0, st,
             reinterpret_cast<R*>(s->H), reinterpret_cast<R*>(w + p.off_ht),
             reinterpret_cast<const R*>(hbuf), (int)d->N, (int)d->K, (int)d->T, total,
             hbuf ? 1 : 0);
  FM_CHECK_LAUNCH("k_hstore");
  return FM_OK;
}

template <typename R>
int Impl<R>::hpass(const fm_dims* d, const fm_state* s, int mode, void* hout, cudaStream_t st) {
  const Plan p = make_plan(d);
  unsigned char* w = reinterpret_cast<unsigned char*>(s->work);
  HpArgs<R> a;
  a.xt = reinterpret_cast<const R*>(s->xt);
  a.W = reinterpret_cast<const R*>(w + p.off_wn);
  a.H = reinterpret_cast<R*>(s->H);
  a.Ht = reinterpret_cast<R*>(w + p.off_ht);
  a.g = reinterpret_cast<const R*>(s->g);
  a.floorp = reinterpret_cast<const R*>(s->floor);
  a.part = reinterpret_cast<R*>(w + p.off_hpart2);
  a.cnt = reinterpret_cast<unsigned*>(w + p.off_hcnt2);
  a.hout = reinterpret_cast<R*>(hout);
  a.F = (int)d->F; a.T = (int)d->T; a.N = (int)d->N; a.K = (int)d->K; a.M = (int)d->M;
  a.mode = mode;
  a.HFR = p.hHFR; a.NS = p.hNS; a.NG = p.hNG; a.S = p.hS;
  const dim3 grid((unsigned)p.htl, (unsigned)(d->B * p.hNG), (unsigned)p.hHS);
  const int nspec = p.hNG == 1 ? (int)d->N : 0;  // specialised builds accumulate every source
  FM_DISPATCH_MP(d->M, {
    if (int rc = with_shape<R, MP>(nspec, k4_of((int)d->K), p.FB, [&](auto nn, auto kc) -> int {
          constexpr int NN = decltype(nn)::value, KC = decltype(kc)::value;
          if constexpr (NN > 0) {
            constexpr int IT = hp_it(NN, KC);
            if (int rc = ensure_smem(k_hpass<R, MP, IT, NN, KC>, p.smem_h)) return rc;
            launch_pdl(k_hpass<R, MP, IT, NN, KC>, grid, dim3(32 * p.FB), p.smem_h, st, a);
            FM_CHECK_LAUNCH("k_hpass");
          } else {
            FM_DISPATCH_IT(p.hIT, {
              if constexpr (IT <= 4) {
                if (int rc = ensure_smem(k_hpass<R, MP, IT, 0, 0>, p.smem_h)) return rc;
                launch_pdl(k_hpass<R, MP, IT, 0, 0>, grid, dim3(32 * p.FB), p.smem_h, st, a);
                FM_CHECK_LAUNCH("k_hpass");
              }
            });
          }
          return FM_OK;
        }))
      return rc;
  });
  return FM_OK;
}

template <typename R>
int Impl<R>::gpass(const fm_dims* d, const fm_state* s, cudaStream_t st) {
  const Plan p = make_plan(d);
  unsigned char* w = reinterpret_cast<unsigned char*>(s->work);
  GpArgs<R> a;
  a.xt = reinterpret_cast<const R*>(s->xt);
  a.W = reinterpret_cast<const R*>(w + p.off_wn);
  a.Ht = reinterpret_cast<const R*>(w + p.off_ht);
  a.g = reinterpret_cast<const R*>(s->g);
  a.floorp = reinterpret_cast<const R*>(s->floor);
  a.lam = reinterpret_cast<R*>(w + p.off_lam);
  a.part = reinterpret_cast<R*>(w + p.off_gpart);
  a.F = (int)d->F; a.T = (int)d->T; a.N = (int)d->N; a.K = (int)d->K; a.M = (int)d->M;
  a.TR = p.gTR; a.S = p.gS;
  const dim3 grid((unsigned)p.gseg, (unsigned)p.nfb, (unsigned)d->B);
  FM_DISPATCH_MP(d->M, {
    if (int rc = with_shape<R, MP>((int)d->N, k4_of((int)d->K), p.FB, [&](auto nn, auto kc) -> int {
          constexpr int NN = decltype(nn)::value, KC = decltype(kc)::value;
          if (int rc = ensure_smem(k_gpass<R, MP, NN, KC>, p.smem_g)) return rc;
          launch_pdl(k_gpass<R, MP, NN, KC>, grid, dim3(32 * p.FB), p.smem_g, st, a);
          FM_CHECK_LAUNCH("k_gpass");
          return FM_OK;
        }))
      return rc;
  });
  return FM_OK;
}

template <typename R>
int Impl<R>::bpass(const fm_dims* d, const fm_state* s, cudaStream_t st) {
  const Plan p = make_plan(d);
  unsigned char* w = reinterpret_cast<unsigned char*>(s->work);
  BpArgs<R> a;
  a.X = reinterpret_cast<const C*>(s->X);
  a.xt = reinterpret_cast<R*>(s->xt);
  a.Q = reinterpret_cast<const C*>(s->Q);
  a.g = reinterpret_cast<const R*>(s->g);
  a.W = reinterpret_cast<const R*>(s->W);
  a.Ht = reinterpret_cast<const R*>(w + p.off_ht);
  a.floorp = reinterpret_cast<const R*>(s->floor);
  a.Wn = reinterpret_cast<R*>(w + p.off_wn);
  a.part = reinterpret_cast<R*>(w + p.off_wpart);
  a.cnt = reinterpret_cast<unsigned*>(w + p.off_bcnt);
  a.llp = reinterpret_cast<double*>(w + p.off_llp);
  a.F = (int)d->F; a.T = (int)d->T; a.N = (int)d->N; a.K = (int)d->K; a.M = (int)d->M;
  a.TR = p.bTR; a.S = p.bS;
  static const int dbg = [] { const char* e = getenv("FM_BP_DBG"); return e ? atoi(e) : 0; }();
  a.dbg = dbg;
  const dim3 grid((unsigned)p.bseg, (unsigned)p.nfb, (unsigned)d->B);
  FM_DISPATCH_MP(d->M, {
    if (int rc = with_shape<R, MP>((int)d->N, k4_of((int)d->K), p.FB, [&](auto nn, auto kc) -> int {
          constexpr int NN = decltype(nn)::value, KC = decltype(kc)::value;
          if constexpr (NN > 0) {
            constexpr int IT = bp_it(NN, KC);
            if (int rc = ensure_smem(k_bpass<R, MP, IT, NN, KC>, p.smem_b)) return rc;
            launch_pdl(k_bpass<R, MP, IT, NN, KC>, grid, dim3(32 * p.FB), p.smem_b, st, a);
            FM_CHECK_LAUNCH("k_bpass");
          } else {
            FM_DISPATCH_IT(p.bIT, {
              if constexpr (IT <= 2) {
                if (int rc = ensure_smem(k_bpass<R, MP, IT, 0, 0>, p.smem_b)) return rc;
                launch_pdl(k_bpass<R, MP, IT, 0, 0>, grid, dim3(32 * p.FB), p.smem_b, st, a);
                FM_CHECK_LAUNCH("k_bpass");
              }
            });
          }
          return FM_OK;
        }))
      return rc;
  });
  return FM_OK;
}

}  // namespace fm
