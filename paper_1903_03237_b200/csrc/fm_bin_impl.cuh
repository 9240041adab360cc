// fm_bin_impl.cuh -- launch logic of the per-bin schedule's k_binw
// (fm_bin.cuh), compiled in its own translation unit (fm_bin.cu).
#pragma once
#include "fm_bin.cuh"
#include "fm_impl.cuh"

namespace fm {

// bins per warp: enough CTAs for ~2 waves of 2 CTAs per SM, each staging its
// mixture's H once for up to 4 x 8 bins
inline int bin_rounds(const fm_dims* d) {
  const long long bins = d->B * d->F;
  long long r = bins / ((long long)BW_WARPS * 4 * 148);
  return (int)std::max<long long>(1, std::min<long long>(4, r));
}

template <typename R>
int Impl<R>::binw(const fm_dims* d, const fm_state* s, cudaStream_t st) {
  if constexpr (sizeof(R) != 4) {
    set_error("k_binw: complex64 only");
    return FM_EINVAL;
  } else {
    const Plan p = make_plan(d);
    unsigned char* w = reinterpret_cast<unsigned char*>(s->work);
    BinArgs<float> a;
    a.X = reinterpret_cast<const float2*>(s->X);
    a.xt = reinterpret_cast<float*>(s->xt);
    a.Q = reinterpret_cast<float2*>(s->Q);
    a.g = reinterpret_cast<float*>(s->g);
    a.W = reinterpret_cast<float*>(s->W);
    a.Wn = reinterpret_cast<float*>(w + p.off_wn);
    a.H = reinterpret_cast<const float*>(s->H);
    a.floorp = reinterpret_cast<const float*>(s->floor);
    a.phi = reinterpret_cast<float*>(w + p.off_phi);
    a.ll_part = reinterpret_cast<double*>(w + p.off_llp);
    a.ld_part = reinterpret_cast<double*>(w + p.off_ldp);
    a.iter = reinterpret_cast<const unsigned*>(w + p.off_cnt) + 1;
    a.status = reinterpret_cast<unsigned long long*>(s->status);
    a.B = (int)d->B; a.F = (int)d->F; a.T = (int)d->T; a.N = (int)d->N; a.K = (int)d->K;
    a.f_offset = d->f_offset;
    a.normalize = d->normalize;
    a.ip_sweeps = d->ip_sweeps;
    a.rounds = bin_rounds(d);
    a.ntile = p.ntile;
    const unsigned gx = (unsigned)((d->F + (long long)BW_WARPS * a.rounds - 1) / ((long long)BW_WARPS * a.rounds));
    const dim3 grid(gx, (unsigned)d->B);
    if (!bin_eligible(d)) {
      set_error("k_binw: dims outside the per-bin schedule");
      return FM_EINVAL;
    }
    FM_DISPATCH_M(d->M, {
      if constexpr (MM <= 4) {
        auto go = [&](auto kern, size_t sm) -> int {
          if (int rc = ensure_smem(kern, sm)) return rc;
          launch_pdl(kern, grid, dim3(32 * BW_WARPS), sm, st, a);
          FM_CHECK_LAUNCH("k_binw");
          return FM_OK;
        };
        int rc = FM_OK;
        if (d->N == 2) rc = go(k_binw<MM, 2, 8>, BwCfg<MM, 2, 8>::smem((int)d->T));
        else if (d->N == 3) rc = go(k_binw<MM, 3, 8>, BwCfg<MM, 3, 8>::smem((int)d->T));
        else rc = go(k_binw<MM, 4, 8>, BwCfg<MM, 4, 8>::smem((int)d->T));
        if (rc) return rc;
      }
    });
    return FM_OK;
  }
}

}  // namespace fm
