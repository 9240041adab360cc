// fm_ipw.cuh -- k_ip for M <= 8: one warp per (bin, mixture), four bins per
// 128-thread CTA, no CTA-wide barrier (spatial.py:172-200, separate.py:222-233).
//
// Same mathematics as k_ip (fm_spatial.cuh): q = V_m^-1 (Q^-1 e_m), Q^-1 and
// log|det Q| from a pivoted Gauss-Jordan on [Q | I], the row updates applied
// to Q^-1 by Sherman-Morrison, log|det Q| by the determinant lemma, then the
// row / gain normalisation and the absorb into W. The M HPD inverses V_m^-1
// are one batched, entry-parallel Gauss-Jordan over all M matrices (M^3
// entries over the warp's 32 lanes), in fp32 for complex64 (as k_ip) and
// fp64 for complex128. A bin is a warp-private chain of ~3M short steps; the
// CTA's four warps (and the SM's other CTAs) interleave their chains instead
// of waiting on each other at __syncthreads.
#pragma once
#include "fm_common.cuh"
#include "fm_linalg.cuh"
#include "fm_spatial.cuh"

namespace fm {

template <typename R, int M> struct IpwSmem {  // one warp's region
  static constexpr size_t al(size_t x) { return (x + 15) & ~size_t(15); }
  using VC = typename std::conditional<sizeof(R) == 4, float2, double2>::type;  // V inverse type
  static constexpr size_t o_Vd = 0;                                             // fp64 V sums
  static constexpr size_t o_Vi = o_Vd + al(sizeof(double2) * M * M * M);        // V^-1 (VC)
  static constexpr size_t o_Qd = o_Vi + (sizeof(R) == 4 ? al(sizeof(VC) * M * M * M) : 0);
  static constexpr size_t o_Ai = o_Qd + al(sizeof(double2) * M * M);
  static constexpr size_t o_vec = o_Ai + al(sizeof(double2) * M * 2 * M);
  static constexpr size_t o_gs = o_vec + al(sizeof(double2) * 3 * M);
  static constexpr size_t o_cs = o_gs + al(sizeof(R) * NMAX * M);
  static constexpr size_t o_rown = o_cs + al(sizeof(R) * NMAX);
  static constexpr size_t o_d0 = o_rown + al(sizeof(double) * M + 2 * sizeof(int) * M);
  static constexpr size_t bytes = o_d0 + al(sizeof(float) * M * M);
};
constexpr int IPW_WARPS = 4;

// Batched in-place Gauss-Jordan inverse of M Hermitian positive-definite
// M x M matrices A[m][i][j] (no pivoting: HPD pivots are positive Schur
// diagonals; the pivot is real, its reciprocal 1/Re p). fail[m] = 1 if a pivot
// of matrix m is not positive and finite (the reference's "non-positive
// normalization", spatial.py:194-198).
template <typename C, int M>
__device__ void warp_inv_hpd_batch(C* A, int* fail, float* d0, float ratio, int lane) {
  using Rr = decltype(C().x);
  constexpr int MM = M * M, TOT = M * MM, NE = (TOT + 31) / 32;
  if (lane < M) fail[lane] = 0;
  for (int e = lane; e < MM; e += 32) d0[e] = ratio * (float)A[(e / M) * MM + (e % M) * (M + 1)].x;
  __syncwarp();
  for (int k = 0; k < M; ++k) {
    C nv[NE];
#pragma unroll
    for (int r = 0; r < NE; ++r) {
      const int e = lane + 32 * r;
      if (e < TOT) {
        const int m = e / MM, ij = e % MM, i = ij / M, j = ij % M;
        const C* Am = A + m * MM;
        const Rr p = Am[k * M + k].x;
        const Rr rp = Rr(1) / p;
        const C aik = Am[i * M + k], akj = Am[k * M + j], aij = Am[ij];
        const C akjr = cmake<C>(akj.x * rp, akj.y * rp);
        const C aikr = cmake<C>(aik.x * rp, aik.y * rp);
        const C other = cmake<C>(aij.x - (aik.x * akjr.x - aik.y * akjr.y),
                                 aij.y - (aik.x * akjr.y + aik.y * akjr.x));
        const bool rk = i == k, ck = j == k;
        C v = rk ? akjr : other;
        v = ck ? (rk ? cmake<C>(rp, 0.0) : cmake<C>(-aikr.x, -aikr.y)) : v;
        nv[r] = v;
        // not positive / finite, or (fp32) a pivot that lost all but ~3 digits
        // of its diagonal: the Schur complement is ill-conditioned
        if (rk && ck && (!(p > Rr(0)) || !isfinite(p) || p <= (Rr)d0[m * M + k])) fail[m] = 1;
      }
    }
    __syncwarp();
#pragma unroll
    for (int r = 0; r < NE; ++r) {
      const int e = lane + 32 * r;
      if (e < TOT) A[e] = nv[r];
    }
    __syncwarp();
  }
}

// The warp-private IP of one bin (A3 + the A4 row / gain normalisation) on
// the warp's IpwSmem region: Vi holds the M V_m (fp32 for complex64, else
// fp64 in Vd), Qd the bin's Q, gs its gains after the MU. fill64(m, Vm)
// writes V_m in fp64 into Vm for the fp32-pivot retry. Leaves the new Q in
// Qd, the normalised gains in gs, the gain scales in cs, and returns the
// status code (0 ok, 1 non-positive norm at bad_m, 2 singular Q) and
// log|det Q| of the result. Shared by k_ip_w and the per-bin schedule's
// k_binw (fm_bin.cuh).
template <typename R, int M, typename Fill64>
__device__ __forceinline__ void ipw_core(unsigned char* sm, int lane, int N, int ip_sweeps,
                                         int normalize, Fill64&& fill64, double& ldet, int& code,
                                         int& bad_m) {
  using L = IpwSmem<R, M>;
  using VC = typename L::VC;
  double2* Vd = reinterpret_cast<double2*>(sm + L::o_Vd);
  VC* Vi = sizeof(R) == 4 ? reinterpret_cast<VC*>(sm + L::o_Vi) : reinterpret_cast<VC*>(Vd);
  double2* Qd = reinterpret_cast<double2*>(sm + L::o_Qd);
  double2* Ai = reinterpret_cast<double2*>(sm + L::o_Ai);
  double2* ub = reinterpret_cast<double2*>(sm + L::o_vec);
  double2* qb = ub + M;
  double2* sk = qb + M;
  R* gs = reinterpret_cast<R*>(sm + L::o_gs);
  R* cs = reinterpret_cast<R*>(sm + L::o_cs);
  double* rown = reinterpret_cast<double*>(sm + L::o_rown);
  int* vfail = reinterpret_cast<int*>(rown + M);
  int* v64 = vfail + M;  // complex64: V_m^-1 kept in fp64 (Vd) after a retry
  float* d0 = reinterpret_cast<float*>(sm + L::o_d0);
  if (lane < NMAX) cs[lane] = R(1);
  __syncwarp();
  // ---- A3: iterative projection (spatial.py:181-199) -------------------------
  for (int e = lane; e < M * 2 * M; e += 32) {  // [Q | I] -> Q^-1 and log|det Q|
    const int r = e / (2 * M), c = e % (2 * M);
    Ai[e] = c < M ? Qd[r * M + c] : make_double2(c - M == r ? 1.0 : 0.0, 0.0);
  }
  __syncwarp();
  ldet = 0.0;
  const bool qok = warp_inv_pivot<M>(Ai, lane, &ldet);
  if (lane < M) v64[lane] = 0;
  warp_inv_hpd_batch<VC, M>(Vi, vfail, d0, sizeof(R) == 4 ? 1e-3f : 0.0f, lane);  // V_m^-1, all m
  if constexpr (sizeof(R) == 4) {
    // an fp32 pivot that is not positive (ill-conditioned V_m) is retried in
    // fp64 from the partials before the reference's error is raised
    for (int m = 0; m < M; ++m) {
      if (!vfail[m]) continue;  // warp-uniform
      double2* Vm = Vd + (size_t)m * M * M;
      fill64(m, Vm);  // V_m in fp64 (the caller's sums)
      __syncwarp();
      const bool ok = warp_inv_hpd<M>(Vm, lane);
      __syncwarp();
      if (lane == 0) {
        vfail[m] = ok ? 0 : 1;
        v64[m] = 1;
      }
      __syncwarp();
    }
  }
  double nprod = 1.0;
  code = qok ? 0 : 2;
  bad_m = 0;  // singular Q -> singular Q V at m = 0
  constexpr int GL = M <= 1 ? 32 : M <= 2 ? 16 : M <= 4 ? 8 : 4;  // lanes per row
  const int ri = lane / GL, sub = lane % GL;
  const bool rv = ri < M;
  for (int sw = 0; sw < ip_sweeps && code == 0; ++sw) {
    for (int m = 0; m < M; ++m) {
      if (vfail[m]) {
        code = 1;
        bad_m = m;
        break;
      }
      const VC* Vm = Vi + (size_t)m * M * M;
      const double2* Vm64 = Vd + (size_t)m * M * M;
      const bool use64 = sizeof(R) == 4 && v64[m];
      if (lane < M) ub[lane] = Ai[lane * 2 * M + M + m];  // u = Q^-1 e_m
      __syncwarp();
      double2 q = make_double2(0.0, 0.0);  // q = V_m^-1 u
      if (rv) {
#pragma unroll
        for (int j = sub; j < M; j += GL) {
          const VC v = Vm[ri * M + j];
          const double2 vv = use64 ? Vm64[ri * M + j] : make_double2((double)v.x, (double)v.y);
          q = cadd(q, cmul(vv, ub[j]));
        }
      }
#pragma unroll
      for (int o = GL / 2; o > 0; o >>= 1) {
        q.x += __shfl_xor_sync(FM_FULL, q.x, o);
        q.y += __shfl_xor_sync(FM_FULL, q.y, o);
      }
      double part = 0.0;
      if (rv && sub == 0) {
        const double2 u = ub[ri];
        part = q.x * u.x + q.y * u.y;  // Re(conj(q_i) u_i)
      }
      const double nrm = warp_sum(part);  // = q^H V q  (spatial.py:193)
      if (!(nrm > 0.0) || !isfinite(nrm)) {
        code = 1;
        bad_m = m;
        break;
      }
      const double isn = drsqrt(nrm);
      if (rv && sub == 0) {  // new row r = conj(q / sqrt(norm))  (spatial.py:199)
        const double2 r = make_double2(q.x * isn, -(q.y * isn));
        qb[ri] = r;
        Qd[m * M + ri] = r;
      }
      __syncwarp();
      double2 sv = make_double2(0.0, 0.0);  // s = (r Q^-1 - e_m^T) / sqrt(norm)
      if (rv) {
#pragma unroll
        for (int j = sub; j < M; j += GL) sv = cadd(sv, cmul(qb[j], Ai[j * 2 * M + M + ri]));
      }
#pragma unroll
      for (int o = GL / 2; o > 0; o >>= 1) {
        sv.x += __shfl_xor_sync(FM_FULL, sv.x, o);
        sv.y += __shfl_xor_sync(FM_FULL, sv.y, o);
      }
      if (rv && sub == 0) {
        if (ri == m) sv.x -= 1.0;
        sk[ri] = make_double2(sv.x * isn, sv.y * isn);
      }
      __syncwarp();
      for (int e = lane; e < M * M; e += 32) {  // Q^-1 -= u s / sqrt(norm)
        const int i = e / M, k = e % M;
        double2* d = Ai + i * 2 * M + M + k;
        *d = csub(*d, cmul(ub[i], sk[k]));
      }
      nprod *= nrm;  // log|det Q| += log sqrt(norm) (determinant lemma)
      if (nprod > 1e150 || nprod < 1e-150) {
        ldet += 0.5 * log(nprod);
        nprod = 1.0;
      }
      __syncwarp();
    }
  }
  ldet += 0.5 * log(nprod);
  // ---- A4: row normalisation, gain normalisation + absorb ---------------------
  if (normalize) {
    if (lane < M) {
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < M; ++j) {
        const double2 q2 = Qd[lane * M + j];
        s += q2.x * q2.x + q2.y * q2.y;
      }
      rown[lane] = sqrt(s);
    }
    __syncwarp();
    for (int e = lane; e < M * M; e += 32) {
      const double r = rown[e / M];
      Qd[e] = make_double2(Qd[e].x / r, Qd[e].y / r);
    }
    for (int e = lane; e < N * M; e += 32) {
      const double r = rown[e % M];
      gs[e] = (R)((double)gs[e] / (r * r));
    }
    double ls = 0.0;
    for (int m = 0; m < M; ++m) ls += log(rown[m]);
    ldet -= ls;
    __syncwarp();
    if (lane < N) {
      R s = 0;
#pragma unroll
      for (int m = 0; m < M; ++m) s += gs[lane * M + m];
      s = s > RT<R>::tiny() ? s : RT<R>::tiny();
      const R scl = R(M) / s;
#pragma unroll
      for (int m = 0; m < M; ++m) gs[lane * M + m] = gs[lane * M + m] * scl;
      cs[lane] = s / R(M);
    }
    __syncwarp();
  }
}

template <typename R, int M>
__global__ void __launch_bounds__(32 * IPW_WARPS) k_ip_w(IpArgs<R> a) {
  pdl_entry();
  using C = cplx<R>;
  using L = IpwSmem<R, M>;
  using VC = typename L::VC;
  extern __shared__ __align__(16) unsigned char small[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long gbf = (long long)blockIdx.x * IPW_WARPS + warp;  // b * F + f
  if (gbf >= (long long)a.B * a.F) return;  // warp-uniform: no CTA barrier below
  const int F = a.F, N = a.N, K = a.K;
  const int b = (int)(gbf / F), f = (int)(gbf % F);
  unsigned char* sm = small + (size_t)warp * L::bytes;
  double2* Vd = reinterpret_cast<double2*>(sm + L::o_Vd);
  VC* Vi = sizeof(R) == 4 ? reinterpret_cast<VC*>(sm + L::o_Vi) : reinterpret_cast<VC*>(Vd);
  double2* Qd = reinterpret_cast<double2*>(sm + L::o_Qd);
  R* gs = reinterpret_cast<R*>(sm + L::o_gs);
  R* cs = reinterpret_cast<R*>(sm + L::o_cs);
  C* Qg = a.Q + ((size_t)b * F + f) * M * M;
  R* gg = a.g + (size_t)b * N * F * M + (size_t)f * M;
  R* Wg = a.W + (size_t)b * (N - a.n0) * F * K + (size_t)f * K;
  const R* Wsg = a.Wsrc + (size_t)b * (N - a.n0) * F * K + (size_t)f * K;
  const unsigned it = *a.iter;
  const long long fglob = a.f_offset + f;
  {  // V_f = (1/T) sum over the segment partials (fixed order, fp64), mirrored
    constexpr int P = M * (M + 1) / 2;
    const C* vp = a.Vpart + ((size_t)b * F + f) * a.nseg * M * P;
    const double invT = 1.0 / (double)a.T;
    for (int e = lane; e < M * P; e += 32) {
      double2 acc = make_double2(0.0, 0.0);
      for (int q = 0; q < a.nseg; ++q) {
        const C c = vp[(size_t)q * M * P + e];
        acc.x += (double)c.x;
        acc.y += (double)c.y;
      }
      const int m = e / P;
      int i = 0, r = e % P;
      while (r >= M - i) {
        r -= M - i;
        ++i;
      }
      const int j = i + r;
      const double2 d = make_double2(acc.x * invT, acc.y * invT);
      if constexpr (sizeof(R) == 4) {
        Vi[((size_t)m * M + i) * M + j] = make_float2((float)d.x, (float)d.y);
        if (i != j) Vi[((size_t)m * M + j) * M + i] = make_float2((float)d.x, (float)-d.y);
      } else {
        Vd[((size_t)m * M + i) * M + j] = d;
        if (i != j) Vd[((size_t)m * M + j) * M + i] = make_double2(d.x, -d.y);
      }
    }
  }
  for (int e = lane; e < M * M; e += 32) Qd[e] = to_d2(Qg[e]);
  for (int e = lane; e < N * M; e += 32)
    gs[e] = a.gnew[(size_t)b * N * F * M + (size_t)(e / M) * F * M + (size_t)f * M + (e % M)];
  __syncwarp();
  double ldet = 0.0;
  int code = 0, bad_m = 0;
  ipw_core<R, M>(sm, lane, N, a.ip_sweeps, a.normalize,
                 [&](int m, double2* Vm) {  // V_m from the partials in fp64
                   constexpr int P = M * (M + 1) / 2;
                   const C* vp = a.Vpart + ((size_t)b * F + f) * a.nseg * M * P + (size_t)m * P;
                   for (int e = lane; e < P; e += 32) {
                     double2 acc = make_double2(0.0, 0.0);
                     for (int q = 0; q < a.nseg; ++q) {
                       const C c = vp[(size_t)q * M * P + e];
                       acc.x += (double)c.x;
                       acc.y += (double)c.y;
                     }
                     int i = 0, r = e;
                     while (r >= M - i) {
                       r -= M - i;
                       ++i;
                     }
                     const int j = i + r;
                     const double2 d = make_double2(acc.x / (double)a.T, acc.y / (double)a.T);
                     Vm[i * M + j] = d;
                     if (i != j) Vm[j * M + i] = make_double2(d.x, -d.y);
                   }
                 },
                 ldet, code, bad_m);
  if (code && lane == 0) report_status(a.status, it, bad_m, fglob, code);
  if (a.normalize) {
    __syncwarp();
    const int Nn = N - a.n0;
    for (int e = lane; e < Nn * K; e += 32) {
      const size_t wi = (size_t)(e / K) * F * K + e % K;
      Wg[wi] = Wsg[wi] * cs[a.n0 + e / K];  // sources.py:202-204
    }
    if (a.n0 && lane == 0) a.u[(size_t)b * F + f] *= cs[0];
  } else if (Wsg != Wg) {  // no absorb: the state W is the W-stepped one
    for (int e = lane; e < (N - a.n0) * K; e += 32) {
      const size_t wi = (size_t)(e / K) * F * K + e % K;
      Wg[wi] = Wsg[wi];
    }
  }
  __syncwarp();
  for (int e = lane; e < M * M; e += 32) Qg[e] = cmake<C>(Qd[e].x, Qd[e].y);
  for (int e = lane; e < N * M; e += 32) gg[(size_t)(e / M) * F * M + (e % M)] = gs[e];
  if (lane < NMAX) a.cs_out[((size_t)b * F + f) * NMAX + lane] = cs[lane];
  if (lane == 0) a.ld_part[(size_t)b * F + f] = ldet;
}

}  // namespace fm
