// fm_linalg.cuh -- warp-level M x M complex dense linear algebra in fp64.
//
// The reference solves the IP row system with numpy.linalg.solve (LAPACK zgesv:
// partial-pivot LU, zgetrf, then zgetrs) at spatial.py:188, takes log|det Q|
// with numpy.linalg.slogdet (zgetrf, separate.py:238 / spatial.py:241) and
// inverts Q with numpy.linalg.inv (zgesv against I, separate.py:122). These
// routines restate that arithmetic for one M x M system per warp (M <= 16),
// matrices in shared memory, fp64 in both precision modes.
#pragma once
#include "fm_common.cuh"

namespace fm {

#define FM_FULL 0xffffffffu

// Partial-pivot LU of the M x M block of A (row stride LD) by one warp, with
// the same row operations applied to columns [M, ncol) (right-hand sides).
// Pivot = first index of max |re|+|im| (izamax in zgetf2); multipliers are
// a * (1/pivot) (zgetf2's reciprocal scaling); the RHS update order is the
// column-oriented one of ztrsm('L','L','N','U'). Returns false on an exactly
// zero pivot (zgetrf info > 0 -> numpy LinAlgError "Singular matrix").
// If logabs != nullptr, *logabs (lane 0) = sum_k log|u_kk| (slogdet).
template <int M>
__device__ bool warp_lu(double2* A, int LD, int ncol, int lane, double* logabs) {
  double la = 0.0;
  for (int k = 0; k < M; ++k) {
    double v = -1.0;
    int idx = lane;
    if (lane >= k && lane < M) v = cabs1(A[lane * LD + k]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      double ov = __shfl_xor_sync(FM_FULL, v, o);
      int oi = __shfl_xor_sync(FM_FULL, idx, o);
      if (ov > v || (ov == v && oi < idx)) {
        v = ov;
        idx = oi;
      }
    }
    if (!(v > 0.0)) {  // zero (or NaN) pivot column
      if (logabs) *logabs = -INFINITY;
      return false;
    }
    if (idx != k) {
      for (int c = lane; c < ncol; c += 32) {
        double2 t = A[k * LD + c];
        A[k * LD + c] = A[idx * LD + c];
        A[idx * LD + c] = t;
      }
    }
    __syncwarp();
    const double2 piv = A[k * LD + k];
    la += log(hypot(piv.x, piv.y));
    const double2 rp = cdiv(make_double2(1.0, 0.0), piv);
    if (lane > k && lane < M) {
      const double2 l = cmul(A[lane * LD + k], rp);
      A[lane * LD + k] = l;
      for (int c = k + 1; c < ncol; ++c) A[lane * LD + c] = csub(A[lane * LD + c], cmul(l, A[k * LD + c]));
    }
    __syncwarp();
  }
  if (logabs) *logabs = la;
  return true;
}

// Back substitution U x = b for the single right-hand side in column M
// (ztrsm('L','U','N','N') order); x written to smem x[0..M).
template <int M>
__device__ void warp_backsub1(const double2* A, int LD, int lane, double2* x) {
  double2 b = make_double2(0.0, 0.0);
  if (lane < M) b = A[lane * LD + M];
  for (int k = M - 1; k >= 0; --k) {
    double2 xk = make_double2(0.0, 0.0);
    if (lane == k) xk = cdiv(b, A[k * LD + k]);
    xk.x = __shfl_sync(FM_FULL, xk.x, k);
    xk.y = __shfl_sync(FM_FULL, xk.y, k);
    if (lane < k) b = csub(b, cmul(xk, A[lane * LD + k]));
    if (lane == k) x[k] = xk;
  }
  __syncwarp();
}

// Back substitution for the M right-hand sides in columns [M, 2M): lane j
// solves column j sequentially. Result overwrites those columns.
template <int M>
__device__ void warp_backsubM(double2* A, int LD, int lane) {
  if (lane < M) {
    const int c = M + lane;
    for (int k = M - 1; k >= 0; --k) {
      double2 xk = cdiv(A[k * LD + c], A[k * LD + k]);
      A[k * LD + c] = xk;
      for (int i = 0; i < k; ++i) A[i * LD + c] = csub(A[i * LD + c], cmul(xk, A[i * LD + k]));
    }
  }
  __syncwarp();
}

// One IP sweep set (spatial.py:181-199) for one frequency bin, by one warp.
// Qd: M x M (row m = q_m^H), fp64, updated in place row by row (Gauss-Seidel:
// row m's system uses rows < m already updated, spatial.py:183-188).
// V: M x M x M weighted covariances (any complex type), V[(m*M+i)*M+j].
// A: scratch M x (M+1); x: scratch M. Returns 0 or an FM_STATUS code and the
// failing row in *bad_m.
template <int M, typename CV>
__device__ int warp_ip_update(double2* Qd, const CV* V, double2* A, double2* x, int sweeps,
                              int lane, int* bad_m) {
  constexpr int LD = M + 1;
  for (int sw = 0; sw < sweeps; ++sw) {
    for (int m = 0; m < M; ++m) {
      const CV* Vm = V + (size_t)m * M * M;
      // A = Q_f V_fm ; rhs = e_m  (spatial.py:184-188)
      for (int e = lane; e < M * M; e += 32) {
        const int r = e / M, c = e % M;
        double2 s = make_double2(0.0, 0.0);
#pragma unroll
        for (int k = 0; k < M; ++k) s = cadd(s, cmul(Qd[r * M + k], to_d2(Vm[k * M + c])));
        A[r * LD + c] = s;
      }
      if (lane < M) A[lane * LD + M] = make_double2(lane == m ? 1.0 : 0.0, 0.0);
      __syncwarp();
      if (!warp_lu<M>(A, LD, M + 1, lane, nullptr)) {
        *bad_m = m;
        return 2;  // FM_STATUS_SINGULAR_QV
      }
      warp_backsub1<M>(A, LD, lane, x);
      // norm = Re(q^H V q)  (spatial.py:193)
      double part = 0.0;
      if (lane < M) {
        double2 s = make_double2(0.0, 0.0);
#pragma unroll
        for (int j = 0; j < M; ++j) s = cadd(s, cmul(to_d2(Vm[lane * M + j]), x[j]));
        const double2 xi = x[lane];
        part = xi.x * s.x + xi.y * s.y;  // Re(conj(x_i) s_i)
      }
      const double norm = warp_sum(part);
      if (!(norm > 0.0) || !isfinite(norm)) {  // spatial.py:194-198
        *bad_m = m;
        return 1;  // FM_STATUS_NONPOS_NORM
      }
      const double sn = sqrt(norm);
      if (lane < M) {  // Q[m, :] = conj(q / sqrt(norm))  (spatial.py:199)
        const double2 xv = x[lane];
        Qd[m * M + lane] = make_double2(xv.x / sn, -(xv.y / sn));
      }
      __syncwarp();
    }
  }
  return 0;
}

}  // namespace fm

namespace fm {

// In-place Gauss-Jordan inverse of one M x M Hermitian positive-definite
// matrix (row-major in smem) by one warp, entry-parallel, no pivoting (HPD
// pivots are the positive Schur-complement diagonals). Returns false if a
// pivot is not positive/finite (rank-deficient V_fm: the reference's
// "non-positive normalization", spatial.py:194-198).
template <int M>
__device__ bool warp_inv_hpd(double2* A, int lane) {
  constexpr int NE = (M * M + 31) / 32;
  for (int k = 0; k < M; ++k) {
    const double2 p = A[k * M + k];
    if (!(p.x > 0.0) || !isfinite(p.x)) return false;
    const double2 rp = crcp(p);
    double2 nv[NE];
#pragma unroll
    for (int r = 0; r < NE; ++r) {
      const int e = lane + 32 * r;
      if (e < M * M) {
        const int i = e / M, j = e % M;
        const double2 aik = A[i * M + k], akj = A[k * M + j], aij = A[e];
        // branch-free select (lanes of one warp take different cases)
        const double2 akjr = cmul(akj, rp);
        const double2 aikr = cmul(aik, rp);
        const double2 other = csub(aij, cmul(aik, akjr));
        const bool rk = i == k, ck = j == k;
        double2 v = rk ? akjr : other;
        v = ck ? (rk ? rp : make_double2(-aikr.x, -aikr.y)) : v;
        nv[r] = v;
      }
    }
    __syncwarp();
#pragma unroll
    for (int r = 0; r < NE; ++r) {
      const int e = lane + 32 * r;
      if (e < M * M) A[e] = nv[r];
    }
    __syncwarp();
  }
  return true;
}

// warp_inv_hpd in fp32 (complex64 mode, M <= 8): the V_fm it inverts were
// accumulated in fp32, and the fp32 pipe (2x the fp64 rate, 4-cycle FMA
// latency) keeps the parallel inversion phase of k_ip off the fp64 pipe that
// all resident CTAs enter together. Same algorithm and selects as above.
template <int M>
__device__ bool warp_inv_hpd_f32(float2* A, int lane) {
  constexpr int NE = (M * M + 31) / 32;
  for (int k = 0; k < M; ++k) {
    const float2 p = A[k * M + k];
    if (!(p.x > 0.0f) || !isfinite(p.x)) return false;
    // HPD: the pivot is real; 1/Re p (no |p|^2, which halves the fp32 range)
    const float rpx = frcp_nr(p.x);
    const float2 rp = make_float2(rpx, 0.0f);
    float2 nv[NE];
#pragma unroll
    for (int r = 0; r < NE; ++r) {
      const int e = lane + 32 * r;
      if (e < M * M) {
        const int i = e / M, j = e % M;
        const float2 aik = A[i * M + k], akj = A[k * M + j], aij = A[e];
        const float2 akjr = make_float2(akj.x * rpx, akj.y * rpx);  // the pivot is real
        const float2 aikr = make_float2(aik.x * rpx, aik.y * rpx);
        const float2 other = make_float2(aij.x - (aik.x * akjr.x - aik.y * akjr.y),
                                         aij.y - (aik.x * akjr.y + aik.y * akjr.x));
        const bool rk = i == k, ck = j == k;
        float2 v = rk ? akjr : other;
        v = ck ? (rk ? rp : make_float2(-aikr.x, -aikr.y)) : v;
        nv[r] = v;
      }
    }
    __syncwarp();
#pragma unroll
    for (int r = 0; r < NE; ++r) {
      const int e = lane + 32 * r;
      if (e < M * M) A[e] = nv[r];
    }
    __syncwarp();
  }
  return true;
}

// Gauss-Jordan with partial pivoting (izamax-style first max |re|+|im|) on
// the augmented [Q | I] (M x 2M, row-major) by one warp; on success the
// right half holds Q^-1 and *logabs = sum_k log|pivot_k| = log|det Q|
// (the LU pivots; slogdet, separate.py:238).
template <int M, typename C2, bool PRODLOG = false>
__device__ bool warp_inv_pivot(C2* A, int lane, double* logabs) {
  using Rc = decltype(C2().x);
  constexpr int W2 = 2 * M;
  constexpr int NE = (M * W2 + 31) / 32;
  // PRODLOG (k_ip): log|det| = 1/2 log prod |pivot|^2, the product carried in
  // fp64 and one log taken when it leaves [1e-150, 1e150] or at the end -- a
  // double log per elimination step sat on warp 0's serial chain (c1 k_ip 22.5
  // -> 20.5 us). The warp-per-bin callers (ipw_core: k_ip_w, k_binw) keep the
  // log per step: with every warp on its own bin the logs overlap other warps'
  // work, and the guarded form measured slower there (c2 k_binw 4.03 -> 4.23 ms)
  double la = 0.0, pprod = 1.0;
  for (int k = 0; k < M; ++k) {
    Rc v = Rc(-1);
    int idx = lane;
    if (lane >= k && lane < M) v = cabs1(A[lane * W2 + k]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const Rc ov = __shfl_xor_sync(FM_FULL, v, o);
      const int oi = __shfl_xor_sync(FM_FULL, idx, o);
      if (ov > v || (ov == v && oi < idx)) {
        v = ov;
        idx = oi;
      }
    }
    if (!(v > Rc(0))) {
      *logabs = -INFINITY;
      return false;
    }
    if (idx != k) {
      for (int c = lane; c < W2; c += 32) {
        const C2 t = A[k * W2 + c];
        A[k * W2 + c] = A[idx * W2 + c];
        A[idx * W2 + c] = t;
      }
    }
    __syncwarp();
    const C2 piv = A[k * W2 + k];
    if constexpr (PRODLOG) {
      pprod *= (double)piv.x * piv.x + (double)piv.y * piv.y;
      if (pprod > 1e150 || pprod < 1e-150) {
        la += 0.5 * log(pprod);
        pprod = 1.0;
      }
    } else {
      la += 0.5 * log((double)piv.x * piv.x + (double)piv.y * piv.y);
    }
    const C2 rp = crcp(piv);
    C2 nv[NE];
#pragma unroll
    for (int r = 0; r < NE; ++r) {
      const int e = lane + 32 * r;
      if (e < M * W2) {
        const int i = e / W2, j = e % W2;
        const C2 akj = cmul(A[k * W2 + j], rp);
        nv[r] = (i == k) ? akj : csub(A[e], cmul(A[i * W2 + k], akj));
      }
    }
    __syncwarp();
#pragma unroll
    for (int r = 0; r < NE; ++r) {
      const int e = lane + 32 * r;
      if (e < M * W2) A[e] = nv[r];
    }
    __syncwarp();
  }
  if constexpr (PRODLOG) la += 0.5 * log(pprod);
  *logabs = la;
  return true;
}


// Cyclic complex Jacobi eigensolver for one Hermitian M x M matrix in shared
// memory, run by one warp (fp64; lanes own the rows / columns a rotation
// touches). On return G is diagonal (eigenvalues on the diagonal, unsorted)
// and the columns of V are the eigenvectors: G_in = V diag(G) V^H.
template <int M>
__device__ void warp_jacobi_eigh(double2* G, double2* V, int lane) {
  for (int e = lane; e < M * M; e += 32) V[e] = make_double2(e / M == e % M ? 1.0 : 0.0, 0.0);
  __syncwarp();
  for (int sweep = 0; sweep < 40; ++sweep) {
    double off = 0.0, dia = 0.0;
    for (int e = lane; e < M * M; e += 32) {
      const double2 v = G[e];
      if (e / M == e % M) dia += v.x * v.x;
      else off += v.x * v.x + v.y * v.y;
    }
    off = warp_sum(off);
    dia = warp_sum(dia);
    if (!(off > 1e-30 * dia) || off == 0.0) break;
    for (int p = 0; p < M - 1; ++p) {
      for (int q = p + 1; q < M; ++q) {
        const double2 apq = G[p * M + q];
        const double mag = sqrt(apq.x * apq.x + apq.y * apq.y);
        if (!(mag > 1e-300)) continue;
        const double app = G[p * M + p].x, aqq = G[q * M + q].x;
        // D = diag(1, e^{-i phi}) makes the pair real; then the real rotation
        // P = [[c, s], [-s, c]] with t = tan(theta) zeroes it (J = D P)
        const double ep_r = apq.x / mag, ep_i = apq.y / mag;  // e^{i phi}
        const double tau = (aqq - app) / (2.0 * mag);
        const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
        const double c = 1.0 / sqrt(1.0 + t * t), sn = t * c;
        // columns: A J  (col_p' = c col_p - s e^{-i phi} col_q, col_q' = s col_p + c e^{-i phi} col_q)
        if (lane < M) {
          const double2 gp = G[lane * M + p], gq = G[lane * M + q];
          const double2 gqe = make_double2(gq.x * ep_r + gq.y * ep_i, gq.y * ep_r - gq.x * ep_i);
          G[lane * M + p] = make_double2(c * gp.x - sn * gqe.x, c * gp.y - sn * gqe.y);
          G[lane * M + q] = make_double2(sn * gp.x + c * gqe.x, sn * gp.y + c * gqe.y);
          const double2 vp = V[lane * M + p], vq = V[lane * M + q];
          const double2 vqe = make_double2(vq.x * ep_r + vq.y * ep_i, vq.y * ep_r - vq.x * ep_i);
          V[lane * M + p] = make_double2(c * vp.x - sn * vqe.x, c * vp.y - sn * vqe.y);
          V[lane * M + q] = make_double2(sn * vp.x + c * vqe.x, sn * vp.y + c * vqe.y);
        }
        __syncwarp();
        // rows: J^H (A J)  (row_p' = c row_p - s e^{i phi} row_q, row_q' = s row_p + c e^{i phi} row_q)
        if (lane < M) {
          const double2 gp = G[p * M + lane], gq = G[q * M + lane];
          const double2 gqe = make_double2(gq.x * ep_r - gq.y * ep_i, gq.y * ep_r + gq.x * ep_i);
          G[p * M + lane] = make_double2(c * gp.x - sn * gqe.x, c * gp.y - sn * gqe.y);
          G[q * M + lane] = make_double2(sn * gp.x + c * gqe.x, sn * gp.y + c * gqe.y);
        }
        __syncwarp();
        if (lane == 0) {
          G[p * M + q] = make_double2(0.0, 0.0);
          G[q * M + p] = make_double2(0.0, 0.0);
          G[p * M + p].y = 0.0;
          G[q * M + q].y = 0.0;
        }
        __syncwarp();
      }
    }
  }
}

}  // namespace fm
