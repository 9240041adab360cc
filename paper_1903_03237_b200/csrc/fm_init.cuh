// fm_init.cuh -- the reference's default spatial initialisation on the device
// (SURVEY §8(f) item 1):
//   G1_f = clamp_psd( (1/T) sum_t x x^H )        spatial.py:93, linalg.py:85-94
//   w, U = hermitian_eig(G1_f)  (descending)      linalg.py:23-33
//   Q_f = U^H                                     spatial.py:100-105, 109-121
// One CTA per bin: all threads accumulate the SCM in fp64 (fixed-order slice
// reduction), then warp 0 diagonalises it with cyclic complex Jacobi
// rotations (fp64, lanes own rows / columns of each rotation), sorts the
// eigenvalues descending and writes Q (rows = conjugated eigenvectors) and
// the clamped eigenvalues. Eigenvectors are unique up to a phase per column;
// every downstream quantity (x~, the likelihood, the images) is invariant to
// that phase, which is how the tests compare with numpy's eigh.
// grid (F, B), block 256.
#pragma once
#include "fm_common.cuh"

namespace fm {

template <typename R> struct InitArgs {
  const cplx<R>* X;  // (B, F, T, M) scaled observation
  cplx<R>* Q;        // (B, F, M, M) out
  double* w;         // (B, F, M) out: clamped eigenvalues, descending (may be null)
  int F, T;
};

template <typename R, int M>
__global__ void __launch_bounds__(256) k_spatial_init(InitArgs<R> a) {
  using C = cplx<R>;
  constexpr int P = M * (M + 1) / 2, S = 256 / P;
  __shared__ double2 G[M * M];  // the SCM, then the rotated matrix
  __shared__ double2 V[M * M];  // eigenvectors (columns)
  __shared__ double2 red[S > 0 ? S * P : 1];
  __shared__ int perm[M];
  const int f = blockIdx.x, b = blockIdx.y, tid = threadIdx.x, lane = tid & 31;
  const int T = a.T;
  const C* Xb = a.X + ((size_t)b * a.F + f) * T * M;
  // ---- SCM: pair p = (i <= k), slice s over frames, fixed-order slice sum
  {
    const int p = tid % P, s = tid / P;
    int i = 0, r = p;
    while (r >= M - i) {
      r -= M - i;
      ++i;
    }
    const int k = i + r;
    double2 acc = make_double2(0.0, 0.0);
    if (s < S) {
      for (int t = s; t < T; t += S) {
        const C xi = Xb[(size_t)t * M + i], xk = Xb[(size_t)t * M + k];
        const double xr = xi.x, xim = xi.y, kr = xk.x, ki = xk.y;
        acc.x += xr * kr + xim * ki;   // Re(x_i conj(x_k))
        acc.y += xim * kr - xr * ki;   // Im(x_i conj(x_k))
      }
      red[s * P + p] = acc;
    }
    __syncthreads();
    if (tid < P) {
      double2 g = make_double2(0.0, 0.0);
      for (int q = 0; q < S; ++q) {
        g.x += red[q * P + tid].x;
        g.y += red[q * P + tid].y;
      }
      g.x /= (double)T;
      g.y /= (double)T;
      int ii = 0, rr = tid;
      while (rr >= M - ii) {
        rr -= M - ii;
        ++ii;
      }
      const int kk = ii + rr;
      if (ii == kk) g.y = 0.0;  // symmetrised (linalg.py:91)
      G[ii * M + kk] = g;
      G[kk * M + ii] = make_double2(g.x, -g.y);
    }
    __syncthreads();
  }
  if (tid >= 32) return;
  // ---- cyclic complex Jacobi (warp 0)
  warp_jacobi_eigh<M>(G, V, lane);
  // ---- clamp (linalg.py:92: w >= 1e-12 * max(max w, 0)), descending order
  double wmax = -INFINITY;
  for (int m = 0; m < M; ++m) wmax = fmax(wmax, G[m * M + m].x);
  const double fl = 1e-12 * fmax(wmax, 0.0);
  if (lane < M) {  // rank = number of eigenvalues before this one in descending order
    const double wl = G[lane * M + lane].x;
    int rank = 0;
    for (int m = 0; m < M; ++m) {
      const double wm = G[m * M + m].x;
      rank += (wm > wl) || (wm == wl && m < lane);
    }
    perm[rank] = lane;
  }
  __syncwarp();
  for (int e = lane; e < M * M; e += 32) {
    const int m = e / M, j = e % M, col = perm[m];
    const double2 v = V[j * M + col];  // Q row m = conj(eigenvector of the m-th largest)
    a.Q[((size_t)b * a.F + f) * M * M + e] = cmake<C>(v.x, -v.y);
  }
  if (a.w && lane < M) a.w[((size_t)b * a.F + f) * M + lane] = fmax(G[perm[lane] * M + perm[lane]].x, fl);
}

}  // namespace fm
