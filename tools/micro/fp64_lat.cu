// Microbenchmark: latency of the warp-level fp64 GJ inverse (M=8) and raw
// DFMA / FFMA dependent chains on B200. nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include "../../paper_1903_03237_b200/csrc/fm_linalg.cuh"
using namespace fm;

__global__ void k_chain(double* out, float* outf, long long* cyc, int n) {
  double a = threadIdx.x * 1e-3, b = 1.0000001, c = 1e-7;
  float af = threadIdx.x * 1e-3f, bf = 1.0000001f, cf = 1e-7f;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = fma(a, b, c);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) af = fmaf(af, bf, cf);
  long long t2 = clock64();
  double s = a;
  for (int i = 0; i < n; ++i) s = 1.0 / (s + 1.0);
  long long t3 = clock64();
  out[threadIdx.x] = a + s;
  outf[threadIdx.x] = af;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; }
}

__global__ void k_gj(double2* A, long long* cyc, int reps) {
  __shared__ double2 S[64];
  const int lane = threadIdx.x;
  for (int e = lane; e < 64; e += 32) S[e] = A[e];
  __syncwarp();
  long long t0 = clock64();
  bool ok = true;
  for (int r = 0; r < reps; ++r) ok &= warp_inv_hpd<8>(S, lane);
  long long t1 = clock64();
  if (lane == 0) { cyc[3] = (t1 - t0) / reps; cyc[4] = ok; }
  for (int e = lane; e < 64; e += 32) A[e] = S[e];
}

int main() {
  double* d; float* f; long long* c; double2* A;
  cudaMalloc(&d, 32 * 8); cudaMalloc(&f, 32 * 4); cudaMalloc(&c, 8 * 8); cudaMalloc(&A, 64 * 16);
  double2 h[64];
  for (int i = 0; i < 8; ++i) for (int j = 0; j < 8; ++j) h[i * 8 + j] = make_double2(i == j ? 8.0 : 0.1 / (1 + i + j), 0.0);
  cudaMemcpy(A, h, sizeof(h), cudaMemcpyHostToDevice);
  const int n = 4096;
  k_chain<<<1, 32>>>(d, f, c, n);
  k_gj<<<1, 32>>>(A, c, 8);
  long long hc[8];
  cudaDeviceSynchronize();
  cudaMemcpy(hc, c, sizeof(hc), cudaMemcpyDeviceToHost);
  printf("dependent DFMA: %.2f cyc, FFMA: %.2f cyc, DDIV+DADD: %.2f cyc\n", (double)hc[0] / n,
         (double)hc[1] / n, (double)hc[2] / n);
  printf("warp_inv_hpd<8>: %lld cyc per inverse (ok=%lld)\n", hc[3], hc[4]);
  return 0;
}
