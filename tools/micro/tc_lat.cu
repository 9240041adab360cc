// tcgen05 latency probe: cycles for [k x tcgen05.mma kind::tf32 (M=128, N=NB, K=8, SS)] +
// commit + mbarrier wait, from one thread of one CTA. Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_1903_03237_b200/csrc tc_lat.cu -o tc_lat
#include <cstdio>
#include <cstdint>
#include "fm_vacc_tc.cuh"
using namespace fm;

template <int NB>
__global__ void probe(long long* out, int reps) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x;
  for (int i = tid; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.f;
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (unsigned)__cvta_generic_to_shared(&tbase)), "r"(32));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  asm volatile("fence.proxy.async.shared::cta;");
  __syncthreads();
  const uint32_t sb = (unsigned)__cvta_generic_to_shared(sm);
  const uint64_t dA = umma_desc(sb, 128, 1024), dB = umma_desc(sb + 32768, 128, 1024);
  constexpr uint32_t ID = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(NB >> 3) << 17) | (8u << 24);
  const int ks[6] = {0, 1, 3, 12, 24, 48};
  unsigned phase = 0;
  if (tid == 0) {
    for (int q = 0; q < 6; ++q) {
      long long best = 1LL << 60, tot = 0;
      for (int r = 0; r < reps; ++r) {
        const long long t0 = clock64();
        for (int k = 0; k < ks[q]; ++k) umma_tf32(tbase, dA + (k & 3) * 16, dB + (k & 3) * 16, ID, k > 0);
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         (unsigned)__cvta_generic_to_shared(&bar)) : "memory");
        mbar_wait(&bar, phase);
        phase ^= 1;
        const long long dt = clock64() - t0;
        best = dt < best ? dt : best;
        tot += dt;
      }
      out[q * 2] = best;
      out[q * 2 + 1] = tot / reps;
    }
    // fence.proxy.async cost
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    out[12] = (clock64() - t0) / reps;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(32));
}

int main() {
  long long* d; cudaMalloc(&d, 64 * sizeof(long long));
  long long h[16];
  for (int nb : {8, 16}) {
    if (nb == 8) { cudaFuncSetAttribute(probe<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536); probe<8><<<1, 128, 65536>>>(d, 50); }
    else { cudaFuncSetAttribute(probe<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536); probe<16><<<1, 128, 65536>>>(d, 50); }
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(h, d, 13 * sizeof(long long), cudaMemcpyDeviceToHost);
    const int ks[6] = {0, 1, 3, 12, 24, 48};
    for (int q = 0; q < 6; ++q) printf("N=%d mmas=%2d: best %lld cyc, mean %lld cyc\n", nb, ks[q], h[q * 2], h[q * 2 + 1]);
    printf("N=%d fence.proxy.async: %lld cyc\n", nb, h[12]);
  }
  return 0;
}
