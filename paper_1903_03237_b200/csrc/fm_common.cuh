// fm_common.cuh -- shared device helpers for the FastMNMF sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <float.h>
#include <stdint.h>

#include <type_traits>

namespace fm {

constexpr int NMAX = 8;  // sources per mixture supported by the fused kernels

// Real type traits: storage/arithmetic type R, its complex pair C, TINY
// (np.finfo(float).tiny in the reference, sources.py:24; FLT_MIN in the
// complex64 mode, SURVEY §8(a) exact-numerics checklist).
template <typename R> struct RT;
template <> struct RT<float> {
  using C = float2;
  static __host__ __device__ constexpr float tiny() { return FLT_MIN; }
};
template <> struct RT<double> {
  using C = double2;
  static __host__ __device__ constexpr double tiny() { return DBL_MIN; }
};

template <typename R> using cplx = typename RT<R>::C;

template <typename C> __host__ __device__ __forceinline__ C cmake(double x, double y) {
  C r;
  r.x = x;
  r.y = y;
  return r;
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {  // a * conj(b)
  return make_double2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) {
  return make_double2(a.x + b.x, a.y + b.y);
}
__device__ __forceinline__ double2 csub(double2 a, double2 b) {
  return make_double2(a.x - b.x, a.y - b.y);
}
__device__ __forceinline__ double2 cdiv(double2 a, double2 b) {
  // Smith's algorithm (what numpy / LAPACK's zladiv family use for robustness)
  if (fabs(b.y) <= fabs(b.x)) {
    double r = b.y / b.x, den = b.x + b.y * r;
    return make_double2((a.x + a.y * r) / den, (a.y - a.x * r) / den);
  } else {
    double r = b.x / b.y, den = b.x * r + b.y;
    return make_double2((a.x * r + a.y) / den, (a.y * r - a.x) / den);
  }
}
__device__ __forceinline__ double cabs1(double2 a) { return fabs(a.x) + fabs(a.y); }
// fp64 1/x and 1/sqrt(x) from the fp32 MUFU estimate + two Newton steps
// (error 1e-7 -> 1e-14 -> ~1 ulp); x must be a normal fp32-range value,
// which holds for the pivots and norms they are used on.
__device__ __forceinline__ double drcp(double x) {
  double r = (double)__frcp_rn((float)x);
  r = r * fma(-x, r, 2.0);
  r = r * fma(-x, r, 2.0);
  return r;
}
__device__ __forceinline__ double drsqrt(double x) {
  double r = (double)rsqrtf((float)x);
  r = r * fma(-0.5 * x * r, r, 1.5);
  r = r * fma(-0.5 * x * r, r, 1.5);
  return r;
}
// 1/p as conj(p)/|p|^2
__device__ __forceinline__ double2 crcp(double2 p) {
  const double inv = drcp(p.x * p.x + p.y * p.y);
  return make_double2(p.x * inv, -p.y * inv);
}
// fp32 complex arithmetic (the complex64 IP path at M <= 8, fm_spatial.cuh)
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float cabs1(float2 a) { return fabsf(a.x) + fabsf(a.y); }
// 1/x for a normal positive fp32 x: MUFU.RCP plus one Newton step (<= 1 ulp)
// -- the IEEE division expands to ~10 instructions with a slow-path call and
// sat on every Gauss-Jordan step of the fp32 inverses
__device__ __forceinline__ float frcp_nr(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return fmaf(r, fmaf(-x, r, 1.0f), r);
}
__device__ __forceinline__ float2 crcp(float2 p) {
  const float inv = frcp_nr(p.x * p.x + p.y * p.y);
  return make_float2(p.x * inv, -p.y * inv);
}
__device__ __forceinline__ float drsqrt(float x) { return rsqrtf(x); }
__device__ __forceinline__ float2 to_c2(double2 a, float2) { return make_float2((float)a.x, (float)a.y); }
__device__ __forceinline__ double2 to_c2(double2 a, double2) { return a; }
__device__ __forceinline__ float2 to_c2(float2 a, float2) { return a; }
__device__ __forceinline__ double2 to_c2(float2 a, double2) { return make_double2(a.x, a.y); }
__device__ __forceinline__ double2 to_d2(float2 a) { return make_double2(a.x, a.y); }
__device__ __forceinline__ double2 to_d2(double2 a) { return a; }

template <typename R> __device__ __forceinline__ R rsqrt_r(R x);
template <> __device__ __forceinline__ float rsqrt_r<float>(float x) { return 1.0f / sqrtf(x); }
template <> __device__ __forceinline__ double rsqrt_r<double>(double x) { return 1.0 / sqrt(x); }

__device__ __forceinline__ float log_r(float x) { return logf(x); }
__device__ __forceinline__ double log_r(double x) { return log(x); }
__device__ __forceinline__ float sqrt_r(float x) { return sqrtf(x); }
// log for the likelihood data term only (reported, never fed back): MUFU-based in fp32
__device__ __forceinline__ float log_fast(float x) { return __logf(x); }
__device__ __forceinline__ double log_fast(double x) { return log(x); }
__device__ __forceinline__ double sqrt_r(double x) { return sqrt(x); }

// Multiplicative-update factor sqrt(num / max(den, TINY))  (sources.py:194, :198;
// separate.py:218-220).
template <typename R> __device__ __forceinline__ R mu_factor(R num, R den) {
  R d = den > RT<R>::tiny() ? den : RT<R>::tiny();
  return sqrt_r(num / d);
}

// Floored model power: numba form `acc if acc > floor else floor` (_kernels.py:232).
template <typename R> __device__ __forceinline__ R floor_max(R acc, R fl) {
  return acc > fl ? acc : fl;
}

// Programmatic dependent launch (sm_90+): let the next kernel in the stream
// start its launch now, then wait until every prerequisite grid has completed
// and its memory is visible. A no-op for kernels launched without the PDL
// attribute. Used at the top of every kernel of the fused iteration so launch
// latency and CTA rasterisation overlap the previous kernel's tail.
__device__ __forceinline__ void pdl_entry() {
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
}

template <typename T> __device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Status key (fastmnmf.h): iteration<<44 | m<<24 | f<<2 | code.
__device__ __forceinline__ void report_status(unsigned long long* status, unsigned it, int m,
                                              long long f, int code) {
  if (!status) return;
  unsigned long long key = ((unsigned long long)it << 44) | ((unsigned long long)m << 24) |
                           ((unsigned long long)f << 2) | (unsigned long long)code;
  atomicMin(status, key);
}

// Vectorised loads/stores of a small contiguous row of R values.
template <typename R, int M> struct RowIO {
  __device__ static __forceinline__ void load(const R* __restrict__ p, R (&v)[M]) {
#pragma unroll
    for (int m = 0; m < M; ++m) v[m] = p[m];
  }
  __device__ static __forceinline__ void store(R* __restrict__ p, const R (&v)[M]) {
#pragma unroll
    for (int m = 0; m < M; ++m) p[m] = v[m];
  }
};
// float rows whose length is a multiple of 4 and whose base is 16-B aligned
// (row length M*4 bytes with M % 4 == 0 keeps every row aligned).
#define FM_ROWIO_F4(MM)                                                              \
  template <> struct RowIO<float, MM> {                                              \
    __device__ static __forceinline__ void load(const float* __restrict__ p,          \
                                                float (&v)[MM]) {                    \
      _Pragma("unroll") for (int m = 0; m < MM; m += 4) {                             \
        float4 q = *reinterpret_cast<const float4*>(p + m);                          \
        v[m] = q.x; v[m + 1] = q.y; v[m + 2] = q.z; v[m + 3] = q.w;                   \
      }                                                                               \
    }                                                                                 \
    __device__ static __forceinline__ void store(float* __restrict__ p,               \
                                                 const float (&v)[MM]) {              \
      _Pragma("unroll") for (int m = 0; m < MM; m += 4) {                             \
        *reinterpret_cast<float4*>(p + m) = make_float4(v[m], v[m + 1], v[m + 2], v[m + 3]); \
      }                                                                               \
    }                                                                                 \
  };
FM_ROWIO_F4(4)
FM_ROWIO_F4(8)
FM_ROWIO_F4(12)
FM_ROWIO_F4(16)
#undef FM_ROWIO_F4

// Complex rows: M complex values, vectorised as 16-B words where possible.
template <typename R, int M> struct CRowIO {
  using C = cplx<R>;
  __device__ static __forceinline__ void load(const C* __restrict__ p, C (&v)[M]) {
    if constexpr (sizeof(R) == 4 && (M % 2) == 0) {
      const float4* q = reinterpret_cast<const float4*>(p);
#pragma unroll
      for (int m = 0; m < M; m += 2) {
        float4 w = q[m / 2];
        v[m].x = w.x; v[m].y = w.y; v[m + 1].x = w.z; v[m + 1].y = w.w;
      }
    } else {
#pragma unroll
      for (int m = 0; m < M; ++m) v[m] = p[m];
    }
  }
  __device__ static __forceinline__ void store(C* __restrict__ p, const C (&v)[M]) {
    if constexpr (sizeof(R) == 4 && (M % 2) == 0) {
      float4* q = reinterpret_cast<float4*>(p);
#pragma unroll
      for (int m = 0; m < M; m += 2) q[m / 2] = make_float4(v[m].x, v[m].y, v[m + 1].x, v[m + 1].y);
    } else {
#pragma unroll
      for (int m = 0; m < M; ++m) p[m] = v[m];
    }
  }
};

}  // namespace fm
