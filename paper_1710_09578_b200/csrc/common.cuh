// common.cuh — shared types and helpers of the sm_100a structured-transform engine.
//
// Complex arithmetic on float2 / double2, the dtype enum mirrored from smat.h,
// strided block views, error plumbing.  Everything in the engine computes on
// (rows, ncols) C-contiguous column blocks (the layout of the reference's
// LinearOperator.forward, pkg/src/linopkit/core.py:128-149).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

#include "../../include/smat.h"

namespace smat {

// ---------------------------------------------------------------- errors ---
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define SMAT_CUDA(call)                                                              \
  do {                                                                               \
    cudaError_t e__ = (call);                                                        \
    if (e__ != cudaSuccess)                                                          \
      throw ::smat::Error(SMAT_CUDA_ERROR, std::string(#call " failed: ") +          \
                                               cudaGetErrorString(e__));             \
  } while (0)

#define SMAT_CHECK(cond, code, msg)                                                  \
  do {                                                                               \
    if (!(cond)) throw ::smat::Error((code), (msg));                                 \
  } while (0)

// ---------------------------------------------------------------- dtypes ---
inline size_t dt_size(int dt) {
  switch (dt) {
    case SMAT_F32: return 4;
    case SMAT_F64: return 8;
    case SMAT_C64: return 8;
    case SMAT_C128: return 16;
    case SMAT_I32: return 4;
    case SMAT_I64: return 8;
  }
  return 0;
}
inline bool dt_complex(int dt) { return dt == SMAT_C64 || dt == SMAT_C128; }
inline bool dt_int(int dt) { return dt == SMAT_I32 || dt == SMAT_I64; }
inline bool dt_double(int dt) { return dt == SMAT_F64 || dt == SMAT_C128 || dt == SMAT_I64; }
inline int dt_real_of(int dt) {
  return dt == SMAT_C64 ? SMAT_F32 : dt == SMAT_C128 ? SMAT_F64 : dt;
}
inline int dt_complex_of(int dt) {
  return (dt == SMAT_F32 || dt == SMAT_C64) ? SMAT_C64 : SMAT_C128;
}

// ------------------------------------------------------------ complex ops ---
template <class R> struct Cx;
template <> struct Cx<float> { using T = float2; };
template <> struct Cx<double> { using T = double2; };
template <class C> struct RealOf;
template <> struct RealOf<float2> { using T = float; };
template <> struct RealOf<double2> { using T = double; };

__host__ __device__ __forceinline__ float2 mk(float a, float b) { return make_float2(a, b); }
__host__ __device__ __forceinline__ double2 mk(double a, double b) { return make_double2(a, b); }

// complex64 add/sub use the packed FP32x2 pipe of sm_100 (FADD2): one
// instruction per complex add instead of two.
__host__ __device__ __forceinline__ float2 operator+(float2 a, float2 b) {
#ifdef __CUDA_ARCH__
  return __fadd2_rn(a, b);
#else
  return mk(a.x + b.x, a.y + b.y);
#endif
}
__host__ __device__ __forceinline__ float2 operator-(float2 a, float2 b) {
#ifdef __CUDA_ARCH__
  return __fadd2_rn(a, make_float2(-b.x, -b.y));
#else
  return mk(a.x - b.x, a.y - b.y);
#endif
}
__host__ __device__ __forceinline__ float2 operator-(float2 a) { return mk(-a.x, -a.y); }
__host__ __device__ __forceinline__ float2& operator+=(float2& a, float2 b) { a = a + b; return a; }
__host__ __device__ __forceinline__ double2 operator+(double2 a, double2 b) { return mk(a.x + b.x, a.y + b.y); }
__host__ __device__ __forceinline__ double2 operator-(double2 a, double2 b) { return mk(a.x - b.x, a.y - b.y); }
__host__ __device__ __forceinline__ double2 operator-(double2 a) { return mk(-a.x, -a.y); }
__host__ __device__ __forceinline__ double2& operator+=(double2& a, double2 b) { a.x += b.x; a.y += b.y; return a; }

// d * (c - i s) for compile-time constants c, s
__device__ __forceinline__ float2 mul_cs(float2 d, float c, float s) {
  const float2 t = __fmul2_rn(d, make_float2(c, c));
  return __ffma2_rn(make_float2(d.y, d.x), make_float2(s, -s), t);
}
__device__ __forceinline__ double2 mul_cs(double2 d, double c, double s) {
  return make_double2(fma(d.x, c, d.y * s), fma(d.y, c, -d.x * s));
}
// a * w where q = (w.x, w.y, -w.y, w.x) (the "quad" twiddle layout of the
// single-precision tables): FMUL2 + FFMA2.
__device__ __forceinline__ float2 cmul_q(float2 a, float4 q) {
  const float2 t = __fmul2_rn(make_float2(a.x, a.x), make_float2(q.x, q.y));
  return __ffma2_rn(make_float2(a.y, a.y), make_float2(q.z, q.w), t);
}

__host__ __device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
__host__ __device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// a * conj(b)
__host__ __device__ __forceinline__ float2 cmulc(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, a.y * b.y), fmaf(a.y, b.x, -a.x * b.y));
}
__host__ __device__ __forceinline__ double2 cmulc(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -a.x * b.y));
}
template <class C> __host__ __device__ __forceinline__ C conj(C a) { return mk(a.x, -a.y); }
template <class C, class R> __host__ __device__ __forceinline__ C scl(C a, R s) {
  return mk(a.x * s, a.y * s);
}

// --------------------------------------------------------------- views -----
// A strided 4-D block: element (o1, o2, i, c) lives at p + o1*s1 + o2*s2 + i*si + c
// (strides in elements).  c runs over `inner` contiguous entries: the columns of
// the (rows, ncols) block, possibly times trailing Kronecker modes.
struct View {
  void* p = nullptr;
  int64_t s1 = 0, s2 = 0, si = 0;
};
struct BatchShape {
  int64_t n1 = 1, n2 = 1, inner = 1;  // counts of o1, o2, c
  int64_t count() const { return n1 * n2 * inner; }
};

__host__ __device__ __forceinline__ int64_t view_base(int64_t b, int64_t n2, int64_t inner,
                                                     int64_t s1, int64_t s2) {
  int64_t c = b % inner;
  int64_t t = b / inner;
  int64_t o2 = t % n2;
  int64_t o1 = t / n2;
  return o1 * s1 + o2 * s2 + c;
}

inline int num_sms(int device) {
  static int cached[64] = {0};
  if (device >= 0 && device < 64 && cached[device]) return cached[device];
  int v = 148;
  cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
  if (device >= 0 && device < 64) cached[device] = v;
  return v;
}

inline bool is_pow2(int64_t n) { return n >= 1 && (n & (n - 1)) == 0; }
inline int ilog2(int64_t n) {
  int l = 0;
  while ((int64_t(1) << l) < n) ++l;
  return l;
}
inline int64_t next_pow2(int64_t n) {
  int64_t m = 1;
  while (m < n) m <<= 1;
  return m;
}

}  // namespace smat
