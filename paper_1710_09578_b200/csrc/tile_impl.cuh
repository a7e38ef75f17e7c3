// tile_impl.cuh — templates of the tiled FFT / FWHT passes (instantiated per
// precision in tile_fft_c64.cu, tile_fft_c128.cu and tile_wht.cu).
//
// One CTA owns CT adjacent batches (columns of the (rows, ncols) block, so one
// row of the tile is a contiguous CT*sizeof(elt)-byte run in HBM) and the full
// length-N transform of each.  Each column is handled by TPC = N/E threads
// holding E = 16 elements in registers; stages exchange through shared memory.
// The reference equivalents are DftPlan._pow2 (kernels.py:95-109), fwht
// (kernels.py:164-190) and the spectrum multiply of Circulant._forward
// (leaves.py:219-224), which here is fused between the forward and inverse
// transforms without leaving registers.
//
// All per-thread index arithmetic is 32-bit: the batch decode uses host-
// computed magic-number division (FastDiv) and per-element offsets are 32-bit
// products widened once (IMAD.WIDE); the launcher checks the ranges.
#pragma once

#include <mutex>
#include <string>
#include <type_traits>
#include <unordered_map>

#include "fft_core.cuh"
#include "tile_kernels.cuh"

namespace smat {

// ------------------------------------------------------------ geometry -----
__host__ __device__ constexpr int tile_E(int N) { return N < 16 ? N : 16; }
__host__ __device__ constexpr int tile_CT_raw(int N, int bytes) {
  return bytes <= 4 ? (N <= 16 ? 128 : N <= 64 ? 64 : N <= 256 ? 32 : N <= 1024 ? 16 : 8)
       : bytes == 8 ? (N <= 16 ? 128 : N <= 32 ? 64 : N <= 128 ? 32 : N <= 512 ? 16 : N <= 1024 ? 8 : 4)
                    : (N <= 8 ? 128 : N <= 16 ? 64 : N <= 32 ? 64 : N <= 64 ? 32 : N <= 256 ? 16 : N <= 512 ? 8 : N <= 2048 ? 4 : 2);
}
// ... clamped so that a CTA never exceeds 1024 threads.
__host__ __device__ constexpr int tile_CT(int N, int bytes) {
  return tile_CT_raw(N, bytes) * (N / tile_E(N)) <= 1024 ? tile_CT_raw(N, bytes) : 1024 / (N / tile_E(N));
}
__host__ __device__ constexpr int tile_threads(int N, int bytes) { return (N / tile_E(N)) * tile_CT(N, bytes); }

// ------------------------------------------------------------- FastDiv -----
// q = n / d for 0 <= n < 2^31, 1 <= d < 2^31:  q = (umulhi(n, m) + n) >> s.
struct FastDiv {
  uint32_t d = 1, m = 1;
  int s = 0;
  FastDiv() = default;
  explicit FastDiv(int64_t dd) {
    SMAT_CHECK(dd >= 1 && dd < (int64_t(1) << 31), SMAT_UNSUPPORTED, "divisor out of 31-bit range");
    d = uint32_t(dd);
    s = 0;
    while ((uint64_t(1) << s) < d) ++s;
    m = uint32_t(((uint64_t(1) << (32 + s)) + d - 1) / d - (uint64_t(1) << 32) + (d == 1 ? 1 : 0));
    if (d == 1) m = 0;
  }
};
// (free function on register copies: member calls on kernel-parameter structs
// would force a local-memory copy of the parameter block)
__device__ __forceinline__ uint32_t fdiv(uint32_t n, uint32_t m, int s) { return (__umulhi(n, m) + n) >> s; }

// Device-side arguments of one FFT tile pass (built from FftArgs).
struct FftDev {
  const void* x;
  void* y;
  int64_t xs1, xs2, ys1, ys2;
  int32_t xsi, ysi;
  FastDiv inner, n2, gdiv, gmod;
  int32_t nb;
  int32_t gin_stride, gout_stride, n_valid_in, n_valid_out;
  const void* pre;
  const void* post;
  const void* mid;
  int32_t mid_stride;
  int32_t mid_gmul;
  int32_t pre_gmul, post_gmul;
  const void* tw;
  const void* tw_lo;
  const void* tw_hi;
  uint32_t tw_mask;
  int32_t tw_lo_bits;
  const void* tw_slices;
  int64_t xsi_hi, ysi_hi;  // two-level row strides (i_lo_bits > 0)
  int32_t i_lo_bits;
  double scale;
  uint32_t flags;
  const int32_t* in_map;  // fused row selection (GEN variant)
  const int32_t* out_map;
  int64_t in_rs, out_rs;
};
// Element offset of row i (two-level when lo_bits > 0).
__device__ __forceinline__ int64_t row_off(int i, int32_t si, int64_t si_hi, int lo_bits) {
  return lo_bits ? int64_t(i & ((1 << lo_bits) - 1)) * si + int64_t(i >> lo_bits) * si_hi : int64_t(i) * si;
}
enum : uint32_t {
  F_XREAL = 1, F_YREAL = 2, F_CONJX = 4, F_CONJY = 8, F_INV = 16, F_MIDCONJ = 32, F_TWINV = 64,
  F_ACC = 128, F_PRECONJ = 256, F_POSTCONJ = 512, F_PAD = 1024, F_TRUNC = 2048, F_SCALE = 4096,
  F_GOFF = 8192, F_TWPRE = 16384
};

struct WhtDev {
  const void* x;
  void* y;
  int64_t xs1, xs2, ys1, ys2;
  int32_t xsi, ysi;
  FastDiv inner, n2;
  int32_t nb;
  int32_t acc;
  // masks (MASK instantiation only)
  FastDiv gdiv, gmod;
  int32_t g_mul, gin_stride, gout_stride, n_valid_in, n_valid_out;
  // two-level rows: (i & i_lo_mask) * si + (i >> i_lo_bits) * si_hi
  int32_t i_lo_bits, i_lo_mask;
  int64_t xsi_hi, ysi_hi;
  // fused row selection (MASK instantiation only)
  const int32_t* in_map;
  const int32_t* out_map;
  int64_t in_rs, out_rs;
  int32_t map_k;
};

// b -> (o1, o2, c) with b = (o1*n2 + o2)*inner + c; returns the offset of the
// batch's first element for strides (s1, s2, 1).
__device__ __forceinline__ void decode_batch(uint32_t b, uint32_t in_d, uint32_t in_m, int in_s, uint32_t n2_d,
                                             uint32_t n2_m, int n2_s, uint32_t& o1, uint32_t& o2, uint32_t& c) {
  const uint32_t t = fdiv(b, in_m, in_s);
  c = b - t * in_d;
  o1 = fdiv(t, n2_m, n2_s);
  o2 = t - o1 * n2_d;
}

// W_Nt^m from the two-level four-step table.
template <class C>
__device__ __forceinline__ C tw2(const C* __restrict__ hi, const C* __restrict__ lo, uint32_t mask, int lo_bits,
                                 uint32_t m) {
  m &= mask;
  return cmul(__ldg(&hi[m >> lo_bits]), __ldg(&lo[m & ((1u << lo_bits) - 1u)]));
}

// -------------------------------------------------------- fft tile pass ----
// >= 1024 resident threads per SM for single precision (64 registers), >= 512
// for double precision (128 registers): two CTAs per SM overlap one CTA's
// HBM phase with the other's shuffle phase.
__host__ __device__ constexpr int tile_resident(int N, int bytes) {
  return bytes <= 8 ? (tile_threads(N, bytes) == 256 ? 768 : 1024) : 512;
}
__host__ __device__ constexpr int tile_min_blocks(int N, int bytes) {
  return tile_resident(N, bytes) / tile_threads(N, bytes) > 0 ? tile_resident(N, bytes) / tile_threads(N, bytes) : 1;
}
// GEN = false is the fast variant the launcher picks when the pass has complex
// input and output, no padding / truncation / pre / post / accumulation and
// a whole number of CTAs: conjugations and the scale fold into sign/scale
// multiplies, so no per-element branch remains.
template <class C, int N, bool MID, bool TW, bool GEN>
__global__ void __launch_bounds__(tile_threads(N, sizeof(C)), tile_min_blocks(N, sizeof(C)))
    fft_tile_kernel(const FftDev p) {
  using R = typename RealOf<C>::T;
  constexpr int E = tile_E(N);
  constexpr int CT = tile_CT(N, sizeof(C));
  constexpr int TPC = N / E;
  constexpr int NST = st_count(N, E);
  constexpr int R0 = st_radix(N, E, 0, false);
  constexpr int RL = MID ? st_radix(N, E, NST - 1, true) : st_radix(N, E, NST - 1, false);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* sm = reinterpret_cast<C*>(smem_raw);
  const int tid = threadIdx.x, cs = tid % CT, j = tid / CT;
  const uint32_t b = blockIdx.x * uint32_t(CT) + uint32_t(cs);
  const bool act = !GEN || int32_t(b) < p.nb;
  const uint32_t f = p.flags;
  int64_t xb = 0, yb = 0;
  int32_t goff = 0;
  if (act) {
    uint32_t o1, o2, c;
    decode_batch(b, p.inner.d, p.inner.m, p.inner.s, p.n2.d, p.n2.m, p.n2.s, o1, o2, c);
    xb = int64_t(o1) * p.xs1 + int64_t(o2) * p.xs2 + c;
    yb = int64_t(o1) * p.ys1 + int64_t(o2) * p.ys2 + c;
    if (f & F_GOFF) {
      const uint32_t q = fdiv(b, p.gdiv.m, p.gdiv.s);
      goff = int32_t(q - fdiv(q, p.gmod.m, p.gmod.s) * p.gmod.d);
    }
  }
  const C* tw = (const C*)p.tw;
  C a[E];
  // ---- load (stage-0 input order: element j + u*TPC + r*N/R0)
  if constexpr (!GEN) {
    const C* xc = (const C*)p.x + xb + int64_t(j) * p.xsi;
    const R sx = ((f & F_CONJX) != 0) != (!MID && (f & F_INV)) ? R(-1) : R(1);
#pragma unroll
    for (int u = 0; u < E / R0; ++u)
#pragma unroll
      for (int r = 0; r < R0; ++r) {
        const int i = u * TPC + r * (N / R0);
        C v = __ldg(&xc[int64_t(i) * p.xsi]);
        v.y *= sx;
        a[u * R0 + r] = v;
      }
  } else {
    const R* xr = (const R*)p.x + xb;
    const C* xc = (const C*)p.x + xb;
#pragma unroll
    for (int u = 0; u < E / R0; ++u)
#pragma unroll
      for (int r = 0; r < R0; ++r) {
        const int i = j + u * TPC + r * (N / R0);
        C v = mk(R(0), R(0));
        const int g = goff + i * p.gin_stride;
        int src = 0;
        if (p.in_map && act) src = __ldg(&p.in_map[g]);
        if (act && (!(f & F_PAD) || g < p.n_valid_in) && src >= 0) {
          const int64_t off = p.in_map ? int64_t(src) * p.in_rs : row_off(i, p.xsi, p.xsi_hi, p.i_lo_bits);
          v = (f & F_XREAL) ? mk(__ldg(&xr[off]), R(0)) : __ldg(&xc[off]);
          if (f & F_CONJX) v = conj(v);
          if (p.pre) {
            const C w = __ldg(&((const C*)p.pre)[p.pre_gmul ? goff * p.pre_gmul + i : g]);
            v = (f & F_PRECONJ) ? cmulc(v, w) : cmul(v, w);
          }
          if (f & F_TWPRE) {
            const C w = tw2<C>((const C*)p.tw_hi, (const C*)p.tw_lo, p.tw_mask, p.tw_lo_bits,
                               uint32_t(goff) * uint32_t(i));
            v = (f & F_TWINV) ? cmulc(v, w) : cmul(v, w);
          }
          if (!MID && (f & F_INV)) v = conj(v);
        }
        a[u * R0 + r] = v;
      }
  }
  fft_stages<C, N, E, CT, false, 0>(a, sm, j, cs, tw);
  if constexpr (MID) {
    constexpr int RF = st_radix(N, E, NST - 1, false);
    const C* mid = (const C*)p.mid;
    const int64_t mbase = int64_t(goff) * p.mid_gmul;
    const R sm_im = (f & F_MIDCONJ) ? R(-1) : R(1);
#pragma unroll
    for (int u = 0; u < E / RF; ++u)
#pragma unroll
      for (int r = 0; r < RF; ++r) {
        const int k = j + u * TPC + r * (N / RF);
        C s = act ? ld_spec(mid, mbase + k * p.mid_stride) : mk(R(0), R(0));
        s.y *= sm_im;
        a[u * RF + r] = conj(cmul(a[u * RF + r], s));
      }
    fft_stages<C, N, E, CT, true, 0>(a, sm, j, cs, tw);
  }
  // ---- store (last-stage output order: element bb + r*N/RL, bb = j + u*TPC)
  R* yr = (R*)p.y + yb;
  C* yc = (C*)p.y + yb;
  const bool pre_conj = MID || (f & F_INV);  // the "inverse" conjugation before twiddle/post
  // fast path: v.x *= s_re, v.y *= s_im  (conj_y and scale folded; pre_conj too when !TW)
  const R sc = (f & F_SCALE) ? R(p.scale) : R(1);
  const R s_re = sc;
  const R s_im = ((f & F_CONJY) != 0) != (!TW && pre_conj) ? -sc : sc;
#pragma unroll
  for (int u = 0; u < E / RL; ++u) {
    const int bb = j + u * TPC;
    if constexpr (TW) {
      // four-step twiddle W^(goff*k), k = bb + r*N/RL: base * step^r
      C wp[4];
      const uint32_t g32 = uint32_t(goff);
      const C* thi = (const C*)p.tw_hi;
      const C* tlo = (const C*)p.tw_lo;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if ((1 << q) < RL) wp[q] = tw2<C>(thi, tlo, p.tw_mask, p.tw_lo_bits, g32 * uint32_t((N / RL) << q));
      C base = tw2<C>(thi, tlo, p.tw_mask, p.tw_lo_bits, g32 * uint32_t(bb));
      C* au = a + u * RL;
      // (conj v) * w  or  (conj v) * conj(w) = conj(v * w)
      const bool twinv = (f & F_TWINV) != 0;
      if (pre_conj != twinv) {
#pragma unroll
        for (int r = 0; r < RL; ++r) au[r] = conj(au[r]);
      }
      au[0] = cmul(au[0], base);
      apply_powers<RL>(au, wp);
#pragma unroll
      for (int r = 1; r < RL; ++r) au[r] = cmul(au[r], base);
      if (twinv) {
#pragma unroll
        for (int r = 0; r < RL; ++r) au[r] = conj(au[r]);
      }
    }
    if constexpr (!GEN) {
      C* yk = yc + int64_t(bb) * p.ysi;
#pragma unroll
      for (int r = 0; r < RL; ++r) {
        C v = a[u * RL + r];
        v.x *= s_re;
        v.y *= s_im;
        yk[int64_t(r * (N / RL)) * p.ysi] = v;
      }
    } else {
#pragma unroll
      for (int r = 0; r < RL; ++r) {
        const int k = bb + r * (N / RL);
        const int g = goff + k * p.gout_stride;
        C v = a[u * RL + r];
        if (!TW && pre_conj) v = conj(v);
        const int dst = (p.out_map && act) ? __ldg(&p.out_map[g]) : 0;
        if (act && (!(f & F_TRUNC) || g < p.n_valid_out) && dst >= 0) {
          if (p.post) {
            const C w = __ldg(&((const C*)p.post)[p.post_gmul ? goff * p.post_gmul + k : g]);
            v = (f & F_POSTCONJ) ? cmulc(v, w) : cmul(v, w);
          }
          if (f & F_CONJY) v = conj(v);
          if (f & F_SCALE) v = scl(v, sc);
          const int64_t off = p.out_map ? int64_t(dst) * p.out_rs : row_off(k, p.ysi, p.ysi_hi, p.i_lo_bits);
          if (f & F_YREAL) {
            yr[off] = (f & F_ACC) ? yr[off] + v.x : v.x;
          } else {
            yc[off] = (f & F_ACC) ? yc[off] + v : v;
          }
        }
      }
    }
  }
}

// -------------------------------------------------------- wht tile pass ----
template <class T>
__device__ __forceinline__ T zero_of() {
  if constexpr (std::is_same<T, float2>::value) return make_float2(0.f, 0.f);
  else if constexpr (std::is_same<T, double2>::value) return make_double2(0.0, 0.0);
  else return T(0);
}

template <class T, int N, bool MASK>
__global__ void __launch_bounds__(tile_threads(N, sizeof(T))) wht_tile_kernel(const WhtDev p) {
  constexpr int E = tile_E(N);
  constexpr int CT = tile_CT(N, sizeof(T));
  constexpr int TPC = N / E;
  constexpr int NST = st_count(N, E);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);
  const int tid = threadIdx.x, cs = tid % CT, j = tid / CT;
  const uint32_t b = blockIdx.x * uint32_t(CT) + uint32_t(cs);
  const bool act = int32_t(b) < p.nb;
  int64_t xb = 0, yb = 0;
  int32_t goff = 0, mcol = 0;
  if (act) {
    uint32_t o1, o2, c;
    decode_batch(b, p.inner.d, p.inner.m, p.inner.s, p.n2.d, p.n2.m, p.n2.s, o1, o2, c);
    xb = int64_t(o1) * p.xs1 + int64_t(o2) * p.xs2 + c;
    yb = int64_t(o1) * p.ys1 + int64_t(o2) * p.ys2 + c;
    if constexpr (MASK) {
      const uint32_t q = fdiv(b, p.gdiv.m, p.gdiv.s);
      goff = int32_t(q - fdiv(q, p.gmod.m, p.gmod.s) * p.gmod.d) * p.g_mul;
      mcol = int32_t(c % uint32_t(p.map_k));
    }
  }
  const T* x = (const T*)p.x + xb;
  T* y = (T*)p.y + yb;
  T a[E];
  constexpr int R0 = st_radix_lin(N, E, 0);
#pragma unroll
  for (int u = 0; u < E / R0; ++u) {
    const int bb = j + u * TPC;
#pragma unroll
    for (int r = 0; r < R0; ++r) {
      const int i = bb * R0 + r;
      bool ok = act;
      if constexpr (MASK) {
        const int g = goff + i * p.gin_stride;
        ok = ok && g < p.n_valid_in;
        if (p.in_map) {
          const int src = ok ? __ldg(&p.in_map[g]) : -1;
          a[u * R0 + r] = src >= 0 ? ((const T*)p.x)[int64_t(src) * p.in_rs + mcol] : zero_of<T>();
          continue;
        }
      }
      a[u * R0 + r] =
          ok ? x[int64_t(i & p.i_lo_mask) * p.xsi + int64_t(i >> p.i_lo_bits) * p.xsi_hi] : zero_of<T>();
    }
  }
  wht_stages<T, N, E, CT, 0>(a, sm, j, cs);
  constexpr int RL = st_radix_lin(N, E, NST - 1);
  constexpr int NSL = st_ns_lin(N, E, NST - 1);
  if (!act) return;
#pragma unroll
  for (int u = 0; u < E / RL; ++u) {
    const int bb = j + u * TPC;
    const int base = (bb / NSL) * (NSL * RL) + (bb % NSL);
#pragma unroll
    for (int r = 0; r < RL; ++r) {
      const int k = base + r * NSL;
      if constexpr (MASK) {
        const int g = goff + k * p.gout_stride;
        if (g >= p.n_valid_out) continue;
        if (p.out_map) {
          const int dst = __ldg(&p.out_map[g]);
          if (dst < 0) continue;
          T* yo = (T*)p.y + int64_t(dst) * p.out_rs + mcol;
          *yo = p.acc ? *yo + a[u * RL + r] : a[u * RL + r];
          continue;
        }
      }
      const int64_t off = int64_t(k & p.i_lo_mask) * p.ysi + int64_t(k >> p.i_lo_bits) * p.ysi_hi;
      y[off] = p.acc ? y[off] + a[u * RL + r] : a[u * RL + r];
    }
  }
}

// ------------------------------------------------------------ launchers ----
template <class K>
inline void set_smem(K kern, size_t bytes) {
  static std::mutex mu;
  static std::unordered_map<uint64_t, size_t> done;
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t key = uint64_t(uintptr_t((const void*)kern)) ^ (uint64_t(dev) << 56);
  std::lock_guard<std::mutex> g(mu);
  auto it = done.find(key);
  if (it != done.end() && it->second >= bytes) return;
  SMAT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
  done[key] = bytes;
}

inline bool fits31(int64_t v) { return v > -(int64_t(1) << 31) && v < (int64_t(1) << 31); }

// Build the device argument block of an FFT tile pass of length N.
inline FftDev make_fft_dev(const FftArgs& a, int N) {
  FftDev d{};
  SMAT_CHECK(a.nb < (int64_t(1) << 31) - 4096, SMAT_UNSUPPORTED, "fft tile: batch count exceeds 2^31");
  SMAT_CHECK(fits31(a.xsi * N) && fits31(a.ysi * N), SMAT_UNSUPPORTED, "fft tile: row stride too large");
  d.x = a.x;
  d.y = a.y;
  d.xs1 = a.xs1; d.xs2 = a.xs2; d.ys1 = a.ys1; d.ys2 = a.ys2;
  d.xsi = int32_t(a.xsi);
  d.ysi = int32_t(a.ysi);
  d.inner = FastDiv(a.inner);
  d.n2 = FastDiv(a.n2);
  d.nb = int32_t(a.nb);
  const bool goff = a.g_mod > 1;
  d.gdiv = FastDiv(a.g_div);
  d.gmod = FastDiv(a.g_mod);
  const int64_t gmax_in = (a.g_mod - 1) + (N - 1) * a.gin_stride;
  const int64_t gmax_out = (a.g_mod - 1) + (N - 1) * a.gout_stride;
  SMAT_CHECK(fits31(gmax_in) && fits31(gmax_out) && fits31((a.g_mod - 1) * a.mid_gmul + (N - 1) * a.mid_stride),
             SMAT_UNSUPPORTED, "fft tile: global row index exceeds 2^31");
  d.gin_stride = int32_t(a.gin_stride);
  d.gout_stride = int32_t(a.gout_stride);
  d.n_valid_in = int32_t(a.n_valid_in < INT32_MAX ? a.n_valid_in : INT32_MAX);
  d.n_valid_out = int32_t(a.n_valid_out < INT32_MAX ? a.n_valid_out : INT32_MAX);
  d.pre = a.pre;
  d.post = a.post;
  d.mid = a.mid;
  d.mid_stride = int32_t(a.mid_stride);
  d.mid_gmul = int32_t(a.mid_gmul);
  SMAT_CHECK(fits31((a.g_mod - 1) * a.pre_gmul + N) && fits31((a.g_mod - 1) * a.post_gmul + N), SMAT_UNSUPPORTED,
             "fft tile: pre/post slice index exceeds 2^31");
  d.pre_gmul = int32_t(a.pre_gmul);
  d.post_gmul = int32_t(a.post_gmul);
  d.tw = a.tw;
  d.tw_lo = a.tw_lo;
  d.tw_hi = a.tw_hi;
  d.tw_mask = uint32_t(a.tw_mask);
  d.tw_lo_bits = a.tw_lo_bits;
  d.tw_slices = a.tw_slices;
  d.i_lo_bits = a.i_lo_bits;
  d.xsi_hi = a.i_lo_bits ? a.xsi_hi : 0;
  d.ysi_hi = a.i_lo_bits ? a.ysi_hi : 0;
  d.scale = a.scale;
  uint32_t f = 0;
  if (a.x_real) f |= F_XREAL;
  if (a.y_real) f |= F_YREAL;
  if (a.conj_x) f |= F_CONJX;
  if (a.conj_y) f |= F_CONJY;
  if (a.inv) f |= F_INV;
  if (a.mid_conj) f |= F_MIDCONJ;
  if (a.tw_inv) f |= F_TWINV;
  if (a.accumulate) f |= F_ACC;
  if (a.pre_conj) f |= F_PRECONJ;
  if (a.post_conj) f |= F_POSTCONJ;
  if (gmax_in >= a.n_valid_in) f |= F_PAD;
  if (gmax_out >= a.n_valid_out) f |= F_TRUNC;
  if (a.scale != 1.0) f |= F_SCALE;
  if (goff) f |= F_GOFF;
  if (a.tw_on && a.tw_pre) f |= F_TWPRE;
  d.flags = f;
  d.in_map = a.in_map;
  d.out_map = a.out_map;
  d.in_rs = a.in_rs;
  d.out_rs = a.out_rs;
  return d;
}

template <class C, int N, bool MID, bool TW, bool GEN>
inline void fft_tile_go(const FftDev& d, int64_t nb, cudaStream_t s) {
  constexpr int CT = tile_CT(N, sizeof(C));
  const size_t smem = N > 1 ? size_t(sm_rows(N)) * CT * sizeof(C) : 0;
  const int64_t blocks = (nb + CT - 1) / CT;
  if (blocks == 0) return;
  set_smem(fft_tile_kernel<C, N, MID, TW, GEN>, smem);
  fft_tile_kernel<C, N, MID, TW, GEN><<<unsigned(blocks), tile_threads(N, sizeof(C)), smem, s>>>(d);
  SMAT_CUDA(cudaGetLastError());
}

template <class C, int N, bool MID, bool TW>
inline void fft_tile_go2(const FftDev& d, int64_t nb, bool fast, cudaStream_t s) {
  if constexpr (N >= 64) {
    if (fast) {
      fft_tile_go<C, N, MID, TW, false>(d, nb, s);
      return;
    }
  }
  fft_tile_go<C, N, MID, TW, true>(d, nb, s);
}

template <class C, int N>
inline void fft_tile_launch(const FftArgs& a, cudaStream_t s) {
  const FftDev d = make_fft_dev(a, N);
  constexpr int CT = tile_CT(N, sizeof(C));
  const bool fast = (a.nb % CT) == 0 && !a.x_real && !a.y_real && !a.pre && !a.post && !a.accumulate &&
                    !(d.flags & (F_PAD | F_TRUNC | F_TWPRE)) && a.i_lo_bits == 0 && !a.in_map && !a.out_map;
  // (an input-side twiddle runs in the generic variant's load loop)
  const bool mid = a.mid != nullptr, tw = a.tw_on != 0 && !a.tw_pre;
  if (mid && tw) fft_tile_go2<C, N, true, true>(d, a.nb, fast, s);
  else if (mid) fft_tile_go2<C, N, true, false>(d, a.nb, fast, s);
  else if (tw) fft_tile_go2<C, N, false, true>(d, a.nb, fast, s);
  else fft_tile_go2<C, N, false, false>(d, a.nb, fast, s);
}

template <class T, int N>
inline void wht_tile_launch(const WhtArgs& a, cudaStream_t s) {
  constexpr int CT = tile_CT(N, sizeof(T));
  SMAT_CHECK(a.nb < (int64_t(1) << 31) - 4096, SMAT_UNSUPPORTED, "fwht tile: batch count exceeds 2^31");
  SMAT_CHECK(fits31(a.xsi * N) && fits31(a.ysi * N), SMAT_UNSUPPORTED, "fwht tile: row stride too large");
  WhtDev d{};
  d.x = a.x; d.y = a.y;
  d.xs1 = a.xs1; d.xs2 = a.xs2; d.ys1 = a.ys1; d.ys2 = a.ys2;
  d.xsi = int32_t(a.xsi); d.ysi = int32_t(a.ysi);
  d.inner = FastDiv(a.inner);
  d.n2 = FastDiv(a.n2);
  d.nb = int32_t(a.nb);
  d.acc = a.accumulate;
  d.i_lo_bits = a.i_lo_bits;
  d.i_lo_mask = a.i_lo_bits ? (1 << a.i_lo_bits) - 1 : -1;
  d.xsi_hi = a.i_lo_bits ? a.xsi_hi : 0;
  d.ysi_hi = a.i_lo_bits ? a.ysi_hi : 0;
  const int64_t gmax_in = (a.g_mod - 1) * a.g_mul + (N - 1) * a.gin_stride;
  const int64_t gmax_out = (a.g_mod - 1) * a.g_mul + (N - 1) * a.gout_stride;
  const bool mask = gmax_in >= a.n_valid_in || gmax_out >= a.n_valid_out || a.in_map || a.out_map;
  d.in_map = a.in_map;
  d.out_map = a.out_map;
  d.in_rs = a.in_rs;
  d.out_rs = a.out_rs;
  d.map_k = int32_t(a.map_k);
  if (mask) {
    SMAT_CHECK(fits31(gmax_in) && fits31(gmax_out), SMAT_UNSUPPORTED, "fwht tile: row index exceeds 2^31");
    d.gdiv = FastDiv(a.g_div);
    d.gmod = FastDiv(a.g_mod);
    d.g_mul = int32_t(a.g_mul);
    d.gin_stride = int32_t(a.gin_stride);
    d.gout_stride = int32_t(a.gout_stride);
    d.n_valid_in = int32_t(a.n_valid_in < INT32_MAX ? a.n_valid_in : INT32_MAX);
    d.n_valid_out = int32_t(a.n_valid_out < INT32_MAX ? a.n_valid_out : INT32_MAX);
  }
  const size_t smem = N > 1 ? size_t(sm_rows(N)) * CT * sizeof(T) : 0;
  const int64_t blocks = (a.nb + CT - 1) / CT;
  if (blocks == 0) return;
  auto go = [&](auto kern) {
    set_smem(kern, smem);
    kern<<<unsigned(blocks), tile_threads(N, sizeof(T)), smem, s>>>(d);
  };
  if (mask) go(wht_tile_kernel<T, N, true>);
  else go(wht_tile_kernel<T, N, false>);
  SMAT_CUDA(cudaGetLastError());
}

#define SMAT_N_SWITCH(FN, T, N, ...)                    \
  switch (N) {                                          \
    case 1: FN<T, 1>(__VA_ARGS__); break;               \
    case 2: FN<T, 2>(__VA_ARGS__); break;               \
    case 4: FN<T, 4>(__VA_ARGS__); break;               \
    case 8: FN<T, 8>(__VA_ARGS__); break;               \
    case 16: FN<T, 16>(__VA_ARGS__); break;             \
    case 32: FN<T, 32>(__VA_ARGS__); break;             \
    case 64: FN<T, 64>(__VA_ARGS__); break;             \
    case 128: FN<T, 128>(__VA_ARGS__); break;           \
    case 256: FN<T, 256>(__VA_ARGS__); break;           \
    case 512: FN<T, 512>(__VA_ARGS__); break;           \
    case 1024: FN<T, 1024>(__VA_ARGS__); break;         \
    case 2048: FN<T, 2048>(__VA_ARGS__); break;         \
    case 4096: FN<T, 4096>(__VA_ARGS__); break;         \
    default: throw Error(SMAT_UNSUPPORTED, "tile length " + std::to_string(N)); \
  }

}  // namespace smat
