// tile_kernels.cu — tiled FFT / FWHT passes for sm_100a.
//
// One CTA owns CT adjacent batches (columns of the (rows, ncols) block, so one
// row of the tile is a contiguous CT*sizeof(elt)-byte run in HBM) and the full
// length-N transform of each.  Each column is handled by TPC = N/E threads
// holding E = 16 elements in registers; stages exchange through shared memory.
// The reference equivalents are DftPlan._pow2 (kernels.py:95-109), fwht
// (kernels.py:164-190) and the spectrum multiply of Circulant._forward
// (leaves.py:219-224), which here is fused between the forward and inverse
// transforms without leaving registers.
#include <mutex>
#include <unordered_map>
#include <vector>

#include "fft_core.cuh"
#include "tile_kernels.cuh"

namespace smat {

// ------------------------------------------------------------ geometry -----
__host__ __device__ constexpr int tile_E(int N) { return N < 16 ? N : 16; }
// Columns per CTA: aim for >= 128 threads and <= 64 KB of shared memory
// (128 KB for the largest tiles).
__host__ __device__ constexpr int tile_CT_raw(int N, int bytes) {
  return bytes <= 4 ? (N <= 16 ? 128 : N <= 64 ? 64 : N <= 256 ? 32 : N <= 1024 ? 16 : 8)
       : bytes == 8 ? (N <= 16 ? 128 : N <= 32 ? 64 : N <= 128 ? 32 : N <= 512 ? 16 : N <= 1024 ? 8 : 4)
                    : (N <= 8 ? 128 : N <= 16 ? 64 : N <= 32 ? 64 : N <= 64 ? 32 : N <= 256 ? 16 : N <= 512 ? 8 : N <= 2048 ? 4 : 2);
}
// ... clamped so that a CTA never exceeds 1024 threads.
__host__ __device__ constexpr int tile_CT(int N, int bytes) {
  return tile_CT_raw(N, bytes) * (N / tile_E(N)) <= 1024 ? tile_CT_raw(N, bytes) : 1024 / (N / tile_E(N));
}

// -------------------------------------------------------- fft tile pass ----
template <class C>
__device__ __forceinline__ C fft_load(const FftArgs& p, bool act, int64_t xb, int64_t goff, int i) {
  using R = typename RealOf<C>::T;
  C v = mk(R(0), R(0));
  const int64_t g = goff + int64_t(i) * p.gin_stride;
  if (act && g < p.n_valid_in) {
    if (p.x_real)
      v = mk(__ldg(&((const R*)p.x)[xb + int64_t(i) * p.xsi]), R(0));
    else
      v = __ldg(&((const C*)p.x)[xb + int64_t(i) * p.xsi]);
    if (p.conj_x) v = conj(v);
    if (p.pre) {
      const C w = __ldg(&((const C*)p.pre)[g]);
      v = p.pre_conj ? cmulc(v, w) : cmul(v, w);
    }
    if (p.inv && !p.mid) v = conj(v);
  }
  return v;
}

template <class C>
__device__ __forceinline__ void fft_store(const FftArgs& p, bool act, int64_t yb, int64_t goff, int k, C v) {
  using R = typename RealOf<C>::T;
  const int64_t g = goff + int64_t(k) * p.gout_stride;
  if (!act || g >= p.n_valid_out) return;
  if (p.inv || p.mid) v = conj(v);
  if (p.tw_on) {
    const uint64_t m = uint64_t(goff * int64_t(k)) & uint64_t(p.tw_mask);
    const C w = cmul(__ldg(&((const C*)p.tw_hi)[m >> p.tw_lo_bits]),
                     __ldg(&((const C*)p.tw_lo)[m & ((uint64_t(1) << p.tw_lo_bits) - 1)]));
    v = p.tw_inv ? cmulc(v, w) : cmul(v, w);
  }
  if (p.post) {
    const C w = __ldg(&((const C*)p.post)[g]);
    v = p.post_conj ? cmulc(v, w) : cmul(v, w);
  }
  if (p.conj_y) v = conj(v);
  if (p.scale != 1.0) v = scl(v, R(p.scale));
  const int64_t off = yb + int64_t(k) * p.ysi;
  if (p.y_real) {
    R* y = (R*)p.y;
    y[off] = p.accumulate ? y[off] + v.x : v.x;
  } else {
    C* y = (C*)p.y;
    y[off] = p.accumulate ? y[off] + v : v;
  }
}

template <class C, int N, int E, int CT, int RL>
__device__ __forceinline__ void fft_store_all(const FftArgs& p, bool act, int64_t yb, int64_t goff,
                                              int j, const C* a) {
  constexpr int TPC = N / E;
#pragma unroll
  for (int u = 0; u < E / RL; ++u)
#pragma unroll
    for (int r = 0; r < RL; ++r) fft_store(p, act, yb, goff, j + u * TPC + r * (N / RL), a[u * RL + r]);
}

template <class C, int N>
__global__ void __launch_bounds__((N / tile_E(N)) * tile_CT(N, sizeof(C)))
    fft_tile_kernel(const FftArgs p) {
  constexpr int E = tile_E(N);
  constexpr int CT = tile_CT(N, sizeof(C));
  constexpr int TPC = N / E;
  constexpr int NST = st_count(N, E);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* sm = reinterpret_cast<C*>(smem_raw);
  const int tid = threadIdx.x, cs = tid % CT, j = tid / CT;
  const int64_t b = int64_t(blockIdx.x) * CT + cs;
  const bool act = b < p.nb;
  int64_t xb = 0, yb = 0, goff = 0;
  if (act) {
    xb = view_base(b, p.n2, p.inner, p.xs1, p.xs2);
    yb = view_base(b, p.n2, p.inner, p.ys1, p.ys2);
    goff = (b / p.g_div) % p.g_mod;
  }
  const C* tw = (const C*)p.tw;
  C a[E];
  constexpr int R0 = st_radix(N, E, 0, false);
#pragma unroll
  for (int u = 0; u < E / R0; ++u)
#pragma unroll
    for (int r = 0; r < R0; ++r) a[u * R0 + r] = fft_load<C>(p, act, xb, goff, j + u * TPC + r * (N / R0));
  fft_stages<C, N, E, CT, false, 0>(a, sm, j, cs, tw);
  constexpr int RL = st_radix(N, E, NST - 1, false);
  if (p.mid) {
    using R = typename RealOf<C>::T;
    const C* mid = (const C*)p.mid;
#pragma unroll
    for (int u = 0; u < E / RL; ++u)
#pragma unroll
      for (int r = 0; r < RL; ++r) {
        const int k = j + u * TPC + r * (N / RL);
        C s = act ? __ldg(&mid[goff + int64_t(k) * p.mid_stride]) : mk(R(0), R(0));
        C v = p.mid_conj ? cmulc(a[u * RL + r], s) : cmul(a[u * RL + r], s);
        a[u * RL + r] = conj(v);
      }
    fft_stages<C, N, E, CT, true, 0>(a, sm, j, cs, tw);
    constexpr int RLM = st_radix(N, E, NST - 1, true);
    fft_store_all<C, N, E, CT, RLM>(p, act, yb, goff, j, a);
  } else {
    fft_store_all<C, N, E, CT, RL>(p, act, yb, goff, j, a);
  }
}

// -------------------------------------------------------- wht tile pass ----
template <class T>
__device__ __forceinline__ T zero_of() {
  if constexpr (std::is_same<T, float2>::value) return make_float2(0.f, 0.f);
  else if constexpr (std::is_same<T, double2>::value) return make_double2(0.0, 0.0);
  else return T(0);
}

template <class T, int N>
__global__ void __launch_bounds__((N / tile_E(N)) * tile_CT(N, sizeof(T)))
    wht_tile_kernel(const WhtArgs p) {
  constexpr int E = tile_E(N);
  constexpr int CT = tile_CT(N, sizeof(T));
  constexpr int TPC = N / E;
  constexpr int NST = st_count(N, E);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);
  const int tid = threadIdx.x, cs = tid % CT, j = tid / CT;
  const int64_t b = int64_t(blockIdx.x) * CT + cs;
  const bool act = b < p.nb;
  int64_t xb = 0, yb = 0, goff = 0;
  if (act) {
    xb = view_base(b, p.n2, p.inner, p.xs1, p.xs2);
    yb = view_base(b, p.n2, p.inner, p.ys1, p.ys2);
    goff = (b / p.g_div) % p.g_mod;
  }
  const T* x = (const T*)p.x;
  T* y = (T*)p.y;
  T a[E];
  constexpr int R0 = st_radix(N, E, 0, false);
#pragma unroll
  for (int u = 0; u < E / R0; ++u) {
    const int bb = j + u * TPC;
#pragma unroll
    for (int r = 0; r < R0; ++r) {
      const int i = bb * R0 + r;
      const int64_t g = goff + int64_t(i) * p.gin_stride;
      a[u * R0 + r] = (act && g < p.n_valid_in) ? x[xb + int64_t(i) * p.xsi] : zero_of<T>();
    }
  }
  wht_stages<T, N, E, CT, 0>(a, sm, j, cs);
  constexpr int RL = st_radix(N, E, NST - 1, false);
  constexpr int NSL = st_ns(N, E, NST - 1, false);
#pragma unroll
  for (int u = 0; u < E / RL; ++u) {
    const int bb = j + u * TPC;
    const int base = (bb / NSL) * (NSL * RL) + (bb % NSL);
#pragma unroll
    for (int r = 0; r < RL; ++r) {
      const int k = base + r * NSL;
      const int64_t g = goff + int64_t(k) * p.gout_stride;
      if (act && g < p.n_valid_out) {
        const int64_t off = yb + int64_t(k) * p.ysi;
        y[off] = p.accumulate ? y[off] + a[u * RL + r] : a[u * RL + r];
      }
    }
  }
}

// ------------------------------------------------------------ dispatch -----
template <class K>
static void set_smem(K kern, size_t bytes) {
  // One attribute call per kernel and device is enough; cache by pointer.
  static std::mutex mu;
  static std::unordered_map<const void*, size_t> done;
  int dev = 0;
  cudaGetDevice(&dev);
  const void* key = (const void*)((uintptr_t)(void*)kern ^ (uintptr_t(dev) << 56));
  std::lock_guard<std::mutex> g(mu);
  auto it = done.find(key);
  if (it != done.end() && it->second >= bytes) return;
  SMAT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
  done[key] = bytes;
}

template <class C, int N>
static void fft_tile_launch(const FftArgs& a, cudaStream_t s) {
  constexpr int E = tile_E(N), CT = tile_CT(N, sizeof(C));
  const size_t smem = size_t(N) * CT * sizeof(C);
  const int threads = (N / E) * CT;
  const int64_t blocks = (a.nb + CT - 1) / CT;
  if (blocks == 0) return;
  SMAT_CHECK(blocks < (int64_t(1) << 31), SMAT_UNSUPPORTED, "fft tile: too many batches");
  set_smem(fft_tile_kernel<C, N>, smem);
  fft_tile_kernel<C, N><<<unsigned(blocks), threads, smem, s>>>(a);
  SMAT_CUDA(cudaGetLastError());
}

template <class T, int N>
static void wht_tile_launch(const WhtArgs& a, cudaStream_t s) {
  constexpr int E = tile_E(N), CT = tile_CT(N, sizeof(T));
  const size_t smem = size_t(N) * CT * sizeof(T);
  const int threads = (N / E) * CT;
  const int64_t blocks = (a.nb + CT - 1) / CT;
  if (blocks == 0) return;
  SMAT_CHECK(blocks < (int64_t(1) << 31), SMAT_UNSUPPORTED, "fwht tile: too many batches");
  set_smem(wht_tile_kernel<T, N>, smem);
  wht_tile_kernel<T, N><<<unsigned(blocks), threads, smem, s>>>(a);
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

void launch_fft_tile(int cdt, int N, const FftArgs& a, cudaStream_t s) {
  if (cdt == SMAT_C64) {
    SMAT_N_SWITCH(fft_tile_launch, float2, N, a, s)
  } else if (cdt == SMAT_C128) {
    SMAT_N_SWITCH(fft_tile_launch, double2, N, a, s)
  } else {
    throw Error(SMAT_BAD_DTYPE, "fft tile: complex dtype required");
  }
}

void launch_wht_tile(int dt, int N, const WhtArgs& a, cudaStream_t s) {
  switch (dt) {
    case SMAT_F32: SMAT_N_SWITCH(wht_tile_launch, float, N, a, s) break;
    case SMAT_F64: SMAT_N_SWITCH(wht_tile_launch, double, N, a, s) break;
    case SMAT_C64: SMAT_N_SWITCH(wht_tile_launch, float2, N, a, s) break;
    case SMAT_C128: SMAT_N_SWITCH(wht_tile_launch, double2, N, a, s) break;
    case SMAT_I32: SMAT_N_SWITCH(wht_tile_launch, int32_t, N, a, s) break;
    case SMAT_I64: SMAT_N_SWITCH(wht_tile_launch, long long, N, a, s) break;
    default: throw Error(SMAT_BAD_DTYPE, "fwht: unsupported dtype");
  }
}

// ------------------------------------------------------ twiddle tables -----
__global__ void tw_init_kernel(double2* d, float2* f, int64_t n, int64_t count, int64_t step) {
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= count) return;
  // exp(-2 pi i (t*step) / n) with the angle reduced exactly in integers.
  const int64_t m = (t * step) % n;
  double s, c;
  sincospi(-2.0 * double(m) / double(n), &s, &c);
  d[t] = make_double2(c, s);
  f[t] = make_float2(float(c), float(s));
}

namespace {
struct TwEntry {
  double2* d = nullptr;
  float2* f = nullptr;
};
std::mutex g_tw_mu;
std::unordered_map<uint64_t, TwEntry> g_tw;  // key: device<<56 | count<<28... (see below)

TwEntry tw_table(int device, int64_t n, int64_t count, int64_t step) {
  const uint64_t key = (uint64_t(device) << 58) ^ (uint64_t(ilog2(n)) << 50) ^
                       (uint64_t(ilog2(count)) << 40) ^ uint64_t(ilog2(step));
  std::lock_guard<std::mutex> g(g_tw_mu);
  auto it = g_tw.find(key);
  if (it != g_tw.end()) return it->second;
  TwEntry e;
  SMAT_CUDA(cudaMalloc(&e.d, count * sizeof(double2)));
  SMAT_CUDA(cudaMalloc(&e.f, count * sizeof(float2)));
  tw_init_kernel<<<unsigned((count + 255) / 256), 256>>>(e.d, e.f, n, count, step);
  SMAT_CUDA(cudaGetLastError());
  SMAT_CUDA(cudaDeviceSynchronize());
  g_tw[key] = e;
  return e;
}
}  // namespace

const void* twiddle4096(int device, bool dbl) {
  TwEntry e = tw_table(device, 4096, 4096, 1);
  return dbl ? (const void*)e.d : (const void*)e.f;
}

TwPair twiddle_pair(int device, int64_t ntot, bool dbl) {
  const int lo_bits = ilog2(ntot) < 12 ? ilog2(ntot) : 12;
  const int64_t lo_n = int64_t(1) << lo_bits;
  const int64_t hi_n = ntot >> lo_bits;
  TwEntry lo = tw_table(device, ntot, lo_n, 1);
  TwEntry hi = tw_table(device, ntot, hi_n, lo_n);
  TwPair p;
  p.lo = dbl ? (const void*)lo.d : (const void*)lo.f;
  p.hi = dbl ? (const void*)hi.d : (const void*)hi.f;
  p.lo_bits = lo_bits;
  return p;
}

}  // namespace smat
