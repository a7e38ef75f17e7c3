// tile_kernels.cu — dispatch of the tiled FFT / FWHT passes and the shared
// device twiddle tables (the device-resident counterpart of the reference's
// DftPlan tables, kernels.py:68-82, shared by every plan on a device).
#include <mutex>
#include <unordered_map>

#include "tile_kernels.cuh"

namespace smat {

void launch_fft_tile_c64_small(int N, const FftArgs& a, cudaStream_t s);
void launch_fft_tile_c64_large(int N, const FftArgs& a, cudaStream_t s);
void launch_fft_tile_c128_small(int N, const FftArgs& a, cudaStream_t s);
void launch_fft_tile_c128_large(int N, const FftArgs& a, cudaStream_t s);

#define SMAT_TMA_DECL(P, N) bool launch_fft_tma_##P##_##N(const FftArgs& a, cudaStream_t s);
SMAT_TMA_DECL(c64, 64)
SMAT_TMA_DECL(c64, 128)
SMAT_TMA_DECL(c64, 256)
SMAT_TMA_DECL(c64, 512)
SMAT_TMA_DECL(c64, 1024)
SMAT_TMA_DECL(c64, 2048)
SMAT_TMA_DECL(c128, 256)
SMAT_TMA_DECL(c128, 512)
SMAT_TMA_DECL(c128, 1024)
SMAT_TMA_DECL(c128, 2048)
#undef SMAT_TMA_DECL

static bool launch_fft_tma_c64(int N, const FftArgs& a, cudaStream_t s) {
  switch (N) {
    case 64: return launch_fft_tma_c64_64(a, s);
    case 128: return launch_fft_tma_c64_128(a, s);
    case 256: return launch_fft_tma_c64_256(a, s);
    case 512: return launch_fft_tma_c64_512(a, s);
    case 1024: return launch_fft_tma_c64_1024(a, s);
    case 2048: return launch_fft_tma_c64_2048(a, s);
    default: return false;
  }
}
static bool launch_fft_tma_c128(int N, const FftArgs& a, cudaStream_t s) {
  switch (N) {
    case 256: return launch_fft_tma_c128_256(a, s);
    case 512: return launch_fft_tma_c128_512(a, s);
    case 1024: return launch_fft_tma_c128_1024(a, s);
    case 2048: return launch_fft_tma_c128_2048(a, s);
    default: return false;
  }
}

// Whether a complex128 outer four-step pass of length N over `inner` columns
// runs on the TMA kernel, which can carry a fused half-length Walsh-Hadamard
// (FftArgs::wht_half): a TMA instantiation exists and whole column tiles.
bool tma_wht_ok(int N, int64_t inner) {
  if (N != 256 && N != 512 && N != 1024 && N != 2048) return false;
  const int ct = N >= 2048 ? 2 : N == 1024 ? 4 : N == 512 ? 8 : 16;  // (TmaGeom::CT, complex128)
  return inner % ct == 0;
}

void launch_fft_tile(int cdt, int N, const FftArgs& a, cudaStream_t s) {
  // persistent TMA-fed variant first (large tiles, complex in and out)
  // (below 256 points only the four-step passes with twiddles / spectra /
  // masks: the plain short passes run at HBM speed on the per-tile kernel)
  const bool pad = (a.g_mod - 1) + (N - 1) * a.gin_stride >= a.n_valid_in;
  const bool trunc = (a.g_mod - 1) + (N - 1) * a.gout_stride >= a.n_valid_out;
  const bool extras = a.mid || a.tw_on || a.pre || a.post || pad || trunc || a.wht_grp;
  if (N >= 256 || (N >= 64 && extras)) {
    if (cdt == SMAT_C64 && launch_fft_tma_c64(N, a, s)) return;
    if (cdt == SMAT_C128 && launch_fft_tma_c128(N, a, s)) return;
  }
  SMAT_CHECK(!a.wht_half, SMAT_UNSUPPORTED, "fused Walsh-Hadamard stages need the TMA pass");
  SMAT_CHECK(!a.wht_grp, SMAT_UNSUPPORTED, "fused Kron Walsh-Hadamard needs the TMA pass");
  if (a.probe_only) return;
  if (cdt == SMAT_C64) {
    if (N <= 64) launch_fft_tile_c64_small(N, a, s);
    else launch_fft_tile_c64_large(N, a, s);
  } else if (cdt == SMAT_C128) {
    if (N <= 64) launch_fft_tile_c128_small(N, a, s);
    else launch_fft_tile_c128_large(N, a, s);
  } else {
    throw Error(SMAT_BAD_DTYPE, "fft tile: complex dtype required");
  }
}

// ------------------------------------------------------ twiddle tables -----
__global__ void tw_init_kernel(double2* d, float2* f, float4* q, int64_t n, int64_t count, int64_t step) {
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= count) return;
  // exp(-2 pi i (t*step) / n) with the angle reduced exactly in integers.
  const int64_t m = (t * step) % n;
  double s, c;
  sincospi(-2.0 * double(m) / double(n), &s, &c);
  d[t] = make_double2(c, s);
  f[t] = make_float2(float(c), float(s));
  q[t] = make_float4(float(c), float(s), -float(s), float(c));  // quad layout for cmul_q
}

namespace {
struct TwEntry {
  double2* d = nullptr;
  float2* f = nullptr;
  float4* q = nullptr;
};
std::mutex g_tw_mu;
std::unordered_map<uint64_t, TwEntry> g_tw;

TwEntry tw_table(int device, int64_t n, int64_t count, int64_t step) {
  const uint64_t key = (uint64_t(device) << 58) ^ (uint64_t(ilog2(n)) << 50) ^
                       (uint64_t(ilog2(count)) << 40) ^ uint64_t(ilog2(step));
  std::lock_guard<std::mutex> g(g_tw_mu);
  auto it = g_tw.find(key);
  if (it != g_tw.end()) return it->second;
  TwEntry e;
  SMAT_CUDA(cudaMalloc(&e.d, count * sizeof(double2)));
  SMAT_CUDA(cudaMalloc(&e.f, count * sizeof(float2)));
  SMAT_CUDA(cudaMalloc(&e.q, count * sizeof(float4)));
  tw_init_kernel<<<unsigned((count + 255) / 256), 256>>>(e.d, e.f, e.q, n, count, step);
  SMAT_CUDA(cudaGetLastError());
  SMAT_CUDA(cudaDeviceSynchronize());
  g_tw[key] = e;
  return e;
}
}  // namespace

// Per-tile four-step twiddle slices: entry g*E + e = W_nt^(g*e) (conjugated
// for inv), one contiguous E-entry slice per tile offset g < nt/E; double2 or
// the quad layout.  The angle is reduced exactly in integers.
__global__ void tw_slice_kernel(double2* d, float4* q, int64_t nt, int64_t E, int inv) {
  for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < nt; t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t m = ((t / E) * (t % E)) % nt;
    double s, c;
    sincospi((inv ? 2.0 : -2.0) * double(m) / double(nt), &s, &c);
    if (d) d[t] = make_double2(c, s);
    if (q) q[t] = make_float4(float(c), float(s), -float(s), float(c));
  }
}

namespace {
std::unordered_map<uint64_t, void*> g_tws;
}

const void* twiddle_slices(int device, int64_t nt, int64_t E, bool inv, bool dbl) {
  const uint64_t key = (uint64_t(device) << 58) ^ (uint64_t(ilog2(nt)) << 40) ^ (uint64_t(ilog2(E)) << 20) ^
                       (uint64_t(inv) << 1) ^ uint64_t(dbl);
  std::lock_guard<std::mutex> g(g_tw_mu);
  auto it = g_tws.find(key);
  if (it != g_tws.end()) return it->second;
  void* p = nullptr;
  SMAT_CUDA(cudaMalloc(&p, size_t(nt) * 16));
  tw_slice_kernel<<<1184, 256>>>(dbl ? (double2*)p : nullptr, dbl ? nullptr : (float4*)p, nt, E, inv ? 1 : 0);
  SMAT_CUDA(cudaGetLastError());
  SMAT_CUDA(cudaDeviceSynchronize());
  g_tws[key] = p;
  return p;
}

const void* twiddle4096(int device, bool dbl) {
  TwEntry e = tw_table(device, 4096, 4096, 1);
  return dbl ? (const void*)e.d : (const void*)e.q;  // single precision: quad layout
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
