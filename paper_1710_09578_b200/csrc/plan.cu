// plan.cu — plan compiler and generic interpreter of the structured-operator tree.
//
// Leaves map onto tiled FFT / FWHT passes (tile_kernels.cu) and pointwise /
// GEMM passes (misc_kernels.cu); composites orchestrate them over strided views
// so that no composite ever materialises a reshaped or transposed copy (the
// reference's Kron._pair_apply loops over columns with reshape/transpose
// copies, composites.py:96-107; here a Kronecker mode is just a stride).
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstring>
#include <mutex>
#include <unordered_map>

#include "plan.cuh"

namespace smat {

// ============================================================ helpers =====
static int cplx_of(int dt) { return dt_complex_of(dt); }

DevBuf* new_buf(Plan& p, int dt, int64_t len) {
  auto b = std::make_unique<DevBuf>();
  b->dt = dt;
  b->len = len;
  b->bytes = size_t(len) * dt_size(dt);
  if (b->bytes) {
    cudaError_t e = cudaMalloc(&b->p, b->bytes);
    if (e != cudaSuccess) {
      cudaGetLastError();
      throw Error(SMAT_OOM, "plan parameter allocation of " + std::to_string(b->bytes) + " bytes failed");
    }
  }
  DevBuf* r = b.get();
  p.bufs.push_back(std::move(b));
  return r;
}

// Host conversion of a parameter array into `target` element type.
static std::vector<unsigned char> convert_host(const smat_param& prm, int target) {
  const int64_t n = prm.len;
  std::vector<unsigned char> out(size_t(n) * dt_size(target));
  auto get = [&](int64_t i, double& re, double& im) {
    re = im = 0;
    switch (prm.dtype) {
      case SMAT_F32: re = ((const float*)prm.data)[i]; break;
      case SMAT_F64: re = ((const double*)prm.data)[i]; break;
      case SMAT_C64: re = ((const float*)prm.data)[2 * i]; im = ((const float*)prm.data)[2 * i + 1]; break;
      case SMAT_C128: re = ((const double*)prm.data)[2 * i]; im = ((const double*)prm.data)[2 * i + 1]; break;
      case SMAT_I32: re = double(((const int32_t*)prm.data)[i]); break;
      case SMAT_I64: re = double(((const int64_t*)prm.data)[i]); break;
      default: throw Error(SMAT_BAD_DTYPE, "parameter dtype");
    }
  };
  if (dt_int(target)) {
    SMAT_CHECK(dt_int(prm.dtype), SMAT_BAD_DTYPE, "integer plan needs integer parameters");
    for (int64_t i = 0; i < n; ++i) {
      int64_t v = prm.dtype == SMAT_I32 ? ((const int32_t*)prm.data)[i] : ((const int64_t*)prm.data)[i];
      if (target == SMAT_I32) ((int32_t*)out.data())[i] = int32_t(v);
      else ((int64_t*)out.data())[i] = v;
    }
    return out;
  }
  SMAT_CHECK(dt_complex(target) || !dt_complex(prm.dtype), SMAT_BAD_DTYPE,
             "complex parameter in a real plan");
  for (int64_t i = 0; i < n; ++i) {
    double re, im;
    get(i, re, im);
    switch (target) {
      case SMAT_F32: ((float*)out.data())[i] = float(re); break;
      case SMAT_F64: ((double*)out.data())[i] = re; break;
      case SMAT_C64: ((float*)out.data())[2 * i] = float(re); ((float*)out.data())[2 * i + 1] = float(im); break;
      case SMAT_C128: ((double*)out.data())[2 * i] = re; ((double*)out.data())[2 * i + 1] = im; break;
    }
  }
  return out;
}

DevBuf* upload_param(Plan& p, const smat_param& prm, int target_dt) {
  DevBuf* b = new_buf(p, target_dt, prm.len);
  if (prm.len) {
    auto h = convert_host(prm, target_dt);
    SMAT_CUDA(cudaMemcpy(b->p, h.data(), h.size(), cudaMemcpyHostToDevice));
  }
  return b;
}

// complex128 device array -> plan complex precision (in place copy into new buffer)
__global__ void c128_to_c64_kernel(const double2* a, float2* b, int64_t n) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    b[i] = make_float2(float(a[i].x), float(a[i].y));
}
static DevBuf* narrow_c128(Plan& p, DevBuf* src, int cdt) {
  if (cdt == SMAT_C128) return src;
  DevBuf* d = new_buf(p, SMAT_C64, src->len);
  c128_to_c64_kernel<<<1184, 256>>>((const double2*)src->p, (float2*)d->p, src->len);
  SMAT_CUDA(cudaGetLastError());
  return d;
}

// ------------------------------------------------------ side streams -------
// One side stream per (device, caller stream): independent callers (threads
// on their own streams, the host path's chunk streams, a stream being
// captured into a CUDA graph) never share one, so a fork neither serialises
// unrelated applies nor drags another caller's work into a capture.
namespace {
std::mutex g_side_mu;
std::unordered_map<uint64_t, cudaStream_t> g_side;
}  // namespace

cudaStream_t Ctx::fork() {
  cudaStream_t side = nullptr;
  {
    const uint64_t key = uint64_t(uintptr_t(stream)) * 64 + uint64_t(device);
    std::lock_guard<std::mutex> lk(g_side_mu);
    auto it = g_side.find(key);
    if (it == g_side.end()) {
      SMAT_CUDA(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
      g_side[key] = side;
    } else {
      side = it->second;
    }
  }
  cudaEvent_t e;
  SMAT_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  SMAT_CUDA(cudaEventRecord(e, stream));
  SMAT_CUDA(cudaStreamWaitEvent(side, e, 0));
  SMAT_CUDA(cudaEventDestroy(e));
  return side;
}

void Ctx::join(cudaStream_t side) {
  cudaEvent_t e;
  SMAT_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  SMAT_CUDA(cudaEventRecord(e, side));
  SMAT_CUDA(cudaStreamWaitEvent(stream, e, 0));
  SMAT_CUDA(cudaEventDestroy(e));
}

// Whether a transform of length Nt runs as a four-step decomposition (else one
// tile pass).  Beyond one tile always; single-precision convolutions of more
// than 2048 points too: a one-tile 4096-point
// convolution keeps only 4 columns per CTA and is load-latency bound, while
// its 64 x 64 four-step runs three passes of 256-byte-row tiles (for C3 the
// intermediate lives mostly in L2).
static bool fourstep(int64_t Nt, bool conv, int cdt) {
  if (Nt > kTileMax) return true;
  return conv && cdt == SMAT_C64 && Nt > 2048;
}

// Split of a four-step transform of length Nt = N1 * N2 (N1 = contiguous /
// middle-pass length).  Must match run_xform.
static void fourstep_split(int64_t Nt, int64_t& N1, int64_t& N2) {
  const int l = ilog2(Nt);
  N1 = int64_t(1) << ((l + 1) / 2);
  N2 = Nt / N1;
}

__global__ void fourstep_perm_kernel(const double2* a, double2* b, int64_t N1, int64_t N2) {
  const int64_t n = N1 * N2;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t k2 = i / N1, k1 = i % N1;
    b[i] = a[k2 + N2 * k1];
  }
}

// A length-n pre/post vector of a four-step transform of length Nt = N1*N2 in
// per-tile order: out[n1*N2 + i] = v[n1 + N1*i] (0 past n), so the strided
// passes (goff = n1, element i) read one contiguous slice per tile.
template <class C>
__global__ void fourstep_vec_kernel(const C* v, C* out, int64_t n, int64_t N1, int64_t N2) {
  const int64_t tot = N1 * N2;
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < tot; q += int64_t(gridDim.x) * blockDim.x) {
    const int64_t n1 = q / N2, i = q % N2, g = n1 + N1 * i;
    out[q] = g < n ? v[g] : C{};
  }
}

// S -> (S[2k], S[2k+1]) and the twiddles W_L^i (i < L/2) of the pruned
// Toeplitz embedding.
__global__ void split_even_odd_kernel(const double2* s, double2* se, double2* so, double2* tw, int64_t L) {
  for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < L / 2; k += int64_t(gridDim.x) * blockDim.x) {
    se[k] = s[2 * k];
    so[k] = s[2 * k + 1];
    double sn, cs;
    sincospi(-2.0 * double(k) / double(L), &sn, &cs);
    tw[k] = make_double2(cs, sn);
  }
}

template <class C>
__global__ void vec_mul_kernel(const C* a, const C* b, C* o, int64_t n) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    o[i] = cmul(a[i], b[i]);
}

// U~ rows in the C5 blocked chain's A2 unit order: unit row g = T' 64 + b,
// T' = k2 NWa + a, holds logical row a + NWa b + N1 k2 of Uw, scaled.
__global__ void utilde_perm_kernel(const double2* Uw, double2* Ut, int64_t P, int64_t r, int64_t N1, int64_t NWa,
                                   double scale) {
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < P * r; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t g = e / r, q = e % r;
    const int64_t Tp = g / 64, b = g % 64, k2 = Tp / NWa, a = Tp % NWa;
    const double2 v = Uw[(a + NWa * b + N1 * k2) * r + q];
    Ut[e] = make_double2(v.x * scale, v.y * scale);
  }
}


// Per-tile (four-step) copy of a pre/post vector of length n for transforms of
// length Nt > kTileMax; nullptr when the transform is a single tile.
static DevBuf* fourstep_vector(Plan& p, const DevBuf* v, int64_t n, int64_t Nt, int cdt) {
  if (!v || Nt <= kTileMax) return nullptr;
  int64_t N1, N2;
  fourstep_split(Nt, N1, N2);
  DevBuf* o = new_buf(p, cdt, Nt);
  if (cdt == SMAT_C128)
    fourstep_vec_kernel<double2><<<1184, 256>>>((const double2*)v->p, (double2*)o->p, n, N1, N2);
  else
    fourstep_vec_kernel<float2><<<1184, 256>>>((const float2*)v->p, (float2*)o->p, n, N1, N2);
  SMAT_CUDA(cudaGetLastError());
  return o;
}

// A convolution spectrum as the plan stores it: four-step order when the
// convolution runs four-step (so the middle pass reads it contiguously per
// tile), then in the plan's complex precision (double2 / float2).
static DevBuf* spectrum_for_plan(Plan& p, DevBuf* src, int cdt) {
  DevBuf* s = src;
  if (fourstep(src->len, true, cdt)) {
    int64_t N1, N2;
    fourstep_split(src->len, N1, N2);
    s = new_buf(p, SMAT_C128, src->len);
    fourstep_perm_kernel<<<1184, 256>>>((const double2*)src->p, (double2*)s->p, N1, N2);
    SMAT_CUDA(cudaGetLastError());
  }
  // single precision: plain float2 entries (the passes form (-w.y, w.x)
  // themselves: half the bytes of the quad layout per tile slice)
  return narrow_c128(p, s, cdt);
}

// ------------------------------------------------------ view utilities -----
// Merge (o1, o2) into a single outer index when both views allow it, so that
// multi-pass transforms see n1 == 1.  Returns false when not mergeable.
static bool merge_outer(Geo& g, Blk& x, Blk& y) {
  if (g.n1 == 1) return true;
  if (g.n2 == 1) {
    g.n2 = g.n1;
    g.n1 = 1;
    x.s2 = x.s1;
    y.s2 = y.s1;
    return true;
  }
  if (x.s1 == g.n2 * x.s2 && y.s1 == g.n2 * y.s2) {
    g.n2 *= g.n1;
    g.n1 = 1;
    return true;
  }
  return false;
}

// Host loop over o1 when the outer dims cannot be merged.
template <class F>
static void for_each_o1(const Geo& g, const Blk& x, const Blk& y, F f) {
  Geo g1 = g;
  g1.n1 = 1;
  for (int64_t o = 0; o < g.n1; ++o) {
    Blk xo = x, yo = y;
    xo.p = (char*)x.p + o * x.s1 * int64_t(dt_size(x.dt));
    yo.p = (char*)y.p + o * y.s1 * int64_t(dt_size(y.dt));
    f(g1, xo, yo);
  }
}

static void fill_views(FftArgs& a, const Blk& x, const Blk& y, const Geo& g) {
  a.x = x.p;
  a.y = y.p;
  a.xs1 = x.s1; a.xs2 = x.s2; a.xsi = x.si;
  a.ys1 = y.s1; a.ys2 = y.s2; a.ysi = y.si;
  a.n2 = g.n2;
  a.inner = g.inner;
  a.nb = g.count();
  a.x_real = !dt_complex(x.dt);
  a.y_real = !dt_complex(y.dt);
}

// Promote a real block into a fresh plan-dtype block.
static Blk promote(Ctx& c, const Blk& x, const Geo& g, int64_t rows) {
  if (x.dt == c.dt) return x;
  Blk t = c.alloc_blk(c.dt, g, rows);
  PointArgs pa;
  pa.x = x.p; pa.x_dt = x.dt; pa.y = t.p; pa.y_dt = t.dt;
  pa.xs1 = x.s1; pa.xs2 = x.s2; pa.xsi = x.si;
  pa.ys1 = t.s1; pa.ys2 = t.s2; pa.ysi = t.si;
  pa.n2 = g.n2; pa.inner = g.inner; pa.nb = g.count(); pa.n = rows;
  c.point(pa);
  return t;
}

static void point_copy(Ctx& c, const Blk& x, const Blk& y, const Geo& g, int64_t rows, bool acc,
                       const void* d = nullptr, bool d_conj = false, bool x_conj = false,
                       double sre = 1.0, double sim = 0.0) {
  PointArgs pa;
  pa.x = x.p; pa.x_dt = x.dt; pa.y = y.p; pa.y_dt = y.dt;
  pa.xs1 = x.s1; pa.xs2 = x.s2; pa.xsi = x.si;
  pa.ys1 = y.s1; pa.ys2 = y.s2; pa.ysi = y.si;
  pa.n2 = g.n2; pa.inner = g.inner; pa.nb = g.count(); pa.n = rows;
  pa.d = d; pa.d_conj = d_conj; pa.x_conj = x_conj; pa.accumulate = acc;
  pa.scale_re = sre; pa.scale_im = sim;
  c.point(pa);
}

// ================================================= FFT-along-axis engine ====
// One logical length-Nt transform of every batch of a view, fused with the
// prologue/epilogue described in FftArgs.  Nt <= 4096 runs as one tile pass;
// larger powers of two run the four-step decomposition Nt = N1*N2:
//   pass 1  stride-N1 length-N2 FFTs, twiddle W_Nt^(n1*k2)   x  -> W
//   pass 2a contiguous length-N1 FFTs written in natural order W -> y
//   pass 2b (convolution) length-N1 FFT * spectrum, IFFT, twiddle^-1  W -> W
//   pass 3  (convolution) stride-N1 length-N2 IFFTs               W -> y
struct XformIO {
  Blk x;
  int64_t x_rows = 0;  // rows of x (rows beyond are zero padding)
  Blk y;
  int64_t y_rows = 0;  // rows of y to write (truncation)
  const void* pre = nullptr;
  bool pre_conj = false;
  const void* mid = nullptr;  // spectrum -> circular convolution
  bool mid_conj = false;
  const void* post = nullptr;
  bool post_conj = false;
  // optional per-tile copies (fourstep_vector) of pre / post for the strided
  // passes of a four-step convolution
  const void* pre_fs = nullptr;
  const void* post_fs = nullptr;
  bool conj_x = false, conj_y = false, inv = false, acc = false;
  double scale = 1.0;
  // x (pass 1) / y (pass 3) already in the blocked four-step row layout of
  // this transform: logical row n1 + N1*k2 at ((n1 / 64) * blk_n2b + k2) * 64 +
  // n1 % 64 (rows of `inner` elements) — the DFSumNode chain keeps its
  // intermediate there, so neither outer pass walks 2 MB-page strides
  bool x_blk = false, y_blk = false;
  int64_t blk_n2b = 0;
  // Walsh-Hadamard over the first half of the outer pass's rows fused into
  // pass 1's input (wht_in) / pass 3's output (wht_out): FftArgs::wht_half
  bool wht_in = false, wht_out = false;
  // fused row selection (single-tile transforms only): see FftArgs::in_map
  const int32_t* in_map = nullptr;
  const int32_t* out_map = nullptr;
  int64_t in_rs = 0, out_rs = 0;
};

static void xform_pass_common(FftArgs& a, Ctx& c) {
  a.tw = twiddle4096(c.device, cplx_of(c.dt) == SMAT_C128);
}

// The inverse four-step twiddle sits between pass 2's IFFT and pass 3; it
// goes to pass 3's input when pass 2's tile has no shared memory left for it
// (double precision, N1 >= 2048).
static bool tw_in_pass3(bool dbl, int64_t N1) { return dbl && N1 >= 2048; }

static void run_xform(Ctx& c, int64_t Nt, Geo g, XformIO io) {
  const int cdt = cplx_of(c.dt);
  const bool dbl = cdt == SMAT_C128;
  if (!fourstep(Nt, io.mid != nullptr, cdt)) {
    SMAT_CHECK(!io.x_blk && !io.y_blk, SMAT_UNSUPPORTED, "blocked rows need a four-step transform");
    FftArgs a;
    fill_views(a, io.x, io.y, g);
    xform_pass_common(a, c);
    a.n_valid_in = io.x_rows;
    a.n_valid_out = io.y_rows;
    a.pre = io.pre; a.pre_conj = io.pre_conj;
    a.mid = io.mid; a.mid_conj = io.mid_conj;
    a.post = io.post; a.post_conj = io.post_conj;
    a.conj_x = io.conj_x; a.conj_y = io.conj_y; a.inv = io.inv && !io.mid;
    a.scale = io.scale; a.accumulate = io.acc;
    a.in_map = io.in_map; a.in_rs = io.in_rs;
    a.out_map = io.out_map; a.out_rs = io.out_rs;
    if (c.wgrp) {
      a.wht_grp = c.wgrp;
      a.wg_xs = c.wg_xs;
      a.wg_ys = c.wg_ys;
      c.wg_used = true;
    }
    c.fft(cdt, int(Nt), a);
    return;
  }
  SMAT_CHECK(!io.in_map && !io.out_map, SMAT_UNSUPPORTED, "fused row selection needs a single-tile transform");
  SMAT_CHECK((!io.wht_in || io.x_blk) && (!io.wht_out || io.y_blk), SMAT_UNSUPPORTED,
             "fused Walsh-Hadamard stages need the blocked chain layout");
  SMAT_CHECK(Nt <= int64_t(kTileMax) * kTileMax, SMAT_UNSUPPORTED,
             "transform length " + std::to_string(Nt) + " exceeds the two-pass limit 2^24");
  if (!merge_outer(g, io.x, io.y)) {
    for_each_o1(g, io.x, io.y, [&](const Geo& g1, const Blk& xo, const Blk& yo) {
      XformIO io1 = io;
      io1.x = xo;
      io1.y = yo;
      run_xform(c, Nt, g1, io1);
    });
    return;
  }
  const int64_t ic = g.inner, O = g.n2;
  const int l = ilog2(Nt);
  const int64_t N1 = int64_t(1) << ((l + 1) / 2);
  const int64_t N2 = Nt / N1;
  // (the blocked single-batch passes address user rows through their row
  // stride, so strided column slices are transformed in place; the batched
  // variant folds (n1, column) into one contiguous index)
  SMAT_CHECK((O == 1 && N1 >= 128) || (io.x.si == ic && io.y.si == ic), SMAT_UNSUPPORTED,
             "four-step FFT needs row-contiguous views");
  const TwPair tw = twiddle_pair(c.device, Nt, dbl);
  // plain inverse transform = conj(F conj(.)) spread over the passes
  bool conj_first = io.conj_x, conj_last = io.conj_y;
  if (io.inv && !io.mid) {
    conj_first = !conj_first;
    conj_last = !conj_last;
  }
  const size_t m0 = c.mark();
  Geo gw;
  gw.n2 = O;
  gw.inner = ic;
  Blk W = c.alloc_blk(cdt, gw, Nt);
  // Blocked intermediate (single outer batch): logical row n1 + N1*k2 of W is
  // stored at ((n1 / B)*N2 + k2)*B + n1 % B, B = 64 — the strided passes then
  // walk W with a B-row stride and the middle pass reads B contiguous rows
  // per block, instead of both walking N1*K-element strides that put every
  // row in its own 2 MB page (translation-bound, tools/tma_probe.cu).  Only
  // the user-layout side of the outer passes stays strided.
  const bool blk = O == 1 && N1 >= 128;
  SMAT_CHECK(blk || (!io.x_blk && !io.y_blk), SMAT_UNSUPPORTED, "blocked rows need the blocked four-step path");
  SMAT_CHECK(!io.y_blk || io.mid, SMAT_UNSUPPORTED, "blocked output rows need the convolution passes");
  constexpr int BL = 6;
  const int64_t B = int64_t(1) << BL;
  auto pass1 = [&]() {
    FftArgs a;
    xform_pass_common(a, c);
    a.x = io.x.p; a.x_real = !dt_complex(io.x.dt);
    a.xs1 = B * io.x.si; a.xs2 = io.x.si; a.xsi = N1 * io.x.si;  // (n1 / B, n1 % B, k2)
    a.y = W.p; a.y_real = 0;
    a.ys1 = N2 * B * ic; a.ys2 = ic; a.ysi = B * ic;
    if (io.x_blk) {  // x in the blocked row layout too
      a.xs1 = io.blk_n2b * B * ic; a.xs2 = ic; a.xsi = B * ic;
    }
    a.n2 = B; a.inner = ic; a.nb = N1 * ic;
    a.g_div = ic; a.g_mod = N1; a.gin_stride = N1;
    a.n_valid_in = io.x_rows;
    a.pre = io.pre; a.pre_conj = io.pre_conj; a.conj_x = conj_first;
    if (io.pre_fs) {
      a.pre = io.pre_fs;
      a.pre_gmul = N2;
    }
    a.tw_on = 1; a.tw_inv = 0; a.tw_lo = tw.lo; a.tw_hi = tw.hi; a.tw_lo_bits = tw.lo_bits; a.tw_mask = Nt - 1;
    a.tw_slices = twiddle_slices(c.device, Nt, N2, false, dbl);
    a.wht_half = io.wht_in ? 1 : 0;
    return a;
  };
  const bool tw3 = tw_in_pass3(dbl, N1);
  auto pass2 = [&]() {  // convolution: W -> W
    FftArgs a;
    xform_pass_common(a, c);
    a.x = W.p; a.y = W.p;
    a.xs1 = W.s2; a.xs2 = N1 * ic; a.xsi = ic;
    a.ys1 = W.s2; a.ys2 = N1 * ic; a.ysi = ic;
    a.n2 = N2; a.inner = ic; a.nb = O * N2 * ic;
    a.g_div = ic; a.g_mod = N2;
    if (blk) {
      a.xs2 = a.ys2 = B * ic;
      a.i_lo_bits = BL; a.xsi_hi = a.ysi_hi = N2 * B * ic;
    }
    // spectra longer than one tile are stored in four-step order
    // (spec_fs[k2*N1 + k1] = spec[k2 + N2*k1], see spectrum_for_plan)
    a.mid = io.mid; a.mid_conj = io.mid_conj; a.mid_stride = 1; a.mid_gmul = N1;
    if (!tw3) {
      a.tw_on = 1; a.tw_inv = 1; a.tw_lo = tw.lo; a.tw_hi = tw.hi; a.tw_lo_bits = tw.lo_bits; a.tw_mask = Nt - 1;
      a.tw_slices = twiddle_slices(c.device, Nt, N1, true, dbl);
    }
    return a;
  };
  auto pass3 = [&]() {  // W -> y
    FftArgs a;
    xform_pass_common(a, c);
    a.x = W.p; a.x_real = 0;
    a.xs1 = 0; a.xs2 = W.s2; a.xsi = N1 * ic;
    a.y = io.y.p; a.y_real = !dt_complex(io.y.dt);
    a.ys1 = 0; a.ys2 = io.y.s2; a.ysi = N1 * io.y.si;
    a.n2 = O; a.inner = N1 * ic; a.nb = O * N1 * ic;
    if (blk) {  // (n1 / B, n1 % B, k2) as in pass 1
      a.xs1 = N2 * B * ic; a.xs2 = ic; a.xsi = B * ic;
      a.ys1 = B * io.y.si; a.ys2 = io.y.si; a.ysi = N1 * io.y.si;
      if (io.y_blk) {
        a.ys1 = io.blk_n2b * B * ic; a.ys2 = ic; a.ysi = B * ic;
      }
      a.n2 = B; a.inner = ic; a.nb = N1 * ic;
    }
    a.g_div = ic; a.g_mod = N1; a.gout_stride = N1;
    a.n_valid_out = io.y_rows;
    a.inv = 1;
    a.wht_half = io.wht_out ? 2 : 0;
    if (tw3) {
      // pass 2's inverse twiddle W^-(n1*k2), applied to this pass's input
      a.tw_on = 1; a.tw_pre = 1; a.tw_inv = 1;
      a.tw_lo = tw.lo; a.tw_hi = tw.hi; a.tw_lo_bits = tw.lo_bits; a.tw_mask = Nt - 1;
      a.tw_slices = twiddle_slices(c.device, Nt, N2, true, dbl);
    }
    a.post = io.post; a.post_conj = io.post_conj; a.conj_y = io.conj_y;
    if (io.post_fs) {
      a.post = io.post_fs;
      a.post_gmul = N2;
    }
    a.scale = io.scale; a.accumulate = io.acc;
    return a;
  };
  // ---- pass 1: x -> W
  if (blk) {
    c.fft(cdt, int(N2), pass1());
  } else {
    FftArgs a;
    xform_pass_common(a, c);
    a.x = io.x.p; a.x_real = !dt_complex(io.x.dt);
    a.xs1 = 0; a.xs2 = io.x.s2; a.xsi = N1 * io.x.si;
    a.y = W.p; a.y_real = 0;
    a.ys1 = 0; a.ys2 = W.s2; a.ysi = N1 * ic;
    a.n2 = O; a.inner = N1 * ic; a.nb = O * N1 * ic;
    a.g_div = ic; a.g_mod = N1; a.gin_stride = N1;
    a.n_valid_in = io.x_rows;
    a.pre = io.pre; a.pre_conj = io.pre_conj; a.conj_x = conj_first;
    if (io.pre_fs) {
      a.pre = io.pre_fs;
      a.pre_gmul = N2;
    }
    a.tw_on = 1; a.tw_inv = 0; a.tw_lo = tw.lo; a.tw_hi = tw.hi; a.tw_lo_bits = tw.lo_bits; a.tw_mask = Nt - 1;
    a.tw_slices = twiddle_slices(c.device, Nt, N2, false, dbl);
    c.fft(cdt, int(N2), a);
  }
  if (!io.mid) {
    // ---- pass 2 (plain): W -> y in natural order
    FftArgs a;
    xform_pass_common(a, c);
    a.x = W.p; a.x_real = 0;
    a.xs1 = W.s2; a.xs2 = N1 * ic; a.xsi = ic;
    a.y = io.y.p; a.y_real = !dt_complex(io.y.dt);
    a.ys1 = io.y.s2; a.ys2 = io.y.si; a.ysi = N2 * io.y.si;
    if (blk) {  // W rows n1 of block k2: B contiguous, then N2*B rows apart
      a.xs2 = B * ic;
      a.i_lo_bits = BL; a.xsi_hi = N2 * B * ic; a.ysi_hi = B * a.ysi;
    }
    a.n2 = N2; a.inner = ic; a.nb = O * N2 * ic;
    a.g_div = ic; a.g_mod = N2; a.gout_stride = N2;
    a.n_valid_out = io.y_rows;
    a.post = io.post; a.post_conj = io.post_conj; a.conj_y = conj_last;
    a.scale = io.scale; a.accumulate = io.acc;
    c.fft(cdt, int(N1), a);
  } else {
    c.fft(cdt, int(N1), pass2());
    c.fft(cdt, int(N2), pass3());
  }
  c.release(m0);
}

// ==================================================== FWHT engine =========
// One FWHT pass over bits [lo, lo+w) of a 2^order transform.  x_rows /
// y_rows mask the global row r = l + 2^lo*m + 2^(lo+w)*h: zero-pad rows
// r >= x_rows on load (first pass only, lo == 0) and skip rows r >= y_rows on
// store (last pass only, lo + w == order) — Partial(Hadamard, arange, arange).
// Fused row selection of a pass: rows of the transform come from / go to rows
// of a compact block through an int32 map (Partial with unique indices).
struct RowMaps {
  const int32_t* in = nullptr;   // first pass: transform row -> compact x row (-1: zero)
  int64_t in_rs = 0;
  const int32_t* out = nullptr;  // last pass: transform row -> compact y row (-1: skip)
  int64_t out_rs = 0;
};

static void wht_pass(Ctx& c, int order, int lo, int w, const Geo& g, const Blk& x, const Blk& y,
                     bool acc, int64_t x_rows, int64_t y_rows, const RowMaps& maps = RowMaps{}) {
  WhtArgs a;
  const int64_t full = int64_t(1) << order;
  if (lo == 0 && maps.in) {
    a.in_map = maps.in;
    a.in_rs = maps.in_rs;
    x_rows = full;  // (every transform row has a map entry)
  }
  if (lo + w == order && maps.out) {
    a.out_map = maps.out;
    a.out_rs = maps.out_rs;
    y_rows = full;
  }
  a.map_k = g.inner;
  const int64_t hi_cnt = int64_t(1) << (order - lo - w);
  a.x = x.p; a.y = y.p;
  a.xs1 = x.s1; a.xs2 = x.s2; a.xsi = x.si;
  a.ys1 = y.s1; a.ys2 = y.s2; a.ysi = y.si;
  a.n2 = g.n2; a.inner = g.inner; a.nb = g.count();
  if (lo > 0 || hi_cnt > 1) {
    // fold: outer1 = O (stride s2), outer2 = high bits, inner = (low bits, c)
    a.xs1 = x.s2; a.xs2 = (int64_t(1) << (lo + w)) * x.si; a.xsi = (int64_t(1) << lo) * x.si;
    a.ys1 = y.s2; a.ys2 = (int64_t(1) << (lo + w)) * y.si; a.ysi = (int64_t(1) << lo) * y.si;
    a.n2 = hi_cnt;
    a.inner = (int64_t(1) << lo) * g.inner;
    a.nb = g.n2 * hi_cnt * a.inner;
    a.g_div = g.inner;
    if (lo == 0) {  // first pass: r = m + 2^w * h, h = (b / ic) % hi
      a.g_mod = hi_cnt;
      a.g_mul = int64_t(1) << w;
      a.gin_stride = a.gout_stride = 1;
    } else {  // r = l + 2^lo * m (+ 2^(lo+w) h, only masked when hi == 1)
      a.g_mod = int64_t(1) << lo;
      a.g_mul = 1;
      a.gin_stride = a.gout_stride = int64_t(1) << lo;
    }
    SMAT_CHECK(x_rows == INT64_MAX || lo == 0, SMAT_UNSUPPORTED, "fwht input mask on a middle pass");
    SMAT_CHECK(y_rows == INT64_MAX || hi_cnt == 1, SMAT_UNSUPPORTED, "fwht output mask on a middle pass");
  }
  a.n_valid_in = x_rows;
  a.n_valid_out = y_rows;
  a.accumulate = acc;
  c.wht(c.dt, 1 << w, a);
}

// Hadamard of order `order` along the rows of x -> y; x has x_rows valid rows
// (zero padding beyond), only the first y_rows rows of the result are written.
static void run_wht(Ctx& c, int order, Geo g, Blk x, Blk y, bool acc, int64_t x_rows = INT64_MAX,
                    int64_t y_rows = INT64_MAX, const RowMaps& maps = RowMaps{}) {
  const int64_t N = int64_t(1) << order;
  SMAT_CHECK((!maps.in && !maps.out) || (g.n1 * g.n2 == 1 && N > 1), SMAT_UNSUPPORTED,
             "fused row selection needs a single batch");
  if (x_rows >= N) x_rows = INT64_MAX;
  if (y_rows >= N) y_rows = INT64_MAX;
  if (N == 1) {
    point_copy(c, x, y, g, 1, acc);
    return;
  }
  if (N <= kTileMax) {
    wht_pass(c, order, 0, order, g, x, y, acc, x_rows, y_rows, maps);
    return;
  }
  if (!merge_outer(g, x, y)) {
    for_each_o1(g, x, y, [&](const Geo& g1, const Blk& xo, const Blk& yo) {
      run_wht(c, order, g1, xo, yo, acc, x_rows, y_rows);
    });
    return;
  }
  // (the first pass reads any row stride; the later ones fold the low row
  // bits with the columns into one contiguous index)
  SMAT_CHECK(y.si == g.inner, SMAT_UNSUPPORTED, "multi-pass FWHT needs a row-contiguous output");
  const int npass = (order + 11) / 12;
  std::vector<int> widths(npass, order / npass);
  for (int i = 0; i < order % npass; ++i) widths[i] += 1;
  const size_t m0 = c.mark();
  Blk T = y;
  const bool y_ok = !acc && y.si == g.inner && y_rows == INT64_MAX && !maps.out;
  if (!y_ok) T = c.alloc_blk(c.dt, g, N);
  int lo = 0;
  for (int p = 0; p < npass; ++p) {
    const bool last = p == npass - 1;
    const Blk& src = p == 0 ? x : T;
    const Blk& dst = (last && !y_ok) ? y : T;
    wht_pass(c, order, lo, widths[p], g, src, dst, last && !y_ok ? acc : false, p == 0 ? x_rows : INT64_MAX,
             last ? y_rows : INT64_MAX, maps);
    lo += widths[p];
  }
  c.release(m0);
}

// ========================================================== leaf nodes =====
struct IdentityNode : Node {
  std::string describe() const override { return "Identity(" + std::to_string(rows) + ")"; }
  bool accepts_real() const override { return true; }
  bool is_identity() const override { return true; }
  void apply(Ctx& c, bool, const Blk& x, const Blk& y, const Geo& g, bool acc) override {
    point_copy(c, x, y, g, rows, acc);
  }
};

struct ZeroNode : Node {
  std::string describe() const override { return "Zero"; }
  bool accepts_real() const override { return true; }
  void apply(Ctx& c, bool adj, const Blk&, const Blk& y, const Geo& g, bool acc) override {
    if (acc) return;
    PointArgs pa;
    pa.y = y.p; pa.y_dt = y.dt;
    pa.ys1 = y.s1; pa.ys2 = y.s2; pa.ysi = y.si;
    pa.n2 = g.n2; pa.inner = g.inner; pa.nb = g.count(); pa.n = adj ? cols : rows;
    c.point(pa);
  }
};

struct DiagNode : Node {
  DevBuf* d = nullptr;
  std::string describe() const override { return "Diagonal(" + std::to_string(rows) + ")"; }
  bool accepts_real() const override { return true; }
  void apply(Ctx& c, bool adj, const Blk& x, const Blk& y, const Geo& g, bool acc) override {
    point_copy(c, x, y, g, rows, acc, d->p, adj);
  }
};

struct DenseNode : Node {
  DevBuf* A = nullptr;
  std::string describe() const override {
    return "Dense(" + std::to_string(rows) + "x" + std::to_string(cols) + ")";
  }
  void apply(Ctx& c, bool adj, const Blk& x0, const Blk& y, const Geo& g, bool acc) override {
    const size_t m0 = c.mark();
    Blk x = promote(c, x0, g, adj ? rows : cols);
    if (!dt_int(c.dt) && blas_available() && g.n1 * g.n2 == 1 && x.si == g.inner && y.si == g.inner) {
      // library GEMM on the row-major blocks viewed column-major:
      //   forward  Y' (K x rows) = X' (K x cols) A^T     (A^T = A's memory, ld cols)
      //   backward Y' (K x cols) = X' (K x rows) conj(A) = X' (A^T)^H
      if (!adj) c.gemm_blas(0, 0, g.inner, rows, cols, x.p, x.si, A->p, cols, acc ? 1.0 : 0.0, y.p, y.si);
      else c.gemm_blas(0, 2, g.inner, cols, rows, x.p, x.si, A->p, cols, acc ? 1.0 : 0.0, y.p, y.si);
      c.release(m0);
      return;
    }
    GemmArgs a;
    a.A = A->p;
    a.lda = cols;
    a.adj = adj;
    a.m = adj ? cols : rows;
    a.k = adj ? rows : cols;
    a.x = x.p; a.y = y.p;
    a.xs1 = x.s1; a.xs2 = x.s2; a.xsi = x.si;
    a.ys1 = y.s1; a.ys2 = y.s2; a.ysi = y.si;
    a.n1 = g.n1; a.n2 = g.n2; a.inner = g.inner;
    a.accumulate = acc;
    c.gemm(a);
    c.release(m0);
  }
};

struct LowRankNode : Node {
  DevBuf *U = nullptr, *V = nullptr, *s = nullptr;
  int64_t r = 0;
  // complex128, rank <= 32: the factors in the padded row layouts of the
  // tensor-core passes (wlr_pitch: c = contraction, e = expansion fragments)
  DevBuf *Uc = nullptr, *Ue = nullptr, *Vc = nullptr, *Ve = nullptr;
  // C5 blocked chain (DFSumNode): U~ = H_{N2b} U / N2b (the Hadamard's k2
  // stages applied ahead), rows in the chain's A2 unit order, both layouts
  DevBuf *Utc = nullptr, *Ute = nullptr;
  std::string describe() const override {
    return "LowRank(rank " + std::to_string(r) + (r <= 32 ? ", FP64 tensor-core halves" : "") + ")";
  }
  // tall-skinny rank-r kernels apply (complex plan, rank <= 32, single batch)
  bool split_ok(const Ctx& c, const Blk& x, const Blk& y, const Geo& g) const {
    (void)y;
    return dt_complex(c.dt) && x.dt == c.dt && r <= 32 && g.n1 * g.n2 == 1;
  }
  // scratch of one contraction: complex128 -> per-CTA partials + the three
  // real W' tables; complex64 -> W (r x K)
  size_t w_bytes(const Ctx& c, const Geo& g) const {
    if (c.dt == SMAT_C128)
      return ((wlr_partial_bytes(c.device, g.inner) + 255) & ~size_t(255)) + size_t(3) * 32 * g.inner * 8;
    return size_t(r) * size_t(g.inner) * dt_size(c.dt);
  }
  static double* w3_of(const Ctx& c, void* w, int64_t K) {
    return reinterpret_cast<double*>(static_cast<char*>(w) + ((wlr_partial_bytes(c.device, K) + 255) & ~size_t(255)));
  }
  // W = F^H x (F = V forward, U backward), diag(s) folded in (conj for the adjoint)
  void contract(Ctx& c, bool adj, const Blk& x, const Geo& g, void* w) const {
    const int64_t kin = adj ? rows : cols;
    if (c.dt == SMAT_C128) {
      WlrMode m;
      m.nw = 1; m.con = true; m.exp = false; m.in = true; m.out = false;
      WlrArgs a;
      a.in.p = x.p; a.in.ld = x.si; a.in.rows = kin;
      a.F = (adj ? Uc : Vc)->p; a.r = r;
      a.nrows = kin; a.n_f = kin; a.n_out = 0; a.K = g.inner;
      a.partial = w;
      c.wlr(m, a, "lowrank_contract");
      c.wlr_fin(w, r, g.inner, s ? s->p : nullptr, adj, w3_of(c, w, g.inner));
      return;
    }
    LowRankArgs la;
    la.F = (adj ? U : V)->p; la.x = x.p; la.w = w; la.rows = kin; la.r = r;
    la.K = g.inner; la.ldx = x.si;
    c.lr_contract(la);
  }
  // y (+)= G W' (G = U forward, V backward)
  void expand(Ctx& c, bool adj, const void* w, const Blk& y, const Geo& g, bool acc) const {
    const int64_t kout = adj ? cols : rows;
    if (c.dt == SMAT_C128) {
      WlrMode m;
      m.nw = 1; m.con = false; m.exp = true; m.in = acc; m.out = true;
      WlrArgs a;
      a.in.p = y.p; a.in.ld = y.si; a.in.rows = kout;
      a.y = y.p; a.yout.g_lo = 1; a.yout.ld = y.si;
      a.F = (adj ? Ve : Ue)->p; a.r = r;
      a.nrows = kout; a.n_out = kout; a.n_f = kout; a.K = g.inner;
      a.w3 = w3_of(c, const_cast<void*>(w), g.inner);
      c.wlr(m, a, "lowrank_expand");
      return;
    }
    LowRankArgs lb;
    lb.F = (adj ? V : U)->p; lb.w = const_cast<void*>(w); lb.y = y.p; lb.rows = kout; lb.r = r;
    lb.K = g.inner; lb.ldy = y.si;
    lb.s = s ? s->p : nullptr; lb.s_conj = adj; lb.accumulate = acc;
    c.lr_expand(lb);
  }
  void apply(Ctx& c, bool adj, const Blk& x0, const Blk& y, const Geo& g, bool acc) override {
    // fwd: y = U diag(s) V^H x ; adj: x' = V diag(conj s) U^H y
    const size_t m0 = c.mark();
    Blk x = promote(c, x0, g, adj ? rows : cols);
    DevBuf* first = adj ? U : V;   // contracted with x (conj-transposed)
    DevBuf* second = adj ? V : U;  // expands back
    const int64_t kin = adj ? rows : cols, kout = adj ? cols : rows;
    if (split_ok(c, x, y, g)) {
      void* w = c.alloc(w_bytes(c, g));
      contract(c, adj, x, g, w);
      expand(c, adj, w, y, g, acc);
      c.release(m0);
      return;
    }
    Blk t = c.alloc_blk(c.dt, g, r);
    GemmArgs a;
    a.A = first->p; a.lda = r; a.adj = 1; a.m = r; a.k = kin;
    a.x = x.p; a.xs1 = x.s1; a.xs2 = x.s2; a.xsi = x.si;
    a.y = t.p; a.ys1 = t.s1; a.ys2 = t.s2; a.ysi = t.si;
    a.n1 = g.n1; a.n2 = g.n2; a.inner = g.inner;
    if (s) { a.rowscale = s->p; a.rowscale_conj = adj; }
    c.gemm(a);
    GemmArgs b;
    b.A = second->p; b.lda = r; b.adj = 0; b.m = kout; b.k = r;
    b.x = t.p; b.xs1 = t.s1; b.xs2 = t.s2; b.xsi = t.si;
    b.y = y.p; b.ys1 = y.s1; b.ys2 = y.s2; b.ysi = y.si;
    b.n1 = g.n1; b.n2 = g.n2; b.inner = g.inner;
    b.accumulate = acc;
    c.gemm(b);
    c.release(m0);
  }
};

struct HadamardNode : Node {
  int order = 0;
  std::string describe() const override { return "Hadamard(" + std::to_string(order) + ")"; }
  void apply(Ctx& c, bool, const Blk& x0, const Blk& y, const Geo& g, bool acc) override {
    const size_t m0 = c.mark();
    Blk x = promote(c, x0, g, rows);
    run_wht(c, order, g, x, y, acc);
    c.release(m0);
  }
};

// Fourier(n): forward DFT (kernels.py:156-161, leaves.py:171-172), backward
// F^H = n * IDFT (leaves.py:174-175); Bluestein for non powers of two
// (kernels.py:83-93, 111-125).
struct FourierNode : Node {
  int64_t n = 0, M = 0;
  DevBuf* chirp = nullptr;   // plan complex precision, length n
  DevBuf* chirp_fs = nullptr;  // its per-tile copy (M > one tile)
  DevBuf* kspec = nullptr;   // FFT_M of the Bluestein kernel, length M
  std::string describe() const override {
    return "Fourier(" + std::to_string(n) + (M ? ", Bluestein M=" + std::to_string(M) : "") + ")";
  }
  bool accepts_real() const override { return true; }
  void apply(Ctx& c, bool adj, const Blk& x, const Blk& y, const Geo& g, bool acc) override {
    XformIO io;
    io.x = x; io.x_rows = n; io.y = y; io.y_rows = n; io.acc = acc;
    if (!M) {
      io.inv = adj;  // F^H = unnormalised inverse
      run_xform(c, n, g, io);
      return;
    }
    io.pre = chirp->p; io.mid = kspec->p; io.post = chirp->p;
    if (chirp_fs) io.pre_fs = io.post_fs = chirp_fs->p;
    io.scale = 1.0 / double(M);
    io.conj_x = adj; io.conj_y = adj;  // F^H y = conj(F conj(y))
    run_xform(c, M, g, io);
  }
};

// Diag(dl) · Fourier(n) · Diag(dr) as ONE transform: the diagonals fold into
// the pre/post vectors of the FFT passes (for Bluestein, into the chirps:
// pre = chirp*dr, post = chirp*dl), so the chain costs no pointwise pass.
//   forward  y = dl * F(dr * x)
//   adjoint  y = conj(dr) * F^H(conj(dl) * x) = conj(dr * F(dl * conj x))
struct DiagFourierNode : Node {
  FourierNode* F = nullptr;
  DevBuf* vr = nullptr;  // applied before the transform (forward): chirp*dr or dr
  DevBuf* vl = nullptr;  // applied after it: chirp*dl or dl (may be the bare chirp)
  DevBuf* vr_fs = nullptr;  // per-tile copies (transform longer than one tile)
  DevBuf* vl_fs = nullptr;
  std::string describe() const override { return "DiagFourierDiag(" + F->describe() + ")"; }
  bool accepts_real() const override { return true; }
  void apply(Ctx& c, bool adj, const Blk& x, const Blk& y, const Geo& g, bool acc) override {
    XformIO io;
    io.x = x; io.x_rows = F->n; io.y = y; io.y_rows = F->n; io.acc = acc;
    io.pre = (adj ? vl : vr) ? (adj ? vl : vr)->p : nullptr;
    io.post = (adj ? vr : vl) ? (adj ? vr : vl)->p : nullptr;
    io.pre_fs = (adj ? vl_fs : vr_fs) ? (adj ? vl_fs : vr_fs)->p : nullptr;
    io.post_fs = (adj ? vr_fs : vl_fs) ? (adj ? vr_fs : vl_fs)->p : nullptr;
    io.conj_x = adj; io.conj_y = adj;
    if (F->M) {
      io.mid = F->kspec->p;
      io.scale = 1.0 / double(F->M);
      run_xform(c, F->M, g, io);
    } else {
      run_xform(c, F->n, g, io);
    }
  }
};

static bool pack_real_pairs(Blk& x, Blk& y, Geo& g, int plan_dt);

// Circulant(c) (leaves.py:207-234): IFFT(spec * FFT(x)); backward uses conj(spec).
struct CirculantNode : Node {
  int64_t n = 0;
  DevBuf* spec = nullptr;
  std::string describe() const override { return "Circulant(" + std::to_string(n) + ")"; }
  bool accepts_real() const override { return true; }
  void apply(Ctx& c, bool adj, const Blk& x0, const Blk& y0, const Geo& g0, bool acc) override {
    Blk x = x0, y = y0;
    Geo g = g0;
    pack_real_pairs(x, y, g, c.dt);
    XformIO io;
    io.x = x; io.x_rows = n; io.y = y; io.y_rows = n; io.acc = acc;
    io.mid = spec->p; io.mid_conj = adj;
    io.scale = 1.0 / double(n);
    run_xform(c, n, g, io);
  }
};

// Toeplitz(col, row_rest) (leaves.py:237-290): circulant embedding of length L.
// Real operator on real data: two real columns (2c, 2c+1) of a (rows, K)
// block are one complex column of the same memory viewed as (rows, K/2)
// complex, and T(a + ib) = Ta + i Tb for real T — one complex transform does
// two real columns and the result lands interleaved exactly where the two
// real outputs belong.
static bool pack_real_pairs(Blk& x, Blk& y, Geo& g, int plan_dt) {
  if (dt_complex(plan_dt) || dt_complex(x.dt) || dt_complex(y.dt) || g.inner % 2) return false;
  auto even = [](int64_t v) { return v % 2 == 0; };
  if (!even(x.s1) || !even(x.s2) || !even(x.si) || !even(y.s1) || !even(y.s2) || !even(y.si)) return false;
  x.dt = y.dt = dt_complex_of(plan_dt);
  x.s1 /= 2; x.s2 /= 2; x.si /= 2;
  y.s1 /= 2; y.s2 /= 2; y.si /= 2;
  g.inner /= 2;
  return true;
}

struct ToeplitzNode : Node {
  int64_t L = 0;
  DevBuf* spec = nullptr;
  // pruned embedding (max(rows, cols) <= L/2): FFT_L of a half-zero input is
  // the two half-length FFTs of x and W_L^i x, and only the first half of
  // the inverse is kept — two length-L/2 convolutions instead of one of L
  DevBuf* spec_e = nullptr;  // S[2k]
  DevBuf* spec_o = nullptr;  // S[2k + 1]
  DevBuf* twid = nullptr;    // W_L^i, i < L/2
  std::string describe() const override {
    return "Toeplitz(" + std::to_string(rows) + "x" + std::to_string(cols) + ", L=" + std::to_string(L) +
           (spec_e ? ", pruned halves" : "") + ")";
  }
  bool accepts_real() const override { return true; }
  void apply(Ctx& c, bool adj, const Blk& x0, const Blk& y0, const Geo& g0, bool acc) override {
    Blk x = x0, y = y0;
    Geo g = g0;
    pack_real_pairs(x, y, g, c.dt);
    XformIO io;
    io.x = x; io.x_rows = adj ? rows : cols;
    io.y = y; io.y_rows = adj ? cols : rows;
    io.acc = acc;
    io.mid_conj = adj;
    io.scale = 1.0 / double(L);
    if (!spec_e) {
      io.mid = spec->p;
      run_xform(c, L, g, io);
      return;
    }
    io.mid = spec_e->p;
    run_xform(c, L / 2, g, io);
    io.mid = spec_o->p;
    io.pre = twid->p;
    io.post = twid->p;
    io.post_conj = true;
    io.acc = true;
    run_xform(c, L / 2, g, io);
  }
};

// ===================================================== composite nodes =====
struct AdjointNode : Node {
  Node* base = nullptr;
  std::string describe() const override { return "Adjoint(" + base->describe() + ")"; }
  bool accepts_real() const override { return base->accepts_real(); }
  void apply(Ctx& c, bool adj, const Blk& x, const Blk& y, const Geo& g, bool acc) override {
    base->apply(c, !adj, x, y, g, acc);
  }
};

// Product(A, B, C) = A·B·C applied right to left (composites.py:49-61).
struct ProductNode : Node {
  std::vector<Node*> f;
  std::string describe() const override {
    std::string s = "Product(";
    for (size_t i = 0; i < f.size(); ++i) s += (i ? ", " : "") + f[i]->describe();
    return s + ")";
  }
  bool accepts_real() const override { return true; }
  void apply(Ctx& c, bool adj, const Blk& x0, const Blk& y, const Geo& g, bool acc) override {
    std::vector<Node*> seq;  // order of application
    if (!adj) seq.assign(f.rbegin(), f.rend());
    else seq.assign(f.begin(), f.end());
    const size_t m0 = c.mark();
    Blk cur = x0;
    if (cur.dt != c.dt && !seq[0]->accepts_real()) cur = promote(c, x0, g, adj ? rows : cols);
    for (size_t i = 0; i < seq.size(); ++i) {
      Node* op = seq[i];
      const int64_t nout = adj ? op->cols : op->rows;
      if (i + 1 == seq.size()) {
        op->apply(c, adj, cur, y, g, acc);
      } else {
        const size_t mk = c.mark();
        Blk nxt = c.alloc_blk(c.dt, g, nout);
        op->apply(c, adj, cur, nxt, g, false);
        // keep nxt alive; release the previous intermediate only if it sits
        // below nxt (stack discipline: we simply never release inside the chain)
        (void)mk;
        cur = nxt;
      }
    }
    c.release(m0);
  }
};

// Sum(*terms): y = sum_k T_k x (new type; the reference expresses it with
// Blocks([[A, B]])·Blocks([[I], [I]]), composites.py:171-178).
struct SumNode : Node {
  std::vector<Node*> t;
  std::string describe() const override {
    std::string s = "Sum(";
    for (size_t i = 0; i < t.size(); ++i) s += (i ? ", " : "") + t[i]->describe();
    return s + ")";
  }
  bool accepts_real() const override { return true; }
  void apply(Ctx& c, bool adj, const Blk& x0, const Blk& y, const Geo& g, bool acc) override {
    const size_t m0 = c.mark();
    Blk xc = x0;
    bool need = false;
    for (Node* op : t) need |= !op->accepts_real();
    if (x0.dt != c.dt && need) xc = promote(c, x0, g, adj ? rows : cols);
    // A rank-r term's contraction (FP64-FMA bound) reads only x: it runs on the
    // side stream while the other terms (memory bound) run here; its expansion
    // accumulates last, after the join.
    // (the same order and allocations in measure / profiling mode, without the
    // fork, so the measured workspace and launch counts match)
    int lr = -1;
    if (t.size() > 1) {
      for (size_t i = 0; i < t.size(); ++i) {
        auto* L = dynamic_cast<LowRankNode*>(t[i]);
        if (L && L->split_ok(c, xc, y, g)) {
          lr = int(i);
          break;
        }
      }
    }
    if (lr >= 0) {
      auto* L = static_cast<LowRankNode*>(t[size_t(lr)]);
      void* w = c.alloc(L->w_bytes(c, g));
      const bool fork = c.can_fork();
      Ctx side = c;
      if (fork) side.stream = c.fork();
      side.launches = 0;
      L->contract(side, adj, xc, g, w);
      c.launches += side.launches;
      bool first = true;
      for (size_t i = 0; i < t.size(); ++i) {
        if (int(i) == lr) continue;
        const Blk& xi = t[i]->accepts_real() ? x0 : xc;
        t[i]->apply(c, adj, xi, y, g, acc || !first);
        first = false;
      }
      if (fork) c.join(side.stream);
      L->expand(c, adj, w, y, g, true);
      c.release(m0);
      return;
    }
    for (size_t i = 0; i < t.size(); ++i) {
      const Blk& xi = t[i]->accepts_real() ? x0 : xc;
      t[i]->apply(c, adj, xi, y, g, acc || i > 0);
    }
    c.release(m0);
  }
};

// Diag·Fourier·Diag (Bluestein, four-step) · Sum(PaddedHadamard, LowRank) —
// the BASELINE C5 chain.  The padded Hadamard H_P (P = 2^order rows, zero
// padding / truncation at the operator's n rows) factors along the
// Bluestein transform's four-step row index r = n1 + N1 k2 (N1 = the middle
// pass length) as H_{N2b}(k2) (x) H_64(b) (x) H_NWa(a), n1 = a + NWa b:
//
//   forward   A1  x -> T1        H_NWa over a, rank-r contraction V^H x of the
//                                input rows (wlr.cu: 64-row x all-column tiles,
//                                FP64 tensor cores)
//             A2  T1 -> T2       H_64 over b, + U~ W' on the output rows
//             B   T2 -> T2'      H_{N2b} over k2 (the FWHT tile pass)
//             Bluestein (Diag·F·Diag folded into its chirps) from T2' in the
//             blocked four-step row layout of the transform
//   backward  the mirror image: Bluestein -> T2' (blocked), B, A2 (with the
//             U~^H contraction of its input rows), A1 (with the V W''
//             expansion of its output rows)
//
// U~ = H_{N2b} U / N2b in A2's row order is built at plan time: adding U~ W'
// ahead of the k2 stages adds U W' after them (the Hadamard is linear, and
// H_{N2b}^2 = N2b I), and in the adjoint U^H z = U~^H (H_{N2b} z).  The
// factor rows are read once per direction — every LowRank tile spans all
// columns — instead of once per column group of a transform tile.
// Blocked layout of T2 / T2' (the Bluestein side): logical row n1 + N1 k2 at
// ((n1 / 64) N2b + k2) 64 + n1 % 64 (XformIO::x_blk / y_blk).  T1: unit rows
// of A2, (k2 NWa + a) 64 + b.
struct DFSumNode : Node {
  Node* fallback = nullptr;       // the generic Product (used when a view does not qualify)
  DiagFourierNode* df = nullptr;
  Node* hp = nullptr;             // PaddedHadamard term
  LowRankNode* lr = nullptr;
  int64_t N1 = 0, N2 = 0, N2b = 0, P = 0, M = 0, NWa = 0;
  std::string describe() const override { return "BlockedChain(" + fallback->describe() + ")"; }
  bool accepts_real() const override { return false; }
  bool usable(const Ctx& c, const Blk& x, const Blk& y, const Geo& g, bool acc) const {
    return !acc && c.dt == SMAT_C128 && g.n1 * g.n2 == 1 && lr->split_ok(c, x, y, g);
  }
  // row maps of the wlr passes (see wlr.cuh); lg(v) = log2 of a power of two
  static int32_t lg(int64_t v) { return ilog2(v); }
  // user rows (unit row = logical row): group T = g / NWa holds rows NWa T + a
  WlrRows user_rows(int64_t ld) const {
    WlrRows m;
    m.g_lo = NWa; m.a_lo = 1; m.ld = ld;
    return m;
  }
  WlrIn user_in(const void* p, int64_t ld, int64_t n) const {
    WlrIn w;
    w.kind = WLR_IN_ROWS; w.p = p; w.ld = ld; w.rows = n;
    return w;
  }
  // T1 as written by A1 (groups T = b + 64 k2 of NWa rows a): row (k2 NWa + a) 64 + b
  WlrRows t1_by_a(int64_t K) const {
    WlrRows m;
    m.gsh = 6; m.g_hi = 64 * NWa; m.g_lo = 1; m.a_lo = 64; m.ld = K;
    return m;
  }
  WlrIn t1_by_a_in(const void* p, int64_t K) const {
    WlrIn w;
    w.kind = WLR_IN_T1A; w.p = p; w.ld = K; w.nwa = NWa; w.n2b = N2b; w.P = P;
    return w;
  }
  // T1 as read by A2 (groups T' = k2 NWa + a of 64 rows b): row 64 T' + b
  WlrRows t1_by_b(int64_t K) const {
    WlrRows m;
    m.g_lo = 64; m.a_lo = 1; m.ld = K;
    return m;
  }
  WlrIn t1_by_b_in(const void* p, int64_t K) const {
    WlrIn w;
    w.kind = WLR_IN_ROWS; w.p = p; w.ld = K; w.rows = P;
    return w;
  }
  // blocked T2 (groups T' = k2 NWa + a, rows b): n1 = a + NWa b ->
  // ((n1 / 64) N2b + k2) 64 + n1 % 64, b = b_lo + (64 / NWa) b_hi
  WlrRows t2_blocked(int64_t K) const {
    WlrRows m;
    m.gsh = lg(NWa); m.g_hi = 64; m.g_lo = 1;
    m.ash = lg(64 / NWa); m.a_lo = NWa; m.a_hi = N2b * 64; m.ld = K;
    return m;
  }
  WlrIn t2_blocked_in(const void* p, int64_t K) const {
    WlrIn w;
    w.kind = WLR_IN_T2B; w.p = p; w.ld = K; w.nwa = NWa; w.n2b = N2b; w.P = P;
    return w;
  }
  // pass B: N2b-point transform over k2, blocked on both sides
  void pass_b(Ctx& c, const void* x, void* y, bool mask_in, int64_t K, int64_t n) const {
    WhtArgs a;
    a.x = x; a.y = y;
    a.xs1 = a.ys1 = N2b * 64 * K; a.xs2 = a.ys2 = K; a.xsi = a.ysi = 64 * K;
    a.n2 = 64; a.inner = K; a.nb = N1 * K;
    a.g_div = K; a.g_mod = N1; a.g_mul = 1; a.gin_stride = a.gout_stride = N1;
    if (mask_in) a.n_valid_in = n;   // backward: unwritten rows >= n read as zero
    else a.n_valid_out = n;          // forward: rows >= n are not stored
    c.wht(c.dt, int(N2b), a);
  }
  // Whether the blocked-side Bluestein pass takes the fused k2 Hadamard stages
  // (TMA kernel): a host-side probe of that pass's launch, cached per
  // (direction, columns, user-side row stride)
  mutable std::mutex fuse_mu;
  mutable std::unordered_map<uint64_t, bool> fuse_memo;
  bool fuse_ok(const Ctx& c, bool adj, const Blk& x, const Blk& y, const Geo& g) const {
    const int64_t K = g.inner;
    if (!tma_wht_ok(int(N2), K)) return false;
    const int64_t ld = adj ? x.si : y.si;
    const uint64_t key = (uint64_t(K) << 33) ^ (uint64_t(ld) << 1) ^ uint64_t(adj);
    {
      std::lock_guard<std::mutex> lk(fuse_mu);
      auto it = fuse_memo.find(key);
      if (it != fuse_memo.end()) return it->second;
    }
    Ctx pc = c;
    pc.measure = true;
    pc.probe = true;
    pc.prof = nullptr;
    pc.top = pc.peak = 0;
    Geo gb;
    gb.inner = K;
    Blk T = pc.alloc_blk(SMAT_C128, gb, P);
    bool ok = true;
    try {
      XformIO io = adj ? df_io(true, x, T, rows) : df_io(false, T, y, rows);
      if (adj) {
        io.y_blk = true; io.y_rows = P; io.wht_out = true;
      } else {
        io.x_blk = true; io.wht_in = true;
      }
      run_xform(pc, M, g, io);
    } catch (const Error& e) {
      if (e.code != SMAT_UNSUPPORTED) throw;
      ok = false;
    }
    std::lock_guard<std::mutex> lk(fuse_mu);
    fuse_memo[key] = ok;
    return ok;
  }
  XformIO df_io(bool adj, const Blk& x, const Blk& y, int64_t n) const {
    XformIO io;
    io.x = x; io.x_rows = n; io.y = y; io.y_rows = n;
    io.pre = (adj ? df->vl : df->vr) ? (adj ? df->vl : df->vr)->p : nullptr;
    io.post = (adj ? df->vr : df->vl) ? (adj ? df->vr : df->vl)->p : nullptr;
    io.pre_fs = (adj ? df->vl_fs : df->vr_fs) ? (adj ? df->vl_fs : df->vr_fs)->p : nullptr;
    io.post_fs = (adj ? df->vr_fs : df->vl_fs) ? (adj ? df->vr_fs : df->vl_fs)->p : nullptr;
    io.conj_x = adj; io.conj_y = adj;
    io.mid = df->F->kspec->p;
    io.scale = 1.0 / double(M);
    io.blk_n2b = N2b;
    return io;
  }
  void apply(Ctx& c, bool adj, const Blk& x0, const Blk& y, const Geo& g, bool acc) override {
    const size_t m0 = c.mark();
    Blk x = promote(c, x0, g, adj ? rows : cols);
    if (!usable(c, x, y, g, acc)) {
      fallback->apply(c, adj, x, y, g, acc);
      c.release(m0);
      return;
    }
    const int64_t K = g.inner, n = rows, r = lr->r;
    Geo gb;
    gb.inner = K;
    Blk Ta = c.alloc_blk(c.dt, gb, P);
    Blk Tb = c.alloc_blk(c.dt, gb, P);
    void* w = c.alloc(lr->w_bytes(c, g));
    double* w3 = LowRankNode::w3_of(c, w, K);
    const void* sv = lr->s ? lr->s->p : nullptr;
    WlrMode ma, mb;
    ma.nw = int(NWa); mb.nw = 64;
    WlrArgs a1, a2;
    a1.r = a2.r = r; a1.K = a2.K = K;
    // the k2 stages of the Hadamard ride in the Bluestein pass on the blocked
    // side when it runs on the TMA kernel, else they are a pass of their own
    const bool fuse_b = fuse_ok(c, adj, x, y, g);
    if (!adj) {
      // y = DF (H_pad x + U diag(s) V^H x)
      ma.con = true;  // A1: x -> T1 (Ta), partials of V^H x
      a1.in = user_in(x.p, x.si, n);
      a1.y = Ta.p; a1.yout = t1_by_a(K);
      a1.F = lr->Vc->p; a1.n_f = n;
      a1.nrows = P; a1.n_out = P;
      a1.partial = w;
      c.wlr(ma, a1, "wht_lowrank_a");
      c.wlr_fin(w, r, K, sv, false, w3);
      mb.exp = true;  // A2: T1 (Ta) -> T2 (Tb), + U~ W'
      a2.in = t1_by_b_in(Ta.p, K);
      a2.y = Tb.p; a2.yout = t2_blocked(K);
      a2.F = lr->Ute->p; a2.n_f = P;
      a2.nrows = P; a2.n_out = P;
      a2.w3 = w3;
      c.wlr(mb, a2, "wht_lowrank_b");
      Blk src = Tb;
      if (!fuse_b) {
        pass_b(c, Tb.p, Ta.p, false, K, n);
        src = Ta;
      }
      XformIO io = df_io(false, src, y, n);
      io.x_blk = true;
      io.wht_in = fuse_b;
      run_xform(c, M, g, io);
    } else {
      // y = (H_pad + V diag(conj s) U^H) DF^H x
      XformIO io = df_io(true, x, Ta, n);
      io.y_blk = true;
      io.y_rows = P;  // rows n..P come out zero (zero-padded post vector)
      io.wht_out = fuse_b;
      run_xform(c, M, g, io);
      Blk t2 = Ta, t1 = Tb;
      if (!fuse_b) {
        pass_b(c, Ta.p, Tb.p, true, K, n);
        t2 = Tb;
        t1 = Ta;
      }
      mb.con = true;  // A2: T2 -> T1, partials of U~^H T2
      a2.in = t2_blocked_in(t2.p, K);
      a2.y = t1.p; a2.yout = t1_by_b(K);
      a2.F = lr->Utc->p; a2.n_f = P;
      a2.nrows = P; a2.n_out = P;
      a2.partial = w;
      c.wlr(mb, a2, "wht_lowrank_b");
      c.wlr_fin(w, r, K, sv, true, w3);
      ma.exp = true;  // A1: T1 -> x', + V W''
      a1.in = t1_by_a_in(t1.p, K);
      a1.y = y.p; a1.yout = user_rows(y.si);
      a1.F = lr->Ve->p; a1.n_f = n;
      a1.nrows = std::min(P, (n + 63) / 64 * 64); a1.n_out = n;
      a1.w3 = w3;
      c.wlr(ma, a1, "wht_lowrank_a");
    }
    c.release(m0);
  }
};

// Kron(A_0, ..., A_{m-1}), np.kron index order (first factor slowest,
// composites.py:96-107): mode a is a strided batched transform.
struct KronNode : Node {
  std::vector<Node*> f;
  std::string describe() const override {
    std::string s = "Kron(";
    for (size_t i = 0; i < f.size(); ++i) s += (i ? ", " : "") + f[i]->describe();
    return s + ")";
  }
  void apply(Ctx& c, bool adj, const Blk& x0, const Blk& y0, const Geo& g0, bool acc) override {
    const size_t m0 = c.mark();
    Geo g = g0;
    Blk x = promote(c, x0, g0, adj ? rows : cols);
    Blk y = y0;
    const int m = int(f.size());
    std::vector<int64_t> sz(m);
    for (int a = 0; a < m; ++a) sz[a] = adj ? f[a]->rows : f[a]->cols;  // current (input) sizes
    auto total = [&]() {
      int64_t t = 1;
      for (int64_t v : sz) t *= v;
      return t;
    };
    if (!merge_outer(g, x, y) || x.si != g.inner || y.si != g.inner) {
      // make both ends contiguous
      Blk xc = c.alloc_blk(c.dt, g0, total());
      point_copy(c, x, xc, g0, total(), false);
      int64_t outrows = adj ? cols : rows;
      Blk yc = c.alloc_blk(c.dt, g0, outrows);
      Geo gc = g0;
      gc.n2 = g0.n1 * g0.n2;
      gc.n1 = 1;
      Blk xcc = xc, ycc = yc;
      xcc.s2 = total() * g0.inner;
      ycc.s2 = outrows * g0.inner;
      apply_modes(c, adj, xcc, ycc, gc, false, sz);
      point_copy(c, yc, y0, g0, outrows, acc);
      c.release(m0);
      return;
    }
    apply_modes(c, adj, x, y, g, acc, sz);
    c.release(m0);
  }

  // Kron(Hadamard(6), A, B), A and B complex64 single-tile transforms of
  // 128 / 256 points (Fourier without Bluestein, Circulant): two passes
  // instead of three — H_64 = H_8 (x) H_8 splits over the A and B passes, each
  // 8-point half running over a tile of 4 or 8 columns x 8 Hadamard rows
  // (warp shuffles across lane bits, FftArgs::wht_grp).  The reference applies every factor
  // mode-wise with per-column copies (composites.py:96-107).
  static bool fft_leaf(const Node* n) {
    if (auto* fo = dynamic_cast<const FourierNode*>(n)) return fo->M == 0 && (fo->n == 128 || fo->n == 256);
    if (auto* ci = dynamic_cast<const CirculantNode*>(n)) return ci->n == 128 || ci->n == 256;
    return false;
  }
  bool fusable(const Ctx& c, const Blk& x, const Blk& y, const Geo& g, bool acc) const {
    if (f.size() != 3 || c.dt != SMAT_C64 || acc || g.n1 * g.n2 != 1 || g.inner % 8) return false;
    if (!dt_complex(x.dt) || !dt_complex(y.dt)) return false;
    auto* h = dynamic_cast<const HadamardNode*>(f[0]);
    return h && h->order == 6 && fft_leaf(f[1]) && fft_leaf(f[2]);
  }
  void run_fused(Ctx& c, bool adj, const Blk& x, const Blk& y, const Geo& g) {
    struct Clear {  // (the fused-WHT request never outlives this call)
      Ctx& c;
      ~Clear() { c.wgrp = 0; }
    } clear{c};
    const int64_t ic = g.inner, na = f[1]->rows, nb = f[2]->rows, plane = na * nb * ic;
    Geo gt;
    gt.inner = ic;
    Blk T = c.alloc_blk(c.dt, gt, 64 * na * nb);
    // pass 1: B over its rows, H_8 over h % 8 (h = 8 hh + lo)
    Geo g1;
    g1.n1 = 8; g1.n2 = na; g1.inner = 8 * ic;
    Blk x1 = x, t1 = T;
    x1.s1 = t1.s1 = 8 * plane; x1.s2 = t1.s2 = nb * ic; x1.si = t1.si = ic;
    c.wgrp = 3; c.wg_xs = c.wg_ys = plane; c.wg_used = false;
    f[2]->apply(c, adj, x1, t1, g1, false);
    SMAT_CHECK(c.wg_used, SMAT_UNSUPPORTED, "kron: fused Walsh-Hadamard not taken");
    // pass 2: A over its rows, H_8 over h / 8
    Geo g2;
    g2.n1 = 8; g2.n2 = nb; g2.inner = 8 * ic;
    Blk t2 = T, y2 = y;
    t2.s1 = y2.s1 = plane; t2.s2 = y2.s2 = ic; t2.si = y2.si = nb * ic;
    c.wgrp = 3; c.wg_xs = c.wg_ys = 8 * plane; c.wg_used = false;
    f[1]->apply(c, adj, t2, y2, g2, false);
    SMAT_CHECK(c.wg_used, SMAT_UNSUPPORTED, "kron: fused Walsh-Hadamard not taken");
  }
  // whether both fused passes run (a launcher probe, cached per direction and width)
  mutable std::mutex fuse_mu;
  mutable std::unordered_map<uint64_t, bool> fuse_memo;
  bool fused_ok(const Ctx& c, bool adj, const Blk& x, const Blk& y, const Geo& g, bool acc) {
    if (!fusable(c, x, y, g, acc)) return false;
    const uint64_t key = (uint64_t(g.inner) << 3) ^ (uint64_t((uintptr_t(x.p) & 15) != 0) << 2) ^
                         (uint64_t((uintptr_t(y.p) & 15) != 0) << 1) ^ uint64_t(adj);
    {
      std::lock_guard<std::mutex> lk(fuse_mu);
      auto it = fuse_memo.find(key);
      if (it != fuse_memo.end()) return it->second;
    }
    Ctx pc = c;
    pc.measure = true;
    pc.probe = true;
    pc.prof = nullptr;
    pc.top = pc.peak = 0;
    bool ok = true;
    try {
      run_fused(pc, adj, x, y, g);
    } catch (const Error& e) {
      if (e.code != SMAT_UNSUPPORTED) throw;
      ok = false;
    }
    std::lock_guard<std::mutex> lk(fuse_mu);
    fuse_memo[key] = ok;
    return ok;
  }

  void apply_modes(Ctx& c, bool adj, const Blk& x, const Blk& y, const Geo& g, bool acc,
                   std::vector<int64_t> sz) {
    if (c.measure && !c.probe && fusable(c, x, y, g, acc)) {
      // sizing / launch counting (placeholder pointers, no probe): the
      // workspace covers the unfused passes too (an apply whose probe fails
      // runs them), the launch count is the fused plan's
      const int64_t l0 = c.launches;
      const size_t m0 = c.mark();
      apply_unfused(c, adj, x, y, g, acc, sz);
      c.release(m0);
      c.launches = l0;
      run_fused(c, adj, x, y, g);
      return;
    }
    if (!c.measure && fused_ok(c, adj, x, y, g, acc)) {
      run_fused(c, adj, x, y, g);
      return;
    }
    apply_unfused(c, adj, x, y, g, acc, sz);
  }
  void apply_unfused(Ctx& c, bool adj, const Blk& x, const Blk& y, const Geo& g, bool acc,
                     std::vector<int64_t> sz) {
    const int m = int(f.size());
    std::vector<int> order;
    for (int a = m - 1; a >= 0; --a)
      if (!f[a]->is_identity()) order.push_back(a);
    const int64_t O = g.n2, ic = g.inner;
    if (order.empty()) {
      int64_t t = 1;
      for (int64_t v : sz) t *= v;
      point_copy(c, x, y, g, t, acc);
      return;
    }
    Blk cur = x;
    for (size_t s = 0; s < order.size(); ++s) {
      const int a = order[s];
      const bool last = s + 1 == order.size();
      int64_t prefix = 1, rest = 1;
      for (int b = 0; b < a; ++b) prefix *= sz[b];
      for (int b = a + 1; b < m; ++b) rest *= sz[b];
      const int64_t nin = sz[a], nout = adj ? f[a]->cols : f[a]->rows;
      Blk dst;
      if (last) {
        dst = y;
      } else {
        Geo gt;
        gt.n2 = O;
        gt.inner = ic;
        dst = c.alloc_blk(c.dt, gt, prefix * nout * rest);
      }
      Geo gm;
      gm.n1 = O;
      gm.n2 = prefix;
      gm.inner = rest * ic;
      Blk xv = cur, yv = dst;
      xv.s1 = cur.s2; xv.s2 = nin * rest * ic; xv.si = rest * ic;
      yv.s1 = dst.s2; yv.s2 = nout * rest * ic; yv.si = rest * ic;
      f[a]->apply(c, adj, xv, yv, gm, last ? acc : false);
      sz[a] = nout;
      cur = dst;
    }
  }
};

// Partial(base, rows, cols) (composites.py:239-320): scatter -> base -> gather.
struct PartialNode : Node {
  Node* base = nullptr;
  DevBuf* ridx = nullptr;  // may be null (all rows)
  DevBuf* cidx = nullptr;
  bool r_unique = true, c_unique = true;
  // base is a Hadamard and both selections are prefixes arange(k): the
  // "Hadamard-padded" operator — zero-pad on load / truncate on store of the
  // FWHT passes, no scatter, gather or padded copies
  int had_order = -1;
  // base is a Hadamard and every selection is duplicate-free: the selection
  // is fused into the FWHT passes as int32 row maps (base row -> compact row,
  // -1 = not selected) — gather on store, scatter on load, no extra passes
  int map_order = -1;
  int64_t map_fourier = 0;  // base is Fourier(n), n a power of two in one tile: maps in the FFT pass
  DevBuf* rmap = nullptr;  // base rows -> selected row position
  DevBuf* cmap = nullptr;  // base cols -> selected col position
  std::string describe() const override {
    return std::string(had_order >= 0     ? "PaddedHadamard("
                       : map_order >= 0   ? "SelectedHadamard("
                       : map_fourier > 0  ? "SelectedFourier("
                                          : "Partial(") +
           base->describe() + ")";
  }
  void apply(Ctx& c, bool adj, const Blk& x0, const Blk& y, const Geo& g, bool acc) override {
    const size_t m0 = c.mark();
    Blk x = promote(c, x0, g, adj ? rows : cols);
    if (had_order >= 0) {
      run_wht(c, had_order, g, x, y, acc, adj ? rows : cols, adj ? cols : rows);
      c.release(m0);
      return;
    }
    if (map_order >= 0 && g.n1 * g.n2 == 1 && x.si == g.inner && y.si == g.inner) {
      RowMaps m;
      DevBuf* in = adj ? rmap : cmap;
      DevBuf* out = adj ? cmap : rmap;
      if (in) {
        m.in = (const int32_t*)in->p;
        m.in_rs = x.si;
      }
      if (out) {
        m.out = (const int32_t*)out->p;
        m.out_rs = y.si;
      }
      run_wht(c, map_order, g, x, y, acc, INT64_MAX, INT64_MAX, m);
      c.release(m0);
      return;
    }
    if (map_fourier > 0 && g.n1 * g.n2 == 1 && x.si == g.inner && y.si == g.inner && dt_complex(c.dt) &&
        !fourstep(map_fourier, false, cplx_of(c.dt))) {
      // Fourier(n) forward DFT / backward F^H (leaves.py:171-175) as one
      // tile pass, selection fused into its load and store
      XformIO io;
      io.x = x; io.x_rows = map_fourier; io.y = y; io.y_rows = map_fourier; io.acc = acc;
      io.inv = adj;
      DevBuf* in = adj ? rmap : cmap;
      DevBuf* out = adj ? cmap : rmap;
      if (in) {
        io.in_map = (const int32_t*)in->p;
        io.in_rs = x.si;
      }
      if (out) {
        io.out_map = (const int32_t*)out->p;
        io.out_rs = y.si;
      }
      run_xform(c, map_fourier, g, io);
      c.release(m0);
      return;
    }
    DevBuf* in_idx = adj ? ridx : cidx;    // scatter side
    DevBuf* out_idx = adj ? cidx : ridx;   // gather side
    const bool in_unique = adj ? r_unique : c_unique;
    const int64_t base_in = adj ? base->rows : base->cols;
    const int64_t base_out = adj ? base->cols : base->rows;
    Blk full_in = x;
    if (in_idx) {
      full_in = c.alloc_blk(c.dt, g, base_in);
      PointArgs z;
      z.y = full_in.p; z.y_dt = c.dt;
      z.ys1 = full_in.s1; z.ys2 = full_in.s2; z.ysi = full_in.si;
      z.n2 = g.n2; z.inner = g.inner; z.nb = g.count(); z.n = base_in;
      c.point(z);
      IndexArgs s;
      s.x = x.p; s.xs1 = x.s1; s.xs2 = x.s2; s.xsi = x.si;
      s.y = full_in.p; s.ys1 = full_in.s1; s.ys2 = full_in.s2; s.ysi = full_in.si;
      s.n2 = g.n2; s.inner = g.inner; s.nb = g.count(); s.n = in_idx->len;
      s.idx = (const int64_t*)in_idx->p;
      s.atomic = !in_unique;
      c.scatter(s);
    }
    if (!out_idx) {
      base->apply(c, adj, full_in, y, g, acc);
    } else {
      Blk full_out = c.alloc_blk(c.dt, g, base_out);
      base->apply(c, adj, full_in, full_out, g, false);
      Blk dst = y;
      if (acc) dst = c.alloc_blk(c.dt, g, out_idx->len);
      IndexArgs s;
      s.x = full_out.p; s.xs1 = full_out.s1; s.xs2 = full_out.s2; s.xsi = full_out.si;
      s.y = dst.p; s.ys1 = dst.s1; s.ys2 = dst.s2; s.ysi = dst.si;
      s.n2 = g.n2; s.inner = g.inner; s.nb = g.count(); s.n = out_idx->len;
      s.idx = (const int64_t*)out_idx->p;
      c.gather(s);
      if (acc) point_copy(c, dst, y, g, out_idx->len, true);
    }
    c.release(m0);
  }
};

// BlockDiag(*blocks) (composites.py:196-236).
struct BlockDiagNode : Node {
  std::vector<Node*> b;
  std::string describe() const override { return "BlockDiag(" + std::to_string(b.size()) + " blocks)"; }
  bool accepts_real() const override {
    for (Node* n : b)
      if (!n->accepts_real()) return false;
    return true;
  }
  void apply(Ctx& c, bool adj, const Blk& x, const Blk& y, const Geo& g, bool acc) override {
    int64_t ri = 0, ro = 0;
    for (Node* n : b) {
      const int64_t nin = adj ? n->rows : n->cols, nout = adj ? n->cols : n->rows;
      n->apply(c, adj, offset_rows(x, ri), offset_rows(y, ro), g, acc);
      ri += nin;
      ro += nout;
    }
  }
};

// Blocks(grid) (composites.py:124-193).
struct BlocksNode : Node {
  int gr = 0, gc = 0;
  std::vector<Node*> cells;  // row-major grid
  std::string describe() const override {
    return "Blocks(" + std::to_string(gr) + "x" + std::to_string(gc) + ")";
  }
  bool accepts_real() const override {
    for (Node* n : cells)
      if (!n->accepts_real()) return false;
    return true;
  }
  void apply(Ctx& c, bool adj, const Blk& x, const Blk& y, const Geo& g, bool acc) override {
    // fwd: y_i = sum_j A_ij x_j ; adj: y_j = sum_i A_ij^H x_i
    const int no = adj ? gc : gr, ni = adj ? gr : gc;
    int64_t ro = 0;
    for (int o = 0; o < no; ++o) {
      int64_t ri = 0, hout = 0;
      for (int i = 0; i < ni; ++i) {
        Node* n = adj ? cells[size_t(i) * gc + o] : cells[size_t(o) * gc + i];
        const int64_t nin = adj ? n->rows : n->cols;
        hout = adj ? n->cols : n->rows;
        n->apply(c, adj, offset_rows(x, ri), offset_rows(y, ro), g, acc || i > 0);
        ri += nin;
      }
      ro += hout;
    }
  }
};

// alpha * base (dparam = alpha): the scaled inverse DFT of kernels.dft and the
// building block of polynomial operators.
struct ScaledNode : Node {
  Node* base = nullptr;
  double re = 1.0, im = 0.0;
  std::string describe() const override { return "Scaled(" + base->describe() + ")"; }
  bool accepts_real() const override { return base->accepts_real(); }
  void apply(Ctx& c, bool adj, const Blk& x, const Blk& y, const Geo& g, bool acc) override {
    const double sim = adj ? -im : im;
    const int64_t nout = adj ? cols : rows;
    if (!acc) {
      base->apply(c, adj, x, y, g, false);
      point_copy(c, y, y, g, nout, false, nullptr, false, false, re, sim);
      return;
    }
    const size_t m0 = c.mark();
    Blk t = c.alloc_blk(c.dt, g, nout);
    base->apply(c, adj, x, t, g, false);
    point_copy(c, t, y, g, nout, true, nullptr, false, false, re, sim);
    c.release(m0);
  }
};

// Sparse(rows, cols, triplets) (leaves.py:100-159): CSR times block forward,
// the conjugate-transposed CSR (built once at plan time, like the reference's
// _csr_adj) backward.
struct SparseNode : Node {
  DevBuf *ptr = nullptr, *col = nullptr, *val = nullptr;
  DevBuf *aptr = nullptr, *acol = nullptr, *aval = nullptr;
  int64_t nnz = 0;
  std::string describe() const override {
    return "Sparse(" + std::to_string(rows) + "x" + std::to_string(cols) + ", nnz " + std::to_string(nnz) + ")";
  }
  void apply(Ctx& c, bool adj, const Blk& x0, const Blk& y, const Geo& g, bool acc) override {
    const size_t m0 = c.mark();
    Blk x = promote(c, x0, g, adj ? rows : cols);
    CsrArgs a;
    a.ptr = (const int64_t*)(adj ? aptr : ptr)->p;
    a.col = (const int64_t*)(adj ? acol : col)->p;
    a.val = (adj ? aval : val)->p;
    a.rows = adj ? cols : rows;
    a.x = x.p; a.xs1 = x.s1; a.xs2 = x.s2; a.xsi = x.si;
    a.y = y.p; a.ys1 = y.s1; a.ys2 = y.s2; a.ysi = y.si;
    a.n2 = g.n2; a.nb_outer = g.n1 * g.n2; a.inner = g.inner;
    a.accumulate = acc;
    c.csr(a);
    c.release(m0);
  }
};

// Polynomial(base, coeffs) = sum_k coeffs[k] base^k (composites.py:323-365),
// Horner's rule on the block: out = c_d x; out = base(out) + c_k x for k < d.
// The backward conjugates the coefficients and applies base^H.
struct PolynomialNode : Node {
  Node* base = nullptr;
  std::vector<std::complex<double>> coef;
  std::string describe() const override {
    return "Polynomial(" + base->describe() + ", degree " + std::to_string(coef.size() - 1) + ")";
  }
  void apply(Ctx& c, bool adj, const Blk& x0, const Blk& y, const Geo& g, bool acc) override {
    const size_t m0 = c.mark();
    const int64_t n = rows;
    Blk x = promote(c, x0, g, n);
    const int d = int(coef.size()) - 1;
    auto cf = [&](int k, double& re, double& im) {
      re = coef[size_t(k)].real();
      im = adj ? -coef[size_t(k)].imag() : coef[size_t(k)].imag();
    };
    double re, im;
    cf(d, re, im);
    if (d == 0) {
      point_copy(c, x, y, g, n, acc, nullptr, false, false, re, im);
      c.release(m0);
      return;
    }
    Blk cur = c.alloc_blk(c.dt, g, n);
    Blk tmp = c.alloc_blk(c.dt, g, n);
    point_copy(c, x, cur, g, n, false, nullptr, false, false, re, im);
    for (int k = d - 1; k >= 0; --k) {
      // the last step lands in y directly unless y accumulates
      Blk dst = (k == 0 && !acc) ? y : tmp;
      base->apply(c, adj, cur, dst, g, false);
      cf(k, re, im);
      if (re != 0.0 || im != 0.0) point_copy(c, x, dst, g, n, true, nullptr, false, false, re, im);
      std::swap(cur, tmp);
    }
    if (acc) point_copy(c, cur, y, g, n, true);
    c.release(m0);
  }
};

// ====================================================== plan building =====
// Device FFT of a complex128 vector (plan-build helper: spectra, Bluestein).
void device_fft_c128(Plan& p, int64_t n, const void* in_dev, void* out_dev) {
  SMAT_CHECK(is_pow2(n), SMAT_NOT_POW2, "device_fft_c128 needs a power of two");
  Ctx c;
  c.device = p.device;
  c.dt = SMAT_C128;
  c.measure = true;
  Blk x, y;
  x.p = (void*)in_dev; x.dt = SMAT_C128; x.si = 1; x.s1 = x.s2 = n;
  y.p = out_dev; y.dt = SMAT_C128; y.si = 1; y.s1 = y.s2 = n;
  Geo g;
  XformIO io;
  io.x = x; io.x_rows = n; io.y = y; io.y_rows = n;
  run_xform(c, n, g, io);
  const size_t need = c.peak;
  void* ws = nullptr;
  if (need) SMAT_CUDA(cudaMalloc(&ws, need));
  c.measure = false;
  c.top = c.peak = 0;
  c.ws = (char*)ws;
  c.ws_size = need;
  try {
    run_xform(c, n, g, io);
    SMAT_CUDA(cudaDeviceSynchronize());
  } catch (...) {
    if (ws) cudaFree(ws);
    throw;
  }
  if (ws) cudaFree(ws);
}

__global__ void chirp_kernel(double2* chirp, int64_t n) {
  for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < n; j += int64_t(gridDim.x) * blockDim.x) {
    // w_j = exp(-i pi (j^2 mod 2n) / n), exact integer reduction (kernels.py:86-87)
    const unsigned long long r = (unsigned long long)(j) * (unsigned long long)(j) % (unsigned long long)(2 * n);
    double s, c;
    sincospi(-double(r) / double(n), &s, &c);
    chirp[j] = make_double2(c, s);
  }
}
__global__ void bluestein_kernel_fill(const double2* chirp, double2* ker, int64_t n, int64_t M) {
  for (int64_t m = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; m < M; m += int64_t(gridDim.x) * blockDim.x) {
    double2 v = make_double2(0, 0);
    if (m < n) v = make_double2(chirp[m].x, -chirp[m].y);
    else if (m > M - n) v = make_double2(chirp[M - m].x, -chirp[M - m].y);
    ker[m] = v;
  }
}

struct Builder {
  Plan& p;
  const smat_node* nodes;
  int n_nodes;
  const int32_t* children;
  int n_children;
  int depth = 0;

  Node* child(const smat_node& nd, int k) {
    SMAT_CHECK(nd.first_child >= 0 && nd.first_child + k < n_children, SMAT_BAD_ARG, "bad child index");
    return build(children[nd.first_child + k]);
  }

  template <class T> T* add() {
    auto u = std::make_unique<T>();
    T* r = u.get();
    p.nodes.push_back(std::move(u));
    return r;
  }

  // elementwise product of two plan-precision complex vectors (either may be null)
  DevBuf* vec_product(DevBuf* a, DevBuf* b, int cdt) {
    if (!a && !b) return nullptr;
    if (!a || !b) return a ? a : b;
    DevBuf* o = new_buf(p, cdt, a->len);
    if (cdt == SMAT_C128)
      vec_mul_kernel<double2><<<1184, 256>>>((const double2*)a->p, (const double2*)b->p, (double2*)o->p, a->len);
    else
      vec_mul_kernel<float2><<<1184, 256>>>((const float2*)a->p, (const float2*)b->p, (float2*)o->p, a->len);
    SMAT_CUDA(cudaGetLastError());
    return o;
  }

  // Product factor list: fold Diag · Fourier · Diag (and Diag · Fourier,
  // Fourier · Diag) into one DiagFourierNode.
  void fuse_diag_fourier(std::vector<Node*>& f) {
    const int cdt = cplx_of(p.dt);
    if (dt_int(p.dt) || !dt_complex(p.dt)) return;
    for (size_t i = 0; i < f.size(); ++i) {
      auto* F = dynamic_cast<FourierNode*>(f[i]);
      if (!F) continue;
      DiagNode* dl = i > 0 ? dynamic_cast<DiagNode*>(f[i - 1]) : nullptr;
      DiagNode* dr = i + 1 < f.size() ? dynamic_cast<DiagNode*>(f[i + 1]) : nullptr;
      if (!dl && !dr) continue;
      auto* n = add<DiagFourierNode>();
      n->F = F;
      n->rows = F->rows;
      n->cols = F->cols;
      DevBuf* chirp = F->M ? F->chirp : nullptr;
      n->vr = vec_product(chirp, dr ? dr->d : nullptr, cdt);
      n->vl = vec_product(chirp, dl ? dl->d : nullptr, cdt);
      const int64_t Nt = F->M ? F->M : F->n;
      n->vr_fs = fourstep_vector(p, n->vr, F->n, Nt, cdt);
      n->vl_fs = fourstep_vector(p, n->vl, F->n, Nt, cdt);
      const size_t lo = dl ? i - 1 : i, hi = dr ? i + 1 : i;
      f.erase(f.begin() + lo, f.begin() + hi + 1);
      f.insert(f.begin() + lo, n);
      i = lo;
    }
  }

  // [DiagFourier (Bluestein, four-step), Sum(PaddedHadamard, LowRank)] ->
  // DFSumNode (the BASELINE C5 chain), when the Hadamard length factors over
  // the Bluestein transform's middle-pass length
  Node* blocked_chain(ProductNode* prod) {
    if (p.dt != SMAT_C128) return nullptr;
    auto* df = dynamic_cast<DiagFourierNode*>(prod->f[0]);
    auto* sum = dynamic_cast<SumNode*>(prod->f[1]);
    if (!df || !sum || !df->F->M || sum->t.size() != 2) return nullptr;
    PartialNode* hp = nullptr;
    LowRankNode* lr = nullptr;
    for (Node* t : sum->t) {
      if (auto* q = dynamic_cast<PartialNode*>(t); q && q->had_order >= 0) hp = q;
      if (auto* q = dynamic_cast<LowRankNode*>(t)) lr = q;
    }
    if (!hp || !lr || lr->r > 32) return nullptr;
    const int64_t M = df->F->M, n = df->F->n;
    if (!fourstep(M, true, SMAT_C128)) return nullptr;
    int64_t N1, N2;
    fourstep_split(M, N1, N2);
    const int64_t P = int64_t(1) << hp->had_order;
    if (N1 < 128 || N1 > kTileMax || P % N1 || P < n || hp->rows != n || hp->cols != n) return nullptr;
    const int64_t N2b = P / N1, NWa = N1 / 64;
    if (N2b < 2 || N2b > N2 || N2b > kTileMax || NWa < 2 || NWa > 64) return nullptr;
    auto* b = add<DFSumNode>();
    b->fallback = prod;
    b->df = df; b->hp = hp; b->lr = lr;
    b->N1 = N1; b->N2 = N2; b->N2b = N2b; b->P = P; b->M = M; b->NWa = NWa;
    build_utilde(lr, n, N1, N2b, NWa);
    p.fused = "blocked Bluestein/Hadamard/LowRank chain (N1=" + std::to_string(N1) + ", N2b=" + std::to_string(N2b) +
              ", Hadamard " + std::to_string(NWa) + " x 64 x " + std::to_string(N2b) + ")";
    return b;
  }

  // U~ = H_{N2b} U / N2b over k2 (U zero-padded to P rows; logical row
  // r = a + NWa b + N1 k2), stored in the blocked chain's A2 unit order:
  // unit row (k2 NWa + a) 64 + b
  DevBuf* build_utilde(LowRankNode* lr, int64_t n, int64_t N1, int64_t N2b, int64_t NWa) {
    const int64_t P = N1 * N2b, r = lr->r;
    DevBuf* Upad = new_buf(p, SMAT_C128, P * r);
    SMAT_CUDA(cudaMemset(Upad->p, 0, Upad->bytes));
    SMAT_CUDA(cudaMemcpy(Upad->p, lr->U->p, size_t(n * r) * 16, cudaMemcpyDeviceToDevice));
    DevBuf* Uw = new_buf(p, SMAT_C128, P * r);
    {
      // N2b-point FWHT over k2 for every (n1, q): rows k2 N1 r elements apart
      Ctx c;
      c.device = p.device;
      c.dt = SMAT_C128;
      WhtArgs a;
      a.x = Upad->p; a.y = Uw->p;
      a.xs1 = a.ys1 = P * r; a.xs2 = a.ys2 = r; a.xsi = a.ysi = N1 * r;
      a.n2 = N1; a.inner = r; a.nb = N1 * r;
      c.wht(SMAT_C128, int(N2b), a);
    }
    DevBuf* Ut = new_buf(p, SMAT_C128, P * r);
    utilde_perm_kernel<<<1184, 256>>>((const double2*)Uw->p, (double2*)Ut->p, P, r, N1, NWa, 1.0 / double(N2b));
    SMAT_CUDA(cudaGetLastError());
    lr->Utc = new_buf(p, SMAT_C128, P * wlr_pitch(false));
    lr->Ute = new_buf(p, SMAT_C128, P * wlr_pitch(true));
    wlr_pad_factor(Ut->p, lr->Utc->p, P, r, false, nullptr);
    wlr_pad_factor(Ut->p, lr->Ute->p, P, r, true, nullptr);
    SMAT_CUDA(cudaDeviceSynchronize());
    drop_buf(Upad);
    drop_buf(Uw);
    drop_buf(Ut);
    return nullptr;
  }
  void drop_buf(DevBuf* b) {
    for (auto it = p.bufs.begin(); it != p.bufs.end(); ++it)
      if (it->get() == b) {
        p.bufs.erase(it);
        return;
      }
  }

  std::vector<Node*> memo;  // shared sub-operators are compiled once

  Node* build(int idx) {
    SMAT_CHECK(idx >= 0 && idx < n_nodes, SMAT_BAD_ARG, "bad node index");
    if (memo.empty()) memo.assign(size_t(n_nodes), nullptr);
    if (memo[size_t(idx)]) return memo[size_t(idx)];
    SMAT_CHECK(++depth < 256, SMAT_BAD_ARG, "operator tree too deep");
    const smat_node& nd = nodes[idx];
    Node* out = nullptr;
    const int cdt = dt_int(p.dt) ? -1 : cplx_of(p.dt);
    switch (nd.kind) {
      case SMAT_IDENTITY: out = add<IdentityNode>(); break;
      case SMAT_ZERO: out = add<ZeroNode>(); break;
      case SMAT_DIAGONAL: {
        auto* n = add<DiagNode>();
        n->d = upload_param(p, nd.param[0], p.dt);
        out = n;
        break;
      }
      case SMAT_DENSE: {
        auto* n = add<DenseNode>();
        SMAT_CHECK(nd.param[0].len == nd.rows * nd.cols, SMAT_BAD_SHAPE, "dense entries size");
        n->A = upload_param(p, nd.param[0], p.dt);
        if (!dt_int(p.dt) && blas_available()) blas_warm(p.device);
        out = n;
        break;
      }
      case SMAT_LOWRANK: {
        auto* n = add<LowRankNode>();
        n->r = nd.iparam[0];
        SMAT_CHECK(n->r >= 1 && nd.param[0].len == nd.rows * n->r && nd.param[1].len == nd.cols * n->r,
                   SMAT_BAD_SHAPE, "lowrank factor sizes");
        n->U = upload_param(p, nd.param[0], p.dt);
        n->V = upload_param(p, nd.param[1], p.dt);
        if (nd.param[2].len) n->s = upload_param(p, nd.param[2], p.dt);
        if (p.dt == SMAT_C128 && n->r <= 32) {
          auto padded = [&](DevBuf* f, int64_t nrows, bool e) {
            DevBuf* b = new_buf(p, SMAT_C128, nrows * wlr_pitch(e));
            wlr_pad_factor(f->p, b->p, nrows, n->r, e, nullptr);
            return b;
          };
          n->Uc = padded(n->U, nd.rows, false);
          n->Ue = padded(n->U, nd.rows, true);
          n->Vc = padded(n->V, nd.cols, false);
          n->Ve = padded(n->V, nd.cols, true);
        }
        out = n;
        break;
      }
      case SMAT_HADAMARD: {
        auto* n = add<HadamardNode>();
        n->order = int(nd.iparam[0]);
        SMAT_CHECK(n->order >= 0 && n->order <= 30, SMAT_BAD_ARG, "hadamard order");
        out = n;
        break;
      }
      case SMAT_FOURIER: {
        SMAT_CHECK(cdt >= 0, SMAT_BAD_DTYPE, "Fourier needs a complex plan");
        auto* n = add<FourierNode>();
        n->n = nd.rows;
        if (!is_pow2(n->n)) {
          n->M = next_pow2(2 * n->n - 1);
          DevBuf* ch = new_buf(p, SMAT_C128, n->n);
          chirp_kernel<<<1184, 256>>>((double2*)ch->p, n->n);
          SMAT_CUDA(cudaGetLastError());
          DevBuf* ker = new_buf(p, SMAT_C128, n->M);
          bluestein_kernel_fill<<<1184, 256>>>((const double2*)ch->p, (double2*)ker->p, n->n, n->M);
          SMAT_CUDA(cudaGetLastError());
          DevBuf* ks = new_buf(p, SMAT_C128, n->M);
          device_fft_c128(p, n->M, ker->p, ks->p);
          n->chirp = narrow_c128(p, ch, cdt);
          n->kspec = spectrum_for_plan(p, ks, cdt);
          n->chirp_fs = fourstep_vector(p, n->chirp, n->n, n->M, cdt);
        }
        out = n;
        break;
      }
      case SMAT_CIRCULANT: {
        SMAT_CHECK(cdt >= 0, SMAT_BAD_DTYPE, "Circulant needs a floating plan");
        const int64_t n = nd.rows;
        SMAT_CHECK(nd.param[0].len == n, SMAT_BAD_SHAPE, "circulant column length");
        if (is_pow2(n)) {
          auto* c = add<CirculantNode>();
          c->n = n;
          DevBuf* cc = upload_param(p, nd.param[0], SMAT_C128);
          DevBuf* sp = new_buf(p, SMAT_C128, n);
          device_fft_c128(p, n, cc->p, sp->p);
          c->spec = spectrum_for_plan(p, sp, cdt);
          out = c;
        } else {
          // C[i,j] = c[(i-j) mod n] == Toeplitz(c, [c[n-1], ..., c[1]]):
          // linear-convolution embedding of length next_pow2(2n-1).
          auto h = convert_host(nd.param[0], SMAT_C128);
          const std::complex<double>* cv = (const std::complex<double>*)h.data();
          auto* t = add<ToeplitzNode>();
          t->L = next_pow2(2 * n - 1);
          std::vector<std::complex<double>> e(size_t(t->L), 0.0);
          for (int64_t i = 0; i < n; ++i) e[size_t(i)] = cv[i];
          for (int64_t j = 1; j < n; ++j) e[size_t(t->L - j)] = cv[n - j];
          DevBuf* eb = new_buf(p, SMAT_C128, t->L);
          SMAT_CUDA(cudaMemcpy(eb->p, e.data(), e.size() * 16, cudaMemcpyHostToDevice));
          DevBuf* sp = new_buf(p, SMAT_C128, t->L);
          device_fft_c128(p, t->L, eb->p, sp->p);
          t->spec = spectrum_for_plan(p, sp, cdt);
          out = t;
        }
        break;
      }
      case SMAT_TOEPLITZ: {
        SMAT_CHECK(cdt >= 0, SMAT_BAD_DTYPE, "Toeplitz needs a floating plan");
        auto* t = add<ToeplitzNode>();
        const int64_t n = nd.rows, m = nd.cols;
        SMAT_CHECK(nd.param[0].len == n && nd.param[1].len == m - 1, SMAT_BAD_SHAPE, "toeplitz sizes");
        t->L = next_pow2(n + m - 1);
        auto hc = convert_host(nd.param[0], SMAT_C128);
        std::vector<std::complex<double>> e(size_t(t->L), 0.0);
        const std::complex<double>* cv = (const std::complex<double>*)hc.data();
        for (int64_t i = 0; i < n; ++i) e[size_t(i)] = cv[i];
        if (m > 1) {
          auto hr = convert_host(nd.param[1], SMAT_C128);
          const std::complex<double>* rv = (const std::complex<double>*)hr.data();
          // embed[L-(m-1):] = row_rest[::-1]  (leaves.py:258-259)
          for (int64_t k = 0; k < m - 1; ++k) e[size_t(t->L - (m - 1) + k)] = rv[m - 2 - k];
        }
        DevBuf* eb = new_buf(p, SMAT_C128, t->L);
        SMAT_CUDA(cudaMemcpy(eb->p, e.data(), e.size() * 16, cudaMemcpyHostToDevice));
        DevBuf* sp = new_buf(p, SMAT_C128, t->L);
        device_fft_c128(p, t->L, eb->p, sp->p);
        t->spec = spectrum_for_plan(p, sp, cdt);
        // pruned halves only when each half is a single tile pass: once the
        // halves go four-step too, one four-step convolution of length L moves
        // fewer bytes (x read and y written once) in half the launches
        const bool prune = !fourstep(t->L / 2, true, cdt);
        if (prune && t->L > kTileMax && t->L / 2 <= kTileMax && std::max(n, m) <= t->L / 2) {
          const int64_t h = t->L / 2;
          DevBuf* se = new_buf(p, SMAT_C128, h);
          DevBuf* so = new_buf(p, SMAT_C128, h);
          DevBuf* tw = new_buf(p, SMAT_C128, h);
          split_even_odd_kernel<<<256, 256>>>((const double2*)sp->p, (double2*)se->p, (double2*)so->p,
                                              (double2*)tw->p, t->L);
          SMAT_CUDA(cudaGetLastError());
          t->spec_e = spectrum_for_plan(p, se, cdt);
          t->spec_o = spectrum_for_plan(p, so, cdt);
          t->twid = narrow_c128(p, tw, cdt);
        }
        out = t;
        break;
      }
      case SMAT_ADJOINT: {
        auto* a = add<AdjointNode>();
        a->base = child(nd, 0);
        out = a;
        break;
      }
      case SMAT_PRODUCT: {
        auto* a = add<ProductNode>();
        for (int k = 0; k < nd.n_children; ++k) a->f.push_back(child(nd, k));
        SMAT_CHECK(!a->f.empty(), SMAT_BAD_ARG, "empty product");
        for (size_t k = 0; k + 1 < a->f.size(); ++k)
          SMAT_CHECK(a->f[k]->cols == a->f[k + 1]->rows, SMAT_BAD_SHAPE, "product chain mismatch");
        fuse_diag_fourier(a->f);
        out = a->f.size() == 1 ? a->f[0] : a;
        if (a->f.size() == 2) {
          if (Node* bc = blocked_chain(a)) out = bc;
        }
        break;
      }
      case SMAT_SUM: {
        auto* a = add<SumNode>();
        for (int k = 0; k < nd.n_children; ++k) a->t.push_back(child(nd, k));
        SMAT_CHECK(!a->t.empty(), SMAT_BAD_ARG, "empty sum");
        out = a;
        break;
      }
      case SMAT_KRON: {
        auto* a = add<KronNode>();
        for (int k = 0; k < nd.n_children; ++k) a->f.push_back(child(nd, k));
        SMAT_CHECK(a->f.size() >= 2, SMAT_BAD_ARG, "kron needs two factors");
        out = a;
        break;
      }
      case SMAT_PARTIAL: {
        auto* a = add<PartialNode>();
        a->base = child(nd, 0);
        if (nd.iparam[0]) {
          a->ridx = upload_param(p, nd.param[0], SMAT_I64);
          a->r_unique = nd.iparam[2] != 0;
        }
        if (nd.iparam[1]) {
          a->cidx = upload_param(p, nd.param[1], SMAT_I64);
          a->c_unique = nd.iparam[3] != 0;
        }
        {
          auto is_prefix = [](const smat_param& prm) {
            if (prm.dtype != SMAT_I64) return false;
            const int64_t* v = (const int64_t*)prm.data;
            for (int64_t i = 0; i < prm.len; ++i)
              if (v[i] != i) return false;
            return true;
          };
          const smat_node& bn = nodes[children[nd.first_child]];
          if (bn.kind == SMAT_HADAMARD && (!nd.iparam[0] || is_prefix(nd.param[0])) &&
              (!nd.iparam[1] || is_prefix(nd.param[1])))
            a->had_order = int(bn.iparam[0]);
          else if (((bn.kind == SMAT_HADAMARD && bn.iparam[0] >= 1) ||
                    (bn.kind == SMAT_FOURIER && is_pow2(bn.rows) && bn.rows >= 2 && bn.rows <= kTileMax &&
                     dt_complex(p.dt))) &&
                   a->r_unique && a->c_unique && (nd.iparam[0] || nd.iparam[1]) && !dt_int(p.dt)) {
            // int32 row maps of the selections (reference composites.py:281-310)
            const int64_t full = bn.kind == SMAT_HADAMARD ? int64_t(1) << bn.iparam[0] : bn.rows;
            auto make_map = [&](const smat_param& prm) {
              std::vector<int32_t> m(size_t(full), -1);
              const int64_t* v = (const int64_t*)prm.data;
              for (int64_t k = 0; k < prm.len; ++k) m[size_t(v[k])] = int32_t(k);
              smat_param mp{m.data(), full, SMAT_I32, 0};
              return upload_param(p, mp, SMAT_I32);
            };
            if (nd.iparam[0] && nd.param[0].dtype == SMAT_I64) a->rmap = make_map(nd.param[0]);
            if (nd.iparam[1] && nd.param[1].dtype == SMAT_I64) a->cmap = make_map(nd.param[1]);
            if ((!nd.iparam[0] || a->rmap) && (!nd.iparam[1] || a->cmap)) {
              if (bn.kind == SMAT_HADAMARD) a->map_order = int(bn.iparam[0]);
              else a->map_fourier = bn.rows;
            }
          }
        }
        out = a;
        break;
      }
      case SMAT_BLOCKDIAG: {
        auto* a = add<BlockDiagNode>();
        for (int k = 0; k < nd.n_children; ++k) a->b.push_back(child(nd, k));
        out = a;
        break;
      }
      case SMAT_BLOCKS: {
        auto* a = add<BlocksNode>();
        a->gr = int(nd.iparam[0]);
        a->gc = int(nd.iparam[1]);
        SMAT_CHECK(a->gr * a->gc == nd.n_children && a->gr > 0, SMAT_BAD_ARG, "blocks grid");
        for (int k = 0; k < nd.n_children; ++k) a->cells.push_back(child(nd, k));
        out = a;
        break;
      }
      case SMAT_SCALED: {
        auto* a = add<ScaledNode>();
        a->base = child(nd, 0);
        a->re = nd.dparam[0];
        a->im = nd.dparam[1];
        SMAT_CHECK(dt_complex(p.dt) || a->im == 0.0, SMAT_BAD_DTYPE, "complex scale in a real plan");
        out = a;
        break;
      }
      case SMAT_SPARSE: {
        SMAT_CHECK(dt_int(p.dt) == false, SMAT_BAD_DTYPE, "Sparse needs a floating plan");
        auto* a = add<SparseNode>();
        const int64_t R = nd.rows, Cn = nd.cols;
        SMAT_CHECK(nd.param[0].dtype == SMAT_I64 && nd.param[0].len == R + 1 && nd.param[1].dtype == SMAT_I64,
                   SMAT_BAD_ARG, "sparse: row_ptr / col_idx must be int64 (rows+1, nnz)");
        const int64_t* rp = (const int64_t*)nd.param[0].data;
        const int64_t* ci = (const int64_t*)nd.param[1].data;
        const int64_t nnz = nd.param[1].len;
        SMAT_CHECK(nd.param[2].len == nnz && rp[0] == 0 && rp[R] == nnz, SMAT_BAD_ARG, "sparse: inconsistent CSR");
        for (int64_t i = 0; i < R; ++i) SMAT_CHECK(rp[i] <= rp[i + 1], SMAT_BAD_ARG, "sparse: row_ptr not monotone");
        for (int64_t k = 0; k < nnz; ++k) SMAT_CHECK(ci[k] >= 0 && ci[k] < Cn, SMAT_BAD_ARG, "sparse: column index");
        a->nnz = nnz;
        a->ptr = upload_param(p, nd.param[0], SMAT_I64);
        a->col = upload_param(p, nd.param[1], SMAT_I64);
        a->val = upload_param(p, nd.param[2], p.dt);
        // conjugate transpose: counting sort by column, stable in the row order
        const bool cv = dt_complex(nd.param[2].dtype);
        auto hv = convert_host(nd.param[2], cv ? SMAT_C128 : SMAT_F64);
        std::vector<int64_t> tp(size_t(Cn) + 1, 0);
        std::vector<int64_t> tc(static_cast<size_t>(nnz));
        std::vector<double> tv(size_t(nnz) * (cv ? 2 : 1));
        for (int64_t k = 0; k < nnz; ++k) ++tp[size_t(ci[k]) + 1];
        for (int64_t j = 0; j < Cn; ++j) tp[size_t(j) + 1] += tp[size_t(j)];
        std::vector<int64_t> fill(tp.begin(), tp.end() - 1);
        const double* hvd = (const double*)hv.data();
        for (int64_t i = 0; i < R; ++i)
          for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
            const int64_t q = fill[size_t(ci[k])]++;
            tc[size_t(q)] = i;
            if (cv) {
              tv[size_t(2 * q)] = hvd[2 * k];
              tv[size_t(2 * q + 1)] = -hvd[2 * k + 1];
            } else {
              tv[size_t(q)] = hvd[k];
            }
          }
        smat_param pp{tp.data(), Cn + 1, SMAT_I64, 0}, pc{tc.data(), nnz, SMAT_I64, 0},
            pv{tv.data(), nnz, cv ? SMAT_C128 : SMAT_F64, 0};
        a->aptr = upload_param(p, pp, SMAT_I64);
        a->acol = upload_param(p, pc, SMAT_I64);
        a->aval = upload_param(p, pv, p.dt);
        out = a;
        break;
      }
      case SMAT_POLYNOMIAL: {
        auto* a = add<PolynomialNode>();
        a->base = child(nd, 0);
        SMAT_CHECK(a->base->rows == a->base->cols && a->base->rows == nd.rows, SMAT_BAD_SHAPE,
                   "polynomial base must be square");
        SMAT_CHECK(nd.param[0].len >= 1, SMAT_BAD_ARG, "polynomial needs coefficients");
        const bool cv = dt_complex(nd.param[0].dtype);
        SMAT_CHECK(!cv || dt_complex(p.dt), SMAT_BAD_DTYPE, "complex coefficients in a real plan");
        auto hc = convert_host(nd.param[0], SMAT_C128);
        const double* h = (const double*)hc.data();
        for (int64_t k = 0; k < nd.param[0].len; ++k) a->coef.emplace_back(h[2 * k], h[2 * k + 1]);
        out = a;
        break;
      }
      default:
        throw Error(SMAT_UNSUPPORTED, "operator kind " + std::to_string(nd.kind) + " has no device path");
    }
    out->rows = nd.rows;
    out->cols = nd.cols;
    --depth;
    memo[size_t(idx)] = out;
    return out;
  }
};

Plan* build_plan(const smat_node* nodes, int n_nodes, const int32_t* children, int n_children, int root,
                 int dt, int device) {
  SMAT_CHECK(dt >= SMAT_F32 && dt <= SMAT_I64, SMAT_BAD_DTYPE, "plan dtype");
  auto p = std::make_unique<Plan>();
  p->dt = dt;
  p->device = device;
  Builder b{*p, nodes, n_nodes, children, n_children};
  p->root = b.build(root);
  p->rows = p->root->rows;
  p->cols = p->root->cols;
  SMAT_CUDA(cudaDeviceSynchronize());
  return p.release();
}

static void run_root(const Plan& p, Ctx& c, bool adj, Blk xb, const Blk& yb, const Geo& g, int64_t nin) {
  if (xb.dt != p.dt && !p.root->accepts_real()) xb = promote(c, xb, g, nin);
  p.root->apply(c, adj, xb, yb, g, false);
}

// Row-major view of a (rows, ncols) block with leading dimension ld.
static Blk row_view(const void* ptr, int dt, int64_t ld, int64_t rows) {
  Blk b;
  b.p = const_cast<void*>(ptr);
  b.dt = dt;
  b.si = ld;
  b.s2 = b.s1 = rows * ld;
  return b;
}

// Copy between a user block (row-major with leading dimension ld, or
// column-major) and a dense row-major block: one pointwise launch.
static void stage_copy(Ctx& c, int dt, const void* src, void* dst, int64_t rows, int64_t ncols, int64_t ld,
                       int layout, bool to_dense) {
  PointArgs pa;
  pa.x = src; pa.x_dt = dt; pa.y = dst; pa.y_dt = dt;
  int64_t us2, usi, uinner_stride;
  if (layout == SMAT_COL_MAJOR) {
    // element (i, col) at col*ld + i: batches o2 = col (stride ld), rows stride 1
    pa.n2 = ncols; pa.inner = 1; pa.nb = ncols; pa.n = rows;
    us2 = ld; usi = 1; uinner_stride = 0;
    const int64_t ds2 = 1, dsi = ncols;
    if (to_dense) { pa.xs2 = us2; pa.xsi = usi; pa.ys2 = ds2; pa.ysi = dsi; }
    else { pa.xs2 = ds2; pa.xsi = dsi; pa.ys2 = us2; pa.ysi = usi; }
  } else {
    pa.n2 = 1; pa.inner = ncols; pa.nb = ncols; pa.n = rows;
    us2 = rows * ld; usi = ld; uinner_stride = 1;
    if (to_dense) { pa.xs2 = us2; pa.xsi = usi; pa.ys2 = rows * ncols; pa.ysi = ncols; }
    else { pa.xs2 = rows * ncols; pa.xsi = ncols; pa.ys2 = us2; pa.ysi = usi; }
  }
  (void)uinner_stride;
  pa.xs1 = pa.xs2 * pa.n2;
  pa.ys1 = pa.ys2 * pa.n2;
  c.point_dt(dt, pa);
}

void run_plan(const Plan& p, Ctx& c, int dir, const void* x, int x_dt, int64_t ldx, void* y, int64_t ldy,
              int64_t ncols, int layout) {
  const bool adj = dir == 1;
  const int64_t nin = adj ? p.rows : p.cols, nout = adj ? p.cols : p.rows;
  const bool col = layout == SMAT_COL_MAJOR;
  SMAT_CHECK(layout == SMAT_ROW_MAJOR || col, SMAT_BAD_ARG, "layout must be SMAT_ROW_MAJOR or SMAT_COL_MAJOR");
  if (ldx <= 0) ldx = col ? nin : ncols;
  if (ldy <= 0) ldy = col ? nout : ncols;
  SMAT_CHECK(ldx >= (col ? nin : ncols) && ldy >= (col ? nout : ncols), SMAT_BAD_ARG,
             "leading dimension smaller than the block");
  Geo g;
  g.inner = ncols;
  if (!col) {
    const Blk xb = row_view(x, x_dt, ldx, nin), yb = row_view(y, p.dt, ldy, nout);
    if (ldx == ncols && ldy == ncols) {
      run_root(p, c, adj, xb, yb, g, nin);
      return;
    }
    // strided rows in place when every pass of the plan can address them
    // (a host-side dry run of the plan decides; no launch happens in it)
    Ctx d = c;
    d.measure = true;
    d.prof = nullptr;
    d.launches = 0;
    bool direct = true;
    try {
      run_root(p, d, adj, xb, yb, g, nin);
    } catch (const Error& e) {
      if (e.code != SMAT_UNSUPPORTED) throw;
      direct = false;
    }
    if (direct) {
      if (c.measure) {
        c.peak = std::max(c.peak, d.peak);
        c.launches += d.launches;
      } else {
        run_root(p, c, adj, xb, yb, g, nin);
      }
      return;
    }
  }
  // staged: dense row-major copies of the strided / column-major sides
  const size_t m0 = c.mark();
  const bool sx = col || ldx != ncols, sy = col || ldy != ncols;
  Blk xb = row_view(x, x_dt, ncols, nin), yb = row_view(y, p.dt, ncols, nout);
  if (sx) {
    xb = c.alloc_blk(x_dt, g, nin);
    stage_copy(c, x_dt, x, xb.p, nin, ncols, ldx, layout, true);
  }
  if (sy) yb = c.alloc_blk(p.dt, g, nout);
  run_root(p, c, adj, xb, yb, g, nin);
  if (sy) stage_copy(c, p.dt, yb.p, y, nout, ncols, ldy, layout, false);
  c.release(m0);
}

}  // namespace smat
