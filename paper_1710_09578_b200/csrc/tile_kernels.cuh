// tile_kernels.cuh — argument blocks and launchers of the tiled FFT / FWHT passes.
#pragma once

#include "common.cuh"

namespace smat {

// One tiled FFT pass: for every batch b of the view, a length-N forward DFT
// along i, with fused prologue/epilogue:
//   load : v = x[b, i]  (real promoted)  -> conj? -> * pre[g_in] -> conj if inv
//   core : forward DFT (N points)      [mid: * spec[g_mid], conj, DFT again]
//   store: conj if inv|mid -> * W_tw^(goff*k) (four-step) -> * post[g_out]
//          -> conj? -> * scale -> y[b, k]  (= or +=, real part or complex)
// with the "global" row indices g_in = goff + i*gin_stride,
// g_out = goff + k*gout_stride, g_mid = goff + k*mid_stride and
// goff = (b / g_div) % g_mod.  Rows with g_in >= n_valid_in load as zero
// (zero padding, leaves.py:269-270, kernels.py:116-118) and rows with
// g_out >= n_valid_out are not stored (truncation, leaves.py:273,
// kernels.py:125).
struct FftArgs {
  const void* x = nullptr;
  void* y = nullptr;
  int64_t xs1 = 0, xs2 = 0, xsi = 0;
  int64_t ys1 = 0, ys2 = 0, ysi = 0;
  int64_t n2 = 1, inner = 1, nb = 0;
  int64_t g_div = 1, g_mod = 1, gin_stride = 1, gout_stride = 1;
  int64_t n_valid_in = INT64_MAX, n_valid_out = INT64_MAX;
  const void* pre = nullptr;
  const void* post = nullptr;
  const void* mid = nullptr;
  int64_t mid_stride = 1;
  int64_t mid_gmul = 1;  // spectrum index = goff*mid_gmul + k*mid_stride
  const void* tw = nullptr;     // W_4096^t table of the working precision
  const void* tw_lo = nullptr;  // four-step twiddle W_Ntot^t, t < 2^tw_lo_bits
  const void* tw_hi = nullptr;  // W_Ntot^(t << tw_lo_bits)
  int64_t tw_mask = 0;          // Ntot - 1
  int32_t tw_lo_bits = 0;
  double scale = 1.0;
  int32_t x_real = 0, y_real = 0, conj_x = 0, conj_y = 0, inv = 0, mid_conj = 0;
  int32_t tw_on = 0, tw_inv = 0, accumulate = 0, pre_conj = 0, post_conj = 0;
  // four-step twiddle on the input (W^(goff*i), after pre) instead of the output
  int32_t tw_pre = 0;
  // pre / post vectors stored per tile ("four-step order"): when nonzero the
  // entry of input row i (output row k) is pre[goff*pre_gmul + i]
  // (post[goff*post_gmul + k]) instead of pre[g_in] (post[g_out]), so a tile's
  // entries are one contiguous slice
  int64_t pre_gmul = 0, post_gmul = 0;
  // optional per-tile four-step twiddle slices (twiddle_slices with E = N,
  // already conjugated for tw_inv): the TMA pass bulk-loads the tile's slice
  // instead of assembling it from tw_lo / tw_hi
  const void* tw_slices = nullptr;
  // two-level row strides (blocked four-step intermediates): when i_lo_bits
  // > 0, row i of x sits at (i % 2^b)*xsi + (i >> b)*xsi_hi, likewise for y
  int32_t i_lo_bits = 0;
  int64_t xsi_hi = 0, ysi_hi = 0;
  // fused row selection (Partial with unique indices; per-tile kernel only):
  // input row g loads x[in_map[g] * in_rs] (zero where < 0), output row g
  // stores to y[out_map[g] * out_rs] (skipped where < 0), both offset by the
  // batch's view origin
  const int32_t* in_map = nullptr;
  const int32_t* out_map = nullptr;
  int64_t in_rs = 0, out_rs = 0;
  // Walsh-Hadamard transform over the first N/2 rows of every tile column
  // fused into the pass (TMA kernel only; the C5 chain's k2 stages of the
  // padded Hadamard): 1 = on the loaded input, before the masks / pre vector
  // and the FFT; 2 = on the output, after the post vector, before the store
  int32_t wht_half = 0;
  // fused 8-point Walsh-Hadamard across a batch index (Kron(Hadamard, ...),
  // KronNode): the batch's inner index is virtual, v = (column group of 4,
  // hh, column % 4) with hh (element strides wg_xs / wg_ys) the Hadamard
  // index; a tile is 4 columns x 8 hh (TMA kernel only, 32-column tiles) and
  // the transform runs across lane bits 2-4 on the loaded input
  int32_t wht_grp = 0;
  int64_t wg_xs = 0, wg_ys = 0;
  // probe only: run every check of the launch (TMA view, shared memory) but
  // launch nothing; launch_fft_tile throws SMAT_UNSUPPORTED where a fused
  // Walsh-Hadamard pass would not run
  int32_t probe_only = 0;
};

// One tiled FWHT pass over the view (stride-1-first stage order).
struct WhtArgs {
  const void* x = nullptr;
  void* y = nullptr;
  int64_t xs1 = 0, xs2 = 0, xsi = 0;
  int64_t ys1 = 0, ys2 = 0, ysi = 0;
  int64_t n2 = 1, inner = 1, nb = 0;
  // global row g = ((b / g_div) % g_mod) * g_mul + i * g{in,out}_stride; rows
  // with g >= n_valid_in load as zero, rows with g >= n_valid_out are not
  // stored (the zero-pad / truncate of Partial(Hadamard, arange, arange))
  int64_t g_div = 1, g_mod = 1, g_mul = 1, gin_stride = 1, gout_stride = 1;
  int64_t n_valid_in = INT64_MAX, n_valid_out = INT64_MAX;
  int32_t accumulate = 0;
  // two-level rows (blocked layouts): row i at (i % 2^i_lo_bits) * {x,y}si +
  // (i >> i_lo_bits) * {x,y}si_hi when i_lo_bits > 0
  int32_t i_lo_bits = 0;
  int64_t xsi_hi = 0, ysi_hi = 0;
  // row selection fused into the pass (Partial with unique indices): global
  // input row g loads x[in_map[g] * in_rs + col] (zero where in_map[g] < 0),
  // output row g stores to y[out_map[g] * out_rs + col] (skipped where < 0);
  // col = (batch index % inner) % map_k.  Single-batch views only.
  const int32_t* in_map = nullptr;
  const int32_t* out_map = nullptr;
  int64_t in_rs = 0, out_rs = 0, map_k = 1;
};

constexpr int kTileMax = 4096;

// Launch one FFT tile pass of length N (power of two, 2..4096) in precision
// `cdt` (SMAT_C64 or SMAT_C128).
void launch_fft_tile(int cdt, int N, const FftArgs& a, cudaStream_t s);
bool tma_wht_ok(int N, int64_t inner);
// Launch one FWHT tile pass of length N (power of two, 2..4096) on dtype dt.
void launch_wht_tile(int dt, int N, const WhtArgs& a, cudaStream_t s);

// Device-resident W_4096^t table of the given precision on `device`.
const void* twiddle4096(int device, bool dbl);
// Device-resident four-step twiddle tables for length `ntot` (pow2).
struct TwPair {
  const void* lo;
  const void* hi;
  int lo_bits;
};
TwPair twiddle_pair(int device, int64_t ntot, bool dbl);
// Per-tile four-step twiddle slices W_nt^(+-g*e) at g*E + e (16 bytes per entry:
// double2, or the float quad layout), cached per device.
const void* twiddle_slices(int device, int64_t nt, int64_t E, bool inv, bool dbl);

}  // namespace smat
