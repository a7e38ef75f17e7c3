// wlr.cuh — fused Walsh-Hadamard + rank-r LowRank passes (complex128, FP64
// tensor cores).  See wlr.cu.
#pragma once

#include "common.cuh"

namespace smat {

// Physical row of unit row g (Hadamard group G = g / NW, position a = g % NW):
//   (G >> gsh) * g_hi + (G & (2^gsh - 1)) * g_lo + (a & (2^ash - 1)) * a_lo + (a >> ash) * a_hi
// (every split of the C5 chain is a power of two); rows are `ld` complex
// elements apart.  Used for the output rows (per-thread stores).
struct WlrRows {
  int32_t gsh = 40, ash = 40;
  int64_t g_hi = 0, g_lo = 0, a_lo = 0, a_hi = 0;
  int64_t ld = 0;
};

// Input rows of a unit (64 unit rows from g0) as ONE tensor-map box:
//   WLR_IN_ROWS  rows g0 .. g0+63 of a block with `rows` rows (rows beyond
//                are zero-filled: the padding of the padded Hadamard)
//   WLR_IN_T1A   the C5 chain's T1 read by NWa-row groups T = g / NWa: row
//                (T / 64) 64 NWa + T % 64 + 64 a
//   WLR_IN_T2B   the blocked T2 read by 64-row groups T' = g / 64 (n1 = a +
//                NWa b, k2): row ((n1 / 64) N2b + k2) 64 + n1 % 64
enum { WLR_IN_ROWS = 0, WLR_IN_T1A = 1, WLR_IN_T2B = 2 };
struct WlrIn {
  int kind = WLR_IN_ROWS;
  const void* p = nullptr;
  int64_t ld = 0;     // row stride (complex elements)
  int64_t rows = 0;   // WLR_IN_ROWS: rows of the block
  int64_t nwa = 1, n2b = 1, P = 0;  // chain geometry (T1A / T2B)
};

// Factor rows: unit row g at F + g * pitch (complex128), zero past rank r —
// laid out at plan time with a padded pitch (wlr_pitch) so that one bulk copy
// of 64 rows lands bank-conflict free for the tensor-core fragments.
int64_t wlr_pitch(bool expansion);

struct WlrArgs {
  WlrIn in;                 // input block (complex128)
  void* y = nullptr;        // output block (complex128)
  WlrRows yout;
  const void* F = nullptr;  // factor rows (wlr_pitch(exp) layout)
  int64_t r = 0;            // rank (<= 32)
  int64_t nrows = 0;        // unit rows covered (g < nrows)
  int64_t n_out = 0;        // output rows g >= n_out are not stored
  int64_t n_f = 0;          // factor rows g >= n_f are zero
  int64_t K = 0;            // columns
  // contraction: per-CTA partial products W_part[cta][q][c] (workspace)
  void* partial = nullptr;
  // expansion: W' as three real tables [32][K]: Re, Im, Re + Im
  const double* w3 = nullptr;
};

// Launch modes (smat_node LowRank / the C5 blocked chain, plan.cu):
//   NW  Hadamard length applied over the unit-row groups (1: none)
//   CON contract the INPUT rows with F^H into the partials
//   EXP add F * W' into the (transformed) output rows
//   IN  read the input block (false: output = F W' only)
//   OUT write the output block
struct WlrMode {
  int nw = 1;
  bool con = false, exp = false, in = true, out = true;
};

// (rows, r) complex128 factor -> the padded wlr layout (dst has rows * wlr_pitch(exp) entries)
void wlr_pad_factor(const void* src, void* dst, int64_t rows, int64_t r, bool expansion, cudaStream_t s);

// grid (CTAs) of a launch over K columns, and the partial-product workspace bytes
int wlr_grid(int device, int64_t K);
size_t wlr_partial_bytes(int device, int64_t K);
// returns the number of kernel launches (1)
int launch_wlr(const WlrMode& m, const WlrArgs& a, int device, cudaStream_t s, bool dry);
// W'[q][c] = scale_q * sum over the CTAs of column chunk c/64 of W_part; scale_q =
// s_q, conj(s_q) (s_conj) or 1 (s null); writes the three real tables w3
int launch_wlr_finalize(const void* partial, int grid, int64_t r, int64_t K, const void* s, bool s_conj, double* w3,
                        cudaStream_t st, bool dry);

}  // namespace smat
