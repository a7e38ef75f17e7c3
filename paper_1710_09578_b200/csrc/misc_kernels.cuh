// misc_kernels.cuh — pointwise, gather/scatter and small-GEMM passes used by the
// generic (unfused) plan interpreter.  Fused plans fold these into the
// prologue/epilogue of the adjacent FFT/FWHT pass instead.
#pragma once

#include "common.cuh"

namespace smat {

// y[o,i,c] (= or +=) scale * dvec[i]^(conj?) * conj?(x[o,i,c])
//   x == nullptr  -> zero fill (or no-op when accumulating)
//   dvec == nullptr -> no diagonal
// x_dt / y_dt may be the real dtype of a complex plan (promote on load / take
// the real part on store).
struct PointArgs {
  const void* x = nullptr;
  void* y = nullptr;
  int x_dt = 0, y_dt = 0;
  int64_t xs1 = 0, xs2 = 0, xsi = 0;
  int64_t ys1 = 0, ys2 = 0, ysi = 0;
  int64_t n2 = 1, inner = 1, nb = 0, n = 0;  // batches and rows
  const void* d = nullptr;                    // diagonal in the plan dtype
  int32_t d_conj = 0, x_conj = 0, accumulate = 0;
  double scale_re = 1.0, scale_im = 0.0;
};
void launch_point(int plan_dt, const PointArgs& a, cudaStream_t s);

// Row gather y[o, r, c] = x[o, idx[r], c] (r < n_out) and scatter
// y[o, idx[r], c] += x[o, r, c] (Partial, composites.py:281-310).
struct IndexArgs {
  const void* x = nullptr;
  void* y = nullptr;
  int64_t xs1 = 0, xs2 = 0, xsi = 0;
  int64_t ys1 = 0, ys2 = 0, ysi = 0;
  int64_t n2 = 1, inner = 1, nb = 0, n = 0;  // n = number of index entries
  const int64_t* idx = nullptr;
  int32_t atomic = 0;
};
void launch_gather(int dt, const IndexArgs& a, cudaStream_t s);
void launch_scatter_add(int dt, const IndexArgs& a, cudaStream_t s);

// CSR sparse times block (Sparse, leaves.py:100-159):
//   y[o, i, c] (= | +=) sum_{k in [ptr[i], ptr[i+1])} val[k] * x[o, col[k], c]
// one warp per (row, batch) pair, lanes over the contiguous columns.
struct CsrArgs {
  const int64_t* ptr = nullptr;
  const int64_t* col = nullptr;
  const void* val = nullptr;  // plan dtype
  int64_t rows = 0;
  const void* x = nullptr;
  void* y = nullptr;
  int64_t xs1 = 0, xs2 = 0, xsi = 0;
  int64_t ys1 = 0, ys2 = 0, ysi = 0;
  int64_t n2 = 1, nb_outer = 1, inner = 1;  // nb_outer = n1 * n2 batches of `inner` columns
  int32_t accumulate = 0;
};
void launch_csr(int dt, const CsrArgs& a, cudaStream_t s);

// Batched GEMM  Y[o] (=|+=) alpha * op(A) * X[o]
//   A: (m x k) row-major with leading dimension lda when !adj,
//      else op(A) = A^H where A is stored (k x m) row-major.
//   X[o]: k rows x inner cols (row stride xsi), Y[o]: m rows x inner.
struct GemmArgs {
  const void* A = nullptr;
  int64_t lda = 0;
  int32_t adj = 0;
  int64_t m = 0, k = 0;
  const void* x = nullptr;
  void* y = nullptr;
  int64_t xs1 = 0, xs2 = 0, xsi = 0;
  int64_t ys1 = 0, ys2 = 0, ysi = 0;
  int64_t n1 = 1, n2 = 1, inner = 1;
  int32_t accumulate = 0;
  // a row-scaling of the result (LowRank's diag(s)) applied before storing
  const void* rowscale = nullptr;
  int32_t rowscale_conj = 0;
};
// Returns the number of kernels launched (counted only when dry).
int launch_gemm(int dt, const GemmArgs& a, int device, cudaStream_t s, bool dry);

// Rank-r (r <= 32) factor kernels of LowRank = U diag(s) V^H on row-contiguous
// (rows, K) blocks (reference vehicle: Product(Dense(U), Dense(V^H)),
// leaves.py:40-46):
//   contract: W (r x K) = F^H X            (F = V forward, U backward; W zeroed first)
//   expand:   Y (=|+=) G diag(s) W          (G = U forward, V backward)
struct LowRankArgs {
  const void* F = nullptr;  // (rows x r) row-major
  const void* x = nullptr;  // (rows x K), row stride ldx
  void* w = nullptr;        // (r x K) contiguous
  void* y = nullptr;        // (rows x K), row stride ldy
  const void* s = nullptr;  // r or null
  int32_t s_conj = 0, accumulate = 0;
  int64_t rows = 0, r = 0, K = 0, ldx = 0, ldy = 0;
};
// cuBLAS GEMM (blas.cu), the Dense leaf's plain library GEMM: column-major
// C (m x n) = op(A) op(B) + beta C, op 0 = N / 2 = C; resolved at run time,
// blas_available() false when libcublas cannot be loaded
bool blas_available();
void blas_warm(int device);
void blas_gemm(int dt, int device, cudaStream_t s, int opa, int opb, int64_t m, int64_t n, int64_t k, const void* A,
               int64_t lda, const void* B, int64_t ldb, double beta_re, void* C, int64_t ldc);

// number of launches (dry) or launch
int launch_lowrank_contract(int dt, const LowRankArgs& a, int device, cudaStream_t s, bool dry);
int launch_lowrank_expand(int dt, const LowRankArgs& a, int device, cudaStream_t s, bool dry);

}  // namespace smat
