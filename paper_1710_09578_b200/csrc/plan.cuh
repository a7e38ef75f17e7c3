// plan.cuh — compiled operator plans: the native replacement of the
// reference's recursive _forward/_backward dispatch (composites.py:49-61,
// 96-113, 171-187, 290-310; leaves.py:40-290).
//
// A plan is a tree of executable nodes built once from the serialised
// smat_node array.  apply() walks the tree on the HOST, launching one fused
// pass per leaf transform (or per group of leaves for the pattern-matched
// fused plans in fused.cu) on a single stream; all buffers come from the
// caller's workspace via a bump allocator whose high-water mark is found by
// a dry run (Ctx::measure), so apply() never allocates.
#pragma once

#include <memory>
#include <string>
#include <vector>

#include "common.cuh"
#include "misc_kernels.cuh"
#include "tile_kernels.cuh"
#include "wlr.cuh"

namespace smat {

// A buffer view: element (o1, o2, i, c) at p + (o1*s1 + o2*s2 + i*si + c) elements.
struct Blk {
  void* p = nullptr;
  int dt = 0;
  int64_t s1 = 0, s2 = 0, si = 0;
};
// Batch geometry shared by the input and output views of one node apply.
struct Geo {
  int64_t n1 = 1, n2 = 1, inner = 1;
  int64_t count() const { return n1 * n2 * inner; }
};

inline Blk offset_rows(const Blk& b, int64_t rows) {
  Blk r = b;
  r.p = (char*)b.p + rows * b.si * int64_t(dt_size(b.dt));
  return r;
}

struct Ctx {
  cudaStream_t stream = nullptr;
  int device = 0;
  int dt = 0;  // plan dtype
  char* ws = nullptr;
  size_t ws_size = 0, top = 0, peak = 0;
  bool measure = false;
  bool probe = false;  // (with measure) ask the launchers whether each pass would run
  int64_t launches = 0;
  // fused 8-point Walsh-Hadamard for the next single-tile transform
  // (KronNode's Hadamard x FFT passes, FftArgs::wht_grp); run_xform consumes it
  int wgrp = 0;
  int64_t wg_xs = 0, wg_ys = 0;
  bool wg_used = false;

  void* alloc(size_t bytes) {
    size_t off = (top + 255) & ~size_t(255);
    top = off + bytes;
    if (top > peak) peak = top;
    if (measure) return (void*)(uintptr_t(0x1000) + off);  // never dereferenced
    SMAT_CHECK(top <= ws_size, SMAT_BAD_ARG,
               "workspace too small: need " + std::to_string(top) + " bytes, have " +
                   std::to_string(ws_size));
    return ws + off;
  }
  // contiguous [n1*n2][rows][inner] buffer of dtype dt
  Blk alloc_blk(int dtype, const Geo& g, int64_t rows) {
    Blk b;
    b.dt = dtype;
    b.si = g.inner;
    b.s2 = rows * g.inner;
    b.s1 = g.n2 * b.s2;
    b.p = alloc(size_t(g.count()) * size_t(rows) * dt_size(dtype));
    return b;
  }
  size_t mark() const { return top; }
  void release(size_t m) { top = m; }

  // optional per-launch profiling (smat_apply_profiled): an event is recorded
  // on the stream before every launch
  std::vector<std::pair<std::string, cudaEvent_t>>* prof = nullptr;
  void note(const std::string& name) {
    if (!prof || measure) return;
    cudaEvent_t e;
    SMAT_CUDA(cudaEventCreate(&e));
    SMAT_CUDA(cudaEventRecord(e, stream));
    prof->emplace_back(name, e);
  }

  // counted launches (skipped in measure mode)
  void fft(int cdt, int N, const FftArgs& a) {
    ++launches;
    // label: precision, length and the fused extras (spectrum, four-step
    // twiddle, pad/truncate/pre/post masks)
    std::string lab = std::string(cdt == SMAT_C128 ? "fft_c128_" : "fft_c64_") + std::to_string(N);
    if (prof) {
      if (a.mid) lab += "_spec";
      if (a.tw_on) lab += a.tw_pre ? "_twin" : "_tw";
      const bool pad = (a.g_mod - 1) + (N - 1) * a.gin_stride >= a.n_valid_in;
      const bool trunc = (a.g_mod - 1) + (N - 1) * a.gout_stride >= a.n_valid_out;
      if (a.pre || a.post || pad || trunc) lab += "_msk";
    }
    note(lab);
    if (!measure) {
      launch_fft_tile(cdt, N, a, stream);
    } else if (probe) {
      FftArgs q = a;
      q.probe_only = 1;
      launch_fft_tile(cdt, N, q, stream);
    }
  }
  void wht(int d, int N, const WhtArgs& a) {
    ++launches;
    note("wht_" + std::to_string(N));
    if (!measure) launch_wht_tile(d, N, a, stream);
  }
  void point(const PointArgs& a) {
    ++launches;
    note("point");
    if (!measure) launch_point(dt, a, stream);
  }
  // pointwise pass in an explicit dtype (staging copies of the apply's user blocks)
  void point_dt(int pdt, const PointArgs& a) {
    ++launches;
    note("stage");
    if (!measure) launch_point(pdt, a, stream);
  }
  void gather(const IndexArgs& a) {
    ++launches;
    note("gather");
    if (!measure) launch_gather(dt, a, stream);
  }
  void scatter(const IndexArgs& a) {
    ++launches;
    note("scatter");
    if (!measure) launch_scatter_add(dt, a, stream);
  }
  void gemm(const GemmArgs& a) {
    launches += launch_gemm(dt, a, device, stream, true);
    note("gemm");
    if (!measure) launch_gemm(dt, a, device, stream, false);
  }
  void csr(const CsrArgs& a) {
    ++launches;
    note("csr");
    if (!measure) launch_csr(dt, a, stream);
  }
  void gemm_blas(int opa, int opb, int64_t m, int64_t n, int64_t k, const void* A, int64_t lda, const void* B,
                 int64_t ldb, double beta, void* C, int64_t ldc) {
    note("gemm_blas");
    if (!measure) blas_gemm(dt, device, stream, opa, opb, m, n, k, A, lda, B, ldb, beta, C, ldc);
  }
  // fused Hadamard + LowRank pass / plain LowRank half on FP64 tensor cores (wlr.cu)
  void wlr(const WlrMode& m, const WlrArgs& a, const char* label) {
    launches += launch_wlr(m, a, device, stream, true);
    note(label);
    if (!measure) launch_wlr(m, a, device, stream, false);
  }
  void wlr_fin(const void* partial, int64_t r, int64_t K, const void* s, bool s_conj, double* w3) {
    const int grid = wlr_grid(device, K);
    launches += launch_wlr_finalize(partial, grid, r, K, s, s_conj, w3, stream, true);
    note("lowrank_finalize");
    if (!measure) launch_wlr_finalize(partial, grid, r, K, s, s_conj, w3, stream, false);
  }
  void lr_contract(const LowRankArgs& a) {
    launches += launch_lowrank_contract(dt, a, device, stream, true);
    note("lowrank_contract");
    if (!measure) launch_lowrank_contract(dt, a, device, stream, false);
  }
  void lr_expand(const LowRankArgs& a) {
    launches += launch_lowrank_expand(dt, a, device, stream, true);
    note("lowrank_expand");
    if (!measure) launch_lowrank_expand(dt, a, device, stream, false);
  }

  // Fork / join with the device's side stream (independent branches of a
  // node run concurrently; graph-capturable event edges).  Disabled in
  // measure and profiling mode (the per-launch profile needs one timeline).
  bool can_fork() const { return !measure && !prof; }
  cudaStream_t fork();               // side stream, ordered after this stream
  void join(cudaStream_t side);      // this stream waits for the side stream
};

// A device array owned by a plan.
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  int dt = 0;
  int64_t len = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};

struct Node {
  int64_t rows = 0, cols = 0;
  virtual ~Node() = default;
  // y (=, or += when acc) op(x) with op = A (adj == false) or A^H.  x has
  // n_in = adj ? rows : cols rows, y has n_out rows; both share geometry g.
  // x.dt is the plan dtype or, for a complex plan, its real dtype when
  // accepts_real() is true; y.dt is the plan dtype.
  virtual void apply(Ctx& c, bool adj, const Blk& x, const Blk& y, const Geo& g, bool acc) = 0;
  virtual bool accepts_real() const { return false; }
  virtual bool is_identity() const { return false; }
  virtual std::string describe() const = 0;
};

struct Plan {
  std::vector<std::unique_ptr<Node>> nodes;
  std::vector<std::unique_ptr<DevBuf>> bufs;
  Node* root = nullptr;
  int dt = 0;
  int device = 0;
  int64_t rows = 0, cols = 0;
  std::string fused;  // name of the pattern-matched fused plan, if any
};

// builders (plan.cu)
Plan* build_plan(const smat_node* nodes, int n_nodes, const int32_t* children, int n_children,
                 int root, int dt, int device);
// y = A x (dir 0) or A^H x (dir 1); x / y row-major with leading dimensions
// ldx / ldy (0: dense) or column-major (layout SMAT_COL_MAJOR)
void run_plan(const Plan& p, Ctx& c, int dir, const void* x, int x_dt, int64_t ldx, void* y, int64_t ldy,
              int64_t ncols, int layout);

// helpers shared with fused.cu
DevBuf* upload_param(Plan& p, const smat_param& prm, int target_dt);
DevBuf* new_buf(Plan& p, int dt, int64_t len);
void device_fft_c128(Plan& p, int64_t n, const void* in_dev, void* out_dev);

}  // namespace smat
