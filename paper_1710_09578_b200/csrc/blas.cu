// blas.cu — the Dense (Matrix) leaf as a plain library GEMM through cuBLAS
// (reference leaves.py:40-46: entries @ x).  No structured transform and no
// LowRank term uses it (those run on the hand-written kernels).
//
// cuBLAS is resolved at run time (dlopen of libcublas.so.12 — the copy torch
// has already loaded, else the toolkit's), so libsmat.so has no link-time
// dependency on it; one handle per (thread, device) and a fixed workspace per
// (thread, device, stream), so that the calls are CUDA-graph capturable.
#include <dlfcn.h>

#include <cstdlib>
#include <mutex>
#include <unordered_map>

#include "misc_kernels.cuh"

namespace smat {

namespace {
using Handle = void*;
using CreateFn = int (*)(Handle*);
using SetStreamFn = int (*)(Handle, cudaStream_t);
using SetWsFn = int (*)(Handle, void*, size_t);
using ZgemmFn = int (*)(Handle, int, int, int, int, int, const double2*, const double2*, int, const double2*, int,
                        const double2*, double2*, int);

using GemmAny = int (*)(Handle, int, int, int, int, int, const void*, const void*, int, const void*, int,
                        const void*, void*, int);

struct Blas {
  bool ok = false;
  CreateFn create = nullptr;
  SetStreamFn set_stream = nullptr;
  SetWsFn set_ws = nullptr;
  ZgemmFn zgemm = nullptr;
  GemmAny sgemm = nullptr, dgemm = nullptr, cgemm = nullptr;
};

const Blas& blas() {
  static Blas b;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libcublas.so.12", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("/usr/local/cuda/lib64/libcublas.so.12", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    b.create = (CreateFn)dlsym(h, "cublasCreate_v2");
    b.set_stream = (SetStreamFn)dlsym(h, "cublasSetStream_v2");
    b.set_ws = (SetWsFn)dlsym(h, "cublasSetWorkspace_v2");
    b.zgemm = (ZgemmFn)dlsym(h, "cublasZgemm_v2");
    b.sgemm = (GemmAny)dlsym(h, "cublasSgemm_v2");
    b.dgemm = (GemmAny)dlsym(h, "cublasDgemm_v2");
    b.cgemm = (GemmAny)dlsym(h, "cublasCgemm_v2");
    b.ok = b.create && b.set_stream && b.set_ws && b.zgemm && b.sgemm && b.dgemm && b.cgemm;
  });
  return b;
}

Handle handle_for(int device) {
  thread_local std::unordered_map<int, Handle> handles;
  auto it = handles.find(device);
  if (it != handles.end()) return it->second;
  const Blas& b = blas();
  Handle h = nullptr;
  SMAT_CHECK(b.create(&h) == 0, SMAT_CUDA_ERROR, "cublasCreate failed");
  handles[device] = h;
  return h;
}

// Bind the handle to stream s with a workspace of its own: cublasSetStream
// resets the handle to cuBLAS's default workspace pool, so the fixed
// workspace is re-attached after every stream switch — one buffer per
// (thread, device, stream), never shared by two streams that may run
// concurrently (the pattern of PyTorch's handle pool).
void bind_stream(Handle h, int device, cudaStream_t s) {
  thread_local std::unordered_map<uint64_t, void*> ws_by_stream;
  constexpr size_t kWs = size_t(32) << 20;
  const Blas& b = blas();
  SMAT_CHECK(b.set_stream(h, s) == 0, SMAT_CUDA_ERROR, "cublasSetStream failed");
  const uint64_t key = uint64_t(uintptr_t(s)) * 64 + uint64_t(device);
  void*& ws = ws_by_stream[key];
  if (!ws) SMAT_CUDA(cudaMalloc(&ws, kWs));  // lives as long as the thread's handle (process)
  SMAT_CHECK(b.set_ws(h, ws, kWs) == 0, SMAT_CUDA_ERROR, "cublasSetWorkspace failed");
}
}  // namespace

bool blas_available() { return blas().ok; }

// create this thread's handle for `device` now (plan build), so that a later
// call inside a CUDA-graph capture allocates nothing
void blas_warm(int device) {
  if (blas().ok) handle_for(device);
}

// Column-major C = op(A) op(B) + beta C in the plan dtype (float32, float64,
// complex64, complex128): the Dense leaf's plain GEMM.
void blas_gemm(int dt, int device, cudaStream_t s, int opa, int opb, int64_t m, int64_t n, int64_t k, const void* A,
               int64_t lda, const void* B, int64_t ldb, double beta_re, void* C, int64_t ldc) {
  const Blas& b = blas();
  SMAT_CHECK(b.ok, SMAT_UNSUPPORTED, "cuBLAS not available");
  SMAT_CHECK(m < (int64_t(1) << 31) && n < (int64_t(1) << 31) && k < (int64_t(1) << 31), SMAT_UNSUPPORTED,
             "gemm dimension exceeds int32");
  Handle h = handle_for(device);
  bind_stream(h, device, s);
  int st = 0;
  if (dt == SMAT_F32) {
    const float one = 1.f, beta = float(beta_re);
    st = b.sgemm(h, opa, opb, int(m), int(n), int(k), &one, A, int(lda), B, int(ldb), &beta, C, int(ldc));
  } else if (dt == SMAT_F64) {
    const double one = 1.0, beta = beta_re;
    st = b.dgemm(h, opa, opb, int(m), int(n), int(k), &one, A, int(lda), B, int(ldb), &beta, C, int(ldc));
  } else if (dt == SMAT_C64) {
    const float2 one = make_float2(1.f, 0.f), beta = make_float2(float(beta_re), 0.f);
    st = b.cgemm(h, opa, opb, int(m), int(n), int(k), &one, A, int(lda), B, int(ldb), &beta, C, int(ldc));
  } else if (dt == SMAT_C128) {
    const double2 one = make_double2(1.0, 0.0), beta = make_double2(beta_re, 0.0);
    st = b.zgemm(h, opa, opb, int(m), int(n), int(k), &one, (const double2*)A, int(lda), (const double2*)B,
                 int(ldb), &beta, (double2*)C, int(ldc));
  } else {
    throw Error(SMAT_BAD_DTYPE, "gemm: unsupported dtype");
  }
  SMAT_CHECK(st == 0, SMAT_CUDA_ERROR, "cublas gemm failed with status " + std::to_string(st));
}

}  // namespace smat
