// solvers.cu — device-resident building blocks of the reference's matrix-free
// solvers (pkg/src/linopkit/solvers.py): batched conjugate gradients
// (_cg_single, solvers.py:75-106, run on every right-hand-side column at
// once), ISTA (solvers.py:163-194), the power method (solvers.py:295-333),
// soft thresholding (solvers.py:22-34) and OMP's atom pick (solvers.py:232-236).
//
// Every vector is an (n, K) C-contiguous float64 / complex128 block (the
// reference computes in np.result_type(rhs, field) >= float64).  The operator
// applications between the steps are ordinary smat_apply calls; the steps here
// keep every per-column scalar (rs, alpha, beta, iteration count, status) in a
// small device array so that an iteration needs no host round trip and a run
// of iterations can be captured in one CUDA graph.
//
// Column reductions are deterministic: a fixed grid of row blocks writes
// partial sums (one per row block and column), and the finalising kernel of
// each step adds them in row-block order.
#include <string>

#include "common.cuh"

namespace smat {
void set_last_error(const std::string& m);
}

namespace {
using namespace smat;

// ---- real / complex helpers (C = double or double2)
__device__ __forceinline__ double abs2_(double a) { return a * a; }
__device__ __forceinline__ double abs2_(double2 a) { return a.x * a.x + a.y * a.y; }
__device__ __forceinline__ double abs_(double a) { return fabs(a); }
__device__ __forceinline__ double abs_(double2 a) { return hypot(a.x, a.y); }
// conj(a) * b
__device__ __forceinline__ double2 vdot_(double a, double b) { return make_double2(a * b, 0.0); }
__device__ __forceinline__ double2 vdot_(double2 a, double2 b) {
  return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
__device__ __forceinline__ double axpy_(double y, double a, double x) { return fma(a, x, y); }
__device__ __forceinline__ double2 axpy_(double2 y, double a, double2 x) {
  return make_double2(fma(a, x.x, y.x), fma(a, x.y, y.y));
}
__device__ __forceinline__ double scale_(double x, double s) { return x * s; }
__device__ __forceinline__ double2 scale_(double2 x, double s) { return make_double2(x.x * s, x.y * s); }
template <class C> __device__ __forceinline__ C zero_();
template <> __device__ __forceinline__ double zero_<double>() { return 0.0; }
template <> __device__ __forceinline__ double2 zero_<double2>() { return make_double2(0.0, 0.0); }

// soft threshold (solvers.py:22-34): real sign(u)*max(|u|-c,0); complex
// u * max(|u|-c,0)/|u| (0 where u == 0)
__device__ __forceinline__ double soft_(double u, double c) {
  const double s = fmax(fabs(u) - c, 0.0);
  return u > 0 ? s : u < 0 ? -s : 0.0 * s;
}
__device__ __forceinline__ double2 soft_(double2 u, double c) {
  const double m = hypot(u.x, u.y);
  const double s = fmax(m - c, 0.0);
  const double f = m != 0.0 ? s / m : 0.0;
  return make_double2(u.x * f, u.y * f);
}

// ---- deterministic column reductions
// Block geometry: CP columns x RP rows per pass (CP*RP <= 256); grid.x column
// groups, grid.y row blocks.  Partial q of column c from row block b at
// part[(b*K + c)*Q + q].
struct RGeo {
  int CP = 32, RP = 8;
  dim3 grid;
};
RGeo rgeo(int64_t n, int64_t K) {
  RGeo g;
  if (K >= 32) {
    g.CP = 32;
    g.RP = 8;
  } else {
    g.CP = int(K);
    g.RP = 256 / int(K);
  }
  const int64_t gx = (K + g.CP - 1) / g.CP;
  int64_t gy = (n + int64_t(g.RP) * 16 - 1) / (int64_t(g.RP) * 16);  // >= 16 rows per thread
  const int64_t cap = gx >= 1184 ? 1 : 1184 / gx;
  if (gy > cap) gy = cap;
  if (gy < 1) gy = 1;
  g.grid = dim3(unsigned(gx), unsigned(gy));
  return g;
}
size_t part_bytes(int64_t n, int64_t K, int Q) {
  const RGeo g = rgeo(n, K);
  return size_t(g.grid.y) * size_t(K) * size_t(Q) * sizeof(double);
}

// F(i, c, acc[Q]) accumulates element (i, c); optionally also transforms it.
template <int Q, class F>
__global__ void __launch_bounds__(256) col_reduce_kernel(int64_t n, int64_t K, int CP, int RP, F f, double* part) {
  __shared__ double sh[256 * Q];
  const int tid = threadIdx.x;
  const int cl = tid % CP, rl = tid / CP;
  const int64_t c = int64_t(blockIdx.x) * CP + cl;
  double acc[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) acc[q] = 0.0;
  if (rl < RP && c < K) {
    for (int64_t i = int64_t(blockIdx.y) * RP + rl; i < n; i += int64_t(gridDim.y) * RP) f(i, c, acc);
  }
#pragma unroll
  for (int q = 0; q < Q; ++q) sh[tid * Q + q] = acc[q];
  __syncthreads();
  if (tid < CP && c < K) {
    double s[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) s[q] = 0.0;
    for (int r = 0; r < RP; ++r)
#pragma unroll
      for (int q = 0; q < Q; ++q) s[q] += sh[(r * CP + tid) * Q + q];
#pragma unroll
    for (int q = 0; q < Q; ++q) part[(int64_t(blockIdx.y) * K + c) * Q + q] = s[q];
  }
}

// Column totals of the partials, deterministic: one 128-thread block per
// column, thread t sums row blocks t, t+128, ... in order, then a fixed-shape
// shared-memory tree.  The finalising kernels run one block per column and
// use the result in thread 0.
template <int Q>
__device__ __forceinline__ bool col_sum(const double* part, int64_t K, int nb, int64_t c, double* out) {
  __shared__ double red[128 * Q];
  const int t = threadIdx.x;
  double v[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) v[q] = 0.0;
  for (int b = t; b < nb; b += 128)
#pragma unroll
    for (int q = 0; q < Q; ++q) v[q] += part[(int64_t(b) * K + c) * Q + q];
#pragma unroll
  for (int q = 0; q < Q; ++q) red[t * Q + q] = v[q];
  __syncthreads();
  for (int h = 64; h > 0; h >>= 1) {
    if (t < h)
#pragma unroll
      for (int q = 0; q < Q; ++q) red[t * Q + q] += red[(t + h) * Q + q];
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < Q; ++q) out[q] = red[q];
  return t == 0;
}

template <int Q, class F>
void reduce(int64_t n, int64_t K, F f, double* part, cudaStream_t s) {
  const RGeo g = rgeo(n, K);
  col_reduce_kernel<Q, F><<<g.grid, 256, 0, s>>>(n, K, g.CP, g.RP, f, part);
  SMAT_CUDA(cudaGetLastError());
}

inline unsigned blocks_for(int64_t n) {
  int64_t b = (n + 255) / 256;
  return unsigned(b > 4736 ? 4736 : b < 1 ? 1 : b);
}

// ============================================================ batched CG ====
// Per-column state (double[K][SMAT_CG_STATE]): see include/smat.h.
enum { CG_RS = 0, CG_THR, CG_ALPHA, CG_BETA, CG_ITERS, CG_STATUS, CG_RES, CG_CURV, CG_NS };

template <class C>
__global__ void cg_init_vec(const C* b, C* x, C* r, C* p, int64_t tot) {
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < tot; e += int64_t(gridDim.x) * blockDim.x) {
    const C v = b[e];
    x[e] = zero_<C>();
    r[e] = v;
    p[e] = v;
  }
}
__global__ void cg_init_fin(const double* part, int nb, int64_t K, double tol, double* st) {
  const int64_t c = blockIdx.x;
  double rr;
  if (!col_sum<1>(part, K, nb, c, &rr)) return;
  double* s = st + c * CG_NS;
  const double nr0 = sqrt(rr);
  s[CG_RS] = rr;
  s[CG_THR] = tol * nr0;
  s[CG_ALPHA] = s[CG_BETA] = 0.0;
  s[CG_ITERS] = 0.0;
  s[CG_CURV] = 0.0;
  // zero right-hand side: x = 0, 0 iterations, converged (solvers.py:81-82)
  s[CG_STATUS] = nr0 == 0.0 ? 1.0 : 0.0;
  s[CG_RES] = 0.0;
}
__global__ void cg_alpha_fin(const double* part, int nb, int64_t K, double* st) {
  const int64_t c = blockIdx.x;
  double* s = st + c * CG_NS;
  if (s[CG_STATUS] != 0.0) return;  // (uniform over the block)
  double v[3];
  if (!col_sum<3>(part, K, nb, c, v)) return;
  const double curv = v[0], slack = 1e-14 * sqrt(v[1]) * sqrt(v[2]);
  if (curv <= slack) {  // BreakdownError (solvers.py:88-93)
    s[CG_STATUS] = 2.0;
    s[CG_CURV] = curv;
    s[CG_ITERS] += 1.0;
    return;
  }
  s[CG_ALPHA] = s[CG_RS] / curv;
}
__global__ void cg_beta_fin(const double* part, int nb, int64_t K, double max_iter, double* st) {
  const int64_t c = blockIdx.x;
  double* s = st + c * CG_NS;
  if (s[CG_STATUS] != 0.0) return;  // (uniform over the block)
  double rs_new;
  if (!col_sum<1>(part, K, nb, c, &rs_new)) return;
  const double it = s[CG_ITERS] + 1.0;
  s[CG_ITERS] = it;
  if (sqrt(rs_new) <= s[CG_THR]) {  // converged (solvers.py:97-98)
    s[CG_STATUS] = 1.0;
    s[CG_RES] = sqrt(rs_new);
    return;
  }
  s[CG_BETA] = rs_new / s[CG_RS];
  s[CG_RS] = rs_new;
  if (it >= max_iter) {  // not converged: residual sqrt(rs_old) (solvers.py:101)
    s[CG_STATUS] = 3.0;
    s[CG_RES] = sqrt(rs_new);
  }
}
template <class C>
__global__ void cg_p_update(const C* r, C* p, const double* st, int64_t K, int64_t tot) {
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < tot; e += int64_t(gridDim.x) * blockDim.x) {
    const double* s = st + (e % K) * CG_NS;
    if (s[CG_STATUS] == 0.0) p[e] = axpy_(r[e], s[CG_BETA], p[e]);
  }
}

template <class C>
void cg_init_t(int64_t n, int64_t K, const void* b, void* x, void* r, void* p, double* st, double tol, double* part,
               cudaStream_t s) {
  const C* bb = (const C*)b;
  reduce<1>(n, K, [=] __device__(int64_t i, int64_t c, double* a) { a[0] += abs2_(bb[i * K + c]); }, part, s);
  cg_init_vec<C><<<blocks_for(n * K), 256, 0, s>>>(bb, (C*)x, (C*)r, (C*)p, n * K);
  cg_init_fin<<<unsigned(K), 128, 0, s>>>(part, int(rgeo(n, K).grid.y), K, tol, st);
  SMAT_CUDA(cudaGetLastError());
}

template <class C>
void cg_step_t(int64_t n, int64_t K, void* x_, void* r_, void* p_, const void* ap_, double* st, int64_t max_iter,
               double* part, cudaStream_t s) {
  C* x = (C*)x_;
  C* r = (C*)r_;
  C* p = (C*)p_;
  const C* ap = (const C*)ap_;
  const int nb = int(rgeo(n, K).grid.y);
  const unsigned cb = unsigned(K);  // one finalising block per column
  // curvature Re<p, Ap>, |p|^2, |Ap|^2 (solvers.py:86-87)
  reduce<3>(
      n, K,
      [=] __device__(int64_t i, int64_t c, double* a) {
        const C pv = p[i * K + c], av = ap[i * K + c];
        a[0] += vdot_(pv, av).x;
        a[1] += abs2_(pv);
        a[2] += abs2_(av);
      },
      part, s);
  cg_alpha_fin<<<cb, 128, 0, s>>>(part, nb, K, st);
  // x += alpha p ; r -= alpha Ap ; |r|^2 (solvers.py:94-96), active columns only
  reduce<1>(
      n, K,
      [=] __device__(int64_t i, int64_t c, double* a) {
        const double* sc = st + c * CG_NS;
        const int64_t e = i * K + c;
        C rv = r[e];
        if (sc[CG_STATUS] == 0.0) {
          const double al = sc[CG_ALPHA];
          x[e] = axpy_(x[e], al, p[e]);
          rv = axpy_(rv, -al, ap[e]);
          r[e] = rv;
        }
        a[0] += abs2_(rv);
      },
      part, s);
  cg_beta_fin<<<cb, 128, 0, s>>>(part, nb, K, double(max_iter), st);
  cg_p_update<C><<<blocks_for(n * K), 256, 0, s>>>(r, p, st, K, n * K);
  SMAT_CUDA(cudaGetLastError());
}

// ================================================================ ISTA =====
// state: [0] l1 of the current x, [1] step counter k
template <class C>
void ista_residual_t(int64_t n, const void* b_, const void* mx_, void* r_, double* trace, double* st, double lam,
                     double* part, cudaStream_t s);
__global__ void ista_trace_fin(const double* part, int nb, double lam, double* trace, double* st) {
  double rr;
  if (!col_sum<1>(part, 1, nb, 0, &rr)) return;
  const int64_t k = int64_t(st[1]);
  trace[k] = lam * st[0] + 0.5 * rr;  // solvers.py:185-187, 190-192
  st[1] = double(k + 1);
}
template <class C>
void ista_residual_t(int64_t n, const void* b_, const void* mx_, void* r_, double* trace, double* st, double lam,
                     double* part, cudaStream_t s) {
  const C* b = (const C*)b_;
  const C* mx = (const C*)mx_;
  C* r = (C*)r_;
  reduce<1>(
      n, 1,
      [=] __device__(int64_t i, int64_t, double* a) {
        C v = b[i];
        const C m = mx[i];
        v = axpy_(v, -1.0, m);
        r[i] = v;
        a[0] += abs2_(v);
      },
      part, s);
  ista_trace_fin<<<1, 128, 0, s>>>(part, int(rgeo(n, 1).grid.y), lam, trace, st);
  SMAT_CUDA(cudaGetLastError());
}
__global__ void ista_l1_fin(const double* part, int nb, double* st) {
  double l1;
  if (!col_sum<1>(part, 1, nb, 0, &l1)) return;
  st[0] = l1;
}
template <class C>
void ista_update_t(int64_t n, void* x_, const void* g_, double alpha, double level, double* st, double* part,
                   cudaStream_t s) {
  C* x = (C*)x_;
  const C* g = (const C*)g_;
  // x <- soft(x + alpha * M^H r, lam * alpha) (solvers.py:188), l1 of the new x
  reduce<1>(
      n, 1,
      [=] __device__(int64_t i, int64_t, double* a) {
        const C v = soft_(axpy_(x[i], alpha, g[i]), level);
        x[i] = v;
        a[0] += abs_(v);
      },
      part, s);
  ista_l1_fin<<<1, 128, 0, s>>>(part, int(rgeo(n, 1).grid.y), st);
  SMAT_CUDA(cudaGetLastError());
}

// ====================================================== power iteration =====
// state: [0] estimate, [1] iterations, [2] done, [3] converged, [4] 1/|w| of
// this step (0: do not normalise), [5] zero flag
__global__ void power_fin(const double* part, int nb, double tol, double* st) {
  const bool done = st[2] != 0.0;
  __syncthreads();  // every thread has read `done` before thread 0 writes the state
  double v[3];
  if (!col_sum<3>(part, 1, nb, 0, v)) return;
  st[4] = 0.0;
  if (done) return;
  const double it = st[1] + 1.0;
  st[1] = it;
  const double est_new = hypot(v[0], v[1]);  // |vdot(v, w)| (solvers.py:321-322)
  const double nw = sqrt(v[2]);
  if (nw == 0.0) {  // operator annihilated the iterate (solvers.py:324-326)
    st[2] = 1.0;
    st[3] = 1.0;
    st[5] = 1.0;
    st[0] = 0.0;
    return;
  }
  st[4] = 1.0 / nw;
  if (it > 1.0 && fabs(est_new - st[0]) <= tol * fmax(est_new, 1e-300)) {  // solvers.py:328
    st[2] = 1.0;
    st[3] = 1.0;
  }
  st[0] = est_new;
}
template <class C>
__global__ void power_norm(C* v, const C* w, const double* st, int64_t n) {
  const double inv = st[4];
  if (inv == 0.0) return;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    v[i] = scale_(w[i], inv);
}
template <class C>
void power_step_t(int64_t n, void* v_, const void* w_, double* st, double tol, double* part, cudaStream_t s) {
  C* v = (C*)v_;
  const C* w = (const C*)w_;
  reduce<3>(
      n, 1,
      [=] __device__(int64_t i, int64_t, double* a) {
        const C vv = v[i], wv = w[i];
        const double2 d = vdot_(vv, wv);
        a[0] += d.x;
        a[1] += d.y;
        a[2] += abs2_(wv);
      },
      part, s);
  power_fin<<<1, 128, 0, s>>>(part, int(rgeo(n, 1).grid.y), tol, st);
  power_norm<C><<<blocks_for(n), 256, 0, s>>>(v, w, st, n);
  SMAT_CUDA(cudaGetLastError());
}

// ===================================================== soft threshold =====
template <class C>
__global__ void soft_kernel(const C* x, C* y, double c, int64_t n) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    y[i] = soft_(x[i], c);
}

// ================================================== OMP atom selection =====
// argmax_i |g[i]| over i not excluded; ties -> lowest index (np.argmax,
// solvers.py:233-235).  Two stages: per-block (value, index) then one block.
template <class C>
__global__ void absmax_part(const C* g, const unsigned char* excl, int64_t n, double* pv, int64_t* pi) {
  __shared__ double sv[256];
  __shared__ int64_t si[256];
  double best = -2.0;
  int64_t bi = INT64_MAX;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const double v = (excl && excl[i]) ? -1.0 : abs_(g[i]);
    if (v > best) {  // strided ascending i: first hit wins ties
      best = v;
      bi = i;
    }
  }
  sv[threadIdx.x] = best;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int h = 128; h > 0; h >>= 1) {
    if (threadIdx.x < h) {
      const double ov = sv[threadIdx.x + h];
      const int64_t oi = si[threadIdx.x + h];
      if (ov > sv[threadIdx.x] || (ov == sv[threadIdx.x] && oi < si[threadIdx.x])) {
        sv[threadIdx.x] = ov;
        si[threadIdx.x] = oi;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    pv[blockIdx.x] = sv[0];
    pi[blockIdx.x] = si[0];
  }
}
__global__ void absmax_fin(const double* pv, const int64_t* pi, int nb, int64_t* out) {
  if (threadIdx.x || blockIdx.x) return;
  double best = -3.0;
  int64_t bi = 0;
  for (int b = 0; b < nb; ++b)
    if (pv[b] > best || (pv[b] == best && pi[b] < bi)) {
      best = pv[b];
      bi = pi[b];
    }
  out[0] = bi;
}

template <class F>
int guarded(F f) {
  try {
    f();
    return SMAT_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return SMAT_BAD_ARG;
  }
}

int need(double* part, size_t have, int64_t n, int64_t K, int Q) {
  if (!part) return SMAT_BAD_ARG;
  return have >= part_bytes(n, K, Q) ? SMAT_OK : SMAT_BAD_ARG;
}

#define SMAT_DISPATCH(dtype, FN, ...)                                                     \
  do {                                                                                    \
    if ((dtype) == SMAT_F64) FN<double>(__VA_ARGS__);                                     \
    else if ((dtype) == SMAT_C128) FN<double2>(__VA_ARGS__);                              \
    else throw Error(SMAT_BAD_DTYPE, "solver vectors must be float64 or complex128");     \
  } while (0)

}  // namespace

extern "C" {

size_t smat_solver_scratch_bytes(int64_t n, int64_t ncols) {
  if (n < 1 || ncols < 1) return 0;
  const size_t a = part_bytes(n, ncols, 3);
  const size_t b = size_t(592) * (sizeof(double) + sizeof(int64_t));  // smat_abs_argmax
  return a > b ? a : b;
}

int smat_cg_init(int32_t dtype, int64_t n, int64_t ncols, const void* b, void* x, void* r, void* p, double* state,
                 double tol, void* scratch, size_t scratch_bytes, void* stream) {
  if (!b || !x || !r || !p || !state || n < 1 || ncols < 1) {
    set_last_error("smat_cg_init: bad argument");
    return SMAT_BAD_ARG;
  }
  if (need((double*)scratch, scratch_bytes, n, ncols, 3) != SMAT_OK) {
    set_last_error("smat_cg_init: scratch too small");
    return SMAT_BAD_ARG;
  }
  return guarded([&] {
    SMAT_DISPATCH(dtype, cg_init_t, n, ncols, b, x, r, p, state, tol, (double*)scratch, (cudaStream_t)stream);
  });
}

int smat_cg_step(int32_t dtype, int64_t n, int64_t ncols, void* x, void* r, void* p, const void* ap, double* state,
                 int64_t max_iter, void* scratch, size_t scratch_bytes, void* stream) {
  if (!x || !r || !p || !ap || !state || n < 1 || ncols < 1) {
    set_last_error("smat_cg_step: bad argument");
    return SMAT_BAD_ARG;
  }
  if (need((double*)scratch, scratch_bytes, n, ncols, 3) != SMAT_OK) {
    set_last_error("smat_cg_step: scratch too small");
    return SMAT_BAD_ARG;
  }
  return guarded([&] {
    SMAT_DISPATCH(dtype, cg_step_t, n, ncols, x, r, p, ap, state, max_iter, (double*)scratch, (cudaStream_t)stream);
  });
}

int smat_ista_residual(int32_t dtype, int64_t n, const void* b, const void* mx, void* r, double* trace,
                       double* state, double lam, void* scratch, size_t scratch_bytes, void* stream) {
  if (!b || !mx || !r || !trace || !state || n < 1) {
    set_last_error("smat_ista_residual: bad argument");
    return SMAT_BAD_ARG;
  }
  if (need((double*)scratch, scratch_bytes, n, 1, 3) != SMAT_OK) {
    set_last_error("smat_ista_residual: scratch too small");
    return SMAT_BAD_ARG;
  }
  return guarded([&] {
    SMAT_DISPATCH(dtype, ista_residual_t, n, b, mx, r, trace, state, lam, (double*)scratch, (cudaStream_t)stream);
  });
}

int smat_ista_update(int32_t dtype, int64_t n, void* x, const void* g, double alpha, double level, double* state,
                     void* scratch, size_t scratch_bytes, void* stream) {
  if (!x || !g || !state || n < 1 || level < 0) {
    set_last_error("smat_ista_update: bad argument");
    return SMAT_BAD_ARG;
  }
  if (need((double*)scratch, scratch_bytes, n, 1, 3) != SMAT_OK) {
    set_last_error("smat_ista_update: scratch too small");
    return SMAT_BAD_ARG;
  }
  return guarded([&] {
    SMAT_DISPATCH(dtype, ista_update_t, n, x, g, alpha, level, state, (double*)scratch, (cudaStream_t)stream);
  });
}

int smat_power_step(int32_t dtype, int64_t n, void* v, const void* w, double* state, double tol, void* scratch,
                    size_t scratch_bytes, void* stream) {
  if (!v || !w || !state || n < 1) {
    set_last_error("smat_power_step: bad argument");
    return SMAT_BAD_ARG;
  }
  if (need((double*)scratch, scratch_bytes, n, 1, 3) != SMAT_OK) {
    set_last_error("smat_power_step: scratch too small");
    return SMAT_BAD_ARG;
  }
  return guarded([&] {
    SMAT_DISPATCH(dtype, power_step_t, n, v, w, state, tol, (double*)scratch, (cudaStream_t)stream);
  });
}

int smat_soft_threshold(int32_t dtype, int64_t n, const void* x, void* y, double c, void* stream) {
  if (!x || !y || n < 0) {
    set_last_error("smat_soft_threshold: bad argument");
    return SMAT_BAD_ARG;
  }
  if (c < 0) {
    set_last_error("threshold must be >= 0");
    return SMAT_BAD_ARG;
  }
  if (n == 0) return SMAT_OK;
  return guarded([&] {
    cudaStream_t s = (cudaStream_t)stream;
    if (dtype == SMAT_F64) soft_kernel<double><<<blocks_for(n), 256, 0, s>>>((const double*)x, (double*)y, c, n);
    else if (dtype == SMAT_C128)
      soft_kernel<double2><<<blocks_for(n), 256, 0, s>>>((const double2*)x, (double2*)y, c, n);
    else throw Error(SMAT_BAD_DTYPE, "soft threshold needs float64 or complex128");
    SMAT_CUDA(cudaGetLastError());
  });
}

int smat_abs_argmax(int32_t dtype, int64_t n, const void* g, const unsigned char* excluded, int64_t* out_index,
                    void* scratch, size_t scratch_bytes, void* stream) {
  if (!g || !out_index || n < 1 || !scratch) {
    set_last_error("smat_abs_argmax: bad argument");
    return SMAT_BAD_ARG;
  }
  const int nb = int(blocks_for(n) > 592 ? 592 : blocks_for(n));
  if (scratch_bytes < size_t(nb) * (sizeof(double) + sizeof(int64_t))) {
    set_last_error("smat_abs_argmax: scratch too small");
    return SMAT_BAD_ARG;
  }
  return guarded([&] {
    cudaStream_t s = (cudaStream_t)stream;
    double* pv = (double*)scratch;
    int64_t* pi = (int64_t*)(pv + nb);
    if (dtype == SMAT_F64) absmax_part<double><<<nb, 256, 0, s>>>((const double*)g, excluded, n, pv, pi);
    else if (dtype == SMAT_C128) absmax_part<double2><<<nb, 256, 0, s>>>((const double2*)g, excluded, n, pv, pi);
    else throw Error(SMAT_BAD_DTYPE, "argmax needs float64 or complex128");
    absmax_fin<<<1, 32, 0, s>>>(pv, pi, nb, out_index);
    SMAT_CUDA(cudaGetLastError());
  });
}

}  // extern "C"
