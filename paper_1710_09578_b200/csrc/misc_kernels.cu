// misc_kernels.cu — pointwise / index / GEMM passes of the generic interpreter.
//
// Reference counterparts: Diagonal._forward/_backward (leaves.py:90-94),
// Identity copy (leaves.py:72-76), Zero (leaves.py:58-62), the Blocks/Sum
// accumulation (composites.py:171-178), Partial scatter/gather
// (composites.py:281-310) and Dense matmul (leaves.py:40-46).
#include <type_traits>

#include "misc_kernels.cuh"

namespace smat {

template <class P> struct IsCx : std::false_type {};
template <> struct IsCx<float2> : std::true_type {};
template <> struct IsCx<double2> : std::true_type {};
template <class P> struct RealT { using T = P; };
template <> struct RealT<float2> { using T = float; };
template <> struct RealT<double2> { using T = double; };

template <class P> __device__ __forceinline__ P zval() {
  if constexpr (IsCx<P>::value) return mk(typename RealT<P>::T(0), typename RealT<P>::T(0));
  else return P(0);
}
template <class P> __device__ __forceinline__ P pmul(P a, P b) {
  if constexpr (IsCx<P>::value) return cmul(a, b);
  else return a * b;
}
template <class P> __device__ __forceinline__ P pconj(P a) {
  if constexpr (IsCx<P>::value) return conj(a);
  else return a;
}
template <class P> __device__ __forceinline__ P padd(P a, P b) { return a + b; }

// ------------------------------------------------------------ pointwise ----
template <class P, bool XR, bool YR>
__global__ void point_kernel(const PointArgs a) {
  using R = typename RealT<P>::T;
  const int64_t total = a.nb * a.n;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += stride) {
    const int64_t c = e % a.inner;
    const int64_t t = e / a.inner;
    const int64_t i = t % a.n;
    const int64_t o = t / a.n;
    const int64_t o2 = o % a.n2, o1 = o / a.n2;
    P v = zval<P>();
    if (a.x) {
      const int64_t xo = o1 * a.xs1 + o2 * a.xs2 + i * a.xsi + c;
      if constexpr (XR) v = mk(((const R*)a.x)[xo], R(0));
      else v = ((const P*)a.x)[xo];
      if (a.x_conj) v = pconj(v);
      if (a.d) {
        P w = ((const P*)a.d)[i];
        if (a.d_conj) w = pconj(w);
        v = pmul(v, w);
      }
      if constexpr (IsCx<P>::value) {
        if (a.scale_re != 1.0 || a.scale_im != 0.0) v = cmul(v, mk(R(a.scale_re), R(a.scale_im)));
      } else if constexpr (std::is_floating_point<P>::value) {
        if (a.scale_re != 1.0) v = v * R(a.scale_re);
      }
    } else if (a.accumulate) {
      continue;
    }
    const int64_t yo = o1 * a.ys1 + o2 * a.ys2 + i * a.ysi + c;
    if constexpr (YR) {
      R* y = (R*)a.y;
      y[yo] = a.accumulate ? y[yo] + v.x : v.x;
    } else {
      P* y = (P*)a.y;
      y[yo] = a.accumulate ? padd(y[yo], v) : v;
    }
  }
}

static unsigned ew_blocks(int64_t total) {
  int64_t b = (total + 255) / 256;
  if (b > 148 * 16) b = 148 * 16;
  return unsigned(b < 1 ? 1 : b);
}

template <class P>
static void point_dispatch(const PointArgs& a, bool xr, bool yr, cudaStream_t s) {
  const int64_t total = a.nb * a.n;
  if (total == 0) return;
  if constexpr (IsCx<P>::value) {
    if (xr && yr) point_kernel<P, true, true><<<ew_blocks(total), 256, 0, s>>>(a);
    else if (xr) point_kernel<P, true, false><<<ew_blocks(total), 256, 0, s>>>(a);
    else if (yr) point_kernel<P, false, true><<<ew_blocks(total), 256, 0, s>>>(a);
    else point_kernel<P, false, false><<<ew_blocks(total), 256, 0, s>>>(a);
  } else {
    point_kernel<P, false, false><<<ew_blocks(total), 256, 0, s>>>(a);
  }
  SMAT_CUDA(cudaGetLastError());
}

void launch_point(int dt, const PointArgs& a, cudaStream_t s) {
  const bool xr = a.x && dt_complex(dt) && !dt_complex(a.x_dt);
  const bool yr = dt_complex(dt) && !dt_complex(a.y_dt);
  switch (dt) {
    case SMAT_F32: point_dispatch<float>(a, false, false, s); break;
    case SMAT_F64: point_dispatch<double>(a, false, false, s); break;
    case SMAT_C64: point_dispatch<float2>(a, xr, yr, s); break;
    case SMAT_C128: point_dispatch<double2>(a, xr, yr, s); break;
    case SMAT_I32: point_dispatch<int32_t>(a, false, false, s); break;
    case SMAT_I64: point_dispatch<long long>(a, false, false, s); break;
    default: throw Error(SMAT_BAD_DTYPE, "pointwise: bad dtype");
  }
}

// ------------------------------------------------------ gather / scatter ---
template <class P>
__global__ void gather_kernel(const IndexArgs a) {
  const int64_t total = a.nb * a.n;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += stride) {
    const int64_t c = e % a.inner, t = e / a.inner, r = t % a.n, o = t / a.n;
    const int64_t o2 = o % a.n2, o1 = o / a.n2;
    const int64_t src = a.idx[r];
    ((P*)a.y)[o1 * a.ys1 + o2 * a.ys2 + r * a.ysi + c] =
        ((const P*)a.x)[o1 * a.xs1 + o2 * a.xs2 + src * a.xsi + c];
  }
}

template <class P> __device__ __forceinline__ void atomic_add_p(P* p, P v) {
  if constexpr (IsCx<P>::value) {
    atomicAdd(&p->x, v.x);
    atomicAdd(&p->y, v.y);
  } else if constexpr (std::is_same<P, long long>::value) {
    atomicAdd((unsigned long long*)p, (unsigned long long)v);
  } else {
    atomicAdd(p, v);
  }
}

template <class P>
__global__ void scatter_kernel(const IndexArgs a) {
  const int64_t total = a.nb * a.n;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += stride) {
    const int64_t c = e % a.inner, t = e / a.inner, r = t % a.n, o = t / a.n;
    const int64_t o2 = o % a.n2, o1 = o / a.n2;
    const int64_t dst = a.idx[r];
    const P v = ((const P*)a.x)[o1 * a.xs1 + o2 * a.xs2 + r * a.xsi + c];
    P* y = &((P*)a.y)[o1 * a.ys1 + o2 * a.ys2 + dst * a.ysi + c];
    if (a.atomic) atomic_add_p(y, v);
    else *y = padd(*y, v);
  }
}

#define SMAT_DT_SWITCH(dt, FN, ...)                               \
  switch (dt) {                                                   \
    case SMAT_F32: FN<float>(__VA_ARGS__); break;                 \
    case SMAT_F64: FN<double>(__VA_ARGS__); break;                \
    case SMAT_C64: FN<float2>(__VA_ARGS__); break;                \
    case SMAT_C128: FN<double2>(__VA_ARGS__); break;              \
    case SMAT_I32: FN<int32_t>(__VA_ARGS__); break;               \
    case SMAT_I64: FN<long long>(__VA_ARGS__); break;             \
    default: throw Error(SMAT_BAD_DTYPE, "bad dtype");            \
  }

template <class P> static void gather_go(const IndexArgs& a, cudaStream_t s) {
  gather_kernel<P><<<ew_blocks(a.nb * a.n), 256, 0, s>>>(a);
}
template <class P> static void scatter_go(const IndexArgs& a, cudaStream_t s) {
  scatter_kernel<P><<<ew_blocks(a.nb * a.n), 256, 0, s>>>(a);
}
void launch_gather(int dt, const IndexArgs& a, cudaStream_t s) {
  if (a.nb * a.n == 0) return;
  SMAT_DT_SWITCH(dt, gather_go, a, s)
  SMAT_CUDA(cudaGetLastError());
}
void launch_scatter_add(int dt, const IndexArgs& a, cudaStream_t s) {
  if (a.nb * a.n == 0) return;
  SMAT_DT_SWITCH(dt, scatter_go, a, s)
  SMAT_CUDA(cudaGetLastError());
}

// ------------------------------------------------------------ CSR SpMM ----
template <class P>
__global__ void __launch_bounds__(256) csr_kernel(const CsrArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const P* val = (const P*)a.val;
  for (int64_t w = warp; w < a.rows * a.nb_outer; w += nwarps) {
    const int64_t i = w % a.rows, o = w / a.rows;
    const int64_t o2 = o % a.n2, o1 = o / a.n2;
    const P* xb = (const P*)a.x + o1 * a.xs1 + o2 * a.xs2;
    P* yr = (P*)a.y + o1 * a.ys1 + o2 * a.ys2 + i * a.ysi;
    const int64_t k0 = a.ptr[i], k1 = a.ptr[i + 1];
    // two 32-column halves per pass share each (col, val) load; the nonzero
    // loop is unrolled by 4 so that up to 8 gathered x rows are in flight
    for (int64_t c = lane; c < a.inner; c += 64) {
      const bool two = c + 32 < a.inner;
      P acc0 = zval<P>(), acc1 = zval<P>();
      int64_t k = k0;
      for (; k + 4 <= k1; k += 4) {
        int64_t j[4];
        P v[4], x0[4], x1[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          j[q] = __ldg(&a.col[k + q]) * a.xsi;
          v[q] = val[k + q];
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          x0[q] = xb[j[q] + c];
          x1[q] = two ? xb[j[q] + c + 32] : zval<P>();
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          acc0 = padd(acc0, pmul(v[q], x0[q]));
          acc1 = padd(acc1, pmul(v[q], x1[q]));
        }
      }
      for (; k < k1; ++k) {
        const int64_t jj = a.col[k] * a.xsi;
        acc0 = padd(acc0, pmul(val[k], xb[jj + c]));
        if (two) acc1 = padd(acc1, pmul(val[k], xb[jj + c + 32]));
      }
      yr[c] = a.accumulate ? padd(yr[c], acc0) : acc0;
      if (two) yr[c + 32] = a.accumulate ? padd(yr[c + 32], acc1) : acc1;
    }
  }
}
// Narrow blocks (fewer than 32 columns, e.g. the solvers' single vectors):
// G = next_pow2(inner) lanes per row, 32 / G rows per warp, so a K = 1
// matrix-vector product runs one row per lane instead of one per warp.
template <class P>
__global__ void __launch_bounds__(256) csr_narrow_kernel(const CsrArgs a, int G) {
  const int lane = threadIdx.x & 31, sub = lane / G, gl = lane % G, per = 32 / G;
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int64_t total = a.rows * a.nb_outer;
  const P* val = (const P*)a.val;
  for (int64_t w = warp * per + sub; w < total; w += nwarps * per) {
    const int64_t i = w % a.rows, o = w / a.rows;
    const int64_t o2 = o % a.n2, o1 = o / a.n2;
    const P* xb = (const P*)a.x + o1 * a.xs1 + o2 * a.xs2;
    P* yr = (P*)a.y + o1 * a.ys1 + o2 * a.ys2 + i * a.ysi;
    const int64_t k0 = a.ptr[i], k1 = a.ptr[i + 1];
    for (int64_t c = gl; c < a.inner; c += G) {
      P acc = zval<P>();
      int64_t k = k0;
      for (; k + 4 <= k1; k += 4) {
        int64_t j[4];
        P v[4], xv[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          j[q] = __ldg(&a.col[k + q]) * a.xsi;
          v[q] = val[k + q];
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) xv[q] = xb[j[q] + c];
#pragma unroll
        for (int q = 0; q < 4; ++q) acc = padd(acc, pmul(v[q], xv[q]));
      }
      for (; k < k1; ++k) acc = padd(acc, pmul(val[k], xb[a.col[k] * a.xsi + c]));
      yr[c] = a.accumulate ? padd(yr[c], acc) : acc;
    }
  }
}

template <class P> static void csr_go(const CsrArgs& a, cudaStream_t s) {
  if (a.inner < 32) {
    int G = 1;
    while (G < a.inner) G <<= 1;
    const int64_t warps = (a.rows * a.nb_outer + (32 / G) - 1) / (32 / G);
    int64_t b = (warps + 7) / 8;
    if (b > 148 * 32) b = 148 * 32;
    csr_narrow_kernel<P><<<unsigned(b < 1 ? 1 : b), 256, 0, s>>>(a, G);
    return;
  }
  int64_t warps = a.rows * a.nb_outer;
  int64_t b = (warps + 7) / 8;
  if (b > 148 * 32) b = 148 * 32;
  csr_kernel<P><<<unsigned(b < 1 ? 1 : b), 256, 0, s>>>(a);
}
void launch_csr(int dt, const CsrArgs& a, cudaStream_t s) {
  if (a.rows * a.nb_outer == 0 || a.inner == 0) return;
  SMAT_DT_SWITCH(dt, csr_go, a, s)
  SMAT_CUDA(cudaGetLastError());
}

// ----------------------------------------------------------------- GEMM ----
// 64x64 output tile per CTA (256 threads, 4x4 per thread), K in chunks of 16
// through shared memory; optional split-K with atomic accumulation for the
// tall-skinny reductions of LowRank (V^H X with k ~ 1e6, m ~ 32).
constexpr int GBM = 64, GBN = 64, GBK = 16;

template <class P>
__global__ void __launch_bounds__(256) gemm_kernel(const GemmArgs a, int64_t k_chunk, int atomic_out) {
  __shared__ P As[GBK][GBM + 1];
  __shared__ P Xs[GBK][GBN + 1];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int64_t m0 = int64_t(blockIdx.y) * GBM;
  // blockIdx.x enumerates (batch, column tile)
  const int64_t ntile = (a.inner + GBN - 1) / GBN;
  const int64_t o = blockIdx.x / ntile;
  const int64_t n0 = (blockIdx.x % ntile) * GBN;
  const int64_t o2 = o % a.n2, o1 = o / a.n2;
  const P* X = (const P*)a.x + o1 * a.xs1 + o2 * a.xs2;
  P* Y = (P*)a.y + o1 * a.ys1 + o2 * a.ys2;
  const P* A = (const P*)a.A;
  const int64_t kbeg = int64_t(blockIdx.z) * k_chunk;
  const int64_t kend = min(a.k, kbeg + k_chunk);
  P acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) acc[i][jj] = zval<P>();
  for (int64_t k0 = kbeg; k0 < kend; k0 += GBK) {
    for (int l = threadIdx.x; l < GBK * GBM; l += 256) {
      const int kk = l / GBM, mm = l % GBM;
      const int64_t gk = k0 + kk, gm = m0 + mm;
      P v = zval<P>();
      if (gk < kend && gm < a.m) v = a.adj ? pconj(A[gk * a.lda + gm]) : A[gm * a.lda + gk];
      As[kk][mm] = v;
    }
    for (int l = threadIdx.x; l < GBK * GBN; l += 256) {
      const int kk = l / GBN, nn = l % GBN;
      const int64_t gk = k0 + kk, gn = n0 + nn;
      Xs[kk][nn] = (gk < kend && gn < a.inner) ? X[gk * a.xsi + gn] : zval<P>();
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < GBK; ++kk) {
      P av[4], xv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) xv[jj] = Xs[kk][tx + 16 * jj];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) acc[i][jj] = padd(acc[i][jj], pmul(av[i], xv[jj]));
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t gm = m0 + ty + 16 * i;
    if (gm >= a.m) continue;
    P rs = zval<P>();
    bool has_rs = a.rowscale != nullptr;
    if (has_rs) {
      rs = ((const P*)a.rowscale)[gm];
      if (a.rowscale_conj) rs = pconj(rs);
    }
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
      const int64_t gn = n0 + tx + 16 * jj;
      if (gn >= a.inner) continue;
      P v = acc[i][jj];
      if (has_rs) v = pmul(v, rs);
      P* yp = &Y[gm * a.ysi + gn];
      if (atomic_out) atomic_add_p(yp, v);
      else *yp = a.accumulate ? padd(*yp, v) : v;
    }
  }
}

template <class P> static int gemm_go(const GemmArgs& a, int device, cudaStream_t s, bool dry) {
  const int64_t ntile = (a.inner + GBN - 1) / GBN;
  const int64_t mt = (a.m + GBM - 1) / GBM;
  const int64_t nbt = a.n1 * a.n2 * ntile;
  // split K when the output grid cannot fill the machine
  const int64_t want = int64_t(num_sms(device)) * 4;
  int64_t splits = 1;
  if (nbt * mt < want && a.k > 4 * GBK) {
    splits = (want + nbt * mt - 1) / (nbt * mt);
    const int64_t max_split = (a.k + 255) / 256;
    if (splits > max_split) splits = max_split;
    if (splits > 65535) splits = 65535;
    if (splits < 1) splits = 1;
  }
  int64_t k_chunk = (a.k + splits - 1) / splits;
  k_chunk = ((k_chunk + GBK - 1) / GBK) * GBK;
  splits = (a.k + k_chunk - 1) / k_chunk;
  if (splits < 1) splits = 1;
  SMAT_CHECK(nbt < (int64_t(1) << 31) && mt < 65536, SMAT_UNSUPPORTED, "gemm grid too large");
  const int atomic_out = splits > 1;
  if (dry) return (atomic_out && !a.accumulate) ? 2 : 1;
  if (atomic_out && !a.accumulate) {
    // zero the output view first
    PointArgs z;
    z.y = a.y;
    z.y_dt = -1;
    z.ys1 = a.ys1; z.ys2 = a.ys2; z.ysi = a.ysi;
    z.n2 = a.n2; z.inner = a.inner; z.nb = a.n1 * a.n2 * a.inner; z.n = a.m;
    point_dispatch<P>(z, false, false, s);
  }
  const dim3 grid_dims{unsigned(nbt), unsigned(mt), unsigned(splits)};
  gemm_kernel<P><<<grid_dims, 256, 0, s>>>(a, k_chunk, atomic_out);
  SMAT_CUDA(cudaGetLastError());
  return (atomic_out && !a.accumulate) ? 2 : 1;
}

int launch_gemm(int dt, const GemmArgs& a, int device, cudaStream_t s, bool dry) {
  if (a.m == 0 || a.inner == 0 || a.n1 * a.n2 == 0) return 0;
  switch (dt) {
    case SMAT_F32: return gemm_go<float>(a, device, s, dry);
    case SMAT_F64: return gemm_go<double>(a, device, s, dry);
    case SMAT_C64: return gemm_go<float2>(a, device, s, dry);
    case SMAT_C128: return gemm_go<double2>(a, device, s, dry);
    default: throw Error(SMAT_BAD_DTYPE, "gemm: unsupported dtype");
  }
}

}  // namespace smat
