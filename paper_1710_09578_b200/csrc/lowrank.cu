// lowrank.cu — rank-r contraction / expansion kernels of a complex64
// LowRank = U diag(s) V^H (complex128 terms run on the FP64 tensor cores,
// wlr.cu).
//
// The reference expresses a low-rank term as Product(Dense(U), Dense(V^H))
// (two OpenBLAS matmuls, leaves.py:40-46).  On the device both halves are
// tall-skinny (rows >> r <= 32) and FMA bound:
//   contract  W = F^H X : a reduction over all rows -> CTAs own row slabs and
//             keep a private r x 128 tile in registers (4 x 4 complex outputs
//             per thread), adding it to W with one atomic per output per CTA;
//   expand    Y (=|+=) G diag(s) W : W' = diag(s) W lives in shared memory,
//             persistent CTAs stream 32-row chunks of G and write Y rows.
// All operand traffic is staged through shared memory with cp.async double
// buffering (the next chunk lands while the current one is multiplied), and
// the accumulate read of Y is issued before the chunk's multiply, so no warp
// waits on HBM latency inside the FMA loop.
#include <type_traits>

#include "misc_kernels.cuh"

namespace smat {

namespace {
template <class P> struct LRT;
template <> struct LRT<float2> { using R = float; };
template <> struct LRT<double2> { using R = double; };

template <class P> __device__ __forceinline__ P lr_zero() {
  using R = typename LRT<P>::R;
  return mk(R(0), R(0));
}
// acc += conj(f) * x
template <class P> __device__ __forceinline__ void fma_cx(P& acc, P f, P x) {
  acc.x = fma(f.x, x.x, fma(f.y, x.y, acc.x));
  acc.y = fma(f.x, x.y, fma(-f.y, x.x, acc.y));
}
// acc += g * w
template <class P> __device__ __forceinline__ void fma_nx(P& acc, P g, P w) {
  acc.x = fma(g.x, w.x, fma(-g.y, w.y, acc.x));
  acc.y = fma(g.x, w.y, fma(g.y, w.x, acc.y));
}

// 16-byte (or 8-byte) global -> shared async copy; src_bytes = 0 zero-fills.
template <int B>
__device__ __forceinline__ void cp_async(void* dst, const void* src, bool valid) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
  const int n = valid ? B : 0;
  if constexpr (B == 16) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(n) : "memory");
  } else {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(n) : "memory");
  }
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
}  // namespace

constexpr int LR_CT = 128;  // columns per CTA tile
constexpr int LR_RC = 16;   // rows per contract chunk
constexpr int LR_RE = 32;   // rows per expand chunk

// ---------------------------------------------------------------- contract --
template <class P>
__global__ void __launch_bounds__(256, 2) lr_contract_kernel(const LowRankArgs a, int64_t rows_per_cta) {
  extern __shared__ __align__(16) unsigned char lr_smem[];
  P* xs = reinterpret_cast<P*>(lr_smem);        // [2][LR_RC][LR_CT]
  P* fs = xs + 2 * LR_RC * LR_CT;               // [2][LR_RC][32]
  const int tid = threadIdx.x, tx = tid % 32, ty = tid / 32;
  const int64_t c0 = int64_t(blockIdx.y) * LR_CT;
  const int64_t r0 = int64_t(blockIdx.x) * rows_per_cta;
  const int64_t r1 = min(a.rows, r0 + rows_per_cta);
  const P* X = (const P*)a.x;
  const P* F = (const P*)a.F;
  const int nch = r1 > r0 ? int((r1 - r0 + LR_RC - 1) / LR_RC) : 0;
  auto issue = [&](int ch) {
    const int64_t rr = r0 + int64_t(ch) * LR_RC;
    const int64_t prr = rr;
    P* xd = xs + (ch & 1) * LR_RC * LR_CT;
    P* fd = fs + (ch & 1) * LR_RC * 32;
    for (int l = tid; l < LR_RC * LR_CT; l += 256) {
      const int k = l / LR_CT, c = l % LR_CT;
      const int64_t row = rr + k, col = c0 + c;
      const bool ok = row < r1 && col < a.K;
      cp_async<sizeof(P)>(&xd[l], ok ? &X[(prr + k) * a.ldx + col] : X, ok);
    }
    for (int l = tid; l < LR_RC * 32; l += 256) {
      const int k = l / 32, q = l % 32;
      const int64_t row = rr + k;
      const bool ok = row < r1 && q < a.r;
      cp_async<sizeof(P)>(&fd[l], ok ? &F[row * a.r + q] : F, ok);
    }
    cp_commit();
  };
  P acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = lr_zero<P>();
  if (nch > 0) issue(0);
  for (int ch = 0; ch < nch; ++ch) {
    if (ch + 1 < nch) {
      issue(ch + 1);
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    const P* xc = xs + (ch & 1) * LR_RC * LR_CT;
    const P* fc = fs + (ch & 1) * LR_RC * 32;
#pragma unroll 4
    for (int k = 0; k < LR_RC; ++k) {
      P f[4], x[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) f[i] = fc[k * 32 + ty + 8 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) x[j] = xc[k * LR_CT + tx + 32 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) fma_cx(acc[i][j], f[i], x[j]);
    }
    __syncthreads();  // buffer (ch & 1) is refilled by issue(ch + 2)
  }
  using R = typename LRT<P>::R;
  R* W = (R*)a.w;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int q = ty + 8 * i;
    if (q >= a.r) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t col = c0 + tx + 32 * j;
      if (col >= a.K) continue;
      atomicAdd(&W[2 * (q * a.K + col)], acc[i][j].x);
      atomicAdd(&W[2 * (q * a.K + col) + 1], acc[i][j].y);
    }
  }
}

// ------------------------------------------------------------------ expand --
template <class P>
__global__ void __launch_bounds__(256, 1) lr_expand_kernel(const LowRankArgs a, int64_t nchunks) {
  extern __shared__ __align__(16) unsigned char lr_smem[];
  P* ws = reinterpret_cast<P*>(lr_smem);  // [32][LR_CT]       W' = diag(s) W
  P* gs = ws + 32 * LR_CT;                // [2][LR_RE][32]    G row chunks
  const int tid = threadIdx.x, tx = tid % 32, ty = tid / 32;
  const int64_t c0 = int64_t(blockIdx.y) * LR_CT;
  const P* W = (const P*)a.w;
  const P* G = (const P*)a.F;
  const P* S = (const P*)a.s;
  P* Y = (P*)a.y;
  auto issue = [&](int64_t ch, int buf) {
    const int64_t rr = ch * LR_RE;
    P* gd = gs + buf * LR_RE * 32;
    for (int l = tid; l < LR_RE * 32; l += 256) {
      const int k = l / 32, q = l % 32;
      const int64_t row = rr + k;
      const bool ok = row < a.rows && q < a.r;
      cp_async<sizeof(P)>(&gd[l], ok ? &G[row * a.r + q] : G, ok);
    }
    cp_commit();
  };
  int64_t ch = blockIdx.x;
  if (ch < nchunks) issue(ch, 0);
  for (int l = tid; l < 32 * LR_CT; l += 256) {
    const int q = l / LR_CT, c = l % LR_CT;
    P v = lr_zero<P>();
    if (q < a.r && c0 + c < a.K) {
      v = W[q * a.K + c0 + c];
      if (S) {
        P sv = S[q];
        if (a.s_conj) sv.y = -sv.y;
        v = cmul(sv, v);
      }
    }
    ws[l] = v;
  }
  for (int it = 0; ch < nchunks; ch += gridDim.x, ++it) {
    const int64_t r0 = ch * LR_RE;
    const int64_t pr0 = r0;
    // previous accumulate values of this chunk's outputs: in flight during the multiply
    P yv[4][4];
    if (a.accumulate) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int64_t row = r0 + ty + 8 * i;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int64_t col = c0 + tx + 32 * j;
          yv[i][j] = (row < a.rows && col < a.K) ? Y[(pr0 + ty + 8 * i) * a.ldy + col] : lr_zero<P>();
        }
      }
    }
    if (ch + gridDim.x < nchunks) {
      issue(ch + gridDim.x, (it + 1) & 1);
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();  // this chunk's G rows (and, first time, W') are visible
    const P* gc = gs + (it & 1) * LR_RE * 32;
    P acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = lr_zero<P>();
#pragma unroll 4
    for (int q = 0; q < 32; ++q) {
      P g[4], w[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) g[i] = gc[(ty + 8 * i) * 32 + q];
#pragma unroll
      for (int j = 0; j < 4; ++j) w[j] = ws[q * LR_CT + tx + 32 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) fma_nx(acc[i][j], g[i], w[j]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t row = r0 + ty + 8 * i;
      if (row >= a.rows) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t col = c0 + tx + 32 * j;
        if (col >= a.K) continue;
        Y[(pr0 + ty + 8 * i) * a.ldy + col] = a.accumulate ? yv[i][j] + acc[i][j] : acc[i][j];
      }
    }
    __syncthreads();  // buffer (it & 1) is refilled two chunks later
  }
}

template <class K>
static void lr_set_smem(K kern, size_t bytes, uint64_t& done_mask) {
  int dev = 0;
  SMAT_CUDA(cudaGetDevice(&dev));
  if (!(done_mask >> dev & 1)) {
    SMAT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
    done_mask |= uint64_t(1) << dev;
  }
}

template <class P>
static int contract_go(const LowRankArgs& a, int device, cudaStream_t s, bool dry) {
  if (dry) return 2;
  SMAT_CHECK(a.r >= 1 && a.r <= 32, SMAT_UNSUPPORTED, "lowrank contract: rank must be <= 32");
  SMAT_CUDA(cudaMemsetAsync(a.w, 0, size_t(a.r * a.K) * sizeof(P), s));
  const int64_t ctiles = (a.K + LR_CT - 1) / LR_CT;
  const int64_t want = int64_t(num_sms(device)) * 2 / ctiles + 1;
  int64_t rows_per = (a.rows + want - 1) / want;
  rows_per = ((rows_per + LR_RC - 1) / LR_RC) * LR_RC;
  if (rows_per < LR_RC) rows_per = LR_RC;
  const int64_t gx = (a.rows + rows_per - 1) / rows_per;
  const size_t smem = size_t(2) * LR_RC * (LR_CT + 32) * sizeof(P);
  static uint64_t done[2] = {0, 0};
  lr_set_smem(lr_contract_kernel<P>, smem, done[sizeof(P) == 16]);
  const dim3 grid_dims{unsigned(gx), unsigned(ctiles), 1u};
  lr_contract_kernel<P><<<grid_dims, 256, smem, s>>>(a, rows_per);
  SMAT_CUDA(cudaGetLastError());
  return 2;
}

template <class P>
static int expand_go(const LowRankArgs& a, int device, cudaStream_t s, bool dry) {
  if (dry) return 1;
  SMAT_CHECK(a.r >= 1 && a.r <= 32, SMAT_UNSUPPORTED, "lowrank expand: rank must be <= 32");
  const int64_t ctiles = (a.K + LR_CT - 1) / LR_CT;
  const int64_t nchunks = (a.rows + LR_RE - 1) / LR_RE;
  int64_t gx = int64_t(num_sms(device)) / ctiles;
  if (gx < 1) gx = 1;
  if (gx > nchunks) gx = nchunks;
  const size_t smem = (size_t(32) * LR_CT + size_t(2) * LR_RE * 32) * sizeof(P);
  static uint64_t done[2] = {0, 0};
  lr_set_smem(lr_expand_kernel<P>, smem, done[sizeof(P) == 16]);
  const dim3 grid_dims{unsigned(gx), unsigned(ctiles), 1u};
  lr_expand_kernel<P><<<grid_dims, 256, smem, s>>>(a, nchunks);
  SMAT_CUDA(cudaGetLastError());
  return 1;
}

int launch_lowrank_contract(int dt, const LowRankArgs& a, int device, cudaStream_t s, bool dry) {
  // (complex128 LowRank terms run on the FP64 tensor cores, wlr.cu)
  if (dt == SMAT_C64) return contract_go<float2>(a, device, s, dry);
  throw Error(SMAT_UNSUPPORTED, "lowrank kernels: complex64 plans only");
}
int launch_lowrank_expand(int dt, const LowRankArgs& a, int device, cudaStream_t s, bool dry) {
  if (dt == SMAT_C64) return expand_go<float2>(a, device, s, dry);
  throw Error(SMAT_UNSUPPORTED, "lowrank kernels: complex64 plans only");
}

}  // namespace smat
