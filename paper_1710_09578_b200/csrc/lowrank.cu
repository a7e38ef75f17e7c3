// lowrank.cu — rank-r contraction / expansion kernels of LowRank = U diag(s) V^H.
//
// The reference expresses the C5 low-rank term as Product(Dense(U), Dense(V^H))
// (two OpenBLAS matmuls, leaves.py:40-46).  On the device both halves are
// tall-skinny (rows ~ 1e6, r = 32, K = 128):
//   contract  W = F^H X : a reduction over all rows -> CTAs own row slabs,
//             accumulate a private 32 x 128 tile in registers and add it to W
//             with one atomic per output per CTA;
//   expand    Y (=|+=) G diag(s) W : W' = diag(s) W lives in shared memory,
//             CTAs stream 32-row chunks of G and write Y with coalesced rows.
// Both are FP64-FMA bound for complex128 (8 flops per complex MAC); register
// tiles of 4 x 4 outputs per thread keep shared-memory traffic at 1 load per
// 8 FMAs.
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
}  // namespace

constexpr int LR_CT = 128;  // columns per CTA tile
constexpr int LR_RC = 16;   // rows per shared chunk (contract)
constexpr int LR_RE = 32;   // rows per chunk (expand)

template <class P>
__global__ void __launch_bounds__(256) lr_contract_kernel(const LowRankArgs a, int64_t rows_per_cta) {
  __shared__ P xs[LR_RC][LR_CT + 1];
  __shared__ P fs[LR_RC][32 + 1];
  const int tid = threadIdx.x, tx = tid % 32, ty = tid / 32;
  const int64_t c0 = int64_t(blockIdx.y) * LR_CT;
  const int64_t r0 = int64_t(blockIdx.x) * rows_per_cta;
  const int64_t r1 = min(a.rows, r0 + rows_per_cta);
  const P* X = (const P*)a.x;
  const P* F = (const P*)a.F;
  P acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = lr_zero<P>();
  for (int64_t rr = r0; rr < r1; rr += LR_RC) {
    for (int l = tid; l < LR_RC * LR_CT; l += 256) {
      const int k = l / LR_CT, c = l % LR_CT;
      const int64_t row = rr + k, col = c0 + c;
      xs[k][c] = (row < r1 && col < a.K) ? X[row * a.ldx + col] : lr_zero<P>();
    }
    for (int l = tid; l < LR_RC * 32; l += 256) {
      const int k = l / 32, q = l % 32;
      const int64_t row = rr + k;
      fs[k][q] = (row < r1 && q < a.r) ? F[row * a.r + q] : lr_zero<P>();
    }
    __syncthreads();
#pragma unroll 4
    for (int k = 0; k < LR_RC; ++k) {
      P f[4], x[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) f[i] = fs[k][ty + 8 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) x[j] = xs[k][tx + 32 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) fma_cx(acc[i][j], f[i], x[j]);
    }
    __syncthreads();
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

template <class P>
__global__ void __launch_bounds__(256, 2) lr_expand_kernel(const LowRankArgs a, int64_t nchunks) {
  extern __shared__ __align__(16) unsigned char lr_smem[];
  P* ws = reinterpret_cast<P*>(lr_smem);           // [32][LR_CT + 1]  W' = diag(s) W
  P* gs = ws + 32 * (LR_CT + 1);                    // [LR_RE][33]      G rows chunk
  const int tid = threadIdx.x, tx = tid % 32, ty = tid / 32;
  const int64_t c0 = int64_t(blockIdx.y) * LR_CT;
  const P* W = (const P*)a.w;
  const P* G = (const P*)a.F;
  const P* S = (const P*)a.s;
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
    ws[q * (LR_CT + 1) + c] = v;
  }
  P* Y = (P*)a.y;
  for (int64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    const int64_t r0 = ch * LR_RE;
    __syncthreads();  // ws ready / previous chunk's gs consumed
    for (int l = tid; l < LR_RE * 32; l += 256) {
      const int k = l / 32, q = l % 32;
      const int64_t row = r0 + k;
      gs[k * 33 + q] = (row < a.rows && q < a.r) ? G[row * a.r + q] : lr_zero<P>();
    }
    __syncthreads();
    P acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = lr_zero<P>();
    for (int q = 0; q < a.r; ++q) {
      P g[4], w[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) g[i] = gs[(ty + 8 * i) * 33 + q];
#pragma unroll
      for (int j = 0; j < 4; ++j) w[j] = ws[q * (LR_CT + 1) + tx + 32 * j];
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
        P* yp = &Y[row * a.ldy + col];
        *yp = a.accumulate ? *yp + acc[i][j] : acc[i][j];
      }
    }
  }
}

template <class P>
static int contract_go(const LowRankArgs& a, int device, cudaStream_t s, bool dry) {
  if (dry) return 2;
  SMAT_CHECK(a.r >= 1 && a.r <= 32, SMAT_UNSUPPORTED, "lowrank contract: rank must be <= 32");
  SMAT_CUDA(cudaMemsetAsync(a.w, 0, size_t(a.r * a.K) * sizeof(P), s));
  const int64_t ctiles = (a.K + LR_CT - 1) / LR_CT;
  const int64_t want = int64_t(num_sms(device)) * 8 / ctiles + 1;
  int64_t rows_per = (a.rows + want - 1) / want;
  rows_per = ((rows_per + LR_RC - 1) / LR_RC) * LR_RC;
  if (rows_per < LR_RC) rows_per = LR_RC;
  const int64_t gx = (a.rows + rows_per - 1) / rows_per;
  const dim3 grid_dims{unsigned(gx), unsigned(ctiles), 1u};
  lr_contract_kernel<P><<<grid_dims, 256, 0, s>>>(a, rows_per);
  SMAT_CUDA(cudaGetLastError());
  return 2;
}

template <class P>
static int expand_go(const LowRankArgs& a, int device, cudaStream_t s, bool dry) {
  if (dry) return 1;
  SMAT_CHECK(a.r >= 1 && a.r <= 32, SMAT_UNSUPPORTED, "lowrank expand: rank must be <= 32");
  const int64_t ctiles = (a.K + LR_CT - 1) / LR_CT;
  const int64_t nchunks = (a.rows + LR_RE - 1) / LR_RE;
  int64_t gx = int64_t(num_sms(device)) * 2 / ctiles + 1;
  if (gx > nchunks) gx = nchunks;
  const size_t smem = (size_t(32) * (LR_CT + 1) + size_t(LR_RE) * 33) * sizeof(P);
  static bool attr_set[2] = {false, false};
  const int slot = sizeof(P) == 16 ? 1 : 0;
  if (!attr_set[slot]) {
    SMAT_CUDA(cudaFuncSetAttribute(lr_expand_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    attr_set[slot] = true;
  }
  const dim3 grid_dims{unsigned(gx), unsigned(ctiles), 1u};
  lr_expand_kernel<P><<<grid_dims, 256, smem, s>>>(a, nchunks);
  SMAT_CUDA(cudaGetLastError());
  return 1;
}

int launch_lowrank_contract(int dt, const LowRankArgs& a, int device, cudaStream_t s, bool dry) {
  if (dt == SMAT_C128) return contract_go<double2>(a, device, s, dry);
  if (dt == SMAT_C64) return contract_go<float2>(a, device, s, dry);
  throw Error(SMAT_UNSUPPORTED, "lowrank kernels: complex plans only");
}
int launch_lowrank_expand(int dt, const LowRankArgs& a, int device, cudaStream_t s, bool dry) {
  if (dt == SMAT_C128) return expand_go<double2>(a, device, s, dry);
  if (dt == SMAT_C64) return expand_go<float2>(a, device, s, dry);
  throw Error(SMAT_UNSUPPORTED, "lowrank kernels: complex plans only");
}

}  // namespace smat
