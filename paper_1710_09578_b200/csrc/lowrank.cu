// lowrank.cu — rank-r contraction / expansion kernels of LowRank = U diag(s) V^H.
//
// The reference expresses the C5 low-rank term as Product(Dense(U), Dense(V^H))
// (two OpenBLAS matmuls, leaves.py:40-46).  On the device both halves are
// tall-skinny (rows ~ 1e6, r = 32, K = 128) and FP64-FMA bound for complex128
// (4 DFMA per complex MAC):
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

// physical row of logical row r (LowRankArgs::rm_n1); chunks start on
// multiples of 32 rows, so rows r0..r0+31 of a chunk stay contiguous
__device__ __forceinline__ int64_t lr_phys(const LowRankArgs& a, int64_t r) {
  if (a.rm_n1 == 0) return r;
  const int64_t n1 = r % a.rm_n1, k2 = r / a.rm_n1;
  return ((n1 >> 6) * a.rm_n2b + k2) * 64 + (n1 & 63);
}

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
    const int64_t prr = lr_phys(a, rr);  // (a chunk is contiguous in either layout)
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
    const int64_t pr0 = lr_phys(a, r0);  // (a 32-row chunk is contiguous in either layout)
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

// ============================================ complex128 on FP64 tensor cores ====
// Both halves as real GEMMs over the interleaved (re, im) layouts, on DMMA
// m8n8k4 tiles (fragments: A[l/4][l%4], B[l%4][l/4], C[l/4][2(l%4) + {0,1}]
// for lane l); every warp owns a 32 x 32 block of C (4 x 4 tiles).
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// expand: C (rows x 2K real) = A (rows x 2r: G as real) * B (2r x 2K) with
// B[2q+p][2c+b] = (b == 0 ? (p == 0 ? Re : -Im) : (p == 0 ? Im : Re)) W'[q][c]:
// C[row][2c] = Re(G W')[row][c], C[row][2c+1] = Im — i.e. Y itself, interleaved.
constexpr int DX_R = 64;    // rows per chunk (2 warp rows of 32)
constexpr int DX_K = 64;    // 2r, rank padded to 32
constexpr int DX_N = 256;   // real columns per CTA (128 complex), in two halves of 128
constexpr int DX_PK = 68;   // padded k stride of the shared operand tiles (doubles)

__global__ void __launch_bounds__(256, 1) lr_expand_dmma_kernel(const LowRankArgs a, int64_t nchunks) {
  extern __shared__ __align__(16) unsigned char lr_smem[];
  double* Bs = reinterpret_cast<double*>(lr_smem);  // [DX_N][DX_PK]
  double* As = Bs + DX_N * DX_PK;                   // [2][DX_R][DX_PK]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 2, wn = warp & 3;
  const int64_t cc0 = int64_t(blockIdx.y) * (DX_N / 2);
  const double2* W = (const double2*)a.w;
  const double2* G = (const double2*)a.F;
  const double2* S = (const double2*)a.s;
  double2* Y = (double2*)a.y;
  auto issue = [&](int64_t ch, int buf) {
    const int64_t rr = ch * DX_R;
    double* ad = As + buf * DX_R * DX_PK;
    for (int l = tid; l < DX_R * 32; l += 256) {
      const int m = l >> 5, q = l & 31;
      const int64_t row = rr + m;
      const bool ok = row < a.rows && q < a.r;
      cp_async<16>(&ad[m * DX_PK + 2 * q], ok ? (const void*)&G[row * a.r + q] : (const void*)G, ok);
    }
    cp_commit();
  };
  int64_t ch = blockIdx.x;
  if (ch < nchunks) issue(ch, 0);
  for (int e = tid; e < DX_N * DX_K; e += 256) {
    const int n = e / DX_K, k = e % DX_K;
    const int q = k >> 1, p = k & 1, c = n >> 1, b = n & 1;
    double v = 0.0;
    if (q < a.r && cc0 + c < a.K) {
      double2 w = W[q * a.K + cc0 + c];
      if (S) {
        double2 sv = S[q];
        if (a.s_conj) sv.y = -sv.y;
        w = cmul(sv, w);
      }
      v = b == 0 ? (p == 0 ? w.x : -w.y) : (p == 0 ? w.y : w.x);
    }
    Bs[n * DX_PK + k] = v;
  }
  for (int it = 0; ch < nchunks; ch += gridDim.x, ++it) {
    if (ch + gridDim.x < nchunks) {
      issue(ch + gridDim.x, (it + 1) & 1);
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();  // this chunk's G rows (and, first time, B') are visible
    const double* A = As + (it & 1) * DX_R * DX_PK;
    const int64_t r0 = ch * DX_R;
#pragma unroll 1
    for (int h = 0; h < 2; ++h) {
      double2 yv[4][4];
      if (a.accumulate) {
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
          for (int ni = 0; ni < 4; ++ni) {
            const int64_t row = r0 + wm * 32 + mi * 8 + (lane >> 2);
            const int64_t col = cc0 + h * 64 + wn * 16 + ni * 4 + (lane & 3);
            yv[mi][ni] = (row < a.rows && col < a.K) ? Y[row * a.ldy + col] : make_double2(0.0, 0.0);
          }
      }
      double acc[4][4][2];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
#pragma unroll 4
      for (int kk = 0; kk < DX_K / 4; ++kk) {
        const int k = kk * 4 + (lane & 3);
        double af[4], bf[4];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) af[mi] = A[(wm * 32 + mi * 8 + (lane >> 2)) * DX_PK + k];
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) bf[ni] = Bs[(h * 128 + wn * 32 + ni * 8 + (lane >> 2)) * DX_PK + k];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
          for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
      }
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) {
          const int64_t row = r0 + wm * 32 + mi * 8 + (lane >> 2);
          const int64_t col = cc0 + h * 64 + wn * 16 + ni * 4 + (lane & 3);
          if (row < a.rows && col < a.K) {
            double2 v = make_double2(acc[mi][ni][0], acc[mi][ni][1]);
            if (a.accumulate) v = make_double2(v.x + yv[mi][ni].x, v.y + yv[mi][ni].y);
            Y[row * a.ldy + col] = v;
          }
        }
    }
    __syncthreads();  // buffer (it & 1) is refilled two chunks later
  }
}

// contract: C (2r x K) = A (2r x 2R) * B (2R x K) over the chunk's R rows,
// A[2q+a][2row+p] = (a == 0 ? (p == 0 ? Re : Im) : (p == 0 ? -Im : Re)) F[row][q]
// (the block form of conj(F)), B[2row+p][c] = X[row][c].{re, im};
// C[2q][c] = Re W[q][c], C[2q+1][c] = Im W[q][c].  Row slabs per CTA, the
// partial W added with one atomic per element and CTA.
constexpr int DC_R = 32;    // rows per chunk (k' = 64)
constexpr int DC_XP = 132;  // padded row stride of the X chunk (complex)
constexpr int DC_FP = 33;   // padded row stride of the F chunk (complex)

__global__ void __launch_bounds__(256, 1) lr_contract_dmma_kernel(const LowRankArgs a, int64_t rows_per_cta) {
  extern __shared__ __align__(16) unsigned char lr_smem[];
  double2* Xs = reinterpret_cast<double2*>(lr_smem);  // [2][DC_R][DC_XP]
  double2* Fs = Xs + 2 * DC_R * DC_XP;                // [2][DC_R][DC_FP]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 2, wn = warp & 3;
  const int64_t c0 = int64_t(blockIdx.y) * 128;
  const int64_t r0 = int64_t(blockIdx.x) * rows_per_cta;
  const int64_t r1 = min(a.rows, r0 + rows_per_cta);
  const double2* X = (const double2*)a.x;
  const double2* F = (const double2*)a.F;
  const int nch = r1 > r0 ? int((r1 - r0 + DC_R - 1) / DC_R) : 0;
  auto issue = [&](int ch) {
    const int64_t rr = r0 + int64_t(ch) * DC_R;
    double2* xd = Xs + (ch & 1) * DC_R * DC_XP;
    double2* fd = Fs + (ch & 1) * DC_R * DC_FP;
    for (int l = tid; l < DC_R * 128; l += 256) {
      const int k = l >> 7, c = l & 127;
      const int64_t row = rr + k, col = c0 + c;
      const bool ok = row < r1 && col < a.K;
      cp_async<16>(&xd[k * DC_XP + c], ok ? (const void*)&X[row * a.ldx + col] : (const void*)X, ok);
    }
    for (int l = tid; l < DC_R * 32; l += 256) {
      const int k = l >> 5, q = l & 31;
      const int64_t row = rr + k;
      const bool ok = row < r1 && q < a.r;
      cp_async<16>(&fd[k * DC_FP + q], ok ? (const void*)&F[row * a.r + q] : (const void*)F, ok);
    }
    cp_commit();
  };
  double acc[4][4][2];
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
  if (nch > 0) issue(0);
  for (int ch = 0; ch < nch; ++ch) {
    if (ch + 1 < nch) {
      issue(ch + 1);
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    const double2* xc = Xs + (ch & 1) * DC_R * DC_XP;
    const double2* fc = Fs + (ch & 1) * DC_R * DC_FP;
#pragma unroll 4
    for (int kk = 0; kk < 2 * DC_R / 4; ++kk) {
      const int kp = kk * 4 + (lane & 3);  // k' = 2*row + p
      const int row = kp >> 1, p = kp & 1;
      double af[4], bf[4];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) {
        const int m = wm * 32 + mi * 8 + (lane >> 2);  // m = 2q + a
        const double2 fv = fc[row * DC_FP + (m >> 1)];
        af[mi] = (m & 1) == 0 ? (p == 0 ? fv.x : fv.y) : (p == 0 ? -fv.y : fv.x);
      }
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) {
        const double* xr = reinterpret_cast<const double*>(&xc[row * DC_XP + wn * 32 + ni * 8 + (lane >> 2)]);
        bf[ni] = xr[p];
      }
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
    }
    __syncthreads();  // buffer (ch & 1) is refilled by issue(ch + 2)
  }
  double* Wd = (double*)a.w;
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int m = wm * 32 + mi * 8 + (lane >> 2);
        const int q = m >> 1, part = m & 1;
        const int64_t col = c0 + wn * 32 + ni * 8 + 2 * (lane & 3) + e;
        if (q < a.r && col < a.K) atomicAdd(&Wd[2 * (q * a.K + col) + part], acc[mi][ni][e]);
      }
}

// (dynamic shared-memory opt-in, once per kernel and device)
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

// DMMA variants are opt-in (SMAT_LR_DMMA=1): with one 8-warp CTA per SM they
// measured slower than the DFMA kernels (C5: contract 2.22 vs 1.44 ms, expand
// 1.77 vs 1.55 ms per launch) — the tensor-core pipe needs more warps in flight
// than the shared-memory footprint of these tiles allows.
static bool lr_dmma() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("SMAT_LR_DMMA");
    on = (e && e[0] == '1') ? 1 : 0;
  }
  return on == 1;
}

static int contract_dmma_go(const LowRankArgs& a, int device, cudaStream_t s, bool dry) {
  if (dry) return 2;
  SMAT_CHECK(a.r >= 1 && a.r <= 32, SMAT_UNSUPPORTED, "lowrank contract: rank must be <= 32");
  SMAT_CUDA(cudaMemsetAsync(a.w, 0, size_t(a.r * a.K) * sizeof(double2), s));
  const int64_t ctiles = (a.K + 127) / 128;
  const int64_t want = int64_t(num_sms(device)) / ctiles + 1;
  int64_t rows_per = (a.rows + want - 1) / want;
  rows_per = ((rows_per + DC_R - 1) / DC_R) * DC_R;
  if (rows_per < DC_R) rows_per = DC_R;
  const int64_t gx = (a.rows + rows_per - 1) / rows_per;
  const size_t smem = size_t(2) * DC_R * (DC_XP + DC_FP) * sizeof(double2);
  static uint64_t done = 0;
  lr_set_smem(lr_contract_dmma_kernel, smem, done);
  const dim3 grid_dims{unsigned(gx), unsigned(ctiles), 1u};
  lr_contract_dmma_kernel<<<grid_dims, 256, smem, s>>>(a, rows_per);
  SMAT_CUDA(cudaGetLastError());
  return 2;
}

static int expand_dmma_go(const LowRankArgs& a, int device, cudaStream_t s, bool dry) {
  if (dry) return 1;
  SMAT_CHECK(a.r >= 1 && a.r <= 32, SMAT_UNSUPPORTED, "lowrank expand: rank must be <= 32");
  const int64_t ctiles = (a.K + DX_N / 2 - 1) / (DX_N / 2);
  const int64_t nchunks = (a.rows + DX_R - 1) / DX_R;
  int64_t gx = int64_t(num_sms(device)) / ctiles;
  if (gx < 1) gx = 1;
  if (gx > nchunks) gx = nchunks;
  const size_t smem = (size_t(DX_N) * DX_PK + size_t(2) * DX_R * DX_PK) * sizeof(double);
  static uint64_t done = 0;
  lr_set_smem(lr_expand_dmma_kernel, smem, done);
  const dim3 grid_dims{unsigned(gx), unsigned(ctiles), 1u};
  lr_expand_dmma_kernel<<<grid_dims, 256, smem, s>>>(a, nchunks);
  SMAT_CUDA(cudaGetLastError());
  return 1;
}

int launch_lowrank_contract(int dt, const LowRankArgs& a, int device, cudaStream_t s, bool dry) {
  if (dt == SMAT_C128 && lr_dmma() && !a.rm_n1) return contract_dmma_go(a, device, s, dry);
  if (dt == SMAT_C128) return contract_go<double2>(a, device, s, dry);
  if (dt == SMAT_C64) return contract_go<float2>(a, device, s, dry);
  throw Error(SMAT_UNSUPPORTED, "lowrank kernels: complex plans only");
}
int launch_lowrank_expand(int dt, const LowRankArgs& a, int device, cudaStream_t s, bool dry) {
  if (dt == SMAT_C128 && lr_dmma() && !a.rm_n1) return expand_dmma_go(a, device, s, dry);
  if (dt == SMAT_C128) return expand_go<double2>(a, device, s, dry);
  if (dt == SMAT_C64) return expand_go<float2>(a, device, s, dry);
  throw Error(SMAT_UNSUPPORTED, "lowrank kernels: complex plans only");
}

}  // namespace smat
