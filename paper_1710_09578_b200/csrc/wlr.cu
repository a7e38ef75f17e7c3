// wlr.cu — fused Walsh-Hadamard + rank-r LowRank passes (complex128) on the
// FP64 tensor cores.
//
// The reference's low-rank term is two OpenBLAS matmuls, Product(Dense(U),
// Dense(V^H)) (leaves.py:40-46), and the padded Hadamard a Partial around the
// numpy fwht (composites.py:281-310, kernels.py:164-190).  For C5 both halves
// of the rank-32 product are tall-skinny (1e6 rows, K = 128 columns): the
// contraction W = V^H X reads every row of X, the expansion Y += U W' writes
// every row of Y.  A pass whose tile is "many rows x few columns" (the FFT /
// FWHT tiles) would have to re-read the factor rows once per column group
// (8x the data from L2), so the LowRank work lives in passes whose tile is
// 64 rows x ALL columns (two 64-column chunks), and the Hadamard splits so
// that two of its stages run in those passes too:
//
//   H_P = H_{2^9} (k2) (x) H_64 (b) (x) H_32 (a),  row r = a + 32 b + 2048 k2
//
//   forward   A1: x -> T1   H_32 over a + partials of V^H x (input rows)
//             A2: T1 -> T2  H_64 over b + U~ W' (output rows)
//   backward  A2: T2 -> T1  H_64 over b + partials of U~^H (input rows)
//             A1: T1 -> x   H_32 over a + V W'' (output rows)
//
// (U~ = H_{2^9} U / 512 in A2's row order: the remaining k2 stages are linear,
// so adding U~ W' before them adds U W' after them; plan.cu builds it.)
//
// Kernel: persistent, one 256-thread CTA per SM, every CTA on a fixed 64-column
// chunk; units of 64 unit-rows x 64 columns stream through a two-deep ring of
// shared-memory stages filled by 1-D bulk copies (cp.async.bulk, one per row,
// mbarrier completion) issued by warp 0 — the data rows plus the unit's 64
// factor rows.  Per unit: contraction on the FP64 tensor cores (mma.sync
// m8n8k4 f64; the complex product as three real products, Gauss), the
// Hadamard stages in shared memory (stride-1-first radix-8 / radix-4
// butterflies), the expansion (three real products into fragments, combined
// and added to the transformed rows), then coalesced 16-byte stores.
// Contraction partials stay in registers for the whole kernel and are
// written once per CTA; a finalize kernel sums them in a fixed order
// (deterministic, no atomics) and folds diag(s).
#include <algorithm>
#include <cstring>
#include <mutex>
#include <set>

#include "tma.cuh"
#include "wlr.cuh"

namespace smat {

namespace {

constexpr int TR = 64;              // unit rows
constexpr int KC = 64;              // columns per chunk
constexpr int RK = 32;              // padded rank
// shared-memory row pitches (bytes).  The tensor-core fragments read 16-byte
// entries of rows lane%4 (contraction: data and factor rows) or lane/4
// (expansion: factor rows); a pitch of 2 (mod 8) or 4 (mod 8) 16-byte units
// puts those rows on distinct bank groups.  The data tile is a tensor-map
// box of KCB = 66 columns (the two extra columns are never used), so it lands
// with that pitch; the factor rows are stored padded in global memory.
constexpr int KCB = KC + 2;
constexpr int DP = KCB * 16;        // 1056
constexpr int FPC = (RK + 2) * 16;  // 544, contraction
constexpr int FPE = (RK + 4) * 16;  // 576, expansion
constexpr int NTHR = 256;
// ring depth per CTA and CTAs per SM: one single-stage CTA per ~half SM, so
// that while one CTA waits for its tile or stores, the other multiplies
constexpr int NST = 1;
constexpr int MINB = 2;

template <bool EXP>
struct WlrGeom {
  static constexpr int FP = EXP ? FPE : FPC;
  static constexpr int DATA = TR * DP;
  static constexpr int STAGE = DATA + TR * FP;
  static constexpr int SMEM = NST * STAGE + 64;
};

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2,
                                            int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

template <int NW>
__device__ __forceinline__ int64_t wlr_phys(const WlrRows& m, int64_t g) {
  constexpr int LW = NW >= 64 ? 6 : NW >= 32 ? 5 : NW >= 16 ? 4 : NW >= 8 ? 3 : NW >= 4 ? 2 : NW >= 2 ? 1 : 0;
  const int64_t G = g >> LW, a = g & (NW - 1);
  return (G >> m.gsh) * m.g_hi + (G & ((int64_t(1) << m.gsh) - 1)) * m.g_lo + (a & ((int64_t(1) << m.ash) - 1)) * m.a_lo +
         (a >> m.ash) * m.a_hi;
}

__device__ __forceinline__ int ilog2_dev(int v) { return 31 - __clz(v); }

__device__ __forceinline__ double2 ld2(const unsigned char* p) { return *reinterpret_cast<const double2*>(p); }
__device__ __forceinline__ void st2(unsigned char* p, double2 v) { *reinterpret_cast<double2*>(p) = v; }

// In-register Walsh-Hadamard of R points, stride-1-first (kernels.py:181-189).
template <int R>
__device__ __forceinline__ void wht_reg(double2 (&v)[8]) {
#pragma unroll
  for (int h = 1; h < R; h <<= 1)
#pragma unroll
    for (int b = 0; b < R; b += 2 * h)
#pragma unroll
      for (int q = 0; q < h; ++q) {
        const double2 x = v[b + q], y = v[b + q + h];
        v[b + q] = make_double2(x.x + y.x, x.y + y.y);
        v[b + q + h] = make_double2(x.x - y.x, x.y - y.y);
      }
}

// One radix-R stage over the 64 rows of a unit, for column c: group j holds
// rows base(j) + k * S (k < R).  Stage 1 (S = 1): R = min(NW, 8) consecutive
// rows, base = R j.  Stage 2 (S = 8, NW > 8): R = NW / 8 rows 8 apart inside
// each NW-row group, base = NW (j / 8) + j % 8.
template <int R, int S, int NW>
__device__ __forceinline__ void wht_stage(unsigned char* dbuf, int c, int p) {
  constexpr int NG = TR / R;
#pragma unroll
  for (int j = p; j < NG; j += NTHR / KC) {
    const int b0 = S == 1 ? R * j : NW * (j / 8) + j % 8;
    double2 v[8];
#pragma unroll
    for (int k = 0; k < R; ++k) v[k] = ld2(dbuf + (b0 + k * S) * DP + c * 16);
    wht_reg<R>(v);
#pragma unroll
    for (int k = 0; k < R; ++k) st2(dbuf + (b0 + k * S) * DP + c * 16, v[k]);
  }
}

template <int NW, bool CON, bool EXP, bool IN, bool OUT>
__global__ void __launch_bounds__(NTHR, MINB)
    wlr_kernel(const __grid_constant__ CUtensorMap xmap, const WlrArgs a, const int nchunks, const int nunits) {
  using G = WlrGeom<EXP>;
  constexpr int FP = G::FP;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NST * G::STAGE);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ch = int(blockIdx.x) % nchunks;
  const int64_t c0 = int64_t(ch) * KC;
  const int kcv = int(min(int64_t(KC), a.K - c0));  // valid columns of this CTA's chunk
  const int r = int(a.r);
  const int gs = int(gridDim.x);
  double2* Y = reinterpret_cast<double2*>(a.y);
  const double2* F = reinterpret_cast<const double2*>(a.F);
  const int lgw = a.in.kind == WLR_IN_ROWS ? 0 : ilog2_dev(int(a.in.nwa));

  auto rows_valid = [&](int64_t lim, int64_t g0) -> int {
    const int64_t v = lim - g0;
    return v <= 0 ? 0 : v >= TR ? TR : int(v);
  };
  // one thread: the unit's input box (one tensor-map copy) and its factor
  // rows (one bulk copy of the padded rows) into stage s
  auto issue = [&](int u, int s) {
    const int64_t g0 = int64_t(u / nchunks) * TR;
    unsigned char* dbuf = smem + s * G::STAGE;
    unsigned char* fbuf = dbuf + G::DATA;
    const int rf = rows_valid(min(a.n_f, a.nrows), g0);
    const uint32_t fbytes = uint32_t(rf) * FP;
    mbar_arrive_expect_tx(&bars[s], (IN ? uint32_t(G::DATA) : 0u) + fbytes);
    if constexpr (IN) {
      const int cw = int(2 * c0);
      if (a.in.kind == WLR_IN_ROWS) {
        tma_load_2d(dbuf, &xmap, &bars[s], cw, int(g0));
      } else if (a.in.kind == WLR_IN_T1A) {
        const int T0 = int(g0 >> lgw);
        tma_load_4d(dbuf, &xmap, &bars[s], cw, 0, T0 & 63, T0 >> 6);
      } else {
        const int Tp = int(g0 >> 6);
        tma_load_5d(dbuf, &xmap, &bars[s], cw, 0, 0, Tp & int(a.in.nwa - 1), Tp >> lgw);
      }
    }
    if (rf) bulk_load(fbuf, F + g0 * (FP / 16), fbytes, &bars[s]);
  };

  if (tid == 0) {
    if constexpr (IN) tma_prefetch_desc(&xmap);
    for (int st = 0; st < NST; ++st) mbar_init(&bars[st], 1);
    fence_barrier_init();
    for (int st = 0; st < NST; ++st)
      if (int(blockIdx.x) + st * gs < nunits) issue(blockIdx.x + st * gs, st);
  }
  __syncthreads();

  // contraction partials: q-tile mt (rows 8mt.. of W), product p (Gauss), pair
  double acc[4][3][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int p = 0; p < 3; ++p) acc[i][p][0] = acc[i][p][1] = 0.0;
  // expansion: this lane's W' fragments for every k-step (q = 4ks + lane%4,
  // column 8*warp + lane/4 of the chunk)
  double wb[EXP ? 8 : 1][3];
  if constexpr (EXP) {
    const int64_t col = c0 + 8 * warp + (lane >> 2);
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      const int q = 4 * ks + (lane & 3);
      const bool ok = col < a.K && q < r;
#pragma unroll
      for (int p = 0; p < 3; ++p) wb[ks][p] = ok ? a.w3[(int64_t(p) * RK + q) * a.K + col] : 0.0;
    }
  }

  for (int u = blockIdx.x, it = 0; u < nunits; u += gs, ++it) {
    const int s = it % NST;
    unsigned char* dbuf = smem + s * G::STAGE;
    unsigned char* fbuf = dbuf + G::DATA;
    const int64_t g0 = int64_t(u / nchunks) * TR;
    mbar_wait(&bars[s], uint32_t((it / NST) & 1));
    // zero what the copies did not fill: the whole tile without an input,
    // factor rows past the factor's end
    const int rf = rows_valid(min(a.n_f, a.nrows), g0);
    if (!IN || rf < TR) {
      if (!IN) {
        for (int e = tid; e < TR * KCB; e += NTHR) st2(dbuf + e * 16, make_double2(0.0, 0.0));
      }
      for (int e = rf * (FP / 16) + tid; e < TR * (FP / 16); e += NTHR) st2(fbuf + e * 16, make_double2(0.0, 0.0));
      __syncthreads();
    }

    if constexpr (CON) {
      // W_part[q][c] += sum_t conj(F[t][q]) X[t][c]  (warp: 8 columns, all 32 q)
      //   T1 = Fr Xr, T2 = Fi Xi, T3 = (Fr - Fi)(Xr + Xi):  Re = T1 + T2, Im = T3 - T1 + T2
      const int cb = (8 * warp + (lane >> 2)) * 16;
#pragma unroll 2
      for (int ks = 0; ks < TR / 4; ++ks) {
        const int row = 4 * ks + (lane & 3);
        const double2 xv = ld2(dbuf + row * DP + cb);
        const double bs = xv.x + xv.y;
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) {
          const double2 fv = ld2(fbuf + row * FP + (8 * mt + (lane >> 2)) * 16);
          dmma(acc[mt][0], fv.x, xv.x);
          dmma(acc[mt][1], fv.y, xv.y);
          dmma(acc[mt][2], fv.x - fv.y, bs);
        }
      }
    }
    if constexpr (NW > 1) {
      if constexpr (CON) __syncthreads();  // contraction reads of the untransformed rows are done
      const int c = tid % KC, p = tid / KC;
      wht_stage<(NW < 8 ? NW : 8), 1, NW>(dbuf, c, p);  // strides 1, 2, 4
      __syncthreads();
      if constexpr (NW > 8) {
        wht_stage<NW / 8, 8, NW>(dbuf, c, p);  // strides 8 .. NW/2
        __syncthreads();
      }
    }
    if constexpr (EXP) {
      // Y[t][c] += sum_q G[t][q] W'[q][c]  (warp: 8 columns; rows in two halves)
      //   T1 = Gr Wr, T2 = Gi Wi, T3 = (Gr + Gi)(Wr + Wi):  Re = T1 - T2, Im = T3 - T1 - T2
#pragma unroll 1
      for (int half = 0; half < 2; ++half) {
        double e[4][3][2];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int p = 0; p < 3; ++p) e[i][p][0] = e[i][p][1] = 0.0;
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          const int q = 4 * ks + (lane & 3);
#pragma unroll
          for (int mt = 0; mt < 4; ++mt) {
            const int row = 32 * half + 8 * mt + (lane >> 2);
            const double2 gv = ld2(fbuf + row * FP + q * 16);
            dmma(e[mt][0], gv.x, wb[ks][0]);
            dmma(e[mt][1], gv.y, wb[ks][1]);
            dmma(e[mt][2], gv.x + gv.y, wb[ks][2]);
          }
        }
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) {
          const int row = 32 * half + 8 * mt + (lane >> 2);
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            unsigned char* pp = dbuf + row * DP + (8 * warp + 2 * (lane & 3) + j) * 16;
            const double2 v = ld2(pp);
            st2(pp, make_double2(v.x + e[mt][0][j] - e[mt][1][j], v.y + e[mt][2][j] - e[mt][0][j] - e[mt][1][j]));
          }
        }
      }
      __syncthreads();
    }
    if constexpr (OUT) {
      // thread: column c, rows t = tid / 64 + 4 j (coalesced 1 KB rows)
      const int rout = rows_valid(min(a.n_out, a.nrows), g0);
      const int c = tid % KC;
      if (c < kcv) {
        for (int t = tid / KC; t < rout; t += NTHR / KC)
          Y[wlr_phys<NW>(a.yout, g0 + t) * a.yout.ld + c0 + c] = ld2(dbuf + t * DP + c * 16);
      }
    }
    __syncthreads();  // stage s is free
    if (tid == 0 && u + NST * gs < nunits) {
      fence_proxy_async();
      issue(u + NST * gs, s);
    }
  }

  if constexpr (CON) {
    double2* P = reinterpret_cast<double2*>(a.partial) + int64_t(blockIdx.x) * RK * KC;
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) {
      const int q = 8 * mt + (lane >> 2);
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int c = 8 * warp + 2 * (lane & 3) + j;
        P[q * KC + c] = make_double2(acc[mt][0][j] + acc[mt][1][j], acc[mt][2][j] - acc[mt][0][j] + acc[mt][1][j]);
      }
    }
  }
}

__global__ void wlr_finalize_kernel(const double2* partial, int grid, int nchunks, int64_t r, int64_t K,
                                    const double2* s, int s_conj, double* w3) {
  const int64_t n = int64_t(RK) * K;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += int64_t(gridDim.x) * blockDim.x) {
    const int q = int(e / K);
    const int64_t c = e % K;
    const int ch = int(c / KC), cc = int(c % KC);
    double2 sum = make_double2(0.0, 0.0);
    if (q < r) {
      for (int b = ch; b < grid; b += nchunks) {  // fixed order: deterministic
        const double2 v = partial[(int64_t(b) * RK + q) * KC + cc];
        sum.x += v.x;
        sum.y += v.y;
      }
      if (s) {
        double2 sv = s[q];
        if (s_conj) sv.y = -sv.y;
        sum = cmul(sum, sv);
      }
    }
    w3[e] = sum.x;
    w3[n + e] = sum.y;
    w3[2 * n + e] = sum.x + sum.y;
  }
}

template <int NW, bool CON, bool EXP, bool IN, bool OUT>
void wlr_go(const CUtensorMap& map, const WlrArgs& a, int grid, int nchunks, int nunits, cudaStream_t s) {
  auto kern = wlr_kernel<NW, CON, EXP, IN, OUT>;
  {
    // the shared-memory opt-in is per (kernel, device)
    static std::mutex mu;
    static std::set<int> done;
    int dev = 0;
    SMAT_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    if (!done.count(dev)) {
      SMAT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, WlrGeom<EXP>::SMEM));
      done.insert(dev);
    }
  }
  kern<<<grid, NTHR, WlrGeom<EXP>::SMEM, s>>>(map, a, nchunks, nunits);
  SMAT_CUDA(cudaGetLastError());
}

// Tensor map of the unit input box (8-byte words; a complex128 is two).
bool wlr_in_map(CUtensorMap* map, const WlrIn& in, int64_t K) {
  auto fn = encode_fn();
  if (!fn || (reinterpret_cast<uintptr_t>(in.p) & 15)) return false;
  const cuuint64_t W = cuuint64_t(2 * K), rb = cuuint64_t(in.ld) * 16;  // words per row, row bytes
  cuuint64_t dims[5] = {W, 1, 1, 1, 1}, strides[4] = {16, 16, 16, 16};
  cuuint32_t box[5] = {cuuint32_t(2 * KCB), 1, 1, 1, 1}, estr[5] = {1, 1, 1, 1, 1};
  int rank = 2;
  const cuuint64_t nwa = cuuint64_t(in.nwa), n2b = cuuint64_t(in.n2b);
  if (in.kind == WLR_IN_ROWS) {
    dims[1] = cuuint64_t(in.rows); strides[0] = rb; box[1] = TR;
  } else if (in.kind == WLR_IN_T1A) {
    // (a: NWa rows 64 apart, T % 64: rows 1 apart, T / 64: 64 NWa rows apart)
    rank = 4;
    dims[1] = nwa; dims[2] = 64; dims[3] = cuuint64_t(in.P) / (64 * nwa);
    strides[0] = 64 * rb; strides[1] = rb; strides[2] = 64 * nwa * rb;
    box[1] = cuuint32_t(nwa); box[2] = cuuint32_t(TR / nwa); box[3] = 1;
  } else {
    // (b % (64/NWa): NWa rows apart, b / (64/NWa): 64 N2b rows apart,
    //  a = T' % NWa: rows 1 apart, k2 = T' / NWa: 64 rows apart)
    rank = 5;
    dims[1] = 64 / nwa; dims[2] = nwa; dims[3] = nwa; dims[4] = n2b;
    strides[0] = nwa * rb; strides[1] = 64 * n2b * rb; strides[2] = rb; strides[3] = 64 * rb;
    box[1] = cuuint32_t(64 / nwa); box[2] = cuuint32_t(nwa); box[3] = 1; box[4] = 1;
  }
  for (int k = 0; k < rank - 1; ++k) {
    if (dims[k + 1] == 1) strides[k] = 16;  // (an extent-1 dimension: any legal stride)
    if (strides[k] % 16 || strides[k] >= (cuuint64_t(1) << 40)) return false;
  }
  const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT64, rank, const_cast<void*>(in.p), dims, strides, box,
                        estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

__global__ void wlr_pad_kernel(const double2* src, double2* dst, int64_t rows, int64_t r, int64_t pitch) {
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < rows * pitch;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t g = e / pitch, q = e % pitch;
    dst[e] = q < r ? src[g * r + q] : make_double2(0.0, 0.0);
  }
}

}  // namespace

int64_t wlr_pitch(bool expansion) { return (expansion ? FPE : FPC) / 16; }

void wlr_pad_factor(const void* src, void* dst, int64_t rows, int64_t r, bool expansion, cudaStream_t s) {
  wlr_pad_kernel<<<1184, 256, 0, s>>>(reinterpret_cast<const double2*>(src), reinterpret_cast<double2*>(dst), rows,
                                      r, wlr_pitch(expansion));
  SMAT_CUDA(cudaGetLastError());
}

int wlr_grid(int device, int64_t K) {
  const int nchunks = int((K + KC - 1) / KC);
  const int per = MINB * num_sms(device) / nchunks;
  return nchunks * (per > 0 ? per : 1);
}

size_t wlr_partial_bytes(int device, int64_t K) { return size_t(wlr_grid(device, K)) * RK * KC * 16; }

int launch_wlr(const WlrMode& m, const WlrArgs& a, int device, cudaStream_t s, bool dry) {
  SMAT_CHECK(a.r >= 1 && a.r <= RK, SMAT_UNSUPPORTED, "wlr: rank must be 1..32");
  SMAT_CHECK(a.K >= 1 && m.nw >= 1 && a.nrows % (m.nw > 1 ? m.nw : 1) == 0, SMAT_BAD_ARG, "wlr: bad shape");
  if (dry) return 1;
  const int nchunks = int((a.K + KC - 1) / KC);
  const int grid = wlr_grid(device, a.K);
  const int64_t nub = (a.nrows + TR - 1) / TR;
  SMAT_CHECK(nub * nchunks < (int64_t(1) << 31), SMAT_UNSUPPORTED, "wlr: too many units");
  const int nunits = int(nub * nchunks);
  // (NW groups never straddle units: TR is a multiple of NW)
  CUtensorMap map;
  std::memset(&map, 0, sizeof(map));
  if (m.in) SMAT_CHECK(wlr_in_map(&map, a.in, a.K), SMAT_UNSUPPORTED, "wlr: input view is not TMA-addressable");
#define WLR_CASE(NW_, CON_, EXP_, IN_, OUT_)                                                          \
  if (m.nw == NW_ && m.con == CON_ && m.exp == EXP_ && m.in == IN_ && m.out == OUT_) {              \
    wlr_go<NW_, CON_, EXP_, IN_, OUT_>(map, a, grid, nchunks, nunits, s);                           \
    return 1;                                                                                         \
  }
#define WLR_HAD(NW_)                  \
  WLR_CASE(NW_, true, false, true, true) \
  WLR_CASE(NW_, false, true, true, true)
  // the C5 blocked chain: Hadamard stages with the contraction (input rows)
  // or the expansion (output rows) — N1 = NWa * 64 for the middle-pass length
  WLR_HAD(2)
  WLR_HAD(4)
  WLR_HAD(8)
  WLR_HAD(16)
  WLR_HAD(32)
  WLR_HAD(64)
  // plain LowRank halves
  WLR_CASE(1, true, false, true, false)    // contraction
  WLR_CASE(1, false, true, true, true)     // expansion, y += G W'
  WLR_CASE(1, false, true, false, true)    // expansion, y = G W'
#undef WLR_HAD
#undef WLR_CASE
  throw Error(SMAT_UNSUPPORTED, "wlr: mode not instantiated");
}

int launch_wlr_finalize(const void* partial, int grid, int64_t r, int64_t K, const void* s, bool s_conj, double* w3,
                        cudaStream_t st, bool dry) {
  if (dry) return 1;
  const int nchunks = int((K + KC - 1) / KC);
  const int64_t n = int64_t(RK) * K;
  const int blocks = int(std::min<int64_t>((n + 255) / 256, 1024));
  wlr_finalize_kernel<<<blocks, 256, 0, st>>>(reinterpret_cast<const double2*>(partial), grid, nchunks, r, K,
                                              reinterpret_cast<const double2*>(s), s_conj ? 1 : 0, w3);
  SMAT_CUDA(cudaGetLastError());
  return 1;
}

}  // namespace smat
