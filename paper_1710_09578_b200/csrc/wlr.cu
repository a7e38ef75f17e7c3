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
constexpr int KC = 32;              // columns per unit (and per column chunk)
constexpr int RK = 32;              // padded rank
// shared-memory row pitches (bytes).  The tensor-core fragments read 16-byte
// entries of rows lane%4 (contraction: data and factor rows) or lane/4
// (expansion: factor rows); a pitch of 2 (mod 8) or 4 (mod 8) 16-byte units
// puts those rows on distinct bank groups.  The data tile is a tensor-map
// box of KCB = 34 columns (the two extra columns are never used), so it lands
// with that pitch; the factor rows are stored padded in global memory.
constexpr int KCB = KC + 2;
constexpr int DP = KCB * 16;        // 544
constexpr int FPC = (RK + 2) * 16;  // 544, contraction
constexpr int FPE = (RK + 4) * 16;  // 576, expansion
// One CTA per SM, two consumer groups of four warps (8 columns each) taking
// alternate units, two rings of shared-memory stages — unit data tiles (4
// deep) and unit factor rows (2 deep).  The thread that releases a stage
// issues its refill (the unit NSD / NSF further on), so the data ring runs two
// units ahead of the consumers.  The groups' tensor-core phases (contraction
// / expansion) are serialised in unit order through two mbarriers, so one
// group multiplies while the other transforms and stores (left to themselves
// the groups phase-lock: both multiply at half rate, then both stream); a
// group hands the pipe over when three quarters of its unit's MMAs are issued
// (one arrival per warp), so the other group's waits and first operand loads
// run under its last steps.  The factor rows are needed only in that phase,
// hence their shorter ring.  Eight
// warps, two per SM sub-partition, leave each thread up to 255 registers
// (a ninth, producer warp would cap them at 168 and spill the expansion).
// (The single-stage two-CTA layout measured load + tensor work + transform +
// store in series: 1.39 ms per C5 pass, of which 0.65 ms tensor work.)
constexpr int GTHR = 128;                // threads per consumer group
constexpr int NGRP = 2;                  // consumer groups
constexpr int NTHR = NGRP * GTHR;
#ifndef WLR_NSD
#define WLR_NSD 4
#endif
constexpr int NSD = WLR_NSD;             // data ring stages
#ifndef WLR_NSF
#define WLR_NSF 2
#endif
constexpr int NSF = WLR_NSF;             // factor ring stages
// tensor-phase step after which a warp hands the pipe over (contraction: of
// 16 k-steps; expansion: of 4 row quarters, counted when quarter SIG_QR + 1's
// products have been issued)
#ifndef WLR_SIG_KS
#define WLR_SIG_KS 12
#endif
#ifndef WLR_SIG_QR
#define WLR_SIG_QR 2
#endif
constexpr int SIG_KS = WLR_SIG_KS, SIG_QR = WLR_SIG_QR;
// (timing experiments only, tools/exp_build.py: skip phases; results wrong)
#ifndef WLR_SKIP
#define WLR_SKIP 0
#endif

template <bool EXP>
struct WlrGeom {
  static constexpr int FP = EXP ? FPE : FPC;
  static constexpr int DATA = TR * DP;
  static constexpr int FACT = TR * FP;
  static constexpr int NBAR = NSD + NSF + NGRP;
  static constexpr int ROWT = NGRP * TR * 8;  // per group: the unit's output row offsets
  static constexpr int SMEM = NSD * DATA + NSF * FACT + ROWT + NBAR * 8;
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
  for (int j = p; j < NG; j += GTHR / KC) {
    const int b0 = S == 1 ? R * j : NW * (j / 8) + j % 8;
    double2 v[8];
#pragma unroll
    for (int k = 0; k < R; ++k) v[k] = ld2(dbuf + (b0 + k * S) * DP + c * 16);
    wht_reg<R>(v);
#pragma unroll
    for (int k = 0; k < R; ++k) st2(dbuf + (b0 + k * S) * DP + c * 16, v[k]);
  }
}

__device__ __forceinline__ void mbar_arrive1(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// named barrier of one consumer group (ids 1, 2; 0 is __syncthreads)
__device__ __forceinline__ void group_sync(int grp) {
  asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(GTHR) : "memory");
}

template <int NW, bool CON, bool EXP, bool IN, bool OUT>
__global__ void __launch_bounds__(NTHR, 1)
    wlr_kernel(const __grid_constant__ CUtensorMap xmap, const WlrArgs a, const int nchunks, const int nunits) {
  using G = WlrGeom<EXP>;
  constexpr int FP = G::FP;
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* dring = smem;                  // data tiles
  unsigned char* fring = smem + NSD * G::DATA;  // factor rows
  int64_t* rowt = reinterpret_cast<int64_t*>(fring + NSF * G::FACT);  // [NGRP][TR]
  uint64_t* full = reinterpret_cast<uint64_t*>(fring + NSF * G::FACT + G::ROWT);
  uint64_t* ffull = full + NSD;
  uint64_t* mma_done = ffull + NSF;  // per group: its tensor phase of a unit is issued
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int grp = warp / 4;  // consumer group 0 / 1
  const int ch = int(blockIdx.x) % nchunks;
  const int64_t c0 = int64_t(ch) * KC;
  const int kcv = int(min(int64_t(KC), a.K - c0));  // valid columns of this CTA's chunk
  const int r = int(a.r);
  const int gs = int(gridDim.x);
  // this CTA's units: blockIdx.x + i * gs, i < nloc (gs is a multiple of
  // nchunks, so every unit of the CTA is in column chunk ch)
  const int nloc = int(blockIdx.x) < nunits ? (nunits - 1 - int(blockIdx.x)) / gs + 1 : 0;
  // first unit row of the CTA's i-th unit: unit u = blockIdx.x + i gs covers
  // row block u / nchunks = blockIdx.x / nchunks + i (gs / nchunks)
  const int rb0 = int(blockIdx.x) / nchunks, rbs = gs / nchunks;
  auto unit_g0 = [&](int i) -> int64_t { return int64_t(rb0 + i * rbs) * TR; };
  double2* Y = reinterpret_cast<double2*>(a.y);
  const double2* F = reinterpret_cast<const double2*>(a.F);
  const int lgw = a.in.kind == WLR_IN_ROWS ? 0 : ilog2_dev(int(a.in.nwa));

  auto rows_valid = [&](int64_t lim, int64_t g0) -> int {
    const int64_t v = lim - g0;
    return v <= 0 ? 0 : v >= TR ? TR : int(v);
  };
  if (tid == 0) {
    for (int st = 0; st < NSD; ++st) mbar_init(&full[st], 1);
    for (int st = 0; st < NSF; ++st) mbar_init(&ffull[st], 1);
    for (int g = 0; g < NGRP; ++g) mbar_init(&mma_done[g], GTHR / 32);  // (one arrival per warp)
    fence_barrier_init();
  }
  __syncthreads();

  // unit i's input box (one tensor-map copy) into data stage i % NSD, its
  // factor rows (one bulk copy of the padded rows) into factor stage i % NSF
  auto issue_data = [&](int i) {
    if constexpr (IN) {
      const int64_t g0 = unit_g0(i);
      const int s = i % NSD;
      unsigned char* dbuf = dring + s * G::DATA;
      mbar_arrive_expect_tx(&full[s], uint32_t(G::DATA));
      const int cw = int(2 * c0);
      if (a.in.kind == WLR_IN_ROWS) {
        tma_load_2d(dbuf, &xmap, &full[s], cw, int(g0));
      } else if (a.in.kind == WLR_IN_T1A) {
        const int T0 = int(g0 >> lgw);
        tma_load_4d(dbuf, &xmap, &full[s], cw, 0, T0 & 63, T0 >> 6);
      } else {
        const int Tp = int(g0 >> 6);
        tma_load_5d(dbuf, &xmap, &full[s], cw, 0, 0, Tp & int(a.in.nwa - 1), Tp >> lgw);
      }
    }
  };
  auto issue_factor = [&](int i) {
    const int64_t g0 = unit_g0(i);
    const int sf = i % NSF;
    const int rf = rows_valid(min(a.n_f, a.nrows), g0);
    const uint32_t fbytes = uint32_t(rf) * FP;
    mbar_arrive_expect_tx(&ffull[sf], fbytes);
    if (rf) bulk_load(fring + sf * G::FACT, F + g0 * (FP / 16), fbytes, &ffull[sf]);
  };
  if (tid == 0) {
    if constexpr (IN) tma_prefetch_desc(&xmap);
    for (int i = 0; i < NSD && i < nloc; ++i) issue_data(i);
    for (int i = 0; i < NSF && i < nloc; ++i) issue_factor(i);
  }

  // ---- consumer group grp: units i = grp, grp + 2, ...
  const int gt = tid - grp * GTHR, gw = gt >> 5;  // thread / warp within the group
  // tensor phase of unit i (the group's k-th, i = 2k + grp) starts after unit
  // i - 1's: group 0 waits for group 1's (k-1)-th, group 1 for group 0's k-th
  // (the acquire also waits for the unit's factor rows and zeroes the rows
  // past the factor's end; the release frees their stage)
  auto mma_acquire = [&](int i, unsigned char* fbuf, int rf) {
    if (i > 0 && !(WLR_SKIP & 32)) mbar_wait(&mma_done[1 - grp], uint32_t(((i - 1) / NGRP) & 1));
    mbar_wait(&ffull[i % NSF], uint32_t((i / NSF) & 1));
    if (rf < TR) {
      for (int e = rf * (FP / 16) + gt; e < TR * (FP / 16); e += GTHR) st2(fbuf + e * 16, make_double2(0.0, 0.0));
      group_sync(grp);
    }
  };
  // Hand-over of the tensor pipe: every warp signals once most of its unit's
  // MMAs are issued (SIG of the phase's steps), so the other group's waits,
  // first operand loads and Gauss sums run under this group's last steps
  // instead of after its release barrier; the release then only frees the
  // factor stage.
  auto mma_signal = [&]() {
    __syncwarp();
    if (lane == 0) mbar_arrive1(&mma_done[grp]);
  };
  auto mma_release = [&](int i, bool signalled) {
    if (!signalled) mma_signal();
    fence_proxy_async();
    group_sync(grp);
    if (gt == 0 && i + NSF < nloc) issue_factor(i + NSF);  // (factor stage free)
  };
  // contraction partials: q-tile mt (rows 8mt.. of W), product p (Gauss), pair
  double acc[4][3][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int p = 0; p < 3; ++p) acc[i][p][0] = acc[i][p][1] = 0.0;
  // expansion: this lane's W' fragments for every k-step (q = 4ks + lane%4,
  // column 8*gw + lane/4 of the chunk)
  double wb[EXP ? 8 : 1][3];
  if constexpr (EXP) {
    const int64_t col = c0 + 8 * gw + (lane >> 2);
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      const int q = 4 * ks + (lane & 3);
      const bool ok = col < a.K && q < r;
#pragma unroll
      for (int p = 0; p < 3; ++p) wb[ks][p] = ok ? a.w3[(int64_t(p) * RK + q) * a.K + col] : 0.0;
    }
  }

  for (int i = grp; i < nloc; i += NGRP) {
    const int s = i % NSD, sf = i % NSF;
    unsigned char* dbuf = dring + s * G::DATA;
    unsigned char* fbuf = fring + sf * G::FACT;
    const int64_t g0 = unit_g0(i);
    if constexpr (IN) {
      mbar_wait(&full[s], uint32_t((i / NSD) & 1));
    } else {
      // without an input the tile starts as zeros (output = F W' only)
      for (int e = gt; e < TR * KCB; e += GTHR) st2(dbuf + e * 16, make_double2(0.0, 0.0));
      group_sync(grp);
    }
    const int rf = rows_valid(min(a.n_f, a.nrows), g0);
    // the unit's output row offsets, once per unit (read by the stores after
    // the group barriers of the tensor phase / transform)
    if (OUT && gt < TR) rowt[grp * TR + gt] = wlr_phys<NW>(a.yout, g0 + gt) * a.yout.ld + c0;

    if constexpr (CON) mma_acquire(i, fbuf, rf);
    if constexpr (CON && !(WLR_SKIP & 1)) {
      // W_part[q][c] += sum_t conj(F[t][q]) X[t][c]  (warp: 8 columns, all 32 q)
      //   T1 = Fr Xr, T2 = Fi Xi, T3 = (Fr - Fi)(Xr + Xi):  Re = T1 + T2, Im = T3 - T1 + T2
      // (operands of k-step ks + 1 are loaded and their Gauss sums formed
      // while ks multiplies: no load or add sits between dependent MMAs)
      const int cb = (8 * gw + (lane >> 2)) * 16;
      const unsigned char* xr0 = dbuf + (lane & 3) * DP + cb;
      const unsigned char* fr0 = fbuf + (lane & 3) * FP + (lane >> 2) * 16;
      double2 xv = ld2(xr0), fv[4];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) fv[mt] = ld2(fr0 + mt * 128);
#pragma unroll
      for (int ks = 0; ks < TR / 4; ++ks) {
        const double bs = (WLR_SKIP & 64) ? xv.x : xv.x + xv.y;
        double fd[4];
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) fd[mt] = (WLR_SKIP & 64) ? fv[mt].x : fv[mt].x - fv[mt].y;
        const double2 xc = xv;
        double2 fc[4];
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) fc[mt] = fv[mt];
        if (ks + 1 < TR / 4) {
          xv = ld2(xr0 + (ks + 1) * 4 * DP);
#pragma unroll
          for (int mt = 0; mt < 4; ++mt) fv[mt] = ld2(fr0 + (ks + 1) * 4 * FP + mt * 128);
        }
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) {
          dmma(acc[mt][0], fc[mt].x, xc.x);
          dmma(acc[mt][1], fc[mt].y, xc.y);
          dmma(acc[mt][2], fd[mt], bs);
        }
        if (ks == SIG_KS) mma_signal();
      }
    }
    // (the release's group barrier also ends the contraction's reads of the
    // untransformed rows)
    if constexpr (CON) mma_release(i, !(WLR_SKIP & 1));
    if constexpr (NW > 1 && !(WLR_SKIP & 2)) {
      const int c = gt % KC, p = gt / KC;
      wht_stage<(NW < 8 ? NW : 8), 1, NW>(dbuf, c, p);  // strides 1, 2, 4
      group_sync(grp);
      if constexpr (NW > 8) {
        wht_stage<NW / 8, 8, NW>(dbuf, c, p);  // strides 8 .. NW/2
        group_sync(grp);
      }
    }
    if constexpr (EXP) mma_acquire(i, fbuf, rf);
    if constexpr (EXP && !(WLR_SKIP & 4)) {
      // Y[t][c] += sum_q G[t][q] W'[q][c]  (warp: 8 columns; rows in quarters)
      //   T1 = Gr Wr, T2 = Gi Wi, T3 = (Gr + Gi)(Wr + Wi):  Re = T1 - T2, Im = T3 - T1 - T2
      // Quarter qr + 1's products are issued before quarter qr's rows are
      // read-modified-written, so the shared-memory update runs under the
      // tensor work; the tensor phase is released before the last update.
      double e[2][2][3][2];
      auto mma_q = [&](int qr, double (&eq)[2][3][2]) {
#pragma unroll
        for (int i2 = 0; i2 < 2; ++i2)
#pragma unroll
          for (int p = 0; p < 3; ++p) eq[i2][p][0] = eq[i2][p][1] = 0.0;
        // (k-step ks + 1's factor entries and sums are formed while ks multiplies)
        const unsigned char* g0p = fbuf + (16 * qr + (lane >> 2)) * FP + (lane & 3) * 16;
        double2 gv[2];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) gv[mt] = ld2(g0p + mt * 8 * FP);
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          double2 gc[2];
          double gs2[2];
#pragma unroll
          for (int mt = 0; mt < 2; ++mt) {
            gc[mt] = gv[mt];
            gs2[mt] = gv[mt].x + gv[mt].y;
          }
          if (ks + 1 < 8) {
#pragma unroll
            for (int mt = 0; mt < 2; ++mt) gv[mt] = ld2(g0p + mt * 8 * FP + (ks + 1) * 64);
          }
#pragma unroll
          for (int mt = 0; mt < 2; ++mt) {
            dmma(eq[mt][0], gc[mt].x, wb[ks][0]);
            dmma(eq[mt][1], gc[mt].y, wb[ks][1]);
            dmma(eq[mt][2], gs2[mt], wb[ks][2]);
          }
        }
      };
      auto rmw_q = [&](int qr, const double (&eq)[2][3][2]) {
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          const int row = 16 * qr + 8 * mt + (lane >> 2);
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            unsigned char* pp = dbuf + row * DP + (8 * gw + 2 * (lane & 3) + j) * 16;
            const double2 v = ld2(pp);
            st2(pp, make_double2(v.x + eq[mt][0][j] - eq[mt][1][j], v.y + eq[mt][2][j] - eq[mt][0][j] - eq[mt][1][j]));
          }
        }
      };
      mma_q(0, e[0]);
#pragma unroll
      for (int qr = 0; qr < 4; ++qr) {
        if (qr + 1 < 4) mma_q(qr + 1, e[(qr + 1) & 1]);
        else mma_release(i, true);
        if (qr == SIG_QR) mma_signal();
        rmw_q(qr, e[qr & 1]);
      }
      group_sync(grp);  // (the expanded rows are complete before the stores read them)
    } else if constexpr (EXP) {
      mma_release(i, false);
    }
    if constexpr (OUT && !(WLR_SKIP & 8)) {
      // thread: column c, rows t = gt / 32 + 4 j (coalesced 512-byte rows)
      const int rout = rows_valid(min(a.n_out, a.nrows), g0);
      const int c = gt % KC;
      if (c < kcv) {
        for (int t = gt / KC; t < rout; t += GTHR / KC) Y[rowt[grp * TR + t] + c] = ld2(dbuf + t * DP + c * 16);
      }
    }
    // stage s is free: order this group's generic-proxy accesses before the
    // producer's next asynchronous copy into it, then release it
    fence_proxy_async();
    group_sync(grp);
    if (IN && gt == 0 && i + NSD < nloc) issue_data(i + NSD);  // (data stage free)
  }

  if constexpr (CON) {
    double2* P = reinterpret_cast<double2*>(a.partial) + (int64_t(blockIdx.x) * NGRP + grp) * RK * KC;
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) {
      const int q = 8 * mt + (lane >> 2);
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int c = 8 * gw + 2 * (lane & 3) + j;
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
      for (int b = ch; b < grid; b += nchunks)  // fixed order: deterministic
        for (int g = 0; g < NGRP; ++g) {
          const double2 v = partial[((int64_t(b) * NGRP + g) * RK + q) * KC + cc];
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
  const int per = num_sms(device) / nchunks;
  return nchunks * (per > 0 ? per : 1);
}

size_t wlr_partial_bytes(int device, int64_t K) { return size_t(wlr_grid(device, K)) * NGRP * RK * KC * 16; }

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
