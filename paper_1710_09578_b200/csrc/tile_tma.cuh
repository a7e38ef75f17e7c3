// tile_tma.cuh — persistent, TMA-fed FFT tile pass.
//
// Same math as fft_tile_kernel (tile_impl.cuh), restructured for HBM
// throughput on sm_100a:
//   * persistent CTAs (as many per SM as shared memory allows, up to 4) walk
//     round-robin over tiles of CT columns x N rows;
//   * one elected thread loads a whole tile with a single 5-D TMA box
//     (cp.async.bulk.tensor) into a 2-3 deep ring of landing buffers tracked by
//     mbarriers, together with the tile's side data (spectrum slice, per-tile
//     pre/post vector slice, four-step twiddle slice) as 1-D bulk copies on
//     the same barrier — no load instructions or addresses in the math warps;
//   * the landing buffer doubles as the exchange buffer (rows XOR-swizzled by
//     the writing stage's radix, ex_row in fft_core.cuh, bank-conflict free);
//   * stage twiddles come from a per-CTA staged table (st_twoff layout, odd
//     lane strides; quad layout in single precision, so every twiddle multiply
//     is FMUL2 + FFMA2);
//   * the output tile is staged in the landing buffer and leaves with one TMA
//     store; masked passes (zero padding / truncation) use extent-limited maps.
#pragma once

#include "tile_impl.cuh"
#include "tma.cuh"

namespace smat {

// EP: elements per thread (16 -> radix-16 stages, 32 -> radix-32 stages: one
// exchange fewer for N = 1024); NB: landing buffers per CTA (0 = as many as fit,
// up to 3).
// CTO: columns per tile override (0 = default).
// MS: side slice in every stage — 0 none, 1 spectrum (MID pass), 2 pre/post
// vector (masked pass).
template <class C, int N, int EP = 16, int NB = 0, bool TV = false, int MS = 0, int CTO = 0>
struct TmaGeom {
  static constexpr int E = N < EP ? N : EP;
  // (double-precision 2048-point tiles: two columns, so that two landing
  // buffers plus the spectrum slice or the four-step twiddles fit)
  static constexpr int CT = CTO ? CTO : sizeof(C) == 16 && N >= 2048 ? 2 : tile_CT(N, sizeof(C));
  static constexpr int TPC = N / E;
  static constexpr int T = TPC * CT;
  static constexpr int ROWB = CT * int(sizeof(C));                 // bytes per tile row
  static constexpr int LAY = ROWB >= 128 ? 1 : 128 / ROWB;          // exchange row permutation
  static constexpr size_t BUF = size_t(N) * CT * sizeof(C);         // one dense TMA box
  // the tile's spectrum slice (MS 1, plain entries) or pre / post slice (MS 2)
  static constexpr size_t SPB = MS == 1 ? size_t(N) * sizeof(C) : MS ? size_t(N) * 16 : 0;
  // four-step twiddles: the tile's slice of a precomputed table, bulk-loaded
  // with the tile (TVSL; measured faster than assembling them per CTA from
  // the two-level table even where it costs a landing buffer: C2's twiddle
  // pass 0.224 -> 0.199 ms with a two- instead of three-deep ring).  Short
  // single-precision tiles keep the per-CTA table (TVB): C3's 64-point
  // masked pass ran 0.053 ms that way vs 0.070 ms with slices.
  static constexpr bool TVSL = TV && (sizeof(C) == 16 || N >= 512);
  static constexpr size_t TVSB = TVSL ? size_t(N) * 16 : 0;
  static constexpr size_t STAGE = BUF + SPB + TVSB;
  // staged stage-twiddle table(s) (float4 quads / double2): one when the stage
  // list is a palindrome (the mirrored inverse of the spectrum pass shares it),
  // else a second one for the mirrored list (short transforms only)
  static constexpr bool DUAL = !st_palindrome(N, E);
  // (entries: float4 quads / double2, or plain float2 in the single-precision
  // spectrum passes)
  static constexpr size_t TWE = (MS == 1 && sizeof(C) == 8) ? 8 : 16;
  static constexpr size_t TWB = size_t(N) * TWE * (DUAL ? 2 : 1);
  static constexpr size_t TVB = TV && !TVSL ? size_t(N) * 16 : 0;  // per-tile four-step twiddles
  // ring of landing buffers: tile t computes in one while t+1.. load into the others
  static constexpr int NBUF =
      NB > 0 && (227 * 1024 - int(TWB + TVB) - 64) / int(STAGE) >= NB
          ? NB
          : ((227 * 1024 - int(TWB + TVB) - 64) / int(STAGE) >= 3 ? 3 : 2);
  static constexpr size_t SMEM = NBUF * STAGE + TWB + TVB + 64;
  // resident CTAs per SM: as many as shared memory and 1024 threads allow, up to 4
  static constexpr int MB_S = (227 * 1024) / int(SMEM), MB_T = 1024 / T;
  static constexpr int MINB = (MB_S < MB_T ? MB_S : MB_T) >= 4 ? 4 : (MB_S < MB_T ? MB_S : MB_T) >= 2 ? 2 : 1;
};

// Programmatic dependent launch for the short single-precision passes
// (N <= 128: C3's 64 / 128-point passes, tens of microseconds each, where the
// launch gap between passes is a visible share): the grid is scheduled while
// the previous pass drains and waits (griddepcontrol.wait) before touching
// its input.  Longer passes are compiled without it — the griddepcontrol
// instructions alone slowed C4's 256-point spectrum pass by 9 %.
// (timing experiments only, tools/exp_build.py: skip phases; results wrong)
#ifndef FFT_SKIP
#define FFT_SKIP 0
#endif

template <class C, int N>
constexpr bool kPdl = sizeof(C) == 8 && N <= 128;
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Walsh-Hadamard transform over rows [0, N/2) of every column of a landed /
// staged tile (natural row order, buf[i * CT + cs]), radix-8 stages with
// strides 1, 8, 64, ... (stride-1-first); TPC threads per column hold 8
// elements each (N/2 = 8 TPC).  The load order of each group is rotated by the
// group index so that the two row groups a memory phase touches differ.
// SMAX: the strides handled here (the stages with stride >= SMAX = TPC — the
// bits of the stage-0 element index r — run in registers on the loaded /
// finished elements instead, wht_regs_half).
// SWZ: rows stored at row ^ ((row >> 3) & 1) — the stride-1 stage's threads
// own 8 consecutive 64-byte rows each (512 bytes apart between lanes, all on
// one half of the banks); flipping the low row bit of every other group puts
// neighbouring lanes on opposite halves (a buffer the kernel fills itself).
template <bool SWZ>
__device__ __forceinline__ int wht_row(int row) {
  return SWZ ? row ^ ((row >> 3) & 1) : row;
}
template <class C, int N, int CT, int TPC, int S = 1, int SMAX = N / 2, bool SWZ = false>
__device__ __forceinline__ void tile_wht_half(C* buf, int j, int cs) {
  constexpr int NH = N / 2;
  static_assert(NH == 8 * TPC, "8 elements per thread");
  if constexpr (S < SMAX) {
    constexpr int R = SMAX / S >= 8 ? 8 : SMAX / S;
#pragma unroll
    for (int q = 0; q < 8 / R; ++q) {
      const int gid = j + q * TPC;
      const int base = (gid / S) * (S * R) + gid % S;
      C v[8];
#pragma unroll
      for (int k = 0; k < R; ++k) v[k] = buf[wht_row<SWZ>(base + k * S) * CT + cs];
      wht_small<R>(v);
#pragma unroll
      for (int k = 0; k < R; ++k) buf[wht_row<SWZ>(base + k * S) * CT + cs] = v[k];
    }
    __syncthreads();
    tile_wht_half<C, N, CT, TPC, S * R, SMAX, SWZ>(buf, j, cs);
  }
}

// The remaining Walsh-Hadamard stage of tile_wht_half<..., SMAX = TPC>: a
// thread's stage-0 elements a[r] are rows j + TPC r, so rows < N/2 are r < 8
// and their stride-TPC.. bits are the bits of r — an 8-point transform in
// registers (one shared-memory round trip and barrier fewer).
template <class C>
__device__ __forceinline__ void wht_regs_half(C* a) {
  wht_small<8>(a);
}

// 8-point Walsh-Hadamard over the Kron Hadamard index hh of a tile whose
// column cs = hh * CG + col (CT = 8 CG columns; FftArgs::wht_grp): the hh bits
// that are lane bits (cs bits < 5) run as butterfly stages over warp
// shuffles — no shared memory, no barrier; for CT = 64 the top bit (cs bit 5)
// is folded into the stage-0 load instead (fused_kron_load).
template <class C, int E, int CT>
__device__ __forceinline__ void wht_lanes8(C* a) {
  constexpr int CG = CT / 8;
  const int lane = int(threadIdx.x) & 31;
#pragma unroll
  for (int m = CG; m <= 16; m <<= 1) {
    const bool hi = (lane & m) != 0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const auto ox = __shfl_xor_sync(0xffffffffu, a[e].x, m);
      const auto oy = __shfl_xor_sync(0xffffffffu, a[e].y, m);
      a[e].x = hi ? ox - a[e].x : a[e].x + ox;
      a[e].y = hi ? oy - a[e].y : a[e].y + oy;
    }
  }
}

// launcher-only flags of the TMA pass: the pre (post) vector is stored per
// tile (pre_gmul / post_gmul) and rides with the tile as a bulk-loaded slice
enum : uint32_t { F_SIDEPRE = 1u << 20, F_SIDEPOST = 1u << 21, F_WGRP = 1u << 25 };

// MSK: the masked variant for the Bluestein / pruned-embedding passes — zero
// padding of input rows (g = goff + i*gin_stride >= n_valid_in), truncation of
// output rows, and the pre / post diagonal vectors.  The tensor maps cover rows
// i < ein (loads zero-fill the rest) and k < eout (stores drop the rest); the
// npatch rows from ein on that only some tiles own are loaded one tile ahead by
// npatch*CT threads and written into the landing buffer, and output rows past
// eout are stored directly by the threads that hold them.  A four-step-ordered
// pre or post vector arrives as a slice in the stage's side area (like the
// spectrum of the MID pass).  goff is uniform over a tile (launcher check), so
// the valid counts are per tile.
template <class C, int N, bool MID, bool TW, int EP, int NB, bool TS, bool MSK, int CTO, int WH = 0>
__global__ void __launch_bounds__(TmaGeom<C, N, EP, NB, TW, MID ? 1 : MSK ? 2 : 0, CTO>::T,
                                  TmaGeom<C, N, EP, NB, TW, MID ? 1 : MSK ? 2 : 0, CTO>::MINB)
    fft_tma_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap ymap,
                   const FftDev p, const int ntiles, const int ein, const int eout, const int npatch) {
  using G = TmaGeom<C, N, EP, NB, TW, MID ? 1 : MSK ? 2 : 0, CTO>;
  using R = typename RealOf<C>::T;
  constexpr int E = G::E, CT = G::CT, TPC = G::TPC, LAY = G::LAY;
  constexpr int NST = st_count(N, E);
  constexpr int R0 = st_radix(N, E, 0, false);
  constexpr int RL = MID ? st_radix(N, E, NST - 1, true) : st_radix(N, E, NST - 1, false);
  constexpr int LQ = log2_c(RL);
  // Deferred refill (spectrum passes, ring of two or three buffers): the
  // thread that issued a tile's TMA store does not wait for the engine to
  // finish reading the buffer — its warp would start the next tile late and
  // hold every barrier of it — but refills the buffer from inside the next
  // tile's forward transform, before its last stage: the store has drained by
  // then and the load still has the spectrum multiply and the inverse
  // transform to land (C5 spectrum pass 2.64 -> 2.34 ms, C2 0.285 -> 0.269,
  // C4 0.305 -> 0.274).  The passes with a single transform need the longer
  // load lead (C2's 1024-point twiddle / plain passes 0.207 / 0.183 -> 0.230 /
  // 0.212 ms deferred) and keep the wait.
  // Short transforms (<= 256 points: C4's and C3's passes, 64 KB tiles of
  // many columns) defer in every pass, at the start of the transform (C4
  // 0.886 -> 0.877 ms per step, C3 0.305 -> 0.302).
  constexpr bool DEFER = TS && (MID || N <= 256) && G::NBUF >= 2 && NST >= 2 && !(FFT_SKIP & 1);
  constexpr bool DEFER_START = DEFER && N <= 256;
  int pend_t = -1;
  constexpr bool EARLY = !TS && !MID && MSK && TW && sizeof(C) == 16 && G::NBUF == 1 && NST >= 2 && G::TVSL && !(FFT_SKIP & 1);
  extern __shared__ __align__(128) unsigned char smem_raw[];
  // stage s: [tile data | spectrum slice] at smem_raw + s*STAGE
  auto stage_buf = [&](int s) { return reinterpret_cast<C*>(smem_raw + s * G::STAGE); };
  auto stage_spec = [&](int s) { return smem_raw + s * G::STAGE + G::BUF; };
  auto stage_tv = [&](int s) { return reinterpret_cast<C*>(smem_raw + s * G::STAGE + G::BUF + G::SPB); };
  constexpr bool TVSL = G::TVSL;
  C* tws = reinterpret_cast<C*>(smem_raw + G::NBUF * G::STAGE);  // W_N^t, t < N (float4 quads or double2)
  C* tvs = reinterpret_cast<C*>(smem_raw + G::NBUF * G::STAGE + G::TWB);  // four-step twiddles of the tile
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + G::NBUF * G::STAGE + G::TWB + G::TVB);
  // (early-refill passes: the slice only the epilogue reads completes on its own barrier)
  uint64_t* bars_e = bars + G::NBUF;
  const int tid = threadIdx.x, cs = tid % CT, j = tid / CT;
  const uint32_t f = p.flags;
  const R sx = ((f & F_CONJX) != 0) != (!MID && (f & F_INV)) ? R(-1) : R(1);
  const bool pre_conj = MID || (f & F_INV);
  const bool twinv = (f & F_TWINV) != 0;
  const bool twpre = TW && (f & F_TWPRE) != 0;  // twiddle the input instead of the output
  const R sc = (f & F_SCALE) ? R(p.scale) : R(1);
  const R s_re = sc;
  // (MSK: the inverse conjugation stays explicit, a post vector sits between it and conj_y)
  const R s_im = ((f & F_CONJY) != 0) != (!TW && !MSK && pre_conj) ? -sc : sc;
  const R smid = (f & F_MIDCONJ) ? R(-1) : R(1);

  const bool side_pre = MSK && (f & F_SIDEPRE) != 0, side_post = MSK && (f & F_SIDEPOST) != 0;
  // early-refill passes: the slices read only by the epilogue (post vector,
  // output twiddles) — issued after it, waited for right before the next one
  const int emask = EARLY ? ((side_post ? 2 : 0) | (G::TVSL && !(TW && (f & F_TWPRE)) ? 4 : 0)) : 0;
  auto tile_goff = [&](int t) -> int {
    const uint32_t q = fdiv(uint32_t(t) * CT, p.gdiv.m, p.gdiv.s);
    return int(q - fdiv(q, p.gmod.m, p.gmod.s) * p.gmod.d);
  };
  // parts: 1 = the barrier's byte count and the tile box, 2 = the spectrum /
  // pre / post slice, 4 = the four-step twiddle slice (the early-refill passes
  // issue them apart: the box and the slice the prologue reads as soon as the
  // landing buffer is dead, the slice the epilogue reads after it)
  auto issue = [&](int t, int s, int parts = 7) {
    uint32_t o1, o2, c0;
    decode_batch(uint32_t(t) * CT, p.inner.d, p.inner.m, p.inner.s, p.n2.d, p.n2.m, p.n2.s, o1, o2, c0);
    const uint32_t sb = MID ? uint32_t(N * sizeof(C)) : (side_pre || side_post) ? uint32_t(N * sizeof(C)) : 0u;
    const uint32_t eb = ((emask & 2) ? sb : 0u) + ((emask & 4) ? uint32_t(G::TVSB) : 0u);
    if (parts & 1) {
      // (a masked box moves only the ein rows every tile owns)
      mbar_arrive_expect_tx(&bars[s], uint32_t(ein * CT * int(sizeof(C)) + G::TVSB) + sb - eb);
      if (f & F_WGRP)  // (4 real columns x 8 hh: virtual column c0 -> real column c0 / 8)
        tma_load_5d(stage_buf(s), &xmap, &bars[s], int((c0 / 8) * (sizeof(C) / 8)), 0, 0, int(o2), int(o1));
      else
        tma_load_5d(stage_buf(s), &xmap, &bars[s], int(c0 * (sizeof(C) / 8)), 0, 0, int(o2), int(o1));
    }
    if ((parts & emask) && eb) mbar_arrive_expect_tx(&bars_e[s], eb);  // (the epilogue's slices go out in one call)
    if ((parts & 6) && (sb || TVSL)) {
      // the tile's contiguous spectrum (or pre / post) and twiddle slices ride
      // on the same barrier
      const size_t g = size_t(tile_goff(t));
      if (sb && (parts & 2)) {
        const unsigned char* src =
            MID ? reinterpret_cast<const unsigned char*>(p.mid) + g * p.mid_gmul * sizeof(C)
                : side_pre ? reinterpret_cast<const unsigned char*>(p.pre) + g * p.pre_gmul * sizeof(C)
                           : reinterpret_cast<const unsigned char*>(p.post) + g * p.post_gmul * sizeof(C);
        bulk_load(stage_spec(s), src, sb, (emask & 2) ? &bars_e[s] : &bars[s]);
      }
      if constexpr (TVSL) {
        if (parts & 4)
          bulk_load(stage_tv(s), reinterpret_cast<const unsigned char*>(p.tw_slices) + g * N * 16, uint32_t(G::TVSB),
                    (emask & 4) ? &bars_e[s] : &bars[s]);
      }
    }
  };
  // rows ein .. ein+npatch-1: thread tid < npatch*CT owns row ein + tid/CT,
  // column tid%CT, and loads it one tile ahead
  const bool powner = MSK && tid < npatch * CT;
  const int prow = ein + tid / CT, pcol = tid % CT;
  auto patch_load = [&](int t) -> C {
    uint32_t o1, o2, c0;
    decode_batch(uint32_t(t) * CT, p.inner.d, p.inner.m, p.inner.s, p.n2.d, p.n2.m, p.n2.s, o1, o2, c0);
    int v = N;
    if (f & F_PAD) {
      const int rem = p.n_valid_in - tile_goff(t);
      v = rem <= 0 ? 0 : min(N, (rem + p.gin_stride - 1) / p.gin_stride);
    }
    const C* xc = (const C*)p.x + (int64_t(o1) * p.xs1 + int64_t(o2) * p.xs2 + c0 + pcol);
    return prow < v ? __ldg(&xc[int64_t(prow) * p.xsi]) : C{};
  };
  if constexpr (kPdl<C, N>) pdl_wait();  // (before any access to the previous pass's output)
  C pval{};
  if (powner && int(blockIdx.x) < ntiles) pval = patch_load(blockIdx.x);

  // tiles are dealt round-robin (tile t = blockIdx.x + i*gridDim.x): at any
  // moment the CTAs work on neighbouring column groups of the same rows, so
  // every DRAM page opened serves all of them
  const int gs = int(gridDim.x);
  if (tid == 0) {
    tma_prefetch_desc(&xmap);
    for (int s = 0; s < G::NBUF; ++s) mbar_init(&bars[s], 1);
    if constexpr (EARLY)
      for (int s = 0; s < G::NBUF; ++s) mbar_init(&bars_e[s], 1);
    fence_barrier_init();
    for (int s = 0; s < G::NBUF; ++s)
      if (int(blockIdx.x) + s * gs < ntiles) issue(blockIdx.x + s * gs, s);
  }
  // four-step twiddle software pipeline: the two-level table lookups of the
  // NEXT tile are issued during the current one
  constexpr int PER = (N + G::T - 1) / G::T;
  C tvlo[TW && !TVSL ? PER : 1], tvhi[TW && !TVSL ? PER : 1];
  auto tv_prefetch = [&](int t) {
    if constexpr (TW && !TVSL) {
      const uint32_t q = fdiv(uint32_t(t) * CT, p.gdiv.m, p.gdiv.s);
      const uint32_t g32 = q - fdiv(q, p.gmod.m, p.gmod.s) * p.gmod.d;
      const C* thi = (const C*)p.tw_hi;
      const C* tlo = (const C*)p.tw_lo;
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        const int k = tid + i * G::T;
        const uint32_t m = (g32 * uint32_t(k < N ? k : 0)) & p.tw_mask;
        tvhi[i] = __ldg(&thi[m >> p.tw_lo_bits]);
        tvlo[i] = __ldg(&tlo[m & ((1u << p.tw_lo_bits) - 1u)]);
      }
    }
  };
  if (int(blockIdx.x) < ntiles) tv_prefetch(blockIdx.x);
  // staged stage-twiddle table (st_twoff layout) from the global W_4096 table;
  // the spectrum passes' mirrored inverse transform runs the same stage list
  // when it is a palindrome and shares the table, else reads a second one
  constexpr bool DUAL = MID && G::DUAL;
  // (16-byte entries: float4 quads or double2)
  C* tws_mir = reinterpret_cast<C*>(reinterpret_cast<unsigned char*>(tws) + (DUAL ? N * int(G::TWE) : 0));
#pragma unroll
  for (int half = 0; half < (DUAL ? 2 : 1); ++half) {
    const bool mir = half == 1;
    for (int e = tid; e < N - st_radix(N, E, 0, mir); e += G::T) {
      int t4096 = 0;
#pragma unroll
      for (int S = 1; S < NST; ++S) {
        const int RS = st_radix(N, E, S, mir), NS = st_ns(N, E, S, mir), OFF = st_twoff(N, E, S, mir);
        if (e >= OFF && e < OFF + NS * (RS - 1)) {
          const int k = (e - OFF) / (RS - 1), r = (e - OFF) % (RS - 1) + 1;
          t4096 = (r * k * (4096 / (NS * RS))) & 4095;
        }
      }
      C* dst = mir ? tws_mir : tws;
      if constexpr (sizeof(C) == 8) {
        const float4 q = __ldg(reinterpret_cast<const float4*>(p.tw) + t4096);
        if constexpr (MID) dst[e] = make_float2(q.x, q.y);  // (plain entries, st_tw_mul<true>)
        else reinterpret_cast<float4*>(dst)[e] = q;
      } else {
        dst[e] = __ldg(reinterpret_cast<const C*>(p.tw) + t4096);
      }
    }
  }
  __syncthreads();

  for (int t = blockIdx.x, it = 0; t < ntiles; t += gs, ++it) {
    // ---- per-thread batch geometry
    const uint32_t b = uint32_t(t) * CT + cs;
    uint32_t o1, o2, c;
    decode_batch(b, p.inner.d, p.inner.m, p.inner.s, p.n2.d, p.n2.m, p.n2.s, o1, o2, c);
    const int64_t yb = int64_t(o1) * p.ys1 + int64_t(o2) * p.ys2 + c;
    int32_t goff = 0;
    if (f & F_GOFF) {
      const uint32_t q = fdiv(b, p.gdiv.m, p.gdiv.s);
      goff = int32_t(q - fdiv(q, p.gmod.m, p.gmod.s) * p.gmod.d);
    }
    // valid input rows i < vin, output rows k < vout of this tile
    int vin = N, vout = N;
    if constexpr (MSK) {
      // (ceil(rem / stride); the four-step strides are powers of two: a shift)
      auto cdiv = [](int rem, int st) {
        return (st & (st - 1)) == 0 ? (rem + st - 1) >> (__ffs(st) - 1) : (rem + st - 1) / st;
      };
      if (f & F_PAD) {
        const int rem = p.n_valid_in - goff;
        vin = rem <= 0 ? 0 : min(N, cdiv(rem, p.gin_stride));
      }
      if (f & F_TRUNC) {
        const int rem = p.n_valid_out - goff;
        vout = rem <= 0 ? 0 : min(N, cdiv(rem, p.gout_stride));
      }
    }
    if constexpr (TW && !TVSL) {
      // goff is uniform over the tile's CT columns (launcher checks): the
      // twiddles W^(goff*k) (conjugated for the inverse) are shared by all
      // columns — finish the lookups prefetched during the previous tile into
      // shared memory (the previous epilogue's reads are fenced by its
      // trailing barrier), then start the next tile's lookups.
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        const int k = tid + i * G::T;
        if (k < N) {
          C v = cmul(tvhi[i], tvlo[i]);
          if (twinv) v = conj(v);
          if constexpr (sizeof(C) == 8) reinterpret_cast<float4*>(tvs)[k] = make_float4(v.x, v.y, -v.y, v.x);
          else tvs[k] = v;
        }
      }
      if (t + gs < ntiles) tv_prefetch(t + gs);
      if (twpre) __syncthreads();  // read right below, by other threads
    }
    // ---- stage 0 from the landing buffer (natural row order)
    const int sidx = it % G::NBUF;
    C* buf = stage_buf(sidx);
    const C* tvt = TVSL ? stage_tv(sidx) : tvs;  // this tile's four-step twiddles
    mbar_wait(&bars[sidx], uint32_t((it / G::NBUF) & 1));
    if constexpr (MSK) {
      if (npatch > 0) {
        // rows ein.. were zero-filled by the TMA box: drop in the prefetched
        // values, then prefetch the next tile's
        if (powner) buf[prow * CT + pcol] = pval;
        __syncthreads();
        if (powner && t + gs < ntiles) pval = patch_load(t + gs);
      }
    }
    // (the fused half Walsh-Hadamard: strides < TPC in shared memory, the
    // rest in registers once loaded; the row mask applies after it)
    constexpr bool WHREG = (WH == 1 || WH == 2) && R0 == E && N / R0 == TPC && RL == E;
    if constexpr (WH == 1 && !(FFT_SKIP & 2)) {
      if constexpr (WHREG) tile_wht_half<C, N, CT, TPC, 1, TPC>(buf, j, cs);  // (ends with a barrier)
      else tile_wht_half<C, N, CT, TPC>(buf, j, cs);
    }
    C a[E];
#pragma unroll
    for (int u = 0; u < E / R0; ++u)
#pragma unroll
      for (int r = 0; r < R0; ++r) {
        // (rows past the tile's valid count were not loaded: zero padding)
        const int i = j + u * TPC + r * (N / R0);
        if constexpr (WH == 3 && CT == 64) {
          // (hh's top bit, cs bit 5: own and partner column of the landed row)
          const C o = buf[i * CT + cs], q = buf[i * CT + (cs ^ 32)];
          a[u * R0 + r] = (cs & 32) ? q - o : o + q;
        } else if constexpr (WH == 1 && WHREG) {
          a[u * R0 + r] = buf[i * CT + cs];
        } else {
          // (rows past the tile's valid count were not loaded: zero padding)
          a[u * R0 + r] = (!MSK || i < vin) ? buf[i * CT + cs] : C{};
        }
      }
    if constexpr (WH == 1 && WHREG) {
      if constexpr (!(FFT_SKIP & 2)) wht_regs_half(a);
      // rows >= N/2 (r >= 8) were not loaded; rows vin.. of the first half
      // are truncated Hadamard outputs
#pragma unroll
      for (int r = 8; r < E; ++r) a[r] = C{};
      if (vin < N / 2) {
#pragma unroll
        for (int r = 0; r < 8; ++r)
          if (!(j + r * TPC < vin)) a[r] = C{};
      }
    }
    if ((MSK && p.pre) || twpre) {
      // conj_x, the pre vector, the input twiddle, then the inverse conjugation
      if (f & F_CONJX) {
#pragma unroll
        for (int e = 0; e < E; ++e) a[e].y = -a[e].y;
      }
      if constexpr (MSK) {
        if (p.pre) {
          const C* pv = (const C*)p.pre;
          const C* ps = reinterpret_cast<const C*>(stage_spec(sidx));
          const bool pc = (f & F_PRECONJ) != 0;
          if (side_pre) {
            // (a per-tile slice is zero past the vector's end, and so are the
            // input rows: no guard)
            if (pc) {
#pragma unroll
              for (int u = 0; u < E / R0; ++u)
#pragma unroll
                for (int r = 0; r < R0; ++r)
                  a[u * R0 + r] = cmulc(a[u * R0 + r], ps[j + u * TPC + r * (N / R0)]);
            } else {
#pragma unroll
              for (int u = 0; u < E / R0; ++u)
#pragma unroll
                for (int r = 0; r < R0; ++r)
                  a[u * R0 + r] = cmul(a[u * R0 + r], ps[j + u * TPC + r * (N / R0)]);
            }
          } else {
#pragma unroll
            for (int u = 0; u < E / R0; ++u)
#pragma unroll
              for (int r = 0; r < R0; ++r) {
                const int i = j + u * TPC + r * (N / R0);
                if (i < vin) {
                  const C w = __ldg(&pv[p.pre_gmul ? goff * p.pre_gmul + i : goff + i * p.gin_stride]);
                  a[u * R0 + r] = pc ? cmulc(a[u * R0 + r], w) : cmul(a[u * R0 + r], w);
                }
              }
          }
        }
      }
      if constexpr (TW) {
        if (twpre) {
#pragma unroll
          for (int u = 0; u < E / R0; ++u)
#pragma unroll
            for (int r = 0; r < R0; ++r)
              a[u * R0 + r] = tw_mul<true>(a[u * R0 + r], tvt, j + u * TPC + r * (N / R0));
        }
      }
      if (!MID && (f & F_INV)) {
#pragma unroll
        for (int e = 0; e < E; ++e) a[e].y = -a[e].y;
      }
    } else if (sx < R(0)) {
#pragma unroll
      for (int e = 0; e < E; ++e) a[e].y = -a[e].y;
    }
    if constexpr (WH == 3) {
      static_assert(CT == 32 || CT == 64, "the fused Kron Walsh-Hadamard needs 32- or 64-column tiles");
      if constexpr (!(FFT_SKIP & 4)) wht_lanes8<C, E, CT>(a);
    }
    // Early refill (direct-store masked complex128 passes with one landing
    // buffer): once the last stage's inputs are in registers nothing reads
    // the landing buffer again, so the next tile's box is issued there — its
    // latency runs under the last radix-16 stage, the epilogue and the stores
    // instead of after them — together with the slice the prologue reads (the
    // fused output Walsh-Hadamard keeps the whole side area for its rows, WH = 2).
    auto early_refill = [&]() {
      __syncthreads();
      if (tid == 0 && t + G::NBUF * gs < ntiles) {
        fence_proxy_async();
        issue(t + G::NBUF * gs, sidx,
              1 | (WH != 2 && side_pre ? 2 : 0) | (WH != 2 && twpre ? 4 : 0));
      }
    };
    auto deferred_refill = [&]() {
      if (tid == 0 && pend_t >= 0) {
        bulk_wait_read0();
        issue(pend_t, (it + G::NBUF - 1) % G::NBUF);
        pend_t = -1;
      }
    };
    if constexpr (!(FFT_SKIP & 1)) {
      if constexpr (DEFER_START) deferred_refill();
      if constexpr (DEFER && !DEFER_START) fft_stages<C, N, E, CT, false, 0, LAY, N, true, MID>(a, buf, j, cs, tws, deferred_refill);
      else if constexpr (EARLY) fft_stages<C, N, E, CT, false, 0, LAY, N, true, MID>(a, buf, j, cs, tws, early_refill);
      else fft_stages<C, N, E, CT, false, 0, LAY, N, true, MID>(a, buf, j, cs, tws);
    }
    if constexpr (MID) {
      constexpr int RF = st_radix(N, E, NST - 1, false);
      // the tile's spectrum slice landed in shared memory with the data
      if constexpr (sizeof(C) == 8) {
        // plain spectrum: conj(a*s) = conj(a s); conj(a*conj s) = conj(a) s
        const float2* ms = reinterpret_cast<const float2*>(stage_spec(sidx));
        // (the conjugation variant chosen once per tile, not per element)
        if ((f & F_MIDCONJ) != 0) {
#pragma unroll
          for (int u = 0; u < E / RF; ++u)
#pragma unroll
            for (int r = 0; r < RF; ++r)
              a[u * RF + r] = cmul_f2(conj(a[u * RF + r]), ms[j + u * TPC + r * (N / RF)]);
        } else {
#pragma unroll
          for (int u = 0; u < E / RF; ++u)
#pragma unroll
            for (int r = 0; r < RF; ++r)
              a[u * RF + r] = conj(cmul_f2(a[u * RF + r], ms[j + u * TPC + r * (N / RF)]));
        }
      } else {
        // conj(a s) or conj(a conj(s)), the sign chosen once per tile
        const C* mid = reinterpret_cast<const C*>(stage_spec(sidx));
        if (smid < R(0)) {
#pragma unroll
          for (int u = 0; u < E / RF; ++u)
#pragma unroll
            for (int r = 0; r < RF; ++r) {
              const C sv = mid[j + u * TPC + r * (N / RF)];
              C& v = a[u * RF + r];
              v = mk(fma(v.x, sv.x, v.y * sv.y), fma(v.x, sv.y, -v.y * sv.x));
            }
        } else {
#pragma unroll
          for (int u = 0; u < E / RF; ++u)
#pragma unroll
            for (int r = 0; r < RF; ++r) {
              const C sv = mid[j + u * TPC + r * (N / RF)];
              C& v = a[u * RF + r];
              v = mk(fma(v.x, sv.x, -v.y * sv.y), fma(-v.x, sv.y, -v.y * sv.x));
            }
        }
      }
      if constexpr (!(FFT_SKIP & 1)) fft_stages<C, N, E, CT, true, 0, LAY, N, true, MID>(a, buf, j, cs, tws_mir);
    }
    // all exchange reads of the landing buffer are done after this barrier
    // (the early refill's barrier already was that point)
    if constexpr (!EARLY) __syncthreads();
    // (the epilogue still reads a post slice or output twiddle slice of the stage)
    const bool late_refill = side_post || (TVSL && !twpre);
    if constexpr (!TS && !EARLY) {
      // the landing buffer is free: start the load NBUF tiles ahead (after the
      // epilogue when it still reads the stage's side area)
      if (!late_refill && tid == 0 && t + G::NBUF * gs < ntiles) {
        fence_proxy_async();
        issue(t + G::NBUF * gs, sidx);
      }
    }
    // ---- epilogue: four-step twiddle, conj/scale, then either direct stores
    //      (TS = false) or a staged tile written back by one TMA store
    C* yc = (C*)p.y + yb;
    if constexpr (EARLY) {
      // (the epilogue's slices were issued after the previous tile's epilogue)
      if (emask) mbar_wait(&bars_e[sidx], uint32_t((it / G::NBUF) & 1));
    }
#pragma unroll
    for (int u = 0; u < E / RL; ++u) {
      const int bb = j + u * TPC;
      C* au = a + u * RL;
      if constexpr ((TW || MSK) && sizeof(C) == 16) {
        // (folded into s_im otherwise; tile-uniform branches outside the
        // element loops, no per-element selects: complex128 outer passes
        // 2.34 / 2.07 -> 2.20 / 1.88 ms)
        if (pre_conj) {
#pragma unroll
          for (int r = 0; r < RL; ++r) au[r].y = -au[r].y;
        }
        if constexpr (TW) {
          if (!twpre) {
#pragma unroll
            for (int r = 0; r < RL; ++r) au[r] = tw_mul<true>(au[r], tvt, bb + r * (N / RL));
          }
        }
      } else if constexpr (TW || MSK) {
        // (single precision: the select folds into the packed twiddle multiply)
#pragma unroll
        for (int r = 0; r < RL; ++r) {
          C v = pre_conj ? conj(au[r]) : au[r];
          if constexpr (TW) {
            if (!twpre) v = tw_mul<true>(v, tvt, bb + r * (N / RL));
          }
          au[r] = v;
        }
      }
      if constexpr (MSK) {
        if (p.post) {
          const C* qv = (const C*)p.post;
          const C* qs = reinterpret_cast<const C*>(stage_spec(sidx));
          const bool qc = (f & F_POSTCONJ) != 0;
          if (side_post) {
            // (the slice is zero past the vector's end; rows >= vout are never stored)
            if (qc) {
#pragma unroll
              for (int r = 0; r < RL; ++r) au[r] = cmulc(au[r], qs[bb + r * (N / RL)]);
            } else {
#pragma unroll
              for (int r = 0; r < RL; ++r) au[r] = cmul(au[r], qs[bb + r * (N / RL)]);
            }
          } else {
#pragma unroll
            for (int r = 0; r < RL; ++r) {
              const int k = bb + r * (N / RL);
              if (k < vout) {
                const C w = __ldg(&qv[p.post_gmul ? goff * p.post_gmul + k : goff + k * p.gout_stride]);
                au[r] = qc ? cmulc(au[r], w) : cmul(au[r], w);
              }
            }
          }
        }
      }
      C* yk = yc + int64_t(bb) * p.ysi;
      if (s_re != R(1) || s_im != R(1)) {
#pragma unroll
        for (int r = 0; r < RL; ++r) {
          au[r].x *= s_re;
          au[r].y *= s_im;
        }
      }
      if constexpr (WH == 2 && WHREG && !(FFT_SKIP & 2)) wht_regs_half(au);
      if constexpr (WH == 2 && !TS) {
        // Direct-store variant of the fused output Walsh-Hadamard: its
        // shared-memory stages (strides < TPC over the first N/2 rows, 32 KB
        // for a 4-column complex128 tile) run in the stage's side area, dead
        // once the post multiply above has read it — the landing buffer is
        // being refilled meanwhile — and the finished rows go straight to HBM.
        static_assert(WHREG && E == RL && G::SPB + G::TVSB >= size_t(N / 2) * CT * sizeof(C),
                      "the side area must hold the first half of the tile");
        C* scr = reinterpret_cast<C*>(stage_spec(sidx));
        __syncthreads();  // every thread has read its post / twiddle slice entries
#pragma unroll
        for (int r = 0; r < 8; ++r) scr[wht_row<true>(bb + r * TPC) * CT + cs] = au[r];
        __syncthreads();
        if constexpr (!(FFT_SKIP & 2)) tile_wht_half<C, N, CT, TPC, 1, TPC, true>(scr, j, cs);  // (ends with a barrier)
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const int k = bb + r * TPC;
          if (k < vout) yk[int64_t(r * TPC) * p.ysi] = scr[wht_row<true>(k) * CT + cs];
        }
      } else {
#pragma unroll
        for (int r = 0; r < RL; ++r) {
          const int k = bb + r * (N / RL);
          if constexpr (TS) {
            buf[k * CT + cs] = au[r];
          } else if (!MSK || k < vout) {
            yk[int64_t(r * (N / RL)) * p.ysi] = au[r];
          }
        }
      }
      if constexpr (MSK && TS) {
        // rows eout <= k < vout lie outside the store map: the tiles that own
        // such rows write them directly
        if (vout > eout) {
#pragma unroll
          for (int r = 0; r < RL; ++r) {
            const int k = bb + r * (N / RL);
            if (k >= eout && k < vout) yk[int64_t(r * (N / RL)) * p.ysi] = au[r];
          }
        }
      }
    }
    if constexpr (EARLY) {
      __syncthreads();  // side area read
      if (tid == 0 && t + G::NBUF * gs < ntiles) {
        fence_proxy_async();
        issue(t + G::NBUF * gs, sidx,
              (WH != 2 && side_pre ? 0 : 2) | (WH != 2 && twpre ? 0 : 4));
      }
    } else if constexpr (!TS) {
      if (TW || late_refill) __syncthreads();  // tile twiddles are rebuilt next / side area read
      if (late_refill && tid == 0 && t + G::NBUF * gs < ntiles) {
        fence_proxy_async();
        issue(t + G::NBUF * gs, sidx);
      }
    }
    if constexpr (TS) {
      if constexpr (WH == 2 && !(FFT_SKIP & 2)) {
        __syncthreads();
        if constexpr (WHREG) tile_wht_half<C, N, CT, TPC, 1, TPC>(buf, j, cs);
        else tile_wht_half<C, N, CT, TPC>(buf, j, cs);
      }
      fence_proxy_async();  // this thread's tile writes -> visible to the TMA engine
      __syncthreads();
      if (tid == 0) {
        uint32_t q1, q2, c0;
        decode_batch(uint32_t(t) * CT, p.inner.d, p.inner.m, p.inner.s, p.n2.d, p.n2.m, p.n2.s, q1, q2, c0);
        if (f & F_WGRP)
          tma_store_5d(&ymap, buf, int((c0 / 8) * (sizeof(C) / 8)), 0, 0, int(q2), int(q1));
        else
          tma_store_5d(&ymap, buf, int(c0 * (sizeof(C) / 8)), 0, 0, int(q2), int(q1));
        bulk_commit();
        // refill the buffer once the store has read it — here, or (DEFER) from
        // inside the next tile, where this thread no longer has to wait
        if constexpr (DEFER) {
          pend_t = t + G::NBUF * gs < ntiles ? t + G::NBUF * gs : -1;
        } else if (t + G::NBUF * gs < ntiles) {
          bulk_wait_read0();
          issue(t + G::NBUF * gs, sidx);
        }
      }
    }
  }
  if constexpr (TS) {
    if (tid == 0) bulk_wait0();
  }
}

// Launch when the pass qualifies (complex in/out, no masks, TMA-compatible
// view); returns false so the caller falls back to the per-tile kernel.
template <class C, int N, int EP, int NB, int CTO = 0>
inline bool fft_tma_launch_v(const FftArgs& a, cudaStream_t s) {
  using G = TmaGeom<C, N, EP, NB, false, false, CTO>;
  if (a.x_real || a.y_real || a.accumulate || a.in_map || a.out_map) return false;
  if (a.inner % G::CT != 0) return false;
  const FftDev d0 = make_fft_dev(a, N);
  const bool pad = (d0.flags & F_PAD) != 0, trunc = (d0.flags & F_TRUNC) != 0;
  const bool msk = pad || trunc || a.pre || a.post;
  // per-tile shared four-step twiddles / spectrum slices / valid row counts
  // need goff uniform across a tile, and the slice must be contiguous
  if ((a.tw_on || a.mid || msk) && a.g_mod > 1 && (a.g_div % G::CT) != 0) return false;
  if (a.mid && a.mid_stride != 1) return false;
  if (msk && (a.mid || a.gin_stride < 1 || a.gout_stride < 1)) return false;
  // masked maps: rows split as (i % rlo, i / rlo) with the smallest rlo the
  // 256-entry box limit allows, covering the rows valid for every tile
  const int64_t rlo = N > 256 ? N / 256 : 1;
  auto extent = [&](int64_t nv, int64_t gs) {
    const int64_t rem = nv - (a.g_mod - 1);
    int64_t v = rem <= 0 ? 0 : (rem + gs - 1) / gs;
    if (v > N) v = N;
    return (v / rlo) * rlo;
  };
  // (a fused Walsh-Hadamard over the first N/2 input rows needs all of them
  // landed: the row mask applies after it, in registers)
  const int64_t ein = a.wht_half == 1 ? N / 2 : pad ? extent(a.n_valid_in, a.gin_stride) : N;
  const int64_t eout = trunc ? extent(a.n_valid_out, a.gout_stride) : N;
  if (ein == 0) return false;
  if (a.wht_half && !(msk && a.tw_on && !a.mid)) return false;
  if (a.wht_half == 2 && eout > N / 2) return false;
  // rows from ein that only some tiles own (the tile with goff = 0 owns the most)
  int64_t npatch = 0;
  if (pad && !a.wht_half) {
    int64_t v0 = (a.n_valid_in + a.gin_stride - 1) / a.gin_stride;
    if (v0 > N) v0 = N;
    npatch = v0 - ein;
    if (npatch * G::CT > G::T) return false;
  }
  FftDev d = d0;
  if (a.wht_grp) d.flags |= F_WGRP;
  if (msk && a.pre && a.pre_gmul) d.flags |= F_SIDEPRE;
  else if (msk && a.post && a.post_gmul) d.flags |= F_SIDEPOST;
  const int64_t n1 = a.nb / (a.n2 * a.inner);
  // two-level rows (blocked four-step intermediate): the row split of the map
  // is the blocking itself; masks and direct row accesses stay single-level
  const int64_t blo = a.i_lo_bits ? (int64_t(1) << a.i_lo_bits) : 0;
  if (blo && (msk || blo > 256 || N / blo > 256 || N % blo)) return false;
  CUtensorMap map, ymap;
  if (a.wht_grp) {
    // fused Kron Walsh-Hadamard: both sides as {columns, hh, rows, o2, o1}
    // with 4-column x 8-hh boxes (single-dimension rows: N <= 256)
    if ((G::CT != 32 && G::CT != 64) || N > 256 || msk || a.tw_on || blo || a.wht_half ||
        a.inner % G::CT || a.x_real || a.y_real)
      return false;
    const int64_t ic = a.inner / 8;
    auto gmap = [&](CUtensorMap* m, const void* ptr, int64_t s1, int64_t s2, int64_t si, int64_t sw) {
      auto fn = encode_fn();
      if (!fn || (reinterpret_cast<uintptr_t>(ptr) & 15)) return false;
      const int64_t w = int64_t(sizeof(C) / 8), e = int64_t(sizeof(C));
      const int64_t n1v = a.nb / (a.n2 * a.inner);
      cuuint64_t dims[5] = {cuuint64_t(ic * w), 8, cuuint64_t(N), cuuint64_t(a.n2), cuuint64_t(n1v)};
      cuuint64_t strides[4] = {cuuint64_t(sw * e), cuuint64_t(si * e), cuuint64_t(s2 * e), cuuint64_t(s1 * e)};
      for (int k = 0; k < 4; ++k) {
        if (dims[k + 1] == 1) strides[k] = 16;
        if (strides[k] % 16 || strides[k] >= (cuuint64_t(1) << 40)) return false;
      }
      cuuint32_t box[5] = {cuuint32_t(G::CT / 8 * w), 8, cuuint32_t(N), 1, 1}, estr[5] = {1, 1, 1, 1, 1};
      return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 5, const_cast<void*>(ptr), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    };
    if (!gmap(&map, a.x, a.xs1, a.xs2, a.xsi, a.wg_xs) || !gmap(&ymap, a.y, a.ys1, a.ys2, a.ysi, a.wg_ys))
      return false;
  }
  const bool pin = pad || a.wht_half == 1;
  if (a.wht_grp) {
    // (maps built above)
  } else if (!make_view_map(&map, a.x, sizeof(C), n1, a.xs1, a.n2, a.xs2, N, a.xsi, a.inner, G::CT,
                            blo ? blo : pin ? rlo : 0, pin ? ein : 0, pin, blo ? a.xsi_hi : 0)) {
    return false;
  }
  // TMA-store epilogue when the output view is TMA-compatible as well
  // complex128 1024-point masked twiddle passes (one landing buffer, two CTAs
  // per SM: the C5 outer passes) store per thread and refill the buffer early
  const bool direct = sizeof(C) == 16 && NB == 1 && msk && a.tw_on && !a.mid && !a.wht_grp && !blo;
  const bool ts = eout > 0 && !direct &&
                  (a.wht_grp ? true
                             : make_view_map(&ymap, a.y, sizeof(C), n1, a.ys1, a.n2, a.ys2, N, a.ysi, a.inner, G::CT,
                                             blo ? blo : trunc ? rlo : 0, trunc ? eout : 0, trunc,
                                             blo ? a.ysi_hi : 0));
  if (!ts && (blo || a.wht_grp)) return false;  // direct stores are single-level, ungrouped
  if (!ts) ymap = map;
  const int64_t ntiles = a.nb / G::CT;
  if (ntiles <= 0) return true;
  int dev = 0;
  cudaGetDevice(&dev);
  auto pick = [&](auto ts_tag, auto mid_tag, auto tw_tag, auto msk_tag, auto wh_tag) {
    constexpr bool TSV = decltype(ts_tag)::value, MV = decltype(mid_tag)::value, TV = decltype(tw_tag)::value,
                   KV = decltype(msk_tag)::value;
    constexpr int WHV = decltype(wh_tag)::value;
    using GV = TmaGeom<C, N, EP, NB, TV, MV ? 1 : KV ? 2 : 0, CTO>;
    if constexpr (GV::SMEM > 232448) {
      return false;  // does not fit one SM: per-tile kernel
    } else {
      if (GV::TVSL && !a.tw_slices) return false;  // needs the precomputed twiddle slices
      if (a.probe_only) return true;
      const int64_t slots = int64_t(num_sms(dev)) * GV::MINB;
      const int grid = int(ntiles < slots ? ntiles : slots);
      auto kern = fft_tma_kernel<C, N, MV, TV, EP, NB, TSV, KV, CTO, WHV>;
      set_smem(kern, GV::SMEM);
      if (kPdl<C, N>) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(unsigned(grid));
        cfg.blockDim = dim3(unsigned(GV::T));
        cfg.dynamicSmemBytes = GV::SMEM;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        SMAT_CUDA(cudaLaunchKernelEx(&cfg, kern, map, ymap, d, int(ntiles), int(ein), int(eout), int(npatch)));
      } else {
        kern<<<grid, GV::T, GV::SMEM, s>>>(map, ymap, d, int(ntiles), int(ein), int(eout), int(npatch));
      }
      return true;
    }
  };
  using T_ = std::true_type;
  using F_ = std::false_type;
  using W0 = std::integral_constant<int, 0>;
  auto pick2 = [&](auto ts_tag) -> bool {
    if (a.wht_grp) {
      if constexpr (decltype(ts_tag)::value && (CTO == 32 || CTO == 64) && G::CT == CTO && N <= 256) {
        using W3 = std::integral_constant<int, 3>;
        return a.mid ? pick(ts_tag, T_{}, F_{}, F_{}, W3{}) : pick(ts_tag, F_{}, F_{}, F_{}, W3{});
      }
      return false;
    }
    if (msk) {
      if (a.tw_on) {
        // (the fused Walsh-Hadamard variants: complex128 passes of the C5 chain)
        if constexpr (sizeof(C) == 16 && N >= 256) {
          if (a.wht_half == 1) return pick(ts_tag, F_{}, T_{}, T_{}, std::integral_constant<int, 1>{});
          if constexpr (decltype(ts_tag)::value || (N == 1024 && NB == 1)) {
            if (a.wht_half == 2) return pick(ts_tag, F_{}, T_{}, T_{}, std::integral_constant<int, 2>{});
          }
        }
        if (a.wht_half) return false;
        return pick(ts_tag, F_{}, T_{}, T_{}, W0{});
      }
      return pick(ts_tag, F_{}, F_{}, T_{}, W0{});
    }
    if (a.mid && a.tw_on) return pick(ts_tag, T_{}, T_{}, F_{}, W0{});
    if (a.mid) return pick(ts_tag, T_{}, F_{}, F_{}, W0{});
    if (a.tw_on) return pick(ts_tag, F_{}, T_{}, F_{}, W0{});
    return pick(ts_tag, F_{}, F_{}, F_{}, W0{});
  };
  const bool ok = ts ? pick2(T_{}) : pick2(F_{});
  if (ok) SMAT_CUDA(cudaGetLastError());
  return ok;
}

// Variant choice (measured, round 1): radix-32 stages and a
// 3-deep landing ring for complex64 >= 1024 points; complex128 1024-point
// passes with one landing buffer and two CTAs (16 warps) per SM except the
// spectrum passes (at 128 registers their FFT + IFFT spills), which keep two
// buffers — these passes are issue-latency bound at 8 warps per SM, and the
// second CTA hides more of it than the lost load lead costs (C5 outer passes
// 2.34 / 2.00 -> 2.09 / 1.78 ms); radix-16 stages everywhere else.  Tried and
// dropped: radix-16 / radix-8 stages for the long complex64 passes, radix-8
// stages for complex128, 1/2/4-column complex128 tiles, single-buffer spectrum
// passes.
template <class C, int N>
inline bool fft_tma_launch(const FftArgs& a, cudaStream_t s) {
  // (the fused Kron Walsh-Hadamard passes, complex64: 128 points on 64-column
  // tiles — 8 columns x 8 hh, 64-byte rows — and 256 points on 32-column tiles)
  if constexpr (sizeof(C) == 8 && N == 128) {
    if (a.wht_grp) return fft_tma_launch_v<C, N, 16, 0, 64>(a, s);
  }
  if constexpr (sizeof(C) == 8 && N == 256) {
    if (a.wht_grp) return fft_tma_launch_v<C, N, 16, 0, 32>(a, s);
  }
  if (a.wht_grp) return false;
  if constexpr (N == 1024 && sizeof(C) == 16) {
    if (!a.mid) return fft_tma_launch_v<C, N, 16, 1>(a, s);
  }
  if constexpr (N >= 1024 && sizeof(C) == 8) return fft_tma_launch_v<C, N, 32, 3>(a, s);
  return fft_tma_launch_v<C, N, 16, 0>(a, s);
}

}  // namespace smat
