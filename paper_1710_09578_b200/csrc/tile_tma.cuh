// tile_tma.cuh — persistent, TMA-fed FFT tile pass.
//
// Same math as fft_tile_kernel's fast variant (tile_impl.cuh), restructured for
// HBM throughput on sm_100a:
//   * persistent CTAs (two per SM) walk over tiles of CT columns x N rows;
//   * one elected thread loads a whole tile with a single 5-D TMA box
//     (cp.async.bulk.tensor) into a dense shared buffer, tracked by an
//     mbarrier — no load instructions, addresses or registers in the math warps;
//   * the landing buffer doubles as the exchange buffer (rows permuted as
//     row ^ ((row >> 4) & (X-1)) to stay bank-conflict free), so a CTA needs
//     one tile of shared memory plus its twiddle table and two CTAs fit per SM:
//     while one CTA shuffles and computes, the other's TMA load is in flight;
//   * stage twiddles come from a per-CTA shared copy of W_N (quad layout in
//     single precision: every twiddle multiply is FMUL2 + FFMA2);
//   * four-step twiddles are looked up before the transform so their latency
//     hides behind it; results leave straight from registers.
#pragma once

#include "tile_impl.cuh"
#include "tma.cuh"

namespace smat {

template <class C, int N>
struct TmaGeom {
  static constexpr int E = tile_E(N);
  static constexpr int CT = tile_CT(N, sizeof(C));
  static constexpr int TPC = N / E;
  static constexpr int T = TPC * CT;
  static constexpr int ROWB = CT * int(sizeof(C));                 // bytes per tile row
  static constexpr int LAY = ROWB >= 128 ? 1 : 128 / ROWB;          // exchange row permutation
  static constexpr size_t BUF = size_t(N) * CT * sizeof(C);         // one dense TMA box
  static constexpr size_t TWB = size_t(N) * 16;                    // W_N (float4 quads / double2)
  // ring of landing buffers: tile t computes in one while t+1.. load into the others
  static constexpr int NBUF = (227 * 1024 - int(TWB) - 64) / int(BUF) >= 3 ? 3 : 2;
  static constexpr size_t SMEM = NBUF * BUF + TWB + 64;
  static constexpr int MINB = (227 * 1024) / int(SMEM) >= 2 && 2 * T <= 1024 ? 2 : 1;
};

template <class C, int N, bool MID, bool TW>
__global__ void __launch_bounds__(TmaGeom<C, N>::T, TmaGeom<C, N>::MINB)
    fft_tma_kernel(const __grid_constant__ CUtensorMap xmap, const FftDev p, const int ntiles) {
  using G = TmaGeom<C, N>;
  using R = typename RealOf<C>::T;
  constexpr int E = G::E, CT = G::CT, TPC = G::TPC, LAY = G::LAY;
  constexpr int NST = st_count(N, E);
  constexpr int R0 = st_radix(N, E, 0, false);
  constexpr int RL = MID ? st_radix(N, E, NST - 1, true) : st_radix(N, E, NST - 1, false);
  constexpr int LQ = log2_c(RL);
  extern __shared__ __align__(128) unsigned char smem_raw[];
  C* bufs = reinterpret_cast<C*>(smem_raw);
  C* tws = reinterpret_cast<C*>(smem_raw + G::NBUF * G::BUF);  // W_N^t, t < N (float4 quads or double2)
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + G::NBUF * G::BUF + G::TWB);
  const int tid = threadIdx.x, cs = tid % CT, j = tid / CT;
  const uint32_t f = p.flags;
  const R sx = ((f & F_CONJX) != 0) != (!MID && (f & F_INV)) ? R(-1) : R(1);
  const bool pre_conj = MID || (f & F_INV);
  const bool twinv = (f & F_TWINV) != 0;
  const R sc = (f & F_SCALE) ? R(p.scale) : R(1);
  const R s_re = sc;
  const R s_im = ((f & F_CONJY) != 0) != (!TW && pre_conj) ? -sc : sc;
  const R smid = (f & F_MIDCONJ) ? R(-1) : R(1);

  auto issue = [&](int t, int s) {
    uint32_t o1, o2, c0;
    decode_batch(uint32_t(t) * CT, p.inner.d, p.inner.m, p.inner.s, p.n2.d, p.n2.m, p.n2.s, o1, o2, c0);
    mbar_arrive_expect_tx(&bars[s], uint32_t(G::BUF));
    tma_load_5d(bufs + s * (G::BUF / sizeof(C)), &xmap, &bars[s], int(c0 * (sizeof(C) / 8)), 0, 0, int(o2),
                int(o1));
  };

  if (tid == 0) {
    tma_prefetch_desc(&xmap);
    for (int s = 0; s < G::NBUF; ++s) mbar_init(&bars[s], 1);
    fence_barrier_init();
    for (int s = 0; s < G::NBUF; ++s)
      if (int(blockIdx.x + s * gridDim.x) < ntiles) issue(blockIdx.x + s * gridDim.x, s);
  }
  // shared copy of W_N from the global W_4096 table (stride 4096/N)
  {
    constexpr int st = 4096 / N;
    if constexpr (sizeof(C) == 8) {
      const float4* g = reinterpret_cast<const float4*>(p.tw);
      float4* s = reinterpret_cast<float4*>(tws);
      for (int t = tid; t < N; t += G::T) s[t] = __ldg(&g[t * st]);
    } else {
      const C* g = reinterpret_cast<const C*>(p.tw);
      for (int t = tid; t < N; t += G::T) tws[t] = __ldg(&g[t * st]);
    }
  }
  __syncthreads();

  for (int t = blockIdx.x, it = 0; t < ntiles; t += gridDim.x, ++it) {
    // ---- per-thread batch geometry and four-step twiddles (latency hidden
    //      behind the TMA wait and the transform)
    const uint32_t b = uint32_t(t) * CT + cs;
    uint32_t o1, o2, c;
    decode_batch(b, p.inner.d, p.inner.m, p.inner.s, p.n2.d, p.n2.m, p.n2.s, o1, o2, c);
    const int64_t yb = int64_t(o1) * p.ys1 + int64_t(o2) * p.ys2 + c;
    int32_t goff = 0;
    if (f & F_GOFF) {
      const uint32_t q = fdiv(b, p.gdiv.m, p.gdiv.s);
      goff = int32_t(q - fdiv(q, p.gmod.m, p.gmod.s) * p.gmod.d);
    }
    C wbase[E / RL];
    C wp[LQ > 0 ? LQ : 1];
    if constexpr (TW) {
      const uint32_t g32 = uint32_t(goff);
      const C* thi = (const C*)p.tw_hi;
      const C* tlo = (const C*)p.tw_lo;
#pragma unroll
      for (int q = 0; q < LQ; ++q) wp[q] = tw2<C>(thi, tlo, p.tw_mask, p.tw_lo_bits, g32 * uint32_t((N / RL) << q));
#pragma unroll
      for (int u = 0; u < E / RL; ++u)
        wbase[u] = tw2<C>(thi, tlo, p.tw_mask, p.tw_lo_bits, g32 * uint32_t(j + u * TPC));
    }
    // ---- stage 0 from the landing buffer (natural row order)
    const int sidx = it % G::NBUF;
    C* buf = bufs + sidx * (G::BUF / sizeof(C));
    mbar_wait(&bars[sidx], uint32_t((it / G::NBUF) & 1));
    C a[E];
#pragma unroll
    for (int u = 0; u < E / R0; ++u)
#pragma unroll
      for (int r = 0; r < R0; ++r) {
        C v = buf[(j + u * TPC + r * (N / R0)) * CT + cs];
        v.y *= sx;
        a[u * R0 + r] = v;
      }
    fft_stages<C, N, E, CT, false, 0, LAY, N, true>(a, buf, j, cs, tws);
    if constexpr (MID) {
      constexpr int RF = st_radix(N, E, NST - 1, false);
      const C* mid = (const C*)p.mid + goff * p.mid_gmul;
#pragma unroll
      for (int u = 0; u < E / RF; ++u)
#pragma unroll
        for (int r = 0; r < RF; ++r) {
          const int k = j + u * TPC + r * (N / RF);
          C sv = __ldg(&mid[k * p.mid_stride]);
          sv.y *= smid;
          a[u * RF + r] = conj(cmul(a[u * RF + r], sv));
        }
      fft_stages<C, N, E, CT, true, 0, LAY, N, true>(a, buf, j, cs, tws);
    }
    // ---- the landing buffer is free: start the load NBUF tiles ahead
    __syncthreads();
    if (tid == 0 && t + G::NBUF * int(gridDim.x) < ntiles) {
      fence_proxy_async();
      issue(t + G::NBUF * gridDim.x, sidx);
    }
    // ---- epilogue straight from registers
    C* yc = (C*)p.y + yb;
#pragma unroll
    for (int u = 0; u < E / RL; ++u) {
      const int bb = j + u * TPC;
      C* au = a + u * RL;
      if constexpr (TW) {
        if (pre_conj != twinv) {
#pragma unroll
          for (int r = 0; r < RL; ++r) au[r] = conj(au[r]);
        }
        au[0] = cmul(au[0], wbase[u]);
        apply_powers<RL>(au, wp);
#pragma unroll
        for (int r = 1; r < RL; ++r) au[r] = cmul(au[r], wbase[u]);
        if (twinv) {
#pragma unroll
          for (int r = 0; r < RL; ++r) au[r] = conj(au[r]);
        }
      }
      C* yk = yc + int64_t(bb) * p.ysi;
#pragma unroll
      for (int r = 0; r < RL; ++r) {
        C v = au[r];
        v.x *= s_re;
        v.y *= s_im;
        yk[int64_t(r * (N / RL)) * p.ysi] = v;
      }
    }
  }
}

// Launch when the pass qualifies (complex in/out, no masks, TMA-compatible
// view); returns false so the caller falls back to the per-tile kernel.
template <class C, int N>
inline bool fft_tma_launch(const FftArgs& a, cudaStream_t s) {
  using G = TmaGeom<C, N>;
  if (a.x_real || a.y_real || a.pre || a.post || a.accumulate) return false;
  if (a.inner % G::CT != 0) return false;
  const FftDev d = make_fft_dev(a, N);
  if (d.flags & (F_PAD | F_TRUNC)) return false;
  const int64_t n1 = a.nb / (a.n2 * a.inner);
  CUtensorMap map;
  if (!make_view_map(&map, a.x, sizeof(C), n1, a.xs1, a.n2, a.xs2, N, a.xsi, a.inner, G::CT)) return false;
  const int64_t ntiles = a.nb / G::CT;
  if (ntiles <= 0) return true;
  int dev = 0;
  cudaGetDevice(&dev);
  const int64_t slots = int64_t(num_sms(dev)) * G::MINB;
  const int grid = int(ntiles < slots ? ntiles : slots);
  auto kern = fft_tma_kernel<C, N, false, false>;
  if (a.mid && a.tw_on) kern = fft_tma_kernel<C, N, true, true>;
  else if (a.mid) kern = fft_tma_kernel<C, N, true, false>;
  else if (a.tw_on) kern = fft_tma_kernel<C, N, false, true>;
  set_smem(kern, G::SMEM);
  kern<<<grid, G::T, G::SMEM, s>>>(map, d, int(ntiles));
  SMAT_CUDA(cudaGetLastError());
  return true;
}

}  // namespace smat
