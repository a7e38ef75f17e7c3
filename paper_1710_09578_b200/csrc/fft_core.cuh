// fft_core.cuh — register/shared-memory FFT and FWHT building blocks (sm_100a).
//
// Replaces the numpy radix-2 DIT of the reference (DftPlan._pow2,
// pkg/src/linopkit/kernels.py:95-109: bit-reversal gather + log2 n full-array
// passes) by a Stockham auto-sort formulation computed in registers: every
// thread owns E elements of one column, performs radix-R butterflies on them
// (R in {2,4,8,16}, constant twiddles folded at compile time) and exchanges
// through shared memory between stages.  No bit-reversal pass exists; input
// and output are both in natural order, so the first stage loads straight
// from HBM and the last stage stores straight to HBM.
//
// The FWHT (kernels.py:164-190) uses the same thread/element geometry without
// twiddles and keeps the reference's stage order (stride 1, 2, 4, ... — stride-1
// first, kernels.py:181-189), which makes fp64 results bit-identical to the
// reference and integer results exact.
//
// Shared-memory layout: element (row, column-slot cs) of a tile lives at
// sm[(row + row/16) * CT + cs].  Skipping one row every 16 rows puts the rows
// a warp touches in the radix-16 scatter (rows 16 apart) on different bank
// halves/quarters, so every exchange runs at the 256-byte-per-warp minimum.
#pragma once

#include "common.cuh"

namespace smat {

// ------------------------------------------------------ stage bookkeeping --
// A length-N transform with E elements per thread runs stages of radix E and
// at most one smaller remainder stage.  The FFT puts the remainder in the
// middle when the E-stages split evenly around it (E^q/2, rem, E^q/2): the
// list is then a palindrome, so the mirrored list the spectrum passes use for
// their inverse transform is the same list and shares one staged twiddle
// table.  Otherwise (and for the FWHT, whose stage order is fixed) the list is
// linear (E, E, ..., rem); the mirrored list is its reverse.
__host__ __device__ constexpr int st_count(int N, int E) {
  int s = 0, m = 1;
  while (m < N) {
    m *= (N / m >= E ? E : N / m);
    ++s;
  }
  return s;
}
__host__ __device__ constexpr int st_radix_lin(int N, int E, int s) {
  int m = 1, r = 1;
  for (int i = 0; i <= s; ++i) {
    r = (N / m >= E ? E : N / m);
    m *= r;
  }
  return r;
}
__host__ __device__ constexpr int st_ns_lin(int N, int E, int s) {
  int m = 1;
  for (int i = 0; i < s; ++i) m *= st_radix_lin(N, E, i);
  return m;
}
__host__ __device__ constexpr bool st_palindrome(int N, int E) {
  return st_count(N, E) % 2 == 1 || st_radix_lin(N, E, st_count(N, E) - 1) == E;
}
__host__ __device__ constexpr int st_radix_fwd(int N, int E, int s) {
  if (st_radix_lin(N, E, st_count(N, E) - 1) == E || st_count(N, E) % 2 == 0) return st_radix_lin(N, E, s);
  // odd stage count with a remainder: move it to the middle
  const int mid = st_count(N, E) / 2;
  return s == mid ? st_radix_lin(N, E, st_count(N, E) - 1) : E;
}
__host__ __device__ constexpr int st_radix(int N, int E, int s, bool mirror) {
  return mirror ? st_radix_fwd(N, E, st_count(N, E) - 1 - s) : st_radix_fwd(N, E, s);
}
__host__ __device__ constexpr int st_ns(int N, int E, int s, bool mirror) {
  int m = 1;
  for (int i = 0; i < s; ++i) m *= st_radix(N, E, i, mirror);
  return m;
}

__device__ __forceinline__ int sm_row(int row) { return row + (row >> 4); }
__host__ __device__ constexpr int sm_rows(int N) { return N + N / 16; }

// ----------------------------------------------------- constant twiddles ---
// d * W_32^t, W_32 = exp(-2*pi*i/32), t in [0, 16) known at compile time:
// W_32^t = cos(pi t/16) - i sin(pi t/16).
template <class C>
__device__ __forceinline__ C mul_w32(C d, const int t) {
  using R = typename RealOf<C>::T;
  constexpr double cs[9] = {1.0,
                            0.98078528040323044913,
                            0.92387953251128675613,
                            0.83146961230254523708,
                            0.70710678118654752440,
                            0.55557023301960222474,
                            0.38268343236508977173,
                            0.19509032201612826785,
                            0.0};
  if (t == 0) return d;
  if (t == 8) return mk(d.y, -d.x);
  // cos(pi t/16) = cs[t] (t <= 8) or -cs[16 - t]; sin(pi t/16) = cs[8 - t] or cs[t - 8]
  const R c = t <= 8 ? R(cs[t]) : R(-cs[16 - t]);
  const R s = t <= 8 ? R(cs[8 - t]) : R(cs[t - 8]);
  return mul_cs(d, c, s);
}

__host__ __device__ constexpr int bitrev_c(int v, int bits) {
  int r = 0;
  for (int i = 0; i < bits; ++i) r |= ((v >> i) & 1) << (bits - 1 - i);
  return r;
}
__host__ __device__ constexpr int log2_c(int n) { return n <= 1 ? 0 : 1 + log2_c(n / 2); }
__host__ __device__ constexpr int ctz_c(int v) { return (v & 1) ? 0 : 1 + ctz_c(v >> 1); }

// In-register forward DFT of R = 1..32 points, natural order in and out.
template <int R, class C>
__device__ __forceinline__ void dft_small(C* a) {
  if constexpr (R > 1) {
#pragma unroll
    for (int half = R / 2; half >= 1; half >>= 1) {
#pragma unroll
      for (int blk = 0; blk < R; blk += 2 * half) {
#pragma unroll
        for (int q = 0; q < half; ++q) {
          C x = a[blk + q], y = a[blk + q + half];
          a[blk + q] = x + y;
          a[blk + q + half] = mul_w32(x - y, q * (32 / (2 * half)));
        }
      }
    }
    C t[R];
#pragma unroll
    for (int i = 0; i < R; ++i) t[i] = a[bitrev_c(i, log2_c(R))];
#pragma unroll
    for (int i = 0; i < R; ++i) a[i] = t[i];
  }
}

// In-register Walsh-Hadamard of R points, stride-1-first (kernels.py:181-189).
template <int R, class T>
__device__ __forceinline__ void wht_small(T* a) {
#pragma unroll
  for (int h = 1; h < R; h <<= 1) {
#pragma unroll
    for (int blk = 0; blk < R; blk += 2 * h) {
#pragma unroll
      for (int q = 0; q < h; ++q) {
        T x = a[blk + q], y = a[blk + q + h];
        a[blk + q] = x + y;
        a[blk + q + h] = x - y;
      }
    }
  }
}

// a[r] *= w^r for r = 1..R-1 where wp[b] = w^(2^b) are table values: every
// power is a product of at most log2(R) correctly rounded factors.
template <int r, class C>
__device__ __forceinline__ C power_of(const C* wp) {
  constexpr int lo = ctz_c(r);
  constexpr int rest = r & (r - 1);
  C w = wp[lo];
  if constexpr (rest & 2) w = cmul(w, wp[1]);
  if constexpr (rest & 4) w = cmul(w, wp[2]);
  if constexpr (rest & 8) w = cmul(w, wp[3]);
  if constexpr (rest & 16) w = cmul(w, wp[4]);
  return w;
}
template <int R, int r = 1, class C>
__device__ __forceinline__ void apply_powers(C* a, const C* wp) {
  if constexpr (r < R) {
    a[r] = cmul(a[r], power_of<r>(wp));
    apply_powers<R, r + 1>(a, wp);
  }
}

// a * W^t from a twiddle table: quad layout (float4) in single precision
// (FMUL2 + FFMA2), plain double2 in double precision; TWS selects a shared-
// memory table (plain loads) instead of the global one (__ldg).
template <bool TWS>
__device__ __forceinline__ float2 tw_mul(float2 a, const float2* tw, int t) {
  const float4* q = reinterpret_cast<const float4*>(tw) + t;
  return cmul_q(a, TWS ? *q : __ldg(q));
}
template <bool TWS>
__device__ __forceinline__ double2 tw_mul(double2 a, const double2* tw, int t) {
  return cmul(a, TWS ? tw[t] : __ldg(&tw[t]));
}

// a * w for a plain float2 w on the packed FP32x2 pipe: FMUL2 + FFMA2 with
// (-w.y, w.x) formed in registers
__device__ __forceinline__ float2 cmul_f2(float2 a, float2 w) {
  const float2 p = __fmul2_rn(make_float2(a.x, a.x), w);
  return __ffma2_rn(make_float2(a.y, a.y), make_float2(-w.y, w.x), p);
}

// Staged stage twiddle of the TMA pass.  F2: a single-precision table of plain
// float2 entries (8 bytes: half the shared-memory traffic of the quads, one
// more instruction per multiply to form (-w.y, w.x)) — used by the spectrum
// passes, whose FFT + IFFT make shared memory their tightest pipe; the other
// passes keep the quads (C2 plain pass 188 -> 200 us with float2 entries).
template <bool F2>
__device__ __forceinline__ float2 st_tw_mul(float2 a, const float2* tw, int t) {
  if constexpr (F2) {
    return cmul_f2(a, tw[t]);
  } else {
    return tw_mul<true>(a, tw, t);
  }
}
template <bool F2>
__device__ __forceinline__ double2 st_tw_mul(double2 a, const double2* tw, int t) { return cmul(a, tw[t]); }

// Spectrum entry i (plan layout: float2 / double2).
__device__ __forceinline__ float2 ld_spec(const float2* mid, int64_t i) { return __ldg(mid + i); }

__device__ __forceinline__ double2 ld_spec(const double2* mid, int64_t i) { return __ldg(mid + i); }

// Exchange-buffer row map.  LAY == 0: padded rows (row + row/16, the buffer
// holds sm_rows(N) rows).  LAY = X > 0: dense rows permuted as
// row ^ ((row >> SH) & (X - 1)) — X = rows per 128 bytes, SH = log2 of the
// writing stage's radix — so the radix-R scatter (rows R apart) spreads over
// all bank groups without padding, which lets a dense TMA landing buffer
// double as the exchange buffer.
template <int LAY, int SH = 4>
__device__ __forceinline__ int ex_row(int row) {
  if constexpr (LAY == 0) return row + (row >> 4);
  else if constexpr (LAY == 1) return row;
  else return row ^ ((row >> SH) & (LAY - 1));
}

// Staged twiddle table (shared-memory tables of the TMA pass): stage s with
// stride NS > 1 and radix R reads W_N^(r*k*N/(NS*R)) at
// st_twoff(s) + k*(R-1) + r-1 — consecutive butterflies k sit (R-1) entries
// apart, an odd stride, so a warp's lookups are bank-conflict free.  The
// table holds N - R0 entries.
__host__ __device__ constexpr int st_twoff(int N, int E, int s, bool mirror) {
  int off = 0, ns = 1;
  for (int i = 0; i < s; ++i) {
    const int r = st_radix(N, E, i, mirror);
    if (ns > 1) off += ns * (r - 1);
    ns *= r;
  }
  return off;
}

// ------------------------------------------------- block FFT (Stockham) ----
// Thread (j, cs) of a tile holds, at stage s (radix R, stride NS), the inputs
// of butterflies bb = j + u*TPC (u < E/R): elements bb + r*N/R.  Outputs go to
// (bb/NS)*NS*R + bb%NS + r*NS.  `tw` is W_TWN^t (t < TWN).
// `hook` runs once the inputs of the LAST stage are in registers (after the
// last exchange read; multi-stage transforms only): from there on the
// exchange buffer is dead for this thread — the TMA pass refills it there.
struct NoHook {
  __device__ __forceinline__ void operator()() const {}
};
template <class C, int N, int E, int CT, bool MIR, int S, int LAY = 0, int TWN = 4096, bool TWS = false,
          bool TF2 = false, class Hook = NoHook>
__device__ __forceinline__ void fft_stages(C* a, C* sm, int j, int cs, const C* __restrict__ tw,
                                           const Hook& hook = Hook{}) {
  constexpr int NST = st_count(N, E);
  if constexpr (S < NST) {
    constexpr int R = st_radix(N, E, S, MIR);
    constexpr int NS = st_ns(N, E, S, MIR);
    constexpr int TPC = N / E;
    constexpr int SH = log2_c(R);
#pragma unroll
    for (int u = 0; u < E / R; ++u) {
      if constexpr (NS > 1) {
        const int k = (j + u * TPC) & (NS - 1);
        if constexpr (TWS) {
          // staged shared table (see st_twoff)
          const int t0 = st_twoff(N, E, S, MIR) + k * (R - 1) - 1;
#pragma unroll
          for (int r = 1; r < R; ++r) a[u * R + r] = st_tw_mul<TF2>(a[u * R + r], tw, t0 + r);
        } else {
          constexpr int step = TWN / (NS * R);
          const int ks = k * step;
#pragma unroll
          for (int r = 1; r < R; ++r) a[u * R + r] = tw_mul<false>(a[u * R + r], tw, r * ks);
        }
      }
      dft_small<R>(a + u * R);
    }
    if constexpr (S + 1 < NST) {
      constexpr int R2 = st_radix(N, E, S + 1, MIR);
      __syncthreads();  // previous readers of sm are done
#pragma unroll
      for (int u = 0; u < E / R; ++u) {
        const int bb = j + u * TPC;
        const int k = bb & (NS - 1);
        const int base = (bb - k) * R + k;
#pragma unroll
        for (int r = 0; r < R; ++r) sm[ex_row<LAY, SH>(base + r * NS) * CT + cs] = a[u * R + r];
      }
      __syncthreads();
#pragma unroll
      for (int u = 0; u < E / R2; ++u) {
        const int bb = j + u * TPC;
#pragma unroll
        for (int r = 0; r < R2; ++r) a[u * R2 + r] = sm[ex_row<LAY, SH>(bb + r * (N / R2)) * CT + cs];
      }
      if constexpr (S + 2 == NST) hook();
      fft_stages<C, N, E, CT, MIR, S + 1, LAY, TWN, TWS, TF2, Hook>(a, sm, j, cs, tw, hook);
    }
  }
}

// Generic in-tile FWHT: group g handles strides S_g..S_g*R/2 in registers.
template <class T, int N, int E, int CT, int S>
__device__ __forceinline__ void wht_stages(T* a, T* sm, int j, int cs) {
  constexpr int NST = st_count(N, E);
  if constexpr (S < NST) {
    constexpr int R = st_radix_lin(N, E, S);
#pragma unroll
    for (int u = 0; u < E / R; ++u) wht_small<R>(a + u * R);
    if constexpr (S + 1 < NST) {
      constexpr int NS = st_ns_lin(N, E, S);
      constexpr int R2 = st_radix_lin(N, E, S + 1);
      constexpr int NS2 = st_ns_lin(N, E, S + 1);
      constexpr int TPC = N / E;
      __syncthreads();
#pragma unroll
      for (int u = 0; u < E / R; ++u) {
        const int bb = j + u * TPC;
        const int base = (bb / NS) * (NS * R) + (bb % NS);
#pragma unroll
        for (int r = 0; r < R; ++r) sm[sm_row(base + r * NS) * CT + cs] = a[u * R + r];
      }
      __syncthreads();
#pragma unroll
      for (int u = 0; u < E / R2; ++u) {
        const int bb = j + u * TPC;
        const int base = (bb / NS2) * (NS2 * R2) + (bb % NS2);
#pragma unroll
        for (int r = 0; r < R2; ++r) a[u * R2 + r] = sm[sm_row(base + r * NS2) * CT + cs];
      }
      wht_stages<T, N, E, CT, S + 1>(a, sm, j, cs);
    }
  }
}

}  // namespace smat
