// lsu_probe.cu — the C5 four-step tile patterns of layout_probe.cu moved by the
// load/store units instead of the TMA engine: per-thread 16-byte cp.async
// (LDGSTS) loads into a shared ring, then per-thread 16-byte stores (LDS + STG)
// or one TMA store of the tile.  Thread / row mapping as in the FFT passes
// (thread (j, cs): rows j + r * TPC of column slot cs), 256 threads per CTA.
//   S  spectrum tile, row-blocked layout: 2048 rows x 32 B, rows 2 KB apart in
//      64-row blocks 128 MB apart
//   O  outer tile, row-blocked layout: 1024 rows x 64 B, 128 KB apart
//   U  outer tile, user layout: 1024 rows x 64 B, 4 MB apart
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_exp/lsu_probe tools/lsu_probe.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

// byte offset of (tile t, row, 16-byte chunk) — kind 0 S, 1 O, 2 U
__device__ __forceinline__ size_t addr(int kind, int t, int row, int chunk) {
  const size_t KB = 1024, MB = KB * KB;
  if (kind == 0) {
    const int cp = t % 64, k2 = t / 64;
    return size_t(cp) * 32 + size_t(row % 64) * 2 * KB + size_t(k2) * 128 * KB + size_t(row / 64) * 128 * MB +
           size_t(chunk) * 16;
  } else if (kind == 1) {
    const int cg = t % 32, n1 = t / 32;
    return size_t(cg) * 64 + size_t(n1 % 64) * 2 * KB + size_t(row) * 128 * KB + size_t(n1 / 64) * 128 * MB +
           size_t(chunk) * 16;
  } else {
    const int cg = t % 32, n1 = t / 32;
    return size_t(cg) * 64 + size_t(n1) * 2 * KB + size_t(row) * 4 * MB + size_t(chunk) * 16;
  }
}

// MODE 0: cp.async loads + LDS/STG stores; 1: cp.async loads + register
// round trip (LDG -> STG, no shared memory); 2: LDG prefetch one tile ahead into registers -> STG
template <int NB, int MODE>
__global__ void __launch_bounds__(256) lsu_copy(const unsigned char* __restrict__ in, unsigned char* __restrict__ out,
                                                int kind, int ntiles) {
  extern __shared__ __align__(128) unsigned char sm[];
  constexpr int TB = 65536;
  const int CT = kind == 0 ? 2 : 4;        // 16-byte chunks per row
  const int TPC = 256 / CT;                // rows per sweep
  const int tid = threadIdx.x, cs = tid % CT, j = tid / CT;
  const int gs = gridDim.x;
  if (MODE == 0) {
    auto issue = [&](int t, int s) {
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        const int row = j + r * TPC;
        const unsigned char* g = in + addr(kind, t, row, cs);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su(sm + s * TB + (row * CT + cs) * 16)), "l"(g)
                     : "memory");
      }
    };
    for (int s = 0; s < NB - 1; ++s) {
      if (int(blockIdx.x) + s * gs < ntiles) issue(blockIdx.x + s * gs, s);
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
    for (int t = blockIdx.x, it = 0; t < ntiles; t += gs, ++it) {
      const int s = it % NB;
      // refill the slot freed in the previous iteration
      if (t + (NB - 1) * gs < ntiles) issue(t + (NB - 1) * gs, (it + NB - 1) % NB);
      asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group %0;" ::"n"(NB - 1) : "memory");
      __syncthreads();
      // every thread stores rows it did NOT load (as after an FFT exchange)
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        const int row = ((j + 37) % TPC) + r * TPC;
        const int4 v = *reinterpret_cast<const int4*>(sm + s * TB + (row * CT + cs) * 16);
        *reinterpret_cast<int4*>(out + addr(kind, t, row, cs)) = v;
      }
      __syncthreads();
    }
  } else {
    int4 v[16];
    auto ld = [&](int t) {
#pragma unroll
      for (int r = 0; r < 16; ++r)
        v[r] = __ldcg(reinterpret_cast<const int4*>(in + addr(kind, t, j + r * TPC, cs)));
    };
    if (int(blockIdx.x) < ntiles) ld(blockIdx.x);
    for (int t = blockIdx.x; t < ntiles; t += gs) {
      int4 w[16];
#pragma unroll
      for (int r = 0; r < 16; ++r) w[r] = v[r];
      if (t + gs < ntiles) ld(t + gs);
#pragma unroll
      for (int r = 0; r < 16; ++r) *reinterpret_cast<int4*>(out + addr(kind, t, j + r * TPC, cs)) = w[r];
    }
  }
}

template <int NB, int MODE>
static void run(void* a, void* b, int kind, int per_sm) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int smem = MODE == 0 ? NB * 65536 : 0;
  cudaFuncSetAttribute(lsu_copy<NB, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int ntiles = 65536;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e9;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    lsu_copy<NB, MODE><<<sms * per_sm, 256, smem>>>((const unsigned char*)a, (unsigned char*)b, kind, ntiles);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const char* nm[3] = {"S", "O", "U"};
  printf("%s mode=%d NB=%d ctas/SM=%d: %.3f ms  %.2f TB/s  (%s)\n", nm[kind], MODE, NB, per_sm, best,
         2.0 * 4294967296.0 / (best * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  void *a = nullptr, *b = nullptr;
  cudaMalloc(&a, size_t(4) << 30);
  cudaMalloc(&b, size_t(4) << 30);
  cudaMemset(a, 1, size_t(4) << 30);
  for (int kind = 0; kind < 3; ++kind) {
    run<2, 0>(a, b, kind, 1);
    run<3, 0>(a, b, kind, 1);
    run<2, 0>(a, b, kind, 2) /* (two CTAs would not fit beside the real tables) */;
    run<1, 1>(a, b, kind, 1);
    run<1, 1>(a, b, kind, 2);
    run<1, 1>(a, b, kind, 4);
  }
  return 0;
}
