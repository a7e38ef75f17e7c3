// tma_probe.cu — copy bandwidth of TMA boxes vs box row width, to size the
// FFT tile passes' column tiles.  A (rows x 2 KB) array is copied tile by tile
// (W-byte x 256-row boxes, TMA load -> smem -> TMA store), persistent CTAs,
// NB-deep ring; compared with a plain 16-byte LDG/STG copy of the same bytes.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t su(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

template <int W, int NB>
__global__ void __launch_bounds__(128) tma_copy(const __grid_constant__ CUtensorMap in,
                                                const __grid_constant__ CUtensorMap out, int ntiles, int ncolt) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + NB * W * 256);
  const int gs = gridDim.x;
  if (threadIdx.x != 0) return;
  for (int s = 0; s < NB; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;");
  auto issue = [&](int t, int s) {
    const int c = (t % ncolt) * (W / 8), r = (t / ncolt) * 256;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar[s])), "r"(W * 256));
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            su(sm + s * W * 256)),
        "l"(&in), "r"(c), "r"(r), "r"(su(&bar[s]))
        : "memory");
  };
  for (int s = 0; s < NB; ++s)
    if (blockIdx.x + s * gs < ntiles) issue(blockIdx.x + s * gs, s);
  for (int t = blockIdx.x, it = 0; t < ntiles; t += gs, ++it) {
    const int s = it % NB;
    const uint32_t par = (it / NB) & 1;
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
            su(&bar[s])),
        "r"(par)
        : "memory");
    const int c = (t % ncolt) * (W / 8), r = (t / ncolt) * 256;
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(&out),
                 "r"(su(sm + s * W * 256)), "r"(c), "r"(r)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;");
    if (t + NB * gs < ntiles) {
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      issue(t + NB * gs, s);
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Strided variant: the array is M rows of 2 KB viewed as row = n1 + N1*i; a
// tile is W bytes x 256 rows i of one n1 (the access pattern of the strided
// four-step passes: row stride N1 * 2 KB).  Tiles are dealt column-tile first,
// then n1, then the i block.
template <int W, int NB>
__global__ void __launch_bounds__(128) tma_copy3(const __grid_constant__ CUtensorMap in,
                                                 const __grid_constant__ CUtensorMap out, int ntiles, int ncolt,
                                                 int n1s, int order, int blk) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + NB * W * 256);
  const int gs = gridDim.x;
  if (threadIdx.x != 0) return;
  for (int s = 0; s < NB; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;");
  auto coords = [&](int t, int& c, int& n1, int& ib) {
    if (order == 0) {  // column tile fastest, then n1, then the row block
      c = (t % ncolt) * (W / 8);
      n1 = (t / ncolt) % n1s;
      ib = (t / ncolt / n1s) * 256;
    } else {  // n1 fastest
      n1 = t % n1s;
      c = ((t / n1s) % ncolt) * (W / 8);
      ib = (t / n1s / ncolt) * 256;
    }
  };
  auto issue = [&](int t, int s) {
    int c, n1, ib;
    coords(t, c, n1, ib);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar[s])), "r"(W * 256));
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
        "%4}], [%5];" ::"r"(su(sm + s * W * 256)),
        "l"(&in), "r"(c), "r"(n1), "r"(ib), "r"(su(&bar[s]))
        : "memory");
  };
  for (int s = 0; s < NB; ++s)
    if (blockIdx.x + s * gs < ntiles) issue(blockIdx.x + s * gs, s);
  for (int t = blockIdx.x, it = 0; t < ntiles; t += gs, ++it) {
    const int s = it % NB;
    const uint32_t par = (it / NB) & 1;
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
            su(&bar[s])),
        "r"(par)
        : "memory");
    int c, n1, ib;
    coords(t, c, n1, ib);
    if (blk) {
      asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
                       &out),
                   "r"(su(sm + s * W * 256)), "r"(c), "r"(n1 % blk), "r"(ib), "r"(n1 / blk)
                   : "memory");
    } else {
      asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(&out),
                   "r"(su(sm + s * W * 256)), "r"(c), "r"(n1), "r"(ib)
                   : "memory");
    }
    asm volatile("cp.async.bulk.commit_group;");
    if (t + NB * gs < ntiles) {
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      issue(t + NB * gs, s);
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

static PFN_cuTensorMapEncodeTiled_v12000 enc();
static CUtensorMapL2promotion g_promo = CU_TENSOR_MAP_L2_PROMOTION_L2_256B;

template <int W, int NB>
static void run3(void* a, void* b, size_t rows, int n1s, int blocks_per_sm, int order = 0, int blk = 0) {
  CUtensorMap mi, mo;
  const size_t n2 = rows / n1s;
  cuuint64_t dims[3] = {256, cuuint64_t(n1s), n2};
  cuuint64_t str[2] = {2048, cuuint64_t(n1s) * 2048};
  cuuint32_t box[3] = {W / 8, 1, 256};
  cuuint32_t es[4] = {1, 1, 1, 1};
  auto f = enc();
  f(&mi, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, a, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
    CU_TENSOR_MAP_SWIZZLE_NONE, g_promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (blk) {
    // blocked output: logical (n1, i) at row ((n1/blk)*n2 + i)*blk + n1%blk
    cuuint64_t d4[4] = {256, cuuint64_t(blk), n2, cuuint64_t(n1s / blk)};
    cuuint64_t s4[3] = {2048, cuuint64_t(blk) * 2048, cuuint64_t(blk) * n2 * 2048};
    cuuint32_t b4[4] = {W / 8, 1, 256, 1};
    f(&mo, CU_TENSOR_MAP_DATA_TYPE_UINT64, 4, b, d4, s4, b4, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_NONE, g_promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    f(&mo, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, b, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_NONE, g_promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  const int ncolt = 2048 / W;
  const int ntiles = int(n2 / 256) * n1s * ncolt;
  const size_t smem = size_t(NB) * W * 256 + 64;
  cudaFuncSetAttribute(tma_copy3<W, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  const int grid = 148 * blocks_per_sm;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  tma_copy3<W, NB><<<grid, 128, smem>>>(mi, mo, ntiles, ncolt, n1s, order, blk);
  cudaEventRecord(e0);
  for (int k = 0; k < 3; ++k) tma_copy3<W, NB><<<grid, 128, smem>>>(mi, mo, ntiles, ncolt, n1s, order, blk);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("strided TMA box %4d B x 256 rows, row stride %8zu KB, order %d, out block %d, ring %d, %d CTA/SM: %7.1f GB/s  (%s)\n", W,
         size_t(n1s) * 2, order, blk, NB, blocks_per_sm, 2.0 * double(n2 / 256 * 256) * n1s * 2048 * 3 / (ms / 1e3) / 1e9,
         cudaGetErrorString(cudaGetLastError()));
}

__global__ void ldg_copy(const int4* in, int4* out, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    out[i] = in[i];
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
}

template <int W, int NB>
static void run(void* a, void* b, size_t rows, int blocks_per_sm) {
  CUtensorMap mi, mo;
  cuuint64_t dims[2] = {256, rows};  // 2 KB rows of uint64
  cuuint64_t str[1] = {2048};
  cuuint32_t box[2] = {W / 8, 256};
  cuuint32_t es[2] = {1, 1};
  auto f = enc();
  f(&mi, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, a, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  f(&mo, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, b, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int ncolt = 2048 / W;
  const int ntiles = int(rows / 256) * ncolt;
  const size_t smem = size_t(NB) * W * 256 + 64;
  cudaFuncSetAttribute(tma_copy<W, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  const int grid = 148 * blocks_per_sm;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  tma_copy<W, NB><<<grid, 128, smem>>>(mi, mo, ntiles, ncolt);
  cudaEventRecord(e0);
  for (int k = 0; k < 5; ++k) tma_copy<W, NB><<<grid, 128, smem>>>(mi, mo, ntiles, ncolt);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("TMA box %4d B x 256 rows, ring %d, %d CTA/SM (smem %zu KB): %7.1f GB/s  (%s)\n", W, NB, blocks_per_sm,
         smem / 1024, 2.0 * rows * 2048 * 5 / (ms / 1e3) / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const size_t rows = size_t(1) << 20;  // 2 GB
  void *a, *b;
  cudaMalloc(&a, rows * 2048);
  cudaMalloc(&b, rows * 2048);
  cudaMemset(a, 1, rows * 2048);
  run<32, 4>(a, b, rows, 4);
  run<64, 4>(a, b, rows, 2);
  run<64, 4>(a, b, rows, 4);
  run<64, 8>(a, b, rows, 2);
  run<128, 4>(a, b, rows, 2);
  run<128, 2>(a, b, rows, 4);
  run<256, 2>(a, b, rows, 2);
  run<256, 3>(a, b, rows, 1);
  run<512, 1>(a, b, rows, 1);
  // strided rows (four-step passes): 64-byte rows at 2 KB .. 4 MB stride
  for (int n1s : {1, 8, 256, 2048}) run3<64, 4>(a, b, rows, n1s, 2);
  for (int n1s : {1, 256, 2048}) run3<128, 4>(a, b, rows, n1s, 2);
  // L2 promotion at the 4 MB stride
  g_promo = CU_TENSOR_MAP_L2_PROMOTION_NONE;
  run3<64, 4>(a, b, rows, 2048, 2);
  g_promo = CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
  run3<64, 4>(a, b, rows, 2048, 2);
  g_promo = CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  // 4 MB-strided input, blocked (128 KB-strided) output
  run3<64, 4>(a, b, rows, 2048, 2, 0, 64);
  run3<64, 4>(a, b, rows, 256, 2, 0, 64);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const size_t n = rows * 2048 / 16;
  ldg_copy<<<148 * 8, 512>>>((const int4*)a, (int4*)b, n);
  cudaEventRecord(e0);
  for (int k = 0; k < 5; ++k) ldg_copy<<<148 * 8, 512>>>((const int4*)a, (int4*)b, n);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("LDG/STG int4 copy: %7.1f GB/s\n", 2.0 * rows * 2048 * 5 / (ms / 1e3) / 1e9);
  return 0;
}
