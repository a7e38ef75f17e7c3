// layout_probe.cu — TMA copy bandwidth of the C5 four-step intermediate's
// tile patterns (complex128, M = 2^21 rows x 128 columns, 64 KB tiles):
//   S_cur  spectrum tile of the row-blocked layout B[n1/64][k2][n1%64][128]:
//          32 blocks x 64 rows x 32 B (rows 2 KB apart)
//   S_new  spectrum tile of B[n1/64][cg][k2][n1%64][2]: 32 runs of 2 KB
//   O_cur  outer tile of the row-blocked layout: 1024 rows x 64 B, 128 KB apart
//   O_new  outer tile of B[n1/64][cg][k2][n1%64][2]: 1024 rows x 64 B, 2 KB apart
// Each tile is TMA-loaded into a ring slot and TMA-stored with the same map
// into a second array.  Prints TB/s (read + write) per pattern / ring / CTAs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_exp/layout_probe tools/layout_probe.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t su(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

struct Pat {
  int kind;
};

__device__ __forceinline__ void coords(int kind, int t, int* c) {
  for (int i = 0; i < 5; ++i) c[i] = 0;
  if (kind == 0) {  // S_cur: {w, n1%64, k2, n1/64}
    c[0] = (t % 64) * 4;
    c[2] = t / 64;
  } else if (kind == 1) {  // S_new: {w, k2, cg, blk}
    c[1] = t / 64;
    c[2] = t % 64;
  } else if (kind == 2) {  // O_cur: {w, n1%64, k2lo, k2hi, n1/64}
    c[0] = (t % 32) * 8;
    const int n1 = t / 32;
    c[1] = n1 % 64;
    c[4] = n1 / 64;
  } else if (kind == 3) {  // O_new: {w, k2lo, k2hi, cg, blk}
    c[0] = (t % 32) * 8;
    c[3] = (t / 32) % 64;
    c[4] = t / 2048;
  } else if (kind == 4) {  // S_half: {w(4 cols), n1%64, k2, cg4, blk}, half tiles
    c[0] = (t % 2) * 4;
    c[3] = (t / 2) % 32;
    c[2] = t / 64;
  } else if (kind == 5) {  // O_4: {w(n1%64 x 4 cols), k2lo, k2hi, cg4, blk}
    c[0] = (t % 64) * 8;
    c[3] = (t / 64) % 32;
    c[4] = t / 2048;
  } else if (kind == 6) {  // U32: {w, n1, k2lo, k2hi}, tile = n1 pair x col pair
    c[0] = (t % 64) * 4;
    c[1] = (t / 64) * 2;
  } else {  // U64: tile = n1 x 4 cols
    c[0] = (t % 32) * 8;
    c[1] = t / 32;
  }
}

template <int NB>
__global__ void __launch_bounds__(32) copy_kernel(const __grid_constant__ CUtensorMap in,
                                                  const __grid_constant__ CUtensorMap out, int kind, int rank,
                                                  int ntiles) {
  extern __shared__ __align__(128) unsigned char sm[];
  constexpr int TB = 65536;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + NB * TB);
  const int gs = gridDim.x;
  if (threadIdx.x != 0) return;
  for (int s = 0; s < NB; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;");
  auto issue = [&](int t, int s) {
    int c[5];
    coords(kind, t, c);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar[s])), "r"(TB));
    if (rank == 4)
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
          "%5}], [%6];" ::"r"(su(sm + s * TB)),
          "l"(&in), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(su(&bar[s]))
          : "memory");
    else
      asm volatile(
          "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
          "%5, %6}], [%7];" ::"r"(su(sm + s * TB)),
          "l"(&in), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(su(&bar[s]))
          : "memory");
  };
  for (int s = 0; s < NB; ++s)
    if (int(blockIdx.x) + s * gs < ntiles) issue(blockIdx.x + s * gs, s);
  for (int t = blockIdx.x, it = 0; t < ntiles; t += gs, ++it) {
    const int s = it % NB;
    const uint32_t par = (it / NB) & 1;
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
            su(&bar[s])),
        "r"(par)
        : "memory");
    int c[5];
    coords(kind, t, c);
    if (rank == 4)
      asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
                       &out),
                   "r"(su(sm + s * TB)), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3])
                   : "memory");
    else
      asm volatile(
          "cp.async.bulk.tensor.5d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4, %5, %6}], [%1];" ::"l"(&out),
          "r"(su(sm + s * TB)), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4])
          : "memory");
    asm volatile("cp.async.bulk.commit_group;");
    if (t + NB * gs < ntiles) {
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      issue(t + NB * gs, s);
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
}

static bool make(CUtensorMap* m, void* p, int kind, int* rank) {
  const cuuint64_t KB = 1024, MB = KB * KB;
  cuuint64_t d[5], s[4];
  cuuint32_t b[5], e[5] = {1, 1, 1, 1, 1};
  if (kind == 0) {
    *rank = 4;
    cuuint64_t dd[5] = {256, 64, 1024, 32, 1}, ss[4] = {2 * KB, 128 * KB, 128 * MB, 0};
    cuuint32_t bb[5] = {4, 64, 1, 32, 1};
    for (int i = 0; i < 5; ++i) d[i] = dd[i], b[i] = bb[i];
    for (int i = 0; i < 4; ++i) s[i] = ss[i];
  } else if (kind == 1) {
    *rank = 4;
    cuuint64_t dd[5] = {256, 1024, 64, 32, 1}, ss[4] = {2 * KB, 2 * MB, 128 * MB, 0};
    cuuint32_t bb[5] = {256, 1, 1, 32, 1};
    for (int i = 0; i < 5; ++i) d[i] = dd[i], b[i] = bb[i];
    for (int i = 0; i < 4; ++i) s[i] = ss[i];
  } else if (kind == 2) {
    *rank = 5;
    cuuint64_t dd[5] = {256, 64, 256, 4, 32}, ss[4] = {2 * KB, 32 * MB, 128 * KB * 256 / 256 * 1, 0};
    // k2 = k2lo + 256 k2hi: k2 stride 128 KB
    ss[1] = 128 * KB;
    ss[2] = 256 * 128 * KB;
    ss[3] = 1024 * 128 * KB;
    ss[0] = 2 * KB;
    cuuint32_t bb[5] = {8, 1, 256, 4, 1};
    for (int i = 0; i < 5; ++i) d[i] = dd[i], b[i] = bb[i];
    for (int i = 0; i < 4; ++i) s[i] = ss[i];
  } else if (kind == 3) {
    *rank = 5;
    cuuint64_t dd[5] = {256, 256, 4, 64, 32}, ss[4] = {2 * KB, 512 * KB, 2 * MB, 128 * MB};
    cuuint32_t bb[5] = {8, 256, 4, 1, 1};
    for (int i = 0; i < 5; ++i) d[i] = dd[i], b[i] = bb[i];
    for (int i = 0; i < 4; ++i) s[i] = ss[i];
  } else if (kind == 4) {
    *rank = 5;
    cuuint64_t dd[5] = {8, 64, 1024, 32, 32}, ss[4] = {64, 4 * KB, 4 * MB, 128 * MB};
    cuuint32_t bb[5] = {4, 64, 1, 1, 32};
    for (int i = 0; i < 5; ++i) d[i] = dd[i], b[i] = bb[i];
    for (int i = 0; i < 4; ++i) s[i] = ss[i];
  } else if (kind == 5) {
    *rank = 5;
    cuuint64_t dd[5] = {512, 256, 4, 32, 32}, ss[4] = {4 * KB, 1 * MB, 4 * MB, 128 * MB};
    cuuint32_t bb[5] = {8, 256, 4, 1, 1};
    for (int i = 0; i < 5; ++i) d[i] = dd[i], b[i] = bb[i];
    for (int i = 0; i < 4; ++i) s[i] = ss[i];
  } else {
    *rank = 4;
    cuuint64_t dd[5] = {256, 2048, 256, 4, 1}, ss[4] = {2 * KB, 4 * MB, 1024 * MB, 0};
    cuuint32_t bb[5] = {cuuint32_t(kind == 6 ? 4 : 8), cuuint32_t(kind == 6 ? 2 : 1), 256, 4, 1};
    for (int i = 0; i < 5; ++i) d[i] = dd[i], b[i] = bb[i];
    for (int i = 0; i < 4; ++i) s[i] = ss[i];
  }
  CUresult r = enc()(m, CU_TENSOR_MAP_DATA_TYPE_UINT64, *rank, p, d, s, b, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) printf("encode failed kind %d: %d\n", kind, int(r));
  return r == CUDA_SUCCESS;
}

template <int NB>
static void run(void* a, void* bptr, int kind, int per_sm) {
  CUtensorMap mi, mo;
  int rank = 0;
  if (!make(&mi, a, kind, &rank) || !make(&mo, bptr, kind, &rank)) return;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int smem = NB * 65536 + 64;
  cudaFuncSetAttribute(copy_kernel<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int ntiles = 65536;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e9;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    copy_kernel<NB><<<sms * per_sm, 32, smem>>>(mi, mo, kind, rank, ntiles);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const char* nm[8] = {"S_cur", "S_new", "O_cur", "O_new", "S_half", "O_4", "U32", "U64"};
  printf("%s NB=%d ctas/SM=%d: %.3f ms  %.2f TB/s  (%s)\n", nm[kind], NB, per_sm, best,
         2.0 * 4294967296.0 / (best * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  void *a = nullptr, *b = nullptr;
  cudaMalloc(&a, size_t(4) << 30);
  cudaMalloc(&b, size_t(4) << 30);
  cudaMemset(a, 1, size_t(4) << 30);
  for (int kind = 0; kind < 8; ++kind) {
    run<1>(a, b, kind, 2);
    run<2>(a, b, kind, 1);
    run<3>(a, b, kind, 1);
  }
  return 0;
}
