// tma.cuh — Tensor Memory Accelerator + mbarrier helpers (inline PTX, sm_100a).
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <mutex>

#include "common.cuh"

namespace smat {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// 5-D tiled TMA load global -> shared, completion counted on `bar` (bytes).
__device__ __forceinline__ void tma_load_5d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2,
                                            int c3, int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
      : "memory");
}

// 1-D bulk copy global -> shared (16-byte aligned, size a multiple of 16),
// completion counted on `bar` (bytes).
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// 5-D tiled TMA store shared -> global (bulk async-group completion).
__device__ __forceinline__ void tma_store_5d(const CUtensorMap* map, const void* src, int c0, int c1, int c2, int c3,
                                             int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.global.shared::cta.tile.bulk_group"
      " [%0, {%2, %3, %4, %5, %6}], [%1];" ::"l"(reinterpret_cast<uint64_t>(map)),
      "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
      : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// wait until all committed bulk stores have finished READING shared memory
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
// wait until all committed bulk stores have completed
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// ---------------------------------------------------------------- host -----
inline PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// Tensor map of a block view  element (o1, o2, i, c) at p + o1*s1 + o2*s2 + i*si + c
// (element size esz, a multiple of 8 bytes), i < N split as (i % 256, i / 256),
// box = CT columns x all N rows of one (o1, o2).
// Masked views (zero padding / truncation of the rows): rows = R < N makes the
// map cover only rows i < R (R a multiple of rlo, i split as (i % rlo, i / rlo));
// with box_rows = R the box moves only those rows (the kernel treats the rest
// of the tile as zero / does not store it), otherwise loads zero-fill the rows
// beyond and stores drop them.
// Two-level rows (si_hi > 0): row i at (i % rlo)*si + (i / rlo)*si_hi.
inline bool make_view_map(CUtensorMap* map, const void* p, size_t esz, int64_t n1, int64_t s1, int64_t n2,
                          int64_t s2, int64_t N, int64_t si, int64_t inner, int CT, int64_t rlo = 0,
                          int64_t rows = 0, bool box_rows = false, int64_t si_hi = 0) {
  auto fn = encode_fn();
  if (!fn) return false;
  const int64_t w = int64_t(esz / 8);  // 8-byte words per element
  if (rlo == 0) rlo = N < 256 ? N : 256;
  if (rows == 0) rows = N;
  if (rlo > 256 || N / rlo > 256 || rows % rlo != 0 || rows <= 0) return false;
  const int64_t rhi = rows / rlo;
  cuuint64_t dims[5] = {cuuint64_t(inner * w), cuuint64_t(rlo), cuuint64_t(rhi), cuuint64_t(n2), cuuint64_t(n1)};
  cuuint64_t strides[4] = {cuuint64_t(si * int64_t(esz)),
                           cuuint64_t((si_hi ? si_hi : rlo * si) * int64_t(esz)),
                           cuuint64_t(s2 * int64_t(esz)), cuuint64_t(s1 * int64_t(esz))};
  for (int k = 0; k < 4; ++k)
    if (strides[k] % 16 || strides[k] >= (cuuint64_t(1) << 40)) {
      if (!(k >= 1 && dims[k + 1] == 1)) return false;
      strides[k] = 16;  // unused dimension of extent 1
    }
  if ((reinterpret_cast<uintptr_t>(p) & 15) != 0) return false;
  cuuint32_t box[5] = {cuuint32_t(CT * w), cuuint32_t(rlo), cuuint32_t(box_rows ? rhi : N / rlo), 1, 1};
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT64, 5, const_cast<void*>(p), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace smat
