// probe.cu — arithmetic peak probes (smat_probe_peak): the FP64 / FP32
// denominators of bench.py's compute rooflines, measured on the box instead
// of taken from a data sheet (MEASURED_PEAKS.json covers only HBM and bf16).
//
//   kind 0  DFMA           FP64 vector FMA pipe (C5's FFT / FWHT arithmetic)
//   kind 1  DMMA m8n8k4    FP64 tensor core (mma.sync f64)
//   kind 2  DFMA + DMMA    half the warps on each: shows whether the two pipes
//                          overlap (sum > either alone) or share hardware
//   kind 3  FFMA2          packed FP32x2 FMA (C3's single-precision FFT)
//
// Each kernel runs independent FMA chains in registers (no memory traffic)
// on 4 CTAs x 256 threads per SM; the result is flops / CUDA-event time of
// the best of three launches.
#include <cuda_runtime.h>

#include <algorithm>

#include "common.cuh"

namespace smat {
namespace {

constexpr int kChains = 16;

__device__ __forceinline__ void dfma_block(double (&c)[kChains], double a, double b) {
#pragma unroll
  for (int k = 0; k < kChains; ++k) c[k] = fma(a, c[k], b);
}

__device__ __forceinline__ void dmma_block(double (&c)[kChains], double a, double b) {
#pragma unroll
  for (int k = 0; k < kChains; k += 2)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c[k]), "+d"(c[k + 1])
                 : "d"(a), "d"(b));
}

// mode 0: DFMA, 1: DMMA, 2: even warps DFMA / odd warps DMMA
__global__ void __launch_bounds__(256) fp64_probe_kernel(double* out, int iters, int mode) {
  const double a = 1.0 + threadIdx.x * 1e-12, b = 1e-12;
  double c[kChains];
#pragma unroll
  for (int k = 0; k < kChains; ++k) c[k] = double(k);
  const bool mma = mode == 1 || (mode == 2 && (threadIdx.x / 32) % 2 == 1);
  if (mma) {
    for (int it = 0; it < iters; ++it) dmma_block(c, a, b);
  } else {
    // (DFMA: 16 FMAs per thread per block; DMMA: 8 x 256 FMAs per warp per
    // block = 64 per thread; four DFMA blocks per DMMA block keep the two
    // halves' work equal)
    for (int it = 0; it < 4 * iters; ++it) dfma_block(c, a, b);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < kChains; ++k) s += c[k];
  if (s == 12345.678) out[0] = s;  // keep the chains live
}

__global__ void __launch_bounds__(256) ffma2_probe_kernel(float* out, int iters) {
  const float2 a = make_float2(1.0f + threadIdx.x * 1e-7f, 1.0f - threadIdx.x * 1e-7f);
  const float2 b = make_float2(1e-7f, 2e-7f);
  float2 c[kChains];
#pragma unroll
  for (int k = 0; k < kChains; ++k) c[k] = make_float2(float(k), float(-k));
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < kChains; ++k) c[k] = __ffma2_rn(a, c[k], b);
  }
  float s = 0;
#pragma unroll
  for (int k = 0; k < kChains; ++k) s += c[k].x + c[k].y;
  if (s == 12345.678f) out[0] = s;
}

}  // namespace

double probe_peak_tflops(int kind, int device) {
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != device) SMAT_CUDA(cudaSetDevice(device));
  void* out = nullptr;
  SMAT_CUDA(cudaMalloc(&out, 64));
  cudaEvent_t e0, e1;
  SMAT_CUDA(cudaEventCreate(&e0));
  SMAT_CUDA(cudaEventCreate(&e1));
  const int grid = num_sms(device) * 4, threads = 256;
  const int iters = 2048;
  double flops = 0;
  if (kind <= 2) {
    // per thread per iteration: DFMA 4 * 16 FMAs; DMMA 8 mma x 256 FMAs / 32 lanes = 64
    flops = 2.0 * double(grid) * threads * iters * 64.0;
  } else {
    flops = 2.0 * double(grid) * threads * iters * kChains * 2.0;
  }
  float best = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    SMAT_CUDA(cudaEventRecord(e0));
    if (kind <= 2) fp64_probe_kernel<<<grid, threads>>>((double*)out, iters, kind);
    else ffma2_probe_kernel<<<grid, threads>>>((float*)out, iters * 4);
    SMAT_CUDA(cudaEventRecord(e1));
    SMAT_CUDA(cudaEventSynchronize(e1));
    SMAT_CUDA(cudaGetLastError());
    float ms = 0;
    SMAT_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    if (rep > 0) best = std::min(best, ms);  // (first launch: warm-up)
  }
  if (kind == 3) flops *= 4;  // (4x the iterations)
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  if (prev != device) cudaSetDevice(prev);
  return flops / (double(best) * 1e-3) / 1e12;
}

}  // namespace smat
