// dmma_rate.cu — FP64 tensor-core (mma.sync m8n8k4 f64) throughput per SM vs
// warps per SM and independent accumulators per warp, to size the rank-r
// LowRank passes (wlr.cu).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_exp/dmma_rate tools/dmma_rate.cu
#include <cuda_runtime.h>

#include <cstdio>

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

template <int NACC>
__global__ void kern(double* out, int iters, double a0, double b0) {
  double acc[NACC][2];
  for (int i = 0; i < NACC; ++i) acc[i][0] = acc[i][1] = 0.0;
  double a = a0 + threadIdx.x, b = b0 - threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) dmma(acc[i], a, b);
  }
  double s = 0;
  for (int i = 0; i < NACC; ++i) s += acc[i][0] + acc[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int NACC>
static void run(int warps) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, size_t(sms) * warps * 32 * 8);
  const int iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  kern<NACC><<<sms, warps * 32>>>(out, 16, 1.0, 2.0);
  cudaEventRecord(e0);
  kern<NACC><<<sms, warps * 32>>>(out, iters, 1.0, 2.0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = double(sms) * warps * iters * NACC * 512.0;
  printf("warps/SM %2d  acc/warp %2d : %.2f TFLOP/s\n", warps, NACC, flops / (ms * 1e-3) / 1e12);
  cudaFree(out);
}

int main() {
  for (int w : {4, 8, 12, 16, 32}) {
    run<4>(w);
    run<8>(w);
    run<12>(w);
  }
  return 0;
}
