// dmma_probe.cu — FP64 tensor-core (mma.sync f64) throughput on this GPU,
// next to plain DFMA, to decide how the rank-32 LowRank kernels compute.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dmma884(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[8][2] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[k][0]), "+d"(c[k][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
  for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dmma1684(double* out, int iters) {
  double a0 = 1.0 + threadIdx.x * 1e-9, a1 = 1.0 - threadIdx.x * 1e-9, b = 0.5;
  double c[8][4] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(c[k][0]), "+d"(c[k][1]), "+d"(c[k][2]), "+d"(c[k][3])
                   : "d"(a0), "d"(a1), "d"(b));
  }
  double s = 0;
  for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1] + c[k][2] + c[k][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dfma(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1e-9;
  double c[16] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k) c[k] = fma(a, c[k], b);
  }
  double s = 0;
  for (int k = 0; k < 16; ++k) s += c[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 148 * 16 * 1024 * sizeof(double));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096;
  for (int blocks_per_sm : {2, 4, 8}) {
    const int grid = 148 * blocks_per_sm, thr = 256;
    float ms;
    dmma884<<<grid, thr>>>(out, 16);
    cudaEventRecord(e0);
    dmma884<<<grid, thr>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * grid * (thr / 32) * double(iters) * 8 * (8 * 8 * 4);
    printf("blocks/SM %d  dmma m8n8k4 : %.2f TFLOP/s\n", blocks_per_sm, fl / ms / 1e9);
    dmma1684<<<grid, thr>>>(out, 16);
    cudaEventRecord(e0);
    dmma1684<<<grid, thr>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * grid * (thr / 32) * double(iters) * 8 * (16 * 8 * 4);
    printf("blocks/SM %d  dmma m16n8k4: %.2f TFLOP/s\n", blocks_per_sm, fl / ms / 1e9);
    dfma<<<grid, thr>>>(out, 16);
    cudaEventRecord(e0);
    dfma<<<grid, thr>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * grid * thr * double(iters) * 16;
    printf("blocks/SM %d  dfma        : %.2f TFLOP/s\n", blocks_per_sm, fl / ms / 1e9);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
