// Micro-probe: FP64/FP32 FMA throughput and HBM copy bandwidth on this B200.
#include <cstdio>
#include <cuda_runtime.h>
template <typename T>
__global__ void fma_loop(T* out, int iters, T a, T b) {
  T x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      x0 = x0 * a + b; x1 = x1 * a + b; x2 = x2 * a + b; x3 = x3 * a + b;
      x4 = x4 * a + b; x5 = x5 * a + b; x6 = x6 * a + b; x7 = x7 * a + b;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void copyk(const float4* __restrict__ a, float4* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t s = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += s) b[i] = a[i];
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("name %s sms %d smem/blk optin %zu l2 %d clock %d memclk %d busw %d\n", p.name, p.multiProcessorCount,
         p.sharedMemPerBlockOptin, p.l2CacheSize, p.clockRate, p.memoryClockRate, p.memoryBusWidth);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  void* out; cudaMalloc(&out, 148 * 8 * 1024 * 8);
  int iters = 4096; float ms;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    fma_loop<double><<<148 * 8, 256>>>((double*)out, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
  }
  double fl = 2.0 * 148 * 8 * 256 * (double)iters * 16 * 8;
  printf("fp64 fma: %.2f TFLOP/s\n", fl / ms / 1e9);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    fma_loop<float><<<148 * 8, 256>>>((float*)out, iters, 1.0000001f, 1e-9f);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
  }
  printf("fp32 fma: %.2f TFLOP/s\n", fl / ms / 1e9);
  size_t n = (size_t)1 << 30;  // 4 GiB floats... use 1 Gi bytes*4
  float4 *a, *b; cudaMalloc(&a, n); cudaMalloc(&b, n);
  cudaMemset(a, 0, n);
  for (int blocks : {148 * 4, 148 * 8, 148 * 16}) {
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      copyk<<<blocks, 512>>>(a, b, n / 16);
      cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    printf("copy blocks %d: %.1f GB/s\n", blocks, 2.0 * n / best / 1e6);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
