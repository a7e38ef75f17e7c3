// tile_tma_c64.cu — instantiations of the persistent TMA-fed FFT tile pass (float2).
#include "tile_tma.cuh"

namespace smat {

bool launch_fft_tma_c64(int N, const FftArgs& a, cudaStream_t s) {
  switch (N) {
    case 256: return fft_tma_launch<float2, 256>(a, s);
    case 512: return fft_tma_launch<float2, 512>(a, s);
    case 1024: return fft_tma_launch<float2, 1024>(a, s);
    case 2048: return fft_tma_launch<float2, 2048>(a, s);
    default: return false;
  }
}

}  // namespace smat
