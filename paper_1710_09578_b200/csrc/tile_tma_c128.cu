// tile_tma_c128.cu — instantiations of the persistent TMA-fed FFT tile pass (double2).
#include "tile_tma.cuh"

namespace smat {

bool launch_fft_tma_c128(int N, const FftArgs& a, cudaStream_t s) {
  switch (N) {
    case 256: return fft_tma_launch<double2, 256>(a, s);
    case 512: return fft_tma_launch<double2, 512>(a, s);
    case 1024: return fft_tma_launch<double2, 1024>(a, s);
    default: return false;
  }
}

}  // namespace smat
