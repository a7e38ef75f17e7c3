// tile_tma_c64_64.cu — 64-point instantiations of the persistent TMA-fed FFT
// tile pass (float2); one file per length so they compile in parallel.
#include "tile_tma.cuh"

namespace smat {

bool launch_fft_tma_c64_64(const FftArgs& a, cudaStream_t s) { return fft_tma_launch<float2, 64>(a, s); }

}  // namespace smat
