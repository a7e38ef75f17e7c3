// tile_tma_c128_2048.cu — 2048-point instantiations of the persistent TMA-fed FFT
// tile pass (double2); one file per length so they compile in parallel.
#include "tile_tma.cuh"

namespace smat {

bool launch_fft_tma_c128_2048(const FftArgs& a, cudaStream_t s) { return fft_tma_launch<double2, 2048>(a, s); }

}  // namespace smat
