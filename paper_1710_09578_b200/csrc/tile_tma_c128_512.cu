// tile_tma_c128_512.cu — 512-point instantiations of the persistent TMA-fed FFT
// tile pass (double2); one file per length so they compile in parallel.
#include "tile_tma.cuh"

namespace smat {

bool launch_fft_tma_c128_512(const FftArgs& a, cudaStream_t s) { return fft_tma_launch<double2, 512>(a, s); }

}  // namespace smat
