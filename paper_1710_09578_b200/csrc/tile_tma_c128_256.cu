// tile_tma_c128_256.cu — 256-point instantiations of the persistent TMA-fed FFT
// tile pass (double2); one file per length so they compile in parallel.
#include "tile_tma.cuh"

namespace smat {

bool launch_fft_tma_c128_256(const FftArgs& a, cudaStream_t s) { return fft_tma_launch<double2, 256>(a, s); }

}  // namespace smat
