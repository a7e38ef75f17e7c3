// tile_fft_c128_small.cu — instantiations of the tiled FFT pass (double2, N in {1,2,4,8,16,32,64}).
#include "tile_impl.cuh"

namespace smat {

void launch_fft_tile_c128_small(int N, const FftArgs& a, cudaStream_t s) {
  switch (N) {
    case 1: fft_tile_launch<double2, 1>(a, s); break;
    case 2: fft_tile_launch<double2, 2>(a, s); break;
    case 4: fft_tile_launch<double2, 4>(a, s); break;
    case 8: fft_tile_launch<double2, 8>(a, s); break;
    case 16: fft_tile_launch<double2, 16>(a, s); break;
    case 32: fft_tile_launch<double2, 32>(a, s); break;
    case 64: fft_tile_launch<double2, 64>(a, s); break;
    default: throw Error(SMAT_UNSUPPORTED, "tile length " + std::to_string(N) + " not in tile_fft_c128_small");
  }
}

}  // namespace smat
