// tile_fft_c128_large.cu — instantiations of the tiled FFT pass (double2, N in {128,256,512,1024,2048,4096}).
#include "tile_impl.cuh"

namespace smat {

void launch_fft_tile_c128_large(int N, const FftArgs& a, cudaStream_t s) {
  switch (N) {
    case 128: fft_tile_launch<double2, 128>(a, s); break;
    case 256: fft_tile_launch<double2, 256>(a, s); break;
    case 512: fft_tile_launch<double2, 512>(a, s); break;
    case 1024: fft_tile_launch<double2, 1024>(a, s); break;
    case 2048: fft_tile_launch<double2, 2048>(a, s); break;
    case 4096: fft_tile_launch<double2, 4096>(a, s); break;
    default: throw Error(SMAT_UNSUPPORTED, "tile length " + std::to_string(N) + " not in tile_fft_c128_large");
  }
}

}  // namespace smat
