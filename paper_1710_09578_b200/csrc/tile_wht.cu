// tile_wht.cu — instantiations of the tiled FWHT pass for every element type.
#include "tile_impl.cuh"

namespace smat {

void launch_wht_tile(int dt, int N, const WhtArgs& a, cudaStream_t s) {
  switch (dt) {
    case SMAT_F32: SMAT_N_SWITCH(wht_tile_launch, float, N, a, s) break;
    case SMAT_F64: SMAT_N_SWITCH(wht_tile_launch, double, N, a, s) break;
    case SMAT_C64: SMAT_N_SWITCH(wht_tile_launch, float2, N, a, s) break;
    case SMAT_C128: SMAT_N_SWITCH(wht_tile_launch, double2, N, a, s) break;
    case SMAT_I32: SMAT_N_SWITCH(wht_tile_launch, int32_t, N, a, s) break;
    case SMAT_I64: SMAT_N_SWITCH(wht_tile_launch, long long, N, a, s) break;
    default: throw Error(SMAT_BAD_DTYPE, "fwht: unsupported dtype");
  }
}

}  // namespace smat
