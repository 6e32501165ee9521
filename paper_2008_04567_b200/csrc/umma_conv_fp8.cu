// fp8 (e4m3 x / w, bf16 b / z / y) instantiations of the tcgen05 convolution kernel, kind::f8f6f4.
#include "umma_conv_kernel.cuh"

namespace wpk {
cudaError_t umma_launch_fp8(int ak, int ek, cudaLaunchConfig_t &lc, const CUtensorMap &tmA, const CUtensorMap &tmB,
                            const CUtensorMap &tmY, const CUtensorMap &tmP, const UmmaArgs &a) {
    return umma_launch_dt<DT_FP8>(ak, ek, lc, tmA, tmB, tmY, tmP, a);
}
}  // namespace wpk
