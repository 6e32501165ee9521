// bf16 instantiations of the tcgen05 convolution kernel (one translation unit per dtype).
#include "umma_conv_kernel.cuh"

namespace wpk {
cudaError_t umma_launch_bf16(int ak, int ek, cudaLaunchConfig_t &lc, const CUtensorMap &tmA, const CUtensorMap &tmB,
                            const CUtensorMap &tmY, const CUtensorMap &tmP, const UmmaArgs &a) {
    return umma_launch_dt<DT_BF16>(ak, ek, lc, tmA, tmB, tmY, tmP, a);
}
}  // namespace wpk
