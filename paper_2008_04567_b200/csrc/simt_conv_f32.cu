// KB2 instantiations for f32 (see simt_conv.cuh).
#include "simt_conv.cuh"
WPK_SIMT_TABLE_IMPL(float, simt_get_f32, 1)
