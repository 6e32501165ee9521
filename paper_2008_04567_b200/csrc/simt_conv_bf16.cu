// KB2 instantiations for bf16 (see simt_conv.cuh).
#include "simt_conv.cuh"
WPK_SIMT_TABLE_IMPL(__nv_bfloat16, simt_get_bf16, 0)
