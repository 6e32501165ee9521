// KB2 instantiations for f16 (see simt_conv.cuh).
#include "simt_conv.cuh"
WPK_SIMT_TABLE_IMPL(__half, simt_get_f16, 0)
