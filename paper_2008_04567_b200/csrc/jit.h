// WPK_FAMILY_JIT: NVRTC-specialised direct convolution (jit.cpp).
#pragma once
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "wpk_internal.h"

namespace wpk {

// Every compile-time constant of the generated kernel for (shape, genes); also the cache key.
std::string jit_defines(const ConvDesc &d, const Config &c);
// The loaded kernel for (shape, genes) on `device`: compiled (NVRTC) or taken from the cache.
bool jit_kernel(const ConvDesc &d, const Config &c, int device, cudaKernel_t *out, std::string *err);
// Compile the not-yet-cached JIT configs of `cfgs` on `threads` host threads (<= 0: all cores).
void jit_precompile(const ConvDesc &d, const std::vector<Config> &cfgs, int threads);
// Compile only (no CUDA context needed): cubin size, or the NVRTC log in *err.
bool jit_compile_only(const ConvDesc &d, const Config &c, size_t *cubin_bytes, std::string *err);
void jit_set_cache_dir(const char *dir);
void jit_stats(long long *compiles, long long *mem_hits, long long *disk_hits, long long *failures, double *seconds);

}  // namespace wpk
