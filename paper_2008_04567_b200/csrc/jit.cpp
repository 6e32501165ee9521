// WPK_FAMILY_JIT: the paper's code-generation step ("compile the generated codes
// just-in-time ... then execute them to get the runtime"; PAPER.md:179 multi-threaded compilation
// and a cache keep the search fast). For one candidate, the direct-convolution template of the
// SIMT family (the paper's schedule genes T_x, T_y, T_z, Tile_x, Tile_y, Tile_z, Tile_rz,
// PAPER.md:89-93) is emitted as CUDA source with every shape parameter, stride, layout and gene a
// compile-time constant -- the filter loops unroll, the address arithmetic folds -- and compiled
// for sm_100a with NVRTC into a cubin, loaded with cudaLibraryLoadData.
//
// Cache: process-wide (key = the full generated constant set), optionally mirrored on disk
// (wpk_jit_set_cache_dir / WPK_JIT_CACHE_DIR; one file per key holding the key and the cubin). The
// tuner compiles the new candidates of a generation on a pool of host threads before measuring
// them (jit_precompile), and reports compile time separately (wpk_jit_stats).
//
// Arithmetic: identical to the SIMT family (fp32 FMA, c ascending then r then s, bias + optional
// residual, ReLU, one RN conversion), so the two families agree bit for bit.
#include <cuda_runtime.h>
#include <nvrtc.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "jit.h"

namespace wpk {

// ---- the template (no headers: conversions through PTX cvt) -----------------------------------
static const char *kJitSource = R"JIT(
typedef unsigned short u16;
typedef unsigned long long u64;
#if WPK_E == 4
typedef float T;
__device__ __forceinline__ float ld_f(const T *p) { return *p; }
__device__ __forceinline__ void st_f(T *p, float v) { *p = v; }
#else
typedef u16 T;
__device__ __forceinline__ float ld_f(const T *p) {
    const u16 h = *p;
#if WPK_BF16
    return __int_as_float(((int)h) << 16);
#else
    float f;
    asm("cvt.f32.f16 %0, %1;" : "=f"(f) : "h"(h));
    return f;
#endif
}
__device__ __forceinline__ void st_f(T *p, float v) {
    u16 h;
#if WPK_BF16
    asm("cvt.rn.bf16.f32 %0, %1;" : "=h"(h) : "f"(v));
#else
    asm("cvt.rn.f16.f32 %0, %1;" : "=h"(h) : "f"(v));
#endif
    *p = h;
}
#endif

extern "C" __global__ void __launch_bounds__(BX * BY * BZ) wpk_jit_conv(const T *__restrict__ x, const T *__restrict__ w,
                                                                        const T *__restrict__ b, T *__restrict__ y,
                                                                        const T *__restrict__ z) {
    const int q0 = blockIdx.x * (BX * TILE_X) + threadIdx.x;
    const int p0 = blockIdx.y * (BY * TILE_Y) + threadIdx.y;
    const int n = blockIdx.z / KBLOCKS;
    const int k0 = (blockIdx.z % KBLOCKS) * (BZ * TILE_Z) + threadIdx.z;
    float acc[TILE_Z][TILE_Y][TILE_X];
#pragma unroll
    for (int j = 0; j < TILE_Z; ++j)
#pragma unroll
        for (int i = 0; i < TILE_Y; ++i)
#pragma unroll
            for (int l = 0; l < TILE_X; ++l) acc[j][i][l] = 0.f;
    bool kval[TILE_Z];
    int cbase[TILE_Z];
#pragma unroll
    for (int j = 0; j < TILE_Z; ++j) {
        const int k = k0 + j * BZ;
        kval[j] = k < KK;
        cbase[j] = kval[j] ? (k / KPG) * CPG : 0;
    }
    const T *xn = x + (long long)n * XS_N;
#pragma unroll 1
    for (int c = 0; c < CPG; c += TRZ) {
#pragma unroll
        for (int cc = 0; cc < TRZ; ++cc) {
            const int ci = c + cc;
            if (CPG % TRZ == 0 || ci < CPG) {
#pragma unroll
                for (int r = 0; r < RR; ++r) {
#pragma unroll
                    for (int s = 0; s < SS; ++s) {
                        float wv[TILE_Z];
#pragma unroll
                        for (int j = 0; j < TILE_Z; ++j) {
                            const int k = k0 + j * BZ;
                            wv[j] = kval[j] ? ld_f(w + (long long)k * WS_K + (long long)ci * WS_C + r * WS_R + s * WS_S) : 0.f;
                        }
#pragma unroll
                        for (int i = 0; i < TILE_Y; ++i) {
                            const int hi = (p0 + i * BY) * SH - PH + r * DH;
                            const bool hok = (p0 + i * BY) < PP && hi >= 0 && hi < HH;
#pragma unroll
                            for (int l = 0; l < TILE_X; ++l) {
                                const int wi = (q0 + l * BX) * SW - PW + s * DW;
                                const bool ok = hok && (q0 + l * BX) < QQ && wi >= 0 && wi < WW;
#if GROUPS == 1
                                const float xv = ok ? ld_f(xn + (long long)ci * XS_C + (long long)hi * XS_H + (long long)wi * XS_W) : 0.f;
#pragma unroll
                                for (int j = 0; j < TILE_Z; ++j) acc[j][i][l] = fmaf(xv, wv[j], acc[j][i][l]);
#else
#pragma unroll
                                for (int j = 0; j < TILE_Z; ++j) {
                                    const float xv = (ok && kval[j])
                                        ? ld_f(xn + (long long)(cbase[j] + ci) * XS_C + (long long)hi * XS_H + (long long)wi * XS_W) : 0.f;
                                    acc[j][i][l] = fmaf(xv, wv[j], acc[j][i][l]);
                                }
#endif
                            }
                        }
                    }
                }
            }
        }
    }
#pragma unroll
    for (int j = 0; j < TILE_Z; ++j) {
        const int k = k0 + j * BZ;
        if (!kval[j]) continue;
        const float bias = (EPI >= 1) ? ld_f(b + k) : 0.f;
#pragma unroll
        for (int i = 0; i < TILE_Y; ++i) {
            const int p = p0 + i * BY;
            if (p >= PP) continue;
#pragma unroll
            for (int l = 0; l < TILE_X; ++l) {
                const int q = q0 + l * BX;
                if (q >= QQ) continue;
                float v = acc[j][i][l] + bias;
                const long long yi = (long long)n * YS_N + (long long)k * YS_K + (long long)p * YS_P + (long long)q * YS_Q;
                if (EPI == 3) v += ld_f(z + yi);
                if (EPI >= 2) v = fmaxf(v, 0.f);
                st_f(y + yi, v);
            }
        }
    }
}
)JIT";

// ---- cache -----------------------------------------------------------------------------------------
struct JitEntry {
    std::string cubin;
    std::string log;                       // compile log on failure
    bool failed = false;
    std::map<int, cudaKernel_t> kernel;    // per device
    std::map<int, cudaLibrary_t> lib;
};

static std::mutex g_mu;
static std::map<std::string, JitEntry> g_cache;
static std::string g_dir;
static bool g_dir_init = false;
static std::atomic<long long> g_compiles{0}, g_mem_hits{0}, g_disk_hits{0}, g_failures{0};
static std::atomic<long long> g_compile_ns{0};

static std::string cache_dir() {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!g_dir_init) {
        g_dir_init = true;
        if (const char *e = getenv("WPK_JIT_CACHE_DIR")) g_dir = e;
    }
    return g_dir;
}

void jit_set_cache_dir(const char *dir) {
    std::lock_guard<std::mutex> lk(g_mu);
    g_dir_init = true;
    g_dir = dir ? dir : "";
}

static void add(std::string &s, const char *name, long long v) {
    s += "#define ";
    s += name;
    s += " ";
    s += std::to_string(v);
    s += "\n";
}

// Every constant the generated kernel depends on; also the cache key.
std::string jit_defines(const ConvDesc &d, const Config &c) {
    const int *g = c.genes;
    const long long cpg = d.c / d.g;
    std::string s;
    add(s, "WPK_E", d.elem());
    add(s, "WPK_BF16", d.dtype == WPK_BF16 ? 1 : 0);
    add(s, "BX", g[0]); add(s, "BY", g[1]); add(s, "BZ", g[2]);
    add(s, "TILE_X", g[3]); add(s, "TILE_Y", g[4]); add(s, "TILE_Z", g[5]); add(s, "TRZ", g[6]);
    add(s, "HH", d.h); add(s, "WW", d.w); add(s, "KK", d.k); add(s, "RR", d.r); add(s, "SS", d.s);
    add(s, "PP", d.p); add(s, "QQ", d.q);
    add(s, "SH", d.sh); add(s, "SW", d.sw); add(s, "PH", d.ph); add(s, "PW", d.pw); add(s, "DH", d.dh); add(s, "DW", d.dw);
    add(s, "CPG", cpg); add(s, "KPG", d.k / d.g); add(s, "GROUPS", d.g);
    const int tz = g[2] * g[5];
    add(s, "KBLOCKS", (d.k + tz - 1) / tz);
    add(s, "EPI", d.epilogue);
    if (d.layout == WPK_NCHW) {
        add(s, "XS_N", (long long)d.c * d.h * d.w); add(s, "XS_C", (long long)d.h * d.w); add(s, "XS_H", d.w); add(s, "XS_W", 1);
        add(s, "WS_K", cpg * d.r * d.s); add(s, "WS_C", (long long)d.r * d.s); add(s, "WS_R", d.s); add(s, "WS_S", 1);
        add(s, "YS_N", (long long)d.k * d.p * d.q); add(s, "YS_K", (long long)d.p * d.q); add(s, "YS_P", d.q); add(s, "YS_Q", 1);
    } else {
        add(s, "XS_N", (long long)d.h * d.w * d.c); add(s, "XS_C", 1); add(s, "XS_H", (long long)d.w * d.c); add(s, "XS_W", d.c);
        add(s, "WS_K", (long long)d.r * d.s * cpg); add(s, "WS_C", 1); add(s, "WS_R", (long long)d.s * cpg); add(s, "WS_S", cpg);
        add(s, "YS_N", (long long)d.p * d.q * d.k); add(s, "YS_K", 1); add(s, "YS_P", (long long)d.q * d.k); add(s, "YS_Q", d.k);
    }
    return s;
}

static unsigned long long fnv64(const std::string &s) {
    unsigned long long h = 1469598103934665603ull;
    for (unsigned char ch : s) h = (h ^ ch) * 1099511628211ull;
    return h;
}

static std::string disk_path(const std::string &dir, const std::string &key) {
    char b[64];
    snprintf(b, sizeof b, "/wpk_jit_%016llx.bin", fnv64(key));
    return dir + b;
}

static bool disk_load(const std::string &key, std::string *cubin) {
    const std::string dir = cache_dir();
    if (dir.empty()) return false;
    FILE *f = fopen(disk_path(dir, key).c_str(), "rb");
    if (!f) return false;
    std::string all;
    char buf[65536];
    size_t n;
    while ((n = fread(buf, 1, sizeof buf, f)) > 0) all.append(buf, n);
    fclose(f);
    // file = key, '\0', cubin (the key guards against hash collisions)
    const size_t z = all.find('\0');
    if (z == std::string::npos || all.compare(0, z, key) != 0) return false;
    *cubin = all.substr(z + 1);
    return !cubin->empty();
}

static void disk_store(const std::string &key, const std::string &cubin) {
    const std::string dir = cache_dir();
    if (dir.empty()) return;
    const std::string path = disk_path(dir, key);
    const std::string tmp = path + ".tmp." + std::to_string((long long)std::hash<std::thread::id>()(std::this_thread::get_id()));
    FILE *f = fopen(tmp.c_str(), "wb");
    if (!f) return;
    fwrite(key.data(), 1, key.size(), f);
    fputc('\0', f);
    fwrite(cubin.data(), 1, cubin.size(), f);
    fclose(f);
    rename(tmp.c_str(), path.c_str());   // atomic publish
}

// NVRTC compile of one key (thread-safe; different programs compile concurrently).
static bool nvrtc_compile(const std::string &key, std::string *cubin, std::string *log) {
    const auto t0 = std::chrono::steady_clock::now();
    const std::string src = key + kJitSource;
    nvrtcProgram prog;
    if (nvrtcCreateProgram(&prog, src.c_str(), "wpk_jit_conv.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS) {
        *log = "nvrtcCreateProgram failed";
        return false;
    }
    const char *opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "--device-as-default-execution-space",
                          "-lineinfo"};
    const nvrtcResult r = nvrtcCompileProgram(prog, 4, opts);
    size_t ls = 0;
    nvrtcGetProgramLogSize(prog, &ls);
    if (ls > 1) {
        log->resize(ls);
        nvrtcGetProgramLog(prog, &(*log)[0]);
    }
    bool ok = (r == NVRTC_SUCCESS);
    if (ok) {
        size_t n = 0;
        ok = nvrtcGetCUBINSize(prog, &n) == NVRTC_SUCCESS && n > 0;
        if (ok) {
            cubin->resize(n);
            ok = nvrtcGetCUBIN(prog, &(*cubin)[0]) == NVRTC_SUCCESS;
        }
    }
    nvrtcDestroyProgram(&prog);
    g_compile_ns += (long long)std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count();
    ++g_compiles;
    if (!ok) ++g_failures;
    return ok;
}

// Make sure the cubin for `key` exists in the process cache (disk, else NVRTC). Thread-safe.
static bool ensure_cubin(const std::string &key, std::string *err) {
    {
        std::lock_guard<std::mutex> lk(g_mu);
        auto it = g_cache.find(key);
        if (it != g_cache.end()) {
            if (it->second.failed) {
                if (err) *err = "JIT compile failed: " + it->second.log;
                return false;
            }
            ++g_mem_hits;
            return true;
        }
    }
    JitEntry e;
    if (disk_load(key, &e.cubin)) {
        ++g_disk_hits;
    } else if (!nvrtc_compile(key, &e.cubin, &e.log)) {
        e.failed = true;
    } else {
        disk_store(key, e.cubin);
    }
    std::lock_guard<std::mutex> lk(g_mu);
    auto ins = g_cache.emplace(key, std::move(e));   // a concurrent compile of the same key: first wins
    if (ins.first->second.failed) {
        if (err) *err = "JIT compile failed: " + ins.first->second.log;
        return false;
    }
    return true;
}

bool jit_kernel(const ConvDesc &d, const Config &c, int device, cudaKernel_t *out, std::string *err) {
    const std::string key = jit_defines(d, c);
    if (!ensure_cubin(key, err)) return false;
    std::lock_guard<std::mutex> lk(g_mu);
    JitEntry &e = g_cache[key];
    auto it = e.kernel.find(device);
    if (it != e.kernel.end()) {
        *out = it->second;
        return true;
    }
    cudaLibrary_t lib;
    cudaError_t ce = cudaLibraryLoadData(&lib, e.cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
    if (ce != cudaSuccess) {
        if (err) *err = std::string("cudaLibraryLoadData: ") + cudaGetErrorString(ce);
        return false;
    }
    cudaKernel_t k;
    ce = cudaLibraryGetKernel(&k, lib, "wpk_jit_conv");
    if (ce != cudaSuccess) {
        if (err) *err = std::string("cudaLibraryGetKernel: ") + cudaGetErrorString(ce);
        return false;
    }
    e.lib[device] = lib;
    e.kernel[device] = k;
    *out = k;
    return true;
}

void jit_precompile(const ConvDesc &d, const std::vector<Config> &cfgs, int threads) {
    std::vector<std::string> keys;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        for (const Config &c : cfgs) {
            if (c.family != WPK_FAMILY_JIT) continue;
            std::string k = jit_defines(d, c);
            if (!g_cache.count(k) && std::find(keys.begin(), keys.end(), k) == keys.end()) keys.push_back(k);
        }
    }
    if (keys.empty()) return;
    if (threads <= 0) threads = (int)std::max(1u, std::thread::hardware_concurrency());
    threads = std::min<int>(threads, (int)keys.size());
    std::atomic<size_t> next{0};
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t)
        pool.emplace_back([&] {
            for (size_t i = next++; i < keys.size(); i = next++) ensure_cubin(keys[i], nullptr);
        });
    for (auto &th : pool) th.join();
}

bool jit_compile_only(const ConvDesc &d, const Config &c, size_t *cubin_bytes, std::string *err) {
    const std::string key = jit_defines(d, c);
    if (!ensure_cubin(key, err)) return false;
    std::lock_guard<std::mutex> lk(g_mu);
    if (cubin_bytes) *cubin_bytes = g_cache[key].cubin.size();
    return true;
}

void jit_stats(long long *compiles, long long *mem_hits, long long *disk_hits, long long *failures, double *seconds) {
    if (compiles) *compiles = g_compiles.load();
    if (mem_hits) *mem_hits = g_mem_hits.load();
    if (disk_hits) *disk_hits = g_disk_hits.load();
    if (failures) *failures = g_failures.load();
    if (seconds) *seconds = (double)g_compile_ns.load() * 1e-9;
}

}  // namespace wpk
