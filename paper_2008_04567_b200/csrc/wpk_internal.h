// Internal declarations shared by the libwpk.so translation units (host C++ and CUDA).
// Never included by oracle/ (task rule ③: the oracle shares no code with the product).
#pragma once

#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include "wpk.h"

namespace wpk {

// --- error reporting -----------------------------------------------------------------------------
void set_error(const std::string &msg);
wpk_status fail(wpk_status st, const std::string &msg);

// --- the GEMM view of one convolution (PAPER.md:86-93 O_conv shape, generalised) ----------------
struct ConvDesc {
    int n, c, h, w, k, r, s;
    int sh, sw, ph, pw, dh, dw, g;
    int layout, epilogue;
    int p, q;          // output spatial size
    int dtype;         // wpk_dtype
    int device = 0;    // CUDA device of the plan (SM count for one-wave checks)
    // fused depthwise + pointwise plan (wpk_dwpw_plan): (n, c, h, w, r, s, strides, pads, dils) are
    // the depthwise conv's (groups = C), k the pointwise output channels; p, q the depthwise output;
    // `epilogue` applies to the pointwise output, dw_epi to the depthwise intermediate
    int fused_dw = 0;
    int dw_epi = 0;
    long long M() const { return (long long)n * p * q; }
    long long flops() const {
        if (fused_dw) return 2LL * n * p * q * c * ((long long)r * s + k);
        return 2LL * n * k * p * q * (c / g) * r * s;
    }
    // bytes per element of y / b / z (the output side) and of x / w (the input side): they differ
    // only for WPK_FP8E4M3 (e4m3 x and w, bf16 b, z and y)
    int elem() const { return (dtype == WPK_BF16 || dtype == WPK_F16 || dtype == WPK_FP8E4M3) ? 2 : 4; }
    int in_elem() const { return dtype == WPK_FP8E4M3 ? 1 : elem(); }
    int out_dtype() const { return dtype == WPK_FP8E4M3 ? WPK_BF16 : dtype; }
};

struct Config {
    int family = WPK_FAMILY_SIMT;
    int genes[WPK_NUM_GENES] = {0, 0, 0, 0, 0, 0, 0};
    bool operator==(const Config &o) const {
        if (family != o.family) return false;
        for (int i = 0; i < WPK_NUM_GENES; ++i)
            if (genes[i] != o.genes[i]) return false;
        return true;
    }
    bool operator<(const Config &o) const {
        if (family != o.family) return family < o.family;
        for (int i = 0; i < WPK_NUM_GENES; ++i)
            if (genes[i] != o.genes[i]) return genes[i] < o.genes[i];
        return false;
    }
};

// Gene domains of one family ("schedule template", PAPER.md:59 / 65).
struct Space {
    int family;
    std::vector<std::vector<int>> dom;   // 7 domains
    std::vector<const char *> names;
};
const Space &family_space(int family);
// Hardware/shape constraints; on false, *why says which ("verified first").
bool config_valid(const ConvDesc &d, const Config &cfg, std::string *why);
Config default_config(const ConvDesc &d, int family);
int default_family(const ConvDesc &d);
bool family_applicable(const ConvDesc &d, int family, std::string *why);

// --- UMMA family: derived launch geometry --------------------------------------------------------
struct UmmaGeom {
    int bm, bn, bk, stages, splits, raster, ctas_per_sm, acc_stages;
    int c_blocks, num_kb, kb_per_split, m_tiles, n_tiles;
    long long work;
    int cpad;           // channel count as stored for the kernel (C rounded up to the alignment)
    int pair;           // 1: tcgen05 CTA pair (cta_group::2, cluster of 2), 256 x BLOCK_N tiles
    int kdual;          // 1: two accumulators per tile (even / odd 16-wide K steps), summed in the epilogue
    int prod_rr;        // 1: TMA producers deal K blocks round robin over 3 warps (A_MODE 4 / 6)
    int kgroup;         // K blocks per full / empty barrier group: 2 for A_MODE 5 / 6, else 1
    int a_mode;         // 0: TMA im2col (or tiled for 1x1), 1: explicit im2col matrix in the workspace,
                        // 2: element gather into smem, 3: pixel-segment gather (C <= 4)
    int seg_sp;         // A_MODE 3: filter columns per row padded to whole 16-byte chunks
    int seg_hp, seg_wp; // A_MODE 3: zero-padded image height / width (pixels of 4 channels)
    int seg_fast;       // A_MODE 3: every 16-byte chunk is one aligned copy (tf32, or 16-bit with dil_w 1)
    int seg_two;        // A_MODE 3: a second, one-pixel-shifted image copy (16-bit, odd stride_w)
    int a_tiled;        // 1: A fetched by a plain 2-D TMA tile load (1x1, stride 1, pad 0), else im2col
    int epi_bufs;       // staging buffers per epilogue warp (2 = double-buffered TMA stores)
    int epi_tma;        // 1: epilogue stages 32x128-byte tiles in smem and TMA-stores them
    int csplit;         // 1: split-K reduced inside a cluster of SPLIT_K CTAs through DSMEM
    int recv_stride;    // csplit: bytes per received partial row (BN/S fp32 + 16 B pad)
    size_t smem_bytes;
    size_t epi_off, bias_off, bar_off;   // byte offsets of the epilogue staging, bias, barriers
    int tmem_cols;
};
bool umma_geometry(const ConvDesc &d, const Config &cfg, UmmaGeom *g, std::string *why);

// --- device-side entry points (implemented in .cu files) -----------------------------------------
struct Workspace {
    char *base = nullptr;
    size_t bytes = 0;
};

struct Plan;
size_t workspace_bytes(Plan &p, const Config &cfg, bool host_staging);
// Launch everything for one run on `stream`; returns number of kernel launches or -1 (error set).
// (w_dw, b_dw: the depthwise weights / bias of a fused depthwise+pointwise plan, else unused)
int launch_conv(Plan &p, const Config &cfg, const void *x, const void *w, const void *b, void *y,
                void *stream, char *ws, size_t ws_bytes, const void *z = nullptr, const void *w_dw = nullptr,
                const void *b_dw = nullptr);
int device_sm_count(int device);
// environment knob read once per process (experiments and debugging only)
int env_knob(const char *name, int dflt);
int device_l2_bytes(int device);

struct Plan {
    ConvDesc d;
    int device = 0;
    Config cfg;
    // workspace
    char *ws_user = nullptr;
    size_t ws_user_bytes = 0;
    char *ws_own = nullptr;
    size_t ws_own_bytes = 0;
    // Persistent per-plan state in the workspace (the workspace belongs to ONE plan): the packed
    // weights and the zeroed split-K counters. Both are keyed by (workspace base, config) as well
    // as by the weight pointer / counter address; reset_ws_state() forgets them whenever the
    // workspace changes or another config has run over it.
    const void *packed_for = nullptr;
    int packed_cfg_family = -1;
    Config packed_cfg;
    const char *state_ws = nullptr;   // workspace base the state below refers to
    int last_launches = 0;
    void *map_cache = nullptr;   // UmmaMapCache (umma_conv.h)
    unsigned long long *dbg = nullptr;   // per-plan kernel timeline (tools only; overrides the global)
    // UMMA geometry of the last config launched (host-side cost of a run: one comparison, not a
    // re-derivation; WPK_* environment knobs are therefore read when a config is first used)
    Config geom_cfg;
    UmmaGeom geom;
    bool geom_ok = false;
    char *counters_at = nullptr; // split-K counters known to be zero at this address
    size_t counters_bytes = 0;
    Config counters_cfg;
    void reset_ws_state() {
        packed_for = nullptr;
        packed_cfg_family = -1;
        counters_at = nullptr;
        counters_bytes = 0;
        state_ws = nullptr;
    }
    // tune stats
    double best_us = 0, tune_seconds = 0;
    int measured = 0, rounds = 0;
};

}  // namespace wpk
