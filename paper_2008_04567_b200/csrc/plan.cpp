// Plan creation, shape validation, schedule templates (gene spaces) and config validity.
//
// Shape rules: SURVEY.md §8(b) "Validation -> errors"; output size P/Q: floor formula (reading c3).
// Schedule templates with tunable hyper-parameters: PAPER.md:59 (§2.2); chromosome encoding
// s = {c_0..c_{n-1}}: PAPER.md:64-65; "verified first in order to meet certain constraints ...
// the product of all dimension values is positive and <= 1024": PAPER.md:68.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <string>

#include "wpk_internal.h"
#include "jit.h"

namespace wpk {

static thread_local std::string g_last_error;

void set_error(const std::string &msg) { g_last_error = msg; }

wpk_status fail(wpk_status st, const std::string &msg) {
    g_last_error = msg;
    return st;
}

static int out_size(int in, int pad, int dil, int f, int stride) {
    long long num = (long long)in + 2LL * pad - (long long)dil * (f - 1) - 1;
    if (num < 0) return 0;
    return (int)(num / stride + 1);
}

static wpk_status to_desc(const wpk_conv2d_shape *s, int dtype, ConvDesc *d) {
    if (!s) return fail(WPK_ERR_INVALID_ARGUMENT, "shape is NULL");
    if (s->struct_size != sizeof(wpk_conv2d_shape))
        return fail(WPK_ERR_INVALID_ARGUMENT, "wpk_conv2d_shape.struct_size mismatch (ABI version)");
    if (dtype < WPK_F32 || dtype > WPK_FP8E4M3) return fail(WPK_ERR_INVALID_ARGUMENT, "bad dtype");
    if (s->layout != WPK_NCHW && s->layout != WPK_NHWC) return fail(WPK_ERR_INVALID_ARGUMENT, "bad layout");
    if (s->epilogue < WPK_EPI_NONE || s->epilogue > WPK_EPI_BIAS_ADD_RELU)
        return fail(WPK_ERR_INVALID_ARGUMENT, "bad epilogue");
    const int dims[] = {s->n, s->c, s->h, s->w, s->k, s->r, s->s, s->stride_h, s->stride_w,
                        s->dil_h, s->dil_w, s->groups};
    for (int v : dims)
        if (v < 1) return fail(WPK_ERR_SHAPE, "every dimension, stride, dilation and groups must be >= 1");
    if (s->pad_h < 0 || s->pad_w < 0) return fail(WPK_ERR_SHAPE, "padding must be >= 0");
    if (s->c % s->groups || s->k % s->groups) return fail(WPK_ERR_SHAPE, "C and K must be divisible by groups");
    *d = ConvDesc{s->n, s->c, s->h, s->w, s->k, s->r, s->s, s->stride_h, s->stride_w, s->pad_h,
                  s->pad_w, s->dil_h, s->dil_w, s->groups, s->layout, s->epilogue, 0, 0, dtype};
    d->p = out_size(s->h, s->pad_h, s->dil_h, s->r, s->stride_h);
    d->q = out_size(s->w, s->pad_w, s->dil_w, s->s, s->stride_w);
    if (d->p < 1 || d->q < 1) return fail(WPK_ERR_SHAPE, "output is empty (P or Q < 1)");
    const double elems[] = {(double)s->n * s->c * s->h * s->w, (double)s->k * (s->c / s->groups) * s->r * s->s,
                            (double)s->n * s->k * d->p * d->q};
    for (double e : elems)
        if (e > 4.0e9) return fail(WPK_ERR_UNSUPPORTED, "tensor larger than 2^32 elements");
    return WPK_OK;
}

// ----------------------------------------------------------------------------------------------
// Schedule templates
// ----------------------------------------------------------------------------------------------
static Space make_space(int family) {
    Space sp;
    sp.family = family;
    if (family == WPK_FAMILY_SIMT || family == WPK_FAMILY_JIT) {
        // the paper's own gene set: threads per block and outputs per thread (the JIT
        // family compiles the same template per candidate with NVRTC)
        sp.dom = {{1, 2, 4, 8, 16, 32}, {1, 2, 4, 8, 16, 32}, {1, 2, 4, 8, 16, 32},
                  {1, 2, 4}, {1, 2, 4}, {1, 2, 4}, {1, 2, 4, 8}};
        sp.names = {"T_x", "T_y", "T_z", "Tile_x", "Tile_y", "Tile_z", "Tile_rz"};
    } else if (family == WPK_FAMILY_UMMA) {
        sp.dom = {{16, 32, 64, 96, 128, 192, 256}, {2, 3, 4, 5, 6, 7, 8}, {1, 2, 4, 8, 16},
                  {0, 1, 2, 3, 4, 5, 6, 7}, {0, 1, 2, 3, 4, 5, 6}, {1, 2, 4}, {128, 256}};
        sp.names = {"BLOCK_N", "STAGES", "SPLIT_K", "MODE", "A_MODE", "ACC_STAGES", "BLOCK_M"};
    } else if (family == WPK_FAMILY_GEMM32) {
        sp.dom = {{64, 128}, {64, 128}, {8, 16}, {4, 8}, {1, 2, 4, 8}, {0}, {0}};
        sp.names = {"BLOCK_M", "BLOCK_N", "BLOCK_K", "THREAD_TILE", "SPLIT_K", "-", "-"};
    } else {
        sp.dom = {{1, 2, 4, 8}, {1, 2, 4}, {64, 128, 256, 512}, {1}, {0}, {0}, {0}};
        sp.names = {"VEC_C", "PIX_PER_THREAD", "THREADS", "-", "-", "-", "-"};
    }
    return sp;
}

const Space &family_space(int family) {
    static const Space spaces[5] = {make_space(0), make_space(1), make_space(2), make_space(3), make_space(4)};
    return spaces[family < 0 || family > 4 ? 0 : family];
}

static bool in_domain(const Space &sp, const Config &cfg, std::string *why) {
    for (int g = 0; g < WPK_NUM_GENES; ++g) {
        const auto &d = sp.dom[g];
        if (std::find(d.begin(), d.end(), cfg.genes[g]) == d.end()) {
            if (why) *why = std::string("gene ") + sp.names[g] + " = " + std::to_string(cfg.genes[g]) + " not in its domain";
            return false;
        }
    }
    return true;
}

bool family_applicable(const ConvDesc &d, int family, std::string *why) {
    auto no = [&](const char *m) { if (why) *why = m; return false; };
    if (d.dtype == WPK_FP8E4M3 && family != WPK_FAMILY_UMMA)
        return no("FP8 (e4m3) runs on the tcgen05 family only (kind::f8f6f4)");
    if (d.fused_dw) {   // the depthwise result is the A operand of the tcgen05 pointwise GEMM
        if (family != WPK_FAMILY_UMMA) return no("fused depthwise+pointwise runs on the tcgen05 family only");
        if (d.dtype != WPK_BF16 && d.dtype != WPK_F16) return no("fused depthwise+pointwise needs bf16 or fp16 data");
        return true;
    }
    if (family == WPK_FAMILY_SIMT) return true;   // the SIMT kernel handles every valid shape, layout and dtype
    if (family == WPK_FAMILY_JIT) return true;    // so does its NVRTC-specialised twin
    if (family == WPK_FAMILY_DW) {
        if (d.g < 2) return no("DW family needs groups > 1 (depthwise or grouped)");
        return true;
    }
    if (family == WPK_FAMILY_GEMM32) {
        if (d.dtype != WPK_F32) return no("GEMM32 family is the exact-fp32 path (dtype F32)");
        if (d.g != 1) return no("GEMM32 family needs groups == 1");
        return true;
    }
    if (family == WPK_FAMILY_UMMA) {
        if (d.dtype == WPK_F32) return no("UMMA family needs tf32/bf16/fp16 (F32 is the exact CUDA-core path)");
        if (d.g != 1) {   // general groups on the tensor cores (gconv_tc.cu, A_MODE 1)
            if (d.c == d.g && d.k == d.g) return no("UMMA family: depthwise convs run on the DW family");
            if (d.dtype != WPK_BF16 && d.dtype != WPK_F16) return no("UMMA grouped conv needs bf16 / fp16");
            if (d.layout != WPK_NHWC) return no("UMMA grouped conv needs NHWC");
            if ((d.c / d.g) % 4) return no("UMMA grouped conv needs C/groups % 4 == 0");
            if (d.k / d.g > 256) return no("UMMA grouped conv needs K/groups <= 256");
            if ((double)d.n * d.h * d.w * d.c >= 2147483647.0 || (double)d.M() * d.k >= 2147483647.0)
                return no("UMMA grouped conv needs < 2^31 elements per tensor");
            return true;
        }
        if (d.sh > 8 || d.sw > 8) return no("TMA im2col traversal stride must be <= 8");
        // TMA im2col 4-D bounding-box corners must lie in [-128, 127] (cuda.h cuTensorMapEncodeIm2col)
        int lo_h = -d.ph, lo_w = -d.pw, up_h = d.ph - (d.r - 1) * d.dh, up_w = d.pw - (d.s - 1) * d.dw;
        for (int v : {lo_h, lo_w, up_h, up_w})
            if (v < -128 || v > 127) return no("TMA im2col corner out of [-128,127]");
        if ((d.r - 1) * d.dh > 65535 || (d.s - 1) * d.dw > 65535) return no("im2col offset too large");
        return true;
    }
    return no("unknown family");
}

static int round_up(int a, int b) { return (a + b - 1) / b * b; }

bool umma_geometry(const ConvDesc &d, const Config &cfg, UmmaGeom *g, std::string *why) {
    auto no = [&](const std::string &m) { if (why) *why = m; return false; };
    const int e = d.in_elem();    // bytes per x / w element (the K-major operands)
    const int eo = d.elem();      // bytes per y element
    g->bm = cfg.genes[6];
    g->bn = cfg.genes[0];
    g->bk = 128 / e;           // one 128-byte swizzle atom of K per stage
    g->stages = cfg.genes[1];
    g->splits = cfg.genes[2];
    g->raster = cfg.genes[3] & 1;
    g->pair = (cfg.genes[3] >> 1) & 1;   // tcgen05 CTA pair (cta_group::2): 256-row tiles over two SMs
    // MODE bit 2: dual accumulators. Consecutive MMAs into one accumulator wait for its
    // read-modify-write (~107 cycles for 128 x 128 x 16 vs 64 of tensor work, tools/mma_ring.cu);
    // a 128-row tile alternates its K steps between two accumulators, summed by the epilogue
    g->kdual = (cfg.genes[3] >> 2) & 1;
    g->ctas_per_sm = 1;
    g->a_mode = cfg.genes[4];
    // A_MODE 4: the TMA producer of A_MODE 0 with its K blocks dealt round robin over three
    // producer warps (A and B boxes of a stage from one thread) instead of an A / B warp split
    g->prod_rr = 0;
    g->kgroup = 1;
    if (g->a_mode == 4) {
        g->a_mode = 0;
        g->prod_rr = 1;
    }
    // A_MODE 5 / 6: the TMA producers of A_MODE 0 / 4 with K groups -- two consecutive K blocks of a
    // work item per full / empty barrier pair (one expect_tx, one wait and one MMA commit per two
    // blocks); STAGES counts K-block slots, so it must be even and >= 4 (>= 2 groups in flight)
    if (g->a_mode == 5 || g->a_mode == 6) {
        static const int no_kgroup = env_knob("WPK_NO_KGROUP", 0);   // A/B experiments only
        if (no_kgroup) return no("A_MODE 5/6 disabled (WPK_NO_KGROUP)");
        if (g->stages % 2 || g->stages < 4) return no("A_MODE 5/6 (K groups of 2) need an even STAGES >= 4");
        g->prod_rr = (g->a_mode == 6) ? 1 : 0;
        g->a_mode = 0;
        static const int kg_half = env_knob("WPK_KG_HALF", 0);   // experiment: two groups of STAGES/2 blocks
        g->kgroup = kg_half ? g->stages / 2 : 2;
    }
    g->acc_stages = cfg.genes[5];
    g->seg_sp = 0; g->seg_hp = 0; g->seg_wp = 0; g->seg_fast = 0; g->seg_two = 0;
    if (d.dtype == WPK_FP8E4M3 && g->a_mode != 0)
        return no("FP8 (e4m3) is instantiated for the TMA A producers only (A_MODE 0 / 4)");
    if (d.g > 1) {
        // grouped conv on the tensor cores (gconv_tc.cu, internal A_MODE 7): one tile = 128 pixels x
        // BLOCK_N / Np groups; the only gene is BLOCK_N (a multiple of the per-group MMA width Np)
        const int kpg = d.k / d.g;
        const int np = std::max(16, round_up(kpg, 16));
        if (cfg.genes[4] != 1 || g->stages != 2 || g->splits != 1 || cfg.genes[3] != 0 || g->acc_stages != 1 || g->bm != 128)
            return no("UMMA grouped conv: genes must be {BLOCK_N, 2, 1, 0, 1, 1, 128}");
        if (g->bn % np) return no("UMMA grouped conv: BLOCK_N must be a multiple of the per-group MMA width");
        if (g->bn / np > d.g) return no("UMMA grouped conv: BLOCK_N covers more groups than the layer has");
        g->a_mode = 7;
        g->cpad = d.c;
        g->c_blocks = (d.r * d.s * (d.c / d.g) + 63) / 64;
        g->num_kb = g->c_blocks;
        g->kb_per_split = g->num_kb;
        g->m_tiles = (int)((d.M() + 127) / 128);
        g->n_tiles = (d.g + g->bn / np - 1) / (g->bn / np);
        g->work = (long long)g->m_tiles * g->n_tiles;
        g->epi_tma = 0; g->csplit = 0; g->pair = 0; g->kdual = 0; g->prod_rr = 0; g->a_tiled = 0;
        g->smem_bytes = 1024 + 2 * 16384 + 2 * (size_t)np * 128 + 64;
        int cols = 32;
        while (cols < g->bn) cols <<= 1;
        g->tmem_cols = cols;
        return true;
    }
    if (d.fused_dw) {
        // fused depthwise + pointwise: the A producer computes the depthwise conv (internal A_MODE 5);
        // the gene's other producers do not apply, K = the depthwise channels (C % 8 == 0)
        // A_MODE 0: the persistent tcgen05 kernel with a depthwise producer (internal A_MODE 5);
        // A_MODE 1: the one-tile-per-CTA kernel of dwpw.cu (internal A_MODE 6), whose only free
        // parameter is none: canonical genes {cover(K_out), 2, 1, 0, 1, 1, 128}
        if (cfg.genes[4] != 0 && cfg.genes[4] != 1)
            return no("fused depthwise+pointwise: A_MODE 0 (persistent, depthwise producer warps) or 1 (one tile per CTA)");
        if ((cfg.genes[3] >> 1) & 3) return no("fused depthwise+pointwise: no CTA pairs / dual accumulators");
        // the depthwise result of an M tile is computed once per N tile: BLOCK_N must cover K_out
        // (up to the widest tile) so that no tile recomputes it
        int cover = 16;
        for (int v : {16, 32, 64, 96, 128, 192, 256}) {
            cover = v;
            if (v >= std::min(round_up(d.k, 16), 256)) break;
        }
        if (g->bn < cover) return no("fused depthwise+pointwise: BLOCK_N must cover K_out (min(K_out, 256))");
        if (cfg.genes[4] == 1) {
            if (g->bn != cover || g->stages != 2 || cfg.genes[3] != 0 || g->acc_stages != 1 || g->bm != 128)
                return no("fused depthwise+pointwise A_MODE 1: genes must be {cover(K_out), 2, SPLIT_K, 0, 1, 1, 128}");
            // SPLIT_K: the 64-channel chunks split over SPLIT_K CTAs per tile (fp32 partials in the
            // workspace, summed in split order by a second kernel)
            const int nkc = (d.c + 63) / 64;
            const int per = (nkc + g->splits - 1) / g->splits;
            if (g->splits > nkc || (long long)(g->splits - 1) * per >= nkc)
                return no("fused depthwise+pointwise A_MODE 1: SPLIT_K leaves an empty split");
            if (d.k % 8) return no("fused depthwise+pointwise A_MODE 1: K_out % 8 == 0 (16-byte output rows)");
            if (d.k > 512) return no("fused depthwise+pointwise A_MODE 1: K_out <= 512 (TMEM columns)");
            if (d.M() >= 2147483647LL - 128) return no("fused depthwise+pointwise A_MODE 1: M < 2^31");
            g->a_mode = 6;
            g->cpad = d.c;
            g->c_blocks = (d.c + 63) / 64;
            g->num_kb = g->c_blocks;
            g->kb_per_split = (g->num_kb + g->splits - 1) / g->splits;
            g->m_tiles = (int)((d.M() + 127) / 128);
            g->n_tiles = 1;
            g->work = (long long)g->m_tiles * g->splits;
            g->epi_tma = 0; g->csplit = 0; g->pair = 0; g->kdual = 0; g->prod_rr = 0; g->a_tiled = 0;
            g->smem_bytes = 1024 + 2 * 16384 + 2 * (size_t)round_up(d.k, 16) * 128 + 64;
            int cols = 32;
            while (cols < round_up(d.k, 16)) cols <<= 1;
            g->tmem_cols = cols;
            return true;
        }
        g->a_mode = 5;
        g->cpad = d.c;
        g->c_blocks = (d.c + g->bk - 1) / g->bk;
        g->num_kb = g->c_blocks;
    } else if ((g->a_mode == 1 || g->a_mode == 2) && d.c >= 64) {
        return no("A_MODE 1/2 (explicit im2col / gather) is reserved for layers with C < 64");
    }
    if (g->a_mode == 5) {
        // (fused depthwise producer: set above)
    } else if (g->a_mode == 3) {
        // pixel-segment gather (C <= 4): activations stored NHWC with 4 channels per pixel (8 or 16
        // bytes); K row = (r, s', c) with s' padded to Sp so that one 16-byte smem chunk holds whole
        // pixels of a single filter row; weights for s' >= S and c >= C are zero.
        if (d.c > 4) return no("A_MODE 3 (pixel-segment gather) needs C <= 4");
        if (g->stages < 3) return no("A_MODE 3 keeps two stages of copies in flight: STAGES >= 3");
        if ((double)d.n * d.h * d.w * 4 >= 2147483647.0) return no("segment gather needs < 2^31 input elements");
        const int ppc = 16 / (4 * e);                         // pixels per 16-byte chunk: 2 (16-bit), 1 (tf32)
        g->seg_sp = round_up(d.s, ppc);
        g->cpad = d.r * g->seg_sp * 4;
        // the activations are re-laid into an explicitly zero-padded image (no bounds checks in
        // the gather); the extra columns cover the dummy filter columns s' in [S, Sp)
        g->seg_hp = d.h + 2 * d.ph;
        // one 16-byte copy per chunk when its PPC pixels are adjacent (dil_w 1); with an odd stride a
        // second copy of the image shifted by one pixel keeps every chunk 16-byte aligned (rows of
        // odd q*stride_w read the shifted copy)
        g->seg_fast = (ppc == 1) || d.dw == 1;
        g->seg_two = (ppc == 2 && d.dw == 1 && d.sw % 2 == 1) ? 1 : 0;
        g->seg_wp = round_up(d.w + 2 * d.pw + (g->seg_sp - d.s) * d.dw + g->seg_two, 2);   // even: 16-B rows
        if ((long long)d.n * g->seg_hp > 65535) return no("segment gather re-layout grid: N * (H + 2 pad_h) > 65535");
        if ((double)d.n * g->seg_hp * g->seg_wp * 4 * (1 + g->seg_two) >= 2147483647.0)
            return no("segment gather needs < 2^31 padded elements");
        g->c_blocks = (g->cpad + g->bk - 1) / g->bk;
        g->num_kb = g->c_blocks;
    } else if (g->a_mode == 1 || g->a_mode == 2) {
        // explicit im2col (1: A = [M][R*S*C] materialised in the workspace, then a plain GEMM) or the
        // fused gather producer (2: the same K order built directly in shared memory)
        g->cpad = round_up(d.r * d.s * d.c, 8);   // 8-element vectors in the im2col kernel
        g->c_blocks = (g->cpad + g->bk - 1) / g->bk;
        g->num_kb = g->c_blocks;
        if (g->a_mode == 1 && (double)d.M() * g->cpad * e > 4.0e9) return no("explicit im2col matrix larger than 4 GB");
        if (g->a_mode == 1 && (size_t)128 * g->cpad * e > 48 * 1024) return no("explicit im2col row block exceeds 48 KB of smem");
        if (g->a_mode == 2 && (double)d.n * d.c * d.h * d.w >= 2147483647.0) return no("gather producer needs < 2^31 input elements");
    } else {
        g->cpad = round_up(d.c, 16 / e);    // TMA global strides must be multiples of 16 B
        g->c_blocks = (g->cpad + g->bk - 1) / g->bk;
        g->num_kb = d.r * d.s * g->c_blocks;
    }
    if (g->splits > g->num_kb) return no("SPLIT_K larger than the number of K blocks");
    if (g->splits > 1 && d.epilogue == WPK_EPI_BIAS_ADD_RELU) return no("the residual epilogue needs SPLIT_K = 1");
    g->kb_per_split = (g->num_kb + g->splits - 1) / g->splits;
    if ((long long)(g->splits - 1) * g->kb_per_split >= g->num_kb) return no("SPLIT_K leaves an empty split");
    g->m_tiles = (int)((d.M() + g->bm - 1) / g->bm);
    g->n_tiles = (d.k + g->bn - 1) / g->bn;
    g->work = (long long)g->m_tiles * g->n_tiles * g->splits;
    if (g->work >= 2147483647LL / 2) return no("too many work items (tiles x splits >= 2^30)");
    if (g->kdual) {
        if (!g->pair && g->bm != 128) return no("dual accumulators: 1-CTA 128-row tiles or CTA pairs (BLOCK_M 256 over two SMs alternates its MMAs already)");
        if (g->splits != 1) return no("dual accumulators need SPLIT_K = 1");
        if (g->a_mode != 0) return no("dual accumulators are instantiated for the TMA A producer (A_MODE 0)");
    }
    if (g->pair) {
        if (g->bm != 256) return no("a CTA pair computes 256-row tiles (BLOCK_M must be 256)");
        if (g->a_mode >= 2) return no("CTA pairs do not support the gather producers");
    }
    size_t stage = g->pair ? (size_t)128 * 128 + (size_t)(g->bn / 2) * 128 : (size_t)g->bm * 128 + (size_t)g->bn * 128;
    if (g->bm == 256 && g->a_mode == 0 && !(d.r == 1 && d.s == 1 && d.sh == 1 && d.sw == 1 && d.ph == 0 && d.pw == 0))
        ;   // a 256-pixel im2col box is one TMA (pixelsPerColumn <= 1024)
    // A operand: a 1x1 / stride-1 / unpadded conv is a plain GEMM on x viewed as [N*H*W][C]
    g->a_tiled = (g->a_mode == 1 || (g->a_mode != 5 && d.r == 1 && d.s == 1 && d.sh == 1 && d.sw == 1 && d.ph == 0 && d.pw == 0 &&
                                      g->cpad == d.c && !getenv("WPK_A_IM2COL"))) ? 1 : 0;
    // epilogue through shared memory + TMA store: NHWC output, whole 128-byte column chunks
    // (split-K: the owner split stores the output the same way; the others store fp32 partials in
    // 32-column chunks, which always divide a 128-byte output chunk)
    const int cw = 128 / eo;
    g->epi_tma = (d.layout == WPK_NHWC && g->bn % cw == 0 && ((long long)d.k * eo) % 16 == 0 &&
                  !getenv("WPK_EPI_DIRECT")) ? 1 : 0;
    const size_t smem_cap = 227 * 1024;
    const size_t bias_bytes = (size_t)round_up(d.k, 256) * 4;   // fp32, zero-padded past K
    const size_t fixed = 1024 /*align slack*/ + bias_bytes + 256 /*barriers*/;
    // 8 epilogue warps x {2, else 1} staging buffers x 32 rows x 128 B
    g->epi_bufs = (g->epi_tma && (size_t)g->stages * stage + 8 * 2 * 4096 + fixed <= smem_cap) ? 2 : 1;
    size_t off = (size_t)g->stages * stage;
    g->epi_off = off;
    if (g->epi_tma) off += (size_t)8 * g->epi_bufs * 4096;
    // Split-K inside a thread-block cluster (DSMEM reduction): the S splits of a tile are the S CTAs
    // of one cluster, each CTA owns BN/S output columns and receives the others' fp32 partials of
    // them into its (by then idle) pipeline stages. Needs one tile per CTA (grid = work), whole
    // 128-byte output chunks per owner, and the receive area within the stage buffers.
    g->csplit = 0;
    g->recv_stride = 0;
    if (g->splits > 1 && g->splits <= 8 && (g->splits & (g->splits - 1)) == 0 && !g->pair && g->a_mode == 0 &&
        g->epi_tma && !getenv("WPK_NO_CSPLIT")) {
        const int slice = g->bn / g->splits;
        const size_t rstride = (size_t)slice * 4 + 16;
        const size_t recv = (size_t)(g->splits - 1) * g->bm * rstride;
        // (one wave only: with one tile per CTA, later waves would pay the whole prologue again)
        if (g->bn % (g->splits * cw) == 0 && recv <= (size_t)g->stages * stage && g->work <= device_sm_count(d.device)) {
            g->csplit = 1;
            g->recv_stride = (int)rstride;
        }
    }
    g->bias_off = off;
    off += bias_bytes;
    g->bar_off = off;
    off += 256;
    g->smem_bytes = 1024 /*align slack*/ + off;
    if (g->smem_bytes > smem_cap) return no("STAGES x tile exceeds shared memory");
    int cols = g->acc_stages * (g->pair ? 1 : g->bm / 128) * g->bn * (g->kdual ? 2 : 1);
    int alloc = 32;
    while (alloc < cols) alloc <<= 1;
    g->tmem_cols = alloc;
    if (alloc * g->ctas_per_sm > 512) return no("TMEM columns exceed 512 per SM");
    if (g->bn > round_up(d.k, 16) * 2 && g->bn > 16) return no("BLOCK_N more than 2x the output channels");
    return true;
}

bool config_valid(const ConvDesc &d, const Config &cfg, std::string *why) {
    if (cfg.family < 0 || cfg.family > 4) { if (why) *why = "bad family"; return false; }
    if (!family_applicable(d, cfg.family, why)) return false;
    if (!in_domain(family_space(cfg.family), cfg, why)) return false;
    const int *gn = cfg.genes;
    if (cfg.family == WPK_FAMILY_SIMT || cfg.family == WPK_FAMILY_JIT) {
        long long threads = (long long)gn[0] * gn[1] * gn[2];
        if (threads < 1 || threads > 1024) {
            if (why) *why = "T_x*T_y*T_z must be in [1, 1024]";
            return false;
        }
        if (cfg.family == WPK_FAMILY_SIMT && d.elem() == 2 && gn[6] != 1) {   // 16-bit SIMT variants are instantiated with Tile_rz = 1 only
            if (why) *why = "Tile_rz must be 1 for 16-bit dtypes on the SIMT family";
            return false;
        }
        long long gy = (d.p + (long long)gn[1] * gn[4] - 1) / ((long long)gn[1] * gn[4]);
        long long gz = (long long)d.n * ((d.k + (long long)gn[2] * gn[5] - 1) / ((long long)gn[2] * gn[5]));
        if (gy > 65535 || gz > 65535) { if (why) *why = "grid y/z exceeds 65535"; return false; }
        return true;
    }
    if (cfg.family == WPK_FAMILY_UMMA) {
        UmmaGeom g;
        return umma_geometry(d, cfg, &g, why);
    }
    if (cfg.family == WPK_FAMILY_GEMM32) {
        if ((d.k + gn[1] - 1) / gn[1] > 65535) { if (why) *why = "grid y exceeds 65535"; return false; }
        const int nk = (d.r * d.s * round_up(d.c, 4) + gn[2] - 1) / gn[2];
        if (gn[4] > 1 && (gn[4] > nk || (long long)(gn[4] - 1) * ((nk + gn[4] - 1) / gn[4]) >= nk)) {
            if (why) *why = "SPLIT_K leaves an empty split";
            return false;
        }
        if (gn[4] > 1 && (double)gn[4] * d.M() * d.k * 4 > 8.0e9) { if (why) *why = "split-K partials exceed 8 GB"; return false; }
        return true;
    }
    // DW: depthwise (vector over channels = groups) or grouped (vector over a group's outputs)
    int vec = gn[0];
    if (d.elem() * vec > 16) { if (why) *why = "VEC_C*elem > 16 bytes"; return false; }
    if (d.c == d.g && d.k == d.g) {
        if (d.c % vec) { if (why) *why = "VEC_C must divide C"; return false; }
        if (d.layout == WPK_NCHW && vec != 1) { if (why) *why = "NCHW depthwise needs VEC_C = 1"; return false; }
    } else if ((d.k / d.g) % vec) {
        if (why) *why = "grouped: VEC_C must divide K/groups";
        return false;
    }
    return true;
}

int default_family(const ConvDesc &d) {
    if (d.dtype == WPK_FP8E4M3) return WPK_FAMILY_UMMA;   // the only family with an e4m3 kernel
    if (d.g > 1) return WPK_FAMILY_DW;   // depthwise and grouped kernels
    if (family_applicable(d, WPK_FAMILY_UMMA, nullptr)) return WPK_FAMILY_UMMA;
    if (family_applicable(d, WPK_FAMILY_GEMM32, nullptr)) return WPK_FAMILY_GEMM32;
    return WPK_FAMILY_SIMT;
}

Config default_config(const ConvDesc &d, int family) {
    Config c;
    c.family = family;
    if (family == WPK_FAMILY_SIMT || family == WPK_FAMILY_JIT) {
        int g[7] = {16, 4, 4, 1, 1, 1, 1};
        std::memcpy(c.genes, g, sizeof g);
        return c;
    }
    if (family == WPK_FAMILY_GEMM32) {
        // 64 x 64 CTA tiles of 4 x 4 outputs per thread, 16-deep K steps, no split: the most common
        // tuned choice on ResNet-50 (profiles/r1e_suite_f32.md)
        int g[7] = {64, 64, 16, 4, 1, 0, 0};
        std::memcpy(c.genes, g, sizeof g);
        return c;
    }
    if (family == WPK_FAMILY_DW) {
        const bool depthwise = d.c == d.g && d.k == d.g;
        int vec = (depthwise && d.layout == WPK_NCHW) ? 1 : 16 / d.elem();
        while (vec > 1 && (depthwise ? d.c : d.k / d.g) % vec) vec >>= 1;
        int g[7] = {vec, 1, 256, 1, 0, 0, 0};
        std::memcpy(c.genes, g, sizeof g);
        return c;
    }
    // UMMA default: BLOCK_M 128; BLOCK_N 128 when that still leaves < ~1 wave of 256-wide tiles
    // (more SMs busy), else the widest (<= 256) that does not pad K by more than 2x -- per-SM L2->SMEM
    // feed (~70 B/clk, tools/tma_bench.cu) bounds a K step and wide tiles have the best FLOP/byte.
    int bn = 16;
    for (int v : {256, 128, 64, 32, 16}) {
        if (v > 16 && v / 2 >= d.k) continue;
        bn = v;
        break;
    }
    const long long mt = (d.M() + 127) / 128;
    if (bn == 256 && mt * ((d.k + 255) / 256) < 120) bn = 128;
    if (d.fused_dw) {   // fused depthwise + pointwise: 128-row 1-CTA tiles, the depthwise producer,
        // the narrowest BLOCK_N that covers K_out (the depthwise result is computed once per M tile)
        for (int v : {16, 32, 64, 96, 128, 192, 256}) {
            bn = v;
            if (v >= std::min(round_up(d.k, 16), 256)) break;
        }
        int g1[7] = {bn, 2, 1, 0, 1, 1, 128};   // the one-tile-per-CTA kernel (dwpw.cu) when it applies
        std::memcpy(c.genes, g1, sizeof g1);
        if (config_valid(d, c, nullptr)) return c;
        int g[7] = {bn, 4, 1, 0, 0, 2, 128};
        std::memcpy(c.genes, g, sizeof g);
        for (int st = 8; st >= 2; --st) {
            c.genes[1] = st;
            if (config_valid(d, c, nullptr)) return c;
        }
        return c;   // (the plan call reports it invalid)
    }
    // large layers: a tcgen05 CTA pair (256 x BLOCK_N over two SMs) halves B traffic per SM
    // (not for short-K layers: with 1-2 K blocks per tile a pair's accumulators are seen ~3 us
    // after the commit, DESIGN.md §10 finding 13, while 1-CTA 128 x 256 tiles stream)
    const int kblocks = d.r * d.s * ((d.c + 63) / 64);
    const bool big = ((d.M() + 255) / 256) * ((d.k + bn - 1) / bn) >= 2 * 148 && bn >= 128 && d.c >= 64 && kblocks > 2;
    c.genes[0] = bn; c.genes[1] = 4; c.genes[2] = 1; c.genes[3] = 0; c.genes[4] = (d.c <= 4) ? 3 : (d.c < 16) ? 1 : 0;
    c.genes[5] = 2; c.genes[6] = 128;
    if (big) { c.genes[3] = 2; c.genes[6] = 256; }
    // small-C layers (pixel-segment gather): many short tiles -> 256-row tiles, and few stages
    // (the gather keeps STAGES-1 of them in flight; more only costs shared memory)
    const bool seg = d.c <= 4 && c.genes[4] == 3;
    if (seg && d.M() >= 256LL * 148) c.genes[6] = 256;
    for (int am : {c.genes[4], 2, 0}) {   // small C: explicit im2col, else the gather producer
        c.genes[4] = am;
        bool ok = false;
        for (int st = (seg && am == 3) ? 4 : 8; st >= 2 && !ok; --st) {
            c.genes[1] = st;
            ok = config_valid(d, c, nullptr);
        }
        if (ok) break;
    }
    // Split-K is left to the tuner: its fixup re-reads fp32 partials and is only a win for
    // very deep, very narrow layers.
    if (!config_valid(d, c, nullptr)) {   // shape too odd for the defaults: fall back to SIMT
        return default_config(d, WPK_FAMILY_SIMT);
    }
    return c;
}

}  // namespace wpk

using namespace wpk;

extern "C" {

const char *wpk_last_error(void) { return g_last_error.c_str(); }

void wpk_tune_options_init(wpk_tune_options *o) {
    if (!o) return;
    std::memset(o, 0, sizeof *o);
    o->struct_size = sizeof *o;
    o->world = 1;
    o->warmup = 3;
    o->reps = 11;
    o->l2_flush = 2;
    o->eval_mode = WPK_EVAL_MEASURED;
    o->family = WPK_FAMILY_AUTO;
    o->ga_pop = 48; o->ga_elites = 4; o->ga_pool = 48; o->ga_max_gen = 50;
    o->ga_mutation = 0.1; o->ga_eps = 0.02;
    o->rl_envs = 1; o->rl_horizon = 64; o->rl_epochs = 4; o->rl_minibatch = 16;
    o->rl_gamma = 0.99; o->rl_mu = 0.95; o->rl_clip = 0.2; o->rl_c1 = 0.15; o->rl_c2 = 20.0;
    o->rl_lr = 1e-4; o->rl_keep_prob = 0.85;
    o->rl_hidden[0] = 512; o->rl_hidden[1] = 1024; o->rl_hidden[2] = 1024; o->rl_hidden[3] = 512;
    o->rl_alpha_mode = 0;
    o->rl_adv_norm = 1;
    o->rl_restart_every = 1;
    o->seed_default = 1;
    o->finalists = 4;
}

wpk_status wpk_conv2d_output_dims(const wpk_conv2d_shape *shape, int32_t *p, int32_t *q) {
    if (!p || !q) return fail(WPK_ERR_INVALID_ARGUMENT, "NULL output pointer");
    ConvDesc d;
    wpk_status st = to_desc(shape, WPK_F32, &d);
    if (st != WPK_OK && st != WPK_ERR_UNSUPPORTED) return st;
    if (st == WPK_ERR_UNSUPPORTED) {   // dims are still well defined
        set_error("");
    }
    *p = d.p;
    *q = d.q;
    if (d.p < 1 || d.q < 1) return fail(WPK_ERR_SHAPE, "output is empty");
    return WPK_OK;
}

wpk_status wpk_conv2d_plan(const wpk_conv2d_shape *shape, wpk_dtype dtype, int device, wpk_plan *out) {
    if (!out) return fail(WPK_ERR_INVALID_ARGUMENT, "out is NULL");
    *out = nullptr;
    if (device < 0) return fail(WPK_ERR_INVALID_ARGUMENT, "device must be >= 0");
    ConvDesc d;
    wpk_status st = to_desc(shape, (int)dtype, &d);
    if (st != WPK_OK) return st;
    d.device = device;
    if (d.dtype == WPK_FP8E4M3) {
        std::string why;
        if (!family_applicable(d, WPK_FAMILY_UMMA, &why)) return fail(WPK_ERR_UNSUPPORTED, "FP8 (e4m3): " + why);
    }
    Plan *p = new (std::nothrow) Plan();
    if (!p) return fail(WPK_ERR_OUT_OF_MEMORY, "host allocation failed");
    p->d = d;
    p->device = device;
    p->cfg = default_config(d, default_family(d));
    std::string why;
    if (!config_valid(d, p->cfg, &why)) {
        delete p;
        return fail(WPK_ERR_EXHAUSTED, "no valid default config: " + why);
    }
    *out = reinterpret_cast<wpk_plan>(p);
    return WPK_OK;
}

wpk_status wpk_dwpw_plan(const wpk_conv2d_shape *dw, int32_t k_out, wpk_epilogue pw_epilogue, wpk_dtype dtype,
                         int device, wpk_plan *out) {
    if (!out) return fail(WPK_ERR_INVALID_ARGUMENT, "out is NULL");
    *out = nullptr;
    if (device < 0) return fail(WPK_ERR_INVALID_ARGUMENT, "device must be >= 0");
    if (k_out < 1) return fail(WPK_ERR_SHAPE, "k_out must be >= 1");
    if (pw_epilogue < WPK_EPI_NONE || pw_epilogue > WPK_EPI_BIAS_RELU)
        return fail(WPK_ERR_INVALID_ARGUMENT, "fused depthwise+pointwise: pointwise epilogue NONE / BIAS / BIAS_RELU");
    ConvDesc d;
    wpk_status st = to_desc(dw, (int)dtype, &d);
    if (st != WPK_OK) return st;
    if (d.g != d.c || d.k != d.c) return fail(WPK_ERR_SHAPE, "fused depthwise+pointwise: the first conv must be depthwise (groups == C == K)");
    if (d.epilogue == WPK_EPI_BIAS_ADD_RELU) return fail(WPK_ERR_UNSUPPORTED, "fused depthwise+pointwise: no residual epilogue on the depthwise conv");
    if (d.layout != WPK_NHWC) return fail(WPK_ERR_UNSUPPORTED, "fused depthwise+pointwise: NHWC only");
    if (d.dtype != WPK_BF16 && d.dtype != WPK_F16) return fail(WPK_ERR_UNSUPPORTED, "fused depthwise+pointwise: bf16 / fp16 only");
    if (d.c % 8) return fail(WPK_ERR_UNSUPPORTED, "fused depthwise+pointwise: C must be a multiple of 8 (16-byte vectors)");
    if ((double)d.n * d.c * d.h * d.w >= 2147483647.0) return fail(WPK_ERR_UNSUPPORTED, "fused depthwise+pointwise: input >= 2^31 elements");
    d.device = device;
    d.fused_dw = 1;
    d.dw_epi = d.epilogue;
    d.epilogue = pw_epilogue;
    d.k = k_out;
    d.g = 1;
    if ((double)d.n * d.p * d.q * d.k > 4.0e9) return fail(WPK_ERR_UNSUPPORTED, "tensor larger than 2^32 elements");
    Plan *p = new (std::nothrow) Plan();
    if (!p) return fail(WPK_ERR_OUT_OF_MEMORY, "host allocation failed");
    p->d = d;
    p->device = device;
    p->cfg = default_config(d, WPK_FAMILY_UMMA);
    std::string why;
    if (!config_valid(d, p->cfg, &why)) {
        delete p;
        return fail(WPK_ERR_EXHAUSTED, "no valid default config: " + why);
    }
    *out = reinterpret_cast<wpk_plan>(p);
    return WPK_OK;
}

wpk_status wpk_conv2d_get_config(wpk_plan plan, int32_t *family, int32_t *genes) {
    if (!plan || !family || !genes) return fail(WPK_ERR_INVALID_ARGUMENT, "NULL argument");
    Plan *p = reinterpret_cast<Plan *>(plan);
    *family = p->cfg.family;
    std::memcpy(genes, p->cfg.genes, sizeof p->cfg.genes);
    return WPK_OK;
}

int32_t wpk_conv2d_config_valid(wpk_plan plan, int32_t family, const int32_t *genes) {
    if (!plan || !genes) { set_error("NULL argument"); return 0; }
    Plan *p = reinterpret_cast<Plan *>(plan);
    Config c;
    c.family = family;
    std::memcpy(c.genes, genes, sizeof c.genes);
    std::string why;
    if (!config_valid(p->d, c, &why)) { set_error(why); return 0; }
    return 1;
}

wpk_status wpk_conv2d_set_config(wpk_plan plan, int32_t family, const int32_t *genes) {
    if (!plan || !genes) return fail(WPK_ERR_INVALID_ARGUMENT, "NULL argument");
    Plan *p = reinterpret_cast<Plan *>(plan);
    Config c;
    c.family = family;
    std::memcpy(c.genes, genes, sizeof c.genes);
    std::string why;
    if (!config_valid(p->d, c, &why)) return fail(WPK_ERR_INVALID_CONFIG, why);
    p->cfg = c;   // launch_conv re-keys the workspace state on the config
    return WPK_OK;
}

wpk_status wpk_conv2d_invalidate(wpk_plan plan) {
    if (!plan) return fail(WPK_ERR_INVALID_ARGUMENT, "NULL plan");
    reinterpret_cast<Plan *>(plan)->reset_ws_state();
    return WPK_OK;
}

wpk_status wpk_jit_compile(wpk_plan plan, const int32_t *genes, size_t *cubin_bytes) {
    if (!plan || !genes) return fail(WPK_ERR_INVALID_ARGUMENT, "NULL argument");
    Plan *p = reinterpret_cast<Plan *>(plan);
    Config c;
    c.family = WPK_FAMILY_JIT;
    for (int g = 0; g < WPK_NUM_GENES; ++g) c.genes[g] = genes[g];
    std::string why;
    if (!config_valid(p->d, c, &why)) return fail(WPK_ERR_INVALID_CONFIG, "JIT config invalid: " + why);
    size_t n = 0;
    if (!jit_compile_only(p->d, c, &n, &why)) return fail(WPK_ERR_INTERNAL, why);
    if (cubin_bytes) *cubin_bytes = n;
    return WPK_OK;
}

wpk_status wpk_jit_set_cache_dir(const char *dir) {
    jit_set_cache_dir(dir);
    return WPK_OK;
}

wpk_status wpk_jit_stats(int64_t *compiles, int64_t *mem_hits, int64_t *disk_hits, int64_t *failures,
                         double *compile_seconds) {
    long long c, m, dh, f;
    double s;
    jit_stats(&c, &m, &dh, &f, &s);
    if (compiles) *compiles = c;
    if (mem_hits) *mem_hits = m;
    if (disk_hits) *disk_hits = dh;
    if (failures) *failures = f;
    if (compile_seconds) *compile_seconds = s;
    return WPK_OK;
}

wpk_status wpk_family_describe(int32_t family, int32_t *counts, int32_t *values, const char **names) {
    if (family < 0 || family > 4 || !counts || !values) return fail(WPK_ERR_INVALID_ARGUMENT, "bad argument");
    const Space &sp = family_space(family);
    for (int g = 0; g < WPK_NUM_GENES; ++g) {
        counts[g] = (int)sp.dom[g].size();
        for (size_t i = 0; i < sp.dom[g].size() && i < 32; ++i) values[g * 32 + i] = sp.dom[g][i];
        if (names) names[g] = sp.names[g];
    }
    return WPK_OK;
}

int32_t wpk_conv2d_last_launch_count(wpk_plan plan) {
    return plan ? reinterpret_cast<Plan *>(plan)->last_launches : 0;
}

wpk_status wpk_conv2d_tune_stats(wpk_plan plan, double *best_us, int32_t *measured, int32_t *rounds,
                                 double *seconds) {
    if (!plan) return fail(WPK_ERR_INVALID_ARGUMENT, "NULL plan");
    Plan *p = reinterpret_cast<Plan *>(plan);
    if (best_us) *best_us = p->best_us;
    if (measured) *measured = p->measured;
    if (rounds) *rounds = p->rounds;
    if (seconds) *seconds = p->tune_seconds;
    return WPK_OK;
}

}  // extern "C"
