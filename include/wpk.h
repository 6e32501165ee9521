/*
 * wpk.h -- C ABI of the B200-native Woodpecker-DL hot path (libwpk.so).
 *
 * The operation (§2.2 Halide listing; PAPER.md:15 and SPEC.md:136 for the fused
 * epilogue): forward 2-D convolution for inference,
 *
 *   y[n,k,p,q] = act( b[k] + sum_{c<C/g, r<R, s<S}
 *                     x[n, g(k)*C/g + c, p*stride_h - pad_h + r*dil_h, q*stride_w - pad_w + s*dil_w]
 *                     * w[k, c, r, s] ),           act = ReLU | identity,  x = 0 outside the image,
 *   P = floor((H + 2 pad_h - dil_h (R-1) - 1)/stride_h) + 1   (same for Q with W, S),
 *
 * together with the per-layer search that picks the kernel configuration ("identify most efficient
 * codes per operator"; GA §2.3; RL-search §2.4).
 *
 * Conventions
 *  - Every call returns wpk_status; no C++ exception crosses the ABI. On error a human-readable
 *    message is available from wpk_last_error() (thread-local; valid until the next call on the
 *    same thread).
 *  - Device pointers are CUDA device pointers on the plan's device (allocated by the caller, e.g.
 *    by PyTorch). Host pointers are plain process memory. Nothing here takes a torch type.
 *  - Layouts (dense, row-major in the order given):
 *      WPK_NCHW: x [N][C][H][W],  w [K][C/g][R][S] (KCRS),  y [N][K][P][Q]
 *      WPK_NHWC: x [N][H][W][C],  w [K][R][S][C/g] (KRSC),  y [N][P][Q][K]
 *      b [K] (or NULL iff epilogue == WPK_EPI_NONE); residual z (WPK_EPI_BIAS_ADD_RELU) laid out as y.
 *  - dtypes: x, w, b, y share one element type (except WPK_FP8E4M3, below):
 *      WPK_F32  float32, exact fp32 FMA on CUDA cores (strict-comparison path)
 *      WPK_TF32 float32 in/out, tf32 tensor-core products, fp32 accumulate
 *      WPK_BF16 bfloat16 in/out, fp32 accumulate;  WPK_F16 float16 in/out, fp32 accumulate.
 *      WPK_FP8E4M3 (NEXT-4): x and w are OCP float8 e4m3 ("e4m3fn": 1 sign, 4 exponent, 3 mantissa
 *               bits, bias 7, no infinities; torch.float8_e4m3fn), b, z and y are bfloat16;
 *               tcgen05.mma kind::f8f6f4 with fp32 accumulate. Tensor-core family only
 *               (WPK_FAMILY_UMMA, A_MODE 0, 4, 5 or 6, groups 1); other families return
 *               WPK_ERR_UNSUPPORTED at plan time. x and w are taken as given (no scaling: a
 *               per-tensor scale folds into w and b outside the library).
 *    The accumulator is fp32; bias is up-converted to fp32 and added before ReLU; the output is
 *    rounded to nearest-even once.
 */
#ifndef WPK_H
#define WPK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define WPK_API __attribute__((visibility("default")))
#else
#define WPK_API
#endif

#define WPK_ABI_VERSION 1
#define WPK_NUM_GENES 7

typedef enum {
    WPK_OK = 0,
    WPK_ERR_INVALID_ARGUMENT = 1, /* NULL / misaligned pointer, bad enum, bad option value     */
    WPK_ERR_SHAPE = 2,            /* any dim < 1, P or Q < 1, C % g != 0, K % g != 0            */
    WPK_ERR_UNSUPPORTED = 3,      /* device not sm_100                                          */
    WPK_ERR_INVALID_CONFIG = 4,   /* genes outside the family's space or violating a constraint */
    WPK_ERR_EXHAUSTED = 5,        /* no valid config could be sampled / every candidate failed  */
    WPK_ERR_CUDA = 6,             /* CUDA runtime/driver error (message in wpk_last_error)      */
    WPK_ERR_OUT_OF_MEMORY = 7,    /* workspace too small / allocation failure                   */
    WPK_ERR_INTERNAL = 8          /* broken invariant (e.g. ranks disagree on the chosen config) */
} wpk_status;

typedef enum { WPK_F32 = 0, WPK_TF32 = 1, WPK_BF16 = 2, WPK_F16 = 3, WPK_FP8E4M3 = 4 } wpk_dtype;
typedef enum { WPK_NCHW = 0, WPK_NHWC = 1 } wpk_layout;
/* WPK_EPI_BIAS_ADD_RELU: y = max(conv + b + z, 0) with a residual z of y's shape, layout and dtype
 * (the last conv of a ResNet block fused with its shortcut add). Run it
 * with wpk_conv2d_run_residual; the tcgen05 family supports it with SPLIT_K = 1. */
typedef enum { WPK_EPI_NONE = 0, WPK_EPI_BIAS = 1, WPK_EPI_BIAS_RELU = 2, WPK_EPI_BIAS_ADD_RELU = 3 } wpk_epilogue;
typedef enum { WPK_SEARCH_GA = 0, WPK_SEARCH_RL = 1, WPK_SEARCH_RANDOM = 2 } wpk_search;
typedef enum { WPK_EVAL_MEASURED = 0, WPK_EVAL_REPLAY = 1, WPK_EVAL_SYNTHETIC = 2 } wpk_eval_mode;

/* Kernel families ("schedule templates"). Each has 7 genes (PAPER.md:65 chromosome
 * s = {c_0..c_6}); their meaning per family is listed by wpk_family_describe().
 *   WPK_FAMILY_SIMT : direct conv on CUDA cores, genes = the paper's
 *                     (T_x, T_y, T_z, Tile_x, Tile_y, Tile_z, Tile_rz), T_x*T_y*T_z<=1024;
 *                     every shape, dtype, layout and groups
 *   WPK_FAMILY_UMMA : tcgen05 implicit GEMM, genes = (BLOCK_N, STAGES, SPLIT_K, MODE,
 *                     A_MODE, ACC_STAGES, BLOCK_M); MODE bit 0 = raster order, bit 1 = CTA pair
 *                     (cta_group::2, 256-row tiles across two SMs, BLOCK_M must be 256), bit 2 =
 *                     dual accumulators (1-CTA BLOCK_M 128 or a pair, SPLIT_K 1: even / odd K steps
 *                     into two TMEM accumulators summed by the epilogue); A_MODE 0 = TMA im2col producer
 *                     (plain TMA tiles for 1x1/s1/p0), 1 = explicit im2col matrix in the workspace,
 *                     2 = fused gather producer (im2col built in shared memory; small-C layers),
 *                     3 = pixel-segment gather (C <= 4), 4 = A_MODE 0 with the K blocks dealt round
 *                     robin over three TMA producer warps (A + B of a stage from one thread),
 *                     5 / 6 = A_MODE 0 / 4 with K groups: two consecutive K blocks share one full /
 *                     empty barrier pair (STAGES = K-block slots, even, >= 4). Grouped plans
 *                     (1 < groups < C, NHWC 16-bit) accept only A_MODE 1 = the tensor-core grouped
 *                     kernel, genes {BLOCK_N, 2, 1, 0, 1, 1, 128} (a handful of valid points: set them
 *                     with wpk_conv2d_set_config / measure, a sampled search rejects most draws);
 *                     fused depthwise+pointwise plans
 *                     accept A_MODE 0 (depthwise producer warps) and 1 (one tile per CTA)
 *   WPK_FAMILY_DW   : grouped conv on CUDA cores, groups > 1: depthwise (groups == C == K, vector
 *                     over channels) or general groups (vector over VEC_C outputs of one group,
 *                     VEC_C | K/groups), genes = (VEC_C, PIX_PER_THREAD, THREADS, -, -, -, -)
 *   WPK_FAMILY_GEMM32 : exact-fp32 implicit GEMM on CUDA cores (WPK_F32, groups == 1), genes =
 *                     (BLOCK_M, BLOCK_N, BLOCK_K, THREAD_TILE, SPLIT_K, -, -); the F32 default;
 *                     SPLIT_K > 1 sums per-split fp32 partials in split order (deterministic)
 *   WPK_FAMILY_JIT  : the SIMT template generated per candidate with every shape parameter and gene
 *                     a compile-time constant and compiled just in time with NVRTC for sm_100a
 *                     (PAPER.md:68 Step2 "compile the generated codes just-in-time ... then execute
 *                     them"); same genes and arithmetic as SIMT (bit-identical results), every Tile_rz
 *                     for every dtype. Compiled cubins are cached per process and, with a cache
 *                     directory, on disk; the tuner compiles each generation's new candidates on a
 *                     pool of host threads before measuring them. Opt-in (never a
 *                     plan's default): tune with family = WPK_FAMILY_JIT or set_config. */
typedef enum {
    WPK_FAMILY_SIMT = 0, WPK_FAMILY_UMMA = 1, WPK_FAMILY_DW = 2, WPK_FAMILY_GEMM32 = 3, WPK_FAMILY_JIT = 4,
    WPK_FAMILY_AUTO = -1
} wpk_family;

/* Operator shape: the first 9 entries of the paper's O_conv generalised with
 * explicit symmetric padding, dilation and groups (reading c2, c4). */
typedef struct {
    uint32_t struct_size; /* = sizeof(wpk_conv2d_shape) */
    int32_t n, c, h, w, k, r, s;
    int32_t stride_h, stride_w, pad_h, pad_w, dil_h, dil_w, groups;
    int32_t layout;   /* wpk_layout   */
    int32_t epilogue; /* wpk_epilogue */
} wpk_conv2d_shape;

/* All-gather of `bytes_per_rank` bytes from every rank: recv[r*bytes_per_rank ...] = send of rank
 * r. Must be called collectively by every rank in the same order. Return 0 on success. Used by
 * wpk_conv2d_tune to share fitness records when candidate evaluation is sharded over GPUs
 * (BASELINE.json north_star: "an NCCL all-gather of fitness values"). */
typedef int (*wpk_exchange_fn)(void *ctx, const void *send, size_t bytes_per_rank, void *recv);

typedef struct {
    uint32_t struct_size;     /* = sizeof(wpk_tune_options); fill with wpk_tune_options_init */
    uint64_t seed;            /* counter-RNG seed (default 0)                                   */
    int32_t rank, world;      /* this process's rank and the number of ranks (default 0, 1)    */
    wpk_exchange_fn exchange; /* required when world > 1                                        */
    void *exchange_ctx;
    int32_t warmup, reps;     /* timing protocol: W untimed + R reps (1..1024) bracketed by device
                                 globaltimer stamps, interquartile mean (defaults 3, 11) */
    int32_t l2_flush;         /* cache policy of a timed rep: 0 = warm (back-to-back single launches),
                               * 1 = read a 2x-L2 buffer before each single-launch rep, 2 (default) = one
                               * rep is a CUDA graph of P back-to-back launches over P copies of x / y
                               * with P x (|x| + |y|) >= 2 x L2 (every launch reads cold inputs; the
                               * stamps, ~2-us steps on this part, span P launches; consecutive
                               * launches overlap through PDL as in a network step), beta = span / P */
    int32_t eval_mode;        /* wpk_eval_mode (default MEASURED)                               */
    int32_t family;           /* wpk_family to search; WPK_FAMILY_AUTO = the plan's default      */
    const char *record_path;  /* if set: append every measured record as JSONL (with world > 1
                               * every rank writes the same gathered table: give each its own path) */
    const char *replay_path;  /* if set with EVAL_REPLAY: read records instead of measuring     */
    const char *log_path;     /* if set: per-generation (GA) / per-step (RL) history JSONL      */
    double synthetic[1 + 2 * WPK_NUM_GENES]; /* EVAL_SYNTHETIC: base, w[7], c*[7] */
    /* GA (defaults per DESIGN.md reading c15) */
    int32_t ga_pop, ga_elites, ga_pool, ga_max_gen;
    double ga_mutation, ga_eps;
    /* PPO (defaults per DESIGN.md readings c21-c24) */
    int32_t rl_envs, rl_horizon, rl_epochs, rl_minibatch;
    double rl_gamma, rl_mu, rl_clip, rl_c1, rl_c2, rl_lr, rl_keep_prob;
    int32_t rl_hidden[4];     /* 512, 1024, 1024, 512                                          */
    int32_t rl_alpha_mode;    /* 0 = the paper's alpha_t = (0.8 alpha + beta)/t, 1 = EMA        */
    int32_t rl_adv_norm;      /* 1 = normalise advantages per update batch (default 1)          */
    int32_t rl_restart_every; /* >0: envs restart from the best-ever config every N updates (1)  */
    int32_t max_seconds;      /* wall-clock cap for one tune (0 = none)                         */
    int32_t seed_default;     /* 1 (default): the plan's expert default config is one of the first
                               * candidates (GA individual 0, RL env 0, first random sample)      */
    const char *cache_dir;    /* if set: tuning-result cache. One JSON file per key =
                               * operator identity (shapes, filter, stride, padding;
                               * plus dilation, groups, dtype, layout, epilogue) + family + device.
                               * A hit whose recorded budget >= the request costs 0 evaluations.
                               * Writes are atomic (temp file + rename). With world > 1 a hit is
                               * used only if every rank's lookup returns the same record.       */
    int32_t finalists;        /* EVAL_MEASURED: the top-k configs by measured beta are re-timed on
                               * EVERY rank after the search and the one with the lowest median
                               * across ranks is chosen (SURVEY.md 8(d) protocol item 2; the
                               * single best-ever timing is biased low). 0 = off; default 4.     */
} wpk_tune_options;

typedef struct wpk_plan_s *wpk_plan;

/* Fill defaults (seed 0, rank 0, world 1, W=3, R=11, L2 flush, measured, GA 48/4/48/50/0.1/0.02,
 * PPO E=1 T=64 epochs 4 minibatch 16 gamma .99 mu .95 clip .2 c1 .15 c2 20 lr 1e-4 keep .85,
 * 4 finalists). Stop decisions (max_seconds, a fatal CUDA error on any rank) are collective:
 * every rank leaves the search after the same exchange. */
WPK_API void wpk_tune_options_init(wpk_tune_options *opts);

/* Output spatial size (host only; no device needed). WPK_ERR_SHAPE if P or Q < 1. */
WPK_API wpk_status wpk_conv2d_output_dims(const wpk_conv2d_shape *shape, int32_t *p, int32_t *q);

/* Validate the shape, form the implicit-GEMM view, choose the kernel family for (dtype, groups,
 * alignment) and a deterministic valid default config: groups > 1 -> WPK_FAMILY_DW (depthwise or
 * grouped kernel); WPK_F32 -> WPK_FAMILY_GEMM32; tf32/bf16/f16 -> WPK_FAMILY_UMMA when the TMA
 * im2col limits hold, else WPK_FAMILY_SIMT. Host only: no CUDA call is made until the first
 * run/tune. `device` is the CUDA ordinal the plan will run on. *out owns host state only. */
WPK_API wpk_status wpk_conv2d_plan(const wpk_conv2d_shape *shape, wpk_dtype dtype, int device, wpk_plan *out);

/* Search the plan's configuration space with GA / RL / random search, at most `budget` distinct
 * measured configs; on success the best config found becomes the plan's config. A candidate that
 * fails (launch error, invalid) scores beta = +inf and is recorded, not returned; returns
 * WPK_ERR_EXHAUSTED only if every candidate failed. With EVAL_REPLAY / EVAL_SYNTHETIC no GPU is
 * touched and the result is a pure function of (shape, dtype, search, budget, seed, records),
 * identical for every world size. opts may be NULL (defaults). */
WPK_API wpk_status wpk_conv2d_tune(wpk_plan plan, wpk_search search, int32_t budget, const wpk_tune_options *opts);

/* Time the plan's current config with the tuner's protocol (the fitness measurement of a candidate,
 * PAPER.md:68): `warmup` untimed runs, then `reps` runs each bracketed by device %globaltimer
 * stamps under the cache policy l2_flush (0 / 1 / 2, see wpk_tune_options), interquartile mean in
 * microseconds -> *us.
 * Uses its own synthetic buffers and stream, synchronises; WPK_ERR_CUDA if the launch fails. */
WPK_API wpk_status wpk_conv2d_measure(wpk_plan plan, int32_t warmup, int32_t reps, int32_t l2_flush, double *us);

/* Run the convolution on `stream` (a cudaStream_t; NULL = legacy default stream). Asynchronous:
 * no host synchronisation, no allocation once a workspace is set. Pointers must be 16-byte
 * aligned device pointers laid out as described above. Packed weights are cached per w pointer
 * (weights are inference constants); after mutating w in place call
 * wpk_conv2d_invalidate. One stream at a time per plan. */
WPK_API wpk_status wpk_conv2d_run(wpk_plan plan, const void *x, const void *w, const void *b, void *y, void *stream);

/* run for WPK_EPI_BIAS_ADD_RELU plans: z is the residual, a device tensor laid out exactly like y
 * (it may not alias y). WPK_ERR_INVALID_ARGUMENT if the plan's epilogue is not BIAS_ADD_RELU, if z
 * or b is NULL, or if z is not 16-byte aligned; wpk_conv2d_run on such a plan fails the same way. */
WPK_API wpk_status wpk_conv2d_run_residual(wpk_plan plan, const void *x, const void *w, const void *b, const void *z,
                                           void *y, void *stream);

/* Fused depthwise + pointwise convolution ("the MobileNet block"; the
 * operator fusion of PAPER.md:15 and :35 -- "one CUDA kernel function for the fused operator"):
 *   t = RN(dw_epilogue(depthwise_conv(x, w_dw) + b_dw))        (PAPER.md:47's conv with groups = C)
 *   y = pw_epilogue(t (*) w_pw + b_pw)                          (a 1x1 conv, stride 1, pad 0)
 * in ONE kernel: the tcgen05 pointwise GEMM's A operand (row = output pixel of the depthwise conv,
 * K = its C channels) is computed by producer warps in shared memory and never written to global
 * memory. t is rounded to the I/O dtype exactly as the unfused depthwise conv would store it, so the
 * fused result equals the unfused chain's (bit for bit on exact-integer inputs).
 *  dw:  the depthwise conv's shape (groups == C == K, NHWC, C % 8 == 0; stride / pad / dilation
 *       any; dw->epilogue = NONE / BIAS / BIAS_RELU is applied to t); k_out = pointwise output
 *       channels; pw_epilogue = NONE / BIAS / BIAS_RELU. dtype BF16 or F16.
 *  Errors: WPK_ERR_SHAPE (not depthwise, k_out < 1, as wpk_conv2d_plan), WPK_ERR_UNSUPPORTED
 *  (NCHW, other dtypes, C % 8 != 0, residual epilogues), WPK_ERR_INVALID_ARGUMENT.
 *  The plan is tuned, configured and sized with the wpk_conv2d_* calls (tcgen05 family, A_MODE 0 =
 *  the depthwise producer; no CTA pairs); run it with wpk_dwpw_run only. */
WPK_API wpk_status wpk_dwpw_plan(const wpk_conv2d_shape *dw, int32_t k_out, wpk_epilogue pw_epilogue, wpk_dtype dtype,
                                 int device, wpk_plan *out);
/* x [N][H][W][C]; w_dw [C][R][S] (torch's depthwise weight [C][1][R][S], or NHWC [C][R][S][1]);
 * b_dw [C] (NULL iff dw epilogue NONE); w_pw [K][C] (torch [K][C][1][1] or NHWC [K][1][1][C]);
 * b_pw [K] (NULL iff pw epilogue NONE); y [N][P][Q][K]. All device pointers, 16-byte aligned, the
 * plan's dtype. Asynchronous on `stream`; the repacked w_dw is cached per pointer. */
WPK_API wpk_status wpk_dwpw_run(wpk_plan plan, const void *x, const void *w_dw, const void *b_dw, const void *w_pw,
                                const void *b_pw, void *y, void *stream);

/* Same as run, but x and y are HOST pointers: copies x host->device, runs, copies y back, all on
 * `stream`, then synchronises the stream. Device staging buffers live in the workspace. */
WPK_API wpk_status wpk_conv2d_run_host(wpk_plan plan, const void *x_host, const void *w, const void *b,
                               void *y_host, void *stream);

/* Same as run_host without the final synchronisation: the H2D copy, the kernels and the D2H copy
 * are only enqueued on `stream`; y_host is valid after the caller synchronises that stream (x_host
 * must stay untouched until then). Pinned host memory makes the copies asynchronous, so plans on
 * different streams overlap their copies with each other's kernels. */
WPK_API wpk_status wpk_conv2d_run_host_async(wpk_plan plan, const void *x_host, const void *w, const void *b,
                                             void *y_host, void *stream);

WPK_API void wpk_conv2d_destroy(wpk_plan plan);
WPK_API const char *wpk_last_error(void);

/* Workspace: bytes the current config needs (layout transform, channel pad, packed weights,
 * split-K partials, host-run staging). The caller may provide it (e.g. a torch tensor); if never
 * set, the plan allocates and owns one on first run. set_workspace with a too-small buffer ->
 * WPK_ERR_OUT_OF_MEMORY. */
WPK_API wpk_status wpk_conv2d_workspace_size(wpk_plan plan, size_t *bytes);
WPK_API wpk_status wpk_conv2d_set_workspace(wpk_plan plan, void *dev_ptr, size_t bytes);

/* Current config: *family and genes[0..6]. set_config validates (WPK_ERR_INVALID_CONFIG). */
WPK_API wpk_status wpk_conv2d_get_config(wpk_plan plan, int32_t *family, int32_t *genes);
WPK_API wpk_status wpk_conv2d_set_config(wpk_plan plan, int32_t family, const int32_t *genes);
/* 1 if (family, genes) is valid for this plan, else 0 (and the reason in wpk_last_error). */
WPK_API int32_t wpk_conv2d_config_valid(wpk_plan plan, int32_t family, const int32_t *genes);

/* Drop the packed-weight / tensor-map caches (call after mutating weights in place). The
 * workspace holds persistent per-plan state (packed weights, self-resetting split-K counters):
 * it belongs to ONE plan and may not be shared by plans whose runs can interleave; the state is
 * re-derived whenever the workspace or the plan's config changes. */
WPK_API wpk_status wpk_conv2d_invalidate(wpk_plan plan);

/* Inference batch-norm folded into the convolution's weights and bias (constant folding; SURVEY.md
 * 8(f) NEXT-1b): for  y = gamma * (conv(x, w) + b - mean) / sqrt(var + eps) + beta  it writes
 *   w_out[k, ...] = w[k, ...] * s_k,   b_out[k] = (b[k] - mean[k]) * s_k + beta[k],
 *   s_k = gamma[k] / sqrt(var[k] + eps),
 * computed in fp32 and rounded once to the plan's dtype, so that run(x, w_out, b_out) computes the
 * conv + BN (+ the plan's epilogue). w / w_out: the plan's weight layout and dtype (w_out may alias
 * w); b: [K] in the plan's dtype or NULL (= 0); b_out [K] in the plan's dtype; gamma, beta, mean,
 * var: fp32 [K]. All device pointers, enqueued on `stream` (no sync). Call wpk_conv2d_invalidate
 * if w_out is a weight buffer the plan has already packed. */
WPK_API wpk_status wpk_conv2d_fold_batchnorm(wpk_plan plan, const void *w, const void *b, const float *gamma,
                                             const float *beta, const float *mean, const float *var, float eps,
                                             void *w_out, void *b_out, void *stream);

/* Describe a family's gene domains: for gene g, domain values are written to
 * values[g*32 .. g*32+counts[g]-1] (at most 32 per gene). names may be NULL. */
WPK_API wpk_status wpk_family_describe(int32_t family, int32_t *counts, int32_t *values, const char **names);

/* Number of kernel launches the last wpk_conv2d_run issued on its stream (for bench accounting). */
WPK_API int32_t wpk_conv2d_last_launch_count(wpk_plan plan);

/* Tuning history of the last tune: best beta (us), number of distinct measured configs,
 * generations/steps, wall seconds. */
WPK_API wpk_status wpk_conv2d_tune_stats(wpk_plan plan, double *best_us, int32_t *measured, int32_t *rounds,
                                 double *seconds);

/* JIT family (WPK_FAMILY_JIT). wpk_jit_compile: generate and compile (NVRTC, sm_100a) the kernel of
 * the plan's shape with `genes`, or take it from the cache; no GPU is needed. *cubin_bytes (may be
 * NULL) receives the cubin size. WPK_ERR_INVALID_CONFIG if the genes are invalid for the JIT family,
 * WPK_ERR_INTERNAL with the NVRTC log in wpk_last_error if compilation fails.
 * wpk_jit_set_cache_dir: directory for the on-disk cubin cache (NULL or "" = memory only; default
 * from the environment variable WPK_JIT_CACHE_DIR). The directory must exist; files are written
 * atomically (temp + rename) and carry their key, so concurrent processes may share it.
 * wpk_jit_stats: process-wide counters since load: NVRTC compiles, in-memory hits, disk hits,
 * failed compiles, and the summed compile wall time in seconds (any pointer may be NULL). */
WPK_API wpk_status wpk_jit_compile(wpk_plan plan, const int32_t *genes, size_t *cubin_bytes);
WPK_API wpk_status wpk_jit_set_cache_dir(const char *dir);
WPK_API wpk_status wpk_jit_stats(int64_t *compiles, int64_t *mem_hits, int64_t *disk_hits, int64_t *failures,
                                 double *compile_seconds);

/* RL-search learner primitives, exported so the C++ learner can be checked against the oracle
 * (tests/test_tuner_parity.py). dims[0..5] = {obs, h1, h2, h3, h4, A+1}. params is the flat
 * concatenation of (W1[h1][obs], b1, ..., W5[A+1][h4], b5) in float64. Computes the PPO loss
 * -L and its gradient for one batch; mask (B x h4, or NULL) is the dropout mask. */
WPK_API wpk_status wpk_ppo_loss_grad(const int32_t *dims, const double *params, int32_t batch, const double *obs,
                             const int32_t *actions, const double *old_logp, const double *adv,
                             const double *v_old, const double *consts /* c1, c2, clip */,
                             const double *mask, double keep, double *loss, double *grad);
/* GAE by backward recursion: adv[T] from r[T], v[T+1]. */
WPK_API wpk_status wpk_gae(int32_t T, const double *r, const double *v, double gamma, double mu, double *adv);
/* Observation O_conv with the feature scaling of DESIGN.md reading c24b. */
WPK_API wpk_status wpk_observation(const wpk_conv2d_shape *shape, const int32_t *genes, double alpha_us, double *obs17);

#ifdef __cplusplus
}
#endif
#endif /* WPK_H */
