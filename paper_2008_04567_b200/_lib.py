"""ctypes binding of libwpk.so (include/wpk.h). Argument marshalling only.

The library is built in-tree by `__graft_entry__.build()` (nvcc, sm_100a). If it is missing this
module raises: there is no CPU or eager-PyTorch fallback for any operation of the hot path.
"""
from __future__ import annotations

import ctypes
import os
import re

_HERE = os.path.dirname(os.path.abspath(__file__))
# WPK_LIB: an alternative in-tree build of the same library (A/B experiments on one GPU box)
LIB_PATH = os.environ.get("WPK_LIB") or os.path.join(_HERE, "libwpk.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "wpk.h")

NUM_GENES = 7

# enums (wpk.h)
OK, ERR_INVALID_ARGUMENT, ERR_SHAPE, ERR_UNSUPPORTED, ERR_INVALID_CONFIG, ERR_EXHAUSTED, ERR_CUDA, \
    ERR_OUT_OF_MEMORY, ERR_INTERNAL = range(9)
STATUS_NAMES = ["OK", "INVALID_ARGUMENT", "SHAPE", "UNSUPPORTED", "INVALID_CONFIG", "EXHAUSTED", "CUDA",
                "OUT_OF_MEMORY", "INTERNAL"]
DTYPES = {"f32": 0, "tf32": 1, "bf16": 2, "f16": 3, "fp8": 4}   # fp8 = WPK_FP8E4M3
LAYOUTS = {"nchw": 0, "nhwc": 1}
EPILOGUES = {"none": 0, "bias": 1, "bias_relu": 2, "bias_add_relu": 3}
SEARCHES = {"ga": 0, "rl": 1, "random": 2}
EVAL_MODES = {"measured": 0, "replay": 1, "synthetic": 2}
FAMILIES = {"simt": 0, "umma": 1, "dw": 2, "gemm32": 3, "jit": 4, "auto": -1}


class WpkError(RuntimeError):
    def __init__(self, status: int, msg: str):
        self.status = status
        super().__init__(f"wpk error {STATUS_NAMES[status] if 0 <= status < 9 else status}: {msg}")


class Shape(ctypes.Structure):
    _fields_ = [("struct_size", ctypes.c_uint32)] + [(n, ctypes.c_int32) for n in (
        "n", "c", "h", "w", "k", "r", "s", "stride_h", "stride_w", "pad_h", "pad_w", "dil_h", "dil_w",
        "groups", "layout", "epilogue")]


EXCHANGE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p)


class TuneOptions(ctypes.Structure):
    _fields_ = [
        ("struct_size", ctypes.c_uint32),
        ("seed", ctypes.c_uint64),
        ("rank", ctypes.c_int32), ("world", ctypes.c_int32),
        ("exchange", EXCHANGE_FN), ("exchange_ctx", ctypes.c_void_p),
        ("warmup", ctypes.c_int32), ("reps", ctypes.c_int32),
        ("l2_flush", ctypes.c_int32), ("eval_mode", ctypes.c_int32), ("family", ctypes.c_int32),
        ("record_path", ctypes.c_char_p), ("replay_path", ctypes.c_char_p), ("log_path", ctypes.c_char_p),
        ("synthetic", ctypes.c_double * (1 + 2 * NUM_GENES)),
        ("ga_pop", ctypes.c_int32), ("ga_elites", ctypes.c_int32), ("ga_pool", ctypes.c_int32),
        ("ga_max_gen", ctypes.c_int32),
        ("ga_mutation", ctypes.c_double), ("ga_eps", ctypes.c_double),
        ("rl_envs", ctypes.c_int32), ("rl_horizon", ctypes.c_int32), ("rl_epochs", ctypes.c_int32),
        ("rl_minibatch", ctypes.c_int32),
        ("rl_gamma", ctypes.c_double), ("rl_mu", ctypes.c_double), ("rl_clip", ctypes.c_double),
        ("rl_c1", ctypes.c_double), ("rl_c2", ctypes.c_double), ("rl_lr", ctypes.c_double),
        ("rl_keep_prob", ctypes.c_double),
        ("rl_hidden", ctypes.c_int32 * 4),
        ("rl_alpha_mode", ctypes.c_int32),
        ("rl_adv_norm", ctypes.c_int32),
        ("rl_restart_every", ctypes.c_int32),
        ("max_seconds", ctypes.c_int32),
        ("seed_default", ctypes.c_int32),
        ("cache_dir", ctypes.c_char_p),
        ("finalists", ctypes.c_int32),
    ]


_lib = None


def load():
    """Load libwpk.so (raises if it was not built: no fallback path exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`. "
                           "There is no CPU fallback.")
    lib = ctypes.CDLL(LIB_PATH)
    P = ctypes.c_void_p
    I32, I32P = ctypes.c_int32, ctypes.POINTER(ctypes.c_int32)
    D, DP = ctypes.c_double, ctypes.POINTER(ctypes.c_double)
    sig = {
        "wpk_tune_options_init": (None, [ctypes.POINTER(TuneOptions)]),
        "wpk_conv2d_output_dims": (I32, [ctypes.POINTER(Shape), I32P, I32P]),
        "wpk_conv2d_plan": (I32, [ctypes.POINTER(Shape), I32, ctypes.c_int, ctypes.POINTER(P)]),
        "wpk_conv2d_tune": (I32, [P, I32, I32, ctypes.POINTER(TuneOptions)]),
        "wpk_conv2d_measure": (I32, [P, I32, I32, I32, DP]),
        "wpk_conv2d_run": (I32, [P, P, P, P, P, P]),
        "wpk_conv2d_run_residual": (I32, [P, P, P, P, P, P, P]),
        "wpk_dwpw_plan": (I32, [ctypes.POINTER(Shape), I32, I32, I32, ctypes.c_int, ctypes.POINTER(P)]),
        "wpk_dwpw_run": (I32, [P, P, P, P, P, P, P, P]),
        "wpk_conv2d_fold_batchnorm": (I32, [P, P, P, P, P, P, P, ctypes.c_float, P, P, P]),
        "wpk_conv2d_run_host": (I32, [P, P, P, P, P, P]),
        "wpk_conv2d_run_host_async": (I32, [P, P, P, P, P, P]),
        "wpk_conv2d_destroy": (None, [P]),
        "wpk_last_error": (ctypes.c_char_p, []),
        "wpk_conv2d_workspace_size": (I32, [P, ctypes.POINTER(ctypes.c_size_t)]),
        "wpk_conv2d_set_workspace": (I32, [P, P, ctypes.c_size_t]),
        "wpk_conv2d_get_config": (I32, [P, I32P, I32P]),
        "wpk_conv2d_set_config": (I32, [P, I32, I32P]),
        "wpk_conv2d_config_valid": (I32, [P, I32, I32P]),
        "wpk_conv2d_invalidate": (I32, [P]),
        "wpk_family_describe": (I32, [I32, I32P, I32P, ctypes.POINTER(ctypes.c_char_p)]),
        "wpk_conv2d_last_launch_count": (I32, [P]),
        "wpk_conv2d_tune_stats": (I32, [P, DP, I32P, I32P, DP]),
        "wpk_ppo_loss_grad": (I32, [I32P, DP, I32, DP, I32P, DP, DP, DP, DP, DP, D, DP, DP]),
        "wpk_gae": (I32, [I32, DP, DP, D, D, DP]),
        "wpk_observation": (I32, [ctypes.POINTER(Shape), I32P, D, DP]),
        "wpk_jit_compile": (I32, [P, I32P, ctypes.POINTER(ctypes.c_size_t)]),
        "wpk_jit_set_cache_dir": (I32, [ctypes.c_char_p]),
        "wpk_jit_stats": (I32, [ctypes.POINTER(ctypes.c_int64)] * 4 + [DP]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def last_error() -> str:
    return (load().wpk_last_error() or b"").decode(errors="replace")


def check(status: int):
    if status != OK:
        raise WpkError(status, last_error())


def header_symbols() -> list[str]:
    """Every function declared WPK_API in include/wpk.h."""
    txt = open(HEADER_PATH).read()
    return re.findall(r"^WPK_API[^(]*?\b(wpk_\w+)\s*\(", txt, flags=re.M)


def make_shape(n, c, h, w, k, r, s, stride=1, pad=0, dil=1, groups=1, layout="nchw", epilogue="bias_relu") -> Shape:
    sh, sw = (stride, stride) if isinstance(stride, int) else stride
    ph, pw = (pad, pad) if isinstance(pad, int) else pad
    dh, dw = (dil, dil) if isinstance(dil, int) else dil
    return Shape(ctypes.sizeof(Shape), n, c, h, w, k, r, s, sh, sw, ph, pw, dh, dw, groups,
                 LAYOUTS[layout], EPILOGUES[epilogue])


def family_describe(family: str | int):
    fam = FAMILIES[family] if isinstance(family, str) else family
    counts = (ctypes.c_int32 * NUM_GENES)()
    values = (ctypes.c_int32 * (NUM_GENES * 32))()
    names = (ctypes.c_char_p * NUM_GENES)()
    check(load().wpk_family_describe(fam, counts, values, names))
    doms = [[values[g * 32 + i] for i in range(counts[g])] for g in range(NUM_GENES)]
    return [n.decode() for n in names], doms


def jit_set_cache_dir(path: str | None):
    """On-disk cubin cache of the JIT family (None = memory only)."""
    check(load().wpk_jit_set_cache_dir(path.encode() if path else None))


def jit_stats() -> dict:
    """Process-wide JIT counters: NVRTC compiles, memory / disk cache hits, failures, compile seconds."""
    v = [ctypes.c_int64() for _ in range(4)]
    sec = ctypes.c_double()
    check(load().wpk_jit_stats(*[ctypes.byref(x) for x in v], ctypes.byref(sec)))
    return {"compiles": v[0].value, "mem_hits": v[1].value, "disk_hits": v[2].value, "failures": v[3].value,
            "compile_seconds": sec.value}
