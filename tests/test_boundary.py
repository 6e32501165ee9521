"""C-ABI boundary tests that need no GPU: the library loads, exports every symbol include/wpk.h
declares, struct sizes agree with the C compiler's, and host-side validation maps bad shapes and
configs to the documented wpk_status codes."""
import ctypes
import os
import subprocess

import pytest

import oracle
import workloads
from paper_2008_04567_b200 import _lib as L
from paper_2008_04567_b200.conv import make_options

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    lib = L.load()
    names = L.header_symbols()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n
    out = subprocess.check_output(["nm", "-D", "--defined-only", L.LIB_PATH]).decode()
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    assert set(names) <= exported


def test_struct_sizes_match_c(tmp_path):
    src = tmp_path / "sz.c"
    src.write_text('#include <stdio.h>\n#include "wpk.h"\nint main(){printf("%zu %zu\\n", '
                   'sizeof(wpk_tune_options), sizeof(wpk_conv2d_shape));}\n')
    exe = tmp_path / "sz"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    a, b = map(int, subprocess.check_output([str(exe)]).split())
    assert (a, b) == (ctypes.sizeof(L.TuneOptions), ctypes.sizeof(L.Shape))


def _plan(shape, dtype="bf16"):
    lib = L.load()
    h = ctypes.c_void_p()
    st = lib.wpk_conv2d_plan(ctypes.byref(shape), L.DTYPES[dtype], 0, ctypes.byref(h))
    return st, h


@pytest.mark.parametrize("kw,status", [
    (dict(n=0), L.ERR_SHAPE), (dict(c=0), L.ERR_SHAPE), (dict(stride=0), L.ERR_SHAPE),
    (dict(h=1, pad=0), L.ERR_SHAPE),                                  # 3x3 on 1x1 -> empty output
    (dict(groups=2, c=3), L.ERR_SHAPE), (dict(groups=2, c=4, k=7), L.ERR_SHAPE),
    (dict(pad=-1), L.ERR_SHAPE),
])
def test_shape_validation(kw, status):
    base = dict(n=1, c=4, h=8, w=8, k=8, r=3, s=3, stride=1, pad=1, dil=1, groups=1)
    base.update(kw)
    shp = L.make_shape(**base)
    st, h = _plan(shp)
    assert st == status, L.last_error()
    assert L.last_error()


@pytest.mark.parametrize("dtype", ["f32", "tf32", "bf16", "f16"])
def test_general_groups_plan(dtype):
    """General grouped conv (1 < groups < C, NEXT-4): planned on the grouped (DW) family, with the
    output vector dividing K/groups; SIMT valid too; the GEMM families are kept out."""
    lib = L.load()
    shp = L.make_shape(2, 32, 9, 9, 48, 3, 3, 1, 1, groups=8, layout="nhwc")   # C/g = 4, K/g = 6
    st, h = _plan(shp, dtype)
    assert st == L.OK, L.last_error()
    fam, genes = ctypes.c_int32(), (ctypes.c_int32 * 7)()
    L.check(lib.wpk_conv2d_get_config(h, ctypes.byref(fam), genes))
    assert fam.value == L.FAMILIES["dw"] and 6 % genes[0] == 0
    assert lib.wpk_conv2d_config_valid(h, L.FAMILIES["dw"], (ctypes.c_int32 * 7)(4, 1, 256, 1, 0, 0, 0)) == 0
    assert lib.wpk_conv2d_config_valid(h, L.FAMILIES["simt"], (ctypes.c_int32 * 7)(16, 4, 4, 1, 1, 1, 1)) == 1
    umma = (ctypes.c_int32 * 7)(64, 4, 1, 0, 0, 2, 128)
    g32 = (ctypes.c_int32 * 7)(64, 64, 8, 4, 1, 0, 0)
    assert lib.wpk_conv2d_config_valid(h, L.FAMILIES["umma"], umma) == 0
    assert lib.wpk_conv2d_config_valid(h, L.FAMILIES["gemm32"], g32) == 0
    lib.wpk_conv2d_destroy(h)


def test_bad_struct_size_and_null():
    lib = L.load()
    shp = L.make_shape(1, 4, 8, 8, 8, 3, 3, 1, 1)
    shp.struct_size = 4
    st, _ = _plan(shp)
    assert st == L.ERR_INVALID_ARGUMENT
    assert lib.wpk_conv2d_plan(None, 0, 0, ctypes.byref(ctypes.c_void_p())) == L.ERR_INVALID_ARGUMENT
    assert lib.wpk_conv2d_run(None, None, None, None, None, None) == L.ERR_INVALID_ARGUMENT


@pytest.mark.parametrize("layer", workloads.resnet50(32) + workloads.vgg16(64) + workloads.mobilenet_v2(1)
                         + workloads.table1() + [workloads.CONFIG1], ids=lambda l: l.name)
def test_output_dims_and_default_plan(oracle_lib, layer):
    from paper_2008_04567_b200 import output_dims
    pq = output_dims(layer.n, layer.c, layer.h, layer.w, layer.k, layer.r, layer.s, layer.stride, layer.pad,
                     layer.dil, layer.groups)
    assert pq == oracle.out_dims(layer.n, layer.c, layer.h, layer.w, layer.k, layer.r, layer.s, layer.stride,
                                 layer.pad, layer.dil, layer.groups)
    for dtype in ("f32", "tf32", "bf16", "f16"):
        shp = L.make_shape(layer.n, layer.c, layer.h, layer.w, layer.k, layer.r, layer.s, layer.stride, layer.pad,
                           layer.dil, layer.groups, "nhwc")
        st, h = _plan(shp, dtype)
        assert st == L.OK, L.last_error()
        lib = L.load()
        fam, genes = ctypes.c_int32(), (ctypes.c_int32 * 7)()
        L.check(lib.wpk_conv2d_get_config(h, ctypes.byref(fam), genes))
        if layer.groups > 1:
            assert fam.value == L.FAMILIES["dw"]
        elif dtype == "f32":
            assert fam.value == L.FAMILIES["gemm32"]
        else:
            assert fam.value == L.FAMILIES["umma"]
        assert lib.wpk_conv2d_config_valid(h, fam, genes) == 1
        lib.wpk_conv2d_destroy(h)


def test_set_config_validation():
    lib = L.load()
    shp = L.make_shape(1, 64, 56, 56, 64, 3, 3, 1, 1, layout="nhwc")
    st, h = _plan(shp, "f32")
    assert st == 0
    bad = (ctypes.c_int32 * 7)(32, 32, 2, 1, 1, 1, 1)         # 2048 threads > 1024
    assert lib.wpk_conv2d_set_config(h, 0, bad) == L.ERR_INVALID_CONFIG
    assert "1024" in L.last_error()
    ok = (ctypes.c_int32 * 7)(16, 8, 4, 1, 1, 1, 1)
    assert lib.wpk_conv2d_set_config(h, 0, ok) == L.OK
    notin = (ctypes.c_int32 * 7)(7, 8, 4, 1, 1, 1, 1)
    assert lib.wpk_conv2d_set_config(h, 0, notin) == L.ERR_INVALID_CONFIG
    # f32 cannot use the tensor-core family
    umma = (ctypes.c_int32 * 7)(64, 4, 1, 0, 0, 2, 128)
    assert lib.wpk_conv2d_set_config(h, 1, umma) == L.ERR_INVALID_CONFIG
    g32 = (ctypes.c_int32 * 7)(128, 64, 16, 4, 2, 0, 0)
    assert lib.wpk_conv2d_set_config(h, 3, g32) == L.OK
    g32_bad = (ctypes.c_int32 * 7)(128, 64, 16, 2, 1, 0, 0)   # THREAD_TILE 2 not in {4, 8}
    assert lib.wpk_conv2d_set_config(h, 3, g32_bad) == L.ERR_INVALID_CONFIG
    lib.wpk_conv2d_destroy(h)
    st, h = _plan(shp, "bf16")
    assert lib.wpk_conv2d_set_config(h, 3, g32) == L.ERR_INVALID_CONFIG   # GEMM32 is f32-only
    too_deep = (ctypes.c_int32 * 7)(256, 8, 1, 0, 0, 2, 128)   # 8 x 48 KB stages > 227 KB
    assert lib.wpk_conv2d_set_config(h, 1, too_deep) == L.ERR_INVALID_CONFIG
    assert lib.wpk_conv2d_set_config(h, 1, umma) == L.OK
    lib.wpk_conv2d_destroy(h)


def test_family_describe_matches_paper_genes():
    names, doms = L.family_describe("simt")
    assert names == ["T_x", "T_y", "T_z", "Tile_x", "Tile_y", "Tile_z", "Tile_rz"]
    names, doms = L.family_describe("umma")
    assert names[0] == "BLOCK_N" and 128 in doms[0]
    names, doms = L.family_describe("gemm32")
    assert names[:5] == ["BLOCK_M", "BLOCK_N", "BLOCK_K", "THREAD_TILE", "SPLIT_K"] and doms[3] == [4, 8]


def test_options_defaults():
    o = make_options()
    assert (o.warmup, o.reps, o.world, o.ga_pop, o.ga_elites) == (3, 11, 1, 48, 4)
    assert (o.rl_c1, o.rl_c2) == (0.15, 20.0)
    assert list(o.rl_hidden) == [512, 1024, 1024, 512]


def test_residual_epilogue_host_validation():
    """WPK_EPI_BIAS_ADD_RELU: split-K configs are invalid; the plain run entry point and the
    host-buffer call refuse a residual plan before touching the device."""
    from paper_2008_04567_b200 import Conv2dPlan
    plan = Conv2dPlan(2, 64, 8, 8, 128, 3, 3, 1, 1, layout="nhwc", epilogue="bias_add_relu", dtype="bf16", device=0)
    assert plan.config_valid(1, [128, 4, 1, 0, 0, 2, 128])
    assert not plan.config_valid(1, [128, 4, 2, 0, 0, 2, 128])
    lib = L.load()
    fake = ctypes.c_void_p(0x1000)
    assert lib.wpk_conv2d_run(plan.handle, fake, fake, fake, fake, None) == 1          # WPK_ERR_INVALID_ARGUMENT
    assert lib.wpk_conv2d_run_residual(plan.handle, fake, fake, fake, None, fake, None) == 1
    assert lib.wpk_conv2d_run_host(plan.handle, fake, fake, fake, fake, None) == 1


def test_missing_library_fails_loudly(tmp_path):
    """No CPU or eager fallback: with the shared library absent the binding raises on first use
    (checked in a fresh interpreter pointing WPK_LIB at a path that does not exist)."""
    import subprocess
    import sys
    env = dict(os.environ, WPK_LIB=str(tmp_path / "absent" / "libwpk.so"))
    code = ("import paper_2008_04567_b200._lib as L\n"
            "try:\n    L.load()\nexcept RuntimeError as e:\n    print('RAISED', 'no CPU fallback' in str(e))\n")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                         cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))), timeout=120)
    assert "RAISED True" in out.stdout, out.stdout + out.stderr


def test_fp8_plans_host_validation():
    """WPK_FP8E4M3 (e4m3 x / w, bf16 y): tcgen05 family only, TMA A producers only (no GPU needed:
    plan + config validation are host logic)."""
    lib = L.load()
    st, h = _plan(L.make_shape(n=2, c=192, h=11, w=13, k=200, r=3, s=3, stride=1, pad=1, layout="nhwc"), dtype="fp8")
    assert st == 0
    fam, g = ctypes.c_int32(), (ctypes.c_int32 * L.NUM_GENES)()
    assert lib.wpk_conv2d_get_config(h, ctypes.byref(fam), g) == 0
    assert fam.value == 1 and g[4] in (0, 4)            # tcgen05, TMA A producer
    for am in (1, 2, 3):                                # gather / explicit im2col: not instantiated for e4m3
        genes = (ctypes.c_int32 * L.NUM_GENES)(128, 4, 1, 0, am, 2, 128)
        assert lib.wpk_conv2d_config_valid(h, 1, genes) == 0
    for fam_id, genes in ((0, (16, 4, 4, 1, 1, 1, 1)), (3, (64, 64, 16, 4, 1, 0, 0)), (4, (16, 4, 4, 1, 1, 1, 1))):
        assert lib.wpk_conv2d_config_valid(h, fam_id, (ctypes.c_int32 * L.NUM_GENES)(*genes)) == 0
    assert b"FP8" in lib.wpk_last_error()
    lib.wpk_conv2d_destroy(h)
    st, h = _plan(L.make_shape(n=1, c=32, h=8, w=8, k=32, r=3, s=3, stride=1, pad=1, groups=32, layout="nhwc"),
                  dtype="fp8")
    assert st == L.ERR_UNSUPPORTED
    assert b"groups" in lib.wpk_last_error() or b"depthwise" in lib.wpk_last_error()


def test_dwpw_plan_host_validation():
    """wpk_dwpw_plan (fused depthwise + pointwise): shape / layout / dtype / channel checks, the
    default config (tcgen05, A_MODE 0 = the depthwise producer, no pairs) and the run-entry guards
    (host logic: no GPU needed)."""
    lib = L.load()

    def plan(c=144, k=24, groups=None, layout="nhwc", dtype="bf16", epi="bias_relu", pw=1):
        shp = L.make_shape(n=1, c=c, h=14, w=14, k=c, r=3, s=3, stride=1, pad=1,
                           groups=c if groups is None else groups, layout=layout, epilogue=epi)
        h = ctypes.c_void_p()
        return lib.wpk_dwpw_plan(ctypes.byref(shp), k, pw, L.DTYPES[dtype], 0, ctypes.byref(h)), h

    st, h = plan()
    assert st == 0, L.last_error()
    fam, g = ctypes.c_int32(), (ctypes.c_int32 * L.NUM_GENES)()
    assert lib.wpk_conv2d_get_config(h, ctypes.byref(fam), g) == 0
    assert fam.value == 1 and g[4] in (0, 1) and (g[3] >> 1) & 3 == 0   # 1: the one-tile-per-CTA kernel
    assert lib.wpk_conv2d_config_valid(h, 1, (ctypes.c_int32 * L.NUM_GENES)(32, 2, 1, 0, 1, 1, 128)) == 1
    assert lib.wpk_conv2d_config_valid(h, 1, (ctypes.c_int32 * L.NUM_GENES)(32, 4, 1, 0, 1, 1, 128)) == 0   # canonical only
    assert lib.wpk_conv2d_config_valid(h, 1, (ctypes.c_int32 * L.NUM_GENES)(64, 4, 2, 1, 0, 2, 256)) == 1
    assert lib.wpk_conv2d_config_valid(h, 1, (ctypes.c_int32 * L.NUM_GENES)(64, 4, 1, 2, 0, 2, 256)) == 0   # pair
    assert lib.wpk_conv2d_config_valid(h, 1, (ctypes.c_int32 * L.NUM_GENES)(64, 4, 1, 0, 4, 2, 128)) == 0   # A_MODE 4
    assert lib.wpk_conv2d_config_valid(h, 0, (ctypes.c_int32 * L.NUM_GENES)(16, 4, 4, 1, 1, 1, 1)) == 0     # SIMT
    # the plain run entry points refuse a fused plan (before touching any pointer)
    assert lib.wpk_conv2d_run(h, 16, 16, 16, 16, None) == L.ERR_INVALID_ARGUMENT
    assert b"wpk_dwpw_run" in lib.wpk_last_error()
    lib.wpk_conv2d_destroy(h)
    assert plan(groups=1)[0] == L.ERR_SHAPE                      # first conv not depthwise
    assert plan(k=0)[0] == L.ERR_SHAPE
    assert plan(c=12)[0] == L.ERR_UNSUPPORTED                    # C % 8
    assert plan(layout="nchw")[0] == L.ERR_UNSUPPORTED
    assert plan(dtype="f32")[0] == L.ERR_UNSUPPORTED
    assert plan(dtype="fp8")[0] == L.ERR_UNSUPPORTED
    assert plan(epi="bias_add_relu")[0] == L.ERR_UNSUPPORTED
    assert plan(pw=3)[0] == L.ERR_INVALID_ARGUMENT               # residual pointwise epilogue
    # a plain conv plan refuses the fused run entry point
    st, h = _plan(L.make_shape(n=1, c=16, h=8, w=8, k=16, r=3, s=3, stride=1, pad=1, layout="nhwc"))
    assert st == 0
    assert lib.wpk_dwpw_run(h, 16, 16, 16, 16, 16, 16, None) == L.ERR_INVALID_ARGUMENT
    lib.wpk_conv2d_destroy(h)


def test_grouped_tensor_core_configs_host_validation():
    """1 < groups < C on the tcgen05 family (gconv_tc.cu): only {BLOCK_N, 2, 1, 0, 1, 1, 128} with
    BLOCK_N a multiple of the per-group MMA width max(16, K/g rounded to 16) and at most `groups`
    groups per tile; NHWC 16-bit only, C/g % 4 == 0; depthwise stays on the DW family."""
    lib = L.load()

    def plan(c, k, g, layout="nhwc", dtype="bf16"):
        st, h = _plan(L.make_shape(n=2, c=c, h=14, w=14, k=k, r=3, s=3, stride=1, pad=1, groups=g, layout=layout),
                      dtype=dtype)
        assert st == 0, L.last_error()
        return h

    def ok(h, bn, rest=(2, 1, 0, 1, 1, 128)):
        return lib.wpk_conv2d_config_valid(h, 1, (ctypes.c_int32 * L.NUM_GENES)(bn, *rest)) == 1

    h = plan(128, 128, 32)                      # K/g = 4 -> Np 16: 1..16 groups per tile
    assert [bn for bn in (16, 32, 64, 96, 128, 192, 256) if ok(h, bn)] == [16, 32, 64, 96, 128, 192, 256]
    assert not ok(h, 64, (4, 1, 0, 1, 1, 128)) and not ok(h, 64, (2, 2, 0, 1, 1, 128))
    assert not ok(h, 64, (2, 1, 0, 0, 2, 128))   # A_MODE 0 (TMA im2col) has no grouped variant
    lib.wpk_conv2d_destroy(h)
    h = plan(1024, 1024, 32)                    # K/g = 32 -> Np 32
    assert not ok(h, 16) and ok(h, 32) and ok(h, 256) and not ok(h, 96 + 16)
    lib.wpk_conv2d_destroy(h)
    h = plan(32, 48, 4)                         # 4 groups: at most 4 x 16 columns
    assert ok(h, 64) and not ok(h, 96)
    lib.wpk_conv2d_destroy(h)
    for kw in (dict(layout="nchw"), dict(dtype="f32"), dict(dtype="tf32")):
        h = plan(128, 128, 32, **kw)
        assert not ok(h, 64)
        lib.wpk_conv2d_destroy(h)
    h = plan(24, 24, 4)                          # C/g = 6
    assert not ok(h, 16) and b"% 4" in lib.wpk_last_error()
    lib.wpk_conv2d_destroy(h)
    h = plan(32, 32, 32)                         # depthwise
    assert not ok(h, 16) and b"depthwise" in lib.wpk_last_error()
    lib.wpk_conv2d_destroy(h)


def test_dwpw_plan_refuses_batchnorm_fold():
    lib = L.load()
    shp = L.make_shape(n=1, c=144, h=14, w=14, k=144, r=3, s=3, stride=1, pad=1, groups=144, layout="nhwc")
    h = ctypes.c_void_p()
    assert lib.wpk_dwpw_plan(ctypes.byref(shp), 24, 1, L.DTYPES["bf16"], 0, ctypes.byref(h)) == 0
    f = ctypes.c_void_p(16)
    st = lib.wpk_conv2d_fold_batchnorm(h, f, None, f, f, f, f, ctypes.c_float(1e-5), f, f, None)
    assert st == L.ERR_UNSUPPORTED and b"fused" in lib.wpk_last_error()
    lib.wpk_conv2d_destroy(h)
