"""JIT family (WPK_FAMILY_JIT, NEXT-2): the paper's Step2 "compile the generated codes just-in-time"
 with a compile cache. Host-only checks: NVRTC compiles the generated
kernel for sm_100a without a GPU, invalid genes are rejected, the in-memory and on-disk caches are
hit instead of recompiling."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _plan(*a, **k):
    from paper_2008_04567_b200 import Conv2dPlan
    k.setdefault("device", 0)
    return Conv2dPlan(*a, **k)


def test_jit_family_space_is_the_papers_gene_set():
    from paper_2008_04567_b200 import _lib as L
    names_simt, dom_simt = L.family_describe("simt")
    names_jit, dom_jit = L.family_describe("jit")
    assert names_jit == ["T_x", "T_y", "T_z", "Tile_x", "Tile_y", "Tile_z", "Tile_rz"] == names_simt
    assert dom_jit == dom_simt


@pytest.mark.parametrize("dtype", ["f32", "tf32", "bf16", "f16"])
@pytest.mark.parametrize("layout", ["nchw", "nhwc"])
def test_jit_compiles_every_dtype_layout(dtype, layout):
    p = _plan(2, 6, 9, 11, 10, 3, 3, 2, 1, dil=2, dtype=dtype, layout=layout)
    # Tile_rz 4 on a 16-bit dtype: not instantiated in the precompiled SIMT family, fine for JIT
    assert p.config_valid("jit", [8, 4, 2, 2, 1, 2, 4])
    assert p.jit_compile([8, 4, 2, 2, 1, 2, 4]) > 1000


def test_jit_grouped_and_residual_epilogue():
    p = _plan(1, 8, 6, 6, 8, 3, 3, 1, 1, groups=4, dtype="bf16", layout="nhwc")
    assert p.jit_compile([4, 4, 2, 1, 2, 1, 2]) > 1000
    q = _plan(1, 8, 6, 6, 8, 1, 1, 1, 0, dtype="f32", layout="nchw", epilogue="bias_add_relu")
    assert q.jit_compile([8, 8, 2, 1, 1, 1, 1]) > 1000


def test_jit_rejects_invalid_genes():
    from paper_2008_04567_b200 import _lib as L
    p = _plan(1, 4, 8, 8, 8, 3, 3, 1, 1, dtype="f32", layout="nchw")
    assert not p.config_valid("jit", [32, 32, 2, 1, 1, 1, 1])       # 2048 threads > 1024
    with pytest.raises(L.WpkError) as e:
        p.jit_compile([32, 32, 2, 1, 1, 1, 1])
    assert e.value.status == L.ERR_INVALID_CONFIG
    with pytest.raises(L.WpkError):
        p.jit_compile([3, 4, 4, 1, 1, 1, 1])                          # T_x = 3 not in its domain


def test_jit_memory_cache_hit():
    from paper_2008_04567_b200 import _lib as L
    p = _plan(1, 5, 7, 7, 6, 3, 3, 1, 1, dtype="f32", layout="nhwc")
    genes = [4, 4, 4, 1, 2, 1, 1]
    n1 = p.jit_compile(genes)
    s1 = L.jit_stats()
    assert p.jit_compile(genes) == n1
    s2 = L.jit_stats()
    assert s2["compiles"] == s1["compiles"] and s2["mem_hits"] == s1["mem_hits"] + 1


_CHILD = r"""
import sys, json
sys.path.insert(0, %r)
from paper_2008_04567_b200 import Conv2dPlan, _lib as L
p = Conv2dPlan(1, 3, 10, 10, 7, 5, 5, 1, 2, dtype="bf16", layout="nchw", device=0)
n = p.jit_compile([8, 8, 1, 1, 1, 1, 1])
print(json.dumps(dict(L.jit_stats(), bytes=n)))
"""


def test_jit_disk_cache_across_processes(tmp_path):
    """A second process with the same cache directory loads the cubin instead of compiling it."""
    import json
    env = dict(os.environ, WPK_JIT_CACHE_DIR=str(tmp_path))
    out = []
    for _ in range(2):
        r = subprocess.run([sys.executable, "-c", _CHILD % ROOT], env=env, capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr
        out.append(json.loads(r.stdout.strip().splitlines()[-1]))
    assert out[0]["compiles"] == 1 and out[0]["disk_hits"] == 0
    assert out[1]["compiles"] == 0 and out[1]["disk_hits"] == 1
    assert out[0]["bytes"] == out[1]["bytes"]
    assert len([f for f in os.listdir(tmp_path) if f.startswith("wpk_jit_")]) == 1
