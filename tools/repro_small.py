"""Run one small conv (exact-integer inputs) under a given UMMA config and compare with the oracle;
a short command for compute-sanitizer.  usage: python tools/repro_small.py N C H W K R S stride pad dil dtype layout genes..."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch
import workloads
from workloads import ConvLayer
from paper_2008_04567_b200 import Conv2dPlan
from _util import to_layout, from_layout, oracle_full

v = sys.argv[1:]
n, c, h, w, k, r, s, st, pd, dl = [int(t) for t in v[:10]]
dtype, layout = v[10], v[11]
genes = [int(t) for t in v[12:19]]
L = ConvLayer("repro", n, c, h, w, k, r, s, st, pd, dl)
x, wt, b = workloads.generate(L, dtype, "int", seed=29)
ref = oracle_full(L, x, wt, b)
plan = Conv2dPlan(n, c, h, w, k, r, s, st, pd, dl, layout=layout, dtype=dtype)
plan.set_config(1, genes)
xl, wl = to_layout(x, wt, layout)
y = plan.run(xl.cuda(), wl.cuda(), b.cuda())
torch.cuda.synchronize()
got = from_layout(y.cpu(), layout).double()
bad = (got - torch.as_tensor(ref)).abs() > 0
print("mismatches", int(bad.sum()), "of", bad.numel())
