"""Minimal driver for ncu captures: one warm forward + one profiled forward.
usage: python tools/prof_run.py CONFIG BATCH [lr]   (lr: the config's low-rank ToleranceSpec)"""
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import ctypes as C  # noqa: E402

import torch  # noqa: E402

from paper_1708_02207_b200 import _lib, configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 256
cfg = configs.CONFIGS[name]
lowrank = len(sys.argv) > 3 and sys.argv[3] == "lr"
prob = configs.make_problem(name, compression=lowrank)
plan = prob.plan()
info = plan.info()
Z = torch.from_numpy(configs.draw_Z(cfg, batch=max(B, cfg.batch))[:B].copy()).cuda()
ll = torch.empty(B, dtype=torch.float64, device="cuda")
ns = info.leaf_depth + 3
for it in range(2):
    st = np.zeros(ns)
    rc = plan.lib.hdd_forward_batch_timed(plan.handle, C.c_void_p(Z.data_ptr()), B, None,
                                          C.c_void_p(ll.data_ptr()), None, st.ctypes.data_as(_lib._f64p), ns)
    if not os.environ.get("HDD_PROF_IGNORE_ERR"):      # A/B builds with deliberately wrong numerics
        plan.check(rc)
torch.cuda.synchronize()
names = ["kappa", "leaf"] + [f"merge_d{d}" for d in range(info.leaf_depth - 1, -1, -1)] + ["finalize"]
print(name, B, {n: round(float(v), 3) for n, v in zip(names, st)}, "total", round(float(st.sum()), 3))
clk = (C.c_longlong * 64)()
plan.lib.hdd_debug_leaf_clocks(clk)
c = [int(v) for v in clk]
print("leaf CTA(0,0) clocks: base", c[1] - c[0])
for r in range(5, -1, -1):
    base = 10 + 8 * (5 - r)
    prev = c[1] if r == 5 else c[10 + 8 * (5 - (r + 1)) + 3]
    ph = [c[base + i] - (prev if i == 0 else c[base + i - 1]) for i in range(4)]
    print(f"  level {r}: A {ph[0]}  B {ph[1]} (chol {c[base + 4] - c[base]})  C {ph[2]}  D {ph[3]}")
print("  total", c[63] - c[0])

mc = (C.c_longlong * 256)()
plan.lib.hdd_debug_merge_clocks(mc)
print("merge CTA(0,0) phase cycles: maps / gather / eliminate / sigma+factors / Schur update")
for d in range(info.leaf_depth - 1, -1, -1):
    c = [int(mc[d * 8 + i]) for i in range(6)]
    if c[0] == 0:
        continue
    c67 = [int(mc[d * 8 + 6]), int(mc[d * 8 + 7])]
    fend = int(mc[(d + 16) * 8]) if d < 16 else 0
    extra = (f"   [tier M: first factor {c67[0] - c[2]} (warp 0 alone {fend - c[2]}), first row apply {c67[1] - c67[0]}]"
             if c67[0] > c[2] else "")
    print(f"  d{d}: " + "  ".join(str(c[i + 1] - c[i]) for i in range(5)) + f"   total {c[5] - c[0]}" + extra)
