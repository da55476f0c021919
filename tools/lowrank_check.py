"""Low-rank (H-matrix) storage: error vs the dense path for several eps."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1708_02207_b200 as hb  # noqa: E402
from paper_1708_02207_b200 import configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 8
cfg = configs.CONFIGS[name]
Z = configs.draw_Z(cfg)[:B]
dense = configs.make_problem(name)
S0 = hb.forward_functionals_batch(dense, Z)
l0 = hb.log_likelihood_batch(dense, Z)
for eps in (1e-4, 1e-6, 1e-8):
    pr = configs.make_problem(name, compression=hb.ToleranceSpec(eps, 16, 32))
    S = hb.forward_functionals_batch(pr, Z)
    ll = hb.log_likelihood_batch(pr, Z)
    es = np.max(np.abs(S - S0)) / np.max(np.abs(S0))
    el = np.max(np.abs(ll - l0) / np.abs(l0))
    print(f"{name} eps {eps:.0e}: S rel err {es:.3e}  ll rel err {el:.3e}", flush=True)
