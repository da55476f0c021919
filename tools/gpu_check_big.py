"""GPU check of the larger configs against the reference goldens + direct solve."""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1708_02207_b200 as hb  # noqa: E402
from paper_1708_02207_b200 import configs  # noqa: E402


def main(names):
    import torch
    for name in names:
        g = np.load(ROOT / "tests" / "golden" / f"cfg_{name}.npz")
        t0 = time.time()
        prob = configs.make_problem(name)
        S = hb.forward_functionals_batch(prob, g["Z"])
        ll = hb.log_likelihood_batch(prob, g["Z"])
        err = max(np.max(np.abs(S[b] - g["S"][b])) / np.max(np.abs(g["S"][b])) for b in range(S.shape[0]))
        errl = np.max(np.abs(ll - g["ll"]) / np.abs(g["ll"]))
        info = prob.plan().info()
        print(f"{name}: S rel {err:.3e}  ll rel {errl:.3e}  (plan+run {time.time() - t0:.1f}s, bcap {info.max_batch},"
              f" ws {info.workspace_bytes / 2**30:.2f} GiB)", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["C3"])
