"""Copy the synthetic experiment data (y, sigma) of C1-C5 from the golden
fixtures (made by the live reference, tests/golden/make_golden.py) into the
package data file paper_1708_02207_b200/data/protocol.npz."""
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
out = {}
for name in ["C1", "C2", "C3", "C4", "C5"]:
    with np.load(ROOT / "tests" / "golden" / f"cfg_{name}.npz") as d:
        out[f"{name}_y"] = d["y"]
        out[f"{name}_sigma"] = d["sigma"]
        out[f"{name}_obs_kind"] = d["obs_kind"]
        out[f"{name}_obs_id"] = d["obs_id"]
np.savez_compressed(ROOT / "paper_1708_02207_b200" / "data" / "protocol.npz", **out)
print("wrote protocol.npz")
