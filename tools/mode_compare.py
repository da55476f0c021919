"""Adjoint vs primal throughput per config (device-resident Z, CUDA events)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_1708_02207_b200 as hb  # noqa: E402
from paper_1708_02207_b200 import configs  # noqa: E402

for name, B in [("C2", 1024), ("C3", 1024), ("C5", 128)]:
    cfg = configs.CONFIGS[name]
    Z = torch.from_numpy(configs.draw_Z(cfg, batch=max(B, cfg.batch))[:B].copy()).cuda()
    for mode in (0, 1):
        prob = configs.make_problem(name, mode=mode)
        hb.log_likelihood_batch(prob, Z)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            hb.log_likelihood_batch(prob, Z)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        print(f"{name} mode {mode}: {ms:.2f} ms per {B} -> {B / ms * 1e3:.0f} samples/s", flush=True)
        del prob
        torch.cuda.empty_cache()
