"""Throughput of every BASELINE config on one GPU (device-resident Z, CUDA events),
plus the low-rank C5 path and the full-solution sweep; one JSON line per case.

usage: python tools/config_sweep.py [--reps 3] > profiles/rNN_configs.jsonl

Batches are sized so each case runs in seconds (C3/C4/C5 use a prefix of their
BASELINE batch; throughput is per-sample work, batch-size independent once the
GPU is full).  Step roofline = algorithmic flops (bench.flops_split) / time.
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1708_02207_b200 as hb  # noqa: E402
from paper_1708_02207_b200 import configs  # noqa: E402

CASES = [("C1", 64, False, "forward"), ("C2", 1024, False, "forward"), ("C3", 1024, False, "forward"),
         ("C4", 1024, False, "forward"), ("C5", 512, False, "forward"), ("C5", 512, True, "forward"),
         ("C2", 1024, False, "solve")]


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    return float(np.median([a.elapsed_time(b) for a, b in ev]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--full", action="store_true",
                    help="the BASELINE batch of every config (C3 8192, C4 65536, C5 16384; sub-batched), 1 rep")
    args = ap.parse_args()
    cases = CASES
    if args.full:
        cases = [(n, configs.CONFIGS[n].batch, lr, "forward") for n, lr in
                 (("C1", False), ("C2", False), ("C3", False), ("C4", False), ("C5", False), ("C5", True))]
        args.reps = 1
    for name, B, lowrank, kind in cases:
        cfg = configs.CONFIGS[name]
        prob = configs.make_problem(name, compression=lowrank)
        Z = torch.from_numpy(configs.draw_Z(cfg, batch=max(B, 1))[:B].copy()).cuda()
        if kind == "forward":
            fn = lambda: hb.log_likelihood_batch(prob, Z)  # noqa: E731
        else:
            fn = lambda: hb.solve_batch(prob, Z)  # noqa: E731
        ms = timed(fn, args.reps)
        leaf_fl, merge_fl = bench.flops_split(cfg.level)
        fl = leaf_fl + sum(merge_fl.values())
        info = (prob.solve_plan() if kind == "solve" else prob.plan()).info()
        line = {"config": name, "case": kind + ("+lowrank" if lowrank else ""), "batch": B,
                "ms": ms, "samples_per_s": B / (ms * 1e-3),
                "step_tflops": fl * B / (ms * 1e-3) / 1e12,
                "frac_fp64": fl * B / (ms * 1e-3) / 1e12 / bench.FP64_PEAK_TFLOPS,
                "flops_per_sample": fl, "mode": int(info.mode), "sub_batch": int(info.max_batch)}
        print(json.dumps(line), flush=True)
        del prob
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
