"""Benchmark of the batched HDD likelihood (one JSON line on rank 0).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl ours|reference]

Workload (default C4, the BASELINE flagship): the 513x513-node problem, n_z = 32, 16
subdomain means, the FIXED global batch of 65,536 Z rows sharded over the N GPUs
(strong scaling: rank r evaluates rows parallel.shard_rows(65536, N, r)).  A step =
one batched likelihood evaluation of every rank's rows, the NCCL all-gather of the
log-likelihoods and the global posterior weights / argmax.

* value      samples/s of the whole job (65,536 / the max-over-ranks step time), Z
             resident in HBM, CUDA events around each step on the launching stream,
             L2 flushed (256 MiB memset) between steps;
* e2e        the same through the public API with HOST buffers (pinned numpy Z ->
             log_likelihood_batch -> hdd_forward_batch_host: H2D of Z, D2H of ll
             inside every timed step; sub-batch copies overlap compute);
* roofline   the dominant kernel stage (largest share of the step, CUDA events per
             stage over a timed pass): algorithmic FP64 flops (DESIGN.md "flop
             accounting") / its time, against the measured FP64 DGEMM peak; `traffic`
             comes from a committed ncu --set full capture of the same config and
             stage (profiles/traffic.json) or is null;
* per_config the other BASELINE configs on this GPU (C1, C2, C3 whole batches; C5 dense
             and low-rank on bounded prefixes), CUDA-event timed;
* cpu_baseline  the reference's CPU path on the host cores (rank 0, N = 1): the
             installed reference `hddsolve` under baseline/_ref (C1-C3: its HDD
             likelihood `bayes.log_likelihood`; C4/C5: its `oracle.direct_solve`,
             the only reference path that reaches levels 9/10 in seconds — its HDD caps
             the mesh at level 8), one forked worker per core x 1 BLAS thread; the
             oracle port when baseline/_ref is absent.
`--impl reference` times that CPU path as the reference arm.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

FP64_PEAK_TFLOPS = 35.46       # cuBLAS DGEMM 8192^3 sustained, profiles/fp64_peaks_r01.jsonl
FP64_PEAK_SRC = "measured cuBLAS DGEMM sustained on this pool's B200 (profiles/fp64_peaks_r01.jsonl)"
REF_DIR = ROOT / "baseline" / "_ref"


def hbm_peak():
    try:
        with open(ROOT / "MEASURED_PEAKS.json") as f:
            return float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


# --------------------------------------------------------------------------
# algorithmic flop model: sum over every node of the full
# reference tree of ng^3/3 + ng^2 (k+1) + k^2 ng + 2 k ng, k = pruned boundary
# --------------------------------------------------------------------------
def _split(r, depth):
    i0, i1, j0, j1 = r
    axis = depth % 2
    if axis == 0 and i1 - i0 == 1:
        axis = 1
    elif axis == 1 and j1 - j0 == 1:
        axis = 0
    if axis == 0:
        mid = (i0 + i1) // 2
        return (i0, mid, j0, j1), (mid, i1, j0, j1), axis
    mid = (j0 + j1) // 2
    return (i0, i1, j0, mid), (i0, i1, mid, j1), axis


def node_flops(r, depth, N):
    i0, i1, j0, j1 = r
    if i1 - i0 == 1 and j1 - j0 == 1:
        return 0.0
    _, _, axis = _split(r, depth)
    ng = (j1 - j0 - 1) if axis == 0 else (i1 - i0 - 1)
    # pruned perimeter: nodes not on the domain boundary
    k = 0
    xs = range(max(i0, 1), min(i1, N - 1) + 1)
    ys = range(max(j0 + 1, 1), min(j1 - 1, N - 1) + 1)
    for j in (j0, j1):
        if 0 < j < N:
            k += len(xs)
    for i in (i0, i1):
        if 0 < i < N:
            k += len(ys)
    return ng ** 3 / 3 + ng * ng * (k + 1) + k * k * ng + 2 * k * ng


def flops_split(level):
    """(leaf-kernel flops, merge flops per depth) per sample, 16x16 leaves."""
    N = 1 << level
    dl = max(0, 2 * (level - 4))
    leaf = 0.0
    merge = {}

    def rec(r, d):
        nonlocal leaf
        f = node_flops(r, d, N)
        if d >= dl:
            leaf += f
        else:
            merge[d] = merge.get(d, 0.0) + f
        if r[1] - r[0] == 1 and r[3] - r[2] == 1:
            return
        a, b, _ = _split(r, d)
        rec(a, d + 1)
        rec(b, d + 1)

    rec((0, N, 0, N), 0)
    return leaf, merge


# --------------------------------------------------------------------------
class ClockSampler:
    def __init__(self, dev_index):
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(dev_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_power_brake": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                try:
                    mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                except AttributeError:
                    mask = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for n, bit in names.items():
                    if mask & bit:
                        self.reasons.add(n)
            except Exception:
                pass
            self._stop.wait(0.05)

    def __enter__(self):
        if self.nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t is not None:
            self._t.join()

    def summary(self):
        med = float(np.median(self.samples)) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "n_samples": len(self.samples)}


# --------------------------------------------------------------------------
# the reference's CPU path (reported baseline and the --impl reference arm)
# --------------------------------------------------------------------------
_CPU = {}


def _cpu_setup(cfg_name):
    """Build (once, before forking) the CPU evaluator of one config.  Returns a
    description of the path."""
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    from paper_1708_02207_b200 import configs
    cfg = configs.CONFIGS[cfg_name]
    obs = configs.observations(cfg)
    y, sigma = configs.observed_data(cfg)
    _CPU.update(cfg=cfg, obs=obs, y=y, sigma=sigma)
    if (REF_DIR / "hddsolve").is_dir():
        sys.path.insert(0, str(REF_DIR))
        import hddsolve as hs
        from hddsolve import bayes as rb, oracle as ro
        from oracle import fields, geometry
        if cfg.level > hs.mesh.MAX_LEVEL:
            hs.mesh.MAX_LEVEL = cfg.level          # the reference caps the mesh at level 8
        mesh = hs.build_mesh(cfg.level)
        fo = fields.SineKLField(geometry.Grid(cfg.level), cfg.n_z)

        class KL:                                    # duck-typed param (bayes.py:183)
            n_z = cfg.n_z

            def kappa(self, z):
                return hs.CoefficientField(fo.kappa_values(z))

        if cfg.level <= 8:
            tree = hs.build_tree(mesh)
            model = rb.MeasurementModel(obs, sigma, y)
            prob = rb.BayesProblem(tree, KL(), np.ones(mesh.n_nodes), np.zeros(4 * (mesh.m - 1)), model)
            _CPU["fn"] = lambda z: rb.log_likelihood(prob, z)
            return "reference", "hddsolve.bayes.log_likelihood (reference HDD functional path, baseline/_ref)"
        param = KL()
        rects = {}
        from oracle.geometry import rect_of_node_id
        for kind, ident in obs:
            if kind == "mean":
                r, _ = rect_of_node_id(cfg.level, ident)
                h = mesh.h
                rects[ident] = hs.Rect(r[0] * h, r[1] * h, r[2] * h, r[3] * h)
        f1, g0 = np.ones(mesh.n_nodes), np.zeros(4 * (mesh.m - 1))

        def fn(z):
            u = ro.direct_solve(mesh, param.kappa(z), f1, g0)
            s = np.array([ro.direct_mean(mesh, u, rects[i]) if k == "mean" else u[i] for k, i in obs])
            return rb.gaussian_log_likelihood(y, s, sigma)

        _CPU["fn"] = fn
        return "reference", ("hddsolve.oracle.direct_solve + direct_mean (baseline/_ref; the reference HDD caps the "
                             f"mesh at level 8 — MAX_LEVEL raised to {cfg.level} at run time — and takes ~136 s per "
                             "level-9 sample, so its sparse-LU truth path is the fastest reference CPU path here)")
    from oracle import direct, fields, geometry, hdd_port
    grid = geometry.Grid(cfg.level)
    fo = fields.SineKLField(grid, cfg.n_z)
    if cfg.level <= 8:
        port = hdd_port.HDDPort(cfg.level, obs)
        _CPU["fn"] = lambda z: hdd_port.gaussian_ll(y, port.forward(fo.kappa_values(z)), sigma)
        return "port", "oracle/hdd_port.py (restatement of the reference HDD functional path)"
    from oracle import configs as ocfg

    def fn(z):
        return hdd_port.gaussian_ll(y, ocfg.observe(grid, direct.solve(grid, fo.kappa_values(z)), obs), sigma)

    _CPU["fn"] = fn
    return "port", "oracle/direct.py (restatement of reference oracle.direct_solve)"


def _cpu_worker(Z):
    from threadpoolctl import threadpool_limits
    threadpool_limits(1)
    return [float(_CPU["fn"](z)) for z in Z]


def time_cpu(Z, n_workers):
    """(samples/s, wall s, ll) of the prepared CPU path on the rows of Z."""
    import multiprocessing as mp
    chunks = [c for c in np.array_split(np.arange(Z.shape[0]), n_workers) if len(c)]
    t0 = time.time()
    with mp.get_context("fork").Pool(len(chunks)) as pool:
        res = pool.map(_cpu_worker, [Z[c] for c in chunks])
    wall = time.time() - t0
    return Z.shape[0] / wall, wall, np.concatenate([np.array(r) for r in res])


def cpu_rows_per_step(cfg_name, cores):
    return {"C1": 64, "C2": cores, "C3": cores}.get(cfg_name, cores)


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cores = len(os.sched_getaffinity(0))
    from paper_1708_02207_b200 import configs
    cfg = configs.CONFIGS[args.config]
    kind, path = _cpu_setup(args.config)
    per_step = cpu_rows_per_step(args.config, cores)
    Zall = configs.draw_Z(cfg)
    rows = lambda i: Zall[(i * per_step + np.arange(per_step)) % Zall.shape[0]]  # noqa: E731
    for w in range(args.warmup):
        time_cpu(rows(w), min(per_step, cores))
    t_all = 0.0
    for s in range(args.steps):
        _, wall, _ = time_cpu(rows(args.warmup + s), min(per_step, cores))
        t_all += wall
    value = args.steps * per_step / t_all
    line = {
        "impl": "reference", "metric": f"likelihood evals/s ({args.config}, {cfg.level}-level grid, n_z={cfg.n_z})",
        "value": value, "unit": "samples/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * t_all / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded protocol, DESIGN.md)",
        "config": {"workload": args.config, "global_batch": cfg.batch, "batch_per_step": per_step,
                   "grid_nodes": (1 << cfg.level) + 1, "n_z": cfg.n_z, "n_obs": len(configs.observations(cfg)),
                   "parallelism": "host cores (one forked worker per core, rank 0 only)"},
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": min(per_step, cores), "kind": kind,
                         "sample": f"{per_step} distinct Z rows of {args.config} per step, forked workers x 1 BLAS "
                                   f"thread: {path}"},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------
def traffic_from_capture(cfg_name, stage, samples_per_launch):
    """DRAM bytes (read + write) per launch of `stage`: the per-sample figure of a
    committed ncu --set full capture of the same config and kernel
    (profiles/traffic.json) times the samples of one launch, or None."""
    try:
        with open(ROOT / "profiles" / "traffic.json") as f:
            rec = json.load(f).get(cfg_name, {}).get(stage)
    except Exception:
        return None
    if not rec:
        return None
    return {"bytes_per_launch": rec["dram_bytes_per_sample"] * samples_per_launch,
            "samples_per_launch": samples_per_launch, "source": rec["source"], "binding": rec.get("binding")}


def per_config_measurements(dev):
    """Samples/s of the other BASELINE configs on this GPU (device-resident Z,
    CUDA events, median of 3 after one warm-up)."""
    import torch
    import paper_1708_02207_b200 as hb
    from paper_1708_02207_b200 import configs
    cases = [("C1", 64, False), ("C2", 1024, False), ("C3", 8192, False), ("C5", 1088, False), ("C5", 544, True)]
    out = {}
    for name, B, lowrank in cases:
        cfg = configs.CONFIGS[name]
        prob = configs.make_problem(name, device=dev.index, compression=lowrank)
        Z = torch.from_numpy(configs.draw_Z(cfg, batch=max(B, cfg.batch))[:B].copy()).to(dev)
        hb.log_likelihood_batch(prob, Z)
        torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            hb.log_likelihood_batch(prob, Z, sync=False)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        from paper_1708_02207_b200.bayes import synchronize
        synchronize(prob)
        ms = float(np.median(ts))
        leaf_fl, merge_fl = flops_split(cfg.level)
        fl = leaf_fl + sum(merge_fl.values())
        key = name + ("_lowrank" if lowrank else "")
        out[key] = {"samples_per_s": B / (ms * 1e-3), "batch": B, "ms": ms,
                    "batch_note": "whole BASELINE batch" if B == cfg.batch else f"first {B} rows of {cfg.batch}",
                    "step_fp64_frac": fl * B / (ms * 1e-3) / 1e12 / FP64_PEAK_TFLOPS,
                    "compression": list(cfg.compression) if lowrank else None}
        prob._plan = None
        del prob, Z
        import gc
        gc.collect()
        torch.cuda.empty_cache()
    return out


def main_rank(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)

    import ctypes as C
    from paper_1708_02207_b200 import _lib, bayes, configs
    from paper_1708_02207_b200.parallel import gather_ragged, posterior_weights_device, shard_rows

    cfg = configs.CONFIGS[args.config]
    G = cfg.batch if args.batch <= 0 else args.batch          # fixed global batch (strong scaling)
    lo, hi = shard_rows(G, world, rank)
    B = hi - lo
    counts = [shard_rows(G, world, r)[1] - shard_rows(G, world, r)[0] for r in range(world)]
    problem = configs.make_problem(args.config, device=local)
    plan = problem.plan()
    info = plan.info()
    Zall = configs.draw_Z(cfg, batch=max(G, cfg.batch))[:G]
    Zl = np.ascontiguousarray(Zall[lo:hi])
    Zd = torch.from_numpy(Zl).to(dev)
    ll = torch.empty(B, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)
    n_stages = info.leaf_depth + 3
    stage = np.zeros(n_stages)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def step():
        plan.check(plan.lib.hdd_forward_batch(plan.handle, C.c_void_p(Zd.data_ptr()), B, None,
                                              C.c_void_p(ll.data_ptr()), C.c_void_p(stream.cuda_stream)))
        ll_all = gather_ragged(ll, counts) if world > 1 else ll
        return posterior_weights_device(ll_all)

    for _ in range(args.warmup):
        step()
    plan.check(plan.lib.hdd_sync(plan.handle, C.c_void_p(stream.cuda_stream)))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.zero_()
            ev[i][0].record(stream)
            w, idx_t, lse_t = step()
            ev[i][1].record(stream)
        torch.cuda.synchronize()
    plan.check(plan.lib.hdd_sync(plan.handle, C.c_void_p(stream.cuda_stream)))
    if world > 1:
        dist.barrier()
    idx, lse, n_w = int(idx_t.item()), float(lse_t.item()), int(w.numel())
    ms = float(np.mean([a.elapsed_time(b) for a, b in ev]))
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = G / (ms_max * 1e-3)

    # per-stage (kernel) times: one timed pass over the first two sub-batches (per-sample
    # stage cost does not depend on the batch once a sub-batch fills the GPU), same
    # stream, CUDA events between launches; stage_ms is scaled to the whole step
    flush.zero_()
    B_st = min(B, 2 * info.max_batch)
    plan.check(plan.lib.hdd_forward_batch_timed(plan.handle, C.c_void_p(Zd.data_ptr()), B_st, None,
                                                C.c_void_p(ll.data_ptr()), C.c_void_p(stream.cuda_stream),
                                                stage.ctypes.data_as(_lib._f64p), n_stages))
    stage *= B / B_st

    # ---- e2e through the public API: pinned host Z -> device -> ll -> host ----
    Zh = torch.from_numpy(Zl).pin_memory()
    Zh_np = Zh.numpy()
    n_e2e = 2
    e2e_ms = []
    if world > 1:
        dist.barrier()
    for _ in range(n_e2e):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = bayes.log_likelihood_batch(problem, Zh_np)      # hdd_forward_batch_host: H2D, compute, D2H
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
    assert np.array_equal(out, ll.cpu().numpy())              # same numbers as the device-resident path
    t = torch.tensor([float(np.mean(e2e_ms))], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_max = float(t.item())

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel stage ----
    leaf_fl, merge_fl = flops_split(cfg.level)
    dl = info.leaf_depth
    names = ["kappa", "leaf"] + [f"merge_d{d}" for d in range(dl - 1, -1, -1)] + ["finalize"]
    flops = {"kappa": 2.0 * cfg.n_z * 2 * (1 << cfg.level) ** 2, "leaf": leaf_fl, "finalize": 0.0}
    for d, f in merge_fl.items():
        flops[f"merge_d{d}"] = f
    shares = {n: float(stage[i]) for i, n in enumerate(names)}
    n_sub = math.ceil(B / info.max_batch)
    # group the stages by the kernel they launch (the names of the ncu launch list): the
    # dominant KERNEL is the instantiation with the largest share of the step, which may
    # run at several tree depths
    def stage_kernel(n):
        if n == "kappa":
            return "kappa_kernel"
        if n == "finalize":
            return "finalize_kernel"
        buf = C.create_string_buffer(160)
        dep = -1 if n == "leaf" else int(n.split("_d")[1])
        lib_plan.check(lib_plan.lib.hdd_plan_stage_kernel(lib_plan.handle, dep, min(B, info.max_batch), buf, 160))
        return buf.value.decode()

    lib_plan = plan
    by_kernel = {}
    for n in names:
        if shares[n] <= 0.0:
            continue
        g = by_kernel.setdefault(stage_kernel(n), {"ms": 0.0, "flops_per_sample": 0.0, "stages": []})
        g["ms"] += shares[n]
        g["flops_per_sample"] += flops.get(n, 0.0)
        g["stages"].append(n)
    step_ms_sum = sum(shares.values())
    for g in by_kernel.values():
        g["share_of_step"] = g["ms"] / step_ms_sum
        g["achieved_tflops"] = g["flops_per_sample"] * B / (g["ms"] * 1e-3) / 1e12
        g["frac_fp64"] = g["achieved_tflops"] / FP64_PEAK_TFLOPS
    top = max(by_kernel, key=lambda kname: by_kernel[kname]["ms"])
    top_g = by_kernel[top]
    top_ms = top_g["ms"]
    launches_top = n_sub * len(top_g["stages"])                 # launches of that kernel per step
    achieved = top_g["achieved_tflops"]
    total_fl = leaf_fl + sum(merge_fl.values())
    hbm_gbs, hbm_src = hbm_peak()
    kappa_bytes = (2 * (1 << cfg.level) ** 2 * 8 + cfg.n_z * 8) * B
    # DRAM traffic of the same launches from the committed ncu captures (per-sample bytes
    # of each stage x the samples of one launch, averaged over the kernel's launches)
    trs = {n: traffic_from_capture(args.config, n, B / n_sub) for n in top_g["stages"]}
    have = [n for n in top_g["stages"] if trs[n] is not None]
    tr = None
    if have:
        tr = {"bytes_per_launch": sum(trs[n]["bytes_per_launch"] for n in have) / len(have),
              "samples_per_launch": B / n_sub, "captured_stages": have,
              "source": [trs[n]["source"] for n in have],
              "note": "mean over the kernel's captured launches (one per depth) of the ncu per-sample DRAM bytes "
                      "x the samples of one launch"}
    algo_per_launch = top_g["flops_per_sample"] * B / launches_top

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cores = len(os.sched_getaffinity(0))
        kind, path = _cpu_setup(args.config)
        n_s = cpu_rows_per_step(args.config, cores)
        v, wall, ll_cpu = time_cpu(Zl[:n_s], min(cores, n_s))
        ll_gpu = ll.cpu().numpy()[:n_s]
        cpu = {"value": v, "unit": "samples/s", "cores": min(cores, n_s), "kind": kind,
               "sample": f"first {n_s} Z rows of {args.config} ({wall:.1f} s wall, setup excluded), forked workers x "
                         f"1 BLAS thread: {path}",
               "max_rel_ll_diff_vs_gpu": float(np.max(np.abs(ll_cpu - ll_gpu) / np.abs(ll_cpu)))}

    per_cfg = None
    if world == 1 and not args.no_per_config:
        ll_host = ll.cpu().numpy()
        plan = None                      # release the flagship plan's workspace first
        problem._plan = None
        del Zd, ll, flush
        import gc
        gc.collect()
        torch.cuda.empty_cache()
        per_cfg = per_config_measurements(dev)
        del ll_host

    # forward kernels per sub-batch + the posterior-weights kernel per step
    launches = args.steps * (info.n_kernels_per_batch * n_sub + 1)
    line = {
        "metric": f"likelihood evals/s ({args.config}, {cfg.level}-level grid, n_z={cfg.n_z})",
        "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_max, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded protocol, DESIGN.md)",
        "config": {"workload": args.config, "global_batch": G, "batch_per_gpu": B, "sub_batches_per_gpu": n_sub,
                   "grid_nodes": (1 << cfg.level) + 1, "n_z": cfg.n_z, "n_obs": info.n_obs,
                   "parallelism": f"dp{world} (fixed global batch, Z rows sharded, NCCL all-gather of ll)",
                   "l2": "flushed between steps (256 MiB memset); per-step working set "
                         f"{info.workspace_bytes / 2**30:.2f} GiB > L2"},
        "roofline": {"bound": "tensor", "kernel": top, "stages": top_g["stages"], "achieved": achieved,
                     "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s", "frac": achieved / FP64_PEAK_TFLOPS,
                     "traffic": None if tr is None else tr["bytes_per_launch"],
                     "traffic_source": None if tr is None else tr,
                     "algorithmic_flops_per_launch": algo_per_launch,
                     "launches_per_step": launches_top,
                     "avg_launch_ms": top_ms / launches_top,
                     "peak_source": FP64_PEAK_SRC,
                     "kernel_share_of_step": top_ms / step_ms_sum},
        "kernels": by_kernel,
        "step_roofline": {"achieved_tflops": total_fl * G / (ms_max * 1e-3) / 1e12,
                          "frac_fp64": total_fl * G / (ms_max * 1e-3) / 1e12 / FP64_PEAK_TFLOPS / world,
                          "flops_per_sample": total_fl},
        "stage_ms": shares,
        "stage_ms_note": f"one CUDA-event-timed pass over the first {B_st} rows, scaled to the {B}-row step",
        "kappa_hbm": {"achieved_gbs": kappa_bytes / (shares["kappa"] * 1e-3) / 1e9, "peak": hbm_gbs,
                      "peak_source": hbm_src},
        "e2e": {"value": G / (e2e_max * 1e-3), "unit": "samples/s",
                "h2d_bytes_per_step": int(B * cfg.n_z * 8), "d2h_bytes_per_step": int(B * 8),
                "ms_per_step": e2e_max, "steps": n_e2e,
                "path": "bayes.log_likelihood_batch(numpy pinned Z) -> hdd_forward_batch_host"},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "posterior": {"argmax": idx, "log_evidence_minus_logB": lse - math.log(n_w)},
        "cpu_baseline": cpu,
        "per_config": per_cfg,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def _spawned(local_rank, args, world, port):
    os.environ.update(RANK=str(local_rank), LOCAL_RANK=str(local_rank), WORLD_SIZE=str(world),
                      LOCAL_WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    main_rank(args)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C4")
    ap.add_argument("--batch", type=int, default=0, help="global batch (default: the config's BASELINE batch)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-per-config", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # launched without torchrun: form the N-rank NCCL job ourselves
        import socket
        import torch
        import torch.multiprocessing as mp
        n_dev = torch.cuda.device_count()
        if n_dev < args.gpus:
            raise SystemExit(f"bench.py --gpus {args.gpus}: only {n_dev} CUDA devices visible")
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        mp.start_processes(_spawned, args=(args, args.gpus, port), nprocs=args.gpus, start_method="spawn")
        return
    if "WORLD_SIZE" in os.environ and int(os.environ["WORLD_SIZE"]) != args.gpus:
        raise SystemExit(f"bench.py --gpus {args.gpus} but WORLD_SIZE={os.environ['WORLD_SIZE']}")
    main_rank(args)


if __name__ == "__main__":
    main()
