"""Benchmark of the batched HDD likelihood (one JSON line on rank 0).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

A step = one batched likelihood evaluation of the config's Z batch (C2:
1024 samples of the 129x129-node problem) per GPU, followed by the NCCL
all-gather of the log-likelihoods and the global posterior weights / argmax
(weak scaling: every rank evaluates its own B rows).

* value      samples/s over all ranks, Z resident in HBM, CUDA events around
             each step on the launching stream, L2 flushed (256 MiB memset)
             between steps, max over ranks;
* e2e        the same through the public Python API with pinned host Z:
             H2D of Z and D2H of ll inside every timed step;
* roofline   dominant kernel (largest share of the step): algorithmic FP64
             flops / its average CUDA-event time,
             against the measured FP64 DGEMM peak (profiles/fp64_peaks_r01.jsonl);
* cpu_baseline  the oracle port of the reference HDD path (oracle/hdd_port.py)
             on the host cores, forked workers x 1 BLAS thread, bounded sample.
`--impl reference` times that same CPU path as the reference arm.
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
    dl = 2 * (level - 4)
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
def cpu_port_worker(args):
    """Forked worker: oracle port of the reference HDD path on a few samples."""
    idx, Z, level, obs, y, sigma, n_z = args
    from threadpoolctl import threadpool_limits
    from oracle import hdd_port
    threadpool_limits(1)
    port = _PORT["port"]
    fo = _PORT["field"]
    out = []
    for z in Z:
        s = port.forward(fo.kappa_values(z))
        out.append(hdd_port.gaussian_ll(y, s, sigma))
    return idx, out


_PORT = {}


def time_cpu_port(cfg_name, n_samples, n_workers):
    """Returns (samples/s, cores, wall seconds, build seconds, ll)."""
    import multiprocessing as mp
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    from oracle import fields, geometry, hdd_port
    from paper_1708_02207_b200 import configs
    cfg = configs.CONFIGS[cfg_name]
    obs = configs.observations(cfg)
    y, sigma = configs.observed_data(cfg)
    t0 = time.time()
    _PORT["port"] = hdd_port.HDDPort(cfg.level, obs)
    _PORT["field"] = fields.SineKLField(geometry.Grid(cfg.level), cfg.n_z)
    build_s = time.time() - t0
    Z = configs.draw_Z(cfg)[:n_samples]
    chunks = np.array_split(np.arange(n_samples), n_workers)
    ctx = mp.get_context("fork")
    t0 = time.time()
    with ctx.Pool(n_workers) as pool:
        res = pool.map(cpu_port_worker, [(i, Z[c], cfg.level, obs, y, sigma, cfg.n_z)
                                         for i, c in enumerate(chunks) if len(c)])
    wall = time.time() - t0
    ll = np.concatenate([np.array(r[1]) for r in sorted(res)])
    return n_samples / wall, n_workers, wall, build_s, ll


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cores = len(os.sched_getaffinity(0))
    from paper_1708_02207_b200 import configs
    cfg = configs.CONFIGS[args.config]
    per_step = {"C1": 64, "C2": cores, "C3": cores}.get(args.config, cores)
    for _ in range(args.warmup):
        time_cpu_port(args.config, min(per_step, cores), min(per_step, cores))
    vals = []
    t_all = 0.0
    for _ in range(args.steps):
        v, c, wall, build_s, _ = time_cpu_port(args.config, per_step, min(per_step, cores))
        vals.append(v)
        t_all += wall
    value = args.steps * per_step / t_all
    line = {
        "impl": "reference", "metric": f"likelihood evals/s ({args.config}, {cfg.level}-level grid, n_z={cfg.n_z})",
        "value": value, "unit": "samples/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * t_all / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded protocol, DESIGN.md)",
        "config": {"workload": args.config, "batch_per_step": per_step, "grid_nodes": (1 << cfg.level) + 1,
                   "n_z": cfg.n_z, "n_obs": len(configs.observations(cfg)),
                   "parallelism": "host cores (one forked worker per core, rank 0 only)"},
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": min(per_step, cores), "kind": "port",
                         "sample": f"{per_step} Z rows per step of {args.config}, forked workers x 1 BLAS thread, "
                                   "oracle/hdd_port.py (restatement of the reference HDD functional path)"},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C2")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return

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
    from paper_1708_02207_b200.parallel import gather_log_likelihood, posterior_weights_device

    cfg = configs.CONFIGS[args.config]
    B = cfg.batch
    problem = configs.make_problem(args.config, device=local)
    plan = problem.plan()
    info = plan.info()
    Zall = configs.draw_Z(cfg, batch=B * world)
    Zl = np.ascontiguousarray(Zall[rank * B:(rank + 1) * B])
    Zd = torch.from_numpy(Zl).to(dev)
    ll = torch.empty(B, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)
    n_stages = info.leaf_depth + 3
    stage = np.zeros(n_stages)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def step(timed_stages):
        if timed_stages is not None:
            rc = plan.lib.hdd_forward_batch_timed(plan.handle, C.c_void_p(Zd.data_ptr()), B, None,
                                                  C.c_void_p(ll.data_ptr()), C.c_void_p(stream.cuda_stream),
                                                  timed_stages.ctypes.data_as(_lib._f64p), n_stages)
        else:
            rc = plan.lib.hdd_forward_batch(plan.handle, C.c_void_p(Zd.data_ptr()), B, None,
                                            C.c_void_p(ll.data_ptr()), C.c_void_p(stream.cuda_stream))
        plan.check(rc)
        return gather_log_likelihood(ll, world)

    for _ in range(args.warmup):
        posterior_weights_device(step(None))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.zero_()
            ev[i][0].record(stream)
            ll_all = step(None)
            w, idx_t, lse_t = posterior_weights_device(ll_all)
            ev[i][1].record(stream)
        torch.cuda.synchronize()
    idx, lse, n_w = int(idx_t.item()), float(lse_t.item()), int(w.numel())
    step_ms = [a.elapsed_time(b) for a, b in ev]
    ms = float(np.mean(step_ms))
    # per-stage (kernel) times: separate pass, same stream, CUDA events between launches
    for _ in range(args.steps):
        flush.zero_()
        step(stage)
    stage /= args.steps
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = world * B / (ms_max * 1e-3)

    # ---- e2e through the public API: pinned host Z -> device -> ll -> host ----
    Zh = torch.from_numpy(Zl).pin_memory()
    llh = torch.empty(B, dtype=torch.float64).pin_memory()
    for _ in range(2):
        bayes.log_likelihood_batch(problem, Zh.to(dev, non_blocking=True))
    torch.cuda.synchronize()
    e2e_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for i in range(args.steps):
        flush.zero_()
        e2e_ev[i][0].record(stream)
        Zs = Zh.to(dev, non_blocking=True)
        out = bayes.log_likelihood_batch(problem, Zs)
        llh.copy_(out, non_blocking=True)
        e2e_ev[i][1].record(stream)
    torch.cuda.synchronize()
    e2e_ms = float(np.mean([a.elapsed_time(b) for a, b in e2e_ev]))
    t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_ms = float(t.item())

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel ----
    leaf_fl, merge_fl = flops_split(cfg.level)
    dl = info.leaf_depth
    names = ["kappa", "leaf"] + [f"merge_d{d}" for d in range(dl - 1, -1, -1)] + ["finalize"]
    flops = {"kappa": 2.0 * cfg.n_z * 2 * (1 << cfg.level) ** 2, "leaf": leaf_fl, "finalize": 0.0}
    for d, f in merge_fl.items():
        flops[f"merge_d{d}"] = f
    shares = {n: float(stage[i]) for i, n in enumerate(names)}
    top = max(shares, key=shares.get)
    top_ms = shares[top]
    achieved = flops[top] * B / (top_ms * 1e-3) / 1e12
    total_fl = leaf_fl + sum(merge_fl.values())
    hbm_gbs, hbm_src = hbm_peak()
    kappa_bytes = (2 * (1 << cfg.level) ** 2 * 8 + cfg.n_z * 8) * B

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cores = len(os.sched_getaffinity(0))
        n_s = {"C1": 64, "C2": 2 * cores, "C3": cores}.get(args.config, cores)
        v, c, wall, build_s, ll_cpu = time_cpu_port(args.config, n_s, min(cores, n_s))
        ll_gpu = ll.cpu().numpy()[:n_s]
        cpu = {"value": v, "unit": "samples/s", "cores": c, "kind": "port",
               "sample": f"first {n_s} Z rows of {args.config} ({wall:.1f} s wall, tree build {build_s:.1f} s "
                         "excluded), forked workers x 1 BLAS thread, oracle/hdd_port.py",
               "max_rel_ll_diff_vs_gpu": float(np.max(np.abs(ll_cpu - ll_gpu) / np.abs(ll_cpu)))}

    # forward kernels per sub-batch + the posterior-weights kernel per step
    launches = args.steps * (info.n_kernels_per_batch * math.ceil(B / info.max_batch) + 1)
    # measured DRAM bytes per launch of the dominant kernel (ncu --set full capture,
    # profiles/r01_ncu_full_leaf_v4_C2.csv: 23.6 KB per leaf-sample) scaled to this launch;
    # the leaf's binding resource is shared-memory bandwidth (same capture)
    traffic = None
    binding = None
    if top == "leaf":
        traffic = {"bytes": 23.6e3 * B * ((1 << cfg.level) // 16) ** 2,
                   "source": "ncu dram__bytes_read+write, leaf2_kernel<2> C2: 1184 MB / (49 leaves x 1024)"}
        binding = {"resource": "instruction issue + shared-memory wavefronts (3 CTAs/SM, latency-bound per CTA)",
                   "issue_active_pct": 59.3, "smem_wavefront_util_pct": 68.7, "dmma_pipe_pct": 11.7,
                   "source": "profiles/r01_ncu_full_leaf_v13_C2.csv"}
    line = {
        "metric": f"likelihood evals/s ({args.config}, {cfg.level}-level grid, n_z={cfg.n_z})",
        "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded protocol, DESIGN.md)",
        "config": {"workload": args.config, "batch_per_gpu": B, "global_batch": B * world,
                   "grid_nodes": (1 << cfg.level) + 1, "n_z": cfg.n_z, "n_obs": info.n_obs,
                   "parallelism": f"dp{world} (Z rows sharded, NCCL all-gather of ll)",
                   "l2": "flushed between steps (256 MiB memset); per-step working set "
                         f"{info.workspace_bytes / 2**30:.2f} GiB > L2"},
        "roofline": {"bound": "tensor", "kernel": top, "achieved": achieved, "peak": FP64_PEAK_TFLOPS,
                     "unit": "TFLOP/s", "frac": achieved / FP64_PEAK_TFLOPS, "traffic": traffic,
                     "peak_source": FP64_PEAK_SRC,
                     "kernel_share_of_step": top_ms / sum(shares.values()),
                     "binding_resource": binding,
                     "algorithmic_flops_per_launch": flops[top] * B},
        "step_roofline": {"achieved_tflops": total_fl * B / (ms_max * 1e-3) / 1e12,
                          "frac_fp64": total_fl * B / (ms_max * 1e-3) / 1e12 / FP64_PEAK_TFLOPS,
                          "flops_per_sample": total_fl},
        "stage_ms": shares,
        "kappa_hbm": {"achieved_gbs": kappa_bytes / (shares["kappa"] * 1e-3) / 1e9, "peak": hbm_gbs,
                      "peak_source": hbm_src},
        "e2e": {"value": world * B / (e2e_ms * 1e-3), "unit": "samples/s",
                "h2d_bytes_per_step": int(B * cfg.n_z * 8), "d2h_bytes_per_step": int(B * 8),
                "ms_per_step": e2e_ms},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "posterior": {"argmax": idx, "log_evidence_minus_logB": lse - math.log(n_w)},
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
