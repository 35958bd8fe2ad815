"""Headline benchmark: HT truncations/sec (fp64, d=64, n=1000, k=50) on B200.

One step = ``truncate(X, fixed_rank(50))`` on the non-orthogonal sum
X = add(A, C) of two seeded Gaussian HT tensors (rank 100 -> 50): bottom-up
Householder orthogonalisation, top-down reduced Gramians, batched Jacobi
eigendecompositions, projection -- reference arith.py:325-352.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line (rank 0).  Under torchrun (N > 1) every rank truncates its
own replica tensor (independent objects, no collective on the data path);
``value`` is the whole-job rate, the step time is the max over ranks.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "HT truncations/sec (fp64, d=64,n=1000,k=50) at 1/2/4/8 GPU; % of FP64/HBM roofline"
UNIT = "truncations/s"


def algorithmic_flops(d: int, n: int, K: int, r: int) -> float:
    """SURVEY §8(d) / Appendix A count for one truncation (balanced tree, d = 2^p)."""
    leaves = d
    inner = d - 2
    f = leaves * (4 * n * K**2 - 4 / 3 * K**3 + 9 * K**3 + 2 * n * K * r)
    f += inner * (8 * K**4 - 4 / 3 * K**3 + 6 * K**4 + 9 * K**3 + 2 * r * K**3 + 2 * r**2 * K**2 + 2 * r**3 * K)
    f += 4 * K**3 + 2 * K**2 + 4 * K**3 + 2 * r * K**2 + 2 * r**2 * K
    return float(f)


def storage(d, n, k):
    return d * n * k + (d - 2) * k**3 + k**2


class ClockSampler:
    """nvidia-smi-equivalent NVML sampling of SM clocks and throttle reasons during the timed region."""

    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4, "hw_slowdown": 0x8,
        "sync_boost": 0x10, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
        "hw_power_brake_slowdown": 0x80, "display_clock_setting": 0x100,
    }

    def __init__(self, index: int):
        self.samples, self.reasons = [], set()
        self._stop = threading.Event()
        self.max_mhz = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover - NVML missing
            self._nv = None
            self.error = str(e)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self._nv.nvmlDeviceGetClockInfo(self._h, self._nv.NVML_CLOCK_SM))
                mask = self._nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for name, bit in self.REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.05)

    def __enter__(self):
        if self._nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._nv is not None:
            self._t.join()

    def summary(self):
        if self._nv is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        med = float(np.median(self.samples)) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def dgemm_peak_tflops():
    """Measured FP64 roofline denominator on this box: cuBLAS DGEMM 4096^3 (best of 5).
    MEASURED_PEAKS.json carries only bf16 and HBM figures."""
    import torch

    a = torch.randn(4096, 4096, dtype=torch.float64, device="cuda")
    b = torch.randn(4096, 4096, dtype=torch.float64, device="cuda")
    for _ in range(2):
        a @ b
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        a @ b
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return 2 * 4096**3 / best / 1e9


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_truncation(x, k, threads):
    """The oracle port (numpy -> OpenBLAS, same LAPACK calls as the reference) on host cores."""
    from threadpoolctl import threadpool_limits

    from oracle import htucker_oracle as orc

    with threadpool_limits(limits=threads):
        t0 = time.perf_counter()
        t = orc.truncate(x, orc.Ctl(max_rank=k))
        dt = time.perf_counter() - t0
    return t, dt


def parity_summary(T, t_ref, x):
    """Checker only: GPU result vs the oracle port on the same inputs (relative error
    through the orthogonalised difference, SURVEY finding 0.3.3; identical ranks)."""
    from oracle import htucker_oracle as orc

    leaves, transfer, root = T.to_numpy()
    got = orc.HT(orc.balanced_tree(T.tree.d), leaves, transfer, root)
    err = orc.orth_difference_norm(got, t_ref) / orc.norm(x)
    return {"rel_err_vs_oracle": err, "ranks_equal": got.ranks == t_ref.ranks, "tol": 1e-10}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# ---------------------------------------------------------------------------
# reference arm: the reference's own CPU algorithm (oracle port), rank 0 only
# ---------------------------------------------------------------------------


def run_reference(args, rank, world):
    if rank != 0:
        return None
    from oracle import htucker_oracle as orc

    threads = cpu_threads()
    _, _, x = orc.c2_inputs(args.d, args.n, args.k)
    times = []
    budget_s = 150.0
    warm = min(args.warmup, 1)
    for _ in range(warm):
        cpu_truncation(x, args.k, threads)
    t_start = time.perf_counter()
    for i in range(args.steps):
        _, dt = cpu_truncation(x, args.k, threads)
        times.append(dt)
        if time.perf_counter() - t_start > budget_s:
            break
    total = sum(times)
    value = len(times) / total
    sample = (f"{len(times)} full C2 d={args.d} truncations (requested {args.steps}; capped at ~{budget_s:.0f}s), "
              f"numpy {np.__version__} / OpenBLAS, {threads} threads, {cpu_model()}")
    return {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": world,
        "steps": len(times), "warmup": warm, "ms_per_step": 1e3 * total / len(times), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded Gaussian, SURVEY §8(d))",
        "config": config_dict(args),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def config_dict(args):
    return {"workload": f"C2: truncate(add(A,C)) d={args.d} n={args.n} rank {2 * args.k}->{args.k}",
            "d": args.d, "n": args.n, "k": args.k, "pre_truncation_rank": 2 * args.k,
            "seeds": [2 * int(round(math.log2(args.d))), 2 * int(round(math.log2(args.d))) + 1],
            "l2_policy": f"inputs {8 * storage(args.d, args.n, 2 * args.k) / 1e6:.0f} MB > 126 MB L2 (no flush needed)",
            "parallelism": "replica per GPU"}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_1708_03340_b200 as htb
    from paper_1708_03340_b200 import _lib
    from oracle import htucker_oracle as orc

    torch.cuda.set_device(local_rank)
    lib = _lib.load()
    # every rank: its own replica (seed offset by rank) -- independent objects
    a, c, x = orc.c2_inputs(args.d, args.n, args.k, seed_base=2 * int(round(math.log2(args.d))) + 2 * rank)
    tree = htb.build_balanced_tree(args.d)
    ad = htb.HTensor(tree, a.U, a.B, a.root)
    cd = htb.HTensor(tree, c.U, c.B, c.root)
    xd = htb.add(ad, cd)  # X resident in HBM (547 MB at d=64: larger than L2)
    del ad, cd
    ctl = htb.TruncationControl.fixed_rank(args.k)
    for _ in range(args.warmup):
        htb.truncate(xd, ctl)
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()

    stream = torch.cuda.current_stream()
    with ClockSampler(local_rank) as clk:
        barrier()
        torch.cuda.synchronize()
        n0 = lib.ht_launch_count()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            T = htb.truncate(xd, ctl)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        launches = lib.ht_launch_count() - n0
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = world * 1e3 / ms

    # per-kernel event timing (separate instrumented steps right after the timed region)
    lib.ht_profile_enable(1)
    prof_steps = 2
    for _ in range(prof_steps):
        htb.truncate(xd, ctl)
    torch.cuda.synchronize()
    prof = _lib.profile_report()
    lib.ht_profile_enable(0)

    # end-to-end through the public API: pinned host X -> H2D -> truncate -> D2H of T
    host_x = xd.to_host_arena()
    sizes, ranks = xd.host_layout()
    out_host = None
    torch.cuda.synchronize()
    e2e_steps = max(1, min(args.steps, 5))
    for _ in range(1):
        xh = htb.HTensor.from_host_arena(tree, sizes, ranks, host_x)
        out_host = htb.truncate(xh, ctl).to_host_arena(out_host)
    torch.cuda.synchronize()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    f0.record(stream)
    for _ in range(e2e_steps):
        xh = htb.HTensor.from_host_arena(tree, sizes, ranks, host_x)
        Th = htb.truncate(xh, ctl)
        out_host = Th.to_host_arena(out_host)
    f1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = f0.elapsed_time(f1) / e2e_steps
    if world > 1:
        t = torch.tensor([e2e_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    h2d = host_x.numel() * 8
    d2h = out_host.numel() * 8

    if rank != 0:
        return None

    peak64 = dgemm_peak_tflops()
    peaks = measured_peaks()
    # dominant kernel roofline (algorithmic flops / event-timed duration on the launching stream)
    dom_name, dom = max(prof.items(), key=lambda kv: kv[1]["ms"])
    step_ms_prof = sum(v["ms"] for v in prof.values()) / prof_steps
    if dom["flops"] > 0:
        ach = dom["flops"] / (dom["ms"] * 1e-3) / 1e12
        roof = {"kernel": dom_name, "bound": "tensor", "achieved": ach, "peak": peak64, "unit": "TFLOP/s",
                "frac": ach / peak64, "traffic": None,
                "peak_source": "cuBLAS DGEMM 4096^3 measured in this run (FP64; DMMA/DFMA microbench 37.1 TF, "
                               "profiles/r01_fp64_peak_microbench.jsonl)",
                "launches_per_step": dom["launches"] / prof_steps,
                "share_of_step": dom["ms"] / prof_steps / step_ms_prof}
    else:
        bw = dom["bytes"] / (dom["ms"] * 1e-3) / 1e9
        roof = {"kernel": dom_name, "bound": "hbm", "achieved": bw, "peak": peaks.get("hbm_gbs", 6521.1),
                "unit": "GB/s", "frac": bw / peaks.get("hbm_gbs", 6521.1), "traffic": None}
    flops = algorithmic_flops(args.d, args.n, 2 * args.k, args.k)
    step_tf = flops / (ms * 1e-3) / 1e12
    kernels = {k: {"ms_per_step": v["ms"] / prof_steps, "launches_per_step": v["launches"] / prof_steps,
                   "tflops": (v["flops"] / (v["ms"] * 1e-3) / 1e12) if v["flops"] else None}
               for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"])}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded Gaussian factors, SURVEY §8(d))",
        "config": config_dict(args),
        "roofline": roof,
        "roofline_step": {"bound": "tensor", "achieved": step_tf, "peak": peak64, "unit": "TFLOP/s",
                          "frac": step_tf / peak64, "flops_per_truncation": flops},
        "kernels": kernels,
        "e2e": {"value": world * 1e3 / e2e_ms, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": e2e_ms},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    if world == 1 and not args.no_cpu_baseline:
        threads = cpu_threads()
        t_ref, dt = cpu_truncation(x, args.k, threads)
        line["cpu_baseline"] = {"value": 1.0 / dt, "unit": UNIT, "cores": threads, "kind": "port",
                                "sample": f"1 full C2 d={args.d} truncation (oracle port: numpy {np.__version__} "
                                          f"-> OpenBLAS, same LAPACK calls as the reference), {cpu_model()}"}
        line["parity"] = parity_summary(T, t_ref, x)
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--d", type=int, default=64)
    ap.add_argument("--n", type=int, default=1000)
    ap.add_argument("--k", type=int, default=50)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        line = run_reference(args, rank, world)
    else:
        if world > 1:
            import torch
            import torch.distributed as dist

            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl")
        line = run_ours(args, rank, world, local_rank)
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()
    if line is not None:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
