"""Secondary measurements on one B200: the C2 weak-scaling sweep
(d = 2^p, p = 3..8: add, truncate, truncate of the orthogonalised tensor, <T,T>;
time vs log2 d), C1, C3 (operator apply + eps/cap truncation) and one C5 shard
(d = 32 leaves of n = 2048, four rank-100 tensors summed to rank 400 -> 100: the
subtree one GPU owns in the 8-GPU layout).  Device times from CUDA events on the
launching stream, after warm-up; inputs are seeded Gaussian factors.

    python tools/sweep.py [--only c2,c1,c3,c5] > profiles/r01_sweep.jsonl
"""
import argparse
import json
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_03340_b200 as htb  # noqa: E402
from paper_1708_03340_b200 import problems  # noqa: E402
from bench import algorithmic_flops  # noqa: E402


def timed(fn, reps, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def c2(p, reps):
    d = 2 ** p
    tree = htb.build_balanced_tree(d)
    a = htb.HTensor(tree, *htb.gaussian_factors(tree, 1000, 50, 2 * p))
    c = htb.HTensor(tree, *htb.gaussian_factors(tree, 1000, 50, 2 * p + 1))
    ctl = htb.TruncationControl.fixed_rank(50)
    x = htb.add(a, c)
    t = htb.truncate(x, ctl)
    xo = htb.orthogonalize(x)
    ms_add = timed(lambda: htb.add(a, c), reps)
    ms_tr = timed(lambda: htb.truncate(x, ctl), reps)
    ms_tro = timed(lambda: htb.truncate(xo, ctl), reps)
    ms_ip = timed(lambda: htb.inner_product_device(t, t), reps)
    fl = algorithmic_flops(d, 1000, 100, 50)
    return {"config": "C2", "d": d, "log2_d": p, "n": 1000, "K": 100, "r": 50,
            "add_ms": ms_add, "truncate_ms": ms_tr, "truncations_per_s": 1e3 / ms_tr,
            "truncate_gflops": fl / (ms_tr * 1e-3) / 1e9,
            "truncate_orthogonal_input_ms": ms_tro, "inner_product_ms": ms_ip,
            "add_truncate_ip_ms": ms_add + ms_tr + ms_ip}


def c1(reps):
    tree = htb.build_balanced_tree(8)
    a = htb.gaussian_htensor(tree, 64, 10, 0, scaled=False)
    c = htb.gaussian_htensor(tree, 64, 10, 1, scaled=False)
    x = htb.add(htb.scale(a, 2.0), htb.scale(c, 1e-10))
    ctl = htb.TruncationControl.fixed_rank(10)
    ms = timed(lambda: htb.truncate(x, ctl), reps)
    return {"config": "C1", "d": 8, "n": 64, "K": 20, "r": 10, "truncate_ms": ms, "truncations_per_s": 1e3 / ms}


def c3(reps):
    tree = htb.build_balanced_tree(16)
    x = htb.gaussian_htensor(tree, 256, 30, 16)
    op = problems.laplace_sum_operator(tree, 256)
    y = htb.apply_operator(op, x)
    ny = htb.norm(y)
    ctl = htb.TruncationControl(eps=1e-8 * ny, max_rank=30)
    y = htb.apply_operator(op, x, lazy=False)
    ms_apply = timed(lambda: htb.apply_operator(op, x, lazy=False), reps)
    ms_norm = timed(lambda: htb.norm(y), reps)
    ms_tr = timed(lambda: htb.truncate(y, ctl), reps)
    t = htb.truncate(y, ctl)
    # Kronecker-fused workflow: F_t never materialised, ||Y|| taken on the device inside
    # the truncation (HT_CTL_RELATIVE_EPS)
    rctl = htb.TruncationControl.relative_accuracy(1e-8, max_rank=30)
    ms_fused = timed(lambda: htb.truncate(htb.apply_operator(op, x), rctl), reps)
    ms_lazy_apply = timed(lambda: htb.apply_operator(op, x), reps)
    tf = htb.truncate(htb.apply_operator(op, x), rctl)
    return {"config": "C3", "d": 16, "n": 256, "K": 60, "r": 30, "apply_ms": ms_apply, "norm_ms": ms_norm,
            "truncate_ms": ms_tr, "apply_norm_truncate_ms": ms_apply + ms_norm + ms_tr,
            "fused_apply_truncate_ms": ms_fused, "lazy_apply_ms": ms_lazy_apply,
            "ranks_out": sorted(set(t.ranks.values())), "ranks_out_fused": sorted(set(tf.ranks.values()))}


def c5_shard(reps):
    d, n = 32, 2048
    tree = htb.build_balanced_tree(d)
    parts = [htb.HTensor(tree, *htb.gaussian_factors(tree, n, 100, s)) for s in range(4)]
    x = htb.add(htb.add(htb.add(parts[0], parts[1]), parts[2]), parts[3])
    ctl = htb.TruncationControl.fixed_rank(100)
    ms_add = timed(lambda: htb.add(htb.add(htb.add(parts[0], parts[1]), parts[2]), parts[3]), max(1, reps // 4), 1)
    ms_tr = timed(lambda: htb.truncate(x, ctl), reps, 1)
    fl = algorithmic_flops(d, n, 400, 100)
    return {"config": "C5 shard (one GPU's subtree of the 8-GPU layout)", "d": d, "n": n, "K": 400, "r": 100,
            "add3_ms": ms_add, "truncate_ms": ms_tr, "truncate_gflops": fl / (ms_tr * 1e-3) / 1e9,
            "x_bytes": 8 * (d * n * 400 + (d - 2) * 400 ** 3 + 400 ** 2)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="c2,c1,c3,c5")
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    only = a.only.split(",")
    dev = torch.cuda.get_device_name(0)
    if "c1" in only:
        print(json.dumps({**c1(50), "gpu": dev}), flush=True)
    if "c2" in only:
        rows = []
        for p in range(3, 9):
            r = c2(p, a.reps)
            rows.append(r)
            print(json.dumps({**r, "gpu": dev}), flush=True)
            torch.cuda.empty_cache()
        # least-squares fit  t = a + b log2 d  (the reference's acceptance model)
        xs = [r["log2_d"] for r in rows]
        ys = [r["truncate_ms"] for r in rows]
        mx, my = sum(xs) / len(xs), sum(ys) / len(ys)
        b = sum((u - mx) * (v - my) for u, v in zip(xs, ys)) / sum((u - mx) ** 2 for u in xs)
        print(json.dumps({"config": "C2 fit", "model": "truncate_ms = a + b*log2(d) (1 GPU: work grows ~ d)",
                          "a": my - b * mx, "b": b, "per_leaf_us": [1e3 * r["truncate_ms"] / r["d"] for r in rows]}),
              flush=True)
    if "c3" in only:
        print(json.dumps({**c3(a.reps), "gpu": dev}), flush=True)
    if "c5" in only:
        print(json.dumps({**c5_shard(3), "gpu": dev}), flush=True)


if __name__ == "__main__":
    main()
