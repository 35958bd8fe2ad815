"""Throughput of repeated C2 d=64 truncations with 1 vs 2 vs 3 in flight (streams):
the latency-bound phases of one truncation (Cholesky, eigensolver, split-K sums) leave
most SMs idle, which a concurrent truncation can fill (experiments)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_03340_b200 as htb  # noqa: E402

tree = htb.build_balanced_tree(64)
x = htb.add(htb.HTensor(tree, *htb.gaussian_factors(tree, 1000, 50, 12)),
            htb.HTensor(tree, *htb.gaussian_factors(tree, 1000, 50, 13)))
ctl = htb.TruncationControl.fixed_rank(50)
T0 = htb.truncate(x, ctl)
for nstreams in (1, 2, 3):
    streams = [torch.cuda.Stream() for _ in range(nstreams)]
    outs = [[htb.HTensor.empty(tree, *T0.host_layout()) for _ in range(2)] for _ in streams]
    main = torch.cuda.current_stream()

    def run(n, e_start):
        for s in streams:
            s.wait_event(e_start)
        for i in range(n):
            q = i % nstreams
            with torch.cuda.stream(streams[q]):
                htb.truncate(x, ctl, out=outs[q][(i // nstreams) % 2])
        for s in streams:
            ev = torch.cuda.Event()
            ev.record(s)
            main.wait_event(ev)

    e = torch.cuda.Event()
    e.record(main)
    run(12 * nstreams, e)
    torch.cuda.synchronize()
    steps = 40
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    run(steps, e0)
    e1.record(main)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    print(f"{nstreams} in flight: {ms:.3f} ms per truncation ({1e3 / ms:.1f}/s)", flush=True)
