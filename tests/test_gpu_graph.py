"""CUDA-graph replay of repeated fixed-rank truncations (driver.cu truncate_graph):
replays must reproduce the eager launches bit for bit, and the Cholesky-QR red flag
read behind the ORTH graph must still route rank-deficient input to the Householder
re-run (reference semantics: arith.py:325-352 with kernels.py:24-32's QR)."""

import numpy as np
import pytest

from oracle import htucker_oracle as orc
from tests.htconv import rel_err, to_host

pytestmark = pytest.mark.gpu


def _arrays(t):
    leaves, transfer, root = t.to_numpy()
    return [np.asarray(v) for _, v in sorted(leaves.items())] + \
           [np.asarray(v) for _, v in sorted(transfer.items())] + [np.asarray(root)]


def _truncs(htb, x, ctl, n):
    out = []
    for _ in range(n):
        out.append(_arrays(htb.truncate(x, ctl)))
    return out


@pytest.mark.parametrize("d,n,k", [(8, 300, 24), (16, 200, 40)])
def test_graph_replay_bitwise_equals_eager(cuda_ok, d, n, k):
    import paper_1708_03340_b200 as htb

    tree = htb.build_balanced_tree(d)
    x = htb.add(htb.gaussian_htensor(tree, n, k, 3), htb.gaussian_htensor(tree, n, k, 4))
    ctl = htb.TruncationControl.fixed_rank(k)
    htb.set_graph_mode(False)
    try:
        eager = _truncs(htb, x, ctl, 1)[0]
    finally:
        htb.set_graph_mode(True)
    c0, r0 = htb.graph_stats()
    got = _truncs(htb, x, ctl, 4)
    c1, r1 = htb.graph_stats()
    assert r1 - r0 >= 2, "repeated truncations of one tensor should replay the captured graph"
    assert c1 - c0 <= 2
    for g in got:
        for a, b in zip(g, eager):
            assert np.array_equal(a, b)
    ref = orc.truncate(to_host(x), orc.Ctl(max_rank=k))
    assert rel_err(to_host(htb.truncate(x, ctl)), ref) <= 1e-10


def test_graph_replay_routes_rank_deficient_input_to_householder(cuda_ok):
    import paper_1708_03340_b200 as htb

    tree = htb.build_balanced_tree(8)
    a = htb.gaussian_htensor(tree, 120, 12, 7)
    x = htb.add(a, a)  # rank 24 frames of rank 12: Cholesky-QR must raise its flag
    ctl = htb.TruncationControl.fixed_rank(12)
    f0 = htb.qr_fallback_count()
    outs = _truncs(htb, x, ctl, 4)
    assert htb.qr_fallback_count() - f0 == 4
    # replays take the Householder branch on the device (conditional node), no host check
    from paper_1708_03340_b200 import _lib
    assert _lib.load().ht_graph_device_fallback() == 1
    ref = orc.truncate(to_host(x), orc.Ctl(max_rank=12))
    leaves, transfer, root = htb.truncate(x, ctl).to_numpy()
    for o in outs[1:]:
        for p, q in zip(o, outs[0]):
            assert np.array_equal(p, q)
    got = orc.HT(orc.balanced_tree(8), {t: np.array(v) for t, v in leaves.items()},
                 {t: np.array(v) for t, v in transfer.items()}, np.array(root))
    assert orc.orth_difference_norm(got, ref) / orc.norm(ref) <= 1e-10


def _fresh_copy(htb, x):
    """The same values in a new arena (new addresses, same layout)."""
    sizes, ranks = x.host_layout()
    y = htb.HTensor.empty(x.tree, sizes, ranks, orthogonal=x.orthogonal)
    y._arena.copy_(x._arena)
    return y


@pytest.mark.parametrize("deficient", [False, True])
def test_graph_relocation_bitwise_equals_eager(cuda_ok, deficient, request):
    """Replays on moved buffers (new input, output and workspace addresses) relocate the
    cached graph instead of capturing again, and still reproduce the eager launches bit
    for bit -- including the device-side Householder branch (conditional body)."""
    import paper_1708_03340_b200 as htb

    tree = htb.build_balanced_tree(8)
    a = htb.gaussian_htensor(tree, 150, 14, 11)
    c = a if deficient else htb.gaussian_htensor(tree, 150, 14, 12)
    x = htb.add(a, c, lazy=False)
    ctl = htb.TruncationControl.fixed_rank(13)
    htb.set_graph_relocation(True)  # opt-in (off by default)
    request.addfinalizer(lambda: htb.set_graph_relocation(False))
    htb.set_graph_mode(False)
    try:
        eager = _arrays(htb.truncate(x, ctl))
    finally:
        htb.set_graph_mode(True)
    for _ in range(3):  # capture + replay on x
        htb.truncate(x, ctl)
    c0, _ = htb.graph_stats()
    m0 = htb.graph_relocations()
    keep = []
    for i in range(6):
        y = _fresh_copy(htb, x)
        keep.append(y)  # keep the buffers alive: every call sees new addresses
        got = _arrays(htb.truncate(y, ctl))
        for p, q in zip(got, eager):
            assert np.array_equal(p, q), f"relocated replay {i} differs from the eager truncation"
    c1, _ = htb.graph_stats()
    assert htb.graph_relocations() - m0 >= 4, "moved buffers should relocate the cached graph"
    assert c1 - c0 <= 1


def test_graph_relocation_whole_graph_update_path(cuda_ok):
    """Same check with relocation forced through cudaGraphExecUpdate (HT_RELOC_UPDATE=1),
    the path used where the driver refuses per-node updates inside conditional bodies."""
    import os
    import subprocess
    import sys

    code = (
        "import numpy as np, paper_1708_03340_b200 as htb\n"
        "from tests.test_gpu_graph import _arrays, _fresh_copy\n"
        "htb.set_graph_relocation(True)\n"
        "tree = htb.build_balanced_tree(8)\n"
        "a = htb.gaussian_htensor(tree, 120, 12, 5)\n"
        "for c in (htb.gaussian_htensor(tree, 120, 12, 6), a):\n"
        "    x = htb.add(a, c, lazy=False); ctl = htb.TruncationControl.fixed_rank(11)\n"
        "    htb.set_graph_mode(False); ref = _arrays(htb.truncate(x, ctl)); htb.set_graph_mode(True)\n"
        "    [htb.truncate(x, ctl) for _ in range(3)]\n"
        "    m0 = htb.graph_relocations(); keep = []\n"
        "    for i in range(4):\n"
        "        y = _fresh_copy(htb, x); keep.append(y)\n"
        "        assert all(np.array_equal(p, q) for p, q in zip(_arrays(htb.truncate(y, ctl)), ref))\n"
        "    assert htb.graph_relocations() - m0 >= 3\n"
        "print('ok')\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, HT_RELOC_UPDATE="1", PYTHONPATH=root)
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


def test_fixed_rank_truncate_raises_on_non_finite_input(cuda_ok):
    """Fixed-rank truncate is asynchronous; a non-finite Gramian recorded by a queued
    (eager or graph-replayed) truncation is raised at the next host synchronisation."""
    import paper_1708_03340_b200 as htb

    tree = htb.build_balanced_tree(8)
    x = htb.add(htb.gaussian_htensor(tree, 100, 10, 1), htb.gaussian_htensor(tree, 100, 10, 2))
    ctl = htb.TruncationControl.fixed_rank(10)
    for _ in range(3):  # capture the graph on these buffers
        htb.truncate(x, ctl)
    htb.synchronize()
    x._arena[5] = float("nan")  # poison a leaf entry in place: the replay sees it
    t = htb.truncate(x, ctl)
    with pytest.raises(RuntimeError, match="not finite|converge"):
        t.to_numpy()
    htb.synchronize()  # the sticky word was cleared by the raise
    htb.set_graph_mode(False)
    try:
        htb.truncate(x, ctl)
        with pytest.raises(RuntimeError):
            htb.synchronize()
    finally:
        htb.set_graph_mode(True)


def test_host_resident_tensor_rejected(cuda_ok):
    import paper_1708_03340_b200 as htb

    tree = htb.build_balanced_tree(4)
    f = htb.gaussian_factors(tree, 20, 3, 0)
    xh = htb.HTensor(tree, *f, device="cpu")
    with pytest.raises(ValueError, match="CUDA"):
        htb.truncate(xh, htb.TruncationControl.fixed_rank(2))


def test_out_buffers_replay_without_relocation(cuda_ok):
    """add(..., out=) / truncate(..., out=) write into fixed buffers: the results equal the
    allocating calls bit for bit, alternating buffer pairs replay their own captured graphs
    (no relocation), and wrong shapes / data-dependent ranks are rejected."""
    import paper_1708_03340_b200 as htb

    tree = htb.build_balanced_tree(8)
    a, c = htb.gaussian_htensor(tree, 150, 16, 5), htb.gaussian_htensor(tree, 150, 16, 6)
    ctl = htb.TruncationControl.fixed_rank(16)
    ref = _arrays(htb.truncate(htb.add(a, c), ctl))
    x0 = htb.add(a, c)
    xb = [htb.HTensor.empty(tree, *x0.host_layout()) for _ in range(2)]
    t0 = htb.truncate(x0, ctl)
    tb = [htb.HTensor.empty(tree, *t0.host_layout()) for _ in range(2)]
    for i in range(6):
        x = htb.add(a, c, out=xb[i % 2])
        t = htb.truncate(x, ctl, out=tb[i % 2])
        assert t is tb[i % 2]
        for u, v in zip(_arrays(t), ref):
            np.testing.assert_array_equal(u, v)
    r0 = htb.graph_relocations()
    for i in range(4):
        htb.truncate(htb.add(a, c, out=xb[i % 2]), ctl, out=tb[i % 2])
    assert htb.graph_relocations() == r0
    with pytest.raises(ValueError):
        htb.truncate(x0, htb.TruncationControl.fixed_rank(8), out=tb[0])
    with pytest.raises(ValueError):
        htb.truncate(x0, htb.TruncationControl.accuracy(1e-3), out=tb[0])
    with pytest.raises(ValueError):
        htb.add(a, a, out=tb[0])


def test_concurrent_truncations_on_streams_match_serial(cuda_ok):
    """Several truncations in flight on separate streams (each with its own output buffer
    and workspace; the benchmark's pipelining) reproduce the serial result bit for bit,
    and cached graphs shared between streams are re-pointed only after their last launch."""
    import torch

    import paper_1708_03340_b200 as htb

    tree = htb.build_balanced_tree(8)
    x = htb.add(htb.gaussian_htensor(tree, 200, 20, 7), htb.gaussian_htensor(tree, 200, 20, 8))
    ctl = htb.TruncationControl.fixed_rank(20)
    ref = _arrays(htb.truncate(x, ctl))
    streams = [torch.cuda.Stream() for _ in range(3)]
    t0 = htb.truncate(x, ctl)
    outs = [htb.HTensor.empty(tree, *t0.host_layout()) for _ in range(4)]  # fewer than stream x buffer pairs
    main = torch.cuda.current_stream()
    done = []
    for i in range(24):
        s = streams[i % 3]
        s.wait_stream(main) if i < 3 else None
        with torch.cuda.stream(s):
            htb.truncate(x, ctl, out=outs[i % 4])
            ev = torch.cuda.Event()
            ev.record(s)
        done.append((ev, i % 4))
    for s in streams:
        main.wait_stream(s)
    torch.cuda.synchronize()
    for o in outs:
        for u, v in zip(_arrays(o), ref):
            np.testing.assert_array_equal(u, v)


def test_more_address_combinations_than_the_cache_run_eagerly(cuda_ok):
    """A caller cycling through more result buffers than the graph cache holds (24 per
    shape) must not pay a capture per call: warm graphs are never evicted, the overflow
    runs eagerly, and every result equals the eager one."""
    import paper_1708_03340_b200 as htb

    tree = htb.build_balanced_tree(4)
    x = htb.add(htb.gaussian_htensor(tree, 60, 7, 1), htb.gaussian_htensor(tree, 60, 7, 2), lazy=False)
    ctl = htb.TruncationControl.fixed_rank(6)
    htb.set_graph_mode(False)
    try:
        ref = _arrays(htb.truncate(x, ctl))
    finally:
        htb.set_graph_mode(True)
    first = htb.truncate(x, ctl)
    outs = [htb.HTensor.empty(tree, *first.host_layout()) for _ in range(30)]
    c0, _ = htb.graph_stats()
    for rnd in range(4):
        for o in outs:
            got = _arrays(htb.truncate(x, ctl, out=o))
            assert all(np.array_equal(p, q) for p, q in zip(got, ref))
    c1, r1 = htb.graph_stats()
    assert c1 - c0 <= 26, f"{c1 - c0} captures for 30 rotating buffers: the cache is thrashing"
