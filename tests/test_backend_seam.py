"""The solver plugin seam (reference solvers.py:28-106) on the host: GpuBackend and
ShardedBackend offer every method the reference's solvers call on ``backend.``,
with the reference SerialBackend's parameters.  When the reference source is
present (build container) both are read from it; elsewhere the list below, taken
from solvers.py, stands in.  (The device arithmetic behind the methods is covered
by the -m gpu tests, e.g. test_gpu_backend.py against the reference's own CG run.)"""

import inspect
import os
import re

import pytest

from paper_1708_03340_b200.backend import GpuBackend
from paper_1708_03340_b200.dist import ShardedBackend

REF_SOLVERS = "/root/reference/pkg/src/htucker/solvers.py"
# solvers.py:28-72 (SerialBackend) -- the seam's eleven methods and their parameters
SEAM = {"lift": ["tensor"], "retrieve": ["tensor"], "lift_operator": ["op"], "apply": ["op", "x"],
        "add": ["x", "y"], "scale": ["x", "alpha"], "truncate": ["x", "ctl"], "inner_product": ["x", "y"],
        "norm": ["x"], "leaf_map": ["x", "dim", "matrix"], "max_rank": ["x"]}


def _reference_seam():
    """Methods the reference solvers call on ``backend.`` and SerialBackend's parameters."""
    src = open(REF_SOLVERS).read()
    called = sorted(set(re.findall(r"backend\.([a-z_]+)\(", src)))
    body = src[src.index("class SerialBackend"):src.index("class DistBackend")]
    params = {m.group(1): [p.split(":")[0].strip() for p in m.group(2).split(",")[1:] if p.strip()]
              for m in re.finditer(r"def ([a-z_]+)\(self((?:, [^)]*)?)\)", body)}
    return called, params


@pytest.mark.parametrize("cls", [GpuBackend, ShardedBackend])
def test_backend_offers_the_seam(cls):
    if os.path.exists(REF_SOLVERS):
        called, params = _reference_seam()
        assert set(called) <= set(params), "every called method is part of SerialBackend"
        seam = {name: params[name] for name in called}
        assert set(seam) == set(SEAM)
    else:
        seam = SEAM
    for name, ref_params in seam.items():
        assert callable(getattr(cls, name, None)), f"{cls.__name__}.{name} missing"
        sig = inspect.signature(getattr(cls, name))
        ours = [p for p in sig.parameters if p != "self"]
        assert len(ours) >= len(ref_params), f"{cls.__name__}.{name}{sig} vs {ref_params}"
        required = [p for p, v in sig.parameters.items() if p != "self" and v.default is inspect.Parameter.empty
                    and v.kind in (v.POSITIONAL_ONLY, v.POSITIONAL_OR_KEYWORD)]
        assert len(required) <= len(ref_params), f"{cls.__name__}.{name} needs more arguments than the seam passes"
