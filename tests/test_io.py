"""HT01 interchange (reference format.py:467-553) against bytes the reference itself
wrote (tests/golden/io.npz, made by tests/golden/make_golden.py::golden_io), plus the
reference's ParseError cases.  Host-only: the arrays live in a CPU arena."""

import struct

import numpy as np
import pytest

from tests.goldens import load


def _x():
    import paper_1708_03340_b200 as htb

    z = load("io.npz")
    return htb, z, z["blob"].tobytes()


def test_deserialize_reference_bytes_then_serialize_bit_exact():
    htb, z, blob = _x()
    x = htb.deserialize(blob, device="cpu")
    assert x.shape == (4, 5, 3, 6, 2)
    for t in range(9):
        assert np.array_equal(np.asarray(x.node_array(t)), z[f"x/{t}"])
    assert htb.serialize(x) == blob
    assert htb.serialized_size(x) == len(blob)


@pytest.mark.parametrize("cut,offset", [(3, 0), (10, 10), (40, 40), (-8, 1072)])
def test_parse_errors_carry_offsets(cut, offset):
    htb, _, blob = _x()
    with pytest.raises(htb.ParseError) as e:
        htb.deserialize(blob[:cut], device="cpu")
    assert e.value.offset == offset


def test_parse_errors_magic_dim_root_rank_trailing():
    htb, _, blob = _x()
    with pytest.raises(htb.ParseError) as e:
        htb.deserialize(b"HT02" + blob[4:], device="cpu")
    assert e.value.offset == 0
    with pytest.raises(htb.ParseError) as e:
        htb.deserialize(blob[:4] + struct.pack("<I", 1) + blob[8:], device="cpu")
    assert e.value.offset == 4
    bad_root = bytearray(blob)
    bad_root[16 + 8 * 5:16 + 8 * 5 + 8] = struct.pack("<Q", 2)
    with pytest.raises(htb.ParseError):
        htb.deserialize(bytes(bad_root), device="cpu")
    with pytest.raises(htb.ParseError) as e:
        htb.deserialize(blob + b"\0" * 8, device="cpu")
    assert e.value.offset == len(blob)
    assert issubclass(htb.ParseError, ValueError)
