"""CKVT trace I/O (trace.hpp:227-367).

The golden file tests/golden/synthetic_small.ckvt was written by the compiled
reference itself (tests/golden/make_trace_golden.py).  Our memory-mapped
reader must return the reference generator's matrices and metadata, our
writer must reproduce the file byte for byte, and corrupted files must fail
with the reference's ParseError codes (checked against the compiled
reference's read_trace when oracle/_ref is available)."""
import os
import struct

import numpy as np
import pytest

from paper_2412_03213_b200 import trace as T
from tests._inputs import port

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "synthetic_small.ckvt")
L_, T_, D_ = 48, 6, 128


def test_read_golden_matches_reference_generator():
    b = T.read_trace(GOLDEN)
    assert (b.n_layers, b.n_heads) == (2, 2)
    assert b.metadata == {"generator": "synthetic-mixture", "n_centers": "8", "seed": "7"}
    for layer in range(2):
        for h in range(2):
            tr = port().generate_head(port().mix_seed(7, layer, h), L_, T_)
            got = b.at(layer, h)
            for name in T.NAMES:
                assert np.array_equal(getattr(got, name), getattr(tr, name)), name
    assert isinstance(b.traces[0].prompt_keys.base, np.memmap) or \
        isinstance(b.traces[0].prompt_keys, np.memmap)


def test_write_is_byte_identical(tmp_path):
    b = T.read_trace(GOLDEN)
    out = tmp_path / "rt.ckvt"
    T.write_trace(b, str(out))
    assert out.read_bytes() == open(GOLDEN, "rb").read()
    b2 = T.read_trace(str(out), mmap=False)
    assert all(np.array_equal(getattr(x, n), getattr(y, n))
               for x, y in zip(b.traces, b2.traces) for n in T.NAMES)


def _corrupt(tmp_path, name, fn):
    raw = bytearray(open(GOLDEN, "rb").read())
    raw = fn(raw)
    p = tmp_path / name
    p.write_bytes(bytes(raw))
    return str(p)


CASES = {
    "bad_magic": (lambda r: b"CKVX" + r[4:], T.ParseCode.BadMagic),
    "bad_version": (lambda r: r[:4] + struct.pack("<I", 2) + r[8:], T.ParseCode.BadVersion),
    "zero_dim": (lambda r: r[:12] + struct.pack("<I", 0) + r[16:], T.ParseCode.DimOverflow),
    "huge_dim": (lambda r: r[:20] + struct.pack("<I", 1 << 30) + r[24:], T.ParseCode.DimOverflow),
    "truncated": (lambda r: r[:-100], T.ParseCode.Truncated),
    "short_header": (lambda r: r[:10], T.ParseCode.Truncated),
    "trailing": (lambda r: r + b"x", T.ParseCode.TrailingData),
    "bad_meta": (lambda r: r[:-3] + b"}}}", T.ParseCode.BadMetadata),
    # corrupt metadata AND trailing bytes: the reference reports the metadata
    "bad_meta_trailing": (lambda r: r[:-3] + b"}}}" + b"xy", T.ParseCode.BadMetadata),
}


@pytest.mark.parametrize("case", sorted(CASES))
def test_corrupt_files_raise_reference_codes(tmp_path, case):
    fn, code = CASES[case]
    p = _corrupt(tmp_path, case + ".ckvt", fn)
    with pytest.raises(T.ParseError) as ei:
        T.read_trace(p)
    assert ei.value.parse_code == code
    from oracle.oracle import Oracle, ref_available
    if ref_available():
        assert Oracle("reference").lib.ref_read_trace_status(p.encode()) == 1 + int(code)


def test_missing_file_is_io_error(tmp_path):
    with pytest.raises(T.TraceIoError):
        T.read_trace(str(tmp_path / "nope.ckvt"))
