"""CKVT trace files: the reference's binary trace format
(trace.hpp:227-367), read memory-mapped and shipped to the device KV store.

Format (trace.hpp:229-234): magic "CKVT", u32 version = 1, u32 n_layers,
n_heads, d, L, T (little endian); then per head, layer-major, the five
matrices prompt_keys [L,d], prompt_values [L,d], decode_queries [T,d],
decode_keys [T,d], decode_values [T,d] as little-endian float32 row-major;
then a u32-length-prefixed UTF-8 JSON object of string metadata.

`read_trace` validates like the reference (same checks, same ParseError
codes and messages) but does not copy the payload: every matrix is a view
into one np.memmap, so a multi-GB trace opens instantly and pages in as the
device upload reads it.  `write_trace` produces byte-identical files to the
reference's writer (tests/test_trace.py checks against the compiled
reference).  `to_device` rounds to bf16 (the device KV store)
and uploads K/V/Q for a Session or the sharded path.
"""
from __future__ import annotations

import json
import os
import struct
from dataclasses import dataclass, field
from enum import IntEnum

import numpy as np

from ._native import CkvError

MAGIC = b"CKVT"
VERSION = 1
MAX_TOTAL_FLOATS = 1 << 33  # trace.hpp:240
NAMES = ("prompt_keys", "prompt_values", "decode_queries", "decode_keys", "decode_values")


class ParseCode(IntEnum):
    """ParseError::Code (common.hpp:41-48)."""

    BadMagic = 0
    BadVersion = 1
    Truncated = 2
    DimOverflow = 3
    BadMetadata = 4
    TrailingData = 5


class ParseError(CkvError, ValueError):
    def __init__(self, code: ParseCode, msg: str):
        super().__init__(-1, msg)
        self.parse_code = code


class TraceIoError(CkvError, OSError):
    """IoError (common.hpp:33-36)."""

    def __init__(self, msg: str):
        super().__init__(-1, msg)


@dataclass
class HeadTrace:
    """trace.hpp:24-50 (arrays are float32 views)."""

    prompt_keys: np.ndarray
    prompt_values: np.ndarray
    decode_queries: np.ndarray
    decode_keys: np.ndarray
    decode_values: np.ndarray

    @property
    def d(self) -> int:
        return int(self.prompt_keys.shape[1])


@dataclass
class TraceBundle:
    """trace.hpp:52-82: traces are layer-major (index = layer * n_heads + head)."""

    n_layers: int
    n_heads: int
    traces: list = field(default_factory=list)
    metadata: dict = field(default_factory=dict)

    def at(self, layer: int, head: int) -> HeadTrace:
        return self.traces[layer * self.n_heads + head]

    def validate(self) -> None:
        """TraceBundle::validate / HeadTrace::validate (trace.hpp:36-49, 68-80)."""
        from ._native import ValidationError
        if self.n_layers == 0 or self.n_heads == 0:
            raise ValidationError(1, "TraceBundle: n_layers and n_heads must be >= 1")
        if len(self.traces) != self.n_layers * self.n_heads:
            raise ValidationError(1, "TraceBundle: trace count does not match n_layers * n_heads")
        f = self.traces[0]
        d, L, T = f.d, f.prompt_keys.shape[0], f.decode_queries.shape[0]
        for tr in self.traces:
            if (tr.d != d or tr.prompt_keys.shape[0] != L or tr.decode_queries.shape[0] != T):
                raise ValidationError(1, "TraceBundle: heads disagree on d/L/T")
            for name, rows in zip(NAMES, (L, L, T, T, T)):
                m = getattr(tr, name)
                if m.shape != (rows, d):
                    raise ValidationError(1, f"HeadTrace: bad shape for {name}")
                if not np.isfinite(m).all():
                    raise ValidationError(1, f"HeadTrace: non-finite values in {name}")


def read_trace(path: str, mmap: bool = True) -> TraceBundle:
    """read_trace (trace.hpp:305-367), memory-mapped."""
    try:
        size = os.path.getsize(path)
        fh = open(path, "rb")
    except OSError:
        raise TraceIoError(f"cannot open for reading: {path}")
    with fh:
        head = fh.read(28)
    if len(head) < 4:
        raise ParseError(ParseCode.Truncated, "trace file: truncated payload")
    if head[:4] != MAGIC:
        raise ParseError(ParseCode.BadMagic, "trace file: bad magic")
    if len(head) < 8:
        raise ParseError(ParseCode.Truncated, "trace file: truncated payload")
    version = struct.unpack_from("<I", head, 4)[0]
    if version != VERSION:
        raise ParseError(ParseCode.BadVersion, f"trace file: unsupported version {version}")
    if len(head) < 28:
        raise ParseError(ParseCode.Truncated, "trace file: truncated payload")
    n_layers, n_heads, d, L, T = struct.unpack_from("<5I", head, 8)
    if n_layers == 0 or n_heads == 0 or d == 0 or L == 0:
        raise ParseError(ParseCode.DimOverflow, "trace file: zero dimension in header")
    heads = n_layers * n_heads
    per_head = (L * 2 + T * 3) * d
    if heads > (1 << 24) or per_head > MAX_TOTAL_FLOATS or heads * per_head > MAX_TOTAL_FLOATS:
        raise ParseError(ParseCode.DimOverflow, "trace file: dimensions exceed supported size")
    payload = heads * per_head * 4
    if size < 28 + payload + 4:
        raise ParseError(ParseCode.Truncated, "trace file: truncated payload")
    if mmap:
        data = np.memmap(path, dtype="<f4", mode="r", offset=28, shape=(heads * per_head,))
    else:
        data = np.fromfile(path, dtype="<f4", count=heads * per_head, offset=28)
    with open(path, "rb") as fh:
        fh.seek(28 + payload)
        meta_len = struct.unpack("<I", fh.read(4))[0]
        meta = fh.read(meta_len)
        if len(meta) != meta_len:
            raise ParseError(ParseCode.Truncated, "trace file: truncated payload")
        # the reference parses the metadata before its trailing-byte check
        # (trace.hpp:353-365), so corrupt metadata wins over extra bytes
        try:
            md = json.loads(meta.decode("utf-8"))
            if not isinstance(md, dict) or not all(isinstance(v, str) for v in md.values()):
                raise ValueError
        except (ValueError, UnicodeDecodeError):
            raise ParseError(ParseCode.BadMetadata, "trace file: corrupt metadata block")
        if fh.read(1):
            raise ParseError(ParseCode.TrailingData, "trace file: trailing data")
    traces = []
    off = 0
    for _ in range(heads):
        mats = []
        for rows in (L, L, T, T, T):
            mats.append(data[off:off + rows * d].reshape(rows, d))
            off += rows * d
        traces.append(HeadTrace(*mats))
    return TraceBundle(n_layers, n_heads, traces, md)


def write_trace(bundle: TraceBundle, path: str) -> None:
    """write_trace (trace.hpp:268-303): byte-identical to the reference's."""
    bundle.validate()
    f = bundle.traces[0]
    try:
        fh = open(path, "wb")
    except OSError:
        raise TraceIoError(f"cannot open for writing: {path}")
    with fh:
        fh.write(MAGIC)
        fh.write(struct.pack("<6I", VERSION, bundle.n_layers, bundle.n_heads, f.d,
                             f.prompt_keys.shape[0], f.decode_queries.shape[0]))
        for tr in bundle.traces:
            for name in NAMES:
                fh.write(np.ascontiguousarray(getattr(tr, name), "<f4").tobytes())
        # nlohmann::json of a std::map: keys sorted, compact separators
        meta = json.dumps(dict(sorted(bundle.metadata.items())), separators=(",", ":"),
                          ensure_ascii=False).encode("utf-8")
        fh.write(struct.pack("<I", len(meta)))
        fh.write(meta)


def to_device(bundle: TraceBundle, device=None, layers=None, decode_kv: bool = False):
    """Round a trace to the device KV store (bf16) and upload it: returns
    (K, V) int16 bf16-bit tensors [units, L, d] and Q float32 [units, T, d]
    (bf16-representable), plus the decode keys / values [units, T, d] (bf16
    bits) with decode_kv; units in bundle order (layer-major), optionally a
    subset of layers.  The f32 -> bf16 rounding runs on the device
    (round-to-nearest-even, as SURVEY §8a N1's parity inputs)."""
    import torch
    dev = device or torch.device("cuda", torch.cuda.current_device())
    sel = [tr for i, tr in enumerate(bundle.traces)
           if layers is None or i // bundle.n_heads in layers]
    # one head at a time from the read-only map (a host copy per matrix)
    bf = lambda a: torch.from_numpy(np.array(a, dtype=np.float32)).to(dev).to(torch.bfloat16)
    K = torch.stack([bf(tr.prompt_keys).view(torch.int16) for tr in sel])
    V = torch.stack([bf(tr.prompt_values).view(torch.int16) for tr in sel])
    Q = torch.stack([bf(tr.decode_queries).float() for tr in sel])
    if not decode_kv:
        return K, V, Q
    dK = torch.stack([bf(tr.decode_keys).view(torch.int16) for tr in sel])
    dV = torch.stack([bf(tr.decode_values).view(torch.int16) for tr in sel])
    return K, V, Q, dK, dV
