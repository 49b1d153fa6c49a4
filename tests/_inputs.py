"""Seeded synthetic inputs (reference generator, trace.hpp:134-198, through
the C oracle port), rounded to bf16-representable f32."""
from __future__ import annotations

import numpy as np

from oracle.oracle import Oracle, to_bf16_representable

_port = None


def port() -> Oracle:
    global _port
    if _port is None:
        _port = Oracle("port")
    return _port


def head(seed: int, layer: int, kv_head: int, L: int, T: int = 64):
    p = port()
    tr = p.generate_head(p.mix_seed(seed, layer, kv_head), L, T)
    return dict(K=to_bf16_representable(tr.prompt_keys), V=to_bf16_representable(tr.prompt_values),
                Q=to_bf16_representable(tr.decode_queries),
                dK=to_bf16_representable(tr.decode_keys),
                dV=to_bf16_representable(tr.decode_values))


def bf16_bits(x: np.ndarray) -> np.ndarray:
    """bf16-representable f32 -> uint16 bit patterns."""
    return (np.ascontiguousarray(x, np.float32).view(np.uint32) >> 16).astype(np.uint16)
