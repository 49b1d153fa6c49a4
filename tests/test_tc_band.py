"""The tensor-core assignment's error band (ckv_assign_tc.cu header), checked
numerically on the host: for fp16 operands h(k), h(dir) (round to nearest,
saturated, flushed below the normal range, as f32_to_f16_tc) and fp32
accumulation, every score is within half the band of the exact
dot_f64(k, dir) the reference ranks by (clustering.hpp:104-115), so the exact
argmax is always among the in-band candidates.

band = kn (2 eps_u + 2^-13) 1.01 + 2.02 kerr_u, kn = |k| + |k - h(k)|,
eps_u = max_c |dir_c - h(dir_c)|, kerr_u = max_k |k - h(k)|.
"""
import numpy as np
import pytest


def to_bf16(x):
    u = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    r = ((u >> 16) & 1) + 0x7FFF
    return ((u + r) >> 16 << 16).astype(np.uint32).view(np.float32)


def h16(x):
    """f32_to_f16_tc (ckv_common.cuh): RN, saturate to +-65504, flush subnormals."""
    x = np.clip(np.asarray(x, np.float32), -65504.0, 65504.0)
    h = x.astype(np.float16)
    h[np.abs(h) < np.float16(2.0 ** -14)] = 0
    return h.astype(np.float32)


def band_check(keys, dirs, rng):
    k16, d16 = h16(keys), h16(dirs)
    eps = np.sqrt(((dirs.astype(np.float64) - d16) ** 2).sum(1)).max()
    kerr_k = np.sqrt(((keys.astype(np.float64) - k16) ** 2).sum(1))
    kerr = kerr_k.max()
    kn = np.sqrt((keys.astype(np.float64) ** 2).sum(1)) + kerr_k
    band = kn * (2 * eps + 2.0 ** -13) * 1.01 + 2.02 * kerr
    exact = keys.astype(np.float64) @ dirs.astype(np.float64).T
    # fp32 accumulation of the (exact) products in a random order per key
    prod = k16[:, None, :].astype(np.float64) * d16[None, :, :].astype(np.float64)
    perm = rng.permutation(keys.shape[1])
    acc = np.zeros(exact.shape, np.float32)
    for j in perm:
        acc = (acc + prod[:, :, j].astype(np.float32)).astype(np.float32)
    err = np.abs(acc.astype(np.float64) - exact)
    assert np.all(err <= 0.5 * band[:, None]), float((err / band[:, None]).max())
    # the exact argmax is in band of the computed max
    M = acc.max(1)
    best = exact.argmax(1)
    assert np.all(acc[np.arange(len(best)), best] >= M - band)
    return band


def unit_dirs(rng, c):
    d = rng.standard_normal((c, 128)).astype(np.float32)
    return (d / np.linalg.norm(d, axis=1, keepdims=True)).astype(np.float32)


@pytest.mark.parametrize("scale", [1e-3, 1.0, 30.0])
def test_band_bounds_scores(scale):
    rng = np.random.default_rng(7)
    keys = to_bf16(rng.standard_normal((64, 128)) * scale)
    band_check(keys, unit_dirs(rng, 96), rng)


def test_band_tiny_and_huge_keys():
    """Keys outside fp16's normal range: the conversion error enters the band."""
    rng = np.random.default_rng(3)
    keys = rng.standard_normal((32, 128)).astype(np.float32)
    keys[0] *= 1e-6      # subnormal in fp16: flushed
    keys[1, :4] = 1e5    # beyond 65504: saturated
    keys = to_bf16(keys)
    band = band_check(keys, unit_dirs(rng, 64), rng)
    assert band[1] > band[2]


def test_fp16_band_narrower_than_bf16():
    """The reason for fp16 operands: a ~6x narrower band than bf16's."""
    rng = np.random.default_rng(5)
    dirs = unit_dirs(rng, 409)
    eps16 = np.sqrt(((dirs.astype(np.float64) - h16(dirs)) ** 2).sum(1)).max()
    eps_bf = np.sqrt(((dirs.astype(np.float64) - to_bf16(dirs)) ** 2).sum(1)).max()
    b16 = 2 * eps16 + 2.0 ** -13
    bbf = 2 * eps_bf + 2.0 ** -13
    assert bbf / b16 > 4.0
