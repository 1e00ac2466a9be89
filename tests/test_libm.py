"""The hot path's transcendentals are glibc's, bit for bit.

The reference calls std::sin / cos / log / atan2 / hypot (glibc 2.39, FMA
ifunc builds on these hosts) in Box-Muller (rng.hpp:47-61), the Shoemake
quaternion (rng.hpp:66-76), FK (hand.cpp:286-288), rotation_between
(geometry.hpp:129-143) and the friction projection (wrench.cpp:96).
paper_2511_07418_b200/csrc/lg_libm.h restates those algorithms; the oracle
(CPU) and the device (GPU) both use it.  Every argument set below covers the
ranges the pipeline produces plus random bit patterns.
"""
import math

import numpy as np
import pytest

from oracle import orc_py as orc


def _args(fn, n, seed):
    rng = np.random.default_rng(seed)
    if fn in ("sin", "cos"):
        parts = [rng.uniform(-1e-7, 1e-7, n // 8), rng.uniform(-0.13, 0.13, n // 8),
                 rng.uniform(-0.9, 0.9, n // 8), rng.uniform(-2.5, 2.5, n // 8),
                 rng.uniform(0, 2 * math.pi, n // 4),  # Box-Muller / roll phases
                 rng.uniform(-50, 50, n // 8), rng.uniform(-1e6, 1e6, n // 8)]
        return np.concatenate(parts), None
    if fn == "log":
        u = (rng.integers(0, 2 ** 53, n, dtype=np.uint64) >> np.uint64(0)).astype(np.float64) * 2.0 ** -53
        u = np.maximum(u, 1e-300)  # rng.hpp:54
        near1 = rng.uniform(0.9, 1.1, n // 4)
        bits = rng.integers(0, 0x7FF0000000000000, n // 4, dtype=np.int64).view(np.float64)
        return np.concatenate([u, near1, bits]), None
    if fn == "atan2":
        t = rng.uniform(0, math.pi, n // 2)
        s = np.abs(np.sin(t)) * rng.uniform(0.5, 2, n // 2)
        c = np.cos(t) * rng.uniform(0.5, 2, n // 2)
        y2, x2 = rng.uniform(-10, 10, n // 2), rng.uniform(-10, 10, n // 2)
        y2[::3] *= 1e-9
        x2[1::3] *= 1e-9
        return np.concatenate([s, y2]), np.concatenate([c, x2])
    x, y = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    y[::3] *= 1e-6
    return x, y


@pytest.mark.parametrize("fn", ["sin", "cos", "log", "atan2", "hypot"])
def test_oracle_libm_is_glibc_bit_for_bit(fn):
    x, y = _args(fn, 2_000_000, 1)
    got = orc.libm(fn, x, y)
    ref = orc.glibc(fn, x, y)
    bad = np.flatnonzero(got.view(np.int64) != ref.view(np.int64))
    assert bad.size == 0, (fn, bad.size, x[bad[:3]], got[bad[:3]], ref[bad[:3]])


@pytest.mark.parametrize("fn", ["sin", "cos", "log"])
def test_glibc_helper_is_python_math(fn):
    """orc.glibc really is the host libm: Python's math module calls it too."""
    x, _ = _args(fn, 4000, 2)
    ref = np.array([getattr(math, fn)(v) if (fn != "log" or v > 0) else -math.inf for v in x])
    assert np.array_equal(orc.glibc(fn, x).view(np.int64), ref.view(np.int64))


@pytest.mark.gpu
@pytest.mark.parametrize("fn", ["sin", "cos", "log", "atan2", "hypot"])
def test_device_libm_is_glibc_bit_for_bit(ctx, fn):
    import paper_2511_07418_b200 as lg
    x, y = _args(fn, 4_000_000, 3)
    got = lg.api.libm_eval(ctx, fn, x, y)
    ref = orc.glibc(fn, x, y)
    bad = np.flatnonzero(got.view(np.int64) != ref.view(np.int64))
    assert bad.size == 0, (fn, bad.size, x[bad[:3]], got[bad[:3]], ref[bad[:3]])


def test_hypot_exceeds_is_glibc_hypot_gt_cap():
    """The friction-disc test hypot(x, y) > cap (wrench.cpp:96-104) decided
    through the squared-norm bound == glibc's hypot compared with cap, on
    random pairs and caps placed at, one ulp around and 2^-44 around the
    glibc value (where the bound must defer to the exact hypot)."""
    rng = np.random.default_rng(11)
    n = 400_000
    x = rng.normal(size=n) * 10.0 ** rng.uniform(-6, 2, size=n)
    y = rng.normal(size=n) * 10.0 ** rng.uniform(-6, 2, size=n)
    h = orc.glibc("hypot", x, y)
    pick = rng.integers(0, 7, size=n)
    cap = np.select([pick == 0, pick == 1, pick == 2, pick == 3, pick == 4, pick == 5],
                    [h, np.nextafter(h, 0), np.nextafter(h, np.inf), h * (1 + 2 ** -44),
                     h * (1 - 2 ** -44), h * rng.uniform(0.5, 2, size=n)], h * 0.0)
    got = orc.hypot_exceeds(x, y, cap)
    assert np.array_equal(got, h > cap)
