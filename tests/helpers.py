"""Shared test helpers: bitwise comparison with NaN == NaN."""
import numpy as np


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def assert_bitwise(got, want, what=""):
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    assert got.shape == want.shape, (what, got.shape, want.shape)
    both_nan = np.isnan(got) & np.isnan(want)
    same = (bits(got) == bits(want)) | both_nan
    if not same.all():
        idx = np.argwhere(~same)[:5]
        detail = [(tuple(int(i) for i in ix), float(got[tuple(ix)]), float(want[tuple(ix)])) for ix in idx]
        raise AssertionError(f"{what}: {int((~same).sum())} of {same.size} values differ, first {detail}")


def max_rel_err(got, want):
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    fin = np.isfinite(want) & np.isfinite(got)
    if not fin.any():
        return 0.0
    d = np.abs(got[fin] - want[fin]) / np.maximum(np.abs(want[fin]), np.finfo(float).tiny)
    return float(d.max())
