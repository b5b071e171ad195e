"""The interval slab test of the packet traversal (cast.cu `pslab_axis` /
`pslab_test`, DESIGN.md §8 "Interval packets") is conservative: for tiles
of 4x8 pinhole rays sharing an origin and random boxes, whenever any ray's
own slab test (box widened by delta) passes, the test of the box widened
by 2 delta against the per-axis interval of the tile's directions passes
too -- including tiles whose direction interval contains 0 on an axis.
Checked in FP64 with numpy (the claim is about the formula; the kernel's
FP32 rounding is covered by the second delta)."""
import numpy as np


def ray_hits(o, d, lo, hi, delta, U):
    with np.errstate(divide="ignore"):
        inv = 1.0 / d
    a = (lo - (o + delta)) * inv
    b = (hi - (o - delta)) * inv
    tn = max(np.minimum(a, b).max(), 0.0)
    tf = min(np.maximum(a, b).min(), U)
    return tn <= tf


def interval_hits(o, dmin, dmax, lo, hi, dp, U):
    near, far = [], []
    for ax in range(3):
        l, h = dmin[ax], dmax[ax]
        if l > 0 or h < 0:
            i0, i1 = 1.0 / l, 1.0 / h
        else:
            i0, i1 = 1.0 / min(l, -1e-30), 1.0 / max(h, 1e-30)
        a = lo[ax] - (o[ax] + dp)
        b = hi[ax] - (o[ax] - dp)
        p = (a * i0, a * i1, b * i0, b * i1)
        if (i0 < 0) != (i1 < 0):
            near.append(max(a * i1, b * i0))
            far.append(np.inf)
        else:
            near.append(min(p))
            far.append(max(p))
    return max(max(near), 0.0) <= min(min(far), U)


def test_interval_slab_is_conservative():
    rng = np.random.default_rng(0)
    fx, W, H = 252.907, 480, 270
    hits = false_pos = 0
    for trial in range(6000):
        u0, v0 = rng.integers(0, W - 4), rng.integers(0, H - 8)
        yaw, pitch = rng.uniform(0, 2 * np.pi), rng.uniform(-0.2, 0.2)
        if trial % 3 == 0:  # tiles straddling the image centre lines: intervals containing 0
            u0, v0, yaw, pitch = W // 2 - 2, H // 2 - 4, 0.0, 0.0
        cy, sy, cp, sp = np.cos(yaw), np.sin(yaw), np.cos(pitch), np.sin(pitch)
        R = np.array([[cy, -sy, 0], [sy, cy, 0], [0, 0, 1]]) @ np.array([[cp, 0, sp], [0, 1, 0], [-sp, 0, cp]])
        o = np.array([rng.uniform(-8, 8), rng.uniform(-8, 8), rng.uniform(1, 2)])
        ds = np.array([R @ np.array([1.0, -(u0 + k % 4 + 0.5 - W / 2) / fx, -(v0 + k // 4 + 0.5 - H / 2) / fx])
                       for k in range(32)])
        c = o + ds[13] * rng.uniform(-2, 12) + rng.normal(0, 0.3, 3)
        e = np.abs(rng.normal(0, 0.3, 3)) + rng.choice([1e-3, 0.05])
        lo, hi = c - e, c + e
        delta, U = 1e-4, rng.choice([10.0, rng.uniform(0.5, 10)])
        any_ray = any(ray_hits(o, d, lo, hi, delta, U) for d in ds)
        iv = interval_hits(o, ds.min(0), ds.max(0), lo, hi, 2 * delta, U)
        assert iv or not any_ray, (trial, lo, hi)
        hits += any_ray
        false_pos += iv and not any_ray
    assert hits > 500
    assert false_pos < 0.05 * hits  # and it still culls
