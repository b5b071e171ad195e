"""Test helpers: turn scenegen sensor dicts into oracle ray specs, and the
parity comparison rules of SURVEY.md §8(c) (written once, used by every
GPU parity test).  Contains no ray-casting arithmetic."""
from __future__ import annotations

import numpy as np

import oracle


def oracle_rays(sensor: dict, kind: str = "depth") -> dict:
    """scenegen sensor dict -> oracle.cast ``rays`` dict."""
    if sensor["kind"] == "pinhole":
        d = dict(model=oracle.PINHOLE, kind=oracle.DEPTH if kind == "depth" else oracle.RANGE,
                 poses=sensor["poses"], max_range=sensor["max_range"])
        d.update(sensor["cam"])
        return d
    if sensor["kind"] == "beams":
        return dict(model=oracle.BEAMS, beams=sensor["beams"], poses=sensor["poses"],
                    max_range=sensor["max_range"])
    return dict(model=oracle.RAYS, orig=sensor["orig"], dir=sensor["dir"],
                max_range=sensor["max_range"])


# SURVEY.md §8(c) / BASELINE.json north_star: |d| <= max(1e-5 m, 1e-6 * ref)
DIST_ABS = 1e-5
DIST_REL = 1e-6


def amb_bound(n: int, frac: float = 2e-4, floor: int = 8) -> int:
    """Default upper bound on the rays a parity test may exclude as ambiguous:
    near-ties of generic workloads are rare (measured: 2 of 388 800 c2
    stereo rays), so a flag that fired on every silhouette or edge ray would
    exceed it."""
    return max(floor, int(frac * n))


def compare(ref: "oracle.OracleResult", dist, seg, face, what="", max_amb=None, max_graze=None):
    """Apply the parity rules; returns a dict of counts, raises on failure.

    distance: every ray within max(1e-5, 1e-6*ref) of the oracle's FP64 t;
    on a tie ray (AMB_TIE) the other tied candidate's t (ref.t2, within
    1e-5 m of t by construction) is accepted too, and on a graze ray
    (AMB_GRAZE: a near candidate within FP64 rounding of its triangle's
    boundary in front of the winner, reading R24) the grazed
    candidate's t.
    seg / face: bit-exact on every ray that is not ambiguous (oracle AMB_*).
    Bounds: at most ``max_amb`` ambiguous rays (default amb_bound(n)) and at
    most ``max_graze`` graze rays (default max(2, 1e-5 n)) -- tests that aim
    rays at edges on purpose pass their own bounds.
    """
    dist = np.asarray(dist, np.float64).reshape(-1)
    n = len(dist)
    tol = np.maximum(DIST_ABS, DIST_REL * np.abs(ref.t64))
    err = np.abs(dist - ref.t64)
    tie = (ref.amb & oracle.AMB_TIE) != 0
    graze = (ref.amb & oracle.AMB_GRAZE) != 0
    with np.errstate(invalid="ignore"):
        tol2 = np.maximum(DIST_ABS, DIST_REL * np.abs(ref.t2))
        # the oracle only flags a tie whose other candidate is within AMB_EPS
        assert np.all(~tie | graze | (np.abs(ref.t2 - ref.t64) <= oracle.AMB_EPS)), f"{what}: tie t2 too far"
        alt = (tie | graze) & (np.abs(dist - ref.t2) <= tol2)
    bad_d = np.nonzero((err > tol) & ~alt)[0]
    amb = ref.amb != 0
    out = dict(n=n, ambiguous=int(amb.sum()), ties=int(tie.sum()), grazes=int(graze.sum()),
               graze_alt=int((graze & alt & (err > tol)).sum()),
               max_err=float(err.max()) if len(err) else 0.0)
    msgs = []
    lim_amb = amb_bound(n) if max_amb is None else max_amb
    lim_graze = max(2, int(1e-5 * n)) if max_graze is None else max_graze
    if out["ambiguous"] > lim_amb:
        msgs.append(f"{what}: {out['ambiguous']} ambiguous rays of {n} exceed the bound {lim_amb}")
    if out["grazes"] > lim_graze:
        msgs.append(f"{what}: {out['grazes']} graze rays of {n} exceed the bound {lim_graze}")
    if len(bad_d):
        i = bad_d[0]
        msgs.append(f"{what}: {len(bad_d)} distance mismatches; first #{i}: gpu={dist[i]!r} "
                    f"oracle={ref.t64[i]!r} seg {seg.reshape(-1)[i] if seg is not None else '-'}"
                    f"/{ref.seg[i]} face {face.reshape(-1)[i] if face is not None else '-'}/{ref.face[i]} "
                    f"amb={ref.amb[i]} t2={ref.t2[i]!r}")
    for name, got, exp in (("seg", seg, ref.seg), ("face", face, ref.face)):
        if got is None:
            continue
        got = np.asarray(got).reshape(-1)
        bad = np.nonzero((got != exp) & ~amb)[0]
        out[f"{name}_mismatch"] = int(len(bad))
        out[f"{name}_diff_ambiguous"] = int(((got != exp) & amb).sum())
        if len(bad):
            i = bad[0]
            msgs.append(f"{what}: {len(bad)} {name} mismatches; first #{i}: gpu={got[i]} "
                        f"oracle={exp[i]} dist gpu={dist[i]!r} oracle={ref.t64[i]!r} "
                        f"t2={ref.t2[i]!r} amb={ref.amb[i]}")
    if msgs:
        raise AssertionError("\n".join(msgs))
    return out


def valid_compare(ref: "oracle.OracleResult", valid, what="", max_amb=None):
    """Stereo shadow mask (f2) parity: bit-exact on every ray the oracle does
    not flag ambiguous, with the ambiguous count bounded (amb_bound(n) by
    default).  Returns the number of shadowed (invalid) pixels."""
    valid = np.asarray(valid).reshape(-1)
    amb = ref.amb != 0
    n_amb = int(amb.sum())
    lim = amb_bound(len(valid)) if max_amb is None else max_amb
    assert n_amb <= lim, f"{what}: {n_amb} ambiguous rays of {len(valid)} exceed the bound {lim}"
    bad = np.nonzero((valid != ref.valid) & ~amb)[0]
    assert len(bad) == 0, f"{what}: {len(bad)} valid mismatches, first {bad[:5]}"
    return int((ref.valid == 0).sum())


def compare_extras(ref: "oracle.OracleResult", normal=None, bary=None, point=None, face=None, what=""):
    """Per-hit channels on every ray whose face equals the oracle's (all
    non-ambiguous rays, by compare()): normal within 1e-6 per component,
    barycentrics within 1e-6 absolute, point within max(1e-5, 1e-6 |p|)."""
    same = np.ones(len(ref.t64), bool) if face is None else (np.asarray(face).reshape(-1) == ref.face)
    msgs = []
    if normal is not None:
        n = np.asarray(normal, np.float64).reshape(-1, 3)
        err = np.abs(n - ref.normal).max(1)
        bad = np.nonzero(same & (err > 1e-6))[0]
        if len(bad):
            msgs.append(f"{what}: {len(bad)} normal mismatches, first {bad[0]}: {n[bad[0]]} vs {ref.normal[bad[0]]}")
    if bary is not None:
        b = np.asarray(bary, np.float64).reshape(-1, 2)
        err = np.abs(b - ref.bary).max(1)
        bad = np.nonzero(same & (err > 1e-6))[0]
        if len(bad):
            msgs.append(f"{what}: {len(bad)} bary mismatches, first {bad[0]}: {b[bad[0]]} vs {ref.bary[bad[0]]}")
    if point is not None:
        p = np.asarray(point, np.float64).reshape(-1, 3)
        err = np.abs(p - ref.point).max(1)
        tol = np.maximum(DIST_ABS, DIST_REL * np.abs(ref.point).max(1))
        bad = np.nonzero(same & (err > tol))[0]
        if len(bad):
            msgs.append(f"{what}: {len(bad)} point mismatches, first {bad[0]}: {p[bad[0]]} vs {ref.point[bad[0]]}")
    if msgs:
        raise AssertionError("\n".join(msgs))
    return int(same.sum())


# SURVEY.md §8(c) "Full-scale certificate": the reported hit lies on the
# reported face within the 1e-5 m parity band.
CERT_BAND = 1e-5


def certify_all(sc, sensor, kind, dist, seg, face, what="", env_chunk=64):
    """Certificate of EVERY ray of a full-size cast: for
    each hit, the oracle's FP64 plane-hit t of the reported face equals the
    reported distance within the parity tolerance, the hit lies on that face
    (within CERT_BAND), and seg is that face's label; each miss reports
    max_range, -1, -1.  Optimality (no closer face) is checked by oracle.cast
    on samples.  Returns the number of certified hits."""
    rays = oracle_rays(sensor, kind)
    n_env = len(sc.env_off) - 1
    per_env = len(dist) // n_env
    max_range = np.float32(sensor["max_range"])
    hits = 0
    for e0 in range(0, n_env, env_chunk):
        e1 = min(n_env, e0 + env_chunk)
        q = np.arange(e0 * per_env, e1 * per_env, dtype=np.int64)
        d, s, f = dist[q].astype(np.float64), seg[q], face[q]
        miss = f < 0
        bad = np.nonzero(miss & ((dist[q] != max_range) | (s != -1)))[0]
        assert len(bad) == 0, f"{what}: miss #{q[bad[0]]} reports {dist[q][bad[0]]!r}/{s[bad[0]]}"
        t_face, outside, label = oracle.certify(sc, rays, f, query=q)
        h = ~miss
        tol = np.maximum(DIST_ABS, DIST_REL * np.abs(t_face))
        with np.errstate(invalid="ignore"):
            bad_t = np.nonzero(h & ~(np.abs(d - t_face) <= tol))[0]
            bad_in = np.nonzero(h & ~(outside <= CERT_BAND))[0]
            bad_rng = np.nonzero(h & ~((t_face > 0) & (t_face <= max_range + DIST_ABS)))[0]
        bad_seg = np.nonzero(h & (label != s))[0]
        for name, b, info in (("distance", bad_t, t_face), ("on-face", bad_in, outside),
                              ("range", bad_rng, t_face), ("label", bad_seg, label)):
            if len(b):
                i = b[0]
                raise AssertionError(f"{what}: {len(b)} {name} certificate failures; first ray "
                                     f"{q[i]}: dist={d[i]!r} face={f[i]} seg={s[i]} oracle={info[i]!r}")
        hits += int(h.sum())
    return hits
