"""Pins for the CPU oracle (-m "not gpu").

The oracle (oracle/oracle.c) is checked here against things other than
itself: closed forms, analytic geometry, invariants and an independent
Moller-Trumbore brute force written in numpy.  Each test names the passage
or DESIGN.md reading it pins.  A plausible mistake in the oracle (dropped
term, wrong sign, transposed pose, wrong face numbering, wrong tie rule,
wrong range/depth scaling) fails at least one of these.
"""
from __future__ import annotations

import math
import os

import numpy as np
import pytest

import oracle
import scenegen as sg

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def cast_pinhole(sc, cam, poses, kind=oracle.DEPTH, max_range=10.0, **kw):
    rays = dict(model=oracle.PINHOLE, kind=kind, poses=poses, max_range=max_range, **cam)
    return oracle.cast(sc, rays, **kw)


def cast_rays(sc, orig, dirs, max_range=100.0, **kw):
    return oracle.cast(sc, dict(model=oracle.RAYS, orig=orig, dir=dirs, max_range=max_range), **kw)


def quad_mesh(size=100.0, name="quad"):
    """Square in the plane x = 0 (normal +x), side `size`."""
    h = size / 2
    v = np.asarray([[0, -h, -h], [0, h, -h], [0, h, h], [0, -h, h]], np.float32)
    return sg.Mesh(name, v, np.asarray([[0, 1, 2], [0, 2, 3]], np.int32))


def _golden_c1():
    vals = {}
    with open(os.path.join(GOLDEN, "c1_camera.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            k, v = line.split(None, 1)
            vals[k] = v.strip()
    return vals


# --------------------------------------------------------------------------
# closed forms
# --------------------------------------------------------------------------

def test_c1_worked_example_golden():
    """SURVEY.md §8(c) config-1 worked example (tests/golden/c1_camera.txt)."""
    g = _golden_c1()
    sc, s = sg.config1()
    d = cast_pinhole(sc, s["cam"], s["poses"], oracle.DEPTH)
    r = cast_pinhole(sc, s["cam"], s["poses"], oracle.RANGE)
    depth = d.t64.reshape(16, 16)
    rng_ = r.t64.reshape(16, 16)
    hit = np.zeros((16, 16), bool)
    hit[6:10, 6:10] = True
    assert np.all(depth[hit] == float(g["depth"]))
    assert np.all(depth[~hit] == float(g["miss_distance"]))
    assert np.all(d.seg.reshape(16, 16)[hit] == int(g["label"]))
    assert np.all(d.seg.reshape(16, 16)[~hit] == -1)
    assert np.all(d.face.reshape(16, 16)[~hit] == -1)
    # the near face is the cube's -x side = faces 0, 1 of box_mesh
    assert set(np.unique(d.face.reshape(16, 16)[hit])) <= {0, 1}
    want = {1: float(g["range_|x'|=1/16_|y'|=1/16"]), 3: float(g["range_|x'|=1/16_|y'|=3/16"]),
            9: float(g["range_|x'|=3/16_|y'|=3/16"])}
    for v in range(6, 10):
        for u in range(6, 10):
            a, b = abs(2 * u - 15), abs(2 * v - 15)  # 1 or 3 (in 1/16 units)
            assert abs(rng_[v, u] - want[a * b]) < 1e-9, (u, v)
    # the 4 pixels on the split diagonal of the near face are exact ties
    amb = d.amb.reshape(16, 16)
    assert amb[hit].astype(bool).sum() == 4
    assert np.all(amb[~hit] == 0)


@pytest.mark.parametrize("dist", [1.5, 3.7, 9.25])
def test_plane_depth_constant_range_over_cos(dist):
    """Camera facing a plane at distance d: depth = d at every pixel, range =
    d / cos(theta) (north_star)."""
    dist = float(np.float32(dist))  # the plane position is an FP32 input
    cam = sg.pinhole(40, 30, 87.0)
    sc = sg.assemble([quad_mesh()], [[(0, 7, sg.make_T(np.eye(3), (dist, 0, 0)))]])
    poses = sg.identity_poses(1)
    d = cast_pinhole(sc, cam, poses, oracle.DEPTH, max_range=100.0)
    r = cast_pinhole(sc, cam, poses, oracle.RANGE, max_range=100.0)
    assert np.all(np.abs(d.t64 - dist) < 1e-12)
    # cos(theta) between the optical axis and the pixel ray, from the angle
    u = np.arange(cam["W"]) + 0.5 - cam["cx"]
    v = np.arange(cam["H"]) + 0.5 - cam["cy"]
    V, U = np.meshgrid(v, u, indexing="ij")
    ax = np.arctan2(np.hypot(U / cam["fx"], V / cam["fy"]), 1.0)
    assert np.allclose(r.t64.reshape(cam["H"], cam["W"]), dist / np.cos(ax), rtol=0, atol=1e-12)
    assert np.all(d.seg == 7)


def test_plane_rotated_sensor_and_scene():
    """Same plane pin with the pair (plane, camera) under a random rigid
    motion: depth stays d within FP32 input rounding."""
    rng = np.random.default_rng(5)
    cam = sg.pinhole(32, 24, 70.0)
    R = sg.random_rotation(rng)
    p = rng.uniform(-5, 5, 3)
    dist = 4.0
    Tq = sg.make_T(R, R @ np.asarray([dist, 0, 0]) + p)
    sc = sg.assemble([quad_mesh()], [[(0, 1, Tq)]])
    poses = sg.make_T(R, p)[None, None]
    d = cast_pinhole(sc, cam, poses, oracle.DEPTH)
    assert np.all(np.abs(d.t64 - dist) < 2e-5)
    assert np.all(d.seg == 1)


def test_cube_slab_analytic():
    """Axis-aligned cube: slab-method t and entry side."""
    rng = np.random.default_rng(11)
    lo, hi = np.asarray([1.0, -0.5, -0.25]), np.asarray([2.0, 0.75, 0.5])
    box = sg.box_mesh("box", lo, hi)
    sc = sg.assemble([box], [[(0, 3, sg.make_T(np.eye(3), (0, 0, 0)))]])
    n = 4000
    o = rng.uniform(-3, 4, (n, 3)).astype(np.float32)
    target = rng.uniform(lo - 0.2, hi + 0.2, (n, 3))
    d = (target - o).astype(np.float32)
    res = cast_rays(sc, o[None], d[None])
    o64, d64 = o.astype(np.float64), d.astype(np.float64)
    with np.errstate(divide="ignore", invalid="ignore"):
        t0 = (lo - o64) / d64
        t1 = (hi - o64) / d64
    tn = np.minimum(t0, t1)
    tf = np.maximum(t0, t1)
    tmin = tn.max(1)
    tmax = tf.min(1)
    inside = np.all((o64 > lo) & (o64 < hi), 1)
    checked = 0
    for i in range(n):
        if inside[i]:
            continue
        hit = tmin[i] <= tmax[i] and tmin[i] > 0
        # skip rays within 1e-7 of an edge (tie between two sides)
        srt = np.sort(tn[i])
        if hit and (srt[2] - srt[1] < 1e-7 or tmax[i] - tmin[i] < 1e-7):
            continue
        if not hit:
            if tmin[i] <= tmax[i] + 1e-7 and tmin[i] > -1e-7:
                continue
            assert res.face[i] == -1 and res.t64[i] == 100.0, i
            continue
        checked += 1
        assert abs(res.t64[i] - tmin[i]) < 1e-9 * max(1, tmin[i]), i
        axis = int(np.argmax(tn[i]))
        side = 2 * axis + (1 if d64[i, axis] < 0 else 0)  # entering +x side when moving -x
        assert res.face[i] // 2 == side, (i, res.face[i], side)
        assert res.seg[i] == 3
    assert checked > 500


@pytest.mark.parametrize("subdiv,ratio", [(0, 0.79465), (1, 0.93417), (2, 0.98225), (3, 0.99547)])
def test_icosphere_from_centre(subdiv, ratio):
    """Camera at the centre of an icosphere of circumradius R: every ray hits,
    r_in <= t <= R, and t * (n_f . d_hat) = distance of the reported face's
    plane (SURVEY.md §8(c) sphere pin; inradius ratios are of the icosphere)."""
    R = 2.0
    mesh = sg.sphere_mesh(R, subdiv)
    # inradius from the mesh: min plane distance over faces (independent check
    # of the quoted ratio)
    v = mesh.verts.astype(np.float64)
    f = mesh.faces
    n = np.cross(v[f[:, 1]] - v[f[:, 0]], v[f[:, 2]] - v[f[:, 0]])
    nh = n / np.linalg.norm(n, axis=1, keepdims=True)
    plane_d = np.abs(np.einsum("ij,ij->i", nh, v[f[:, 0]]))
    assert abs(plane_d.min() / R - ratio) < 2e-4
    sc = sg.assemble([mesh], [[(0, 2, sg.make_T(np.eye(3), (0, 0, 0)))]])
    cam = sg.pinhole(24, 16, 100.0)
    rng = np.random.default_rng(subdiv)
    P = sg.make_T(sg.random_rotation(rng), (0, 0, 0))[None, None]
    res = cast_pinhole(sc, cam, P, oracle.RANGE)
    assert np.all(res.face >= 0)
    assert np.all(res.t64 <= R * (1 + 1e-6)) and np.all(res.t64 >= R * ratio * (1 - 1e-3))
    # recompute each ray direction independently: unit vector through the pixel
    u = np.arange(cam["W"]) + 0.5 - cam["cx"]
    vv = np.arange(cam["H"]) + 0.5 - cam["cy"]
    V, U = np.meshgrid(vv, u, indexing="ij")
    ds = np.stack([np.ones_like(U), -U / cam["fx"], -V / cam["fy"]], -1).reshape(-1, 3)
    ds /= np.linalg.norm(ds, axis=1, keepdims=True)
    dw = ds @ P[0, 0, :, :3].astype(np.float64).T
    cosang = np.abs(np.einsum("ij,ij->i", nh[res.face], dw))
    assert np.allclose(res.t64 * cosang, plane_d[res.face], atol=1e-9)


def test_sphere_from_outside_bounds():
    """Outside camera: hit t between the circumsphere and insphere entry
    distances; rays missing the circumsphere miss."""
    R, subdiv = 1.0, 2
    r_in = 0.98225 * R
    mesh = sg.sphere_mesh(R, subdiv)
    c = np.asarray([4.0, 0.3, -0.2])
    sc = sg.assemble([mesh], [[(0, 1, sg.make_T(np.eye(3), c))]])
    rng = np.random.default_rng(3)
    n = 3000
    o = np.zeros((n, 3), np.float32)
    d = (c + rng.uniform(-1.3, 1.3, (n, 3)) - 0).astype(np.float32)
    res = cast_rays(sc, o[None], d[None])
    d64 = d.astype(np.float64)
    dh = d64 / np.linalg.norm(d64, axis=1, keepdims=True)
    b = dh @ c
    perp2 = np.dot(c, c) - b * b

    def entry(rad):
        disc = rad * rad - perp2
        with np.errstate(invalid="ignore"):
            return b - np.sqrt(disc)

    tR = entry(R) / np.linalg.norm(d64, axis=1)
    tr = entry(r_in) / np.linalg.norm(d64, axis=1)
    miss_R = perp2 > R * R
    assert np.all(res.face[miss_R] == -1)
    hit_r = perp2 < (r_in * 0.999) ** 2
    assert np.all(res.face[hit_r] >= 0)
    h = res.face >= 0
    assert np.all(res.t64[h] >= tR[h] - 1e-9)
    ok = hit_r & h
    assert np.all(res.t64[ok] <= tr[ok] + 1e-9)


def test_lidar_wall_beam_zero():
    """Beam (e=0, a=0) toward a wall at 2 m -> range 2.0."""
    beams = sg.lidar_beams(8, 16)  # a_k = -180 + 22.5k: k = 8 is a = 0
    sc = sg.assemble([quad_mesh()], [[(0, 1, sg.make_T(np.eye(3), (2.0, 0, 0)))]])
    # 8 channels from -45 to 45: no exact 0; use a 9-channel table for e = 0
    beams = sg.lidar_beams(9, 16)
    res = oracle.cast(sc, dict(model=oracle.BEAMS, beams=beams, poses=sg.identity_poses(1),
                               max_range=10.0))
    rr = res.t64.reshape(9, 16)
    assert abs(rr[4, 8] - 2.0) < 1e-7  # float32 beam table is cos/sin rounded
    assert res.seg.reshape(9, 16)[4, 8] == 1


@pytest.mark.parametrize("nseg", [16, 23])
def test_lidar_ring_in_ngon_cylinder(nseg):
    """Horizontal ring inside an n-gon cylinder of circumradius R: range =
    R cos(pi/n) / cos(phi), phi = angle from the facet normal."""
    R = 3.0
    cyl = sg.cylinder_mesh("cyl", R, 4.0, nseg=nseg, closed=False, z0=-2.0)
    sc = sg.assemble([cyl], [[(0, 1, sg.make_T(np.eye(3), (0, 0, 0)))]])
    K = 360
    beams = sg.lidar_beams(3, K, -10.0, 10.0)
    res = oracle.cast(sc, dict(model=oracle.BEAMS, beams=beams, poses=sg.identity_poses(1),
                               max_range=10.0))
    rr = res.t64.reshape(3, K)[1]
    az = np.radians(-180.0 + 360.0 * np.arange(K) / K)
    seg_w = 2 * math.pi / nseg
    # facet k spans [k seg_w, (k+1) seg_w]; its normal points at (k+0.5) seg_w
    phi = (np.mod(az, seg_w) - seg_w / 2)
    want = R * math.cos(math.pi / nseg) / np.cos(phi)
    # beams with az on a facet boundary are ties: skip them
    edge = np.abs(np.abs(phi) - seg_w / 2) < 1e-6
    assert np.allclose(rr[~edge], want[~edge], atol=2e-6)
    assert np.all((rr >= R * math.cos(math.pi / nseg) - 1e-6) & (rr <= R + 1e-6))


def test_lidar_dome_under_ceiling():
    """Dome pattern under a ceiling plane at height h: range = h / sin(e)
    (PAPER.md:228 'Dome LiDAR')."""
    h = 2.5
    ceil = quad_mesh(200.0)
    Rz = np.asarray([[0, 0, -1], [0, 1, 0], [1, 0, 0]], np.float64)  # +x normal -> -z
    sc = sg.assemble([ceil], [[(0, 1, sg.make_T(Rz, (0, 0, h)))]])
    beams = sg.dome_beams(8, 24)
    res = oracle.cast(sc, dict(model=oracle.BEAMS, beams=beams, poses=sg.identity_poses(1),
                               max_range=50.0))
    C, K = 8, 24
    e = np.radians(90.0 / C + (90.0 - 90.0 / C) * np.arange(C) / (C - 1))
    want = np.repeat((h / np.sin(e))[:, None], K, 1)
    assert np.allclose(res.t64.reshape(C, K), want, rtol=1e-6)


# --------------------------------------------------------------------------
# semantics: misses, max range, ties, degenerate faces, numbering
# --------------------------------------------------------------------------

def test_misses_empty_env_and_facing_away():
    """Empty env and a camera facing away -> max_range, -1, -1."""
    cam = sg.pinhole(8, 6, 60.0)
    sc = sg.assemble([sg.cube_mesh()], [[], [(0, 1, sg.make_T(np.eye(3), (-3, 0, 0)))]])
    res = cast_pinhole(sc, cam, sg.identity_poses(2), oracle.DEPTH, max_range=7.5)
    assert np.all(res.t64 == 7.5) and np.all(res.seg == -1) and np.all(res.face == -1)


def test_max_range_inclusive():
    """A hit at exactly t = max_range counts; beyond it is a miss (reading R5);
    hits within 1e-5 of max_range are flagged AMB_RANGE."""
    def run(x, mr):
        sc = sg.assemble([quad_mesh()], [[(0, 1, sg.make_T(np.eye(3), (x, 0, 0)))]])
        o = np.asarray([[[0, 0.1, 0.3]]], np.float32)  # off the quad's diagonal
        d = np.asarray([[[1, 0, 0]]], np.float32)
        return cast_rays(sc, o, d, max_range=mr)
    r = run(10.0, 10.0)
    assert r.face[0] >= 0 and r.t64[0] == 10.0 and r.amb[0] & oracle.AMB_RANGE
    r = run(10.5, 10.0)
    assert r.face[0] == -1 and r.t64[0] == 10.0 and r.amb[0] == 0
    r = run(10.000004, 10.0)
    assert r.face[0] == -1 and r.amb[0] & oracle.AMB_RANGE
    r = run(5.0, 10.0)
    assert r.amb[0] == 0


def test_tie_goes_to_lowest_face_and_is_flagged():
    """Coincident triangles: equal t -> lowest per-env face index (reading
    R11), flagged AMB_TIE."""
    q = quad_mesh()
    sc = sg.assemble([q, q], [[(1, 5, sg.make_T(np.eye(3), (3, 0, 0))),
                               (0, 6, sg.make_T(np.eye(3), (3, 0, 0)))]])
    o = np.zeros((1, 2, 3), np.float32)
    d = np.asarray([[[1, 0.1, 0.05], [1, -0.1, -0.05]]], np.float32)
    r = cast_rays(sc, o, d)
    assert list(r.seg) == [5, 5]
    # instance 0's faces are 0 (y > z half of the quad) and 1; instance 1's
    # coincident copies are 2 and 3
    assert list(r.face) == [0, 1]
    assert np.all(r.amb & oracle.AMB_TIE)


def test_shared_vertex_rays_are_flagged():
    """A ray aimed exactly at a vertex shared by two triangles (generic FP32
    coordinates; origin 0, direction = the vertex) hits both geometrically,
    but the FP64 edge tests of its rounded hit point may exclude one of
    them.  Every such ray must be flagged AMB_TIE (north_star: 'except for
    rays whose two candidate hits lie within 1e-5 m of each other'; DESIGN.md
    reading R24).  Control: rays aimed at the triangles' interiors are not
    flagged."""
    rng = np.random.default_rng(11)
    n_hit = 0
    for trial in range(200):
        a, b, c = rng.uniform(-1, 1, (3, 3))
        e = a + b - c  # across edge ab from c: a planar convex quad
        a, b, c, e = (np.asarray(v + (4.0, 0.0, 0.0), np.float32) for v in (a, b, c, e))  # in front of 0
        m = sg.Mesh("two", np.stack([a, b, c, e]).astype(np.float32),
                    np.asarray([[0, 1, 2], [1, 0, 3]], np.int32))
        sc = sg.assemble([m], [[(0, 1, sg.make_T(np.eye(3), (0, 0, 0)))]])
        d = np.stack([a, b])[None].astype(np.float32)  # aimed at the two shared vertices
        r = cast_rays(sc, np.zeros((1, 2, 3), np.float32), d)
        hit = r.face >= 0
        n_hit += int(hit.sum())
        assert np.all(r.amb[hit] & oracle.AMB_TIE), trial
        # interior points (barycentric weights >= 0.2 each) are unambiguous
        w = 0.2 + 0.4 * rng.dirichlet([4, 4, 4], 8)
        w = w / w.sum(1, keepdims=True)
        q = w @ np.stack([a, b, c]).astype(np.float64)
        r2 = cast_rays(sc, np.zeros((1, 8, 3), np.float32), q[None].astype(np.float32))
        assert np.all(r2.face == 0) and not np.any(r2.amb & oracle.AMB_TIE), trial
    assert n_hit > 300


def test_degenerate_face_kept_for_numbering_never_hit():
    """Zero-area faces keep the numbering and are never hit (reading R12)."""
    v = np.asarray([[0, -5, -5], [0, 5, -5], [0, 5, 5], [0, -5, 5]], np.float32)
    m = sg.Mesh("q", v, np.asarray([[0, 1, 1], [0, 2, 2], [0, 1, 2], [0, 2, 3]], np.int32))
    sc = sg.assemble([m], [[(0, 1, sg.make_T(np.eye(3), (2, 0, 0)))]])
    o = np.zeros((1, 2, 3), np.float32)
    d = np.asarray([[[1, 0.2, -0.1], [1, -0.2, 0.1]]], np.float32)
    r = cast_rays(sc, o, d)
    assert list(r.face) == [2, 3]


def test_double_sided():
    """Triangles are hit from both sides (reading R10)."""
    sc = sg.assemble([quad_mesh()], [[(0, 1, sg.make_T(np.eye(3), (0, 0, 0)))]])
    o = np.asarray([[[-2, 0, 0], [2, 0.5, 0]]], np.float32)
    d = np.asarray([[[1, 0, 0], [-1, 0, 0]]], np.float32)
    r = cast_rays(sc, o, d)
    assert np.all(r.face >= 0) and np.allclose(r.t64, 2.0)


def test_face_numbering_across_instances_and_labels():
    """Per-env face index = prefix sum of instance face counts + local index
    (reading R2); seg = instance label (reading R3)."""
    cube, cyl = sg.cube_mesh(), sg.closed_cylinder_92()
    sc = sg.assemble([cube, cyl], [
        [(1, 10, sg.make_T(np.eye(3), (5, 0, 0))), (0, 20, sg.make_T(np.eye(3), (3, 0, 0)))],
        [(0, 30, sg.make_T(np.eye(3), (3, 0, 0)))]])
    o = np.zeros((2, 1, 3), np.float32)
    d = np.asarray([[[1, 0.01, 0.02]], [[1, 0.01, 0.02]]], np.float32)
    r = cast_rays(sc, o, d)
    # env 0: the cube (instance 1) is nearer; its faces follow the cylinder's 92
    assert r.seg[0] == 20 and 92 <= r.face[0] < 92 + 12
    assert r.face[0] - 92 in (0, 1)  # -x side of the cube
    assert r.seg[1] == 30 and r.face[1] in (0, 1)
    assert abs(r.t64[0] - 2.5) < 1e-9


def test_origin_on_surface_flagged_zero():
    """A candidate within 1e-5 of t = 0 sets AMB_ZERO (parity rule 3)."""
    sc = sg.assemble([quad_mesh()], [[(0, 1, sg.make_T(np.eye(3), (0, 0, 0)))]])
    o = np.asarray([[[1e-6, 0.1, 0.1]]], np.float32)
    d = np.asarray([[[-1, 0.0, 0.0]]], np.float32)
    r = cast_rays(sc, o, d)
    assert r.amb[0] & oracle.AMB_ZERO


def test_sensor_frame_axes():
    """x forward, y left, z up; u grows to the right (-y), v downward (-z)
    (reading R7): an object at (+x, -y, +z) lands in the top-right quadrant."""
    cam = sg.pinhole(20, 20, 90.0)
    sc = sg.assemble([sg.cube_mesh(0.5)], [[(0, 1, sg.make_T(np.eye(3), (4, -1.5, 1.5)))]])
    r = cast_pinhole(sc, cam, sg.identity_poses(1))
    img = r.seg.reshape(20, 20)
    vs, us = np.nonzero(img == 1)
    assert len(us) > 0 and us.min() >= 10 and vs.max() < 10


def test_depth_le_range_and_principal_ray():
    """depth <= range on every hit; equality on the optical axis."""
    sc, s = sg.config2(n_envs=2)
    cam = dict(s["cam"])
    cam.update(W=41, H=21, cx=20.5, cy=10.5)
    d = cast_pinhole(sc, cam, s["poses"], oracle.DEPTH)
    r = cast_pinhole(sc, cam, s["poses"], oracle.RANGE)
    hit = (d.face >= 0) & (r.face >= 0)
    assert hit.sum() > 50
    assert np.all(d.t64[hit] <= r.t64[hit] + 1e-12)
    centre = (np.arange(2) * 21 + 10) * 41 + 20
    for c in centre:
        if d.face[c] >= 0:
            assert abs(d.t64[c] - r.t64[c]) < 1e-12


# --------------------------------------------------------------------------
# independent brute force (different formula) and invariants
# --------------------------------------------------------------------------

def _mt_numpy(tris, o, d, max_range):
    """Independent FP64 Moller-Trumbore (vectorised numpy), closest hit,
    lowest index on equal t."""
    v0, v1, v2 = tris[:, 0], tris[:, 1], tris[:, 2]
    e1, e2 = v1 - v0, v2 - v0
    out_t = np.full(len(o), max_range)
    out_f = np.full(len(o), -1)
    for i in range(len(o)):
        p = np.cross(d[i], e2)
        det = np.einsum("ij,ij->i", e1, p)
        ok = det != 0
        inv = np.where(ok, 1.0 / np.where(ok, det, 1.0), 0.0)
        s = o[i] - v0
        u = np.einsum("ij,ij->i", s, p) * inv
        q = np.cross(s, e1)
        v = (q @ d[i]) * inv
        t = np.einsum("ij,ij->i", e2, q) * inv
        hit = ok & (u >= 0) & (v >= 0) & (u + v <= 1) & (t > 0) & (t <= max_range)
        if hit.any():
            k = np.nonzero(hit)[0]
            j = k[np.lexsort((k, t[k]))[0]]
            out_t[i], out_f[i] = t[j], j
    return out_t, out_f


def test_matches_independent_moller_trumbore():
    """1000 random rays vs a 50-triangle scene == an independent brute force
    with a different intersection formula."""
    rng = np.random.default_rng(42)
    verts = rng.uniform(-2, 2, (150, 3)).astype(np.float32)
    m = sg.Mesh("soup", verts, np.arange(150, dtype=np.int32).reshape(50, 3))
    T = sg.make_T(sg.random_rotation(rng), rng.uniform(-1, 1, 3), 1.3)
    sc = sg.assemble([m], [[(0, 4, T)]])
    n = 1000
    o = rng.uniform(-4, 4, (n, 3)).astype(np.float32)
    d = rng.normal(size=(n, 3)).astype(np.float32)
    res = cast_rays(sc, o[None], d[None], max_range=20.0)
    A, b = T[:, :3].astype(np.float64), T[:, 3].astype(np.float64)
    tris = (verts.astype(np.float64) @ A.T + b).reshape(50, 3, 3)
    t, f = _mt_numpy(tris, o.astype(np.float64), d.astype(np.float64), 20.0)
    amb = res.amb != 0
    assert np.allclose(res.t64, t, rtol=1e-9, atol=1e-12)
    assert np.all((res.face == f) | amb)
    assert (f >= 0).sum() > 100


def _rigid_exact(rng):
    """Random signed axis permutation (a rotation): exact in FP32, so the
    transformed inputs represent exactly the moved scene.  (A translation is
    not FP32-exact in general: it is covered by the generic test.)"""
    perm = rng.permutation(3)
    R = np.zeros((3, 3))
    R[np.arange(3), perm] = rng.choice([-1.0, 1.0], 3)
    if np.linalg.det(R) < 0:
        R[0] *= -1
    return R, np.zeros(3)


def _move(sc, poses, R, p):
    T = sc.inst_T.astype(np.float64)
    T2 = np.empty_like(T)
    T2[:, :, :3] = np.einsum("ij,njk->nik", R, T[:, :, :3])
    T2[:, :, 3] = T[:, :, 3] @ R.T + p
    P = poses.astype(np.float64)
    P2 = np.empty_like(P)
    P2[..., :3] = np.einsum("ij,esjk->esik", R, P[..., :3])
    P2[..., 3] = P[..., 3] @ R.T + p
    sc2 = sg.Scene(sc.meshes, sc.env_off, sc.inst_asset, sc.inst_label, T2.astype(np.float32))
    return sc2, P2.astype(np.float32)


def test_rigid_invariance_exact_group():
    """Scene + sensor moved by an FP32-exact rigid motion: identical outputs
    within 1e-9 (north_star invariance pin)."""
    sc, s = sg.config2(n_envs=3)
    cam = dict(s["cam"], W=60, H=34, cx=30.0, cy=17.0)
    a = cast_pinhole(sc, cam, s["poses"], oracle.RANGE)
    rng = np.random.default_rng(9)
    for _ in range(2):
        R, p = _rigid_exact(rng)
        sc2, P2 = _move(sc, s["poses"], R, p)
        b = cast_pinhole(sc2, cam, P2, oracle.RANGE)
        assert np.allclose(a.t64, b.t64, atol=1e-9, rtol=0)
        ok = (a.amb == 0) & (b.amb == 0)
        assert np.all(a.face[ok] == b.face[ok]) and np.all(a.seg[ok] == b.seg[ok])


def test_rigid_invariance_generic():
    """Generic rotation: equal within FP32 input rounding; seg/face equal away
    from edges (graze > 1e-4) and ties."""
    sc, s = sg.config2(n_envs=2)
    cam = dict(s["cam"], W=60, H=34, cx=30.0, cy=17.0)
    a = cast_pinhole(sc, cam, s["poses"], oracle.DEPTH, graze=True)
    R = sg.random_rotation(np.random.default_rng(1))
    sc2, P2 = _move(sc, s["poses"], R, np.asarray([0.7, -1.1, 0.3]))
    b = cast_pinhole(sc2, cam, P2, oracle.DEPTH)
    far_edge = (a.graze > 1e-4) & (a.amb == 0) & (b.amb == 0)
    assert np.all(a.seg[far_edge] == b.seg[far_edge])
    same = far_edge & (a.face == b.face)
    assert np.allclose(a.t64[same], b.t64[same], atol=1e-4)


def test_query_subset_equals_full():
    """Sampled queries (any order) give the same per-ray answers as a full
    cast -- the sampling used for full-size parity."""
    sc, s = sg.config2(n_envs=4)
    cam = dict(s["cam"], W=30, H=20, cx=15.0, cy=10.0)
    full = cast_pinhole(sc, cam, s["poses"])
    q = np.random.default_rng(0).choice(4 * 600, 300, replace=False)
    sub = cast_pinhole(sc, cam, s["poses"], query=q)
    assert np.array_equal(sub.t64, full.t64[q]) and np.array_equal(sub.face, full.face[q])
    one = cast_pinhole(sc, cam, s["poses"], query=q, n_threads=1)
    assert np.array_equal(one.t64, sub.t64)


# --------------------------------------------------------------------------
# per-hit channels: normal, barycentrics, point
# --------------------------------------------------------------------------

def test_plane_normal_and_point_closed_form():
    """Camera facing a plane at distance d: the normal faces the camera,
    (-1, 0, 0); the point is (d, -x' d, -y' d) (PAPER.md:218 normals, :228
    point clouds)."""
    dist = 3.0
    cam = sg.pinhole(12, 8, 80.0)
    sc = sg.assemble([quad_mesh()], [[(0, 1, sg.make_T(np.eye(3), (dist, 0, 0)))]])
    r = cast_pinhole(sc, cam, sg.identity_poses(1), oracle.DEPTH, extras=True)
    assert np.allclose(r.normal, [-1.0, 0.0, 0.0], atol=1e-15)
    u = np.arange(cam["W"]) + 0.5 - cam["cx"]
    v = np.arange(cam["H"]) + 0.5 - cam["cy"]
    V, U = np.meshgrid(v, u, indexing="ij")
    want = np.stack([np.full(U.shape, dist), -U / cam["fx"] * dist, -V / cam["fy"] * dist], -1)
    assert np.allclose(r.point, want.reshape(-1, 3), atol=1e-12)


def test_barycentric_reproduces_hit_point_and_linear_field():
    """hit = (1-b1-b2) v0 + b1 v1 + b2 v2 over the face's world vertices, and
    a linear per-vertex field interpolates to its value at the hit (SPEC
    S:555-556 'linear-reproduction oracle')."""
    rng = np.random.default_rng(21)
    verts = rng.uniform(-1, 1, (60, 3)).astype(np.float32)
    m = sg.Mesh("soup", verts, np.arange(60, dtype=np.int32).reshape(20, 3))
    T = sg.make_T(sg.random_rotation(rng), (3.0, 0.2, -0.1), 1.1)
    sc = sg.assemble([m], [[(0, 2, T)]])
    o = np.zeros((1, 2000, 3), np.float32)
    d = (rng.uniform([2.0, -1.5, -1.5], [4.0, 1.5, 1.5], (1, 2000, 3))).astype(np.float32)
    r = cast_rays(sc, o, d, extras=True)
    hit = r.face >= 0
    assert hit.sum() > 100
    A, b = T[:, :3].astype(np.float64), T[:, 3].astype(np.float64)
    W = verts.astype(np.float64) @ A.T + b
    tri = W.reshape(20, 3, 3)[r.face[hit]]
    b1, b2 = r.bary[hit, 0], r.bary[hit, 1]
    p = (1 - b1 - b2)[:, None] * tri[:, 0] + b1[:, None] * tri[:, 1] + b2[:, None] * tri[:, 2]
    assert np.allclose(p, r.point[hit], atol=1e-9)
    assert np.all((b1 >= -1e-12) & (b2 >= -1e-12) & (b1 + b2 <= 1 + 1e-12))
    field = 0.7 * tri[..., 0] - 0.2 * tri[..., 2] + 0.5  # linear in position
    interp = (1 - b1 - b2) * field[:, 0] + b1 * field[:, 1] + b2 * field[:, 2]
    assert np.allclose(interp, 0.7 * r.point[hit, 0] - 0.2 * r.point[hit, 2] + 0.5, atol=1e-9)
    assert np.all(r.bary[~hit] == -1.0) and np.all(r.normal[~hit] == 0.0)


def test_vertex_aimed_ray_barycentrics():
    """A ray through vertex v1 (resp. v2) of an isolated triangle has
    barycentrics (1, 0) (resp. (0, 1))."""
    v = np.asarray([[2, -1, -1], [2, 1, -1], [2, 0, 1]], np.float32)
    sc = sg.assemble([sg.Mesh("t", v, np.asarray([[0, 1, 2]], np.int32))],
                     [[(0, 1, sg.make_T(np.eye(3), (0, 0, 0)))]])
    o = np.zeros((1, 3, 3), np.float32)
    d = v[None].copy()
    r = cast_rays(sc, o, d, extras=True)
    assert np.allclose(r.bary, [[0, 0], [1, 0], [0, 1]], atol=1e-12)
    assert np.allclose(r.t64, 1.0)


def test_sphere_normals_face_the_origin():
    """Inside an icosphere every normal points back at the camera (n . d <
    0) and equals the reported face's unit normal up to sign."""
    mesh = sg.sphere_mesh(2.0, 2)
    sc = sg.assemble([mesh], [[(0, 1, sg.make_T(np.eye(3), (0, 0, 0)))]])
    cam = sg.pinhole(16, 12, 100.0)
    r = cast_pinhole(sc, cam, sg.identity_poses(1), oracle.RANGE, extras=True)
    v = mesh.verts.astype(np.float64)[mesh.faces[r.face]]
    n = np.cross(v[:, 1] - v[:, 0], v[:, 2] - v[:, 0])
    n /= np.linalg.norm(n, axis=1, keepdims=True)
    assert np.allclose(np.abs(np.einsum("ij,ij->i", n, r.normal)), 1.0, atol=1e-12)
    # direction of each ray = point / |point| (camera at the origin)
    dirs = r.point / np.linalg.norm(r.point, axis=1, keepdims=True)
    assert np.all(np.einsum("ij,ij->i", r.normal, dirs) < 0)


# --------------------------------------------------------------------------
# stereo shadow mask
# --------------------------------------------------------------------------

def _post_and_wall(wall_x=6.0, post_x=3.0, half_w=0.1):
    wall = quad_mesh(200.0)
    post = sg.box_mesh("post", (-0.01, -half_w, -5.0), (0.01, half_w, 5.0))
    return sg.assemble([wall, post], [[(0, 1, sg.make_T(np.eye(3), (wall_x, 0, 0))),
                                       (1, 2, sg.make_T(np.eye(3), (post_x, 0, 0)))]])


def test_stereo_wall_only_all_valid_and_zero_baseline():
    """One wall and nothing else: every pixel valid; with baseline 0
    every hit pixel is valid."""
    cam = sg.pinhole(32, 8, 70.0)
    sc = sg.assemble([quad_mesh(200.0)], [[(0, 1, sg.make_T(np.eye(3), (4.0, 0, 0)))]])
    r = cast_pinhole(sc, cam, sg.identity_poses(1), stereo=((0.0, -0.2, 0.0), 1e-4))
    assert np.all(r.valid == 1)
    sc2 = _post_and_wall()
    r = cast_pinhole(sc2, cam, sg.identity_poses(1), stereo=((0.0, 0.0, 0.0), 1e-4))
    assert np.all(r.valid == 1)


@pytest.mark.parametrize("baseline", [0.1, 0.3])
def test_stereo_post_shadow_band_closed_form(baseline):
    """Thin post (half-width h at x = P) before a wall (x = W), right camera
    at (0, -b, 0): a wall point at height y is hidden from it iff the
    segment to the camera crosses the post, i.e. |y P/W - b (1 - P/W)| <= h
    (S:546 'band width grows with baseline')."""
    W_, P_, h = 6.0, 3.0, 0.1
    cam = sg.pinhole(400, 4, 60.0)
    sc = _post_and_wall(W_, P_, h)
    r = cast_pinhole(sc, cam, sg.identity_poses(1), max_range=20.0,
                     stereo=((0.0, -baseline, 0.0), 1e-4), extras=True)
    row = np.arange(400) + (1 * 400)  # v = 1
    on_wall = r.seg[row] == 1
    y = r.point[row, 1]
    yp = y * P_ / W_ - baseline * (1 - P_ / W_)
    shadow = np.abs(yp) <= h
    far = np.abs(np.abs(yp) - h) > 2e-3  # away from the band's edges
    sel = on_wall & far
    assert sel.sum() > 200
    assert np.array_equal(r.valid[row][sel] == 0, shadow[sel])
    assert (shadow & on_wall).sum() >= 3
    # the post itself is seen by both cameras: valid
    assert np.all(r.valid[row][r.seg[row] == 2] == 1)


# --------------------------------------------------------------------------
# certificate of a reported face (oracle.certify)
# --------------------------------------------------------------------------

def test_certify_single_triangle_closed_form():
    """One triangle in the plane x = 5 with legs along +y and +z: the ray
    through (5, y, z) has t = 1 (direction (5, y, z)), and the plane hit lies
    outside the face by max(-y, -z, (y + z - 1)/sqrt 2) (signed distances to
    the three edges)."""
    v = np.asarray([[5, 0, 0], [5, 1, 0], [5, 0, 1]], np.float32)
    m = sg.Mesh("tri", v, np.asarray([[0, 1, 2]], np.int32))
    sc = sg.assemble([m, m], [[(0, 7, sg.make_T(np.eye(3), (0, 0, 0))),
                               (1, 9, sg.make_T(np.eye(3), (2.0, 0, 0)))]])
    pts = np.asarray([[0.25, 0.25], [0.8, 0.6], [-0.1, 0.3], [0.0, 0.0], [0.5, 0.5]])
    d = np.concatenate([np.full((len(pts), 1), 5.0), pts], 1)[None].astype(np.float32)
    o = np.zeros_like(d)
    rays = dict(model=oracle.RAYS, orig=o, dir=d, max_range=100.0)
    t, out, lab = oracle.certify(sc, rays, np.zeros(len(pts), np.int32))
    def want_out(k):  # the hit is (5k, k y, k z) on a face with unit legs
        return np.maximum(np.maximum(-k * pts[:, 0], -k * pts[:, 1]), (k * pts.sum(1) - 1) / math.sqrt(2))
    assert np.allclose(t, 1.0, atol=1e-15)
    assert np.allclose(out, want_out(1.0), atol=1e-7)  # FP32 direction inputs
    assert np.all(lab == 7)
    # face 1 is the second instance's copy at x = 7: t = 7/5, label 9
    t1, out1, lab1 = oracle.certify(sc, rays, np.ones(len(pts), np.int32))
    assert np.allclose(t1, 1.4, atol=1e-14) and np.all(lab1 == 9)
    assert np.allclose(out1, want_out(1.4), atol=1e-7)
    # a miss certifies nothing
    tm, outm, labm = oracle.certify(sc, rays, np.full(len(pts), -1, np.int32))
    assert np.all(np.isnan(tm)) and np.all(np.isinf(outm)) and np.all(labm == -1)


def test_certify_agrees_with_cast_on_its_own_answer():
    """On the oracle's own winners (random c2-like scene, 2 envs) the
    certificate reproduces t exactly (same FP64 plane formula), finds every
    hit inside its face and returns the cast's seg."""
    sc, s = sg.config2(n_envs=2)
    cam = sg.pinhole(24, 16, 87.0)
    rays = dict(model=oracle.PINHOLE, kind=oracle.RANGE, poses=s["poses"], max_range=10.0, **cam)
    r = oracle.cast(sc, rays)
    t, out, lab = oracle.certify(sc, rays, r.face)
    hit = r.face >= 0
    assert hit.sum() > 50
    assert np.array_equal(t[hit], r.t64[hit])
    assert np.all(out[hit] <= 1e-12)
    assert np.array_equal(lab, r.seg)
    assert np.all(np.isnan(t[~hit]))


# --------------------------------------------------------------------------
# vertex annotations (f1; "embed vertex-level annotations that
# can be queried"; SPEC S:550-556 query_annotation examples)
# --------------------------------------------------------------------------

def test_annotation_vertex_centroid_and_miss():
    """Ray through vertex v_k -> exactly A(v_k); through the centroid ->
    the mean of the three annotations; a miss -> NaN."""
    v = np.asarray([[2, -1, -1], [2, 1, -1], [2, 0, 1]], np.float32)
    sc = sg.assemble([sg.Mesh("t", v, np.asarray([[0, 1, 2]], np.int32))],
                     [[(0, 1, sg.make_T(np.eye(3), (0, 0, 0)))]])
    A = np.asarray([[1.0, -2.0], [4.0, 0.5], [-3.0, 8.0]], np.float32)
    cen = v.astype(np.float64).mean(0)
    d = np.concatenate([v, cen[None], [[-1.0, 0.0, 0.0]]]).astype(np.float32)[None]
    o = np.zeros_like(d)
    r = cast_rays(sc, o, d, annot=[A])
    assert np.allclose(r.annot[:3], A, atol=1e-12)
    assert np.allclose(r.annot[3], A.astype(np.float64).mean(0), atol=1e-7)  # FP32 centroid direction
    assert np.all(np.isnan(r.annot[4]))


def test_annotation_linear_field_reproduction():
    """A linear field of the object-space vertex coordinates interpolates to
    the same field at the object-space hit point A^-1 (p - b) (S:555-556
    'linear-reproduction oracle'), under a random similarity transform, for
    K = 3 fields; an asset without annotations yields NaN."""
    rng = np.random.default_rng(31)
    verts = rng.uniform(-1, 1, (60, 3)).astype(np.float32)
    soup = sg.Mesh("soup", verts, np.arange(60, dtype=np.int32).reshape(20, 3))
    wall = sg.Mesh("wall", np.asarray([[9, -50, -50], [9, 50, -50], [9, 0, 50]], np.float32),
                   np.asarray([[0, 1, 2]], np.int32))
    T = sg.make_T(sg.random_rotation(rng), (3.0, 0.2, -0.1), 1.1)
    sc = sg.assemble([soup, wall], [[(0, 2, T), (1, 3, sg.make_T(np.eye(3), (0, 0, 0)))]])
    M = np.asarray([[1.0, 0.0, 0.0], [2.0, -1.0, 0.5], [0.0, 0.25, 3.0]])
    c = np.asarray([0.0, 0.5, -1.0])
    field = (verts.astype(np.float64) @ M.T + c).astype(np.float32)
    o = np.zeros((1, 3000, 3), np.float32)
    d = rng.uniform([2.0, -1.5, -1.5], [4.0, 1.5, 1.5], (1, 3000, 3)).astype(np.float32)
    r = cast_rays(sc, o, d, extras=True, annot=[field, None])
    on_soup = (r.face >= 0) & (r.face < 20)
    assert on_soup.sum() > 200 and (r.face == 20).sum() > 100
    A, b = T[:, :3].astype(np.float64), T[:, 3].astype(np.float64)
    p_obj = np.linalg.solve(A, (r.point[on_soup] - b).T).T
    want = p_obj @ M.T + c
    # the FP32-rounded field values carry ~1e-7 relative error
    assert np.allclose(r.annot[on_soup], want, atol=2e-6)
    assert np.all(np.isnan(r.annot[r.face == 20]))


# --------------------------------------------------------------------------
# ambiguity flags: the near-candidate band (reading R24) and the
# stereo shadow band edges (reading R21), pinned on both sides
# --------------------------------------------------------------------------

def _outside_distance(p, a, b, c):
    """In-plane distance (FP64) by which point p (on the triangle's plane)
    lies outside triangle abc, from its barycentric coordinates (a different
    formula from the oracle's edge functions): 0 inside."""
    e1, e2 = b - a, c - a
    G = np.array([[e1 @ e1, e1 @ e2], [e1 @ e2, e2 @ e2]])
    u, v = np.linalg.solve(G, np.array([(p - a) @ e1, (p - a) @ e2]))
    w = 1.0 - u - v
    dist = 0.0
    for lam, (q0, q1, opp) in ((w, (b, c, a)), (u, (c, a, b)), (v, (a, b, c))):
        if lam < 0:  # p beyond the edge opposite the vertex with weight lam
            ed = q1 - q0
            h = np.linalg.norm(np.cross(ed, opp - q0)) / np.linalg.norm(ed)  # altitude
            dist = max(dist, -lam * h)
    return dist


def test_near_candidate_band_is_fp64_rounding():
    """A plane hit just outside an isolated triangle is a near candidate
    (AMB_GRAZE on the otherwise-missing ray) only within FP64 rounding of the
    scene's magnitudes (nu = 2^-40 M, R24), not within a fixed
    1e-9 m: rays that pass the edge by more than 2^-36 M (16 nu) and less
    than 1e-9 m are clean misses; rays through a vertex, or within 2^-46 M of
    the edge, are hits or grazes.  A millimetre-sized triangle puts FP32
    direction quantisation (~1e-10 m) between the two bands."""
    rng = np.random.default_rng(5)
    n_band = n_vert = 0
    for trial in range(60):
        a, b, c = (rng.uniform(-1e-3, 1e-3, 3) + np.array([4e-3, 0, 0]) for _ in range(3))
        a, b, c = (np.asarray(v, np.float32) for v in (a, b, c))
        m = sg.Mesh("tri", np.stack([a, b, c]), np.asarray([[0, 1, 2]], np.int32))
        sc = sg.assemble([m], [[(0, 1, sg.make_T(np.eye(3), (0, 0, 0)))]])
        A, B, C = (v.astype(np.float64) for v in (a, b, c))
        # aim just outside edge AB (away from C), and at the three vertices
        w = rng.uniform(0.1, 0.9, 40)
        out_dir = (A + B) / 2 - C
        off = rng.uniform(0.0, 1e-9, 40)[:, None] * out_dir / np.linalg.norm(out_dir)
        tgt = A + w[:, None] * (B - A) + off
        dirs = np.concatenate([tgt, np.stack([A, B, C])]).astype(np.float32)[None]
        r = cast_rays(sc, np.zeros_like(dirs), dirs, max_range=2.0)
        n = np.cross(B - A, C - A)
        M = 2.0 * np.abs(dirs[0]).max() + np.abs(np.stack([A, B, C])).max()
        for i in range(40):
            dd = dirs[0, i].astype(np.float64)
            t = n @ A / (n @ dd)
            dist = _outside_distance(t * dd, A, B, C)
            if dist > 2.0 ** -36 * M:
                assert r.face[i] == -1 and r.amb[i] == 0, (trial, i, dist)
                n_band += dist < 1e-9
            elif dist <= 2.0 ** -46 * M:  # on the edge within rounding: a hit, or a flagged graze
                assert r.face[i] == 0 or r.amb[i] & oracle.AMB_GRAZE, (trial, i, dist)
        for i in range(40, 43):  # vertex-aimed: a hit, or a flagged graze
            assert r.face[i] == 0 or (r.amb[i] & oracle.AMB_GRAZE and r.t2[i] > 0), (trial, i)
            n_vert += 1
    assert n_band > 1000  # these all sat inside the old fixed 1e-9 m band


def test_graze_never_flags_generic_rays():
    """Negative pin of AMB_GRAZE / AMB_TIE: 20 000 random rays through the
    cluttered c2 scene (generic FP32 directions) come nowhere near FP64
    rounding of an edge, so no ray is a graze and almost none a tie (a
    flag that fired on silhouettes or on every edge crossing would fail)."""
    sc, _ = sg.config2(n_envs=4)
    rng = np.random.default_rng(9)
    o = rng.uniform([-1, -3, -2], [1, 3, 2], (4, 5000, 3)).astype(np.float32)
    d = (rng.uniform([2, -3, -1.5], [8, 3, 1.5], (4, 5000, 3)) - o).astype(np.float32)
    r = cast_rays(sc, o, d, max_range=2.0)
    assert (r.face >= 0).mean() > 0.2
    assert not np.any(r.amb & oracle.AMB_GRAZE)
    assert np.count_nonzero(r.amb & oracle.AMB_TIE) <= 2


def _beams_at(points, pose_T=None):
    """Unit beam table [1][K][3] aimed from the sensor origin at `points`."""
    d = np.asarray(points, np.float64)
    d = d / np.linalg.norm(d, axis=1, keepdims=True)
    return d[None].astype(np.float32)


def _shadow_case(occluder, o2, wall_x=2.0, eps=1e-4, ys=None, zs=None):
    """Wall x = wall_x (200 m quad) + one occluder quad; beams (range) from
    the origin aimed at wall points (wall_x, y, z); second sensor at o2."""
    wall = quad_mesh(200.0)
    sc = sg.assemble([wall, occluder], [[(0, 1, sg.make_T(np.eye(3), (wall_x, 0, 0))),
                                         (1, 2, sg.make_T(np.eye(3), (0, 0, 0)))]])
    pts = np.stack([np.full_like(ys, wall_x), ys, zs], 1)
    beams = _beams_at(pts)
    rays = dict(model=oracle.BEAMS, beams=beams, poses=sg.identity_poses(1), max_range=20.0)
    r = oracle.cast(sc, rays, stereo=(tuple(o2), eps))
    # the hit point in FP64 from the FP32 beam (normalised in FP64, reading R19)
    bd = beams[0].astype(np.float64)
    bd = bd / np.linalg.norm(bd, axis=1, keepdims=True)
    p = bd * (wall_x / bd[:, :1])
    u = np.asarray(o2, np.float64) - p
    L = np.linalg.norm(u, axis=1)
    u = u / L[:, None]
    return r, p, u, L


def test_stereo_shadow_flag_at_eps_closed_form():
    """AMB_SHADOW at the self-hit guard: an occluder in the plane y = y0
    (x in [1, wall_x), never crossed by the primary rays, which stay at
    y > y0) crosses each shadow segment at distance s = (p_y - y0) / -u_y
    from its hit point p.  The oracle must flag exactly the rays with
    |s - eps| <= 1e-5 and mark a pixel invalid exactly when eps < s < L - eps
    (reading R21); both sides of the band are pinned, so a
    flag set on every shadowed ray, or on none, fails."""
    y0, eps, wall_x = -0.25, 1e-4, 2.0
    occ = sg.Mesh("occ", np.asarray([[1.0, y0, -1], [wall_x - 1e-7, y0, -1], [wall_x - 1e-7, y0, 1],
                                     [1.0, y0, 1]], np.float32), np.asarray([[0, 1, 2], [0, 2, 3]], np.int32))
    ys = y0 + np.linspace(0.0, 3e-4, 601)
    zs = np.linspace(-0.3, 0.3, 601)
    r, p, u, L = _shadow_case(occ, (0.0, -4.0, 0.0), wall_x, eps, ys, zs)
    assert np.all(r.face >= 0) and np.all(r.seg == 1)  # every beam reaches the wall
    s = (p[:, 1] - y0) / -u[:, 1]
    x_cross = p[:, 0] + s * u[:, 0]
    crosses = (x_cross >= 1.0) & (np.abs(p[:, 2] + s * u[:, 2]) <= 1.0)
    assert crosses.all()
    clear = np.abs(np.abs(s - eps) - 1e-5) > 1e-9  # off the flag band's own edges
    want_flag = np.abs(s - eps) <= 1e-5
    got_flag = (r.amb & oracle.AMB_SHADOW) != 0
    assert np.array_equal(got_flag[clear], want_flag[clear])
    assert want_flag[clear].sum() >= 20 and (~want_flag[clear]).sum() >= 200
    sharp = np.abs(s - eps) > 1e-9
    assert np.array_equal(r.valid[sharp] == 0, ((s > eps) & (s < L - eps))[sharp])
    assert (r.valid == 0).sum() >= 100 and (r.valid == 1).sum() >= 50


def test_stereo_shadow_flag_at_far_end_closed_form():
    """AMB_SHADOW at the far end L - eps: an occluder in the plane
    y = -b + delta just in front of the second sensor o2 = (0, -b, 0) meets
    each segment at distance s' = delta / -u_y before o2; flagged exactly
    when |s' - eps| <= 1e-5, invalid exactly when s' > eps."""
    b, eps, wall_x = 4.0, 1e-4, 2.0
    delta = 1.2e-4 * 0.7
    occ = sg.Mesh("occ", np.asarray([[-1, -b + delta, -1], [1, -b + delta, -1], [1, -b + delta, 1],
                                     [-1, -b + delta, 1]], np.float32), np.asarray([[0, 1, 2], [0, 2, 3]], np.int32))
    delta = float(np.float32(-b + delta)) + b  # the plane's FP32 position
    ys = np.linspace(-0.5, 0.5, 41).repeat(41)
    zs = np.tile(np.linspace(-6.0, 6.0, 41), 41)
    r, p, u, L = _shadow_case(occ, (0.0, -b, 0.0), wall_x, eps, ys, zs)
    assert np.all(r.face >= 0)
    s2 = delta / -u[:, 1]
    clear = np.abs(np.abs(s2 - eps) - 1e-5) > 1e-9
    want_flag = np.abs(s2 - eps) <= 1e-5
    got_flag = (r.amb & oracle.AMB_SHADOW) != 0
    assert np.array_equal(got_flag[clear], want_flag[clear])
    assert want_flag[clear].sum() >= 20 and (~want_flag[clear]).sum() >= 200
    sharp = np.abs(s2 - eps) > 1e-9
    assert np.array_equal(r.valid[sharp] == 0, (s2 > eps)[sharp])
