"""GPU parity: the CUDA path (through the C ABI) against the FP64 oracle,
element by element on seeded inputs (SURVEY.md §8(c) parity rules):
  distance within max(1e-5 m, 1e-6 * ref) on every ray;
  seg / face bit-exact on every ray the oracle does not flag ambiguous.
Small configs are compared in full; BASELINE's full-size configs are cast
in the launch configuration bench.py times and compared on sampled rays.
"""
from __future__ import annotations

import math

import numpy as np
import pytest
import torch

import oracle
import paper_2503_01471_b200 as agr
import scenegen as sg
from helpers import certify_all, compare, compare_extras, oracle_rays, valid_compare
from gpu_util import cast_sensor, dev, make_scene, to_np

pytestmark = pytest.mark.gpu


def _check_full(sc, sensor, kind="depth", what="", **bounds):
    s = make_scene(sc)
    got = to_np(cast_sensor(s, sensor, kind))
    ref = oracle.cast(sc, oracle_rays(sensor, kind))
    res = compare(ref, got["dist"], got["seg"], got["face"], what, **bounds)
    s.close()
    return res, got, ref


@pytest.mark.parametrize("kind", ["depth", "range"])
def test_c1_full(kind):
    sc, sensor = sg.config1()
    res, got, ref = _check_full(sc, sensor, kind, f"c1 {kind}")
    d = got["dist"].reshape(16, 16)
    assert np.all(d[6:10, 6:10] < 3.0) and d[0, 0] == 10.0
    if kind == "depth":
        assert np.all(d[6:10, 6:10] == 2.0)


@pytest.mark.parametrize("kind", ["depth", "range"])
def test_c2_full(kind):
    sc, sensor = sg.config2()
    res, got, ref = _check_full(sc, sensor, kind, f"c2 {kind}")
    assert (ref.face >= 0).mean() > 0.1


def test_axis_aligned_centre_rays():
    """Odd image sizes put the centre column / row rays exactly on the
    sensor axes, so a tile's direction interval touches or straddles 0
    (the packet traversal's sign-change branch) at the env level and, with
    identity / 90-degree-yaw instance transforms, at the object level."""
    sc1, _ = sg.config1()
    c2, _ = sg.config2(n_envs=3)
    per_env = [[(0, 1, sg.make_T(np.eye(3), (0.0, 0.0, 0.0)))],
               [(0, 2, sg.make_T(sg.rot_z(np.pi / 2), (0.0, 0.0, 0.0)))],
               [(0, 3, sg.make_T(np.eye(3), (0.0, 0.0, 0.0))), (1, 4, c2.inst_T[0])]]
    sc = sg.assemble([sc1.meshes[0], c2.meshes[c2.inst_asset[0]]], per_env)
    poses = np.zeros((3, 2, 3, 4), np.float32)
    for e in range(3):
        poses[e, 0] = sg.make_T(np.eye(3), (0.0, 0.0, 0.0))
        poses[e, 1] = sg.make_T(sg.rot_z(np.pi / 2), (2.5, -3.0, 0.0))
    sensor = dict(kind="pinhole", cam=sg.pinhole(33, 17, 90.0), poses=poses, max_range=10.0)
    for kind in ("depth", "range"):
        # rays exactly on the cube faces' diagonals: 63 ties / 4 grazes of 3366
        res, got, ref = _check_full(sc, sensor, kind, f"axis-aligned {kind}", max_amb=100, max_graze=8)
        assert (ref.face >= 0).mean() > 0.05


@pytest.mark.parametrize("scale", [0.01, 100.0])
def test_scaled_scene_and_sensor(scale):
    """The whole c2 scene, the sensor positions and max_range scaled by
    0.01 / 100 (instances then carry scales of 0.005-0.015 / 50-150): the
    error model's bounds scale with the scene, so parity
    holds at the tolerance of the scaled distances."""
    sc, sensor = sg.config2(n_envs=4)
    T = sc.inst_T.astype(np.float64) * scale
    sc = sg.Scene(sc.meshes, sc.env_off, sc.inst_asset, sc.inst_label, T.astype(np.float32))
    rng = np.random.default_rng(21)
    poses = np.zeros((4, 1, 3, 4), np.float32)
    for e in range(4):
        poses[e, 0] = sg.make_T(sg.rot_z(rng.uniform(-0.4, 0.4)), rng.uniform(-0.5, 0.5, 3) * scale)
    sensor = dict(sensor, poses=poses, max_range=10.0 * scale, cam=sg.pinhole(96, 64, 87.0))
    for kind in ("depth", "range"):
        res, got, ref = _check_full(sc, sensor, kind, f"scale {scale} {kind}")
        assert (ref.face >= 0).mean() > 0.1


def test_sensor_on_a_surface():
    """Sensors placed exactly on a face plane of the config-1 cube (x = 2,
    inside the face, on an edge, on a corner) looking in several directions:
    candidates at t = 0 are excluded by the (0, max_range] rule on both
    sides (AMB_ZERO flags them for seg / face), distances must still match."""
    sc, sensor = sg.config1()
    spots = [(2.0, 0.0, 0.0), (2.0, 0.5, 0.0), (2.0, 0.5, 0.5), (2.0, 0.1, -0.2)]
    yaws = [0.0, np.pi, np.pi / 2]
    poses = np.zeros((1, len(spots) * len(yaws), 3, 4), np.float32)
    k = 0
    for p_ in spots:
        for y in yaws:
            poses[0, k] = sg.make_T(sg.rot_z(y), p_)
            k += 1
    sensor = dict(sensor, poses=poses, cam=sg.pinhole(24, 16, 100.0))
    for kind in ("depth", "range"):
        # every ray starts on the face plane: all AMB_ZERO by construction
        res, got, ref = _check_full(sc, sensor, kind, f"on-surface {kind}", max_amb=sensor["poses"].shape[1] * 24 * 16)
        assert res["ambiguous"] > 0


def test_ragged_multisensor_random_poses():
    """Image sizes that are not tile multiples, 2 sensors per env, random poses."""
    sc, sensor = sg.config2(n_envs=6)
    rng = np.random.default_rng(3)
    poses = np.zeros((6, 2, 3, 4), np.float32)
    for e in range(6):
        for k in range(2):
            poses[e, k] = sg.make_T(sg.rot_z(rng.uniform(-0.6, 0.6)) @ sg.rot_y(rng.uniform(-0.3, 0.3)),
                                    rng.uniform([-1, -1, -1], [1, 1, 1]))
    sensor = dict(sensor, poses=poses, cam=sg.pinhole(37, 19, 100.0))
    for kind in ("depth", "range"):
        _check_full(sc, sensor, kind, f"ragged {kind}")


def test_explicit_rays_random():
    sc, _ = sg.config2(n_envs=8)
    rng = np.random.default_rng(7)
    R = 4000
    o = rng.uniform([-1, -3, -2], [4, 3, 2], (8, R, 3)).astype(np.float32)
    tgt = rng.uniform([2, -3, -1.5], [8, 3, 1.5], (8, R, 3))
    d = (tgt - o).astype(np.float32)
    s = make_scene(sc)
    out = s.cast_rays(torch.from_numpy(o).to(dev()), torch.from_numpy(d).to(dev()), 2.0)
    got = to_np(out)
    ref = oracle.cast(sc, dict(model=oracle.RAYS, orig=o, dir=d, max_range=2.0))
    compare(ref, got["dist"], got["seg"], got["face"], "rays")


def _edge_targeted_rays(sc, n_per_env, rng, eps_list=(0.0, 1e-7, -1e-7, 1e-6, -1e-6, 1e-5, -1e-5)):
    """Rays aimed at points on triangle edges and vertices (world space, FP64),
    nudged across the edge by eps (relative to the edge length): the cases
    where an FP32 test could flip hit <-> miss."""
    E = sc.n_envs
    o = np.zeros((E, n_per_env, 3), np.float32)
    d = np.zeros((E, n_per_env, 3), np.float32)
    verts, faces = sc.verts.astype(np.float64), sc.faces
    voff, foff = sc.vert_off, sc.face_off
    for e in range(E):
        j0, j1 = sc.env_off[e], sc.env_off[e + 1]
        for r in range(n_per_env):
            j = rng.integers(j0, j1)
            a = sc.inst_asset[j]
            f = rng.integers(foff[a], foff[a + 1])
            T = sc.inst_T[j].astype(np.float64)
            tri = verts[voff[a] + faces[f]] @ T[:, :3].T + T[:, 3]
            k = rng.integers(0, 3)
            p0, p1, p2 = tri[k], tri[(k + 1) % 3], tri[(k + 2) % 3]
            w = rng.uniform(0, 1) if rng.uniform() < 0.8 else float(rng.integers(0, 2))
            on_edge = p0 + w * (p1 - p0)
            inward = (p2 - on_edge)
            eps = eps_list[rng.integers(0, len(eps_list))]
            target = on_edge + eps * inward
            org = rng.uniform([-1, -3, -2], [1.5, 3, 2])
            o[e, r] = org
            d[e, r] = target - org
    return o, d


def test_edge_and_vertex_targeted_rays():
    """Silhouette and shared-edge rays: the FP32 filter must defer every
    decision it cannot certify, so seg/face stay exact off the near-ties."""
    sc, _ = sg.config2(n_envs=16)
    rng = np.random.default_rng(11)
    o, d = _edge_targeted_rays(sc, 3000, rng)
    s = make_scene(sc)
    got = to_np(s.cast_rays(torch.from_numpy(o).to(dev()), torch.from_numpy(d).to(dev()), 12.0))
    ref = oracle.cast(sc, dict(model=oracle.RAYS, orig=o, dir=d, max_range=12.0))
    # shared-edge rays are ties by construction (11 % of them), never grazes
    # of more than a few
    res = compare(ref, got["dist"], got["seg"], got["face"], "edge rays", max_amb=len(ref.amb) // 5)
    assert res["ambiguous"] > 100  # the generator really produces near-ties


def test_exact_mode_equals_filter_mode():
    """FP32 filter + FP64 arbitration == all-FP64 traversal, bitwise."""
    sc, sensor = sg.config2(n_envs=16)
    s = make_scene(sc)
    a = to_np(cast_sensor(s, sensor, "range"))
    s.set_exact_mode(True)
    b = to_np(cast_sensor(s, sensor, "range"))
    for k in a:
        assert np.array_equal(a[k], b[k]), k


def test_refit_equals_rebuild_and_repeat_is_deterministic():
    """After new transforms, refit (old topology) == rebuild, bitwise; a
    repeated cast is bitwise identical (SURVEY.md §8(c) GPU self-invariants)."""
    sc, sensor = sg.config5(n_envs=32, ring=3)
    ring = sc.extra["ring_T"]
    s = make_scene(sc)
    for step in (1, 2):
        s.set_instance_transforms(torch.from_numpy(ring[step]).to(dev()))
        s.refit()
        a = to_np(cast_sensor(s, sensor, "depth"))
        a2 = to_np(cast_sensor(s, sensor, "depth"))
        s.set_instance_transforms(torch.from_numpy(ring[step]).to(dev()))
        s.build()
        b = to_np(cast_sensor(s, sensor, "depth"))
        for k in a:
            assert np.array_equal(a[k], a2[k]) and np.array_equal(a[k], b[k]), (step, k)
        sc2 = sg.Scene(sc.meshes, sc.env_off, sc.inst_asset, sc.inst_label, ring[step])
        ref = oracle.cast(sc2, oracle_rays(sensor, "depth"))
        compare(ref, a["dist"], a["seg"], a["face"], f"c5 step {step}")


def test_null_channels_and_channel_independence():
    sc, sensor = sg.config2(n_envs=4)
    s = make_scene(sc)
    full = to_np(cast_sensor(s, sensor))
    only_d = to_np(cast_sensor(s, sensor, channels=("dist",)))
    only_f = to_np(cast_sensor(s, sensor, channels=("face",)))
    assert np.array_equal(full["dist"], only_d["dist"])
    assert np.array_equal(full["face"], only_f["face"])


def test_empty_and_single_instance_envs():
    """Envs with 0, 1 and several instances side by side."""
    cube = sg.cube_mesh()
    per_env = [[], [(0, 3, sg.make_T(np.eye(3), (3, 0, 0)))],
               [(0, 4, sg.make_T(sg.rot_z(0.3), (4, 0.5, 0), 1.2)),
                (0, 5, sg.make_T(np.eye(3), (2.5, -0.6, 0.2), 0.5))], []]
    sc = sg.assemble([cube], per_env)
    sensor = dict(kind="pinhole", cam=sg.pinhole(24, 16, 90.0), poses=sg.identity_poses(4),
                  max_range=10.0)
    res, got, ref = _check_full(sc, sensor, "depth", "empty/single")
    assert np.all(got["seg"].reshape(4, -1)[0] == -1) and np.all(got["seg"].reshape(4, -1)[3] == -1)
    assert (got["seg"].reshape(4, -1)[1] == 3).any()


def test_degenerate_faces_and_max_range_boundary():
    v = np.asarray([[0, -5, -5], [0, 5, -5], [0, 5, 5], [0, -5, 5]], np.float32)
    m = sg.Mesh("q", v, np.asarray([[0, 1, 1], [0, 2, 2], [0, 1, 2], [0, 2, 3]], np.int32))
    sc = sg.assemble([m], [[(0, 1, sg.make_T(np.eye(3), (10.0, 0, 0)))],
                           [(0, 2, sg.make_T(np.eye(3), (10.0 + 2e-6, 0, 0)))],
                           [(0, 3, sg.make_T(np.eye(3), (9.99, 0, 0)))]])
    o = np.zeros((3, 64, 3), np.float32)
    rng = np.random.default_rng(1)
    d = np.concatenate([np.ones((3, 64, 1)), rng.uniform(-0.3, 0.3, (3, 64, 2))], -1).astype(np.float32)
    s = make_scene(sc)
    got = to_np(s.cast_rays(torch.from_numpy(o).to(dev()), torch.from_numpy(d).to(dev()), 10.0))
    ref = oracle.cast(sc, dict(model=oracle.RAYS, orig=o, dir=d, max_range=10.0))
    # envs 0 and 1 put the quad within 1e-5 of max_range: their 128 rays are AMB_RANGE
    res = compare(ref, got["dist"], got["seg"], got["face"], "degenerate/max-range", max_amb=128)
    assert res["ambiguous"] == 128
    f = got["face"].reshape(3, 64)
    assert set(np.unique(f[2])) <= {2, 3}


@pytest.mark.parametrize("node_width", [0, 4])
def test_update_meshes_single_and_degenerate_assets(node_width):
    """A batched mesh update over assets that become a single triangle, all
    zero-area (no leaf at all) and ordinary again: the single-leaf and empty
    BLAS roots (BVH4 and BVH8), the top-down builds around them, and the
    casts in every schedule against the oracle."""
    quad = np.asarray([[0, -2, -2], [0, 2, -2], [0, 2, 2], [0, -2, 2]], np.float32)
    faces = np.asarray([[0, 1, 2], [0, 2, 3]], np.int32)
    sph = sg.sphere_mesh(0.8, 2)
    meshes = [sg.Mesh("a", quad, faces), sg.Mesh("b", quad.copy(), faces), sg.Mesh("c", sph.verts, sph.faces)]
    pos = [(4.0, -0.6, 0.0), (5.0, 0.0, 0.0), (6.0, 3.5, 0.0)]
    per_env = [[(a, a + 1, sg.make_T(np.eye(3), pos[a])) for a in range(3)]] * 2  # two envs, all three assets
    sc = sg.assemble(meshes, per_env)
    s = agr.Scene.from_scenegen(sc, device=0, node_width=node_width)
    s.set_instance_transforms(torch.from_numpy(sc.inst_T).to(dev()))
    s.build()
    new = [quad.copy(), quad.copy(), (sph.verts * 1.1).astype(np.float32)]
    new[0][3] = new[0][0]          # face 1 of asset 0 degenerate: one leaf left
    new[1][:] = new[1][0]          # every vertex of asset 1 equal: no leaf at all
    s.update_meshes([0, 1, 2], torch.from_numpy(np.concatenate(new)).to(dev()))
    s.build()
    sc2 = sg.assemble([sg.Mesh(m.name, v, m.faces) for m, v in zip(meshes, new)], per_env)
    sensor = dict(kind="pinhole", cam=sg.pinhole(48, 32, 90.0), poses=sg.identity_poses(2), max_range=20.0)
    ref = oracle.cast(sc2, oracle_rays(sensor, "depth"))
    for mode in (0, 1, 2, 3):
        s.set_traversal(mode)
        got = to_np(cast_sensor(s, sensor, "depth"))
        compare(ref, got["dist"], got["seg"], got["face"], f"degenerate update mode {mode}", max_amb=64)
    assert set(np.unique(ref.seg)) >= {1, 3} and 2 not in set(np.unique(ref.seg))
    s.close()


def test_lidar_beams_small():
    sc, sensor = sg.config4(n_envs=8)
    sensor = dict(sensor, beams=sg.lidar_beams(32, 64))
    _check_full(sc, sensor, "range", "c4 small")


def test_dome_lidar_small():
    sc, sensor = sg.config4(n_envs=4)
    sensor = dict(sensor, beams=sg.dome_beams(16, 48))
    _check_full(sc, sensor, "range", "dome")


@pytest.mark.parametrize("n_envs", [20, 70])
def test_host_buffer_path_equals_device_path(n_envs):
    """agr_cast_pinhole_host (H2D poses, chunked cast, D2H images) gives the
    device path's bytes: one env per chunk (20 envs) and 3-env chunks with a
    ragged last one (70 envs over AGR_E2E_CHUNKS = 32 chunks)."""
    sc, sensor = sg.config2(n_envs=n_envs)
    s = make_scene(sc)
    a = to_np(cast_sensor(s, sensor, "depth"))
    poses = torch.from_numpy(np.ascontiguousarray(sensor["poses"])).pin_memory()
    out = s.cast_pinhole_host(sensor["cam"], poses, sensor["max_range"], agr.AGR_DEPTH)
    for k in a:
        assert np.array_equal(a[k], out[k].numpy().reshape(-1)), k
    if n_envs != 20:
        s.close()
        return
    # pageable host outputs take the staging path
    H, W = sensor["cam"]["H"], sensor["cam"]["W"]
    pageable = {k: torch.empty((20, 1, H, W), dtype=torch.float32 if k == "dist" else torch.int32)
                for k in ("dist", "seg", "face")}
    s.cast_pinhole_host(sensor["cam"], poses.clone(), sensor["max_range"], agr.AGR_DEPTH, out=pageable)
    for k in a:
        assert np.array_equal(a[k], pageable[k].numpy().reshape(-1)), k
    beams = sg.lidar_beams(16, 32)
    sc4, s4sensor = sg.config4(n_envs=5)
    s4 = make_scene(sc4)
    dev_out = to_np(cast_sensor(s4, dict(s4sensor, beams=beams), "range"))
    host_out = s4.cast_beams_host(torch.from_numpy(beams), torch.from_numpy(s4sensor["poses"]),
                                  s4sensor["max_range"])
    for k in dev_out:
        assert np.array_equal(dev_out[k], host_out[k].numpy().reshape(-1)), k


def test_checksums_independent_of_sharding():
    """Per-env checksums of one scene == those of the same envs split into two
    scenes (the 1-GPU vs n-GPU bitwise check, run on one GPU)."""
    sc, sensor = sg.config2(n_envs=12)
    s = make_scene(sc)
    out = cast_sensor(s, sensor)
    per_env = sensor["cam"]["W"] * sensor["cam"]["H"]
    full = s.checksum(out, per_env).cpu().numpy()
    parts = []
    for e0, e1 in ((0, 5), (5, 12)):
        sub = sc.env_slice(e0, e1)
        ss = make_scene(sub)
        o = cast_sensor(ss, dict(sensor, poses=sensor["poses"][e0:e1]))
        parts.append(ss.checksum(o, per_env).cpu().numpy())
    assert np.array_equal(full, np.concatenate(parts))
    assert len(set(full.tolist())) == 12


# ---- BASELINE full-size configs, sampled -------------------------------------

def _sampled(sc, sensor, kind, n_sample, seed, what):
    s = make_scene(sc)
    got = to_np(cast_sensor(s, sensor, kind))
    n = len(got["dist"])
    q = np.random.default_rng(seed).choice(n, n_sample, replace=False)
    ref = oracle.cast(sc, oracle_rays(sensor, kind), query=q)
    res = compare(ref, got["dist"][q], got["seg"][q], got["face"][q], what)
    s.close()
    return res, got


@pytest.mark.slow
def test_c3_full_size_sampled():
    """c3: 1024 envs, 270x480 depth camera, forest (bench workload)."""
    sc, sensor = sg.config3()
    res, got = _sampled(sc, sensor, "depth", 30000, 3, "c3")
    hit = got["face"] >= 0
    assert 0.3 < hit.mean() < 0.99
    # every output is either max range or a plausible depth
    assert np.all((got["dist"] > 0) & (got["dist"] <= 10.0))
    # every one of the 132.7 M rays: the reported hit is on the reported face
    assert certify_all(sc, sensor, "depth", got["dist"], got["seg"], got["face"], "c3") == hit.sum()


def _silhouette_pixels(seg_img):
    """Flat indices of pixels whose segmentation differs from a 4-neighbour
    (both sides of every outline) in [E][S][H][W] images."""
    e = np.zeros(seg_img.shape, bool)
    dx = seg_img[..., :, 1:] != seg_img[..., :, :-1]
    dy = seg_img[..., 1:, :] != seg_img[..., :-1, :]
    e[..., :, 1:] |= dx
    e[..., :, :-1] |= dx
    e[..., 1:, :] |= dy
    e[..., :-1, :] |= dy
    return np.flatnonzero(e)


@pytest.mark.slow
def test_c3_bench_step_exact_equals_filter_and_silhouettes():
    """Full-size optimality evidence in the launch configuration bench.py
    times (binned-SAH TLAS built once, then set_instance_transforms + refit,
    interval-packet traversal): (a) the all-FP64 per-lane traversal (exact
    mode: every leaf tested in FP64, a different traversal order) equals
    the FP32-filter packet cast bitwise on all 132.7 M c3 rays -- no ray
    loses a closer hit to the FP32 filter or the packet culling; (b) 50 000
    silhouette pixels (a 4-neighbour with another segment: where a culled
    closer hit would show) against the oracle.  The oracle's inputs are the
    scene and the ray ids; the GPU image only chooses which rays to ask."""
    sc, sensor = sg.config3()
    s = make_scene(sc, build=False)
    s.set_tlas_builder(1)
    s.build()
    s.set_instance_transforms(torch.from_numpy(sc.inst_T).to(dev()))  # the bench step
    s.refit()
    a = cast_sensor(s, sensor, "depth")
    s.set_exact_mode(True)
    b = cast_sensor(s, sensor, "depth")
    s.set_exact_mode(False)
    for k in a:
        assert torch.equal(a[k], b[k]), k
    del b
    seg = a["seg"].cpu().numpy()
    got = to_np(a)
    sil = _silhouette_pixels(seg)
    assert len(sil) > 1_000_000
    q = np.random.default_rng(33).choice(sil, 50000, replace=False)
    ref = oracle.cast(sc, oracle_rays(sensor, "depth"), query=q)
    res = compare(ref, got["dist"][q], got["seg"][q], got["face"][q], "c3 silhouettes")
    print("c3 silhouettes:", res)
    s.close()


@pytest.mark.slow
def test_c4_full_size_sampled():
    sc, sensor = sg.config4()
    _, got = _sampled(sc, sensor, "range", 40000, 4, "c4")
    certify_all(sc, sensor, "range", got["dist"], got["seg"], got["face"], "c4")


@pytest.mark.slow
def test_c5_sampled_with_refit_steps():
    """c5 (per GPU at 8 GPUs: 2048 envs), obstacles re-posed every step."""
    sc, sensor = sg.config5(n_envs=2048, ring=4)
    ring = sc.extra["ring_T"]
    s = make_scene(sc)
    rng = np.random.default_rng(5)
    for step in range(1, 4):
        s.set_instance_transforms(torch.from_numpy(ring[step]).to(dev()))
        s.refit()
        got = to_np(cast_sensor(s, sensor, "depth"))
        q = rng.choice(len(got["dist"]), 20000, replace=False)
        sc2 = sg.Scene(sc.meshes, sc.env_off, sc.inst_asset, sc.inst_label, ring[step])
        ref = oracle.cast(sc2, oracle_rays(sensor, "depth"), query=q)
        compare(ref, got["dist"][q], got["seg"][q], got["face"][q], f"c5 step {step}")
        certify_all(sc2, sensor, "depth", got["dist"], got["seg"], got["face"], f"c5 step {step}")


def _flat(out):
    return {k: v.reshape(-1) for k, v in out.items()}


@pytest.mark.slow
def test_c5_bench_step_full_size():
    """c5 at its stated 16384 envs in bench.py's launch configuration: every
    step sets a new transform set and rebuilds the LBVH TLAS (warp-per-env
    build with the SAH-optimal BVH8 collapse), then casts; in step 1 exact
    mode == filter mode bitwise on all 530.8 M rays and 20 000 silhouette rays
    against the oracle; 20 000 sampled rays per step against the oracle and
    every ray of the first 2048 envs certified."""
    sc, sensor = sg.config5(n_envs=16384, ring=3)
    ring = sc.extra["ring_T"]
    s = make_scene(sc, build=False)
    s.set_tlas_builder(0)
    poses = torch.from_numpy(np.ascontiguousarray(sensor["poses"])).to(dev())
    rng = np.random.default_rng(11)
    E_cert = 2048
    per_env = sensor["cam"]["W"] * sensor["cam"]["H"]
    for step in (1, 2):
        s.set_instance_transforms(torch.from_numpy(ring[step]).to(dev()))
        s.build()
        img = s.cast_pinhole(sensor["cam"], poses, sensor["max_range"], agr.AGR_DEPTH)
        sc2 = sg.Scene(sc.meshes, sc.env_off, sc.inst_asset, sc.inst_label, ring[step])
        if step == 1:
            # exact mode == the filtered packet cast on all 530.8 M rays, and
            # 20 000 silhouette rays against the oracle
            s.set_exact_mode(True)
            ex = s.cast_pinhole(sensor["cam"], poses, sensor["max_range"], agr.AGR_DEPTH)
            s.set_exact_mode(False)
            for k in img:
                assert torch.equal(img[k], ex[k]), k
            del ex
            sil = _silhouette_pixels(img["seg"].cpu().numpy())
            qs = np.random.default_rng(14).choice(sil, 20000, replace=False)
            qst = torch.from_numpy(qs).to(dev())
            ref = oracle.cast(sc2, oracle_rays(sensor, "depth"), query=qs)
            compare(ref, img["dist"].reshape(-1)[qst].cpu().numpy(), img["seg"].reshape(-1)[qst].cpu().numpy(),
                    img["face"].reshape(-1)[qst].cpu().numpy(), "c5 silhouettes")
        out = _flat(img)
        del img
        n = out["dist"].numel()
        q = rng.choice(n, 20000, replace=False)
        qt = torch.from_numpy(q).to(dev())
        got = {k: v[qt].cpu().numpy() for k, v in out.items()}
        ref = oracle.cast(sc2, oracle_rays(sensor, "depth"), query=q)
        compare(ref, got["dist"], got["seg"], got["face"], f"c5 full step {step}")
        head = {k: v[: E_cert * per_env].cpu().numpy() for k, v in out.items()}
        sub = sc2.env_slice(0, E_cert)
        sen = dict(sensor, poses=sensor["poses"][:E_cert])
        assert certify_all(sub, sen, "depth", head["dist"], head["seg"], head["face"], f"c5 step {step}") > 0
        del out
    s.close()


@pytest.mark.slow
def test_c4_bench_step_full_size():
    """c4 at its stated 4096 envs in bench.py's launch configuration (SAH
    TLAS built once, transforms set + refit, interval packets on the BVH8):
    exact mode == filter mode bitwise on all 268 M beams, 20 000 silhouette
    beams and 40 000 sampled beams against the oracle, and every ray of the
    first 1024 envs certified."""
    sc, sensor = sg.config4()
    s = make_scene(sc, build=False)
    s.set_tlas_builder(1)
    s.build()
    s.set_instance_transforms(torch.from_numpy(sc.inst_T).to(dev()))
    s.refit()
    beams = torch.from_numpy(np.ascontiguousarray(sensor["beams"])).to(dev())
    poses = torch.from_numpy(np.ascontiguousarray(sensor["poses"])).to(dev())
    img = s.cast_beams(beams, poses, sensor["max_range"])
    # exact mode (all-FP64 per-lane traversal) == the filtered packet cast on
    # all 268 M beams, and 20 000 silhouette beams against the oracle
    s.set_exact_mode(True)
    ex = s.cast_beams(beams, poses, sensor["max_range"])
    s.set_exact_mode(False)
    for k in img:
        assert torch.equal(img[k], ex[k]), k
    del ex
    out = _flat(img)
    sil = _silhouette_pixels(img["seg"].cpu().numpy())
    qs = np.random.default_rng(13).choice(sil, 20000, replace=False)
    qst = torch.from_numpy(qs).to(dev())
    ref = oracle.cast(sc, oracle_rays(sensor, "range"), query=qs)
    compare(ref, out["dist"][qst].cpu().numpy(), out["seg"][qst].cpu().numpy(), out["face"][qst].cpu().numpy(),
            "c4 silhouettes")
    q = np.random.default_rng(12).choice(out["dist"].numel(), 40000, replace=False)
    qt = torch.from_numpy(q).to(dev())
    got = {k: v[qt].cpu().numpy() for k, v in out.items()}
    ref = oracle.cast(sc, oracle_rays(sensor, "range"), query=q)
    compare(ref, got["dist"], got["seg"], got["face"], "c4 full bench step")
    E_cert = 1024
    per_env = sensor["beams"].shape[0] * sensor["beams"].shape[1]
    head = {k: v[: E_cert * per_env].cpu().numpy() for k, v in out.items()}
    sen = dict(sensor, poses=sensor["poses"][:E_cert])
    assert certify_all(sc.env_slice(0, E_cert), sen, "range", head["dist"], head["seg"], head["face"], "c4") > 0
    s.close()


# ---- per-hit channels (normal, barycentrics, point cloud) -------------------

ALL = ("dist", "seg", "face", "normal", "bary", "point")


@pytest.mark.parametrize("kind", ["depth", "range"])
def test_extras_c2_full(kind):
    """Normals facing the sensor, barycentrics and points vs the oracle
    (PAPER.md:218 Fig. 3a normals; :228 barycentrics, point clouds)."""
    sc, sensor = sg.config2(n_envs=16)
    s = make_scene(sc)
    got = to_np(cast_sensor(s, sensor, kind, channels=ALL))
    ref = oracle.cast(sc, oracle_rays(sensor, kind), extras=True)
    compare(ref, got["dist"], got["seg"], got["face"], f"extras {kind}")
    n = compare_extras(ref, got["normal"], got["bary"], got["point"], got["face"], f"extras {kind}")
    assert n > 10000
    # the extras do not change the core channels
    core = to_np(cast_sensor(s, sensor, kind))
    for k in core:
        assert np.array_equal(core[k], got[k]), k


def test_extras_lidar_and_rays():
    sc, sensor = sg.config4(n_envs=6)
    sensor = dict(sensor, beams=sg.lidar_beams(24, 64))
    s = make_scene(sc)
    got = to_np(cast_sensor(s, sensor, "range", channels=ALL))
    ref = oracle.cast(sc, oracle_rays(sensor, "range"), extras=True)
    compare(ref, got["dist"], got["seg"], got["face"], "lidar extras")
    compare_extras(ref, got["normal"], got["bary"], got["point"], got["face"], "lidar extras")
    sc2, _ = sg.config2(n_envs=4)
    rng = np.random.default_rng(17)
    o, d = _edge_targeted_rays(sc2, 2000, rng)
    s2 = make_scene(sc2)
    out = s2.cast_rays(torch.from_numpy(o).to(dev()), torch.from_numpy(d).to(dev()), 12.0, channels=ALL)
    got = to_np(out)
    ref = oracle.cast(sc2, dict(model=oracle.RAYS, orig=o, dir=d, max_range=12.0), extras=True)
    compare(ref, got["dist"], got["seg"], got["face"], "edge extras", max_amb=len(ref.amb) // 5)
    compare_extras(ref, got["normal"], got["bary"], got["point"], got["face"], "edge extras")


def test_extras_host_path():
    sc, sensor = sg.config2(n_envs=9)
    s = make_scene(sc)
    a = to_np(cast_sensor(s, sensor, "range", channels=ALL))
    poses = torch.from_numpy(np.ascontiguousarray(sensor["poses"])).pin_memory()
    out = s.cast_pinhole_host(sensor["cam"], poses, sensor["max_range"], agr.AGR_RANGE, channels=ALL)
    for k in a:
        assert np.array_equal(a[k], out[k].numpy().reshape(-1)), k


# ---- f2: stereo shadow mask --------------------------------------------------------

@pytest.mark.parametrize("baseline", [0.095, 0.5])
def test_stereo_mask_c2(baseline):
    """Stereo shadow mask vs the oracle on c2 envs."""
    sc, sensor = sg.config2(n_envs=12)
    s = make_scene(sc)
    s.set_stereo((0.0, -baseline, 0.0), 1e-4)
    got = to_np(cast_sensor(s, sensor, "depth", channels=("dist", "seg", "face", "valid")))
    ref = oracle.cast(sc, oracle_rays(sensor, "depth"), stereo=((0.0, -baseline, 0.0), 1e-4))
    compare(ref, got["dist"], got["seg"], got["face"], "stereo")
    n_shadow = valid_compare(ref, got["valid"], f"stereo b={baseline}")
    assert n_shadow > 100
    # the mask does not change the other channels
    core = to_np(cast_sensor(s, sensor, "depth"))
    for k in core:
        assert np.array_equal(core[k], got[k]), k


def test_stereo_mask_lidar_and_lane_mode():
    sc, sensor = sg.config4(n_envs=4)
    sensor = dict(sensor, beams=sg.lidar_beams(16, 64))
    s = make_scene(sc)
    s.set_stereo((0.0, 0.0, 0.3), 1e-4)
    chans = ("dist", "seg", "face", "valid")
    got = to_np(cast_sensor(s, sensor, "range", channels=chans))
    ref = oracle.cast(sc, oracle_rays(sensor, "range"), stereo=((0.0, 0.0, 0.3), 1e-4))
    valid_compare(ref, got["valid"], "lidar stereo")
    s.set_traversal(1)
    lane = to_np(cast_sensor(s, sensor, "range", channels=chans))
    for k in got:
        assert np.array_equal(got[k], lane[k]), k


def test_tlas_builders_sah_and_lbvh_agree():
    """The LBVH TLAS (default) and the binned-SAH TLAS give bitwise identical
    images (the BVH only accelerates the plain definition); c3-shaped envs."""
    sc, sensor = sg.config3(n_envs=6)
    s = make_scene(sc)
    a = to_np(cast_sensor(s, sensor, "depth"))
    s.set_tlas_builder(1)
    s.build()
    b = to_np(cast_sensor(s, sensor, "depth"))
    for k in a:
        assert np.array_equal(a[k], b[k]), k
    q = np.random.default_rng(2).choice(len(a["dist"]), 20000, replace=False)
    ref = oracle.cast(sc, oracle_rays(sensor, "depth"), query=q)
    compare(ref, a["dist"][q], a["seg"][q], a["face"][q], "c3 small SAH TLAS")


# ---- f4: sensor presets ----------------------------------------------------------------

@pytest.mark.parametrize("name", sorted(sg.PRESETS))
def test_sensor_presets_match_oracle(name):
    """Every preset of PAPER.md:228 runs through the cast and matches the
    oracle on a c4-shaped room (sampled rays)."""
    sc, sensor = sg.config4(n_envs=3)
    p = sg.preset(name)
    sensor = dict(sensor, kind=p["kind"])
    if p["kind"] == "pinhole":
        sensor["cam"] = p["cam"]
        kind = "range"
    else:
        sensor["beams"] = p["beams"]
        kind = "range"
    s = make_scene(sc)
    got = to_np(cast_sensor(s, sensor, kind))
    n = len(got["dist"])
    q = np.random.default_rng(3).choice(n, min(n, 6000), replace=False)
    ref = oracle.cast(sc, oracle_rays(sensor, kind), query=q)
    compare(ref, got["dist"][q], got["seg"][q], got["face"][q], name)


# ---- f3: per-env unique / deforming meshes ------------------------------------------

def test_update_mesh_per_env_unique_and_deforming():
    """Per-env unique meshes (one asset per env) re-randomised at reset by
    agr_update_mesh: the rebuilt BLAS + refreshed instance
    bounds + TLAS give the oracle's images for the new vertices, including
    faces that become degenerate / non-degenerate."""
    rng = np.random.default_rng(8)
    E = 4
    meshes = [sg.sphere_mesh(0.8, 2, name=f"blob{e}") for e in range(E)]
    per_env = [[(e, 1, sg.make_T(np.eye(3), (3.0, 0.0, 0.0)))] for e in range(E)]
    sc = sg.assemble(meshes, per_env)
    cam = sg.pinhole(64, 48, 70.0)
    sensor = dict(kind="pinhole", cam=cam, poses=sg.identity_poses(E), max_range=10.0)
    s = make_scene(sc)
    for step in range(3):
        new_meshes = []
        for e in range(E):
            v = meshes[e].verts.astype(np.float64)
            v = v * rng.uniform(0.7, 1.3, (len(v), 1)) + rng.uniform(-0.2, 0.2, 3)
            if step == 1:
                v[meshes[e].faces[:5, 1]] = v[meshes[e].faces[:5, 0]]  # some zero-area faces
            vf = v.astype(np.float32)
            new_meshes.append(sg.Mesh(meshes[e].name, vf, meshes[e].faces))
            s.update_mesh(e, torch.from_numpy(vf).to(dev()))
        s.build() if step != 2 else s.refit()
        got = to_np(cast_sensor(s, sensor, "range"))
        sc2 = sg.assemble(new_meshes, per_env)
        ref = oracle.cast(sc2, oracle_rays(sensor, "range"))
        compare(ref, got["dist"], got["seg"], got["face"], f"update step {step}")
    # the binary LBVH export is packed by the create-time build only: after
    # an update it is refused (ESTATE), the leaf order stays available
    with pytest.raises(agr.AgrError, match="create-time"):
        s.debug_export_blas(0)


def _bvh4_canonical(nodes, root):
    """A BLAS BVH4 export as a nested tuple from its root (child boxes as
    bits, leaf refs as stored, internal children recursively): equal for
    equal trees whatever the node numbering."""
    refs = nodes[:, 24:28].view(np.int32)
    bits = nodes[:, :24].view(np.uint32)

    def rec(n):
        out = [bits[n].tobytes()]
        for r in refs[n]:
            out.append(rec(int(r) - root) if r >= 0 else int(r))
        return tuple(out)
    return rec(0)


def test_update_meshes_batched_equals_one_by_one():
    """agr_update_meshes rebuilds several assets of different sizes in one
    batch: every asset's BVH4 is bit-identical to the one agr_update_mesh
    builds alone (the segmented sort keeps each asset's leaf order), the
    untouched assets are unchanged, and the cast matches the oracle."""
    rng = np.random.default_rng(9)
    E = 6
    meshes = [sg.sphere_mesh(0.6 + 0.1 * e, 1 + e % 3, name=f"blob{e}") for e in range(E)]
    per_env = [[(e, e + 1, sg.make_T(sg.rot_z(rng.uniform(0, 6.28)), (3.0, 0.0, 0.2)))] for e in range(E)]
    sc = sg.assemble(meshes, per_env)
    sa, sb = make_scene(sc), make_scene(sc)
    which = [4, 1, 5, 2]
    new = {}
    for a in which:
        v = meshes[a].verts.astype(np.float64)
        new[a] = (v * rng.uniform(0.8, 1.2, (len(v), 1)) + rng.uniform(-0.2, 0.2, 3)).astype(np.float32)
    before = [sa.debug_export_bvh4(a) for a in range(E)]
    sa.update_meshes(which, torch.from_numpy(np.concatenate([new[a] for a in which])).to(dev()))
    for a in which:
        sb.update_mesh(a, torch.from_numpy(new[a]).to(dev()))
    torch.cuda.synchronize()
    for a in range(E):
        # the BVH4 node numbering depends on the build's schedule (blas.cu
        # K5b'); the tree -- boxes, leaves and shape from the root -- does not
        ca, cb = _bvh4_canonical(*sa.debug_export_bvh4(a)), _bvh4_canonical(*sb.debug_export_bvh4(a))
        assert ca == cb, f"asset {a}"
        if a not in which:
            assert ca == _bvh4_canonical(*before[a])
    sa.build()
    cam = sg.pinhole(48, 32, 70.0)
    sensor = dict(kind="pinhole", cam=cam, poses=sg.identity_poses(E), max_range=10.0)
    got = to_np(cast_sensor(sa, sensor, "depth"))
    sc2 = sg.assemble([sg.Mesh(m.name, new.get(a, m.verts), m.faces) for a, m in enumerate(meshes)], per_env)
    ref = oracle.cast(sc2, oracle_rays(sensor, "depth"))
    compare(ref, got["dist"], got["seg"], got["face"], "update_meshes")
    assert (got["face"] >= 0).mean() > 0.05
    v = torch.zeros((len(meshes[1].verts) * 2, 3), device=dev())
    with pytest.raises(agr.AgrError):
        sa.update_meshes([1, 1], v)
    with pytest.raises(agr.AgrError):
        sa.update_meshes([E], v)


def test_c6_unique_terrain_reset_small():
    """c6 shape at small size: one unique terrain asset
    per env, every env's mesh replaced at reset by one agr_update_meshes
    batch; full oracle parity before and after the reset."""
    sc, sensor = sg.config6(n_envs=6, ring=2, n=24)
    sensor = dict(sensor, cam=sg.pinhole(40, 24, 87.0))
    s = make_scene(sc)
    s.set_tlas_builder(0)
    got = to_np(cast_sensor(s, sensor, "depth"))
    ref = oracle.cast(sc, oracle_rays(sensor, "depth"))
    compare(ref, got["dist"], got["seg"], got["face"], "c6 before reset")
    assert (got["face"] >= 0).mean() > 0.5
    ring = sc.extra["ring_V"]
    s.update_meshes(list(range(6)), torch.from_numpy(ring[1]).to(dev()))
    s.build()
    got = to_np(cast_sensor(s, sensor, "depth"))
    V = len(sc.meshes[0].verts)
    sc2 = sg.assemble([sg.Mesh(m.name, ring[1][i * V:(i + 1) * V], m.faces) for i, m in enumerate(sc.meshes)],
                      [[(i, 1, sc.inst_T[i])] for i in range(6)])
    ref = oracle.cast(sc2, oracle_rays(sensor, "depth"))
    compare(ref, got["dist"], got["seg"], got["face"], "c6 after reset")


@pytest.mark.slow
def test_c6_full_size_lane_mode_after_update():
    """c6 at bench size in the bench's launch configuration: 256 unique
    32768-triangle terrains, every mesh replaced by one agr_update_meshes
    batch (plain LBVH), LBVH TLAS rebuilt, one ray per lane; sampled oracle
    parity plus the per-ray certificate of all 8.3 M rays."""
    sc, sensor = sg.config6()
    s = make_scene(sc, trbvh_rounds=0)
    s.set_tlas_builder(0)
    s.set_traversal(1)
    ring = sc.extra["ring_V"]
    s.update_meshes(list(range(sc.n_envs)), torch.from_numpy(ring[1]).to(dev()))
    s.build()
    got = to_np(cast_sensor(s, sensor, "depth"))
    V = len(sc.meshes[0].verts)
    sc2 = sg.assemble([sg.Mesh(m.name, ring[1][i * V:(i + 1) * V], m.faces) for i, m in enumerate(sc.meshes)],
                      [[(i, 1, sc.inst_T[i])] for i in range(sc.n_envs)])
    q = np.random.default_rng(6).choice(len(got["dist"]), 20000, replace=False)
    ref = oracle.cast(sc2, oracle_rays(sensor, "depth"), query=q)
    compare(ref, got["dist"][q], got["seg"][q], got["face"][q], "c6 full size")
    hit = got["face"] >= 0
    assert hit.mean() > 0.5
    assert certify_all(sc2, sensor, "depth", got["dist"], got["seg"], got["face"], "c6") == hit.sum()
    s.close()


# ---- f1: interpolated vertex annotations -------------------------------------------

def _c2_annotations(sc, rng):
    """k = 3 annotations: random values on the cube, the object-space
    coordinates (a linear field) on the cylinder, none on the panel."""
    cube, cyl, _ = sc.meshes
    return [rng.uniform(-5, 5, (len(cube.verts), 3)).astype(np.float32),
            cyl.verts.astype(np.float32).copy(), None]


@pytest.mark.parametrize("kind", ["depth", "range"])
def test_annotations_c2_vs_oracle(kind):
    """Interpolated vertex annotations against the oracle on
    every ray whose face equals the oracle's; NaN on misses and on the
    un-annotated panel."""
    sc, sensor = sg.config2(n_envs=16)
    s = make_scene(sc)
    A = _c2_annotations(sc, np.random.default_rng(17))
    for a, vals in enumerate(A):
        if vals is not None:
            s.set_vertex_annotations(a, torch.from_numpy(vals).to(dev()))
    got = to_np(cast_sensor(s, sensor, kind, channels=("dist", "seg", "face", "annot")))
    ref = oracle.cast(sc, oracle_rays(sensor, kind), annot=A)
    compare(ref, got["dist"], got["seg"], got["face"], "annot")
    ann = got["annot"].reshape(-1, 3)
    same = got["face"] == ref.face
    finite = np.isfinite(ref.annot).all(1)
    assert np.array_equal(np.isfinite(ann).all(1)[same], finite[same])
    err = np.abs(ann[same & finite] - ref.annot[same & finite])
    assert err.max() <= 1e-5 * (1.0 + np.abs(ref.annot[same & finite]).max()), err.max()
    assert (same & finite).sum() > 10000 and (same & ~finite & (ref.face >= 0)).sum() > 100


def test_annotations_host_path_and_errors():
    sc, sensor = sg.config2(n_envs=5)
    s = make_scene(sc)
    with pytest.raises(agr.AgrError):  # no annotations set yet
        cast_sensor(s, sensor, "depth", channels=("dist", "annot"))
    A = _c2_annotations(sc, np.random.default_rng(3))
    s.set_vertex_annotations(0, torch.from_numpy(A[0]).to(dev()))
    with pytest.raises(agr.AgrError):  # k differs from the scene's
        s.set_vertex_annotations(1, torch.from_numpy(A[1][:, :2].copy()).to(dev()))
    with pytest.raises(agr.AgrError):  # vertex count mismatch
        s.set_vertex_annotations(1, torch.from_numpy(A[0]).to(dev()))
    dev_out = to_np(cast_sensor(s, sensor, "depth", channels=("dist", "face", "annot")))
    poses = torch.from_numpy(np.ascontiguousarray(sensor["poses"])).pin_memory()
    host = s.cast_pinhole_host(sensor["cam"], poses, sensor["max_range"], agr.AGR_DEPTH,
                               channels=("dist", "face", "annot"))
    for k in dev_out:
        assert np.array_equal(dev_out[k], host[k].numpy().reshape(-1), equal_nan=True), k


# ---- maximum sizes ---------------------------------------------------------------

@pytest.mark.parametrize("n", [300, 1024])
@pytest.mark.parametrize("builder", [0, 1])
def test_max_instances_per_env(builder, n):
    """AGR_MAX_INSTANCES_PER_ENV (1024) instances in one env -- the largest
    one-CTA TLAS build -- and 300 (a CTA build whose shared memory crosses
    48 KB only with the static part counted), with both TLAS builders,
    rebuild and refit, against the oracle; one more instance is
    EUNSUPPORTED."""
    rng = np.random.default_rng(41)
    per_env = []
    for e in range(2):
        insts = []
        for j in range(n if e == 0 else 37):
            T = sg.make_T(sg.random_rotation(rng), rng.uniform([2, -6, -4], [14, 6, 4]), rng.uniform(0.1, 0.4))
            insts.append((j % 2, j + 1, T))
        per_env.append(insts)
    sc = sg.assemble([sg.cube_mesh(), sg.panel_mesh()], per_env)
    cam = sg.pinhole(48, 32, 90.0)
    sensor = dict(kind="pinhole", cam=cam, poses=sg.identity_poses(2), max_range=20.0)
    s = make_scene(sc, build=False)
    s.set_tlas_builder(builder)
    s.build()
    got = to_np(cast_sensor(s, sensor, "range"))
    ref = oracle.cast(sc, oracle_rays(sensor, "range"))
    compare(ref, got["dist"], got["seg"], got["face"], f"{n} instances, builder {builder}")
    assert (got["face"][: cam["W"] * cam["H"]] >= 0).mean() > (0.3 if n == 1024 else 0.1)
    assert s.info()["n_instances"] == n + 37
    # re-pose everything and refit (topology kept)
    T2 = sc.inst_T.copy()
    T2[:, :, 3] += rng.uniform(-0.3, 0.3, (len(T2), 3)).astype(np.float32)
    s.set_instance_transforms(torch.from_numpy(T2).to(dev()))
    s.refit()
    got = to_np(cast_sensor(s, sensor, "range"))
    sc2 = sg.Scene(sc.meshes, sc.env_off, sc.inst_asset, sc.inst_label, T2)
    ref = oracle.cast(sc2, oracle_rays(sensor, "range"))
    compare(ref, got["dist"], got["seg"], got["face"], f"{n} instances after refit")
    if n == 1024:
        with pytest.raises(agr.AgrError):
            sg_over = sg.assemble([sg.cube_mesh()], [[(0, 1, sg.make_T(np.eye(3), (3, 0, 0)))] * (n + 1)])
            agr.Scene.from_scenegen(sg_over, device=0)


def test_large_image_sampled():
    """A 1920x1080 frame (2.07 M rays, one env, 2 sensors: grid of 129600
    warps) against the oracle on sampled rays, plus the full certificate."""
    sc, _ = sg.config2(n_envs=1)
    cam = sg.pinhole(1920, 1080, 100.0)
    P = sg.identity_poses(1, 2)
    P[0, 1, :, :3] = sg.rot_z(0.3)
    sensor = dict(kind="pinhole", cam=cam, poses=P, max_range=10.0)
    s = make_scene(sc)
    got = to_np(cast_sensor(s, sensor, "depth"))
    q = np.random.default_rng(5).choice(len(got["dist"]), 20000, replace=False)
    ref = oracle.cast(sc, oracle_rays(sensor, "depth"), query=q)
    compare(ref, got["dist"][q], got["seg"][q], got["face"][q], "1080p")
    certify_all(sc, sensor, "depth", got["dist"], got["seg"], got["face"], "1080p")


# ---- ordering and degenerate instances ---------------------------------

def test_host_cast_waits_for_scene_work_on_the_caller_stream():
    """agr_cast_pinhole_host runs on internal streams: it must wait for a
    refit still queued on the caller's stream (delayed here by a long
    sleep kernel) without a caller-side sync, and return the images of the
    new transforms."""
    sc, sensor = sg.config5(n_envs=16, ring=2)
    ring = sc.extra["ring_T"]
    s = make_scene(sc)
    T1 = torch.from_numpy(ring[1]).to(dev())
    poses = torch.from_numpy(np.ascontiguousarray(sensor["poses"])).pin_memory()
    torch.cuda.synchronize()
    torch.cuda._sleep(200_000_000)  # ~0.1 s of GPU time ahead of the update
    s.set_instance_transforms(T1)
    s.refit()
    host = s.cast_pinhole_host(sensor["cam"], poses, sensor["max_range"], agr.AGR_DEPTH)
    dev_out = to_np(cast_sensor(s, sensor, "depth"))
    for k in dev_out:
        assert np.array_equal(dev_out[k], host[k].numpy().reshape(-1)), k
    sc2 = sg.Scene(sc.meshes, sc.env_off, sc.inst_asset, sc.inst_label, ring[1])
    ref = oracle.cast(sc2, oracle_rays(sensor, "depth"))
    compare(ref, host["dist"].numpy().reshape(-1), host["seg"].numpy().reshape(-1),
            host["face"].numpy().reshape(-1), "host cast after queued refit")
    with pytest.raises(agr.AgrError, match="kind"):
        s.cast_pinhole_host(sensor["cam"], poses, sensor["max_range"], 7)


def test_singular_instance_keeps_tlas_boxes_tight():
    """An instance hidden by a zero scale (a common reset trick) is never
    hit and must not widen its TLAS ancestors' boxes to infinity: the env's
    TLAS boxes stay finite, and the images match the oracle."""
    cube = sg.cube_mesh()
    Z = sg.make_T(np.eye(3), (3.0, 0.0, 0.0), 0.0)
    per_env = [[(0, 1, sg.make_T(np.eye(3), (3.0, 0.5, 0.0))), (0, 2, Z),
                (0, 3, sg.make_T(sg.rot_z(0.4), (5.0, -1.0, 0.3))), (0, 4, Z), (0, 5, Z)]]
    sc = sg.assemble([cube], per_env)
    sensor = dict(kind="pinhole", cam=sg.pinhole(64, 48, 90.0), poses=sg.identity_poses(1), max_range=10.0)
    for builder in (0, 1):
        s = make_scene(sc, build=False)
        s.set_tlas_builder(builder)
        s.build()
        nodes, root = s.debug_export_bvh4(-1)
        f = nodes.reshape(-1, 8, 4)
        boxes = f[:, :6, :].transpose(0, 2, 1)  # [node][child][lo.x hi.x lo.y hi.y lo.z hi.z]
        refs = f[:, 6, :].view(np.int32)
        used = refs != np.int32(-2 ** 31)
        b = boxes[used]
        # every child box is finite (and small) or the all-+inf never-hit
        # sentinel of an empty subtree -- never half-infinite
        fin = np.isfinite(b).all(1)
        assert np.all(fin | (b == np.inf).all(1)), builder
        assert fin.sum() >= 2 and np.abs(b[fin]).max() < 10.0, builder
        got = to_np(cast_sensor(s, sensor, "depth"))
        ref = oracle.cast(sc, oracle_rays(sensor, "depth"))
        compare(ref, got["dist"], got["seg"], got["face"], f"singular instances, builder {builder}")
        assert set(np.unique(got["seg"])) <= {-1, 1, 3}


# ---- asset parts: one BLAS per connected-component group ---------------

def _faces_sharing_a_vertex_share_a_part(mesh, part):
    first = {}
    for f, tri in enumerate(mesh.faces):
        for v in tri:
            if int(v) in first and part[first[int(v)]] != part[f]:
                return False
            first.setdefault(int(v), f)
    return True


def test_asset_parts_partition():
    """A tree (open trunk + canopy: two connected components whose boxes
    fill far less than their union box) is split into 2 BLAS parts; a face
    never leaves its component's part; single-component assets and triangle
    soups (> 64 components) stay whole; part_policy 1 never splits."""
    rng = np.random.default_rng(1)
    tree = sg.tree_mesh(rng)
    rock = sg.rock_mesh(rng)
    tris = rng.uniform(-1, 1, (80, 3, 3)).astype(np.float32)
    soup = sg.Mesh("soup", tris.reshape(-1, 3), np.arange(240, dtype=np.int32).reshape(-1, 3))
    meshes = [tree, rock, sg.cube_mesh(), soup]
    sc = sg.assemble(meshes, [[(a, a + 1, sg.make_T(np.eye(3), (3.0 * a, 0, 0))) for a in range(4)]])
    s = make_scene(sc)
    n, part = s.debug_asset_parts(0, len(tree.faces))
    assert n == 2 and set(part.tolist()) == {0, 1}
    assert _faces_sharing_a_vertex_share_a_part(tree, part)
    trunk = part == part[0]
    assert trunk.sum() == 32 and (~trunk).sum() == 1280  # 16-segment trunk, icosphere-3 canopy
    for a in (1, 2, 3):
        assert s.debug_asset_parts(a, len(meshes[a].faces))[0] == 1, a
    info = s.info()
    assert info["n_parts"] == 5 and info["n_items"] == 5
    with pytest.raises(agr.AgrError, match="parts"):
        s.debug_export_blas(0)
    whole = make_scene(sc, parts=False)
    assert whole.debug_asset_parts(0, len(tree.faces))[0] == 1
    assert whole.info()["n_items"] == 4


@pytest.mark.parametrize("builder", [0, 1])
def test_parts_equal_whole_asset_bitwise(builder):
    """Splitting assets into parts changes only the acceleration structure:
    c3-shaped envs cast with and without parts give bitwise identical
    depth, seg, face, normals and barycentrics, after a rebuild and after a
    refit with new poses, in packet and per-lane traversal; and match the
    oracle."""
    sc, sensor = sg.config3(n_envs=8)
    chans = ("dist", "seg", "face", "normal", "bary")
    out = {}
    for parts in (True, False):
        s = make_scene(sc, build=False, parts=parts)
        s.set_tlas_builder(builder)
        s.build()
        a = to_np(cast_sensor(s, sensor, "depth", channels=chans))
        T2 = sc.inst_T.copy()
        T2[:, :2, 3] += np.random.default_rng(4).uniform(-0.5, 0.5, (len(T2), 2)).astype(np.float32)
        s.set_instance_transforms(torch.from_numpy(T2).to(dev()))
        s.refit()
        b = to_np(cast_sensor(s, sensor, "range", channels=chans))
        s.set_traversal(1)
        c = to_np(cast_sensor(s, sensor, "range", channels=chans))
        out[parts] = (a, b, c, s.info())
    for i in range(3):
        for k in chans:
            assert np.array_equal(out[True][i][k].view(np.uint32), out[False][i][k].view(np.uint32)), (i, k)
    assert out[True][3]["n_items"] == out[False][3]["n_items"] + 40 * 8  # every tree: trunk + canopy
    q = np.random.default_rng(12).choice(len(out[True][0]["dist"]), 20000, replace=False)
    ref = oracle.cast(sc, oracle_rays(sensor, "depth"), query=q)
    compare(ref, out[True][0]["dist"][q], out[True][0]["seg"][q], out[True][0]["face"][q], "c3 parts")


def test_parts_update_mesh_stereo_and_exact():
    """A split asset (tree) deformed by agr_update_mesh rebuilds both part
    BLAS and the item boxes; stereo shadows and exact mode run over parts;
    everything matches the oracle / the filter bitwise."""
    rng = np.random.default_rng(6)
    tree = sg.tree_mesh(rng)
    per_env = [[(0, 1, sg.make_T(sg.rot_z(0.3 * e), (4.0, 0.5 * e - 1, -2.5))),
                (1, 2, sg.make_T(np.eye(3), (9.0, 0, 0)))] for e in range(4)]
    sc = sg.assemble([tree, sg.cube_mesh(4.0)], per_env)
    cam = sg.pinhole(96, 64, 90.0)
    sensor = dict(kind="pinhole", cam=cam, poses=sg.identity_poses(4), max_range=12.0)
    s = make_scene(sc)
    assert s.info()["n_parts"] == 3
    v = tree.verts.astype(np.float64) * 1.1 + rng.uniform(-0.05, 0.05, tree.verts.shape)
    vf = v.astype(np.float32)
    s.update_mesh(0, torch.from_numpy(vf).to(dev()))
    s.build()
    sc2 = sg.assemble([sg.Mesh("t", vf, tree.faces), sg.cube_mesh(4.0)], per_env)
    s.set_stereo((0.0, -0.3, 0.0), 1e-4)
    got = to_np(cast_sensor(s, sensor, "depth", channels=("dist", "seg", "face", "valid")))
    ref = oracle.cast(sc2, oracle_rays(sensor, "depth"), stereo=((0.0, -0.3, 0.0), 1e-4))
    # the cube's front face (x = 7) is centred on the optical axis: its
    # diagonal pixels are exact ties (61 of 24576), as in config 1
    compare(ref, got["dist"], got["seg"], got["face"], "tree parts after update", max_amb=64)
    assert valid_compare(ref, got["valid"], "tree parts stereo", max_amb=64) > 50
    assert (got["seg"] == 1).sum() > 500
    s.set_exact_mode(True)
    ex = to_np(cast_sensor(s, sensor, "depth", channels=("dist", "seg", "face", "valid")))
    for k in got:
        assert np.array_equal(got[k], ex[k]), k


# ---- 8-wide nodes for the interval packets ------------------------------

@pytest.mark.parametrize("cfg", [2, 3, 4])
def test_bvh8_packets_equal_bvh4_packets_bitwise(cfg):
    """The interval-packet traversal over the BVH32 copy (default), over a
    BVH8 / BVH16 copy (node_width 8 / 16), over the BVH4 (traversal mode 2), a
    BVH4-only scene (node_width 4) and the per-lane traversal give bitwise
    identical images, after a rebuild and after a refit; and match the
    oracle on samples.  (c2 / c4 envs of <= 32 items have a one-node 32-wide
    TLAS, c3's 91-item envs a deep one.)"""
    if cfg == 2:
        sc, sensor = sg.config2(n_envs=8)
    elif cfg == 3:
        sc, sensor = sg.config3(n_envs=6)
    else:
        sc, sensor = sg.config4(n_envs=6)
        sensor = dict(sensor, beams=sg.lidar_beams(64, 256))
    kind = "range" if cfg == 4 else "depth"
    chans = ("dist", "seg", "face", "normal")
    s = make_scene(sc, build=False)
    s4 = agr.Scene.from_scenegen(sc, device=0, node_width=4)
    s16 = agr.Scene.from_scenegen(sc, device=0, node_width=16)
    s8 = agr.Scene.from_scenegen(sc, device=0, node_width=8)  # the default is 32
    for sc_ in (s4, s16, s8):
        sc_.set_instance_transforms(torch.from_numpy(sc.inst_T).to(dev()))
    for sc_ in (s, s4, s16, s8):
        sc_.set_tlas_builder(1)
        sc_.build()
    imgs = []
    for step in range(2):
        if step == 1:
            T2 = sc.inst_T.copy()
            T2[:, :2, 3] += np.random.default_rng(5).uniform(-0.3, 0.3, (len(T2), 2)).astype(np.float32)
            for sc_ in (s, s4, s16, s8):
                sc_.set_instance_transforms(torch.from_numpy(T2).to(dev()))
                sc_.refit()
        runs = []
        for sc_, mode in ((s, 0), (s, 2), (s4, 0), (s, 1), (s, 3), (s16, 0), (s16, 3), (s8, 0), (s8, 3)):
            sc_.set_traversal(mode)
            runs.append(to_np(cast_sensor(sc_, sensor, kind, channels=chans)))
        for r in runs[1:]:
            for k in chans:
                assert np.array_equal(runs[0][k].view(np.uint32), r[k].view(np.uint32)), (step, k)
        imgs.append(runs[0])
    q = np.random.default_rng(8).choice(len(imgs[0]["dist"]), 10000, replace=False)
    ref = oracle.cast(sc, oracle_rays(sensor, kind), query=q)
    compare(ref, imgs[0]["dist"][q], imgs[0]["seg"][q], imgs[0]["face"][q], f"c{cfg} bvh8")


def test_wide_tile_cameras_all_schedules_bitwise():
    """Small wide-angle images (8x8 .. 64x64 at 87 deg: a 4x8 tile spans
    0.24-2 rad) are cast one ray per lane in auto mode (agr.h); the
    interval packets forced on them (modes 2 / 3, the sign-change branches
    of the interval slab everywhere) give bitwise the same images, and
    those match the oracle in full."""
    sc, sensor = sg.config4(n_envs=8)
    s = make_scene(sc, build=False)
    s.set_tlas_builder(1)
    s.build()
    for H, W in ((8, 8), (16, 16), (31, 33), (64, 64)):
        cam = sg.pinhole(W, H, 87.0)
        sen = dict(kind="pinhole", cam=cam, poses=sensor["poses"], max_range=10.0)
        runs = []
        for mode in (0, 1, 2, 3):
            s.set_traversal(mode)
            runs.append(to_np(cast_sensor(s, sen, "depth", channels=("dist", "seg", "face", "normal"))))
        for r in runs[1:]:
            for k in r:
                assert np.array_equal(runs[0][k].view(np.uint32), r[k].view(np.uint32)), (H, W, k)
        ref = oracle.cast(sc, oracle_rays(sen, "depth"))
        compare(ref, runs[0]["dist"], runs[0]["seg"], runs[0]["face"], f"wide tiles {H}x{W}")
    with pytest.raises(agr.AgrError):
        s.set_traversal(4)
    s.close()


@pytest.mark.parametrize("builder", [0, 1])
def test_tlas_warp_refit_equals_cta_refit_c3_bitwise(builder):
    """c3-shaped envs (91 TLAS items: warp refit, CTA build) refit after new
    transforms give bitwise the TLAS a 140-item-env scene (CTA refit) gives."""
    sc, sensor = sg.config3(n_envs=3)
    per_env = [[(int(sc.inst_asset[i]), int(sc.inst_label[i]), sc.inst_T[i])
                for i in range(int(sc.env_off[e]), int(sc.env_off[e + 1]))] for e in range(3)]
    big = per_env[0] + per_env[1][:89]
    scs = [sg.assemble(sc.meshes, per_env), sg.assemble(sc.meshes, per_env + [big])]
    scenes = [make_scene(x, build=False) for x in scs]
    for x in scenes:
        x.set_tlas_builder(builder)
        x.build()
    for x, scx in zip(scenes, scs):
        T2 = scx.inst_T.copy()
        T2[:, :2, 3] += 0.3
        x.set_instance_transforms(torch.from_numpy(T2).to(dev()))
        x.refit()
    for e in range(3):
        a, ra = scenes[0].debug_export_bvh4(-1 - e)
        b, rb = scenes[1].debug_export_bvh4(-1 - e)
        if builder == 0:  # LBVH: deterministic node numbering
            assert ra == rb and np.array_equal(a.view(np.uint32), b.view(np.uint32)), e
        else:  # the SAH build numbers nodes in the order its warps claim tasks
            assert _bvh4_canonical(a, ra) == _bvh4_canonical(b, rb), e
    for x in scenes:
        x.close()


def test_tlas_warp_path_equals_cta_path_bitwise():
    """Envs of <= 32 TLAS items are LBVH-built, and envs of <= 128 items
    refit, by one warp each (tlas.cu k_tlas_warp) unless some env of the
    scene is larger (then every env takes the CTA path): the same envs give
    bitwise the same BVH4 TLAS and images either way, after an LBVH build
    and after a refit."""
    sc, sensor = sg.config2(n_envs=3)  # 10 items per env
    big = [(int(a), 40 + k, T) for k, (a, T) in enumerate(zip(sc.inst_asset[:10], sc.inst_T[:10]))] * 14
    per_env = [[(int(sc.inst_asset[i]), int(sc.inst_label[i]), sc.inst_T[i])
                for i in range(int(sc.env_off[e]), int(sc.env_off[e + 1]))] for e in range(3)]
    small = sg.assemble(sc.meshes, per_env)
    mixed = sg.assemble(sc.meshes, per_env + [big])  # a 140-item env appended last
    scenes = [make_scene(small), make_scene(mixed)]
    poses = sensor["poses"][:3]
    sen = dict(sensor, poses=poses)
    for step in range(2):
        if step == 1:
            for x, scx in zip(scenes, (small, mixed)):
                T2 = scx.inst_T.copy()
                T2[:, :2, 3] += 0.2
                x.set_instance_transforms(torch.from_numpy(T2).to(dev()))
                x.refit()
        for e in range(3):
            a, ra = scenes[0].debug_export_bvh4(-1 - e)
            b, rb = scenes[1].debug_export_bvh4(-1 - e)
            assert ra == rb
            assert np.array_equal(a.view(np.uint32), b.view(np.uint32)), (step, e)
        img = [to_np(cast_sensor(x, sen if i == 0 else dict(sen, poses=np.concatenate([poses, poses[:1]]))))
               for i, x in enumerate(scenes)]
        n = len(img[0]["dist"])
        for k in img[0]:
            assert np.array_equal(img[0][k].view(np.uint32), img[1][k][:n].view(np.uint32)), (step, k)
    for x in scenes:
        x.close()


# --------------------------------------------------------------------------
# Table II-shaped env step: the
# kinematic stand-in (include/agr_sim.h) + refit + cast, eager and as a
# CUDA graph, against the oracle on the scene the step produced
# --------------------------------------------------------------------------
def _t2_setup(E=16, H=48, W=64):
    sc, sensor = sg.config4(n_envs=E)
    robots0, obst0 = sg.table2_sim_records(sc, sensor["poses"])
    prm = agr.agr_sim_params(dt=0.05, v_max=2.0, tau=0.2, yaw_rate_max=1.5, goal_radius=0.5,
                             lo=(-4.0, -4.0, 0.5), hi=(4.0, 4.0, 3.5), seed=7, env_base=0)
    cam = sg.pinhole(W, H, 87.0)
    return sc, robots0, obst0, prm, cam


def test_sim_step_records():
    """The stand-in keeps static instances exactly, moves obstacles rigidly
    (rotation part stays R_z(angle) A0), keeps robots inside the box and
    writes orthonormal poses; two runs are bitwise identical."""
    sc, robots0, obst0, prm, _ = _t2_setup()
    runs = []
    for _ in range(2):
        robots = torch.from_numpy(robots0.copy()).to(dev())
        obst = torch.from_numpy(obst0.copy()).to(dev())
        poses = torch.empty((sc.n_envs, 1, 3, 4), device=dev())
        T = torch.empty((sc.n_inst, 3, 4), device=dev())
        for _k in range(50):
            agr.sim_kinematic_step(robots, poses, obst, T, prm)
        torch.cuda.synchronize()
        runs.append((poses.cpu().numpy(), T.cpu().numpy(), robots.cpu().numpy()))
    assert all(np.array_equal(a, b) for a, b in zip(runs[0], runs[1]))
    P, Tn, R = runs[0]
    static = sc.inst_label == 0
    assert np.array_equal(Tn[static], sc.inst_T[static])
    A0 = sc.inst_T[:, :, :3].astype(np.float64)
    A = Tn[:, :, :3].astype(np.float64)
    # same column norms and the z row untouched: a yaw rotation of A0
    assert np.allclose(np.linalg.norm(A, axis=1), np.linalg.norm(A0, axis=1), rtol=1e-5, atol=1e-6)
    assert np.array_equal(Tn[:, 2, :3], sc.inst_T[:, 2, :3])
    assert np.array_equal(Tn[:, :2, 3], sc.inst_T[:, :2, 3])
    assert np.any(Tn[~static] != sc.inst_T[~static])
    Rp = P[:, 0, :, :3].astype(np.float64)
    assert np.allclose(Rp @ np.swapaxes(Rp, 1, 2), np.eye(3), atol=1e-6)
    p = P[:, 0, :, 3]
    assert np.all(p >= np.asarray(prm.lo) - 1e-6) and np.all(p <= np.asarray(prm.hi) + 1e-6)
    assert np.all(R.view(np.int32)[:, 10] >= 1)  # every robot drew a goal
    assert np.any(np.abs(p - robots0[:, 0:3]) > 0.1)


def test_sim_step_rejects_bad_params():
    sc, robots0, obst0, prm, _ = _t2_setup(E=2)
    robots = torch.from_numpy(robots0.copy()).to(dev())
    poses = torch.empty((2, 1, 3, 4), device=dev())
    bad = agr.agr_sim_params(dt=0.0, v_max=1.0, tau=0.1)
    with pytest.raises(agr.AgrError):
        agr.sim_kinematic_step(robots, poses, None, None, bad)


def test_table2_env_step_graph_matches_eager_and_oracle():
    """20 dynamic env steps (robots + obstacles move, transforms set, TLAS
    refit, depth + seg cast) replayed from a CUDA graph give bitwise the
    images of the same steps run eagerly, and those images match the oracle
    on the scene and poses the last step produced."""
    sc, robots0, obst0, prm, cam = _t2_setup()
    E, H, W = sc.n_envs, cam["H"], cam["W"]
    results = []
    for use_graph in (False, True):
        s = make_scene(sc)
        s.set_tlas_builder(1)
        s.build()
        robots = torch.from_numpy(robots0.copy()).to(dev())
        obst = torch.from_numpy(obst0.copy()).to(dev())
        poses = torch.empty((E, 1, 3, 4), device=dev())
        T = torch.from_numpy(sc.inst_T.copy()).to(dev())
        out = {"dist": torch.empty((E, 1, H, W), device=dev()),
               "seg": torch.empty((E, 1, H, W), dtype=torch.int32, device=dev()),
               "face": torch.empty((E, 1, H, W), dtype=torch.int32, device=dev())}

        def step():
            agr.sim_kinematic_step(robots, poses, obst, T, prm)
            s.set_instance_transforms(T)
            s.refit()
            s.cast_pinhole(cam, poses, 10.0, agr.AGR_DEPTH, out=out)

        if use_graph:
            step()  # step 1 eagerly, then 19 graph replays
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            # capture records the launches without running them
            with torch.cuda.graph(g):
                step()
            for _ in range(19):
                g.replay()
        else:
            for _ in range(20):
                step()
        torch.cuda.synchronize()
        results.append(({k: v.cpu().numpy() for k, v in out.items()}, poses.cpu().numpy(), T.cpu().numpy()))
        s.close()
    (img_e, P_e, T_e), (img_g, P_g, T_g) = results
    assert np.array_equal(P_e, P_g) and np.array_equal(T_e, T_g)
    for k in img_e:
        assert np.array_equal(img_e[k].view(np.int32), img_g[k].view(np.int32)), k
    sc2 = sc.env_slice(0, E)
    sc2.inst_T = T_e
    sensor = dict(kind="pinhole", cam=cam, poses=P_e, max_range=10.0)
    ref = oracle.cast(sc2, oracle_rays(sensor, "depth"))
    res = compare(ref, img_e["dist"].reshape(-1), img_e["seg"].reshape(-1), img_e["face"].reshape(-1),
                  "t2 env step")
    assert (ref.face >= 0).mean() > 0.5
