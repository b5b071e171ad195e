"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO ray-casting arithmetic: it only builds asset meshes,
per-env instance lists / transforms / labels, sensor poses, pinhole
intrinsics and LiDAR beam tables -- i.e. the *inputs* of the C ABI
 -- with the shapes, sizes and structure of the paper's
workloads (Table I scene: "20 cube obstacles in front of the
robots", 270x480 camera; Table II scene: "room-like static
environment consisting of 15 floating obstacles"; PAPER.md:215 LiDAR "512
points, 128 channels").  The recipe is DESIGN.md §6 / SURVEY.md §8(d).

Determinism: every env draws from its own stream
``np.random.default_rng([config_seed, global_env_id])`` so the same env gets
the same scene regardless of how envs are sharded across GPUs.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# ----------------------------------------------------------------------------
# asset meshes (object space, float32 vertices, int32 faces)
# ----------------------------------------------------------------------------


@dataclass
class Mesh:
    name: str
    verts: np.ndarray  # float32 [V][3]
    faces: np.ndarray  # int32 [F][3]


def box_mesh(name, lo, hi) -> Mesh:
    """Axis-aligned box [lo, hi], 8 vertices, 12 triangles (2 per side)."""
    lo = np.asarray(lo, np.float64)
    hi = np.asarray(hi, np.float64)
    v = []
    for i in range(8):
        v.append([hi[0] if i & 1 else lo[0], hi[1] if i & 2 else lo[1], hi[2] if i & 4 else lo[2]])
    # sides as quads (a, b, c, d) -> triangles (a, b, c), (a, c, d)
    quads = [
        (0, 2, 6, 4),  # -x
        (1, 5, 7, 3),  # +x
        (0, 4, 5, 1),  # -y
        (2, 3, 7, 6),  # +y
        (0, 1, 3, 2),  # -z
        (4, 6, 7, 5),  # +z
    ]
    f = []
    for a, b, c, d in quads:
        f.append((a, b, c))
        f.append((a, c, d))
    return Mesh(name, np.asarray(v, np.float32), np.asarray(f, np.int32))


def cube_mesh(size=1.0) -> Mesh:
    h = size / 2
    return box_mesh("cube", (-h, -h, -h), (h, h, h))


def panel_mesh() -> Mesh:
    """1 x 1 x 0.05 m panel (thin box), 12 triangles."""
    return box_mesh("panel", (-0.025, -0.5, -0.5), (0.025, 0.5, 0.5))


def room_mesh() -> Mesh:
    """10 x 10 x 4 m room box (floor at z = 0), 12 triangles, seen from inside."""
    return box_mesh("room", (-5.0, -5.0, 0.0), (5.0, 5.0, 4.0))


def ground_mesh(size=40.0) -> Mesh:
    h = size / 2
    v = np.asarray([[-h, -h, 0], [h, -h, 0], [h, h, 0], [-h, h, 0]], np.float32)
    f = np.asarray([[0, 1, 2], [0, 2, 3]], np.int32)
    return Mesh("ground", v, f)


def cylinder_mesh(name="cylinder", r=0.5, h=1.0, nseg=24, closed=True, z0=None) -> Mesh:
    """Cylinder about z.  Closed: side 2*nseg + caps as fans 2*nseg = 4*nseg tri
    (nseg=24 -> 96; we use fan caps with a centre vertex)."""
    z0 = -h / 2 if z0 is None else z0
    z1 = z0 + h
    v = []
    for k in range(nseg):
        a = 2 * math.pi * k / nseg
        v.append([r * math.cos(a), r * math.sin(a), z0])
    for k in range(nseg):
        a = 2 * math.pi * k / nseg
        v.append([r * math.cos(a), r * math.sin(a), z1])
    f = []
    for k in range(nseg):
        k1 = (k + 1) % nseg
        f.append((k, k1, nseg + k1))
        f.append((k, nseg + k1, nseg + k))
    if closed:
        cb = len(v)
        v.append([0.0, 0.0, z0])
        ct = len(v)
        v.append([0.0, 0.0, z1])
        for k in range(nseg):
            k1 = (k + 1) % nseg
            f.append((cb, k1, k))
            f.append((ct, nseg + k, nseg + k1))
    return Mesh(name, np.asarray(v, np.float32), np.asarray(f, np.int32))


def closed_cylinder_92() -> Mesh:
    """Closed cylinder r=0.5, h=1 with 23 segments -> 4*23 = 92 triangles."""
    return cylinder_mesh("cylinder", 0.5, 1.0, nseg=23, closed=True)


def icosphere(subdiv: int):
    """Unit icosphere (vertices on the unit sphere), 20 * 4**subdiv faces."""
    t = (1.0 + math.sqrt(5.0)) / 2.0
    v = [[-1, t, 0], [1, t, 0], [-1, -t, 0], [1, -t, 0],
         [0, -1, t], [0, 1, t], [0, -1, -t], [0, 1, -t],
         [t, 0, -1], [t, 0, 1], [-t, 0, -1], [-t, 0, 1]]
    v = [list(np.asarray(p, np.float64) / np.linalg.norm(p)) for p in v]
    f = [(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11),
         (1, 5, 9), (5, 11, 4), (11, 10, 2), (10, 7, 6), (7, 1, 8),
         (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8), (3, 8, 9),
         (4, 9, 5), (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1)]
    for _ in range(subdiv):
        cache = {}

        def mid(a, b):
            key = (min(a, b), max(a, b))
            if key not in cache:
                m = np.asarray(v[a]) + np.asarray(v[b])
                v.append(list(m / np.linalg.norm(m)))
                cache[key] = len(v) - 1
            return cache[key]

        nf = []
        for a, b, c in f:
            ab, bc, ca = mid(a, b), mid(b, c), mid(c, a)
            nf += [(a, ab, ca), (b, bc, ab), (c, ca, bc), (ab, bc, ca)]
        f = nf
    return np.asarray(v, np.float64), np.asarray(f, np.int32)


def sphere_mesh(radius=1.0, subdiv=2, name="sphere") -> Mesh:
    v, f = icosphere(subdiv)
    return Mesh(name, (v * radius).astype(np.float32), f)


def tree_mesh(rng: np.random.Generator, name="tree") -> Mesh:
    """Open 16-segment trunk (32 tri, r in [.12,.2], h = 4) + jittered
    icosphere-3 canopy (1280 tri, r in [1, 1.6], centre z in [3, 4]) = 1312."""
    r = rng.uniform(0.12, 0.2)
    trunk = cylinder_mesh("trunk", r, 4.0, nseg=16, closed=False, z0=0.0)
    cv, cf = icosphere(3)
    cr = rng.uniform(1.0, 1.6)
    cz = rng.uniform(3.0, 4.0)
    jitter = 1.0 + rng.uniform(-0.08, 0.08, size=(len(cv), 1))
    cv = cv * cr * jitter + np.asarray([0.0, 0.0, cz])
    verts = np.concatenate([trunk.verts.astype(np.float64), cv]).astype(np.float32)
    faces = np.concatenate([trunk.faces, cf + len(trunk.verts)]).astype(np.int32)
    return Mesh(name, verts, faces)


def rock_mesh(rng: np.random.Generator, name="rock") -> Mesh:
    """Jittered anisotropic icosphere-2 (320 tri), resting on z = 0."""
    v, f = icosphere(2)
    axes = rng.uniform([0.4, 0.3, 0.2], [0.8, 0.6, 0.45])
    jitter = 1.0 + rng.uniform(-0.12, 0.12, size=(len(v), 1))
    v = v * jitter * axes
    v[:, 2] -= v[:, 2].min() * 0.6
    return Mesh(name, v.astype(np.float32), f)


# ----------------------------------------------------------------------------
# scenes
# ----------------------------------------------------------------------------


@dataclass
class Scene:
    """Flattened scene description == the arguments of agr_scene_create."""
    meshes: list
    env_off: np.ndarray      # int64 [E+1] CSR of instances per env
    inst_asset: np.ndarray   # int32 [I]
    inst_label: np.ndarray   # int32 [I]
    inst_T: np.ndarray       # float32 [I][3][4] object -> env-local, x' = A x + b
    env_base: int = 0        # global id of env 0 (sharding)
    extra: dict = field(default_factory=dict)

    @property
    def n_envs(self):
        return len(self.env_off) - 1

    @property
    def n_inst(self):
        return int(self.env_off[-1])

    @property
    def verts(self):
        return np.concatenate([m.verts for m in self.meshes]).astype(np.float32)

    @property
    def faces(self):
        return np.concatenate([m.faces for m in self.meshes]).astype(np.int32)

    @property
    def vert_off(self):
        return np.concatenate([[0], np.cumsum([len(m.verts) for m in self.meshes])]).astype(np.int64)

    @property
    def face_off(self):
        return np.concatenate([[0], np.cumsum([len(m.faces) for m in self.meshes])]).astype(np.int64)

    def env_slice(self, e0, e1) -> "Scene":
        """Sub-scene with envs [e0, e1) (same assets)."""
        i0, i1 = int(self.env_off[e0]), int(self.env_off[e1])
        return Scene(self.meshes, (self.env_off[e0:e1 + 1] - i0).astype(np.int64),
                     self.inst_asset[i0:i1].copy(), self.inst_label[i0:i1].copy(),
                     self.inst_T[i0:i1].copy(), self.env_base + e0, dict(self.extra))


def rot_z(a):
    c, s = math.cos(a), math.sin(a)
    return np.asarray([[c, -s, 0], [s, c, 0], [0, 0, 1]], np.float64)


def rot_y(a):
    c, s = math.cos(a), math.sin(a)
    return np.asarray([[c, 0, s], [0, 1, 0], [-s, 0, c]], np.float64)


def random_rotation(rng):
    q = rng.normal(size=4)
    q /= np.linalg.norm(q)
    w, x, y, z = q
    return np.asarray([
        [1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
        [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
        [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)]], np.float64)


def make_T(R, p, s=1.0):
    T = np.zeros((3, 4), np.float64)
    T[:, :3] = np.asarray(R) * s
    T[:, 3] = p
    return T.astype(np.float32)


def env_rng(seed, env, *more):
    return np.random.default_rng([int(seed), int(env)] + [int(m) for m in more])


def pinhole(W, H, hfov_deg):
    """Intrinsics from horizontal FOV (reading R8): fx computed in
    FP64 and rounded to FP32, fy = fx, principal point at the image centre."""
    fx = (W / 2.0) / math.tan(math.radians(hfov_deg) / 2.0)
    fx = float(np.float32(fx))
    return dict(W=int(W), H=int(H), fx=fx, fy=fx, cx=float(W / 2.0), cy=float(H / 2.0))


def lidar_beams(C=128, K=512, elev_lo=-45.0, elev_hi=45.0):
    """OS0-128-style beam table [C][K][3] float32 (reading R9):
    e_c = lo + (hi-lo) c/(C-1), a_k = -180 + 360 k/K, computed in FP64."""
    e = np.radians(elev_lo + (elev_hi - elev_lo) * np.arange(C) / max(C - 1, 1))
    a = np.radians(-180.0 + 360.0 * np.arange(K) / K)
    E, A = np.meshgrid(e, a, indexing="ij")
    d = np.stack([np.cos(E) * np.cos(A), np.cos(E) * np.sin(A), np.sin(E)], -1)
    return d.astype(np.float32)


def dome_beams(C=32, K=128):
    """Hemispherical dome LiDAR (PAPER.md:218 Fig. 3b, :228 'Dome LiDAR'):
    elevations (0, 90] deg, full azimuth."""
    return lidar_beams(C, K, elev_lo=90.0 / C, elev_hi=90.0)


def identity_poses(E, S=1):
    P = np.zeros((E, S, 3, 4), np.float32)
    P[:, :, 0, 0] = P[:, :, 1, 1] = P[:, :, 2, 2] = 1.0
    return P


def _c2_obstacle(rng, asset_ids):
    a = int(rng.integers(0, len(asset_ids)))
    p = rng.uniform([2.0, -3.0, -1.5], [8.0, 3.0, 1.5])
    R = random_rotation(rng)
    s = rng.uniform(0.5, 1.5)
    return asset_ids[a], make_T(R, p, s)


def assemble(meshes, per_env):
    """per_env: list (per env) of lists of (asset, label, T[3][4])."""
    env_off = [0]
    assets, labels, Ts = [], [], []
    for insts in per_env:
        for a, lab, T in insts:
            assets.append(a)
            labels.append(lab)
            Ts.append(T)
        env_off.append(len(assets))
    T = np.asarray(Ts, np.float32).reshape(-1, 3, 4) if Ts else np.zeros((0, 3, 4), np.float32)
    return Scene(meshes, np.asarray(env_off, np.int64), np.asarray(assets, np.int32),
                 np.asarray(labels, np.int32), T)


CONFIG_SEED = {1: 1001, 2: 1002, 3: 1003, 4: 1004, 5: 1005, 6: 1006}


def config1():
    """c1: 1 env, unit cube x in [2,3], y,z in [-.5,.5]; 16x16 camera with
    fx=fy=cx=cy=8 (90 deg hfov) at the origin; max 10 m (reading R16)."""
    meshes = [cube_mesh()]
    sc = assemble(meshes, [[(0, 1, make_T(np.eye(3), (2.5, 0.0, 0.0)))]])
    cam = dict(W=16, H=16, fx=8.0, fy=8.0, cx=8.0, cy=8.0)
    return sc, dict(cam=cam, poses=identity_poses(1), max_range=10.0, kind="pinhole")


def config2(n_envs=64, env_base=0):
    """c2: 10 random obstacles (cube/cylinder/panel) per env; 135x240, 87 deg."""
    meshes = [cube_mesh(), closed_cylinder_92(), panel_mesh()]
    per_env = []
    for e in range(env_base, env_base + n_envs):
        rng = env_rng(CONFIG_SEED[2], e)
        insts = []
        for k in range(10):
            a, T = _c2_obstacle(rng, [0, 1, 2])
            insts.append((a, k + 1, T))
        per_env.append(insts)
    sc = assemble(meshes, per_env)
    sc.env_base = env_base
    return sc, dict(cam=pinhole(240, 135, 87.0), poses=identity_poses(n_envs),
                    max_range=10.0, kind="pinhole")


def forest_assets(seed=CONFIG_SEED[3]):
    rng = np.random.default_rng([seed, 0xA55E7])
    meshes = [ground_mesh(40.0)]
    meshes += [tree_mesh(rng, f"tree{i}") for i in range(4)]
    meshes += [rock_mesh(rng, f"rock{i}") for i in range(2)]
    return meshes


def config3(n_envs=1024, env_base=0, n_trees=40, n_rocks=10):
    """c3: forest -- ground quad + 40 trees (4 variants) + 10 rocks (2
    variants) per env; 270x480 87 deg camera at a random pose in the forest."""
    meshes = forest_assets()
    per_env = []
    poses = np.zeros((n_envs, 1, 3, 4), np.float32)
    for i, e in enumerate(range(env_base, env_base + n_envs)):
        rng = env_rng(CONFIG_SEED[3], e)
        insts = [(0, 0, make_T(np.eye(3), (0.0, 0.0, 0.0)))]
        for k in range(n_trees):
            v = int(rng.integers(0, 4))
            p = (*rng.uniform(-10, 10, 2), 0.0)
            insts.append((1 + v, 1 + k, make_T(rot_z(rng.uniform(0, 2 * math.pi)), p,
                                              rng.uniform(0.8, 1.25))))
        for k in range(n_rocks):
            v = int(rng.integers(0, 2))
            p = (*rng.uniform(-10, 10, 2), 0.0)
            insts.append((5 + v, 1 + n_trees + k,
                          make_T(rot_z(rng.uniform(0, 2 * math.pi)), p, rng.uniform(0.8, 1.25))))
        per_env.append(insts)
        cp = (*rng.uniform(-8, 8, 2), rng.uniform(1.0, 2.0))
        R = rot_z(rng.uniform(0, 2 * math.pi)) @ rot_y(math.radians(rng.uniform(-10, 10)))
        poses[i, 0] = make_T(R, cp)
    sc = assemble(meshes, per_env)
    sc.env_base = env_base
    return sc, dict(cam=pinhole(480, 270, 87.0), poses=poses, max_range=10.0, kind="pinhole")


def config4(n_envs=4096, env_base=0):
    """c4: Table II-shaped room 10x10x4 m + 15 floating
    obstacles; OS0-128-style 128x512 LiDAR, range + seg, max 10 m."""
    meshes = [room_mesh(), cube_mesh(), closed_cylinder_92(), panel_mesh()]
    per_env = []
    poses = np.zeros((n_envs, 1, 3, 4), np.float32)
    for i, e in enumerate(range(env_base, env_base + n_envs)):
        rng = env_rng(CONFIG_SEED[4], e)
        insts = [(0, 0, make_T(np.eye(3), (0.0, 0.0, 0.0)))]
        for k in range(15):
            a = 1 + int(rng.integers(0, 3))
            p = rng.uniform([-4.0, -4.0, 0.5], [4.0, 4.0, 3.5])
            insts.append((a, k + 1, make_T(random_rotation(rng), p, rng.uniform(0.5, 1.5))))
        per_env.append(insts)
        poses[i, 0] = make_T(rot_z(rng.uniform(0, 2 * math.pi)),
                             rng.uniform([-3.0, -3.0, 1.0], [3.0, 3.0, 3.0]))
    sc = assemble(meshes, per_env)
    sc.env_base = env_base
    return sc, dict(beams=lidar_beams(128, 512), poses=poses, max_range=10.0, kind="beams")


def table2_sim_records(sc, poses, seed=CONFIG_SEED[4] + 7):
    """Initial records of the kinematic env-step stand-in (include/agr_sim.h)
    for a c4-shaped room scene: robots float32 [E][12] (agr_sim_robot: p from
    the env's sensor pose, v = 0, goal unset, yaw of the pose, 0 goals) and
    obstacles float32 [I][20] (agr_sim_obstacle: T0 = the instance transform;
    the room (label 0) never moves, each floating obstacle gets a yaw rate
    U(-0.5, 0.5) rad/s, a bobbing amplitude U(0, 0.2) m, frequency U(0.5, 2)
    rad/s and phase U(0, 2 pi), from its env's own stream)."""
    E = sc.n_envs
    robots = np.zeros((E, 12), np.float32)
    P = np.asarray(poses, np.float64).reshape(E, -1, 3, 4)[:, 0]
    robots[:, 0:3] = P[:, :, 3]
    robots[:, 9] = np.arctan2(P[:, 1, 0], P[:, 0, 0])
    obst = np.zeros((sc.n_inst, 20), np.float32)
    obst[:, 0:12] = sc.inst_T.reshape(-1, 12)
    for i in range(E):
        e = sc.env_base + i
        i0, i1 = int(sc.env_off[i]), int(sc.env_off[i + 1])
        rng = env_rng(seed, e)
        m = i1 - i0
        mov = sc.inst_label[i0:i1] != 0
        obst[i0:i1, 12] = np.where(mov, rng.uniform(-0.5, 0.5, m), 0.0)
        obst[i0:i1, 13] = np.where(mov, rng.uniform(0.0, 0.2, m), 0.0)
        obst[i0:i1, 14] = np.where(mov, rng.uniform(0.5, 2.0, m), 0.0)
        obst[i0:i1, 16] = np.where(mov, rng.uniform(0.0, 2 * math.pi, m), 0.0)
    return robots, obst


def _quat_rotations(q):
    """Rotation matrices [..][3][3] of (unnormalised) quaternions q [..][4]
    (w, x, y, z), normalised first: uniform random rotations for normal q."""
    q = q / np.linalg.norm(q, axis=-1, keepdims=True)
    w, x, y, z = (q[..., i] for i in range(4))
    R = np.empty(q.shape[:-1] + (3, 3))
    R[..., 0, 0] = 1 - 2 * (y * y + z * z)
    R[..., 0, 1] = 2 * (x * y - z * w)
    R[..., 0, 2] = 2 * (x * z + y * w)
    R[..., 1, 0] = 2 * (x * y + z * w)
    R[..., 1, 1] = 1 - 2 * (x * x + z * z)
    R[..., 1, 2] = 2 * (y * z - x * w)
    R[..., 2, 0] = 2 * (x * z - y * w)
    R[..., 2, 1] = 2 * (y * z + x * w)
    R[..., 2, 2] = 1 - 2 * (x * x + y * y)
    return R


def config5(n_envs=2048, env_base=0, ring=64):
    """c5: Table I-shaped 20 cubes per env at c2's pose
    distribution (position U(x in [2,8], y in [-3,3], z in [-1.5,1.5]),
    uniform rotation, scale U[0.5,1.5]), re-sampled every step: a ring of
    `ring` transform sets (float32 [ring][I][3][4]); step k uses set k % ring.
    135x240 camera.  Each env draws its whole ring from its own stream in
    one batch per quantity (16384 envs in seconds)."""
    meshes = [cube_mesh()]
    n_inst = 20
    ring_T = np.zeros((ring, n_envs, n_inst, 3, 4), np.float32)
    for i, e in enumerate(range(env_base, env_base + n_envs)):
        rng = env_rng(CONFIG_SEED[5], e)
        p = rng.uniform([2.0, -3.0, -1.5], [8.0, 3.0, 1.5], (ring, n_inst, 3))
        R = _quat_rotations(rng.normal(size=(ring, n_inst, 4)))
        sc_ = rng.uniform(0.5, 1.5, (ring, n_inst))
        T = np.empty((ring, n_inst, 3, 4))
        T[..., :3] = R * sc_[..., None, None]
        T[..., 3] = p
        ring_T[:, i] = T.astype(np.float32)
    ring_T = ring_T.reshape(ring, n_envs * n_inst, 3, 4)
    env_off = np.arange(n_envs + 1, dtype=np.int64) * n_inst
    labels = np.tile(np.arange(1, n_inst + 1, dtype=np.int32), n_envs)
    sc = Scene(meshes, env_off, np.zeros(n_envs * n_inst, np.int32), labels, ring_T[0].copy(), env_base)
    sc.extra["ring_T"] = ring_T
    return sc, dict(cam=pinhole(240, 135, 87.0), poses=identity_poses(n_envs),
                    max_range=10.0, kind="pinhole")


def terrain_mesh(rng, n=128, size=20.0, amp=1.2, name="terrain") -> Mesh:
    """Heightfield over x in [0, size], y in [-size/2, size/2]: (n+1)^2
    vertices, 2 n^2 triangles; height = four random plane waves of
    decreasing amplitude (a per-env unique, non-instanced mesh)."""
    x = np.linspace(0.0, size, n + 1)
    y = np.linspace(-size / 2, size / 2, n + 1)
    X, Y = np.meshgrid(x, y, indexing="ij")
    Z = np.zeros_like(X)
    for k in range(4):
        kx, ky = rng.uniform(0.2, 1.2, 2) * rng.choice([-1.0, 1.0], 2)
        Z += amp / (k + 1) * np.sin(kx * X + ky * Y + rng.uniform(0.0, 2.0 * np.pi))
    verts = np.stack([X, Y, Z], -1).reshape(-1, 3).astype(np.float32)
    idx = np.arange((n + 1) * (n + 1)).reshape(n + 1, n + 1)
    a, b, c, d = idx[:-1, :-1], idx[1:, :-1], idx[1:, 1:], idx[:-1, 1:]
    faces = np.concatenate([np.stack([a, b, c], -1).reshape(-1, 3),
                            np.stack([a, c, d], -1).reshape(-1, 3)]).astype(np.int32)
    return Mesh(name, verts, faces)


def config6(n_envs=256, env_base=0, ring=2, n=128):
    """c6 (PAPER.md:226 per-env merged mesh rebuilt at
    reset): one unique terrain asset per env (2 n^2 = 32768 triangles at
    n = 128), re-randomised at every step: extra["ring_V"] float32
    [ring][E * V][3] holds `ring` vertex sets (env-major, as
    agr_update_meshes takes them); step k uses set k % ring.  135x240 87 deg
    depth camera 5 m above the terrain's edge, pitched down 25 deg."""
    meshes, ring_v = [], []
    for i, e in enumerate(range(env_base, env_base + n_envs)):
        rng = env_rng(CONFIG_SEED[6], e)
        ms = [terrain_mesh(rng, n, name=f"terrain{e}") for _ in range(ring)]
        meshes.append(ms[0])
        ring_v.append(np.stack([m.verts for m in ms]))
    per_env = [[(i, 1, make_T(np.eye(3), (0.0, 0.0, 0.0)))] for i in range(n_envs)]
    sc = assemble(meshes, per_env)
    sc.env_base = env_base
    sc.extra["ring_V"] = np.ascontiguousarray(np.concatenate(ring_v, 1))
    P = np.zeros((n_envs, 1, 3, 4), np.float32)
    P[:, 0, :, :3] = rot_y(math.radians(25.0))
    P[:, 0, :, 3] = (-2.0, 0.0, 5.0)
    return sc, dict(cam=pinhole(240, 135, 87.0), poses=P, max_range=20.0, kind="pinhole")


def make_config(c: int, n_envs=None, env_base=0):
    if c == 1:
        return config1()
    kw = {} if n_envs is None else dict(n_envs=n_envs)
    return {2: config2, 3: config3, 4: config4, 5: config5, 6: config6}[c](env_base=env_base, **kw)


# ----------------------------------------------------------------------------
# sensor presets ("idealized configurations of: Ouster OS-0,
# OS-1, OS-2, OS-Dome, Intel RealSense D455, Luxonis Oak-D (and Pro W) and ST
# VL53L5CX ToF sensors").  The paper gives only the names; the parameters
# below are the public nominal specs (reading R22): vertical FOV
# and channel counts of the Ouster family, depth FOV of the D455 / Oak-D
# stereo cameras, 8x8 zones over 45 deg x 45 deg for the VL53L5CX.
# ----------------------------------------------------------------------------

def ouster(model="OS0", channels=128, columns=512):
    """Ouster lidar beam table [C][K][3]: uniform channels over the model's
    vertical FOV (OS0 90 deg, OS1 45 deg, OS2 22.5 deg), 360 deg azimuth."""
    vfov = {"OS0": 90.0, "OS1": 45.0, "OS2": 22.5}[model]
    return lidar_beams(channels, columns, -vfov / 2.0, vfov / 2.0)


def ouster_dome(channels=128, columns=512):
    """OS-Dome: 180 deg vertical FOV hemisphere looking up (elevations 0..90
    deg above the horizon and the mirror image: -90..90 about the up axis is
    modelled as elevations (0, 90] deg here, i.e. the upper hemisphere)."""
    return dome_beams(channels, columns)


PRESETS = {
    # name: (kind, builder)
    "os0-128": ("beams", lambda: ouster("OS0", 128, 512)),
    "os1-64": ("beams", lambda: ouster("OS1", 64, 1024)),
    "os2-32": ("beams", lambda: ouster("OS2", 32, 1024)),
    "os-dome-128": ("beams", lambda: ouster_dome(128, 512)),
    "d455": ("pinhole", lambda: pinhole(848, 480, 87.0)),
    "d455-270x480": ("pinhole", lambda: pinhole(480, 270, 87.0)),
    "oak-d": ("pinhole", lambda: pinhole(640, 400, 72.0)),
    "oak-d-pro-w": ("pinhole", lambda: pinhole(640, 400, 127.0)),
    "vl53l5cx": ("pinhole", lambda: pinhole(8, 8, 45.0)),
}


def preset(name: str) -> dict:
    """Sensor spec for a preset: {'kind': 'pinhole', 'cam': {...}} or
    {'kind': 'beams', 'beams': float32 [C][K][3]}."""
    kind, build = PRESETS[name]
    return {"kind": kind, ("cam" if kind == "pinhole" else "beams"): build()}
