"""Small mixed workload for compute-sanitizer (memcheck / initcheck /
racecheck / synccheck): every kernel family of libagr.so once -- BLAS
builds (create + a batched mesh update with the cooperative top-down
BVH4), TLAS LBVH / SAH builds and refit, pinhole casts in every traversal
schedule (packets BVH8 / BVH4, lanes, exact), beams, explicit rays, extras,
stereo, checksums, deep TLAS (BVH16 / BVH32 copies, the wide SAH-optimal
DP collapses, warp and CTA TLAS paths) and the simulator stand-in."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2503_01471_b200 as agr  # noqa: E402
import scenegen as sg  # noqa: E402

dev = torch.device("cuda", 0)


def T(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to(dev)


sc, sensor = sg.config2(n_envs=3)
s = agr.Scene.from_scenegen(sc)
s.set_instance_transforms(T(sc.inst_T))
for builder in (0, 1):
    s.set_tlas_builder(builder)
    s.build()
s.refit()
cam = dict(sensor["cam"], W=40, H=24)
poses = T(sensor["poses"])
for mode in (0, 1, 2, 3):
    s.set_traversal(mode)
    s.cast_pinhole(cam, poses, 10.0, agr.AGR_DEPTH, channels=("dist", "seg", "face", "normal", "bary", "point"))
s.set_traversal(0)
s.set_stereo()
s.cast_pinhole(cam, poses, 10.0, agr.AGR_RANGE, channels=("dist", "seg", "face", "valid"))
s.set_exact_mode(True)
s.cast_pinhole(cam, poses, 10.0, agr.AGR_DEPTH)
s.set_exact_mode(False)
beams = T(sg.lidar_beams(16, 32))
out = s.cast_beams(beams, poses, 10.0)
s.checksum(out, 16 * 32)
R = 64
o = T(np.zeros((3, R, 3), np.float32))
d = T(np.random.default_rng(0).normal(size=(3, R, 3)).astype(np.float32))
s.cast_rays(o, d, 10.0)
torch.cuda.synchronize()
s.close()

# deep TLAS (round 2): c3 forest envs (91 items: BVH32 by default, the CTA
# TLAS build with the 32-wide DP), the BVH16 copy, and 300 items in one env
# (beyond the DP's 128: greedy wide collapse), both builders + refit, every
# pinhole schedule
sc3, sen3 = sg.config3(n_envs=2)
rng = np.random.default_rng(41)
big = [[(j % 2, j + 1, sg.make_T(sg.random_rotation(rng), rng.uniform([2, -6, -4], [14, 6, 4]),
                                 rng.uniform(0.1, 0.4))) for j in range(n)] for n in (300, 37)]
scb = sg.assemble([sg.cube_mesh(), sg.panel_mesh()], big)
for scx, nw, poses_x in ((sc3, 0, sen3["poses"]), (sc3, 16, sen3["poses"]), (scb, 0, sg.identity_poses(2))):
    sx = agr.Scene.from_scenegen(scx, node_width=nw)
    sx.set_instance_transforms(T(scx.inst_T))
    for builder in (0, 1):
        sx.set_tlas_builder(builder)
        sx.build()
        sx.refit()
        for mode in (0, 3):
            sx.set_traversal(mode)
            sx.cast_pinhole(sg.pinhole(40, 24, 87.0), T(poses_x), 10.0, agr.AGR_DEPTH,
                            channels=("dist", "seg", "face"))
    torch.cuda.synchronize()
    sx.close()

# per-env unique meshes: batched BLAS rebuild (sort, fit, records, top-down BVH4)
E = 4
meshes = [sg.terrain_mesh(np.random.default_rng(e), n=16) for e in range(E)]
sc6 = sg.assemble(meshes, [[(e, 1, sg.make_T(np.eye(3), (0.0, 0.0, 0.0)))] for e in range(E)])
s6 = agr.Scene.from_scenegen(sc6, trbvh_rounds=0, node_width=4)
s6.set_instance_transforms(T(sc6.inst_T))
s6.build()
v = np.concatenate([m.verts * 1.05 for m in meshes]).astype(np.float32)
s6.update_meshes(list(range(E)), T(v))
s6.build()
s6.set_traversal(1)
s6.cast_pinhole(sg.pinhole(24, 16, 87.0), T(sg.identity_poses(E)), 20.0)
torch.cuda.synchronize()
s6.close()

# simulator stand-in + refit + cast (the Table-II env step)
sc4, sen4 = sg.config4(n_envs=2)
robots, obst = sg.table2_sim_records(sc4, sen4["poses"])
s4 = agr.Scene.from_scenegen(sc4)
Tm = T(sc4.inst_T)
s4.set_instance_transforms(Tm)
s4.build()
rb, ob = T(robots), T(obst)
pz = torch.empty((2, 1, 3, 4), device=dev)
prm = agr.agr_sim_params(dt=0.05, v_max=2.0, tau=0.2, yaw_rate_max=1.5, goal_radius=0.5,
                         lo=(-4.0, -4.0, 0.5), hi=(4.0, 4.0, 3.5), seed=1, env_base=0)
for _ in range(2):
    agr.sim_kinematic_step(rb, pz, ob, Tm, prm)
    s4.set_instance_transforms(Tm)
    s4.refit()
    s4.cast_pinhole(sg.pinhole(16, 8, 87.0), pz, 10.0, agr.AGR_DEPTH, channels=("dist", "seg"))
torch.cuda.synchronize()
s4.close()
print("sanitize workload done")
