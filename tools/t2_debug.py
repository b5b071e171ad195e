"""Where does a small Table-II step's time go?  8x8 x 2048 envs static:
eager sim + cast, cast alone, sim alone, graph replay (CUDA events)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2503_01471_b200 as agr, scenegen as sg

E, H, W = int(sys.argv[1]) if len(sys.argv) > 1 else 2048, 8, 8
dev = torch.device("cuda", 0)
sc, sen = sg.config4(n_envs=E)
robots0, obst0 = sg.table2_sim_records(sc, sen["poses"])
s = agr.Scene.from_scenegen(sc)
s.set_tlas_builder(1)
T = torch.from_numpy(sc.inst_T).to(dev)
s.set_instance_transforms(T)
s.build()
cam = sg.pinhole(W, H, 87.0)
robots = torch.from_numpy(robots0).to(dev)
poses = torch.empty((E, 1, 3, 4), device=dev)
out = {"dist": torch.empty((E, 1, H, W), device=dev), "seg": torch.empty((E, 1, H, W), dtype=torch.int32, device=dev)}
prm = agr.agr_sim_params(dt=0.01, v_max=2.0, tau=0.2, yaw_rate_max=1.5, goal_radius=0.5,
                         lo=(-4.0, -4.0, 0.5), hi=(4.0, 4.0, 3.5), seed=2025, env_base=0)
st = torch.cuda.current_stream()


def timeit(fn, n=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(n):
        fn()
    b.record(st)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3


sim = lambda: agr.sim_kinematic_step(robots, poses, None, None, prm)
cast = lambda: s.cast_pinhole(cam, poses, 10.0, agr.AGR_DEPTH, out=out)
print("sim alone us", timeit(sim))
print("cast alone us", timeit(cast))
print("sim+cast eager us", timeit(lambda: (sim(), cast())))
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    sim(); cast()
print("graph replay us", timeit(g.replay))
for mode in (1, 0):
    s.set_traversal(mode)
    print("traversal", mode, "cast us", timeit(cast))
