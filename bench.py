#!/usr/bin/env python
"""Benchmark of the batched ray-casting hot path (BASELINE.json metric:
rays/sec and env-frames/sec at 1/2/4/8 B200; % of roofline).

One step = one pass of the whole per-step hot path over one batch of envs
(SURVEY.md §8(a)): set the instance transforms (a3) + per-env TLAS build
(a2; c5 uses the in-place refit) + one fused cast (a4 ray generation, a5
traversal, a6 FP64 epilogue + stores).  The per-asset BLAS (a1) is built
once at scene creation, as in the paper (the BVH is computed
"exclusively for randomization").

Default workload (N=1): config 3 -- 1024 envs per GPU, forest scene (ground
+ 40 trees + 10 rocks, ~56k triangles per env), 270x480 D455-like depth
camera, depth + segmentation + face index (BASELINE.json configs[2], the
north-star target).  Multi-GPU: one process per GPU (torchrun), each rank
casts its own block of envs (weak scaling: per-GPU work fixed); the step
time is the max over ranks; no data-path collective (envs are independent,
PAPER.md:226).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3|4|5]
    python bench.py --impl reference ...   # the CPU oracle arm
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import scenegen as sg  # noqa: E402

METRIC = "rays/sec and env-frames/sec at 1/2/4/8 B200; % of HBM/FP32 roofline"
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
TRAFFIC_PATH = os.path.join(ROOT, "profiles", "cast_traffic.json")

# Algorithmic thread-instruction costs of one unit of traversal work
# (DESIGN.md §8 "ALU roofline"): per child box test, per
# node pop, per triangle test, per instance entry, per ray (generation +
# epilogue).  Multiplied by each ray's OWN traversal units (counted with one
# ray per lane, so packet over-visits are not counted as useful work); a
# BVH4 node visit is 4 child box tests.
C_BOX, C_LOOP, C_TRI, C_XF, C_RAY = 20, 15, 40, 25, 70
BVH_WIDTH = 4

WORKLOADS = {
    3: "c3: forest, 1024 envs/GPU (ground + 40 trees + 10 rocks, ~56k tri/env), "
       "270x480 D455-like pinhole (87 deg hfov) depth + seg + face, max 10 m",
    4: "c4: Table II-shaped room + 15 floating obstacles, 512 envs/GPU (4096 over 8 GPUs), "
       "OS0-128-style LiDAR 128x512 range + seg, max 10 m",
    5: "c5: Table I-shaped 20 cubes/env re-posed every step (TLAS rebuild), 2048 envs/GPU "
       "(16384 over 8 GPUs), 135x240 depth + seg + face, max 10 m",
    6: "c6 (f3): per-env unique terrain (32768 tri/env), every env's mesh re-randomised and "
       "its BLAS rebuilt every step (agr_update_meshes), 256 envs/GPU, 135x240 depth + seg + face, "
       "max 20 m",
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=3, choices=[3, 4, 5, 6])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--envs", type=int, default=None, help="envs per GPU (default: config's)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-counters", action="store_true")
    ap.add_argument("--trbvh-rounds", type=int, default=None,
                    help="BLAS treelet-restructuring rounds (default 3; 0 for c6, whose BLAS "
                         "are rebuilt every step: there the LBVH alone is the better trade)")
    ap.add_argument("--tlas-builder", default=None, choices=["lbvh", "sah"],
                    help="TLAS builder for agr_build (default: sah for the static c3/c4 "
                         "scenes, lbvh for c5, whose TLAS is rebuilt every step)")
    ap.add_argument("--tlas-step", default=None, choices=["build", "refit"],
                    help="per-step TLAS update (default: refit for c3/c4, whose obstacles "
                         "keep their poses; rebuild for c5, re-posed every step)")
    ap.add_argument("--traversal", default=None, choices=["auto", "lane"],
                    help="auto: warp packets for camera / LiDAR tiles; lane: one ray per lane "
                         "(default: lane for c6, whose terrain seen at grazing angles makes a "
                         "4x8 packet test ~9x the triangles its rays need; auto elsewhere)")
    return ap.parse_args()


def envs_per_gpu(args):
    if args.envs:
        return args.envs
    return {3: 1024, 4: 512, 5: 2048, 6: 256}[args.config]


def make_workload(cfg, n_envs, env_base):
    if cfg == 3:
        return sg.config3(n_envs=n_envs, env_base=env_base)
    if cfg == 4:
        return sg.config4(n_envs=n_envs, env_base=env_base)
    if cfg == 6:
        return sg.config6(n_envs=n_envs, env_base=env_base, ring=2)
    return sg.config5(n_envs=n_envs, env_base=env_base, ring=8)


def blas_launches(n_assets, trbvh_rounds):
    """Kernels one agr_update_meshes batch launches (blas.cu blas_build_batch)."""
    seg_passes = 0
    while n_assets > 1 and ((n_assets - 1) >> (8 * seg_passes)) != 0:
        seg_passes += 1
    n = 5 + 4 * 3  # seg_of, init_bounds, radius, tri_prep, morton; 4 code passes
    if n_assets > 1:
        n += 2 + 3 * seg_passes
    n += 2 + trbvh_rounds + (1 if trbvh_rounds > 0 else 0) + 4
    return n


def env_base(rank, envs_per_rank):
    """Weak scaling: rank r owns global envs [r E, (r+1) E)."""
    return rank * envs_per_rank


def reduce_max(t, world):
    """Max over ranks (step times are max-over-ranks, never wall clock)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t


def combine_checksums(sums, env0=0):
    """One 64-bit digest of per-env checksums (agr_checksum) in global env
    order: sum over envs of checksum_e * (2 e + 1) mod 2^64, so a run on N
    GPUs and a run of the same global envs on one GPU give the same digest."""
    mask = (1 << 64) - 1
    acc = 0
    for i, v in enumerate(np.asarray(sums, np.int64).tolist()):
        acc = (acc + (v & mask) * (2 * (env0 + i) + 1)) & mask
    return f"{acc:016x}"


def gather_checksums(sums, local_ms, world):
    """All-gather every rank's per-env checksums and its local ms/step (the
    only data-path collective of the bench: NCCL under torchrun, outside the
    timed region; BASELINE.json north_star).  Returns (digest over all
    ranks' envs in global order, [ms/step per rank])."""
    import torch
    import torch.distributed as dist
    ms = torch.tensor([local_ms], dtype=torch.float64, device=sums.device)
    if dist.is_available() and dist.is_initialized() and world > 1:
        gs = [torch.zeros_like(sums) for _ in range(world)]
        gm = [torch.zeros_like(ms) for _ in range(world)]
        dist.all_gather(gs, sums)
        dist.all_gather(gm, ms)
        allsums, allms = torch.cat(gs), torch.cat(gm)
    else:
        allsums, allms = sums, ms
    return combine_checksums(allsums.cpu().numpy()), [float(x) for x in allms.cpu()]


def rays_per_env(sensor):
    if sensor["kind"] == "pinhole":
        return sensor["cam"]["W"] * sensor["cam"]["H"] * sensor["poses"].shape[1]
    return sensor["beams"].shape[0] * sensor["beams"].shape[1] * sensor["poses"].shape[1]


def channels_for(cfg):
    return ("dist", "seg") if cfg == 4 else ("dist", "seg", "face")


# --------------------------------------------------------------------------
# clocks sampled during the timed region (NVML)
# --------------------------------------------------------------------------
class ClockSampler:
    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover
            self.nv = None
            self.err = str(e)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.05)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.nv:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.nv:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# --------------------------------------------------------------------------
# CPU oracle (reported baseline; never the target)
# --------------------------------------------------------------------------
def oracle_rate(sc, sensor, kind, n_rays, seed):
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle
    from helpers import oracle_rays
    total = sc.n_envs * rays_per_env(sensor)
    q = np.random.default_rng(seed).choice(total, min(n_rays, total), replace=False)
    t0 = time.perf_counter()
    r = oracle.cast(sc, oracle_rays(sensor, kind), query=q)
    dt = time.perf_counter() - t0
    return len(q) / dt, r.tests / dt, dt, len(q)


def cpu_cores():
    return os.cpu_count() or 1


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg = args.config
    E = envs_per_gpu(args)
    sc, sensor = make_workload(cfg, E, 0)
    kind = "range" if cfg == 4 else "depth"
    per_step = {3: 2500, 4: 20000, 5: 20000, 6: 2000}[cfg]
    for w in range(args.warmup):
        oracle_rate(sc, sensor, kind, per_step // 4, 100 + w)
    times, rays = [], 0
    for k in range(args.steps):
        _, _, dt, n = oracle_rate(sc, sensor, kind, per_step, 1000 + k)
        times.append(dt)
        rays += n
    tot = sum(times)
    value = rays / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "rays/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000 * tot / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOADS[cfg], "envs_per_gpu": E,
                   "rays_per_step": per_step, "sample": "uniform random rays of the workload"},
        "cpu_baseline": {"value": value, "unit": "rays/s", "cores": cpu_cores(), "kind": "oracle",
                         "sample": f"{per_step} random rays per step of the {E}-env workload"},
        "e2e": {"value": value, "unit": "rays/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# --------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist
    import paper_2503_01471_b200 as agr

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    assert world == args.gpus, f"--gpus {args.gpus} but WORLD_SIZE={world}"
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # one process per GPU under torchrun (also for a 1-process torchrun, so
    # the NCCL path is exercised); plain `python bench.py` runs without it
    distributed = "RANK" in os.environ and "MASTER_ADDR" in os.environ
    if distributed:
        dist.init_process_group("nccl", device_id=dev)

    cfg = args.config
    E = envs_per_gpu(args)
    sc, sensor = make_workload(cfg, E, env_base(rank, E))  # this rank's block of global envs
    kind = agr.AGR_RANGE if cfg == 4 else agr.AGR_DEPTH
    chans = channels_for(cfg)
    trbvh_rounds = args.trbvh_rounds if args.trbvh_rounds is not None else (0 if cfg == 6 else 3)
    scene = agr.Scene.from_scenegen(sc, device=local, trbvh_rounds=trbvh_rounds)
    traversal = args.traversal or ("lane" if cfg == 6 else "auto")
    scene.set_traversal(0 if traversal == "auto" else 1)
    tlas_builder = args.tlas_builder or ("lbvh" if cfg in (5, 6) else "sah")
    scene.set_tlas_builder(1 if tlas_builder == "sah" else 0)
    step_refit = (args.tlas_step or ("build" if cfg in (5, 6) else "refit")) == "refit"
    rpe = rays_per_env(sensor)
    rays_per_step = E * rpe
    # inputs resident in HBM before timing
    if cfg == 5:
        ring = torch.from_numpy(sc.extra["ring_T"]).to(dev)
        T_steps = [ring[k] for k in range(ring.shape[0])]
    else:
        T_steps = [torch.from_numpy(sc.inst_T).to(dev)]
    V_steps = None
    if cfg == 6:
        ringv = torch.from_numpy(sc.extra["ring_V"]).to(dev)
        V_steps = [ringv[k] for k in range(ringv.shape[0])]
        all_assets = list(range(len(sc.meshes)))
    poses = torch.from_numpy(sensor["poses"]).to(dev)
    beams = torch.from_numpy(sensor["beams"]).to(dev) if sensor["kind"] == "beams" else None
    scene.set_instance_transforms(T_steps[0])
    scene.build()
    shape = (E, poses.shape[1]) + ((sensor["cam"]["H"], sensor["cam"]["W"]) if beams is None
                                   else tuple(beams.shape[:2]))
    out = {c: torch.empty(shape, dtype=torch.float32 if c == "dist" else torch.int32, device=dev)
           for c in chans}
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def update(k):
        """The per-step scene update: new poses (or, for c6, new meshes) and
        the TLAS refit / rebuild."""
        if V_steps is not None:
            scene.update_meshes(all_assets, V_steps[k % len(V_steps)], stream)
        else:
            scene.set_instance_transforms(T_steps[k % len(T_steps)], stream)
        if step_refit:
            scene.refit(stream)
        else:
            scene.build(stream)

    def step(k):
        update(k)
        if beams is None:
            scene.cast_pinhole(sensor["cam"], poses, sensor["max_range"], kind, out=out, stream=stream)
        else:
            scene.cast_beams(beams, poses, sensor["max_range"], out=out, stream=stream)

    # k_instances + k_tlas + k_cast (+ the batched BLAS rebuild for c6)
    LAUNCHES_PER_STEP = 3 + (blas_launches(len(sc.meshes), trbvh_rounds) if cfg == 6 else 0)
    for w in range(args.warmup):
        step(w)
    torch.cuda.synchronize()

    # ---- timed region: K steps, L2 flushed (untimed) between steps -------
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if distributed:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            flush.zero_()
            e0, e1, e2 = ev[k]
            e0.record(stream)
            update(k)
            e1.record(stream)
            if beams is None:
                scene.cast_pinhole(sensor["cam"], poses, sensor["max_range"], kind, out=out, stream=stream)
            else:
                scene.cast_beams(beams, poses, sensor["max_range"], out=out, stream=stream)
            e2.record(stream)
        torch.cuda.synchronize()
    step_ms = [a.elapsed_time(c) for a, b, c in ev]
    cast_ms = [b.elapsed_time(c) for a, b, c in ev]
    total_ms = sum(step_ms)
    cast_total = sum(cast_ms)
    # per-env checksums of the last step's images and every rank's own
    # ms/step, all-gathered (untimed)
    digest, rank_ms = gather_checksums(scene.checksum(out, rays_per_env(sensor), stream),
                                       total_ms / args.steps, world)
    t = reduce_max(torch.tensor([total_ms, cast_total], dtype=torch.float64, device=dev), world)
    if distributed:
        dist.barrier()
    total_ms, cast_total = float(t[0]), float(t[1])
    ms_per_step = total_ms / args.steps
    value = rays_per_step * world / (total_ms / 1e3 / args.steps)

    # ---- per-ray work counters (separate, untimed counting launch) --------
    counters = lane_counters = None
    if not args.no_counters:
        scene.enable_counters(True)
        step(0)
        torch.cuda.synchronize()
        counters = scene.counters()
        scene.set_traversal(1)  # each ray's own units (algorithmic work)
        step(0)
        torch.cuda.synchronize()
        lane_counters = scene.counters()
        scene.set_traversal(0 if traversal == "auto" else 1)
        scene.enable_counters(False)

    # ---- end to end through the public C ABI with host buffers ------------
    e2e = None
    if not args.no_e2e:
        poses_h = torch.from_numpy(sensor["poses"]).pin_memory()
        out_h = {c: torch.empty(shape, dtype=torch.float32 if c == "dist" else torch.int32,
                                pin_memory=True) for c in chans}
        beams_h = torch.from_numpy(sensor["beams"]).pin_memory() if beams is not None else None

        V_h = [v.cpu().pin_memory() for v in V_steps] if V_steps is not None else None
        V_d = torch.empty_like(V_steps[0]) if V_steps is not None else None

        def e2e_step(k):
            if V_h is not None:  # c6: the step's new meshes come from the host
                V_d.copy_(V_h[k % len(V_h)], non_blocking=True)
                scene.update_meshes(all_assets, V_d, stream)
                scene.refit(stream) if step_refit else scene.build(stream)
            else:
                update(k)
            stream.synchronize()
            if beams_h is None:
                scene.cast_pinhole_host(sensor["cam"], poses_h, sensor["max_range"], kind, out=out_h)
            else:
                scene.cast_beams_host(beams_h, poses_h, sensor["max_range"], out=out_h)

        for w in range(min(args.warmup, 2)):
            e2e_step(w)
        n_e2e = max(3, min(args.steps, 10))
        if distributed:
            dist.barrier()
        t0 = time.perf_counter()
        for k in range(n_e2e):
            e2e_step(k)
        dt = time.perf_counter() - t0
        tt = reduce_max(torch.tensor([dt], dtype=torch.float64, device=dev), world)
        dt = float(tt[0])
        h2d = poses_h.numel() * 4 + (beams_h.numel() * 4 if beams_h is not None else 0) + \
            (V_h[0].numel() * 4 if V_h is not None else 0)
        d2h = sum(v.numel() * 4 for v in out_h.values())
        e2e = {"value": rays_per_step * world * n_e2e / dt, "unit": "rays/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": n_e2e,
               "note": "agr_cast_*_host: H2D poses, chunked cast, D2H of every output image"}

    if distributed:
        dist.destroy_process_group()
    if rank != 0:
        return 0

    # ---- roofline of the dominant kernel (k_cast) -------------------------
    peaks = json.load(open(PEAKS_PATH)) if os.path.exists(PEAKS_PATH) else {}
    clocks = clk.summary()
    cast_s = cast_total / 1e3 / args.steps  # per launch (per rank)
    roof = None
    if lane_counters and lane_counters["rays"] > 0:
        per = {k: lane_counters[k] / lane_counters["rays"] for k in ("nodes", "leaves", "instances")}
        pops = per["nodes"] + per["leaves"] + per["instances"]
        w_ray = BVH_WIDTH * C_BOX * per["nodes"] + C_LOOP * pops + C_TRI * per["leaves"] + \
            C_XF * per["instances"] + C_RAY
        achieved = w_ray * rays_per_step / cast_s / 1e12
        mhz = clocks.get("sm_mhz") or peaks.get("sm_max_mhz", 1965.0)
        peak = 148 * 128 * mhz * 1e6 / 1e12
        traffic = None
        if os.path.exists(TRAFFIC_PATH):
            traffic = json.load(open(TRAFFIC_PATH)).get(f"c{cfg}")
        roof = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "Tinst/s",
                "frac": achieved / peak, "traffic": traffic,
                "kernel": "k_cast", "kernel_ms": 1e3 * cast_s,
                "work_per_ray_inst": w_ray, "per_ray": per,
                "peak_note": "148 SMs x 128 FP32/INT lanes x measured median SM clock "
                             "(DESIGN.md §8); algorithmic instr = counted units x unit costs"}
        out_bytes = rays_per_step * 4 * len(chans)
        hbm_peak = peaks.get("hbm_gbs", 6553.3)
        roof["hbm"] = {"achieved_gbs": out_bytes / cast_s / 1e9, "peak_gbs": hbm_peak,
                       "frac": out_bytes / cast_s / 1e9 / hbm_peak,
                       "bytes_per_launch": out_bytes, "peak_note": "of measured (MEASURED_PEAKS.json)"}

    cpu = None
    if not args.no_cpu_baseline:
        kind_s = "range" if cfg == 4 else "depth"
        n_cpu = {3: 40000, 4: 200000, 5: 200000, 6: 20000}[cfg]
        rate, tests_rate, dt, n = oracle_rate(sc, sensor, kind_s, n_cpu, 7)
        cpu = {"value": rate, "unit": "rays/s", "cores": cpu_cores(), "kind": "oracle",
               "sample": f"{n} uniform random rays of this rank's {E}-env workload ({dt:.1f} s wall)",
               "tri_tests_per_s": tests_rate}

    line = {
        "metric": METRIC, "value": value, "unit": "rays/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32+f64",
        "data": "synthetic",
        "config": {"workload": WORKLOADS[cfg], "envs_per_gpu": E, "rays_per_step_per_gpu": rays_per_step,
                   "channels": list(chans), "parallelism": f"env-sharded x{world}",
                   "l2": "flushed between timed steps (256 MB write, untimed)",
                   "trbvh_rounds": trbvh_rounds, "traversal": traversal,
                   "step": ("update_meshes (every env's BLAS rebuilt)" if cfg == 6 else
                            "set_instance_transforms") + " + TLAS " + ("refit" if step_refit else "rebuild") +
                           " + cast (TLAS builder: " + tlas_builder + ")"},
        "update_ms_per_step": (total_ms - cast_total) / args.steps,
        "checksum": {"digest": digest, "envs": E * world, "last_step": args.steps - 1,
                     "rank_ms_per_step": rank_ms},
        "env_frames_per_sec": E * poses.shape[1] * world / (ms_per_step / 1e3),
        "cast_ms_per_step": cast_total / args.steps,
        "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": LAUNCHES_PER_STEP * args.steps, "clocks": clocks,
        "counters_per_ray": ({k: v / counters["rays"] for k, v in counters.items() if k != "rays"}
                             if counters else None),
        "counters_per_ray_own": ({k: v / lane_counters["rays"] for k, v in lane_counters.items()
                                  if k != "rays"} if lane_counters else None),
    }
    print(json.dumps(line))
    return 0


if __name__ == "__main__":
    sys.exit(main())
