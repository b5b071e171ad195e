#!/usr/bin/env python
"""Benchmark of the batched ray-casting hot path (BASELINE.json metric:
rays/sec and env-frames/sec at 1/2/4/8 B200; % of roofline).

One step = one pass of the whole per-step hot path over one batch of envs
(SURVEY.md §8(a)): set the instance transforms (a3) + per-env TLAS refit or
rebuild (a2/a3) + one fused cast (a4 ray generation, a5 traversal, a6 FP64
epilogue + stores).  The per-asset BLAS (a1) is built once at scene
creation, as in the paper (the BVH is computed "exclusively
for randomization"); c6 (f3) rebuilds every env's BLAS inside the step.

Default workload (N=1): config 3 -- 1024 envs, forest scene (ground + 40
trees + 10 rocks, ~56k triangles per env), 270x480 D455-like depth camera,
depth + segmentation + face index (BASELINE.json configs[2], the north-star
target).

Multi-GPU: one process per GPU.  Under
torchrun the ranks come from the environment; `python bench.py --gpus N`
without it re-launches itself under `torch.distributed.run` (the driver's
own launch line).  Scaling is STRONG by default: the config's total envs
(c3 1024, c4 4096, c5 16384, c6 256) are split into contiguous blocks, GPU g
owning [floor(g E / n), floor((g + 1) E / n)); `--scaling weak` keeps the
per-GPU envs fixed instead.  No collective on the data path (envs are
independent); after the timed region one NCCL all-gather
carries every rank's per-env image checksums and ms/step, and for N > 1
rank 0 re-casts the same global envs alone and checks that the 1-GPU digest
equals the N-GPU one.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3|4|5|6]
    python bench.py --impl reference ...   # the CPU oracle arm
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import scenegen as sg  # noqa: E402

METRIC = "rays/sec and env-frames/sec at 1/2/4/8 B200; % of HBM/FP32 roofline"
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
NCU_PATH = os.path.join(ROOT, "profiles", "cast_ncu.json")  # tools/cast_ncu_summary.py

# Algorithmic thread-instruction costs of one unit of traversal work
# (DESIGN.md §8 "ALU roofline"): per child box test, per
# node pop, per triangle test, per instance entry, per ray (generation +
# epilogue).  Multiplied by each ray's OWN traversal units (counted with one
# ray per lane, so packet over-visits are not counted as useful work); a
# BVH4 node visit is 4 child box tests.
C_BOX, C_LOOP, C_TRI, C_XF, C_RAY = 20, 15, 40, 25, 70
BVH_WIDTH = 4

# Total envs of each config (strong scaling splits them over the GPUs) and
# the per-GPU envs of --scaling weak.
TOTAL_ENVS = {3: 1024, 4: 4096, 5: 16384, 6: 256}
WEAK_ENVS = {3: 1024, 4: 512, 5: 2048, 6: 256}

WORKLOADS = {
    3: "c3: forest (ground + 40 trees + 10 rocks, ~56k tri/env), 270x480 D455-like pinhole "
       "(87 deg hfov) depth + seg + face, max 10 m",
    4: "c4: Table II-shaped room + 15 floating obstacles, OS0-128-style LiDAR 128x512 "
       "range + seg, max 10 m",
    5: "c5: Table I-shaped 20 cubes/env re-posed every step, 135x240 depth + seg + face, max 10 m",
    6: "c6 (f3): per-env unique terrain (32768 tri/env), every env's mesh re-randomised and "
       "its BLAS rebuilt every step (agr_update_meshes), 135x240 depth + seg + face, max 20 m",
}


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=3, choices=[3, 4, 5, 6])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong: the config's total envs split over the GPUs (default); "
                         "weak: a fixed number of envs per GPU")
    ap.add_argument("--envs", type=int, default=None,
                    help="total envs (strong) or envs per GPU (weak); default: the config's")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-counters", action="store_true")
    ap.add_argument("--no-verify", action="store_true",
                    help="skip rank 0's 1-GPU re-cast of all envs (digest check, N > 1)")
    ap.add_argument("--trbvh-rounds", type=int, default=None,
                    help="BLAS treelet-restructuring rounds (default 3; 0 for c6, whose BLAS "
                         "are rebuilt every step: there the LBVH alone is the better trade)")
    ap.add_argument("--tlas-builder", default=None, choices=["lbvh", "sah"],
                    help="TLAS builder for agr_build (default: sah for the static c3/c4 "
                         "scenes, lbvh for c5, whose TLAS is rebuilt every step)")
    ap.add_argument("--tlas-step", default=None, choices=["build", "refit"],
                    help="per-step TLAS update (default: refit for c3/c4, whose obstacles "
                         "keep their poses; rebuild for c5, re-posed every step)")
    ap.add_argument("--traversal", default=None, choices=["auto", "lane", "packet4"],
                    help="auto: warp packets for camera / LiDAR tiles; lane: one ray per lane "
                         "(default: lane for c6, whose terrain seen at grazing angles makes a "
                         "4x8 packet test ~9x the triangles its rays need; auto elsewhere); "
                         "packet4: the interval packets on the 4-wide nodes (A/B)")
    ap.add_argument("--node-width", type=int, default=None, choices=[0, 4, 8, 16, 32],
                    help="agr_create_options.node_width: the interval packets' wide BVH copy (0: the "
                         "library default; 4: none)")
    ap.add_argument("--no-parts", action="store_true",
                    help="one BLAS per asset (agr_create_options.part_policy 1) instead of splitting "
                         "multi-component assets (trees: trunk + canopy) into parts")
    ap.add_argument("--table2", action="store_true",
                    help="only the Table-II-shaped env-step sweep (PAPER.md:276-304): room + 15 "
                         "floating obstacles, 8x8 .. 480x640 depth + seg camera, 128 .. 2048 envs, "
                         "on-device kinematic pose update + (dynamic) refit + cast per step")
    ap.add_argument("--no-table2", action="store_true",
                    help="skip the Table-II sweep that the default run appends to its line")
    ap.add_argument("--t2-res", default="8x8,64x64,270x480,480x640")
    ap.add_argument("--t2-envs", default="128,256,512,1024,2048")
    ap.add_argument("--t2-steps", type=int, default=20)
    ap.add_argument("--t2-traversal", default="auto", choices=["auto", "lane", "packet4"])
    ap.add_argument("--selftest", action="store_true",
                    help="CPU-only check of the multi-rank plumbing (gloo): spawn, env "
                         "sharding, all-gather, digest; no CUDA")
    return ap.parse_args(argv)


# --------------------------------------------------------------------------
# ranks, sharding, collectives
# --------------------------------------------------------------------------
def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def spawn_ranks(n, argv):
    """Re-launch this script as n ranks under torch.distributed.run (the
    same launch line the driver uses); rank 0's JSON line reaches our
    stdout.  Returns the launcher's exit code."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + list(argv)
    return subprocess.call(cmd)


def total_envs(args, world):
    if args.scaling == "weak":
        return (args.envs or WEAK_ENVS[args.config]) * world
    return args.envs or TOTAL_ENVS[args.config]


def shard(E_total, rank, world):
    """GPU g owns global envs [floor(g E / n), floor((g + 1) E / n))
    (SURVEY.md §8(e)): (first env, env count)."""
    lo = E_total * rank // world
    hi = E_total * (rank + 1) // world
    return lo, hi - lo


def env_base(rank, envs_per_rank):
    """Weak scaling: rank r owns global envs [r E, (r+1) E)."""
    return rank * envs_per_rank


def make_workload(cfg, n_envs, env_base):
    if cfg == 3:
        return sg.config3(n_envs=n_envs, env_base=env_base)
    if cfg == 4:
        return sg.config4(n_envs=n_envs, env_base=env_base)
    if cfg == 6:
        return sg.config6(n_envs=n_envs, env_base=env_base, ring=2)
    return sg.config5(n_envs=n_envs, env_base=env_base, ring=8)


def blas_launches(trbvh_rounds, bvh8):
    """Kernels one agr_update_meshes batch launches (blas.cu blas_build_batch):
    seg_of, init_bounds, tri_prep (+ radius), morton; 4 sort passes of hist +
    3-launch scan + scatter; pack_tris, karras, fit; [size copy + treelet
    rounds + depth]; top-down init + top-down BVH4 +
    single-leaf roots [the same three for the BVH8 copy]; asset info
    (checked against the ncu launch list, profiles/r02l_launches_c6.csv)."""
    n = 4 + 4 * 5 + 3
    if trbvh_rounds > 0:
        n += 1 + trbvh_rounds + 1
    n += 3 + (3 if bvh8 else 0) + 1  # (no child-record pass; mesh updates keep the greedy BVH8 collapse)
    return n


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
    only collective of the bench: NCCL under torchrun, outside the timed
    region; BASELINE.json north_star).  Ranks may own different env counts
    (strong scaling), so the counts are gathered first and the sums padded.
    Returns (digest over all ranks' envs in global order, [ms/step per rank])."""
    import torch
    import torch.distributed as dist
    ms = torch.tensor([local_ms], dtype=torch.float64, device=sums.device)
    if dist.is_available() and dist.is_initialized() and world > 1:
        cnt = torch.tensor([sums.numel()], dtype=torch.int64, device=sums.device)
        gc = [torch.zeros_like(cnt) for _ in range(world)]
        dist.all_gather(gc, cnt)
        counts = [int(c.item()) for c in gc]
        pad = torch.zeros(max(counts), dtype=sums.dtype, device=sums.device)
        pad[:sums.numel()] = sums
        gs = [torch.zeros_like(pad) for _ in range(world)]
        gm = [torch.zeros_like(ms) for _ in range(world)]
        dist.all_gather(gs, pad)
        dist.all_gather(gm, ms)
        allsums = torch.cat([g[:c] for g, c in zip(gs, counts)])
        allms = torch.cat(gm)
    else:
        allsums, allms = sums, ms
    return combine_checksums(allsums.cpu().numpy()), [float(x) for x in allms.cpu()]


def rays_per_env(sensor):
    if sensor["kind"] == "pinhole":
        return sensor["cam"]["W"] * sensor["cam"]["H"] * sensor["poses"].shape[1]
    return sensor["beams"].shape[0] * sensor["beams"].shape[1] * sensor["poses"].shape[1]


def channels_for(cfg):
    return ("dist", "seg") if cfg == 4 else ("dist", "seg", "face")


def input_checksums(sc, sensor):
    """Per-env 64-bit digests of the workload INPUTS (instance table,
    transforms, sensor poses) -- the --selftest stand-in for image checksums."""
    import hashlib
    out = []
    P = sensor["poses"].reshape(sc.n_envs, -1)
    for e in range(sc.n_envs):
        i0, i1 = int(sc.env_off[e]), int(sc.env_off[e + 1])
        h = hashlib.sha256()
        for a in (sc.inst_asset[i0:i1], sc.inst_label[i0:i1], sc.inst_T[i0:i1], P[e]):
            h.update(np.ascontiguousarray(a).tobytes())
        out.append(np.frombuffer(h.digest()[:8], np.int64)[0])
    return np.asarray(out, np.int64)


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
            self.h = None
            try:
                # the CUDA device's own GPU (NVML indices ignore CUDA_VISIBLE_DEVICES)
                import torch
                p = torch.cuda.get_device_properties(index)
                bus = f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
                self.h = pynvml.nvmlDeviceGetHandleByPciBusId(bus.encode())
            except Exception:
                self.h = None
            if self.h is None:
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
            time.sleep(0.02)

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
# CPU oracle (reported baseline and parity spot check; never the target)
# --------------------------------------------------------------------------
def _oracle_imports():
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle
    import helpers
    return oracle, helpers


def oracle_sample(sc, sensor, kind, q, n_threads=0):
    """The oracle on ray ids q; returns (result, wall seconds)."""
    oracle, helpers = _oracle_imports()
    t0 = time.perf_counter()
    r = oracle.cast(sc, helpers.oracle_rays(sensor, kind), query=q, n_threads=n_threads)
    return r, time.perf_counter() - t0


def cpu_cores():
    return os.cpu_count() or 1


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def run_reference(args):
    """The reference arm = the oracle as it stands, on this box's host cores,
    one bounded sample of the workload per step (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg = args.config
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    E = total_envs(args, world)
    sc, sensor = make_workload(cfg, E, 0)
    kind = "range" if cfg == 4 else "depth"
    per_step = {3: 2500, 4: 20000, 5: 20000, 6: 2000}[cfg]
    total = sc.n_envs * rays_per_env(sensor)
    for w in range(args.warmup):
        q = np.random.default_rng(100 + w).choice(total, per_step // 4, replace=False)
        oracle_sample(sc, sensor, kind, q)
    times, rays = [], 0
    for k in range(args.steps):
        q = np.random.default_rng(1000 + k).choice(total, per_step, replace=False)
        _, dt = oracle_sample(sc, sensor, kind, q)
        times.append(dt)
        rays += len(q)
    tot = sum(times)
    value = rays / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "rays/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000 * tot / args.steps, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOADS[cfg], "envs_total": E,
                   "rays_per_step": per_step, "sample": "uniform random rays of the workload"},
        "cpu_baseline": {"value": value, "unit": "rays/s", "cores": cpu_cores(), "kind": "oracle",
                         "cpu_model": cpu_model(),
                         "sample": f"{per_step} random rays per step of the {E}-env workload"},
        "e2e": {"value": value, "unit": "rays/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------
# --selftest: the multi-rank plumbing on CPU (gloo), no CUDA
# --------------------------------------------------------------------------
def run_selftest(args):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        dist.init_process_group("gloo")
    E = total_envs(args, world)
    if args.scaling == "weak":
        e0, n = env_base(rank, E // world), E // world
    else:
        e0, n = shard(E, rank, world)
    sc, sensor = make_workload(args.config, n, e0)
    sums = torch.from_numpy(input_checksums(sc, sensor))
    t = time.perf_counter()
    digest, rank_ms = gather_checksums(sums, 1000.0 * (rank + 1), world)
    tmax = reduce_max(torch.tensor([float(rank + 1)], dtype=torch.float64), world)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps({"selftest": True, "n_gpus": world, "envs_total": E, "scaling": args.scaling,
                          "shards": [list(shard(E, r, world)) for r in range(world)]
                          if args.scaling == "strong" else None,
                          "digest": digest, "rank_ms_per_step": rank_ms,
                          "max_over_ranks": float(tmax[0]), "wall_s": time.perf_counter() - t}),
              flush=True)
    return 0


# --------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------
class Workload:
    """One rank's scene, inputs and per-step update, resident on its GPU."""

    def __init__(self, args, cfg, n_envs, e0, dev, agr, torch):
        self.cfg = cfg
        self.sc, self.sensor = make_workload(cfg, n_envs, e0)
        sc, sensor = self.sc, self.sensor
        self.E = n_envs
        self.kind = agr.AGR_RANGE if cfg == 4 else agr.AGR_DEPTH
        self.chans = channels_for(cfg)
        self.trbvh_rounds = args.trbvh_rounds if args.trbvh_rounds is not None else (0 if cfg == 6 else 3)
        self.traversal = args.traversal or ("lane" if cfg == 6 else "auto")
        # the BVH8 copy serves only the interval packets of mode 0: a per-lane
        # scene (c6) keeps BVH4 only, so its per-step BLAS rebuilds skip the
        # 8-wide collapse
        self.scene = agr.Scene.from_scenegen(sc, device=dev.index, trbvh_rounds=self.trbvh_rounds,
                                             parts=not args.no_parts,
                                             node_width=(args.node_width if args.node_width is not None
                                                         else 4 if self.traversal == "lane" else 0))
        self.mode = {"auto": 0, "lane": 1, "packet4": 2}[self.traversal]
        self.scene.set_traversal(self.mode)
        self.tlas_builder = args.tlas_builder or ("lbvh" if cfg in (5, 6) else "sah")
        self.scene.set_tlas_builder(1 if self.tlas_builder == "sah" else 0)
        self.step_refit = (args.tlas_step or ("build" if cfg in (5, 6) else "refit")) == "refit"
        self.rpe = rays_per_env(sensor)
        # inputs resident in HBM before timing
        if cfg == 5:
            ring = torch.from_numpy(sc.extra["ring_T"]).to(dev)
            self.T_steps = [ring[k] for k in range(ring.shape[0])]
        else:
            self.T_steps = [torch.from_numpy(sc.inst_T).to(dev)]
        self.V_steps = None
        if cfg == 6:
            ringv = torch.from_numpy(sc.extra["ring_V"]).to(dev)
            self.V_steps = [ringv[k] for k in range(ringv.shape[0])]
            self.all_assets = list(range(len(sc.meshes)))
        self.poses = torch.from_numpy(sensor["poses"]).to(dev)
        self.beams = torch.from_numpy(sensor["beams"]).to(dev) if sensor["kind"] == "beams" else None
        self.scene.set_instance_transforms(self.T_steps[0])
        self.scene.build()
        self.shape = (n_envs, self.poses.shape[1]) + (
            (sensor["cam"]["H"], sensor["cam"]["W"]) if self.beams is None else tuple(self.beams.shape[:2]))
        self.out = {c: torch.empty(self.shape, dtype=torch.float32 if c == "dist" else torch.int32, device=dev)
                    for c in self.chans}

    def update(self, k, stream):
        """The per-step scene update: new poses (or, for c6, new meshes) and
        the TLAS refit / rebuild."""
        if self.V_steps is not None:
            self.scene.update_meshes(self.all_assets, self.V_steps[k % len(self.V_steps)], stream)
        else:
            self.scene.set_instance_transforms(self.T_steps[k % len(self.T_steps)], stream)
        if self.step_refit:
            self.scene.refit(stream)
        else:
            self.scene.build(stream)

    def cast(self, stream):
        s = self.sensor
        if self.beams is None:
            self.scene.cast_pinhole(s["cam"], self.poses, s["max_range"], self.kind, out=self.out, stream=stream)
        else:
            self.scene.cast_beams(self.beams, self.poses, s["max_range"], out=self.out, stream=stream)

    def step(self, k, stream):
        self.update(k, stream)
        self.cast(stream)

    def checksums(self, stream):
        return self.scene.checksum(self.out, self.rpe, stream)


# --------------------------------------------------------------------------
# Table II-shaped env-step sweep
# --------------------------------------------------------------------------
# The paper's own Aerial Gym numbers (Table II, RTX 3090),
# env-frames/s: context only, another GPU and a full simulator step.
PAPER_T2 = {"8x8": [2951, 5770, 10546, 21690, 37597], "64x64": [2669, 5358, 10097, 16501, 26023],
            "270x480": [1592, 2057, 2408, 2627, 2750], "480x640": [919, 1053, 1136, 1185, 1205]}
PAPER_T2_ENVS = [128, 256, 512, 1024, 2048]


def run_table2(args, dev, agr, torch, env_base=0):
    """One env step = agr_sim_kinematic_step (robots fly to random goals under a
    velocity controller: the "controller-in-the-loop" stand-in, include/agr_sim.h)
    + [dynamic: obstacles drift, agr_set_instance_transforms + agr_refit]
    + agr_cast_pinhole (87 deg hfov, depth + seg, max 10 m), captured once per
    cell as a CUDA graph and replayed; L2 flushed (untimed) between timed
    steps, CUDA events on the launching stream.  'static' is the paper's
    setting ("a room-like static environment consisting of 15 floating
    obstacles"): only the sensors move."""
    res_list = [tuple(int(x) for x in r.split("x")) for r in args.t2_res.split(",")]  # H x W
    env_list = [int(x) for x in args.t2_envs.split(",")]
    E_max = max(env_list)
    base_sc, base_sensor = sg.config4(n_envs=E_max, env_base=env_base)
    robots0, obst0 = sg.table2_sim_records(base_sc, base_sensor["poses"])
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    prm = agr.agr_sim_params(dt=0.01, v_max=2.0, tau=0.2, yaw_rate_max=1.5, goal_radius=0.5,
                             lo=(-4.0, -4.0, 0.5), hi=(4.0, 4.0, 3.5), seed=2025, env_base=env_base)
    cells, launches = [], 0
    for E in env_list:
        sc = base_sc.env_slice(0, E)
        I = sc.n_inst
        scene = agr.Scene.from_scenegen(sc, device=dev.index)
        scene.set_tlas_builder(1)
        scene.set_traversal({"auto": 0, "lane": 1, "packet4": 2}[args.t2_traversal])
        T = torch.from_numpy(sc.inst_T).to(dev)
        scene.set_instance_transforms(T)
        scene.build()
        for H, W in res_list:
            cam = sg.pinhole(W, H, 87.0)
            for mode in ("static", "dynamic"):
                robots = torch.from_numpy(robots0[:E].copy()).to(dev)
                obst = torch.from_numpy(obst0[:I].copy()).to(dev)
                poses = torch.empty((E, 1, 3, 4), dtype=torch.float32, device=dev)
                out = {c: torch.empty((E, 1, H, W), dtype=torch.float32 if c == "dist" else torch.int32,
                                      device=dev) for c in ("dist", "seg")}

                def env_step():
                    if mode == "dynamic":
                        agr.sim_kinematic_step(robots, poses, obst, T, prm)
                        scene.set_instance_transforms(T)
                        scene.refit()
                    else:
                        agr.sim_kinematic_step(robots, poses, None, None, prm)
                    scene.cast_pinhole(cam, poses, 10.0, agr.AGR_DEPTH, out=out)

                per_step = 4 if mode == "dynamic" else 2  # sim (+ k_instances + k_tlas) + k_cast
                env_step()  # un-captured once: allocations / attributes settle
                torch.cuda.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    env_step()
                for _ in range(max(3, args.warmup)):
                    g.replay()
                torch.cuda.synchronize()
                K = args.t2_steps
                ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                      for _ in range(K)]
                for k in range(K):
                    flush.zero_()
                    ev[k][0].record(stream)
                    g.replay()
                    ev[k][1].record(stream)
                torch.cuda.synchronize()
                ms = sum(a.elapsed_time(b) for a, b in ev) / K
                # the same steps back to back without the flush (a simulator
                # loop's steady state: the scene stays in L2)
                w0, w1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                w0.record(stream)
                for k in range(K):
                    g.replay()
                w1.record(stream)
                torch.cuda.synchronize()
                ms_warm = w0.elapsed_time(w1) / K
                launches += per_step * 2 * K
                paper = None
                key = f"{H}x{W}"
                if key in PAPER_T2 and E in PAPER_T2_ENVS:
                    paper = PAPER_T2[key][PAPER_T2_ENVS.index(E)]
                cells.append({"res": f"{H}x{W}", "envs": E, "mode": mode, "ms_per_step": ms,
                              "env_frames_per_sec": E / (ms / 1e3),
                              "ms_per_step_l2_warm": ms_warm,
                              "env_frames_per_sec_l2_warm": E / (ms_warm / 1e3),
                              "rays_per_sec": E * W * H / (ms / 1e3),
                              "paper_rtx3090_fps": paper if mode == "static" else None})
                del g
        scene.close()
    return {"cells": cells, "gpu_launches": launches,
            "step": "graph replay of agr_sim_kinematic_step [+ set_instance_transforms + refit] + cast_pinhole",
            "camera": "pinhole 87 deg hfov, depth + seg, max 10 m",
            "scene": "c4 room 10x10x4 m + 15 floating obstacles per env (SAH TLAS built once)",
            "l2": "flushed between timed steps (256 MB write, untimed)",
            "paper_note": "paper_rtx3090_fps = Table II Aerial Gym FPS (RTX 3090, full simulator step "
                          "with physics + controller; PAPER.md:284-288): context, not a target"}


def table2_main(args, torch, agr):
    """--table2: the sweep alone on one GPU, one JSON line."""
    if int(os.environ.get("RANK", "0")) != 0:
        return 0
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0")))
    torch.cuda.set_device(dev)
    with ClockSampler(dev.index) as clk:
        t2 = run_table2(args, dev, agr, torch)
    head = [c for c in t2["cells"] if c["res"] == "270x480" and c["mode"] == "static"]
    head = max(head, key=lambda c: c["envs"]) if head else t2["cells"][-1]
    line = {"metric": "env-frames/sec (Table II-shaped env step)", "value": head["env_frames_per_sec"],
            "unit": "env-frames/s", "n_gpus": 1, "steps": args.t2_steps, "warmup": max(3, args.warmup),
            "ms_per_step": head["ms_per_step"], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32+f64", "data": "synthetic",
            "config": {"workload": f"t2: {head['res']} depth + seg, {head['envs']} envs, static room + 15 "
                                   "floating obstacles (headline cell of the sweep)",
                       "l2": t2["l2"]},
            "gpu_launches": t2["gpu_launches"], "clocks": clk.summary(), "table2": t2}
    print(json.dumps(line), flush=True)
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return spawn_ranks(args.gpus, sys.argv[1:])
    if args.selftest:
        return run_selftest(args)
    import torch
    import torch.distributed as dist
    import paper_2503_01471_b200 as agr
    if args.table2:
        return table2_main(args, torch, agr)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE={world}; using WORLD_SIZE", file=sys.stderr)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # one process per GPU under torchrun (also for a 1-process torchrun, so
    # the NCCL path is exercised); plain `python bench.py` runs without it
    distributed = "RANK" in os.environ and "MASTER_ADDR" in os.environ
    if distributed:
        dist.init_process_group("nccl", device_id=dev)

    cfg = args.config
    E_total = total_envs(args, world)
    if args.scaling == "weak":
        e0, E = env_base(rank, E_total // world), E_total // world
    else:
        e0, E = shard(E_total, rank, world)
    wl = Workload(args, cfg, E, e0, dev, agr, torch)
    scene, sensor = wl.scene, wl.sensor
    rays_per_step = E * wl.rpe
    rays_total = E_total * wl.rpe
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    # k_instances + k_tlas + k_cast (+ the batched BLAS rebuild for c6)
    LAUNCHES_PER_STEP = 3 + (blas_launches(wl.trbvh_rounds, wl.traversal != "lane") if cfg == 6 else 0)
    for w in range(args.warmup):
        wl.step(w, stream)
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
            e0_, e1_, e2_ = ev[k]
            e0_.record(stream)
            wl.update(k, stream)
            e1_.record(stream)
            wl.cast(stream)
            e2_.record(stream)
        torch.cuda.synchronize()
    step_ms = [a.elapsed_time(c) for a, b, c in ev]
    cast_ms = [b.elapsed_time(c) for a, b, c in ev]
    total_ms = sum(step_ms)
    cast_total = sum(cast_ms)
    # per-env checksums of the last step's images and every rank's own
    # ms/step, all-gathered (untimed)
    digest, rank_ms = gather_checksums(wl.checksums(stream), total_ms / args.steps, world)
    t = reduce_max(torch.tensor([total_ms, cast_total], dtype=torch.float64, device=dev), world)
    if distributed:
        dist.barrier()
    total_ms, cast_total = float(t[0]), float(t[1])
    ms_per_step = total_ms / args.steps
    value = rays_total / (total_ms / 1e3 / args.steps)

    # ---- per-ray work counters (separate, untimed counting launch) --------
    counters = lane_counters = None
    if not args.no_counters:
        scene.enable_counters(True)
        wl.step(0, stream)
        torch.cuda.synchronize()
        counters = scene.counters()
        scene.set_traversal(1)  # each ray's own units (algorithmic work)
        wl.step(0, stream)
        torch.cuda.synchronize()
        lane_counters = scene.counters()
        scene.set_traversal(wl.mode)
        scene.enable_counters(False)

    # ---- end to end through the public C ABI with host buffers ------------
    e2e = None
    if not args.no_e2e:
        poses_h = torch.from_numpy(sensor["poses"]).pin_memory()
        out_h = {c: torch.empty(wl.shape, dtype=torch.float32 if c == "dist" else torch.int32,
                                pin_memory=True) for c in wl.chans}
        beams_h = torch.from_numpy(sensor["beams"]).pin_memory() if wl.beams is not None else None
        V_h = [v.cpu().pin_memory() for v in wl.V_steps] if wl.V_steps is not None else None
        V_d = torch.empty_like(wl.V_steps[0]) if wl.V_steps is not None else None

        def e2e_step(k):
            if V_h is not None:  # c6: the step's new meshes come from the host
                V_d.copy_(V_h[k % len(V_h)], non_blocking=True)
                scene.update_meshes(wl.all_assets, V_d, stream)
                scene.refit(stream) if wl.step_refit else scene.build(stream)
            else:
                wl.update(k, stream)
            # no sync: the host casts wait for the queued scene work themselves
            if beams_h is None:
                scene.cast_pinhole_host(sensor["cam"], poses_h, sensor["max_range"], wl.kind, out=out_h)
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
        # the PCIe ceiling of this path: pinned device->host copy bandwidth of
        # one step's image bytes (torch copies, best of 3; tools/pcie_d2h.py)
        probe_d = torch.empty(d2h // 4, dtype=torch.int32, device=dev)
        probe_h = torch.empty(d2h // 4, dtype=torch.int32, pin_memory=True)
        d2h_gbs = 0.0
        for _ in range(3):
            ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ea.record()
            probe_h.copy_(probe_d, non_blocking=True)
            eb.record()
            torch.cuda.synchronize()
            d2h_gbs = max(d2h_gbs, d2h / (ea.elapsed_time(eb) / 1e3) / 1e9)
        del probe_d, probe_h
        e2e_gbs = d2h * n_e2e / dt / 1e9
        e2e = {"value": rays_total * n_e2e / dt, "unit": "rays/s",
               "h2d_bytes_per_step": h2d * world, "d2h_bytes_per_step": d2h * world, "steps": n_e2e,
               "d2h_gbs": e2e_gbs, "d2h_peak_gbs": d2h_gbs, "d2h_frac": e2e_gbs / d2h_gbs if d2h_gbs else None,
               "note": "agr_cast_*_host: H2D poses, cast in up to 32 env chunks of >= 2^20 rays on one stream while the finished "
                       "chunks' images are copied to pinned host memory on another; d2h_peak_gbs = one "
                       "pinned copy of the same bytes (the PCIe ceiling of this path)"}

    # ---- rank 0 re-casts every global env alone: 1-GPU digest == N-GPU digest
    verify = None
    if world > 1 and not args.no_verify and rank == 0:
        full = Workload(args, cfg, E_total, 0, dev, agr, torch)
        full.update(args.steps - 1, stream)  # the last timed step's scene
        full.cast(stream)
        torch.cuda.synchronize()
        d1 = combine_checksums(full.checksums(stream).cpu().numpy())
        verify = {"one_gpu_digest": d1, "equal": d1 == digest}
        del full
        torch.cuda.empty_cache()
    if distributed:
        dist.barrier()
        dist.destroy_process_group()
    if rank != 0:
        return 0

    # ---- roofline of the dominant kernel (k_cast) -------------------------
    peaks = json.load(open(PEAKS_PATH)) if os.path.exists(PEAKS_PATH) else {}
    clocks = clk.summary()
    cast_s = cast_total / 1e3 / args.steps  # per launch (max over ranks)
    roof = None
    if lane_counters and lane_counters["rays"] > 0:
        per = {k: lane_counters[k] / lane_counters["rays"] for k in ("nodes", "leaves", "instances")}
        pops = per["nodes"] + per["leaves"] + per["instances"]
        w_ray = BVH_WIDTH * C_BOX * per["nodes"] + C_LOOP * pops + C_TRI * per["leaves"] + \
            C_XF * per["instances"] + C_RAY
        achieved = w_ray * rays_per_step / cast_s / 1e12
        mhz = clocks.get("sm_mhz") or peaks.get("sm_max_mhz", 1965.0)
        peak = 148 * 128 * mhz * 1e6 / 1e12
        traffic = ncu = None
        if os.path.exists(NCU_PATH):  # the committed ncu capture of this config's cast
            ncu = json.load(open(NCU_PATH)).get(f"c{cfg}")
            traffic = ncu["traffic"] if ncu else None
        roof = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "Tinst/s",
                "frac": achieved / peak, "traffic": traffic,
                "kernel": "k_cast", "kernel_ms": 1e3 * cast_s,
                "ncu": ncu,  # L2 / L1 hit, FMA / ALU / FP64 pipes, issue activity of the same launch shape
                "work_per_ray_inst": w_ray, "per_ray": per,
                "peak_note": "148 SMs x 128 FP32/INT lanes x measured median SM clock "
                             "(DESIGN.md §8; FMA-loop check in profiles/fma_peak.json); "
                             "algorithmic instr = counted units x unit costs"}
        out_bytes = rays_per_step * 4 * len(wl.chans)
        hbm_peak = peaks.get("hbm_gbs", 6553.3)
        roof["hbm"] = {"achieved_gbs": out_bytes / cast_s / 1e9, "peak_gbs": hbm_peak,
                       "frac": out_bytes / cast_s / 1e9 / hbm_peak,
                       "bytes_per_launch": out_bytes, "peak_note": "of measured (MEASURED_PEAKS.json)"}

    # ---- CPU oracle: baseline rate + parity spot check of step 0's images --
    cpu = parity = None
    if not args.no_cpu_baseline:
        kind_s = "range" if cfg == 4 else "depth"
        wl.step(0, stream)
        torch.cuda.synchronize()
        got = {c: v.cpu().numpy().reshape(-1) for c, v in wl.out.items()}
        total = wl.E * wl.rpe
        n_cpu = {3: 40000, 4: 200000, 5: 200000, 6: 20000}[cfg]
        q = np.random.default_rng(7).choice(total, min(n_cpu, total), replace=False)
        # after update(0) the scene is the generated one: c5 poses ring set 0
        # (= sc.inst_T), c6 meshes ring set 0 (= sc.meshes), c3/c4 never change
        osc = wl.sc
        ref, dt = oracle_sample(osc, sensor, kind_s, q)
        rate = len(q) / dt
        q1 = q[: max(1, len(q) // 32)]
        _, dt1 = oracle_sample(osc, sensor, kind_s, q1, n_threads=1)
        rate1 = len(q1) / dt1
        cpu = {"value": rate, "unit": "rays/s", "cores": cpu_cores(), "kind": "oracle",
               "cpu_model": cpu_model(),
               "sample": f"{len(q)} uniform random rays of rank 0's {wl.E}-env workload ({dt:.1f} s wall)",
               "tri_tests_per_s": ref.tests / dt,
               "one_core": {"value": rate1, "unit": "rays/s", "sample": f"{len(q1)} of those rays"},
               "full_frame_s": rays_total / rate,
               "full_frame_note": "extrapolated: one step of the whole workload at the all-core rate"}
        _, helpers = _oracle_imports()
        try:
            res = helpers.compare(ref, got["dist"][q], got["seg"][q], got["face"][q] if "face" in got else None,
                                  f"bench c{cfg} parity sample")
            parity = {"n": res["n"], "mismatch": 0, "ambiguous": res["ambiguous"], "ties": res["ties"],
                      "grazes": res["grazes"], "max_dist_err_m": res["max_err"],
                      "images": "step 0 (update + cast) after the timed loop"}
        except AssertionError as e:  # reported, never hidden
            parity = {"n": len(q), "failed": str(e)[:1000]}

    line = {
        "metric": METRIC, "value": value, "unit": "rays/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f32+f64",
        "data": "synthetic",
        "config": {"workload": WORKLOADS[cfg], "envs_total": E_total, "envs_rank0": E,
                   "rays_per_step": rays_total, "channels": list(wl.chans),
                   "parallelism": f"env-sharded x{world} ({args.scaling} scaling)",
                   "l2": "flushed between timed steps (256 MB write, untimed)",
                   "trbvh_rounds": wl.trbvh_rounds, "traversal": wl.traversal,
                   "blas_parts": wl.scene.info()["n_parts"], "tlas_items": wl.scene.info()["n_items"],
                   "step": ("update_meshes (every env's BLAS rebuilt)" if cfg == 6 else
                            "set_instance_transforms") + " + TLAS " + ("refit" if wl.step_refit else "rebuild") +
                           " + cast (TLAS builder: " + wl.tlas_builder + ")"},
        "update_ms_per_step": (total_ms - cast_total) / args.steps,
        "checksum": {"digest": digest, "envs": E_total, "last_step": args.steps - 1,
                     "rank_ms_per_step": rank_ms, "verify": verify},
        "env_frames_per_sec": E_total * wl.poses.shape[1] / (ms_per_step / 1e3),
        "cast_ms_per_step": cast_total / args.steps,
        "roofline": roof, "cpu_baseline": cpu, "parity_sample": parity, "e2e": e2e,
        "gpu_launches": LAUNCHES_PER_STEP * args.steps, "clocks": clocks,
        "counters_per_ray": ({k: v / counters["rays"] for k, v in counters.items() if k != "rays"}
                             if counters else None),
        "counters_per_ray_own": ({k: v / lane_counters["rays"] for k, v in lane_counters.items()
                                  if k != "rays"} if lane_counters else None),
    }
    if world == 1 and not args.no_table2:
        # the f4 sweep, after every timed number of the line above (own timing)
        del wl, scene
        torch.cuda.empty_cache()
        line["table2"] = run_table2(args, dev, agr, torch)
    print(json.dumps(line), flush=True)
    return 0 if (verify is None or verify["equal"]) else 3


if __name__ == "__main__":
    sys.exit(main())
