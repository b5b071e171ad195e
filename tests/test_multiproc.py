"""World-size-2 `gloo` tests (CPU) of the multi-GPU host logic used by
bench.py: env sharding (weak scaling, contiguous global env
blocks per rank), per-env input independence from the sharding, and the
max-over-ranks step-time reduction."""
from __future__ import annotations

import hashlib
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench
import scenegen as sg


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _env_digest(sc, e):
    i0, i1 = int(sc.env_off[e]), int(sc.env_off[e + 1])
    h = hashlib.sha256()
    h.update(sc.inst_asset[i0:i1].tobytes())
    h.update(sc.inst_label[i0:i1].tobytes())
    h.update(sc.inst_T[i0:i1].tobytes())
    return np.frombuffer(h.digest()[:8], np.int64)[0]


def _worker(rank, world, port, cfg, E, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sc, sensor = bench.make_workload(cfg, E, bench.env_base(rank, E))
    dig = torch.tensor([_env_digest(sc, e) for e in range(E)], dtype=torch.int64)
    poses = torch.from_numpy(sensor["poses"].reshape(E, -1).copy())
    gathered = [torch.zeros_like(dig) for _ in range(world)]
    dist.all_gather(gathered, dig)
    pg = [torch.zeros_like(poses) for _ in range(world)]
    dist.all_gather(pg, poses)
    t = torch.tensor([10.0 * (rank + 1), 1.0 + rank], dtype=torch.float64)
    tmax = bench.reduce_max(t, world)
    if rank == 0:
        q.put((torch.cat(gathered).numpy(), torch.cat(pg).numpy(), tmax.numpy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("cfg", [3, 5])
def test_two_rank_sharding_matches_single_process(cfg):
    E = 6
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, cfg, E, q)) for r in range(2)]
    for p in procs:
        p.start()
    dig, poses, tmax = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # the 2-rank job covers global envs [0, 2E) exactly once, with the same
    # per-env content as a single process generating all 2E envs
    sc, sensor = bench.make_workload(cfg, 2 * E, 0)
    ref = np.asarray([_env_digest(sc, e) for e in range(2 * E)])
    assert np.array_equal(dig, ref)
    assert np.array_equal(poses, sensor["poses"].reshape(2 * E, -1))
    assert list(tmax) == [20.0, 2.0]  # max over ranks


def test_env_base_is_weak_scaling():
    assert [bench.env_base(r, 1024) for r in range(4)] == [0, 1024, 2048, 3072]


def _ck_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(rank)
    sums = torch.from_numpy(rng.integers(-2**63, 2**63 - 1, 5, dtype=np.int64))
    digest, ms = bench.gather_checksums(sums, 1.5 + rank, world)
    if rank == 0:
        q.put((digest, ms))
    dist.barrier()
    dist.destroy_process_group()


def test_checksum_gather_equals_single_process_digest():
    """bench.gather_checksums (the bench's one collective): the digest of
    two ranks' per-env checksums equals the single-process digest of the
    concatenation in global env order, and every rank's ms is reported."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ck_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    digest, ms = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
    allsums = np.concatenate([np.random.default_rng(r).integers(-2**63, 2**63 - 1, 5, dtype=np.int64)
                              for r in range(2)])
    assert digest == bench.combine_checksums(allsums)
    assert ms == [1.5, 2.5]
    # order matters (global env order), a single changed checksum changes it
    assert bench.combine_checksums(allsums[::-1]) != digest
    alt = allsums.copy()
    alt[7] ^= 1
    assert bench.combine_checksums(alt) != digest


def test_shard_is_strong_scaling():
    """GPU g owns [floor(gN/n), floor((g+1)N/n)); the
    blocks tile [0, N) exactly, also when n does not divide N."""
    for N, n in ((1024, 8), (1024, 3), (16384, 7), (5, 8)):
        blocks = [bench.shard(N, g, n) for g in range(n)]
        assert blocks[0][0] == 0 and sum(c for _, c in blocks) == N
        for (a, c), (b, _) in zip(blocks, blocks[1:]):
            assert a + c == b
    assert [bench.shard(1024, g, 8) for g in range(2)] == [(0, 128), (128, 128)]


@pytest.mark.parametrize("world,cfg,scaling", [(2, 5, "strong"), (3, 3, "strong"), (2, 4, "weak")])
def test_bench_spawn_path_gloo(world, cfg, scaling):
    """`python bench.py --gpus N` without torchrun re-launches itself as N
    ranks under torch.distributed.run (bench.spawn_ranks, the driver's launch
    line); --selftest runs the same sharding + all-gather + digest on CPU
    (gloo).  The N-rank digest of the per-env input checksums equals the
    single-process digest of the same global envs."""
    import json
    import subprocess
    import sys
    E = {5: 40, 3: 7, 4: 6}[cfg]
    cmd = [sys.executable, os.path.join(os.path.dirname(bench.__file__), "bench.py"), "--gpus", str(world),
           "--selftest", "--config", str(cfg), "--envs", str(E), "--scaling", scaling]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr[-2000:]
    line = json.loads([ln for ln in p.stdout.splitlines() if ln.startswith("{")][-1])
    total = E if scaling == "strong" else E * world
    assert line["n_gpus"] == world and line["envs_total"] == total
    assert line["rank_ms_per_step"] == [1000.0 * (r + 1) for r in range(world)]
    assert line["max_over_ranks"] == float(world)
    sc, sensor = bench.make_workload(cfg, total, 0)
    assert line["digest"] == bench.combine_checksums(bench.input_checksums(sc, sensor))
