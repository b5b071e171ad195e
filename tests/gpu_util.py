"""GPU-side test helpers: build a libagr scene from scenegen inputs and run
casts through the C ABI binding.  Argument marshalling only."""
from __future__ import annotations

import numpy as np
import torch

import paper_2503_01471_b200 as agr


def dev():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device (there is no CPU fallback)"
    return torch.device("cuda", 0)


def make_scene(sc, transforms=None, build=True, trbvh_rounds=3, parts=True):
    s = agr.Scene.from_scenegen(sc, device=0, trbvh_rounds=trbvh_rounds, parts=parts)
    T = sc.inst_T if transforms is None else transforms
    if s.n_inst:
        s.set_instance_transforms(torch.from_numpy(np.ascontiguousarray(T, np.float32)).to(dev()))
    if build:
        s.build()
    return s


def cast_sensor(s, sensor, kind="depth", channels=("dist", "seg", "face")):
    poses = torch.from_numpy(np.ascontiguousarray(sensor["poses"], np.float32)).to(dev())
    if sensor["kind"] == "pinhole":
        out = s.cast_pinhole(sensor["cam"], poses, sensor["max_range"],
                             agr.AGR_DEPTH if kind == "depth" else agr.AGR_RANGE, channels=channels)
    else:
        beams = torch.from_numpy(np.ascontiguousarray(sensor["beams"], np.float32)).to(dev())
        out = s.cast_beams(beams, poses, sensor["max_range"], channels=channels)
    torch.cuda.synchronize()
    return out


def to_np(out):
    return {k: v.cpu().numpy().reshape(-1) for k, v in out.items()}
