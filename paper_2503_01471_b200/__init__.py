"""B200-native batched ray caster for parallel robot-simulation sensors.

Thin Python binding over ``lib/libagr.so`` (the C ABI declared in
``include/agr.h``).  This module only marshals arguments: every step of the
hot path (BLAS/TLAS build, ray generation, traversal, arbitration, stores)
runs in the CUDA kernels of ``csrc/``.  PyTorch is used for device memory
and streams only.  There is no CPU fallback: if the library or a GPU is
missing, calls raise.

Paper: Aerial Gym Simulator (arxiv 2503.01471), §III.D.1 lines
226-228 (per-env meshes of transformed sub-meshes, BVH, per-pixel rays,
range vs depth, segmentation and face-index images).
"""
from __future__ import annotations

import ctypes
import os
import re

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libagr.so")
# experiments only: load an alternative build of the same library
LIB_PATH = os.environ.get("AGR_LIB_PATH", LIB_PATH)
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "agr.h")
SIM_HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "agr_sim.h")

AGR_OK, AGR_EINVAL, AGR_ENOMEM, AGR_ECUDA, AGR_ESTATE, AGR_EUNSUPPORTED = 0, -1, -2, -3, -4, -5
AGR_DEPTH, AGR_RANGE = 0, 1
_STATUS = {0: "AGR_OK", -1: "AGR_EINVAL", -2: "AGR_ENOMEM", -3: "AGR_ECUDA", -4: "AGR_ESTATE",
           -5: "AGR_EUNSUPPORTED"}


class AgrError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


class agr_mesh(ctypes.Structure):
    _fields_ = [("verts", ctypes.c_void_p), ("n_verts", ctypes.c_int32),
                ("faces", ctypes.c_void_p), ("n_faces", ctypes.c_int32)]


class agr_instance(ctypes.Structure):
    _fields_ = [("asset", ctypes.c_int32), ("label", ctypes.c_int32)]


class agr_pinhole(ctypes.Structure):
    _fields_ = [("width", ctypes.c_int32), ("height", ctypes.c_int32),
                ("fx", ctypes.c_float), ("fy", ctypes.c_float),
                ("cx", ctypes.c_float), ("cy", ctypes.c_float)]


class agr_outputs(ctypes.Structure):
    _fields_ = [("dist", ctypes.c_void_p), ("seg", ctypes.c_void_p), ("face", ctypes.c_void_p),
                ("normal", ctypes.c_void_p), ("bary", ctypes.c_void_p), ("point", ctypes.c_void_p),
                ("valid", ctypes.c_void_p), ("annot", ctypes.c_void_p)]


# channel -> (torch dtype name, trailing vector size)
CHANNELS = {"dist": ("float32", None), "seg": ("int32", None), "face": ("int32", None),
            "normal": ("float32", 3), "bary": ("float32", 2), "point": ("float32", 3),
            "valid": ("int32", None), "annot": ("float32", "k")}  # k: the scene's annotation width


class agr_create_options(ctypes.Structure):
    _fields_ = [("trbvh_rounds", ctypes.c_int32), ("part_policy", ctypes.c_int32),
                ("node_width", ctypes.c_int32), ("reserved", ctypes.c_int32 * 5)]


class agr_scene_info(ctypes.Structure):
    _fields_ = [("n_assets", ctypes.c_int32), ("n_envs", ctypes.c_int32),
                ("n_instances", ctypes.c_int64), ("n_blas_nodes", ctypes.c_int64),
                ("n_blas_tris", ctypes.c_int64), ("n_tlas_nodes", ctypes.c_int64),
                ("blas_max_depth", ctypes.c_int32), ("tlas_max_depth", ctypes.c_int32),
                ("device_bytes", ctypes.c_int64), ("built", ctypes.c_int32),
                ("n_parts", ctypes.c_int32), ("n_items", ctypes.c_int64)]


class agr_sim_params(ctypes.Structure):
    """include/agr_sim.h: the kinematic env-step stand-in's parameters."""
    _fields_ = [("dt", ctypes.c_float), ("v_max", ctypes.c_float), ("tau", ctypes.c_float),
                ("yaw_rate_max", ctypes.c_float), ("goal_radius", ctypes.c_float),
                ("lo", ctypes.c_float * 3), ("hi", ctypes.c_float * 3),
                ("seed", ctypes.c_uint32), ("env_base", ctypes.c_int32)]


SIM_ROBOT_FLOATS = 12     # sizeof(agr_sim_robot) / 4
SIM_OBSTACLE_FLOATS = 20  # sizeof(agr_sim_obstacle) / 4

_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_SIGS = {
    "agr_abi_version": (_I32, []),
    "agr_last_error": (ctypes.c_char_p, []),
    "agr_scene_create": (_I32, [_I32, ctypes.POINTER(agr_mesh), _I32, _I32, _P,
                                ctypes.POINTER(agr_instance), ctypes.POINTER(_P)]),
    "agr_scene_create_ex": (_I32, [_I32, ctypes.POINTER(agr_mesh), _I32, _I32, _P,
                                   ctypes.POINTER(agr_instance), ctypes.POINTER(agr_create_options),
                                   ctypes.POINTER(_P)]),
    "agr_scene_destroy": (_I32, [_P]),
    "agr_scene_get_info": (_I32, [_P, ctypes.POINTER(agr_scene_info)]),
    "agr_set_instance_transforms": (_I32, [_P, _P, _P]),
    "agr_build": (_I32, [_P, _P]),
    "agr_update_mesh": (_I32, [_P, _I32, _P, _I32, _P]),
    "agr_update_meshes": (_I32, [_P, _I32, _P, _P, _P]),
    "agr_set_vertex_annotations": (_I32, [_P, _I32, _P, _I32, _I32, _P]),
    "agr_refit": (_I32, [_P, _P]),
    "agr_cast_pinhole": (_I32, [_P, ctypes.POINTER(agr_pinhole), _I32, _P, _I32, ctypes.c_float,
                                agr_outputs, _P]),
    "agr_cast_beams": (_I32, [_P, _P, _I32, _I32, _P, _I32, ctypes.c_float, agr_outputs, _P]),
    "agr_cast_rays": (_I32, [_P, _P, _P, _I32, ctypes.c_float, agr_outputs, _P]),
    "agr_cast_pinhole_host": (_I32, [_P, ctypes.POINTER(agr_pinhole), _I32, _P, _I32,
                                     ctypes.c_float, agr_outputs]),
    "agr_cast_beams_host": (_I32, [_P, _P, _I32, _I32, _P, _I32, ctypes.c_float, agr_outputs]),
    "agr_checksum": (_I32, [_P, agr_outputs, ctypes.c_int64, _P, _P]),
    "agr_set_exact_mode": (_I32, [_P, _I32]),
    "agr_set_traversal": (_I32, [_P, _I32]),
    "agr_set_tlas_builder": (_I32, [_P, _I32]),
    "agr_set_stereo": (_I32, [_P, ctypes.c_float, ctypes.c_float, ctypes.c_float, ctypes.c_float]),
    "agr_enable_counters": (_I32, [_P, _I32]),
    "agr_get_counters": (_I32, [_P, _P]),
    "agr_debug_export_blas": (_I32, [_P, _I32, _P, _P, _P, ctypes.POINTER(ctypes.c_int64),
                                     ctypes.POINTER(ctypes.c_int64)]),
    "agr_debug_export_bvh4": (_I32, [_P, _I32, _P, ctypes.POINTER(ctypes.c_int32),
                                     ctypes.POINTER(ctypes.c_int64)]),
    "agr_debug_asset_parts": (_I32, [_P, _I32, _P, ctypes.POINTER(ctypes.c_int32)]),
    "agr_sim_kinematic_step": (_I32, [_P, _I32, _P, _P, ctypes.c_int64, _P,
                                      ctypes.POINTER(agr_sim_params), _P]),
}

_lib = None


def load():
    """dlopen libagr.so (raises if it was not built: there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run `make` (or __graft_entry__.build())")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(lib, name)
            f.restype = res
            f.argtypes = args
        _lib = lib
    return _lib


def header_symbols():
    """Function names declared in include/agr.h and include/agr_sim.h."""
    txt = ""
    for path in (HEADER_PATH, SIM_HEADER_PATH):
        with open(path) as f:
            txt += f.read()
    return sorted(set(re.findall(r"^\s*(?:agr_status|int32_t|const char\*)\s+(agr_\w+)\s*\(", txt, re.M)))


def _check(st):
    if st != AGR_OK:
        raise AgrError(st, load().agr_last_error().decode())


def last_error() -> str:
    return load().agr_last_error().decode()


def _ptr(t):
    """Device/host pointer of a torch tensor or numpy array (None -> NULL)."""
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


def _stream_handle(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream


def _outputs(out: dict):
    return agr_outputs(*(_ptr(out.get(k)) for k in CHANNELS))


class Scene:
    """Owner of an ``agr_scene`` handle (one CUDA device)."""

    def __init__(self, meshes, env_offsets, inst_asset, inst_label, device: int = 0,
                 trbvh_rounds: int = 3, parts: bool = True, node_width: int = 0):
        """meshes: list of (verts float32 [V][3], faces int32 [F][3]) host arrays.
        trbvh_rounds: treelet-restructuring passes on every BLAS (0 = LBVH).
        parts: split multi-component assets into BLAS parts when it pays
        (agr_create_options.part_policy 0); False: one BLAS per asset.
        node_width: the interval packets' wide BVH copy: 8, 16 or 32 (0: 32),
        4: BVH4 only."""
        lib = load()
        self._keep = []
        arr = (agr_mesh * len(meshes))()
        for i, (v, f) in enumerate(meshes):
            v = np.ascontiguousarray(v, np.float32)
            f = np.ascontiguousarray(f, np.int32)
            self._keep += [v, f]
            arr[i] = agr_mesh(v.ctypes.data, len(v), f.ctypes.data, len(f))
        env_offsets = np.ascontiguousarray(env_offsets, np.int64)
        n_inst = int(env_offsets[-1])
        inst = (agr_instance * max(n_inst, 1))()
        ia = np.asarray(inst_asset, np.int32)
        il = np.asarray(inst_label, np.int32)
        for j in range(n_inst):
            inst[j] = agr_instance(int(ia[j]), int(il[j]))
        h = _P()
        opts = agr_create_options(int(trbvh_rounds), 0 if parts else 1, int(node_width))
        _check(lib.agr_scene_create_ex(device, arr, len(meshes), len(env_offsets) - 1,
                                       env_offsets.ctypes.data, inst, ctypes.byref(opts), ctypes.byref(h)))
        self._keep = []
        self.handle = h
        self.device = device
        self.n_envs = len(env_offsets) - 1
        self.annot_k = 0
        self.n_inst = n_inst

    @classmethod
    def from_scenegen(cls, sc, device: int = 0, trbvh_rounds: int = 3, parts: bool = True,
                      node_width: int = 0):
        """Build from a ``scenegen.Scene`` (inputs only; no arithmetic)."""
        return cls([(m.verts, m.faces) for m in sc.meshes], sc.env_off, sc.inst_asset,
                   sc.inst_label, device, trbvh_rounds, parts, node_width)

    def close(self):
        if getattr(self, "handle", None):
            load().agr_scene_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- build ------------------------------------------------------------
    def set_instance_transforms(self, T, stream=None):
        """T: CUDA float32 tensor [n_inst, 3, 4] (object -> env-local)."""
        _check(load().agr_set_instance_transforms(self.handle, _ptr(T), _stream_handle(stream)))

    def update_mesh(self, asset: int, verts, stream=None):
        """verts: CUDA float32 [V, 3] (same V as at create); rebuilds the BLAS."""
        _check(load().agr_update_mesh(self.handle, int(asset), _ptr(verts), int(verts.shape[0]),
                                      _stream_handle(stream)))

    def set_vertex_annotations(self, asset: int, values, stream=None):
        """values: CUDA float32 [V, k] per-vertex annotations of `asset` (same k
        for every asset); casts with the "annot" channel interpolate them."""
        v = values if values.dim() == 2 else values.reshape(values.shape[0], -1)
        _check(load().agr_set_vertex_annotations(self.handle, int(asset), _ptr(v), int(v.shape[0]),
                                                 int(v.shape[1]), _stream_handle(stream)))
        self.annot_k = int(v.shape[1])

    def update_meshes(self, assets, verts, stream=None):
        """Batched update_mesh: ``assets`` a sequence of distinct asset ids,
        ``verts`` CUDA float32 [sum V, 3] (their vertex arrays concatenated in
        that order); all BLAS are rebuilt in one set of launches."""
        a = np.ascontiguousarray(assets, dtype=np.int32)
        _check(load().agr_update_meshes(self.handle, len(a), a.ctypes.data, _ptr(verts),
                                        _stream_handle(stream)))

    def build(self, stream=None):
        _check(load().agr_build(self.handle, _stream_handle(stream)))

    def refit(self, stream=None):
        _check(load().agr_refit(self.handle, _stream_handle(stream)))

    def info(self) -> dict:
        inf = agr_scene_info()
        _check(load().agr_scene_get_info(self.handle, ctypes.byref(inf)))
        return {k: getattr(inf, k) for k, _ in agr_scene_info._fields_}

    # ---- casts ------------------------------------------------------------
    def _alloc(self, shape, channels, device_tensors=True, pin=False):
        import torch
        dev = torch.device("cuda", self.device) if device_tensors else torch.device("cpu")
        out = {}
        for ch in channels:
            dt, vec = CHANNELS[ch]
            if vec == "k":
                if not self.annot_k:
                    raise AgrError(AGR_EINVAL, "annot requested but no vertex annotations set")
                vec = self.annot_k
            shp = tuple(shape) + ((vec,) if vec else ())
            out[ch] = torch.empty(shp, dtype=getattr(torch, dt), device=dev,
                                  pin_memory=pin and not device_tensors)
        return out

    def cast_pinhole(self, cam: dict, poses, max_range: float, kind: int = AGR_DEPTH,
                     out=None, channels=("dist", "seg", "face"), stream=None):
        """poses: CUDA float32 [n_envs, S, 3, 4].  Returns dict of [E,S,H,W] tensors."""
        S = poses.shape[1]
        if out is None:
            out = self._alloc((self.n_envs, S, cam["H"], cam["W"]), channels)
        c = agr_pinhole(cam["W"], cam["H"], cam["fx"], cam["fy"], cam["cx"], cam["cy"])
        _check(load().agr_cast_pinhole(self.handle, ctypes.byref(c), kind, _ptr(poses), S,
                                       float(max_range),
                                       _outputs(out),
                                       _stream_handle(stream)))
        return out

    def cast_beams(self, beams, poses, max_range: float, out=None,
                   channels=("dist", "seg", "face"), stream=None):
        """beams: CUDA float32 [C, K, 3]; poses [n_envs, S, 3, 4]."""
        C, K = beams.shape[0], beams.shape[1]
        S = poses.shape[1]
        if out is None:
            out = self._alloc((self.n_envs, S, C, K), channels)
        _check(load().agr_cast_beams(self.handle, _ptr(beams), C, K, _ptr(poses), S,
                                     float(max_range),
                                     _outputs(out),
                                     _stream_handle(stream)))
        return out

    def cast_rays(self, orig, dirs, max_range: float, out=None,
                  channels=("dist", "seg", "face"), stream=None):
        """orig, dirs: CUDA float32 [n_envs, R, 3] env-local."""
        R = orig.shape[1]
        if out is None:
            out = self._alloc((self.n_envs, R), channels)
        _check(load().agr_cast_rays(self.handle, _ptr(orig), _ptr(dirs), R, float(max_range),
                                    _outputs(out),
                                    _stream_handle(stream)))
        return out

    def cast_pinhole_host(self, cam: dict, poses_host, max_range: float, kind: int = AGR_DEPTH,
                          out=None, channels=("dist", "seg", "face")):
        """End-to-end cast through host buffers (synchronous).  poses_host:
        CPU float32 [n_envs, S, 3, 4]; outputs are CPU tensors (pinned if
        allocated here)."""
        S = poses_host.shape[1]
        if out is None:
            out = self._alloc((self.n_envs, S, cam["H"], cam["W"]), channels, False, pin=True)
        c = agr_pinhole(cam["W"], cam["H"], cam["fx"], cam["fy"], cam["cx"], cam["cy"])
        _check(load().agr_cast_pinhole_host(self.handle, ctypes.byref(c), kind, _ptr(poses_host), S,
                                            float(max_range),
                                            _outputs(out)))
        return out

    def cast_beams_host(self, beams_host, poses_host, max_range: float, out=None,
                        channels=("dist", "seg", "face")):
        C, K = beams_host.shape[0], beams_host.shape[1]
        S = poses_host.shape[1]
        if out is None:
            out = self._alloc((self.n_envs, S, C, K), channels, False, pin=True)
        _check(load().agr_cast_beams_host(self.handle, _ptr(beams_host), C, K, _ptr(poses_host), S,
                                          float(max_range),
                                          _outputs(out)))
        return out

    def checksum(self, out: dict, elems_per_env: int, stream=None):
        import torch
        sums = torch.zeros(self.n_envs, dtype=torch.int64, device=torch.device("cuda", self.device))
        _check(load().agr_checksum(self.handle,
                                   _outputs(out),
                                   int(elems_per_env), _ptr(sums), _stream_handle(stream)))
        return sums

    # ---- test / profiling hooks --------------------------------------------
    def set_exact_mode(self, exact: bool):
        _check(load().agr_set_exact_mode(self.handle, 1 if exact else 0))

    def set_stereo(self, offset=(0.0, -0.095, 0.0), eps: float = 1e-4):
        """Second sensor origin (sensor frame) and self-hit guard for `valid`."""
        _check(load().agr_set_stereo(self.handle, *(float(x) for x in offset), float(eps)))

    def set_tlas_builder(self, builder: int):
        """0 LBVH (Morton + Karras; the default), 1 binned SAH for agr_build."""
        _check(load().agr_set_tlas_builder(self.handle, int(builder)))

    def set_traversal(self, mode: int):
        """0 auto (interval packets for pinhole / beam tiles on the BVH8 when
        built; per-lane rays for pinholes whose 4x8 tile spans > 0.12 rad),
        1 per-lane rays, 2 interval packets on the BVH4 for every camera,
        3 interval packets on the BVH8 for every camera."""
        _check(load().agr_set_traversal(self.handle, int(mode)))

    def enable_counters(self, enable: bool):
        _check(load().agr_enable_counters(self.handle, 1 if enable else 0))

    def counters(self) -> dict:
        c = np.zeros(8, np.int64)
        _check(load().agr_get_counters(self.handle, c.ctypes.data))
        return dict(rays=int(c[0]), nodes=int(c[1]), leaves=int(c[2]), instances=int(c[3]),
                    fp64_tests=int(c[4]), overflow=int(c[5]), tlas_nodes=int(c[6]),
                    empty_entries=int(c[7]))

    def debug_export_blas(self, asset: int):
        nn, nl = ctypes.c_int64(), ctypes.c_int64()
        lib = load()
        _check(lib.agr_debug_export_blas(self.handle, asset, None, None, None,
                                         ctypes.byref(nn), ctypes.byref(nl)))
        nodes = np.zeros((nn.value, 16), np.float32)
        faces = np.zeros(max(nl.value, 1), np.int32)
        codes = np.zeros(max(nl.value, 1), np.uint32)
        _check(lib.agr_debug_export_blas(self.handle, asset, nodes.ctypes.data, faces.ctypes.data,
                                         codes.ctypes.data, ctypes.byref(nn), ctypes.byref(nl)))
        return nodes, faces[:nl.value], codes[:nl.value]


    def debug_asset_parts(self, asset: int, n_faces: int):
        """(n_parts, part of each of the asset's n_faces faces)."""
        n = ctypes.c_int32()
        part = np.zeros(n_faces, np.int32)
        _check(load().agr_debug_asset_parts(self.handle, int(asset), part.ctypes.data, ctypes.byref(n)))
        return n.value, part

    def debug_export_bvh4(self, which: int):
        """BVH4 nodes of asset `which` (>= 0) or of env (-1 - which)'s TLAS."""
        n = ctypes.c_int64()
        root = ctypes.c_int32()
        lib = load()
        _check(lib.agr_debug_export_bvh4(self.handle, which, None, ctypes.byref(root), ctypes.byref(n)))
        nodes = np.zeros((n.value, 32), np.float32)
        _check(lib.agr_debug_export_bvh4(self.handle, which, nodes.ctypes.data, ctypes.byref(root),
                                         ctypes.byref(n)))
        return nodes, root.value


def sim_kinematic_step(robots, poses, obstacles, obst_T, params: agr_sim_params, stream=None):
    """agr_sim_kinematic_step (include/agr_sim.h): the simulator stand-in of
    the Table-II env-step benchmark.  robots: CUDA float32 [E, 12] (one
    agr_sim_robot per env); poses: CUDA float32 [E, 1, 3, 4] (written);
    obstacles: CUDA float32 [I, 20] (agr_sim_obstacle records) or None;
    obst_T: CUDA float32 [I, 3, 4] (written) or None."""
    n_obst = 0 if obstacles is None else int(obstacles.shape[0])
    _check(load().agr_sim_kinematic_step(_ptr(robots), int(robots.shape[0]), _ptr(poses),
                                         _ptr(obstacles), n_obst, _ptr(obst_T),
                                         ctypes.byref(params), _stream_handle(stream)))


def abi_version() -> int:
    return int(load().agr_abi_version())
