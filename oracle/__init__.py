"""CPU brute-force ray-casting oracle -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package.  The product path
(``paper_2503_01471_b200``) never imports it and shares no code with it.

This module is argument marshalling over ``oracle/liboracle.so`` (plain C,
FP64, built from ``oracle/oracle.c``); see ``oracle/oracle.h`` for the
definition it computes and the PAPER.md passages it follows
(§III.D.1).

Parity-pin status: every output (distance, seg, face and the
ambiguity flags) is pinned by closed forms and invariants in
``tests/test_oracle_pins.py``; the paper itself prints no per-ray value.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

RAYS, PINHOLE, BEAMS = 0, 1, 2
DEPTH, RANGE = 0, 1
AMB_TIE, AMB_RANGE, AMB_ZERO, AMB_SHADOW, AMB_GRAZE = 1, 2, 4, 8, 16
NEAR_REL = 2.0 ** -40  # oracle.c ORACLE_NEAR_REL: near-candidate band nu = NEAR_REL * M
AMB_EPS = 1e-5  # metres, SURVEY.md §8(c) parity rules / BASELINE.json north_star


def build() -> str:
    """Compile liboracle.so with gcc (plain C, -O2, pthreads)."""
    src = os.path.join(_HERE, "oracle.c")
    if (not os.path.exists(_LIB_PATH)
            or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src)
            or os.path.getmtime(_LIB_PATH) < os.path.getmtime(os.path.join(_HERE, "oracle.h"))):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-pthread",
                               "-Wall", "-o", _LIB_PATH, src, "-lm"])
    return _LIB_PATH


class _Scene(ctypes.Structure):
    _fields_ = [
        ("n_assets", ctypes.c_int32),
        ("verts", ctypes.c_void_p), ("vert_off", ctypes.c_void_p),
        ("faces", ctypes.c_void_p), ("face_off", ctypes.c_void_p),
        ("n_envs", ctypes.c_int32), ("env_off", ctypes.c_void_p),
        ("inst_asset", ctypes.c_void_p), ("inst_label", ctypes.c_void_p),
        ("inst_T", ctypes.c_void_p),
        ("annot", ctypes.c_void_p), ("annot_k", ctypes.c_int32),
    ]


class _Rays(ctypes.Structure):
    _fields_ = [
        ("model", ctypes.c_int32),
        ("orig", ctypes.c_void_p), ("dir", ctypes.c_void_p), ("R", ctypes.c_int32),
        ("W", ctypes.c_int32), ("H", ctypes.c_int32),
        ("fx", ctypes.c_float), ("fy", ctypes.c_float),
        ("cx", ctypes.c_float), ("cy", ctypes.c_float),
        ("kind", ctypes.c_int32),
        ("beams", ctypes.c_void_p), ("C", ctypes.c_int32), ("K", ctypes.c_int32),
        ("poses", ctypes.c_void_p), ("S", ctypes.c_int32),
        ("max_range", ctypes.c_float),
        ("stereo", ctypes.c_float * 3), ("stereo_eps", ctypes.c_float),
    ]


_lib = None


def _load():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        _lib.oracle_cast.restype = ctypes.c_int
        _lib.oracle_cast.argtypes = [ctypes.POINTER(_Scene), ctypes.POINTER(_Rays),
                                     ctypes.c_void_p, ctypes.c_int64, ctypes.c_double,
                                     ctypes.c_int32] + [ctypes.c_void_p] * 12
        _lib.oracle_last_tests.restype = ctypes.c_int64
        _lib.oracle_certify.restype = ctypes.c_int
        _lib.oracle_certify.argtypes = [ctypes.POINTER(_Scene), ctypes.POINTER(_Rays),
                                        ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                        ctypes.c_int32] + [ctypes.c_void_p] * 3
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data


@dataclass
class OracleResult:
    t64: np.ndarray    # float64 winning t (max_range on miss)
    dist: np.ndarray   # float32(t64)
    seg: np.ndarray    # int32
    face: np.ndarray   # int32
    amb: np.ndarray    # int32 AMB_* bits
    t2: np.ndarray     # float64 second-best candidate t
    graze: np.ndarray  # float64 silhouette diagnostic
    tests: int         # ray/triangle tests performed
    normal: np.ndarray = None  # float64 [n][3] (extras=True)
    bary: np.ndarray = None    # float64 [n][2]
    point: np.ndarray = None   # float64 [n][3]
    valid: np.ndarray = None   # int32 [n] stereo shadow mask (stereo=...)
    annot: np.ndarray = None   # float64 [n][K] interpolated vertex annotations (annot=...)


def cast(scene, rays: dict, query=None, n_threads: int = 0, amb_eps: float = AMB_EPS,
         graze: bool = False, extras: bool = False, stereo=None, annot=None) -> OracleResult:
    """Run the oracle.

    ``scene``: an object with numpy fields ``verts, vert_off, faces, face_off,
    env_off, inst_asset, inst_label, inst_T`` (see scenegen.Scene).
    ``rays``: dict with ``model`` and the fields of oracle_rays.
    ``query``: int64 flat ray ids (default: every ray).
    ``stereo``: (offset xyz in the sensor frame, eps) -> also the shadow mask.
    ``annot``: per-asset list of float [V][K] vertex annotations (None for an
    asset without any) -> also the interpolated annotation of each hit.
    """
    lib = _load()
    sc, r, keep, total = _marshal(scene, rays, annot)
    if query is None:
        query = np.arange(total, dtype=np.int64)
    q = np.ascontiguousarray(query, dtype=np.int64)
    n = len(q)
    out = OracleResult(np.empty(n, np.float64), np.empty(n, np.float32),
                       np.empty(n, np.int32), np.empty(n, np.int32),
                       np.empty(n, np.int32), np.empty(n, np.float64),
                       np.full(n, np.inf), 0)
    if stereo is not None:
        (r.stereo[0], r.stereo[1], r.stereo[2]), r.stereo_eps = stereo[0], stereo[1]
        out.valid = np.empty(n, np.int32)
    if extras:
        out.normal = np.empty((n, 3), np.float64)
        out.bary = np.empty((n, 2), np.float64)
        out.point = np.empty((n, 3), np.float64)
    if annot is not None:
        out.annot = np.empty((n, sc.annot_k), np.float64)
    rc = lib.oracle_cast(ctypes.byref(sc), ctypes.byref(r), _ptr(q), n, amb_eps, n_threads,
                         _ptr(out.t64), _ptr(out.dist), _ptr(out.seg), _ptr(out.face),
                         _ptr(out.amb), _ptr(out.t2), _ptr(out.graze) if graze else None,
                         _ptr(out.normal), _ptr(out.bary), _ptr(out.point), _ptr(out.valid),
                         _ptr(out.annot))
    if rc != 0:
        raise ValueError("oracle_cast rejected its input")
    out.tests = int(lib.oracle_last_tests())
    return out


def certify(scene, rays: dict, face, query=None, n_threads: int = 0):
    """Certificate of reported faces (oracle.h oracle_certify): returns
    ``(t_face, outside, label)`` -- the FP64 plane-hit t of each reported face,
    how far that hit lies outside the face (<= 0 inside) and its label."""
    lib = _load()
    sc, r, keep, total = _marshal(scene, rays)
    if query is None:
        query = np.arange(total, dtype=np.int64)
    q = np.ascontiguousarray(query, dtype=np.int64)
    f = np.ascontiguousarray(face, dtype=np.int32).reshape(-1)
    if len(f) != len(q):
        raise ValueError("one face per queried ray")
    n = len(q)
    t_face, outside, label = np.empty(n, np.float64), np.empty(n, np.float64), np.empty(n, np.int32)
    rc = lib.oracle_certify(ctypes.byref(sc), ctypes.byref(r), _ptr(q), n, _ptr(f), n_threads,
                            _ptr(t_face), _ptr(outside), _ptr(label))
    if rc != 0:
        raise ValueError("oracle_certify rejected its input")
    return t_face, outside, label


def _marshal(scene, rays, annot=None):
    keep = []

    def arr(x, dt):
        a = np.ascontiguousarray(x, dtype=dt)
        keep.append(a)
        return a

    verts = arr(scene.verts, np.float32)
    sc = _Scene(len(scene.vert_off) - 1,
                _ptr(verts), _ptr(arr(scene.vert_off, np.int64)),
                _ptr(arr(scene.faces, np.int32)), _ptr(arr(scene.face_off, np.int64)),
                len(scene.env_off) - 1, _ptr(arr(scene.env_off, np.int64)),
                _ptr(arr(scene.inst_asset, np.int32)), _ptr(arr(scene.inst_label, np.int32)),
                _ptr(arr(scene.inst_T, np.float32)), None, 0)
    if annot is not None:
        K = max(np.asarray(a).reshape(len(m.verts), -1).shape[1]
                for a, m in zip(annot, scene.meshes) if a is not None)
        rows = [np.full((len(m.verts), K), np.nan, np.float32) if a is None
                else np.asarray(a, np.float32).reshape(len(m.verts), K) for a, m in zip(annot, scene.meshes)]
        A = arr(np.concatenate(rows), np.float32)
        sc.annot, sc.annot_k = _ptr(A), K
    m = rays["model"]
    r = _Rays()
    r.model = m
    r.max_range = float(rays["max_range"])
    n_envs = len(scene.env_off) - 1
    if m == RAYS:
        o = arr(rays["orig"], np.float32)
        d = arr(rays["dir"], np.float32)
        r.orig, r.dir, r.R = _ptr(o), _ptr(d), o.shape[1]
        total = n_envs * r.R
    else:
        poses = arr(rays["poses"], np.float32)
        r.poses, r.S = _ptr(poses), poses.shape[1]
        if m == PINHOLE:
            r.W, r.H = int(rays["W"]), int(rays["H"])
            r.fx, r.fy, r.cx, r.cy = (float(rays[k]) for k in ("fx", "fy", "cx", "cy"))
            r.kind = int(rays["kind"])
            total = n_envs * r.S * r.H * r.W
        else:
            b = arr(rays["beams"], np.float32)
            r.beams, r.C, r.K = _ptr(b), b.shape[0], b.shape[1]
            total = n_envs * r.S * r.C * r.K
    return sc, r, keep, total
