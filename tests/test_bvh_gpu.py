"""Structural checks of the GPU LBVH (BLAS) against brute force on small
inputs (SURVEY.md §4 unit layer; §8(c) 'BVH pieces'): Morton codes of known
points, sorted order, every non-degenerate face in exactly one leaf,
boxes containing their children, Karras topology == recursive split."""
from __future__ import annotations

import numpy as np
import pytest

import scenegen as sg
import torch

from gpu_util import dev, make_scene

pytestmark = pytest.mark.gpu


def _expand(v):
    out = 0
    for b in range(10):
        out |= ((v >> b) & 1) << (3 * b)
    return out


def morton_ref(p):
    """Independent bit-loop Morton code of a point in [0, 1]^3 (x in bit 2)."""
    q = [min(int(np.floor(c * 1024.0)), 1023) for c in p]
    q = [max(0, c) for c in q]
    return (_expand(q[0]) << 2) | (_expand(q[1]) << 1) | _expand(q[2])


def test_morton_ref_known_values():
    assert morton_ref((0.9999, 0.9999, 0.9999)) == 0x3FFFFFFF
    assert morton_ref((1 / 1024, 0, 0)) == 4  # lowest x bit lands in bit 2


def _check_blas(mesh):
    """Plain LBVH (no treelet restructuring): the Karras topology is checked."""
    sc = sg.assemble([mesh], [[(0, 0, sg.make_T(np.eye(3), (0, 0, 0)))]])
    s = make_scene(sc, build=False, trbvh_rounds=0, parts=False)
    nodes, leaf_face, codes = s.debug_export_blas(0)
    v = mesh.verts
    tri = v[mesh.faces]
    area2 = np.linalg.norm(np.cross((tri[:, 1] - tri[:, 0]).astype(np.float64),
                                    (tri[:, 2] - tri[:, 0]).astype(np.float64)), axis=1)
    valid = np.nonzero(area2 > 0)[0]
    # every non-degenerate face in exactly one leaf
    assert sorted(leaf_face.tolist()) == sorted(valid.tolist())
    n = len(leaf_face)
    # codes sorted, and equal to the Morton code of the centroid in the
    # centroid bounds (computed independently here)
    lo_t, hi_t = tri.min(1), tri.max(1)
    cent = 0.5 * lo_t + 0.5 * hi_t
    cv = cent[valid]
    clo, chi = cv.min(0), cv.max(0)
    ext = chi - clo
    for i, f in enumerate(leaf_face):
        u = [(cent[f][k] - clo[k]) / ext[k] if ext[k] > 0 else 0.0 for k in range(3)]
        assert codes[i] == morton_ref(np.asarray(u, np.float32)), i
    assert np.all(np.diff(codes.astype(np.int64)) >= 0)
    # equal codes keep ascending face order (stable sort)
    for i in range(n - 1):
        if codes[i] == codes[i + 1]:
            assert leaf_face[i] < leaf_face[i + 1]
    if n < 2:
        return nodes, leaf_face
    # boxes: child boxes contain their subtree's triangles exactly
    refs = nodes[:, 12:14].view(np.int32)

    def box_of(ref):
        if ref < 0:
            f = leaf_face[~ref]
            return lo_t[f], hi_t[f], [f]
        b0lo, b0hi, f0 = box_of(refs[ref, 0])
        b1lo, b1hi, f1 = box_of(refs[ref, 1])
        nd = nodes[ref]
        c0lo, c0hi = nd[[0, 2, 4]], nd[[1, 3, 5]]
        c1lo, c1hi = nd[[6, 8, 10]], nd[[7, 9, 11]]
        assert np.array_equal(c0lo, b0lo) and np.array_equal(c0hi, b0hi)
        assert np.array_equal(c1lo, b1lo) and np.array_equal(c1hi, b1hi)
        return np.minimum(b0lo, b1lo), np.maximum(b0hi, b1hi), f0 + f1

    lo, hi, fs = box_of(0)
    assert sorted(fs) == sorted(valid.tolist())
    assert np.array_equal(lo, lo_t[valid].min(0)) and np.array_equal(hi, hi_t[valid].max(0))

    # Karras topology == recursive split of the sorted keys (brute force)
    keys = [(int(c) << 32) | i for i, c in enumerate(codes)]

    def split(first, last):
        a, b = keys[first], keys[last]
        common = 64 - (a ^ b).bit_length()
        s = first
        for k in range(first, last):
            if 64 - (a ^ keys[k + 1]).bit_length() > common:
                s = k + 1
            else:
                break
        return s

    def rec(first, last):
        """returns set of (lo, hi) leaf ranges of internal nodes"""
        if first == last:
            return []
        sp = split(first, last)
        return [(first, last)] + rec(first, sp) + rec(sp + 1, last)

    def ranges(ref):
        if ref < 0:
            return (~ref, ~ref), []
        (a0, b0), r0 = ranges(refs[ref, 0])
        (a1, b1), r1 = ranges(refs[ref, 1])
        assert b0 + 1 == a1
        return (a0, b1), [(a0, b1)] + r0 + r1

    (a, b), got = ranges(0)
    assert (a, b) == (0, n - 1)
    assert sorted(got) == sorted(rec(0, n - 1))
    return nodes, leaf_face


@pytest.mark.parametrize("mesh_fn", [
    lambda: sg.cube_mesh(),
    lambda: sg.closed_cylinder_92(),
    lambda: sg.sphere_mesh(1.0, 2),
    lambda: sg.tree_mesh(np.random.default_rng(1)),
    lambda: sg.ground_mesh(),
])
def test_blas_structure(mesh_fn):
    _check_blas(mesh_fn())


def test_blas_duplicate_codes_and_degenerates():
    """Many identical centroids (duplicate Morton codes) + zero-area faces."""
    rng = np.random.default_rng(0)
    base = rng.uniform(-1, 1, (3, 3)).astype(np.float32)
    tris = np.concatenate([np.tile(base, (40, 1, 1)), rng.uniform(-1, 1, (30, 3, 3)).astype(np.float32)])
    tris[5, 2] = tris[5, 1]  # degenerate (repeated vertex)
    tris[50, 1] = tris[50, 0]
    v = tris.reshape(-1, 3)
    f = np.arange(len(v), dtype=np.int32).reshape(-1, 3)
    _check_blas(sg.Mesh("dup", v, f))


def test_blas_single_triangle_and_flat_axis():
    v = np.asarray([[0, 0, 0], [1, 0, 0], [0, 1, 0]], np.float32)
    nodes, lf = _check_blas(sg.Mesh("one", v, np.asarray([[0, 1, 2]], np.int32)))
    assert list(lf) == [0]


def test_large_mesh_multiblock_sort():
    """A mesh big enough for a multi-block radix sort (> 1024 keys per tile)."""
    m = sg.sphere_mesh(2.0, 5)  # 20480 faces
    sc = sg.assemble([m], [[(0, 0, sg.make_T(np.eye(3), (0, 0, 0)))]])
    s = make_scene(sc, build=False, parts=False)
    nodes, leaf_face, codes = s.debug_export_blas(0)
    assert sorted(leaf_face.tolist()) == list(range(len(m.faces)))
    assert np.all(np.diff(codes.astype(np.int64)) >= 0)
    for i in np.nonzero(np.diff(codes.astype(np.int64)) == 0)[0]:
        assert leaf_face[i] < leaf_face[i + 1]


LEAF_SHIFT = 29  # agr_internal.cuh: BLAS leaf ref x = first | (count - 1) << 29


def _walk_bvh4(nodes, root, leaf_boxes=None, blas=True):
    """Collect leaves reachable from BVH4 node 0; check every child box
    contains the boxes of its subtree (exactly: the union)."""
    refs = nodes[:, 24:28].view(np.int32)
    leaves = []

    def box(n, k):
        lo = np.asarray([nodes[n, 0 + k], nodes[n, 8 + k], nodes[n, 16 + k]])
        hi = np.asarray([nodes[n, 4 + k], nodes[n, 12 + k], nodes[n, 20 + k]])
        return lo, hi

    def rec(n):
        lo_all, hi_all = np.full(3, np.inf), np.full(3, -np.inf)
        for k in range(4):
            r = refs[n, k]
            if r == np.iinfo(np.int32).min:
                lo, hi = box(n, k)
                assert np.all(np.isinf(lo)) and np.all(np.isinf(hi))
                continue
            lo, hi = box(n, k)
            if r < 0:
                x = ~r
                # BLAS multi-triangle leaf: consecutive records, box = their union
                first, count = (x & ((1 << LEAF_SHIFT) - 1), (x >> LEAF_SHIFT) + 1) if blas else (x, 1)
                group = list(range(first, first + count))
                leaves.extend(group)
                if leaf_boxes is not None:
                    bl = [leaf_boxes(l) for l in group]
                    blo = np.min([b[0] for b in bl], 0)
                    bhi = np.max([b[1] for b in bl], 0)
                    assert np.array_equal(lo, blo) and np.array_equal(hi, bhi)
            else:
                clo, chi = rec(r - root)
                assert np.array_equal(lo, clo) and np.array_equal(hi, chi)
            lo_all, hi_all = np.minimum(lo_all, lo), np.maximum(hi_all, hi)
        return lo_all, hi_all

    rec(0)
    return leaves


@pytest.mark.parametrize("mesh_fn", [lambda: sg.cube_mesh(), lambda: sg.tree_mesh(np.random.default_rng(2)),
                                     lambda: sg.sphere_mesh(1.0, 4)])
def test_bvh4_blas_covers_every_leaf_once(mesh_fn):
    mesh = mesh_fn()
    sc = sg.assemble([mesh], [[(0, 0, sg.make_T(np.eye(3), (0, 0, 0)))]])
    s = make_scene(sc, build=False, parts=False)
    _, leaf_face, _ = s.debug_export_blas(0)
    nodes, root = s.debug_export_bvh4(0)
    tri = mesh.verts[mesh.faces]
    lo_t, hi_t = tri.min(1), tri.max(1)
    leaves = _walk_bvh4(nodes, root, lambda l: (lo_t[leaf_face[l]], hi_t[leaf_face[l]]))
    assert sorted(leaves) == list(range(len(leaf_face)))
    # greedy collapse: nodes have up to 4 children, most internal nodes 4
    cnt = nodes[:, 28].view(np.int32)
    assert cnt.max() <= 4


@pytest.mark.parametrize("trbvh_rounds", [0, 3])
def test_bvh4_blas_is_compact_and_reachable(trbvh_rounds):
    """The BLAS BVH4 is compacted at every build (blas.cu K5b'): the export
    holds exactly the nodes reachable from the root, each reached once, the
    root first, internal refs in range; far fewer nodes than binary nodes;
    the same after a batched mesh update (the c6 path)."""
    meshes = [sg.terrain_mesh(np.random.default_rng(3), n=32), sg.sphere_mesh(1.0, 3), sg.cube_mesh()]
    sc = sg.assemble(meshes, [[(a, a + 1, sg.make_T(np.eye(3), (0, 0, 0)))] for a in range(3)])
    s = make_scene(sc, build=False, trbvh_rounds=trbvh_rounds, parts=False)
    for step in range(2):
        if step == 1:
            v = np.concatenate([m.verts * 1.1 + 0.05 for m in meshes]).astype(np.float32)
            s.update_meshes([0, 1, 2], torch.from_numpy(v).to(dev()))
            torch.cuda.synchronize()
        for a, m in enumerate(meshes):
            nodes, root = s.debug_export_bvh4(a)
            refs = nodes[:, 24:28].view(np.int32)
            seen = np.zeros(len(nodes), np.int32)
            stack = [root]
            while stack:
                n = stack.pop()
                assert root <= n < root + len(nodes)
                seen[n - root] += 1
                stack.extend(int(r) for r in refs[n - root] if r >= 0)
            assert np.all(seen == 1), (a, step)
            if len(m.faces) > 100:
                assert len(nodes) < 0.6 * (len(m.faces) - 1), (a, len(nodes))
            tri = (m.verts * (1.1 if step else 1.0) + (0.05 if step else 0.0)).astype(np.float32)[m.faces]
            if step == 0:
                lb = sum(len(mm.faces) for mm in meshes[:a])  # the asset's first leaf record
                leaves = _walk_bvh4(nodes, root, lambda l, t=tri, lf=s.debug_export_blas(a)[1]:
                                    (t[lf[l - lb]].min(0), t[lf[l - lb]].max(0)))
                assert sorted(leaves) == list(range(lb, lb + len(m.faces)))


def test_bvh4_tlas_covers_every_instance_once():
    sc, _ = sg.config2(n_envs=5)
    s = make_scene(sc)
    for e in range(5):
        nodes, root = s.debug_export_bvh4(-1 - e)
        leaves = _walk_bvh4(nodes, root, blas=False)
        assert sorted(leaves) == list(range(int(sc.env_off[e]), int(sc.env_off[e + 1])))


def _sah_cost(nodes, refs, leaf_face, lo_t, hi_t, ci=1.2, ct=1.0):
    def area(lo, hi):
        d = hi - lo
        return d[0] * d[1] + d[1] * d[2] + d[2] * d[0]

    def rec(ref):
        if ref < 0:
            f = leaf_face[~ref]
            return ct * area(lo_t[f], hi_t[f]), lo_t[f], hi_t[f]
        c0, l0, h0 = rec(refs[ref, 0])
        c1, l1, h1 = rec(refs[ref, 1])
        lo, hi = np.minimum(l0, l1), np.maximum(h0, h1)
        return ci * area(lo, hi) + c0 + c1, lo, hi

    c, lo, hi = rec(0)
    return c / area(lo, hi)


@pytest.mark.parametrize("mesh_fn", [lambda: sg.tree_mesh(np.random.default_rng(1)),
                                     lambda: sg.rock_mesh(np.random.default_rng(2)),
                                     lambda: sg.sphere_mesh(1.0, 3)])
def test_trbvh_keeps_leaves_and_boxes_and_lowers_sah(mesh_fn):
    """Treelet restructuring (f3 BLAS quality): every face still in exactly one
    leaf, every child box the exact union of its subtree, BVH4 consistent, and
    the SAH cost of the binary tree lower than the plain LBVH's."""
    mesh = mesh_fn()
    tri = mesh.verts[mesh.faces]
    lo_t, hi_t = tri.min(1).astype(np.float64), tri.max(1).astype(np.float64)
    costs = {}
    for rounds in (0, 3):
        sc = sg.assemble([mesh], [[(0, 0, sg.make_T(np.eye(3), (0, 0, 0)))]])
        s = make_scene(sc, build=False, trbvh_rounds=rounds, parts=False)
        nodes, leaf_face, _ = s.debug_export_blas(0)
        refs = nodes[:, 12:14].view(np.int32)
        seen = []

        def walk(ref):
            if ref < 0:
                seen.append(leaf_face[~ref])
                f = leaf_face[~ref]
                return lo_t[f], hi_t[f]
            l0, h0 = walk(refs[ref, 0])
            l1, h1 = walk(refs[ref, 1])
            nd = nodes[ref]
            assert np.array_equal(nd[[0, 2, 4]], l0) and np.array_equal(nd[[1, 3, 5]], h0)
            assert np.array_equal(nd[[6, 8, 10]], l1) and np.array_equal(nd[[7, 9, 11]], h1)
            return np.minimum(l0, l1), np.maximum(h0, h1)

        walk(0)
        assert sorted(seen) == list(range(len(mesh.faces)))
        b4, root = s.debug_export_bvh4(0)
        assert sorted(_walk_bvh4(b4, root)) == list(range(len(mesh.faces)))
        costs[rounds] = _sah_cost(nodes, refs, leaf_face, lo_t, hi_t)
    assert costs[3] < costs[0] * 0.97, costs
