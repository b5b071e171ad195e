"""BVH4 level widths of a c6 terrain BLAS (the top-down build's grid barriers)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2503_01471_b200 as agr, scenegen as sg
sc, sen = sg.config6(n_envs=2, ring=1)
s = agr.Scene.from_scenegen(sc, trbvh_rounds=0, parts=False, node_width=4)
nodes, root = s.debug_export_bvh4(0)
refs = nodes[:, 24:28].view(np.int32)
lvl, widths = [root], []
while lvl:
    widths.append(len(lvl))
    lvl = [int(r) for n in lvl for r in refs[n - root] if r >= 0]
print("nodes", len(nodes), "levels", len(widths), widths, "blas depth", s.info()["blas_max_depth"])
