"""Export the binary BLAS (after LBVH + treelet rounds) of c3's assets to
gpurun_out/blas_c3.npz for offline collapse-quality analysis."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2503_01471_b200 as agr, scenegen as sg
sc, _ = sg.config3(n_envs=2)
s = agr.Scene.from_scenegen(sc, parts=False)
out = {}
for a, m in enumerate(sc.meshes):
    nodes, leaf_face, _ = s.debug_export_blas(a)
    tri = m.verts[m.faces]
    out[f"nodes{a}"] = nodes
    out[f"leafbox{a}"] = np.concatenate([tri[leaf_face].min(1), tri[leaf_face].max(1)], 1)
np.savez(os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "gpurun_out", "blas_c3.npz"), **out)
print("assets", len(sc.meshes))
