import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2010_09063_b200 as P
sys.path.insert(0, "tests")
from test_golden_full_gpu import _load, _sampled_blocks
f = _load("cifar_cnn_b256")
B, C, every = int(f["B"]), float(f["clip"]), int(f["every"])
desc = P.build_desc(P.ModelKind.cifar_cnn)
data = P.synth_for_model(desc, B, 0)
model = P.build_from_desc(desc, 0)
eng = P.GradEngine(model, P.Strategy(4), B)
got, norms, nclip = eng.clipped_sum(data.inputs, data.labels, C)
gs = got[::every].astype(np.float64); want = f["clipped_sum"]
bars = np.maximum(1e-5, 3.0 * f["ref_f32_block_rel"])
tag = os.environ.get("TAG", "")
for k, ((lo, hi), bar) in enumerate(zip(_sampled_blocks(f), bars)):
    if hi <= lo: continue
    w, g = want[lo:hi], gs[lo:hi]
    nw = np.linalg.norm(g - w) / np.linalg.norm(w)
    el = np.max(np.abs(g - w) / (np.abs(w) + np.abs(w).max()))
    print(tag, k, f"bar {bar:.1e} normwise {nw:.1e} elem {el:.1e}", "FAIL" if (nw > bar or el > bar) else "")
