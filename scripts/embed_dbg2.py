import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2010_09063_b200 as P
B, L, V, E = 512, 256, 10004, 100
desc = P.build_desc(P.ModelKind.embed, P.ModelOptions(seq_len=L, vocab=V, hidden=E))
data = P.synth_for_model(desc, 3 * B, 5)
cfg = P.DpConfig(clip_norm=0.05, noise_multiplier=1.1, learning_rate=0.5, seed=3)
mv = P.build_from_desc(desc, 0); ev = P.GradEngine(mv, P.Strategy.jacmm, B)
os.environ["PGB_EMB_AGG_SCALAR"] = "1"
ms = P.build_from_desc(desc, 0); es = P.GradEngine(ms, P.Strategy.jacmm, B)
os.environ.pop("PGB_EMB_AGG_SCALAR")
print("info", ev.info(), es.info())
for s in range(3):
    sl = slice(s * B, (s + 1) * B)
    rv = P.dpsgd_step(mv, ev, data.inputs[sl], data.labels[sl], cfg, 7 + s)
    rs = P.dpsgd_step(ms, es, data.inputs[sl], data.labels[sl], cfg, 7 + s)
    d = np.abs(mv.flat_params() - ms.flat_params())[: V * E].reshape(V, E)
    print(s, "norms eq", np.array_equal(rv.pre_clip_norms, rs.pre_clip_norms), "maxdiff", d.max(),
          "nrows", np.count_nonzero(d.max(1)), "cols", np.nonzero(d.max(0))[0][:10])
