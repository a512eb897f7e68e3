import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2010_09063_b200 as P
B, L, V, E = [int(v) for v in sys.argv[1:5]] if len(sys.argv) > 4 else (40, 17, 97, 8)
desc = P.build_desc(P.ModelKind.embed, P.ModelOptions(seq_len=L, vocab=V, hidden=E))
data = P.synth_for_model(desc, B, 5)
for sigma in (0.0, 1.1):
    res = []
    for scalar in (0, 1):
        if scalar: os.environ["PGB_EMB_AGG_SCALAR"] = "1"
        m = P.build_from_desc(desc, 0)
        e = P.GradEngine(m, P.Strategy.jacmm, B)
        os.environ.pop("PGB_EMB_AGG_SCALAR", None)
        p0 = m.flat_params().copy()
        cfg = P.DpConfig(clip_norm=0.05, noise_multiplier=sigma, learning_rate=0.5, seed=3)
        P.dpsgd_step(m, e, data.inputs, data.labels, cfg, 7)
        res.append(m.flat_params() - p0)
    d = np.abs(res[0] - res[1])[: V * E].reshape(V, E)
    print("sigma", sigma, "maxdiff", d.max(), "rows differing", np.nonzero(d.max(1))[0][:20], "cols", np.nonzero(d.max(0))[0])
    print(res[0][:8]); print(res[1][:8])
