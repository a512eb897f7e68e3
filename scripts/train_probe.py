"""Step-by-step fcnn DP training: ours vs the compiled reference (f32), same
batches (bench::train's shuffle), parameter distance after each step."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
import paper_2010_09063_b200 as P  # noqa: E402
from paper_2010_09063_b200.harness import _shuffle  # noqa: E402

kind, strat, n, batch = 1, 1, 256, 32
desc = P.build_desc(P.ModelKind(kind))
od = O.build_desc(kind)
model = P.build_from_desc(desc, 0)
p0 = model.flat_params()
data = P.synth_for_model(desc, n, 3)
cfg = P.DpConfig(clip_norm=1.0, noise_multiplier=1.1, learning_rate=0.1, seed=5)
eng = P.GradEngine(model, P.Strategy(strat), batch)
R = O.RefModel(od, strat, batch, p0, np.float32)
steps = n // batch
order = np.arange(n, dtype=np.int64)
for epoch in range(2):
    _shuffle(order, 5, epoch)
    for s in range(steps):
        idx = order[s * batch:(s + 1) * batch]
        x, y = data.inputs[idx], data.labels[idx]
        rep = P.dpsgd_step(model, eng, x, y, cfg, epoch * steps + s)
        rn, rc = R.step(x, y, 1.0, 1.1, 0.1, 1, 5, epoch * steps + s)
        got, want = model.flat_params().astype(np.float64), R.params().astype(np.float64)
        nd = np.max(np.abs(rep.pre_clip_norms - rn) / rn)
        print(epoch, s, "param rel", np.linalg.norm(got - want) / np.linalg.norm(want),
              "norm rel", nd, "clipped", rep.clipped_count, rc,
              "min |n-C|", np.min(np.abs(rn - 1.0)))
