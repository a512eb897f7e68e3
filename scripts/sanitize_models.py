"""One small DPSGD step per model through the engine (for compute-sanitizer runs)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2010_09063_b200 as P  # noqa: E402

for kind, opts, strat, B in ((P.ModelKind.mnist_cnn, None, P.Strategy.groupconv, 8),
                             (P.ModelKind.cifar_cnn, None, P.Strategy.groupconv, 4),
                             (P.ModelKind.fcnn, None, P.Strategy.norms, 16),
                             (P.ModelKind.logreg, None, P.Strategy.outer, 16),
                             (P.ModelKind.embed, P.ModelOptions(seq_len=64, vocab=500, hidden=16),
                              P.Strategy.jacmm, 8)):
    desc = P.build_desc(kind, opts) if opts else P.build_desc(kind)
    model = P.build_from_desc(desc, 0)
    data = P.synth_for_model(desc, 4 * B, 0)
    eng = P.GradEngine(model, strat, B)
    cfg = P.DpConfig(1.0, 1.1, 0.1, 1, 0)
    for s in range(2):
        rep = P.dpsgd_step(model, eng, data.inputs[s * B:(s + 1) * B], data.labels[s * B:(s + 1) * B],
                           cfg, s)
    P.run_epoch(eng, model, data, cfg, 10)  # multi-step graphs (cross-step PDL for MNIST)
    eng.weighted_grad_sum(data.inputs[:B], data.labels[:B], np.full(B, 0.5, np.float32))
    print(kind.name, "ok", rep.clipped_count, flush=True)
