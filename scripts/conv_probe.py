"""Per-geometry probe of the TMA conv GEMMs: a one-conv model (conv C->D 3x3
p1 on HxW, relu, global avgpool, D=10 classes head-free) per case, eager,
PGB_DEBUG_LAUNCH=1; per-example grads vs the oracle."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
import paper_2010_09063_b200 as P  # noqa: E402

O.port()
cases = [(3, 32, 32, 10), (32, 32, 32, 10), (32, 16, 16, 10), (64, 16, 8, 10), (64, 8, 8, 10),
         (128, 8, 8, 10), (128, 4, 4, 10), (256, 4, 4, 10)]
if len(sys.argv) > 1:
    cases = [cases[int(i)] for i in sys.argv[1:]]
for C, H, W, D in cases:
    layers = [P.LayerSpec(P.LayerKind.conv, C, D, 3, 1, 1), P.LayerSpec(P.LayerKind.relu),
              P.LayerSpec(P.LayerKind.global_avgpool)]
    desc = P.custom_desc(P.ModelKind.cifar_cnn, layers, (C, H, W), D)
    od = O.custom_desc(O.CIFAR_CNN, [(1, C, D, 3, 1, 1), (6, 0, 0, 0, 1, 0), (4, 0, 0, 0, 1, 0)],
                       (C, H, W), D)
    B = 4
    model = P.build_from_desc(desc, 0)
    data = P.synth_for_model(desc, B, 0)
    try:
        eng = P.GradEngine(model, P.Strategy.groupconv, B, P.ExecMode.eager)
        st, nr = eng.per_example_flat(data.inputs, data.labels)
    except Exception as e:
        print(C, H, W, D, "FAIL", str(e)[:120])
        continue
    ws, wnsq, _ = O.per_example_grads(od, data.inputs.astype(np.float64),
                                      data.labels.astype(np.float64), O.init_params(od, 0))
    n0 = od.blocks[0] * B
    err = np.linalg.norm(st[:n0] - ws[:n0]) / np.linalg.norm(ws[:n0])
    print(C, H, W, D, "dW rel", err, "norm rel", np.max(np.abs(nr - np.sqrt(wnsq)) / np.sqrt(wnsq)))
