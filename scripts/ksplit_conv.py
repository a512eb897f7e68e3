import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2010_09063_b200 as P
import oracle as O
O.port()
for (C, H, W, D) in [(32, 16, 16, 64), (32, 32, 32, 32)]:
  for B in (4, 8, 16):
    for flag in (0, 1):
        if flag: os.environ["PGB_NO_KSPLIT"] = "1"
        layers = [P.LayerSpec(P.LayerKind.conv, C, D, 3, 1, 1), P.LayerSpec(P.LayerKind.relu),
                  P.LayerSpec(P.LayerKind.conv, D, D, 3, 1, 1), P.LayerSpec(P.LayerKind.relu),
                  P.LayerSpec(P.LayerKind.conv, D, 10, 3, 1, 1), P.LayerSpec(P.LayerKind.relu),
                  P.LayerSpec(P.LayerKind.global_avgpool)]
        desc = P.custom_desc(P.ModelKind.cifar_cnn, layers, (C, H, W), 10)
        od = O.custom_desc(O.CIFAR_CNN, [(1, C, D, 3, 1, 1), (6, 0, 0, 0, 1, 0), (1, D, D, 3, 1, 1), (6, 0, 0, 0, 1, 0), (1, D, 10, 3, 1, 1),
                                         (6, 0, 0, 0, 1, 0), (4, 0, 0, 0, 1, 0)], (C, H, W), 10)
        model = P.build_from_desc(desc, 0)
        data = P.synth_for_model(desc, B, 0)
        eng = P.GradEngine(model, P.Strategy.groupconv, B)
        st, nr = eng.per_example_flat(data.inputs, data.labels)
        ws, wnsq, _ = O.per_example_grads(od, data.inputs.astype(np.float64), data.labels.astype(np.float64), O.init_params(od, 0))
        os.environ.pop("PGB_NO_KSPLIT", None)
        off = 0; out = []
        for n in od.blocks:
            g, w = st[off:off + B * n], ws[off:off + B * n]
            out.append(f"{np.linalg.norm(g - w) / np.linalg.norm(w):.1e}")
            off += B * n
        print((C, H, W, D), B, "nosplit" if flag else "split", " ".join(out))
