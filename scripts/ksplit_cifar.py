import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2010_09063_b200 as P
import oracle as O
O.port()
desc = P.build_desc(P.ModelKind.cifar_cnn)
od = O.build_desc(O.CIFAR_CNN)
for B in [int(b) for b in os.environ.get("KS_B", "4,8").split(",")]:
    data = P.synth_for_model(desc, B, 0)
    ws, wnsq, _ = O.per_example_grads(od, data.inputs.astype(np.float64), data.labels.astype(np.float64), O.init_params(od, 0))
    for flag in (0, 1):
        if flag: os.environ["PGB_NO_KSPLIT"] = "1"
        model = P.build_from_desc(desc, 0)
        eng = P.GradEngine(model, P.Strategy.groupconv, B)
        st, nr = eng.per_example_flat(data.inputs, data.labels)
        os.environ.pop("PGB_NO_KSPLIT", None)
        off = 0; out = []
        for n in od.blocks:
            g, w = st[off:off + B * n].reshape(B, n), ws[off:off + B * n].reshape(B, n)
            e = np.linalg.norm(g - w, axis=1) / np.linalg.norm(w, axis=1)
            out.append(f"{e.max():.1e}@{e.argmax()}")
            off += B * n
        print(B, "nosplit" if flag else "split", " ".join(out[:8]))
