import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2010_09063_b200 as P
import oracle as O
O.port()
desc = P.build_desc(P.ModelKind.cifar_cnn)
od = O.build_desc(O.CIFAR_CNN)
for B in (4, 8):
    data = P.synth_for_model(desc, B, 0)
    p64 = O.init_params(od, 0)
    x64, y64 = O.synth(od, B, 0)
    _, wn, wclip, want = O.dpsgd_step(od, x64, y64, p64, 1.0, 0.0, 0.1, 1, 0, 0)
    for flag in (0, 1):
        if flag: os.environ["PGB_NO_KSPLIT"] = "1"
        model = P.build_from_desc(desc, 0)
        e = P.GradEngine(model, P.Strategy.groupconv, B)
        got = e.clipped_sum(data.inputs, data.labels, 1.0)[0]
        os.environ.pop("PGB_NO_KSPLIT", None)
        off = 0; out = []
        for k, n in enumerate(od.blocks):
            a, b = got[off:off+n].astype(np.float64), want[off:off+n]
            out.append(f"{k}:{np.linalg.norm(a-b)/max(np.linalg.norm(b),1e-30):.1e}")
            off += n
        print(B, os.environ.get("PGB_KSPLIT_CHAIN"), "nosplit" if flag else "split", " ".join(out))
