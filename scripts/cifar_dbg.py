import sys, os, numpy as np
sys.path.insert(0, os.getcwd())
import paper_2010_09063_b200 as P
B = int(sys.argv[1]) if len(sys.argv) > 1 else 4
desc = P.build_desc(P.ModelKind.cifar_cnn)
model = P.build_from_desc(desc, 0)
data = P.synth_for_model(desc, B, 0)
eng = P.GradEngine(model, P.Strategy.groupconv, B, P.ExecMode.eager)
s, n = eng.per_example_flat(data.inputs, data.labels)
print("ok", n[:4])
