"""e2e epoch driver vs steps per chunk graph (PGB_CHUNK_STEPS), MNIST B=256."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2010_09063_b200 as P  # noqa: E402

B, N = 256, 256 * 234
desc = P.build_desc(P.ModelKind.mnist_cnn)
model = P.build(P.ModelKind.mnist_cnn, 0)
data = P.synth_for_model(desc, N, 0, pinned=True)
eng = P.GradEngine(model, P.Strategy.groupconv, B)
cfg = P.DpConfig(1.0, 1.1, 0.1, 1, 0)
norms = np.empty(N, np.float32)
for cs in (1, 4, 8, 16, 21):
    os.environ["PGB_CHUNK_STEPS"] = str(cs)
    P.run_epoch(eng, model, data, cfg, 0, norms)
    t0 = time.perf_counter()
    P.run_epoch(eng, model, data, cfg, 0, norms)
    dt = time.perf_counter() - t0
    print(f"chunk {cs:>3} steps: {dt / 234 * 1e6:7.1f} us/step, {N / dt / 1e6:.2f} M ex/s", flush=True)
# raw copy of the same dataset in 12.9 MB pieces on a side stream
x = torch.from_numpy(data.inputs.reshape(-1))
d = torch.empty(16 * B * 784, device="cuda")
s = torch.cuda.Stream()
for piece in (B * 784, 16 * B * 784):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with torch.cuda.stream(s):
        for o in range(0, x.numel() - piece + 1, piece):
            d[:piece].copy_(x[o:o + piece], non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"raw H2D of the dataset in {piece * 4} B pieces: {x.numel() * 4 / dt / 1e9:.1f} GB/s", flush=True)
