"""The bench's C2 step alone (diagnostics): K forwards over a >L2 ring of
layers and buffers, captured as one CUDA graph, median of replays.
usage: python tools/step_bench.py [K] [reps]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_02540_b200 as dtq  # noqa: E402
from bench import HBLOCK, K, M, N, make_inputs  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
dev = torch.device("cuda:0")
x_np, w_np, smooth_np = make_inputs()
x, w = torch.from_numpy(x_np).to(dev), torch.from_numpy(w_np).to(dev)
bal = dtq.Balance(torch.from_numpy(smooth_np).to(dev),
                  torch.from_numpy(dtq.hadamard_signs(K, 7)).to(dev), HBLOCK)
ring = max(2, int(300e6 // (M * K * 2 + N * K + M * N * 2)) + 1)
layers = [dtq.QuantLinear.create(w, 8, 8, balance=bal) for _ in range(ring)]
xs = [x.clone() for _ in range(ring)]
ys = [torch.empty((M, N), dtype=torch.float16, device=dev) for _ in range(ring)]
ws = layers[0].workspace(M, dev)


def run():
    for i in range(steps):
        layers[i % ring].forward(xs[i % ring], out=ys[i % ring], workspace=ws)


run()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    run()
ts = []
for _ in range(reps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b) * 1e3 / steps)
print(f"{os.environ.get('DTQ_B200_LIB', 'product')}: step median {np.median(ts):.2f} us "
      f"min {min(ts):.2f} us ({steps} steps x {reps} replays)")
