"""fc1 -> GELU -> fc2 at the stack's 16384 rows, both GELU placements:
GELU in fc1's GEMM epilogue (fc2 quantizes as is) vs GELU as the prologue
of fc2's quantizer.  CUDA-graph batches; per-forward us.  Diagnostics."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_02540_b200 as dtq  # noqa: E402

dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(0)
M, D = 16384, 1152


def layer(K, N):
    w = (torch.randn((N, K), generator=g, device=dev) / K ** 0.5).half()
    bal = dtq.Balance(torch.rand(K, generator=g, device=dev, dtype=torch.float64) + 0.5,
                      torch.from_numpy(dtq.hadamard_signs(K, 7)).to(dev), 128)
    return dtq.QuantLinear.create(w, 8, 8, balance=bal)


fc1, fc2 = layer(D, 4 * D), layer(4 * D, D)
x = (torch.randn((M, D), generator=g, device=dev) * 2).half()
h = torch.empty((M, 4 * D), dtype=torch.float16, device=dev)
y = torch.empty((M, D), dtype=torch.float16, device=dev)
ws = fc2.workspace(M, dev)
gelu = dtq.Prologue(dtq.PROLOGUE_GELU)


def timeit(fn, n=10, reps=10):
    fn()
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        for _ in range(n):
            fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        gr.replay()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3 / n)
    return float(np.median(ts))


r = {
    "fc1": timeit(lambda: fc1.forward(x, out=h, workspace=ws)),
    "fc1+gelu_epilogue": timeit(lambda: fc1.forward(x, out=h, workspace=ws, activation=dtq.ACT_GELU)),
    "fc2": timeit(lambda: fc2.forward(h, out=y, workspace=ws)),
    "fc2+gelu_prologue": timeit(lambda: fc2.forward(h, out=y, workspace=ws, prologue=gelu)),
}
r["gelu_in_epilogue_total"] = r["fc1+gelu_epilogue"] + r["fc2"]
r["gelu_in_prologue_total"] = r["fc1"] + r["fc2+gelu_prologue"]
for k, v in r.items():
    print(f"{k:26s} {v:8.1f} us")
