"""One C2 forward's two kernels, a few times (for ncu captures of the product
kernels at the headline shape; diagnostics)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_02540_b200 as dtq  # noqa: E402
from bench import HBLOCK, K, M, N, make_inputs  # noqa: E402

dev = torch.device("cuda:0")
x_np, w_np, smooth_np = make_inputs()
x, w = torch.from_numpy(x_np).to(dev), torch.from_numpy(w_np).to(dev)
bal = dtq.Balance(torch.from_numpy(smooth_np).to(dev),
                  torch.from_numpy(dtq.hadamard_signs(K, 7)).to(dev), HBLOCK)
layer = dtq.QuantLinear.create(w, 8, 8, balance=bal)
ws = layer.workspace(M, dev)
y = torch.empty((M, N), dtype=torch.float16, device=dev)
for _ in range(5):
    layer.forward(x, out=y, workspace=ws)
torch.cuda.synchronize()
print("ok")
