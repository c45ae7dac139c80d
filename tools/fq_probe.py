"""Per-CTA timeline of the tile quantizer (DTQ_DEBUG_FQ_PROBE=1 diagnostics).

usage: DTQ_DEBUG_FQ_PROBE=1 python tools/fq_probe.py M K
Needs a build with -DFQ_TILE_PROBE (tools/variant.sh probe '-DFQ_TILE_PROBE';
export DTQ_B200_LIB=variants/probe/libdtq_b200.so).
"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_02540_b200 as dtq  # noqa: E402

M, K = int(sys.argv[1]), int(sys.argv[2])
dev = torch.device("cuda:0")
x = (torch.randn(M, K, device=dev) * 2).half()
w = (torch.randn(256, K, device=dev) / K ** 0.5).half()
signs = torch.from_numpy(dtq.hadamard_signs(K, 7)).to(dev)
smooth = torch.rand(K, device=dev, dtype=torch.float64) + 0.5
layer = dtq.QuantLinear.create(w, 8, 8, balance=dtq.Balance(smooth, signs, 128))
for _ in range(3):
    layer.quantize(x)
torch.cuda.synchronize()
lib = dtq.lib()
lib.dtq_diag_fq_probe_ptr.restype = C.c_void_p
ptr = lib.dtq_diag_fq_probe_ptr()
cud = C.CDLL("libcudart.so")
cud.cudaMemset(C.c_void_p(ptr), 0, 65536 * 8 * 8)
layer.quantize(x)
torch.cuda.synchronize()
host = (C.c_uint64 * (65536 * 8))()
cud.cudaMemcpy(host, C.c_void_p(ptr), 65536 * 8 * 8, 2)
a = np.frombuffer(host, dtype=np.uint64).reshape(-1, 8)[:, :5].astype(np.float64)
a = a[a[:, 2] > 0]
t0 = a[:, 3].min()
print(f"CTAs {len(a)}: data-wait {a[:, 0].mean():.0f}  barrier {a[:, 1].mean():.0f}  "
      f"loop {a[:, 2].mean():.0f} cycles (max {a[:, 2].max():.0f}); CTA start spread "
      f"{(a[:, 3].max() - t0) / 1e3:.2f} us, lifetime mean {(a[:, 4] - a[:, 3]).mean() / 1e3:.2f} us, "
      f"last end {(a[:, 4].max() - t0) / 1e3:.2f} us after first start")
