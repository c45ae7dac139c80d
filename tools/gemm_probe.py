"""Per-role wait cycles of the GEMM (DTQ_DEBUG_GEMM_PROBE=1 diagnostics).

usage: DTQ_DEBUG_GEMM_PROBE=1 python tools/gemm_probe.py M N K [wbits]
Needs a diagnostics build (the product kernel has no probes):
  tools/variant.sh diag '-DDTQ_GEMM_DIAG'; export DTQ_B200_LIB=variants/diag/libdtq_b200.so
"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_02540_b200 as dtq  # noqa: E402

M, N, K = (int(v) for v in sys.argv[1:4])
WB = int(sys.argv[4]) if len(sys.argv) > 4 else 8
dev = torch.device("cuda:0")
x = torch.randn(M, K, device=dev).half()
w = (torch.randn(N, K, device=dev) / K ** 0.5).half()
layer = dtq.QuantLinear.create(w, WB, 8)
codes, s, z = layer.quantize(x)
y = torch.empty(M, N, dtype=torch.float16, device=dev)
for _ in range(3):
    layer.gemm(codes, s, z, out=y)
torch.cuda.synchronize()
lib = dtq.lib()
lib.dtq_diag_probe_ptr.restype = C.c_void_p
ptr = lib.dtq_diag_probe_ptr()
buf = torch.zeros(4096 * 8, dtype=torch.int64, device=dev)
C.CDLL(None)
torch.cuda.synchronize()
# zero the probe, run once, read it back
cud = C.CDLL("libcudart.so")
cud.cudaMemset(C.c_void_p(ptr), 0, 4096 * 8 * 8)
layer.gemm(codes, s, z, out=y)
torch.cuda.synchronize()
host = (C.c_uint64 * (4096 * 8))()
cud.cudaMemcpy(host, C.c_void_p(ptr), 4096 * 8 * 8, 2)
a = np.frombuffer(host, dtype=np.uint64).reshape(4096, 8)[:148].astype(np.float64)
names = ["tma empty-wait", "mma full-wait", "mma tempty-wait", "epi tfull-wait",
         "epi store-drain", "total"]
for i, n in enumerate(names):
    print(f"{n:16s} mean {a[:, i].mean():10.0f} cyc  max {a[:, i].max():10.0f}")
