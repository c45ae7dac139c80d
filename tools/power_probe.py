"""GEMM time with random vs all-zero operands, per diagnostics mode
(profiles/r02_gemm_epilogue_smsp.md).

usage: [DTQ_B200_LIB=variants/diag/libdtq_b200.so DTQ_DEBUG_GEMM_EPI=n] [TAG=name]
       python tools/power_probe.py
W8A8 GEMM at C2 (4096 x 4608 x 1152) and 16384 rows, fp16 out, CUDA graph of
20 launches over a >L2 ring of code buffers; "zero" = all-zero activation
codes and zero weights (minimal operand toggling).  Diagnostics.
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_02540_b200 as dtq  # noqa: E402

dev = torch.device("cuda:0")
def run(M, N, K, zero):
    if zero:
        wc = torch.full((N, K), 128, dtype=torch.uint8, device=dev)
        layer = dtq.QuantLinear.from_codes(wc, torch.ones(N, dtype=torch.float64, device=dev) * 1e-2, 8, K)
        codes = torch.zeros((M, K), dtype=torch.uint8, device=dev)
    else:
        wc = torch.randint(0, 256, (N, K), dtype=torch.uint8, device=dev)
        layer = dtq.QuantLinear.from_codes(wc, torch.ones(N, dtype=torch.float64, device=dev) * 1e-2, 8, K)
        codes = torch.randint(0, 256, (M, K), dtype=torch.uint8, device=dev)
    s = torch.rand(M, dtype=torch.float64, device=dev) * 1e-2
    z = torch.randint(0, 256, (M,), dtype=torch.int32, device=dev)
    y = torch.empty(M, N, dtype=torch.float16, device=dev)
    nb = max(2, int(256e6 // (M * K)) + 1)
    cs = [codes.clone() for _ in range(nb)]
    def f():
        for i in range(20):
            layer.gemm(cs[i % nb], s, z, out=y)
    f(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        f()
    ts = []
    for _ in range(7):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); g.replay(); b.record(); b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3 / 20)
    ts.sort()
    return ts[3]
for M, N, K in ((4096, 4608, 1152), (16384, 4608, 1152)):
    r = run(M, N, K, False); z = run(M, N, K, True)
    print(f"{os.environ.get('TAG','')} M={M} N={N} K={K}: random {r:.1f} us  zero {z:.1f} us  ({2*M*N*K/r*1e-6:.0f} / {2*M*N*K/z*1e-6:.0f} TOPS)", flush=True)
