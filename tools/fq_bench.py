"""Fused-quantizer micro-benchmark (diagnostics, not the bench contract).

usage: python tools/fq_bench.py [M K pro rot dtype] ...   e.g.  4096 1152 none 1 f16
Times layer.quantize (fast mode) with CUDA events, L2 flushed between reps.
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_02540_b200 as dtq  # noqa: E402


def one(M, K, pro, rot, dtype, reps=50):
    dev = torch.device("cuda:0")
    dt = {"f16": torch.float16, "bf16": torch.bfloat16, "f32": torch.float32}[dtype]
    g = torch.Generator().manual_seed(0)
    x = (torch.randn(M, K, generator=g) * torch.exp(torch.randn(K, generator=g))).to(dt).to(dev)
    w = (torch.randn(256, K, generator=g) / K ** 0.5).to(torch.float16).to(dev)
    bal = None
    if rot:
        smooth = torch.exp(0.3 * torch.randn(K, generator=g)).double().to(dev)
        signs = torch.from_numpy(dtq.hadamard_signs(K, 7)).to(dev)
        bal = dtq.Balance(smooth, signs, 128)
    layer = dtq.QuantLinear.create(w, 8, 8, balance=bal)
    prologue = None
    sc, sh = torch.randn(K, device=dev) * 0.1, torch.randn(K, device=dev) * 0.1
    if pro == "gelu":
        prologue = dtq.Prologue(dtq.PROLOGUE_GELU)
    elif pro == "mod":
        prologue = dtq.Prologue(dtq.PROLOGUE_MODULATE, sc, sh)
    elif pro == "ln":
        prologue = dtq.Prologue(dtq.PROLOGUE_LN_MODULATE, sc, sh)
    codes = torch.empty(M, (K + 15) // 16 * 16, dtype=torch.uint8, device=dev)[:, :K]
    s = torch.empty(M, dtype=torch.float64, device=dev)
    z = torch.empty(M, dtype=torch.int32, device=dev)
    # a ring of input copies larger than L2 (126 MB): every launch reads cold
    # data; batches of launches between two events (the event clock ticks in
    # ~2 us steps, too coarse for one small kernel)
    nbuf = max(2, int(256e6 // x.numel() // x.element_size()) + 1)
    xs = [x.clone() for _ in range(nbuf)]
    batch = 20

    def run(i=0):
        layer.quantize(xs[i % nbuf], mode=dtq.MODE_FAST, out=(codes, s, z), prologue=prologue)

    run(0)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()       # no host launch overhead in the timing
    with torch.cuda.graph(graph):
        for i in range(batch):
            run(i)
    ts = []
    for r in range(reps // 5 + 3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        graph.replay()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3 / batch)
    ts.sort()
    med = ts[len(ts) // 2]
    nbytes = M * K * (x.element_size() + 1) + 12 * M
    print(f"M={M} K={K} pro={pro} rot={rot} {dtype}: median {med:.2f} us  min {ts[0]:.2f} us  "
          f"{nbytes / med / 1e3:.0f} GB/s", flush=True)


if __name__ == "__main__":
    args = sys.argv[1:] or ["4096", "1152", "none", "1", "f16", "16384", "1152", "none", "1", "f16",
                            "16384", "4608", "gelu", "1", "f16", "16384", "1152", "ln", "1", "f16"]
    for i in range(0, len(args), 5):
        one(int(args[i]), int(args[i + 1]), args[i + 2], int(args[i + 3]), args[i + 4])
