"""W4A8 vs W8A8 layer forward (diagnostics, not the bench contract).

usage: [DTQ_W4_UNPACK=0|1] python tools/w4_bench.py [M K N] ...
Times layer.forward (fused quantizer with smooth + Hadamard -> GEMM, fp16
out) for a W8A8 and a W4A8 layer of the same shape, in CUDA graphs of KB
forwards over a ring of layers and inputs larger than L2 (as the bench's C2
step), and prints the W4 / W8 throughput ratio.
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_02540_b200 as dtq  # noqa: E402

KB = 20


def timed(layers, xs, ys, ws, reps=5):
    n = len(layers)

    def run():
        for i in range(KB):
            layers[i % n].forward(xs[i % n], out=ys[i % n], workspace=ws)

    run()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        run()
    for _ in range(3):
        g.replay()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3 / KB)
    ts.sort()
    return ts[len(ts) // 2]


def one(M, K, N):
    dev = torch.device("cuda:0")
    gen = torch.Generator(device=dev).manual_seed(0)
    signs = torch.from_numpy(dtq.hadamard_signs(K, 7)).to(dev)
    bal = dtq.Balance(torch.rand(K, generator=gen, device=dev, dtype=torch.float64) + 0.5, signs,
                      128)
    per = M * K * 2 + N * K + M * N * 2
    ring = max(2, int(300e6 // per) + 1)
    xs = [torch.randn((M, K), generator=gen, device=dev).half() for _ in range(ring)]
    ys = [torch.empty((M, N), dtype=torch.float16, device=dev) for _ in range(ring)]
    out = {}
    for wb in (8, 4):
        layers = [dtq.QuantLinear.create((torch.randn((N, K), generator=gen, device=dev)
                                          / K ** 0.5).half(), wb, 8, balance=bal)
                  for _ in range(ring)]
        ws = layers[0].workspace(M, dev)
        out[wb] = timed(layers, xs, ys, ws)
        del layers
    ops = 2.0 * M * K * N
    print(f"M={M} K={K} N={N}: W8 {out[8]:.2f} us ({ops / out[8] * 1e-6:.0f} TOPS)  "
          f"W4 {out[4]:.2f} us ({ops / out[4] * 1e-6:.0f} TOPS)  W4/W8 {out[8] / out[4]:.3f}",
          flush=True)


if __name__ == "__main__":
    a = sys.argv[1:] or ["4096", "1152", "3456", "4096", "1152", "1152", "4096", "1152", "4608",
                         "4096", "4608", "1152", "16384", "1152", "3456", "16384", "1152", "4608",
                         "16384", "4608", "1152", "16384", "1152", "1152"]
    for i in range(0, len(a), 3):
        one(int(a[i]), int(a[i + 1]), int(a[i + 2]))
