"""GEMM micro-benchmark (diagnostics, not the bench contract).

usage: python tools/gemm_bench.py [M N K wbits] ...
Times layer.gemm (codes already quantized) with CUDA events, L2 flushed
between reps, against torch._int_mm (cuBLASLt s8xs8->s32, no epilogue) and
fp16 torch.matmul on the same shape.  DTQ_GEMM_CFG selects the tile config.
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_02540_b200 as dtq  # noqa: E402


def timeit(fn, flush, reps=30, batch=10):
    """Mean time per call over batches of `batch` back-to-back calls between
    two events (the event clock ticks in ~2 us steps); fn(i) should rotate
    through inputs larger than L2."""
    fn(0)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()       # no host launch overhead in the timing
    with torch.cuda.graph(graph):
        for i in range(batch):
            fn(i)
    ts = []
    for r in range(max(3, reps // 5)):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        graph.replay()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3 / batch)
    ts.sort()
    return ts[len(ts) // 2]


def one(M, N, K, wbits):
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev).manual_seed(0)
    x = torch.randn(M, K, generator=g, device=dev).half()
    w = (torch.randn(N, K, generator=g, device=dev) / K ** 0.5).half()
    layer = dtq.QuantLinear.create(w, wbits, 8)
    codes, s, z = layer.quantize(x)
    y = torch.empty(M, N, dtype=torch.float16, device=dev)
    flush = None
    nb = max(2, int(256e6 // (M * K)) + 1)   # code buffers cycling through > L2
    cs = [codes.clone() for _ in range(nb)]
    t = timeit(lambda i: layer.gemm(cs[i % nb], s, z, out=y), flush)
    a8s = [torch.randint(-127, 127, (M, K), dtype=torch.int8, device=dev) for _ in range(nb)]
    b8 = torch.randint(-127, 127, (K, N), dtype=torch.int8, device=dev).t().contiguous().t()
    ti = timeit(lambda i: torch._int_mm(a8s[i % nb], b8), flush)
    nh = max(2, int(256e6 // (2 * M * K)) + 1)
    xs = [x.clone() for _ in range(nh)]
    th = timeit(lambda i: torch.matmul(xs[i % nh], w.t(), out=y), flush)
    ops = 2.0 * M * N * K
    print(f"M={M} N={N} K={K} W{wbits}: ours {t:.1f} us {ops / t / 1e6:.0f} TOPS | "
          f"cublasLt int8 {ti:.1f} us {ops / ti / 1e6:.0f} | fp16 {th:.1f} us {ops / th / 1e6:.0f}",
          flush=True)


if __name__ == "__main__":
    a = sys.argv[1:] or ["4096", "4608", "1152", "8", "16384", "3456", "1152", "8",
                         "16384", "1152", "1152", "8", "16384", "4608", "1152", "8",
                         "16384", "1152", "4608", "8", "480", "2304", "1152", "8",
                         "16384", "4608", "1152", "4"]
    for i in range(0, len(a), 4):
        one(int(a[i]), int(a[i + 1]), int(a[i + 2]), int(a[i + 3]))
