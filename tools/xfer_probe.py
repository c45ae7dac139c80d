"""Host<->device copy ceilings and forward_host pipelining (diagnostics).

usage: python tools/xfer_probe.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_02540_b200 as dtq  # noqa: E402

M, K, N = 4096, 1152, 4608
dev = torch.device("cuda:0")
xh = torch.randn(M, K).half().pin_memory()
yh = torch.empty(M, N, dtype=torch.float16).pin_memory()
xd = torch.empty(M, K, dtype=torch.float16, device=dev)
yd = torch.randn(M, N, device=dev).half()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


h2d = t(lambda: xd.copy_(xh, non_blocking=True))
d2h = t(lambda: yh.copy_(yd, non_blocking=True))
print(f"H2D {xh.numel() * 2 / 1e6:.1f} MB: {h2d * 1e3:.0f} us = {xh.numel() * 2 / h2d / 1e6:.1f} GB/s")
print(f"D2H {yh.numel() * 2 / 1e6:.1f} MB: {d2h * 1e3:.0f} us = {yh.numel() * 2 / d2h / 1e6:.1f} GB/s")


def both():
    ev = torch.cuda.Event()
    ev.record()
    s1.wait_event(ev)
    s2.wait_event(ev)
    with torch.cuda.stream(s1):
        xd.copy_(xh, non_blocking=True)
    with torch.cuda.stream(s2):
        yh.copy_(yd, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


print(f"H2D || D2H: {t(both) * 1e3:.0f} us")
w = (torch.randn(N, K, device=dev) / K ** 0.5).half()
layer = dtq.QuantLinear.create(w, 8, 8)
print(f"forward_host: {t(lambda: layer.forward_host(xh, yh)) * 1e3:.0f} us "
      f"(chunks={os.environ.get('DTQ_HOST_CHUNKS', '8')})")

# chunked copies alone: 8 D2H chunks on one stream, and with 8 H2D chunks on another
yc = [(yh[i * 512:(i + 1) * 512], yd[i * 512:(i + 1) * 512]) for i in range(8)]
xc = [(xd[i * 512:(i + 1) * 512], xh[i * 512:(i + 1) * 512]) for i in range(8)]


def d2h_chunks():
    for hb, db in yc:
        hb.copy_(db, non_blocking=True)


def both_chunks():
    ev = torch.cuda.Event()
    ev.record()
    s1.wait_event(ev)
    s2.wait_event(ev)
    for (hb, db), (dd, hs) in zip(yc, xc):
        with torch.cuda.stream(s1):
            dd.copy_(hs, non_blocking=True)
        with torch.cuda.stream(s2):
            hb.copy_(db, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


print(f"8 D2H chunks: {t(d2h_chunks) * 1e3:.0f} us; with 8 H2D chunks: {t(both_chunks) * 1e3:.0f} us")
import time  # noqa: E402
x512 = xd[:512].clone()
y512 = torch.empty(512, N, dtype=torch.float16, device=dev)
ws = layer.workspace(512, dev)
for _ in range(5):
    layer.forward(x512, out=y512, workspace=ws)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(100):
    layer.forward(x512, out=y512, workspace=ws)
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"host enqueue of one 512-row forward: {(t1 - t0) * 1e4:.1f} us")
