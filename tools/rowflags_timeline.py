"""CTA timeline of one forward: quantizer and GEMM CTA start / end times
(globaltimer), to see whether the two kernels overlap (row flags).

Needs a diagnostics build with both probes:
  tools/variant.sh tl '-DDTQ_GEMM_DIAG -DFQ_TILE_PROBE'
  DTQ_B200_LIB=variants/tl/libdtq_b200.so DTQ_DEBUG_GEMM_PROBE=1 DTQ_DEBUG_FQ_PROBE=1 \\
      python tools/rowflags_timeline.py [M K N]
"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_02540_b200 as dtq  # noqa: E402

M, K, N = (int(v) for v in sys.argv[1:4]) if len(sys.argv) > 3 else (4096, 1152, 4608)
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(0)
w = (torch.randn((N, K), generator=g, device=dev) / K ** 0.5).half()
signs = torch.from_numpy(dtq.hadamard_signs(K, 7)).to(dev)
smooth = torch.rand(K, generator=g, device=dev, dtype=torch.float64) + 0.5
layer = dtq.QuantLinear.create(w, 8, 8, balance=dtq.Balance(smooth, signs, 128))
x = (torch.randn((M, K), generator=g, device=dev) * 2).half()
ws = layer.workspace(M, dev)
y = torch.empty((M, N), dtype=torch.float16, device=dev)
for _ in range(5):
    layer.forward(x, out=y, workspace=ws)
torch.cuda.synchronize()
lib = dtq.lib()
lib.dtq_diag_probe_ptr.restype = C.c_void_p
lib.dtq_diag_fq_probe_ptr.restype = C.c_void_p
gp, fp = lib.dtq_diag_probe_ptr(), lib.dtq_diag_fq_probe_ptr()
cud = C.CDLL("libcudart.so")
for p, n in ((gp, 4096 * 8 * 8), (fp, 65536 * 8 * 8)):
    if p:
        cud.cudaMemset(C.c_void_p(p), 0, n)
torch.cuda.synchronize()
# the forward as it runs in a network: several back to back in one CUDA graph
# (no host launch gaps); the probes keep the last forward's CTAs
NG = int(os.environ.get("TL_GRAPH", "3"))
if NG > 0:
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        for _ in range(NG):
            layer.forward(x, out=y, workspace=ws)
    torch.cuda.synchronize()
    for p, n in ((gp, 4096 * 8 * 8), (fp, 65536 * 8 * 8)):
        if p:
            cud.cudaMemset(C.c_void_p(p), 0, n)
    torch.cuda.synchronize()
    gr.replay()
else:
    layer.forward(x, out=y, workspace=ws)
torch.cuda.synchronize()


def read(p, rows):
    host = (C.c_uint64 * (rows * 8))()
    cud.cudaMemcpy(host, C.c_void_p(p), rows * 8 * 8, 2)
    return np.frombuffer(host, dtype=np.uint64).reshape(rows, 8).astype(np.float64)


fq = read(fp, 4096) if fp else None
gm = read(gp, 4096) if gp else None
t0 = None
if fq is not None:
    f = fq[fq[:, 3] > 0]
    t0 = f[:, 3].min()
    print(f"quantizer: {len(f)} CTAs, start {0:.2f}..{(f[:, 3].max() - t0) / 1e3:.2f} us, "
          f"end {(f[:, 4].min() - t0) / 1e3:.2f}..{(f[:, 4].max() - t0) / 1e3:.2f} us")
if gm is not None:
    q = gm[gm[:, 6] > 0]
    t0 = t0 if t0 is not None else q[:, 6].min()
    print(f"gemm:      {len(q)} CTAs, start {(q[:, 6].min() - t0) / 1e3:.2f}..{(q[:, 6].max() - t0) / 1e3:.2f} us, "
          f"end {(q[:, 7].min() - t0) / 1e3:.2f}..{(q[:, 7].max() - t0) / 1e3:.2f} us")
    print(f"gemm wait cycles (mean): tma empty {q[:, 0].mean():.0f}  mma full {q[:, 1].mean():.0f}  "
          f"epi tfull {q[:, 3].mean():.0f}  total {q[:, 5].mean():.0f}")
