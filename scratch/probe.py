import sys, os, ctypes, numpy as np, torch
os.environ['DTQ_DEBUG_GEMM_PROBE'] = '1'
sys.path.insert(0, '.')
import paper_2406_02540_b200 as dtq
M, K, N = [int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (16384, 1152, 4608))]
x = (torch.randn(M, K) * 2).half().cuda(); w = (torch.randn(N, K) / K**.5).half().cuda()
layer = dtq.QuantLinear.create(w, 8, 8)
codes, s, z = dtq.quantize_rows(x)
y = torch.empty(M, N, dtype=torch.float16, device='cuda')
for _ in range(3): layer.gemm(codes, s, z, out=y)
torch.cuda.synchronize()
L = dtq.lib(); L.dtq_diag_probe_ptr.restype = ctypes.c_void_p
ptr = L.dtq_diag_probe_ptr()
buf = np.zeros(148 * 8, np.uint64)
torch.cuda.synchronize()
ctypes.CDLL('libcudart.so.12').cudaMemcpy(ctypes.c_void_p(buf.ctypes.data), ctypes.c_void_p(ptr), ctypes.c_size_t(buf.nbytes), 2)
p = buf.reshape(148, 8).astype(np.float64)
tot = p[:, 5].mean()
names = ['tma empty-wait', 'mma full-wait', 'mma tempty-wait', 'epi0 tfull-wait', 'epi0 store-drain', 'total']
cfg = os.environ.get('DTQ_GEMM_CFG', 'auto'); dbg = os.environ.get('DTQ_DEBUG_GEMM_EPI', '0')
print(f"M={M} cfg={cfg} dbg={dbg}: " + ", ".join(f"{n} {p[:, i].mean() / tot * 100:.0f}%" for i, n in enumerate(names[:5])) + f", total {tot:.0f} cyc")
