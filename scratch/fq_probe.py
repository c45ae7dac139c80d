import sys, os, ctypes, numpy as np, torch
os.environ['DTQ_DEBUG_FQ_PROBE'] = '1'
sys.path.insert(0, '.')
import paper_2406_02540_b200 as dtq
M, K = [int(v) for v in (sys.argv[1:3] if len(sys.argv) > 2 else (4096, 1152))]
bal_on = int(os.environ.get('BAL', '1'))
x = (torch.randn(M, K) * 2).half().cuda(); w = (torch.randn(256, K) / K**.5).half().cuda()
bal = dtq.Balance(torch.rand(K, dtype=torch.float64).cuda() + 0.5, torch.from_numpy(dtq.hadamard_signs(K, 7)).cuda(), 128) if bal_on else None
layer = dtq.QuantLinear.create(w, 8, 8, balance=bal)
torch.cuda.synchronize()
L = dtq.lib(); L.dtq_diag_fq_probe_ptr.restype = ctypes.c_void_p
ptr = L.dtq_diag_fq_probe_ptr()
cudart = ctypes.CDLL('libcudart.so.12')
cudart.cudaMemset(ctypes.c_void_p(ptr), 0, ctypes.c_size_t(65536 * 64))
codes, s, z = layer.quantize(x)
torch.cuda.synchronize()
buf = np.zeros(65536 * 8, np.uint64)
cudart.cudaMemcpy(ctypes.c_void_p(buf.ctypes.data), ctypes.c_void_p(ptr), ctypes.c_size_t(buf.nbytes), 2)
p = buf.reshape(-1, 8).astype(np.float64); p = p[p[:, 4] > 0]
rows = p[:, 4].sum()
print(f"M={M} K={K} bal={bal_on}: warps {len(p)}, rows/warp {p[:,4].mean():.2f}; per-row cycles: wait {p[:,0].sum()/rows:.0f}, pass1 {p[:,1].sum()/rows:.0f}, params {p[:,2].sum()/rows:.0f}, pass2 {p[:,3].sum()/rows:.0f}")
