import sys, os, numpy as np, torch
sys.path.insert(0, '.')
import paper_2406_02540_b200 as dtq
M, K, N = [int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (4096, 1152, 4608))]
wb = int(os.environ.get('WB', '8'))
x = (torch.randn(M, K) * 2).half().cuda(); w = (torch.randn(N, K) / K**.5).half().cuda()
layer = dtq.QuantLinear.create(w, wb, 8)
codes, s, z = dtq.quantize_rows(x)
y = torch.empty(M, N, dtype=torch.float16, device='cuda')
flush = torch.empty(512 << 20, dtype=torch.uint8, device='cuda')
for _ in range(5): layer.gemm(codes, s, z, out=y)
ts = []
for i in range(50):
    flush.fill_(i)
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); layer.gemm(codes, s, z, out=y); b.record()
    torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
t = np.median(ts) * 1e-3
print(f"M={M} K={K} N={N} W{wb} noepi={os.environ.get('DTQ_DEBUG_GEMM_NOEPI','0')}: {t*1e6:.1f} us  {2*M*N*K/t/1e12:.0f} TOPS")
