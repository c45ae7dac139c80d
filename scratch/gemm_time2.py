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
# (a) cold: flush then one launch, mean of 100
ts = []
for i in range(100):
    flush.fill_(i)
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); layer.gemm(codes, s, z, out=y); b.record()
    torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
tc = np.mean(ts) * 1e-3
# (b) warm back-to-back: 50 launches between two events
a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
a.record()
for i in range(50): layer.gemm(codes, s, z, out=y)
b.record(); torch.cuda.synchronize()
tw = a.elapsed_time(b) * 1e-3 / 50
ops = 2 * M * N * K
print(f"M={M} K={K} N={N} W{wb} cfg={os.environ.get('DTQ_GEMM_CFG','auto')} noepi={os.environ.get('DTQ_DEBUG_GEMM_NOEPI','0')}: cold {tc*1e6:.1f} us {ops/tc/1e12:.0f} TOPS | warm b2b {tw*1e6:.1f} us {ops/tw/1e12:.0f} TOPS")
