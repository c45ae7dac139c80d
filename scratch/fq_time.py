import sys, os, numpy as np, torch
sys.path.insert(0, '.')
import paper_2406_02540_b200 as dtq
M, K = [int(v) for v in (sys.argv[1:3] if len(sys.argv) > 2 else (4096, 1152))]
bal_on = int(os.environ.get('BAL', '1'))
x = (torch.randn(M, K) * 2).half().cuda()
w = (torch.randn(256, K) / K**.5).half().cuda()
bal = dtq.Balance(torch.rand(K, dtype=torch.float64).cuda() + 0.5, torch.from_numpy(dtq.hadamard_signs(K, 7)).cuda(), 128) if bal_on else None
layer = dtq.QuantLinear.create(w, 8, 8, balance=bal)
ldc = (K + 15) // 16 * 16
buf = torch.empty(M, ldc, dtype=torch.uint8, device='cuda')
out = (buf[:, :K], torch.empty(M, dtype=torch.float64, device='cuda'), torch.empty(M, dtype=torch.int32, device='cuda'))
flush = torch.empty(512 << 20, dtype=torch.uint8, device='cuda')
for _ in range(5): layer.quantize(x, out=out)
ts = []
for i in range(100):
    flush.fill_(i)
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); layer.quantize(x, out=out); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
tc = np.mean(ts) * 1e-3
a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
a.record()
for i in range(50): layer.quantize(x, out=out)
b.record(); torch.cuda.synchronize(); tw = a.elapsed_time(b) * 1e-3 / 50
by = 3 * M * K + 12 * M
print(f"FQ M={M} K={K} bal={bal_on}: cold {tc*1e6:.1f} us {by/tc/1e9:.0f} GB/s | warm {tw*1e6:.1f} us {by/tw/1e9:.0f} GB/s")
