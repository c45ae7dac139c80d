import sys, os, numpy as np, torch
sys.path.insert(0, '.')
import paper_2406_02540_b200 as dtq
M, K = 4096, 1152
x = (torch.randn(M, K) * 2).half().cuda()
w = (torch.randn(256, K) / K**.5).half().cuda()
bal = dtq.Balance(torch.rand(K, dtype=torch.float64).cuda() + 0.5, torch.from_numpy(dtq.hadamard_signs(K, 7)).cuda(), 128)
layer = dtq.QuantLinear.create(w, 8, 8, balance=bal)
ldc = (K + 15) // 16 * 16
buf = torch.empty(M, ldc, dtype=torch.uint8, device='cuda')
out = (buf[:, :K], torch.empty(M, dtype=torch.float64, device='cuda'), torch.empty(M, dtype=torch.int32, device='cuda'))
flush = torch.empty(512 << 20, dtype=torch.uint8, device='cuda')
y = torch.empty_like(x)
big = torch.empty(64 << 20, dtype=torch.float32, device='cuda')
def timeit(fn, mode, n=50):
    ts = []
    for i in range(n):
        if mode == 'flushw': flush.fill_(i)
        elif mode == 'flushr': flush.fill_(i); big.sum()
        elif mode == 'busy': torch.cuda._sleep(200000)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return np.median(ts) * 1e3, np.mean(ts) * 1e3
for mode in ['busy', 'flushw', 'flushr']:
    for name, fn in [('copy x->y 9.4MB', lambda: y.copy_(x)), ('FQ bal', lambda: layer.quantize(x, out=out)), ('empty-record', lambda: None)]:
        med, mean = timeit(fn, mode)
        print(f"{mode:7s} {name:18s} median {med:6.1f} us  mean {mean:6.1f} us")
