import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2406_02540_b200 as dtq
g = dict(np.load('tests/golden/golden.npz'))
cuda = lambda a: torch.as_tensor(np.ascontiguousarray(a)).cuda()
for wb in (8, 4):
    layer = dtq.QuantLinear.create(cuda(g['w']), wb, 8, bias=cuda(g['bias']))
    x = cuda(g['q_x'])
    codes, s, z = dtq.quantize_rows(x)
    acc = layer.gemm(codes, s, z, out_dtype=torch.int32).cpu().numpy().astype(np.float64)
    y64 = layer.forward(x, out_dtype=torch.float64, mode=dtq.MODE_EXACT).cpu().numpy()
    yref = g[f'w{wb}_y']
    sx = s.cpu().numpy(); sw = g[f'w{wb}_s']
    ynp = (sx[:, None] * sw[None, :]) * acc + g['bias'][None, :]
    d = y64 != yref
    print(wb, 'mismatch', d.sum(), 'maxabs', np.abs(y64 - yref).max(), 'np==ref', (ynp == yref).all(), 'np==gpu', (ynp == y64).all())
    idx = np.argwhere(d)[:5]
    for t, o in idx:
        print(t, o, y64[t, o], yref[t, o], ynp[t, o], acc[t, o], sx[t], sw[o])
    y64b = layer.forward(x, out_dtype=torch.float64, mode=dtq.MODE_EXACT).cpu().numpy()
    print('repeat equal', (y64b == y64).all())
