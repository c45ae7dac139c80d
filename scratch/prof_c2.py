import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2406_02540_b200 as dtq
import bench
x_np, w_np, sm = bench.make_inputs()
M, K, N = bench.M, bench.K, bench.N
x = torch.from_numpy(x_np).cuda(); w = torch.from_numpy(w_np).cuda()
bal = dtq.Balance(torch.from_numpy(sm).cuda(), torch.from_numpy(dtq.hadamard_signs(K, 7)).cuda(), 128)
layer = dtq.QuantLinear.create(w, 8, 8, balance=bal)
y = torch.empty((M, N), dtype=torch.float16, device='cuda')
ws = layer.workspace(M)
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 5):
    layer.forward(x, out=y, workspace=ws)
torch.cuda.synchronize()
print('ok')
