"""Race detection by repetition (compute-sanitizer is closed on this GPU pool):
every GEMM tile configuration (1-CTA / CTA pair x BN 256 / 128, W8A8 and
W4A8 incl. W4 CTA pairs, W4A8 forwards on s8 weights expanded into a
shared workspace) and the quantizer kernels run the same forwards
hundreds of times back to back, interleaved with other shapes so the
persistent kernels' pipelines (mbarrier phases, TMEM double buffer, TMA ring,
converter ring) start in every state; every result must be bit-identical to
the first.  A missing barrier, a phase bug or a TMEM / smem reuse race shows
up as a differing output.

usage: python tools/race_stress.py [reps]      (prints one JSON line per config)
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def child(reps):
    import torch
    import paper_2406_02540_b200 as dtq
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev).manual_seed(0)
    layers, xs = [], []
    for wb, M, K, N, pro in ((8, 300, 256, 512, None), (8, 1000, 1152, 4608, "ln"),
                             (4, 777, 1152, 1152, "gelu"), (4, 2048, 4608, 1152, None),
                             (8, 129, 128, 200, None)):
        signs = torch.from_numpy(dtq.hadamard_signs(K, 7)).to(dev)
        bal = dtq.Balance(torch.rand(K, generator=g, device=dev, dtype=torch.float64) + 0.5,
                          signs, 128)
        w = (torch.randn((N, K), generator=g, device=dev) / K ** 0.5).half()
        layers.append((dtq.QuantLinear.create(w, wb, 8, balance=bal), pro))
        xs.append((torch.randn((M, K), generator=g, device=dev) * 2).half())
    sc = torch.randn(1152, device=dev) * 0.1
    sh = torch.randn(1152, device=dev) * 0.1
    pros = {None: None, "gelu": dtq.Prologue(dtq.PROLOGUE_GELU),
            "ln": dtq.Prologue(dtq.PROLOGUE_LN_MODULATE, sc, sh, 1e-6)}
    # one workspace for every layer, as a network's forward shares it: each
    # W4A8 forward rewrites the s8 weights the previous layer's GEMM read
    ws = torch.zeros(max(dtq.lib().dtq_qlinear_workspace_bytes(l._h, x.shape[0])
                         for (l, _), x in zip(layers, xs)), dtype=torch.uint8, device=dev)
    first = [l.forward(x, prologue=pros[p]).clone() for (l, p), x in zip(layers, xs)]
    acc0 = [l.gemm(*l.quantize(x, prologue=pros[p]), out_dtype=torch.int32).clone()
            for (l, p), x in zip(layers, xs)]
    torch.cuda.synchronize()
    bad = 0
    for r in range(reps):
        for i, ((l, p), x) in enumerate(zip(layers, xs)):
            y = l.forward(x, prologue=pros[p], workspace=ws)
            if (r & 7) == 0:
                a = l.gemm(*l.quantize(x, prologue=pros[p]), out_dtype=torch.int32)
                bad += int(not torch.equal(a, acc0[i]))
            bad += int(not torch.equal(y, first[i]))
    torch.cuda.synchronize()
    print(json.dumps({"config": os.environ.get("DTQ_GEMM_CFG", "auto"),
                      "w4_cta2": os.environ.get("DTQ_GEMM_W4_CTA2", "0"), "reps": reps,
                      "forwards": reps * len(layers), "mismatches": bad}), flush=True)
    return bad


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--child":
        sys.exit(1 if child(int(sys.argv[2])) else 0)
    reps = sys.argv[1] if len(sys.argv) > 1 else "200"
    rc = 0
    for cfg, w4p in (("auto", "0"), ("0", "0"), ("1", "0"), ("2", "1"), ("3", "1")):
        env = dict(os.environ, DTQ_GEMM_W4_CTA2=w4p)
        if cfg != "auto":
            env["DTQ_GEMM_CFG"] = cfg
        rc |= subprocess.run([sys.executable, __file__, "--child", reps], env=env).returncode
    sys.exit(rc)
