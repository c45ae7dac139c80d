"""Measure the fast-mode code mismatch rates against the fp64 oracle chain.

For each fast path (balance only, modulate, modulate + balance, GELU +
balance, LayerNorm-modulate + balance) and input dtype, quantize seeded
activations on the device and compare with the oracle's fp64 chain
(toydit.cpp:339-369 modulate / :83 GELU / fp64 LayerNorm restatement ->
balance.cpp:57-67 scaling -> 128-block rotate_channels -> quant.cpp:140-177).
Prints one JSON line per case and a pooled summary.  Diagnostics only.
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2406_02540_b200 as dtq  # noqa: E402
from oracle.oracle import Oracle  # noqa: E402

orc = Oracle()
DEV = "cuda"


def chain(xd, pro, sc, sh, smooth, signs, eps=1e-6):
    if pro == "gelu":
        xd = orc.gelu(xd)
    elif pro == "mod":
        xd = orc.modulate(xd, sc, sh)
    elif pro == "ln":
        xd = orc.modulate(orc.layernorm(xd, eps), sc, sh)
    if smooth is not None:
        xd = orc.scale_x(xd, smooth)
    if signs is not None:
        xd = orc.rotate_blocks(xd, signs, 128)
    return xd


def main():
    pooled = {}
    for pro in ["none", "mod", "gelu", "ln"]:
        for bal in [False, True]:
            if pro == "none" and not bal:
                continue
            for dt in [torch.float16, torch.bfloat16, torch.float32]:
                for K in [128, 1152, 2304, 4608]:
                    rng = np.random.default_rng(K + 17)
                    M = 2048 if K <= 1152 else 1024
                    x = rng.standard_normal((M, K)) * np.exp(rng.standard_normal(K))
                    x[:, rng.integers(0, K, 4)] *= 30
                    xt = torch.from_numpy(x).to(dt).to(DEV)
                    xd = xt.double().cpu().numpy()
                    sc = (rng.standard_normal(K) * 0.2).astype(np.float32)
                    sh = (rng.standard_normal(K) * 0.1).astype(np.float32)
                    smooth = np.exp(0.3 * rng.standard_normal(K)) if bal else None
                    signs = dtq.hadamard_signs(K, 7) if bal else None
                    b = dtq.Balance(torch.from_numpy(smooth).to(DEV),
                                    torch.from_numpy(signs).to(DEV), 128) if bal else None
                    kind = {"none": 0, "mod": dtq.PROLOGUE_MODULATE, "gelu": dtq.PROLOGUE_GELU,
                            "ln": dtq.PROLOGUE_LN_MODULATE}[pro]
                    p = dtq.Prologue(kind, torch.from_numpy(sc).to(DEV),
                                     torch.from_numpy(sh).to(DEV), 1e-6) if pro != "none" else None
                    codes, s, z = dtq.quantize_rows(xt, mode=dtq.MODE_FAST, balance=b, prologue=p)
                    ref = chain(xd, pro, sc.astype(np.float64), sh.astype(np.float64), smooth,
                                signs)
                    c_ref, s_ref, z_ref = orc.quantize_rows(ref, 8)
                    d = np.abs(codes.cpu().numpy().astype(int) - c_ref.astype(int))
                    srel = float(np.abs(s.cpu().numpy() / s_ref - 1).max())
                    rec = {"pro": pro, "bal": bal, "dtype": str(dt).split(".")[-1], "K": K, "M": M,
                           "max_d": int(d.max()), "n_diff": int((d > 0).sum()),
                           "rate": float((d > 0).mean()), "s_rel_max": srel,
                           "z_diff": int((z.cpu().numpy() != z_ref).sum())}
                    print(json.dumps(rec), flush=True)
                    key = (pro, bal)
                    a = pooled.setdefault(key, [0, 0, 0])
                    a[0] += rec["n_diff"]
                    a[1] += d.size
                    a[2] = max(a[2], rec["max_d"])
    for (pro, bal), (nd, n, md) in pooled.items():
        print(json.dumps({"pooled": f"{pro}/bal={bal}", "rate": nd / n, "n_diff": nd, "n": n,
                          "max_d": md}))


if __name__ == "__main__":
    main()
