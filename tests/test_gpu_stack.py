"""C4 stack parity: two PixArt-alpha blocks' prologue-bearing linears chained
through the device path (fast mode, as the bench stack runs them), each
layer checked against the oracle chain on its own device input.

Per block (toydit.cpp:159-219 order, attention and residuals left out --
they are not on the quantized-linear path):
    x  --LN+modulate--> qkv (1152 -> 3456)            [checked, not chained]
    x  --LN+modulate--> fc1 (1152 -> 4608) + GELU in fc1's GEMM epilogue
       --fp16--> fc2 (4608 -> 1152)                    [block 0]
    x  --LN+modulate--> fc1 --fp16--> GELU prologue of fc2's quantizer --> fc2
                                                       [block 1: the other placement]
    fc2's fp16 output is the next block's x.
Every linear carries smooth + 128-block Hadamard balance.  For each layer,
on sampled token rows (exact: quantization is row-local, quant.cpp:70-73):
  * codes within 1 LSB of the oracle's fp64 chain on <= 1e-4 of codes
    (pooled over the stack, and per layer);
  * the int32 accumulator the oracle computes from the GPU's own codes
    equals the device's (qgemm.cpp:52-60);
  * fp16 y within 1e-3 of max|y_ref| (test_qgemm.cpp:19-26).
The oracle chain: oracle.modulate / oracle.layernorm (no reference LN;
pinned against torch's F.layer_norm in fp64) / oracle.gelu (toydit.cpp:83), then
scale_x + rotate_blocks + quantize_rows, qlinear_acc, qlinear_epilogue.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
import paper_2406_02540_b200 as dtq  # noqa: E402

pytestmark = pytest.mark.gpu

DEV = "cuda"
M, D = 4096, 1152
ROWS = 192
EPS = 1e-6


def _ln_mod(oracle, xd, sc, sh):
    return oracle.modulate(oracle.layernorm(xd, EPS), sc, sh)


def _layer(rng, K, N, oracle):
    w = (rng.standard_normal((N, K)) / np.sqrt(K)).astype(np.float16)
    smooth = np.exp(0.3 * rng.standard_normal(K))
    signs = oracle.hadamard_signs(K, 7)
    bias = rng.standard_normal(N) * 0.05
    bal = dtq.Balance(torch.from_numpy(smooth).to(DEV), torch.from_numpy(signs).to(DEV), 128)
    layer = dtq.QuantLinear.create(torch.from_numpy(w).to(DEV), 8, 8,
                                   bias=torch.from_numpy(bias).to(DEV), balance=bal)
    wc, sw, _ = layer.export()
    return layer, smooth, signs, bias, wc, sw


def _check(oracle, name, layer, x_dev, pre, smooth, signs, bias, wc, sw, rows, prologue, stats,
           act=dtq.ACT_NONE):
    codes, s, z = layer.quantize(x_dev, mode=dtq.MODE_FAST, prologue=prologue)
    y = layer.forward(x_dev, out_dtype=torch.float16, prologue=prologue, activation=act)
    acc = layer.gemm(codes, s, z, out_dtype=torch.int32)
    xr = x_dev[torch.as_tensor(rows, device=DEV)].double().cpu().numpy()
    chain = oracle.rotate_blocks(oracle.scale_x(pre(xr), smooth), signs, 128)
    c_ref, s_ref, _ = oracle.quantize_rows(chain, 8)
    c_gpu = codes.cpu().numpy()[rows]
    d = np.abs(c_gpu.astype(np.int32) - c_ref.astype(np.int32))
    nd = int((d > 0).sum())
    stats.append((name, nd, d.size))
    assert d.max() <= 1, (name, d.max())
    assert nd <= max(1e-4 * d.size, 1), (name, nd, d.size)
    z_gpu = z.cpu().numpy()[rows]
    acc_ref = oracle.qlinear_acc(c_gpu, z_gpu, wc, np.full(wc.shape[0], 128, np.int32))
    assert np.array_equal(acc.cpu().numpy()[rows].astype(np.int64), acc_ref), name
    y_ref = oracle.qlinear_epilogue(acc_ref, s.cpu().numpy()[rows], sw, bias)
    if act == dtq.ACT_GELU:  # gelu(y) in the epilogue: against the oracle's exact-erf GELU
        y_ref = oracle.gelu(y_ref)
    err = np.abs(y.float().cpu().numpy()[rows] - y_ref).max() / np.abs(y_ref).max()
    assert err <= 1e-3, (name, err)
    return y


def test_c4_two_block_chain(oracle):
    rng = np.random.default_rng(2024)
    g = np.exp(rng.standard_normal(D))
    x0 = rng.standard_normal((M, D)) * g
    x0[:, rng.choice(D, 4, replace=False)] *= 30
    x = torch.from_numpy(x0.astype(np.float16)).to(DEV)
    rows = np.sort(rng.choice(M, ROWS, replace=False))
    stats = []
    for blk in range(2):
        sc = (rng.standard_normal(D) * 0.2).astype(np.float32)
        sh = (rng.standard_normal(D) * 0.1).astype(np.float32)
        pro_ln = dtq.Prologue(dtq.PROLOGUE_LN_MODULATE, torch.from_numpy(sc).to(DEV),
                              torch.from_numpy(sh).to(DEV), EPS)
        scd, shd = sc.astype(np.float64), sh.astype(np.float64)
        ln = lambda xr: _ln_mod(oracle, xr, scd, shd)  # noqa: E731
        qkv = _layer(rng, D, 3 * D, oracle)
        _check(oracle, f"b{blk}.qkv", qkv[0], x, ln, *qkv[1:], rows, pro_ln, stats)
        fc1 = _layer(rng, D, 4 * D, oracle)
        epi = blk == 0  # block 0: GELU in fc1's epilogue; block 1: in fc2's quantizer
        h = _check(oracle, f"b{blk}.fc1", fc1[0], x, ln, *fc1[1:], rows, pro_ln, stats,
                   act=dtq.ACT_GELU if epi else dtq.ACT_NONE)
        fc2 = _layer(rng, 4 * D, D, oracle)
        x = _check(oracle, f"b{blk}.fc2", fc2[0], h, (lambda v: v) if epi else oracle.gelu,
                   *fc2[1:], rows, None if epi else dtq.Prologue(dtq.PROLOGUE_GELU), stats)
        assert bool(torch.isfinite(x).all())
    nd = sum(s[1] for s in stats)
    n = sum(s[2] for s in stats)
    for name, a, b in stats:
        print(f"{name}: {a} of {b} codes differ ({a / b:.2e})")
    print(f"stack pooled code mismatch {nd / n:.2e}")
    assert nd <= 1e-4 * n
