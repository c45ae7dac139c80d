"""Seeded random sweep of the device path against the CPU oracle.

Each case draws a shape (M, K, N), weight / activation bit widths, input
dtype and balance (smoothing + 128-block rotation or none), then checks the
bars of SURVEY.md section 8c on that case:
  * codes / s / z of the fast quantizer without balance: bit-exact;
  * codes / s / z of the exact (fp64) quantizer with balance: bit-exact
    against the oracle's scale + rotate + quantize;
  * the GEMM's int32 accumulator from those codes: bit-exact;
  * the fp16 forward: within 1e-3 of max|y_ref| (the reference's norm).
Shapes include K that are not multiples of 128 (the lane-group and exact
kernels), single rows, and N that are not multiples of any tile width.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
import paper_2406_02540_b200 as dtq  # noqa: E402

pytestmark = pytest.mark.gpu

DEV = "cuda"
CASES = 64


def _case(i):
    rng = np.random.default_rng(1000 + i)
    M = int(rng.choice([1, 7, 129, 300, 1024, 2500]))
    K = int(rng.choice([64, 128, 200, 384, 1152, 1280, 2304, 4608]))
    N = int(rng.choice([1, 40, 256, 333, 1152, 4608]))
    wbits = int(rng.choice([2, 4, 6, 8]))
    abits = int(rng.choice([4, 8])) if wbits != 8 else 8
    dtype = [torch.float16, torch.bfloat16, torch.float32][int(rng.integers(0, 3))]
    balance = bool(rng.integers(0, 2)) and K % 128 == 0
    return rng, M, K, N, wbits, abits, dtype, balance


@pytest.mark.parametrize("i", range(CASES))
def test_random_case(oracle, i):
    rng, M, K, N, wbits, abits, dtype, balance = _case(i)
    gains = np.exp(rng.standard_normal(K))
    x = (rng.standard_normal((M, K)) * gains)
    x[:, rng.integers(0, K)] *= 25.0
    xt = torch.from_numpy(x).to(dtype).to(DEV)
    xd = xt.double().cpu().numpy()               # the values the device sees
    w = (rng.standard_normal((N, K)) / np.sqrt(K)).astype(np.float32)
    wt = torch.from_numpy(w).to(DEV)

    bal, xs = None, xd
    if balance:
        smooth = np.exp(0.3 * rng.standard_normal(K))
        signs = dtq.hadamard_signs(K, 7)
        bal = dtq.Balance(torch.from_numpy(smooth).to(DEV), torch.from_numpy(signs).to(DEV), 128)
        xs = oracle.rotate_blocks(oracle.scale_x(xd, smooth), signs, 128)
    layer = dtq.QuantLinear.create(wt, wbits, abits, balance=bal)
    wc, sw, _ = layer.export()                   # codes, scales, row sums
    zw = np.full(N, 1 << (wbits - 1), np.int32)  # symmetric weights: z = 2^(b-1)

    # quantizer: fast mode is bit-exact without balance, exact mode with it
    mode = dtq.MODE_EXACT if balance else dtq.MODE_FAST
    codes, s, z = dtq.quantize_rows(xt, bits=abits, mode=mode, balance=bal)
    c_ref, s_ref, z_ref = oracle.quantize_rows(xs, abits)
    assert np.array_equal(codes.cpu().numpy(), c_ref), (M, K, N, wbits, abits, dtype, balance)
    assert np.array_equal(s.cpu().numpy(), s_ref)
    assert np.array_equal(z.cpu().numpy(), z_ref)

    # GEMM accumulator from the device codes: exact (checked on a row sample
    # so the CPU oracle stays within seconds)
    rows = np.arange(M) if M <= 128 else np.sort(rng.choice(M, 128, replace=False))
    acc = layer.gemm(codes, s, z, out_dtype=torch.int32).cpu().numpy().astype(np.int64)[rows]
    acc_ref = oracle.qlinear_acc(c_ref[rows], z_ref[rows], wc, zw)
    assert np.array_equal(acc, acc_ref)

    # forward (fast mode end to end; fp16 / bf16 / fp32 out) against the
    # fp64 reference epilogue: fp16 within 1e-3 (the reference's norm), bf16
    # within its own rounding (2^-8)
    if abits == 8:
        ydt = [torch.float16, torch.bfloat16, torch.float32][i % 3]
        y = layer.forward(xt, out_dtype=ydt).double().cpu().numpy()[rows]
        y_ref = oracle.qlinear_epilogue(acc_ref, s_ref[rows], sw)
        err = np.abs(y - y_ref).max() / max(np.abs(y_ref).max(), 1e-30)
        # fp16 / fp32 out: the reference's 1e-3 norm (test_qgemm.cpp:19-26),
        # balanced (fast fp32 transforms) or not; bf16 out: its own rounding
        # (2^-9 relative per element)
        tol = 4e-3 if ydt == torch.bfloat16 else 1e-3
        assert err <= tol, (ydt, err)


FAST_CASES = 24


def _fast_case(i):
    rng = np.random.default_rng(5000 + i)
    M = int(rng.choice([3, 64, 500, 2048]))
    K = int(rng.choice([128, 256, 1152, 2304, 4608]))
    dtype = [torch.float16, torch.bfloat16, torch.float32][int(rng.integers(0, 3))]
    pro = ["none", "modulate", "gelu", "ln_modulate"][i % 4]
    return rng, M, K, dtype, pro


def _fast_chain(oracle, xd, pro, sc, sh, smooth, signs, eps=1e-6):
    # the fp64 chain the fast kernel approximates: prologue (toydit.cpp:
    # 339-369 modulate, :83 GELU, or the fp64 LayerNorm restatement -- no
    # reference LN exists), apply_scaling X / s (balance.cpp:57-67), 128-block
    # rotate_channels (balance.cpp:94-107)
    if pro == "gelu":
        xd = oracle.gelu(xd)
    elif pro == "modulate":
        xd = oracle.modulate(xd, sc, sh)
    elif pro == "ln_modulate":
        mu = xd.mean(1, keepdims=True)
        var = ((xd - mu) ** 2).mean(1, keepdims=True)
        xd = oracle.modulate((xd - mu) / np.sqrt(var + eps), sc, sh)
    return oracle.rotate_blocks(oracle.scale_x(xd, smooth), signs, 128)


def test_random_fast_balanced_pooled(oracle):
    # The fast fp32 quantizer with smoothing + rotation (and each fused
    # prologue) against the oracle's fp64 chain, over seeded cases: codes
    # within 1 LSB everywhere, and at most 1e-4 of codes off (north_star),
    # both per case (a case smaller than 1e4 codes may have one) and pooled.
    nd_all, n_all, lines = 0, 0, []
    for i in range(FAST_CASES):
        rng, M, K, dtype, pro = _fast_case(i)
        x = rng.standard_normal((M, K)) * np.exp(rng.standard_normal(K))
        xt = torch.from_numpy(x).to(dtype).to(DEV)
        xd = xt.double().cpu().numpy()
        smooth = np.exp(0.3 * rng.standard_normal(K))
        signs = dtq.hadamard_signs(K, 7)
        sc = (rng.standard_normal(K) * 0.2).astype(np.float32)
        sh = (rng.standard_normal(K) * 0.1).astype(np.float32)
        bal = dtq.Balance(torch.from_numpy(smooth).to(DEV), torch.from_numpy(signs).to(DEV), 128)
        kind = {"none": dtq.PROLOGUE_NONE, "modulate": dtq.PROLOGUE_MODULATE,
                "gelu": dtq.PROLOGUE_GELU, "ln_modulate": dtq.PROLOGUE_LN_MODULATE}[pro]
        p = dtq.Prologue(kind, torch.from_numpy(sc).to(DEV), torch.from_numpy(sh).to(DEV), 1e-6)
        codes, s, z = dtq.quantize_rows(xt, mode=dtq.MODE_FAST, balance=bal, prologue=p)
        ref = _fast_chain(oracle, xd, pro, sc.astype(np.float64), sh.astype(np.float64), smooth,
                          signs)
        c_ref, s_ref, z_ref = oracle.quantize_rows(ref, 8)
        d = np.abs(codes.cpu().numpy().astype(int) - c_ref.astype(int))
        nd = int((d > 0).sum())
        lines.append(f"case {i:2d} {pro:11s} {str(dtype)[6:]:8s} M={M:5d} K={K:5d} "
                     f"diff={nd} rate={nd / d.size:.2e}")
        assert d.max() <= 1, lines[-1]
        assert nd <= max(1e-4 * d.size, 1), lines[-1]
        # the per-token scale is the reference's fp64 s of the row's fp32 range
        assert np.allclose(s.cpu().numpy(), s_ref, rtol=1e-5, atol=0), lines[-1]
        nd_all += nd
        n_all += d.size
    print("\n".join(lines))
    print(f"pooled fast-mode code mismatch rate {nd_all / n_all:.2e} ({nd_all} of {n_all})")
    assert nd_all <= 1e-4 * n_all
