"""GPU parity: the sm_100a path (through the C ABI) against the CPU oracle.

Bars (BASELINE.json north_star):
  * rotation off: u8 codes, f64 per-token scales, i32 zero points and the
    int32 accumulators are bit-exact;
  * rotation on (fast fp32 mode): codes differ by at most 1 LSB on at most
    1e-4 of elements; the exact (fp64) mode is bit-exact with rotation too;
  * fp16 outputs: max|y - y_ref| <= 1e-3 * max|y_ref|;
  * the F64 parity epilogue reproduces the reference's fp64 y bit-for-bit.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
import paper_2406_02540_b200 as dtq  # noqa: E402

pytestmark = pytest.mark.gpu

DEV = "cuda"
REL_TOL = 1e-3


def f64(a):
    return np.asarray(a, dtype=np.float64)


def cuda(a, dtype=None):
    t = torch.as_tensor(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.to(DEV)


def rel_err(y, y_ref):
    return np.abs(np.asarray(y, np.float64) - y_ref).max() / max(np.abs(y_ref).max(), 1e-30)


def activations(rng, M, K, outliers=4):
    g = np.exp(rng.standard_normal(K))
    x = rng.standard_normal((M, K)) * g
    x[:, rng.choice(K, outliers, replace=False)] *= 30.0
    x = x.astype(np.float16)
    x[0] = 0.0
    x[1] = 0.5
    x[2] = np.abs(x[2])
    x[3] = -np.abs(x[3])
    return x


# ------------------------------------------------------------------ quantizer
@pytest.mark.parametrize("mode", [dtq.MODE_FAST, dtq.MODE_EXACT])
@pytest.mark.parametrize("bits", [8, 6, 4, 2])
def test_quantizer_golden_bitexact(golden, mode, bits):
    x = cuda(golden["q_x"])
    codes, s, z = dtq.quantize_rows(x, bits, mode=mode)
    key = "q" if bits == 8 else f"q{bits}"
    assert np.array_equal(codes.cpu().numpy(), golden[f"{key}_codes"])
    assert np.array_equal(s.cpu().numpy(), golden[f"{key}_s"])
    assert np.array_equal(z.cpu().numpy(), golden[f"{key}_z"])


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16, torch.float32, torch.float64])
def test_quantizer_full_size_bitexact(oracle, dtype):
    rng = np.random.default_rng(11)
    x = activations(rng, 4096, 1152)
    xt = torch.from_numpy(x.astype(np.float32)).to(dtype)
    codes, s, z = dtq.quantize_rows(xt.to(DEV))
    c_ref, s_ref, z_ref = oracle.quantize_rows(xt.double().numpy(), 8)
    assert np.array_equal(codes.cpu().numpy(), c_ref)
    assert np.array_equal(s.cpu().numpy(), s_ref)
    assert np.array_equal(z.cpu().numpy(), z_ref)


@pytest.mark.parametrize("K", [8, 40, 128, 136, 200, 1000, 1152, 2304, 2432, 4608, 8192, 9216])
def test_quantizer_ragged_and_wide(oracle, K):
    rng = np.random.default_rng(K)
    x = (rng.standard_normal((37, K)) * 3).astype(np.float16)
    x[5] = 1.0
    codes, s, z = dtq.quantize_rows(cuda(x))
    c_ref, s_ref, z_ref = oracle.quantize_rows(f64(x), 8)
    assert np.array_equal(codes.cpu().numpy(), c_ref)
    assert np.array_equal(s.cpu().numpy(), s_ref) and np.array_equal(z.cpu().numpy(), z_ref)


def test_quantizer_unaligned_pitch(oracle):
    rng = np.random.default_rng(5)
    base = (rng.standard_normal((64, 1160)) * 2).astype(np.float16)
    xt = cuda(base)[:, 3:3 + 1152]          # pitch 1160, misaligned start
    codes, s, z = dtq.quantize_rows(xt)
    c_ref, s_ref, z_ref = oracle.quantize_rows(f64(base[:, 3:3 + 1152]), 8)
    assert np.array_equal(codes.cpu().numpy(), c_ref) and np.array_equal(s.cpu().numpy(), s_ref)


def test_quantizer_row_shards_are_bit_identical():
    # per-token params are row-local (quant.cpp:70-73): any row split of X
    # quantizes to the same bytes -> token-row sharding across GPUs is exact
    rng = np.random.default_rng(3)
    x = cuda(activations(rng, 1000, 1152))
    full = dtq.quantize_rows(x)
    for a, b in [(0, 333), (333, 800), (800, 1000)]:
        part = dtq.quantize_rows(x[a:b])
        for p, f in zip(part, full):
            assert torch.equal(p, f[a:b])


def test_quantizer_nonfinite_sets_status():
    x = torch.randn(8, 256, device=DEV, dtype=torch.float16)
    x[3, 7] = float("inf")
    status = torch.zeros(1, dtype=torch.int32, device=DEV)
    dtq.quantize_rows(x, status=status)
    assert int(status.item()) == 1


# ------------------------------------------------------------------ balance
def test_balance_exact_mode_bitexact(golden):
    bal = dtq.Balance(cuda(golden["bal_smooth"]), cuda(golden["bal_signs"]), 128)
    codes, s, z = dtq.quantize_rows(cuda(golden["q_x"]), mode=dtq.MODE_EXACT, balance=bal)
    assert np.array_equal(codes.cpu().numpy(), golden["bal_codes"])
    assert np.array_equal(s.cpu().numpy(), golden["bal_s"])
    assert np.array_equal(z.cpu().numpy(), golden["bal_z"])
    rot = dtq.Balance(None, cuda(golden["bal_signs"]), 128)
    codes, s, z = dtq.quantize_rows(cuda(golden["q_x"]), mode=dtq.MODE_EXACT, balance=rot)
    assert np.array_equal(codes.cpu().numpy(), golden["rot_codes"])
    assert np.array_equal(s.cpu().numpy(), golden["rot_s"])


@pytest.mark.parametrize("M,K", [(4096, 1152), (1000, 4608), (37, 2304), (5, 128), (300, 2432)])
def test_balance_fast_mode_within_one_lsb(oracle, M, K):
    # the tile quantizer: 4 lanes per block up to K = 2304, 2 beyond; ragged
    # row tiles (M not a multiple of the tile height)
    rng = np.random.default_rng(21 + K)
    x = activations(rng, M, K)
    w = rng.standard_normal((256, K)) / np.sqrt(K)
    smooth = oracle.scaling_mask(np.abs(f64(x)).max(0), np.abs(w).max(0), 0.5)
    signs = oracle.hadamard_signs(K, 7)
    bal = dtq.Balance(cuda(smooth), cuda(signs), 128)
    codes, s, z = dtq.quantize_rows(cuda(x), mode=dtq.MODE_FAST, balance=bal)
    xr = oracle.rotate_blocks(oracle.scale_x(f64(x), smooth), signs, 128)
    c_ref, s_ref, z_ref = oracle.quantize_rows(xr, 8)
    d = np.abs(codes.cpu().numpy().astype(np.int32) - c_ref.astype(np.int32))
    assert d.max() <= 1, f"max code difference {d.max()}"
    assert (d > 0).mean() <= 1e-4, f"{(d > 0).mean():.2e} of codes differ"
    assert np.allclose(s.cpu().numpy(), s_ref, rtol=1e-6)


# ------------------------------------------------------------------ weights
@pytest.mark.parametrize("wb", [8, 4])
def test_weight_prep_bitexact(golden, wb):
    layer = dtq.QuantLinear.create(cuda(golden["w"]), wb, 8)
    codes, s, wsum = layer.export()
    assert np.array_equal(codes, golden[f"w{wb}_codes"])
    assert np.array_equal(s, golden[f"w{wb}_s"])
    zw = 1 << (wb - 1)
    assert np.array_equal(wsum, (golden[f"w{wb}_codes"].astype(np.int64) - zw).sum(1))


def test_weight_prep_balanced_bitexact(golden):
    bal = dtq.Balance(cuda(golden["bal_smooth"]), cuda(golden["bal_signs"]), 128)
    layer = dtq.QuantLinear.create(cuda(golden["w"]), 8, 8, balance=bal)
    codes, s, _ = layer.export()
    assert np.array_equal(codes, golden["bal_wcodes"])
    assert np.array_equal(s, golden["bal_ws"])


def test_w4_from_packed_codes(golden):
    # checkpoint path: the reference's packed nibble stream uploaded as is
    packed = cuda(golden["w4_packed"])
    layer = dtq.QuantLinear.from_codes(packed, cuda(golden["w4_s"]), 4, golden["w"].shape[1],
                                       packed=True)
    codes, s, _ = layer.export()
    assert np.array_equal(codes, golden["w4_codes"])


# ------------------------------------------------------------------ GEMM
@pytest.mark.parametrize("wb", [8, 4])
def test_gemm_golden_acc_and_f64_bitexact(golden, oracle, wb):
    bias = cuda(golden["bias"])
    layer = dtq.QuantLinear.create(cuda(golden["w"]), wb, 8, bias=bias)
    x = cuda(golden["q_x"])
    codes, s, z = dtq.quantize_rows(x)
    acc = layer.gemm(codes, s, z, out_dtype=torch.int32).cpu().numpy()
    acc_ref = oracle.qlinear_acc(golden["q_codes"], golden["q_z"], golden[f"w{wb}_codes"],
                                 golden[f"w{wb}_z"])
    assert np.array_equal(acc.astype(np.int64), acc_ref)
    y64 = layer.forward(x, out_dtype=torch.float64, mode=dtq.MODE_EXACT).cpu().numpy()
    assert np.array_equal(y64, golden[f"w{wb}_y"])           # reference fp64 y, bit-exact
    y16 = layer.forward(x, out_dtype=torch.float16).float().cpu().numpy()
    assert rel_err(y16, golden[f"w{wb}_y"]) <= REL_TOL


@pytest.mark.parametrize("i", [0, 1, 2])
def test_gemm_ragged_shapes(golden, i):
    layer = dtq.QuantLinear.create(cuda(golden[f"rag{i}_w"]), 8, 8, bias=cuda(golden[f"rag{i}_b"]))
    x = cuda(golden[f"rag{i}_x"])
    y64 = layer.forward(x, out_dtype=torch.float64, mode=dtq.MODE_EXACT).cpu().numpy()
    assert np.array_equal(y64, golden[f"rag{i}_y"])
    for dt in (torch.float16, torch.bfloat16, torch.float32):
        y = layer.forward(x, out_dtype=dt).double().cpu().numpy()
        tol = 1e-2 if dt == torch.bfloat16 else REL_TOL
        assert rel_err(y, golden[f"rag{i}_y"]) <= tol


def test_gemm_balanced_layer(golden):
    bal = dtq.Balance(cuda(golden["bal_smooth"]), cuda(golden["bal_signs"]), 128)
    layer = dtq.QuantLinear.create(cuda(golden["w"]), 8, 8, bias=cuda(golden["bias"]), balance=bal)
    x = cuda(golden["q_x"])
    y64 = layer.forward(x, out_dtype=torch.float64, mode=dtq.MODE_EXACT).cpu().numpy()
    assert np.array_equal(y64, golden["bal_y"])
    y16 = layer.forward(x, out_dtype=torch.float16, mode=dtq.MODE_FAST).float().cpu().numpy()
    assert rel_err(y16, golden["bal_y"]) <= REL_TOL


STDIT_SHAPES = [("qkv", 1152, 3456), ("proj", 1152, 1152), ("fc1", 1152, 4608),
                ("fc2", 4608, 1152)]


@pytest.mark.parametrize("wb", [8, 4])
@pytest.mark.parametrize("name,K,N", STDIT_SHAPES)
def test_stdit_shapes_full_size(oracle, wb, name, K, N):
    """Config 1 / 3 shapes at M=4096: int32 acc exact on sampled rows
    (row-local, so a row subset is an exact check), fp16 within 1e-3."""
    rng = np.random.default_rng(K * 7 + N + wb)
    M = 4096
    x = activations(rng, M, K)
    w = (rng.standard_normal((N, K)) / np.sqrt(K)).astype(np.float16)
    bias = rng.standard_normal(N) * 0.1
    layer = dtq.QuantLinear.create(cuda(w), wb, 8, bias=cuda(bias))
    xt = cuda(x)
    codes, s, z = dtq.quantize_rows(xt)
    acc = layer.gemm(codes, s, z, out_dtype=torch.int32)
    y16 = layer.forward(xt, out_dtype=torch.float16)
    rows = np.sort(rng.choice(M, 384, replace=False))
    rows[:4] = [0, 1, 2, 3]
    wc, sw, zw = oracle.make_quant_linear(f64(w), wb)
    c_ref, s_ref, z_ref = oracle.quantize_rows(f64(x[rows]), 8)
    assert np.array_equal(codes.cpu().numpy()[rows], c_ref)
    acc_ref = oracle.qlinear_acc(c_ref, z_ref, wc, zw)
    assert np.array_equal(acc.cpu().numpy()[rows].astype(np.int64), acc_ref)
    y_ref = oracle.qlinear_epilogue(acc_ref, s_ref, sw, bias)
    assert rel_err(y16.float().cpu().numpy()[rows], y_ref) <= REL_TOL


def test_prologue_modulate_exact(oracle):
    rng = np.random.default_rng(8)
    M, K, N = 300, 1152, 640
    x = activations(rng, M, K)
    sc = (rng.standard_normal(K) * 0.2).astype(np.float32)
    sh = (rng.standard_normal(K) * 0.1).astype(np.float32)
    pro = dtq.Prologue(dtq.PROLOGUE_MODULATE, cuda(sc), cuda(sh))
    codes, s, z = dtq.quantize_rows(cuda(x), mode=dtq.MODE_EXACT, prologue=pro)
    xm = oracle.modulate(f64(x), f64(sc), f64(sh))
    c_ref, s_ref, z_ref = oracle.quantize_rows(xm, 8)
    assert np.array_equal(codes.cpu().numpy(), c_ref) and np.array_equal(s.cpu().numpy(), s_ref)
    codes, s, z = dtq.quantize_rows(cuda(x), mode=dtq.MODE_FAST, prologue=pro)
    d = np.abs(codes.cpu().numpy().astype(int) - c_ref.astype(int))
    print(f"fast modulate: {(d > 0).mean():.2e} of codes differ")
    assert d.max() <= 1 and (d > 0).mean() <= 1e-4


@pytest.mark.parametrize("K", [1152, 1408, 3456, 4608])  # odd block counts: idle items
def test_prologue_gelu_and_layernorm_codes(oracle, K):
    # GELU follows toydit.cpp:83 (the oracle's exact-erf gelu); LayerNorm has
    # no reference counterpart, so its chain is the oracle's fp64 LayerNorm,
    # pinned against torch's F.layer_norm (tests/test_oracle.py).  Fast-mode codes
    # against the fp64 chain: within 1 LSB on at most 1e-4 of codes, the
    # north_star bar for fp32 transforms.
    rng = np.random.default_rng(9)
    x = activations(rng, 512, K).astype(np.float32)
    xt = cuda(x)
    xd = f64(x)
    codes, s, z = dtq.quantize_rows(xt, prologue=dtq.Prologue(dtq.PROLOGUE_GELU))
    c_ref, s_ref, z_ref = oracle.quantize_rows(oracle.gelu(xd), 8)
    d = np.abs(codes.cpu().numpy().astype(int) - c_ref.astype(int))
    print(f"GELU K={K}: {(d > 0).mean():.2e} of codes differ")
    assert d.max() <= 1 and (d > 0).mean() <= 1e-4
    sc = (rng.standard_normal(K) * 0.2).astype(np.float32)
    sh = (rng.standard_normal(K) * 0.1).astype(np.float32)
    pro = dtq.Prologue(dtq.PROLOGUE_LN_MODULATE, cuda(sc), cuda(sh), 1e-6)
    codes, s, z = dtq.quantize_rows(xt, prologue=pro)
    ln = oracle.layernorm(xd, 1e-6)
    c_ref, s_ref, z_ref = oracle.quantize_rows(oracle.modulate(ln, f64(sc), f64(sh)), 8)
    d = np.abs(codes.cpu().numpy().astype(int) - c_ref.astype(int))
    print(f"LN-modulate K={K}: {(d > 0).mean():.2e} of codes differ")
    assert d.max() <= 1 and (d > 0).mean() <= 1e-4


def test_overflow_guard_and_shape_errors():
    # K beyond the exact-int32 bound -> OverflowError (qgemm.cpp:29-34 convention)
    K = 70000
    codes = torch.full((1, K), 128, dtype=torch.uint8, device=DEV)
    layer = dtq.QuantLinear.from_codes(codes, torch.ones(1, dtype=torch.float64, device=DEV), 8, K)
    a = torch.zeros((128, (K + 15) // 16 * 16), dtype=torch.uint8, device=DEV)
    with pytest.raises(OverflowError):
        layer.gemm(a[:, :K], torch.ones(128, dtype=torch.float64, device=DEV),
                   torch.zeros(128, dtype=torch.int32, device=DEV))
    small = dtq.QuantLinear.create(torch.randn(16, 64, device=DEV, dtype=torch.float16))
    with pytest.raises(ValueError):
        small.forward(torch.randn(4, 32, device=DEV, dtype=torch.float16))  # X cols != C_in


def test_forward_host_buffers(golden):
    layer = dtq.QuantLinear.create(cuda(golden["w"]), 8, 8, bias=cuda(golden["bias"]))
    x = torch.from_numpy(golden["q_x"]).pin_memory()
    y = torch.empty((x.shape[0], layer.N), dtype=torch.float64).pin_memory()
    layer.forward_host(x, y, mode=dtq.MODE_EXACT)
    assert np.array_equal(y.numpy(), golden["w8_y"])
    x_bad = x.clone()
    x_bad[2, 2] = float("nan")
    with pytest.raises(ValueError):
        layer.forward_host(x_bad, y)


def test_deterministic():
    rng = np.random.default_rng(4)
    x = cuda(activations(rng, 1024, 1152))
    layer = dtq.QuantLinear.create(cuda(rng.standard_normal((2304, 1152)).astype(np.float16)), 4, 8)
    y1 = layer.forward(x)
    y2 = layer.forward(x)
    assert torch.equal(y1, y2)


@pytest.mark.gpu
@pytest.mark.parametrize("wcode", [0, 15])
def test_w4_extreme_codes_exact(wcode):
    # W4 weights enter the MMA as 16*(c - 8): the extremes (-128, +112 as s8)
    # at the largest STDiT K must still give the exact int32 accumulator
    K, N, M = 4608, 256, 512
    codes = torch.full((N, K), wcode, dtype=torch.uint8, device=DEV)
    layer = dtq.QuantLinear.from_codes(codes, torch.ones(N, dtype=torch.float64, device=DEV), 4, K)
    a = torch.full((M, K), 255, dtype=torch.uint8, device=DEV)
    a[1::2] = 0
    z = torch.zeros(M, dtype=torch.int32, device=DEV)
    z[2::4] = 255
    acc = layer.gemm(a, torch.ones(M, dtype=torch.float64, device=DEV), z, out_dtype=torch.int32)
    x = a.cpu().long() - z.cpu().long()[:, None]
    want = x.sum(1, keepdim=True) * (wcode - 8)
    assert torch.equal(acc.cpu().long(), want.expand(M, N))


@pytest.mark.gpu
def test_forward_host_pipelined_chunks_match_device_forward():
    # M >= 1024 with a non-F64 output takes the chunked two-stream host
    # pipeline; rows are independent, so it must equal the device forward
    rng = np.random.default_rng(21)
    M, K, N = 3000, 1152, 640
    x = torch.from_numpy(activations(rng, M, K).astype(np.float16))
    w = torch.from_numpy((rng.standard_normal((N, K)) / K ** 0.5).astype(np.float16))
    signs = torch.from_numpy(dtq.hadamard_signs(K, 7)).to(DEV)
    smooth = torch.from_numpy(rng.uniform(0.5, 2.0, K)).to(DEV)
    layer = dtq.QuantLinear.create(w.to(DEV), 8, 8, balance=dtq.Balance(smooth, signs, 128))
    want = layer.forward(x.to(DEV), out_dtype=torch.float16).cpu()
    xh = x.pin_memory()
    yh = torch.empty((M, N), dtype=torch.float16).pin_memory()
    layer.forward_host(xh, yh)
    assert torch.equal(yh, want)


@pytest.mark.gpu
def test_tile_quantizer_varying_tile_heights_in_one_process():
    # the tile height R (and so the kernel's dynamic smem) changes with M:
    # a small-M launch must not shrink the smem limit a later launch needs
    K = 1152
    signs = torch.from_numpy(dtq.hadamard_signs(K, 7)).to(DEV)
    bal = dtq.Balance(torch.ones(K, dtype=torch.float64, device=DEV) * 1.5, signs, 128)
    for M in (16384, 480, 16384, 37, 4096, 5):
        x = torch.randn(M, K, device=DEV).half()
        codes, s, z = dtq.quantize_rows(x, balance=bal)
        assert codes.shape == (M, K) and bool(torch.isfinite(s).all())


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("K", [1152, 4608, 8192])
def test_quantizer_input_dtypes_wide_rows(oracle, dtype, K):
    # tile kernel (two lanes per block beyond K = 1152, four-row tiles beyond
    # 4608) and, for fp32 rows too wide for a shared-memory tile, the
    # lane-group kernel: codes / s / z bit-exact with no balance
    rng = np.random.default_rng(K + 3)
    x = torch.from_numpy((rng.standard_normal((70, K)) * 3).astype(np.float32)).to(dtype)
    codes, s, z = dtq.quantize_rows(x.to(DEV))
    c_ref, s_ref, z_ref = oracle.quantize_rows(x.double().numpy(), 8)
    assert np.array_equal(codes.cpu().numpy(), c_ref)
    assert np.array_equal(s.cpu().numpy(), s_ref) and np.array_equal(z.cpu().numpy(), z_ref)


@pytest.mark.gpu
@pytest.mark.parametrize("K,N,packed", [(200, 100, False), (1152, 4608, True), (328, 96, True)])
def test_w4_gemm_tails_and_packed_upload(K, N, packed):
    # single-CTA W4A8 tiles read the packed nibbles straight from L2: K tails
    # (the last k-block past the packed row), N tails (rows past N) and the
    # checkpoint path (packed stream uploaded as stored) must give the exact
    # int32 accumulator
    rng = np.random.default_rng(K + N)
    M = 300
    wc = rng.integers(0, 16, (N, K), dtype=np.uint8)
    if packed:
        wp = np.zeros((N, (K + 1) // 2), np.uint8)
        wp |= wc[:, 0::2]
        wp[:, : K // 2] |= (wc[:, 1::2] << 4).astype(np.uint8)
        layer = dtq.QuantLinear.from_codes(cuda(wp), torch.ones(N, dtype=torch.float64, device=DEV),
                                           4, K, packed=True)
    else:
        layer = dtq.QuantLinear.from_codes(cuda(wc), torch.ones(N, dtype=torch.float64, device=DEV),
                                           4, K)
    a = rng.integers(0, 256, (M, K), dtype=np.uint8)
    z = rng.integers(0, 256, M).astype(np.int32)
    ldc = (K + 15) // 16 * 16
    ab = torch.zeros((M, ldc), dtype=torch.uint8, device=DEV)
    ab[:, :K] = cuda(a)
    acc = layer.gemm(ab[:, :K], torch.ones(M, dtype=torch.float64, device=DEV), cuda(z),
                     out_dtype=torch.int32).cpu().numpy().astype(np.int64)
    want = (a.astype(np.int64) - z[:, None]) @ (wc.astype(np.int64) - 8).T
    assert np.array_equal(acc, want)


@pytest.mark.gpu
def test_w4_cta_pair_path_exact(tmp_path):
    # CTA-pair W4A8 tiles (not the default choice; DTQ_GEMM_W4_CTA2=1 lets the
    # tile model pick them) give the same exact accumulators
    import os
    import subprocess
    import sys
    code = r"""
import numpy as np, torch, paper_2406_02540_b200 as dtq
rng = np.random.default_rng(5)
for K, N, M in [(1152, 4608, 600), (200, 100, 300)]:
    wc = rng.integers(0, 16, (N, K), dtype=np.uint8)
    layer = dtq.QuantLinear.from_codes(torch.from_numpy(wc).cuda(),
                                       torch.ones(N, dtype=torch.float64, device="cuda"), 4, K)
    a = rng.integers(0, 256, (M, K), dtype=np.uint8)
    z = rng.integers(0, 256, M).astype(np.int32)
    ldc = (K + 15) // 16 * 16
    ab = torch.zeros((M, ldc), dtype=torch.uint8, device="cuda")
    ab[:, :K] = torch.from_numpy(a).cuda()
    acc = layer.gemm(ab[:, :K], torch.ones(M, dtype=torch.float64, device="cuda"),
                     torch.from_numpy(z).cuda(), out_dtype=torch.int32).cpu().numpy()
    want = (a.astype(np.int64) - z[:, None]) @ (wc.astype(np.int64) - 8).T
    assert np.array_equal(acc.astype(np.int64), want), (K, N, M)
print("ok")
"""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, DTQ_GEMM_W4_CTA2="1", PYTHONPATH=root)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                       timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-3000:]


@pytest.mark.gpu
@pytest.mark.parametrize("K", [1, 5, 13, 67, 127, 129])
def test_w4_odd_k_exact(K):
    # odd K: the W4 nibble words run past (K + 1) / 2 bytes of the row; the
    # GEMM's B operand must carry every column (reference test_qgemm.cpp:64-77
    # draws c_in in 1..128)
    rng = np.random.default_rng(K)
    N, M = 37, 50
    wc = rng.integers(0, 16, (N, K), dtype=np.uint8)
    layer = dtq.QuantLinear.from_codes(cuda(wc), torch.ones(N, dtype=torch.float64, device=DEV),
                                       4, K)
    a = rng.integers(0, 256, (M, K), dtype=np.uint8)
    z = rng.integers(0, 256, M).astype(np.int32)
    ldc = (K + 15) // 16 * 16
    ab = torch.zeros((M, ldc), dtype=torch.uint8, device=DEV)
    ab[:, :K] = cuda(a)
    acc = layer.gemm(ab[:, :K], torch.ones(M, dtype=torch.float64, device=DEV), cuda(z),
                     out_dtype=torch.int32).cpu().numpy().astype(np.int64)
    want = (a.astype(np.int64) - z[:, None]) @ (wc.astype(np.int64) - 8).T
    assert np.array_equal(acc, want)


@pytest.mark.parametrize("wb", [8, 4])
def test_c5_full_size_balanced_row_shards(oracle, wb):
    """BASELINE configs[4] at its full size on one device: M = 131072 token
    rows (STDiT 16 x 512^2, batch 8), fc1 1152 -> 4608, smooth + 128-block
    Hadamard fused into the quantizer.  Properties that hold at any size:
      * the forward of each of 8 row shards (the per-GPU slice at 8 GPUs) is
        bit-identical to the same rows of the whole forward (quant.cpp:70-73:
        per-token params are row-local; qgemm.cpp:52-63: per-row dot);
      * on sampled rows, codes are within 1 LSB of the oracle on <= 1e-4 of
        elements, the int32 accumulators recomputed by the oracle from the
        GPU's own codes are equal, and fp16 y is within 1e-3."""
    rng = np.random.default_rng(131072 + wb)
    M, K, N = 131072, 1152, 4608
    # activations drawn on the device (the oracle checks a row sample only)
    g = torch.exp(torch.randn(K, device=DEV, dtype=torch.float64))
    xt = (torch.randn(M, K, device=DEV, dtype=torch.float64) * g)
    xt[:, :4] *= 30.0
    xt = xt.to(torch.float16)
    xt[0] = 0.0
    xt[1] = 0.5
    w = rng.standard_normal((N, K)) / np.sqrt(K)
    amax = xt[:8192].abs().amax(0).double().cpu().numpy()
    smooth = oracle.scaling_mask(amax, np.abs(w).max(0), 0.5)
    signs = oracle.hadamard_signs(K, 7)
    bal = dtq.Balance(cuda(smooth), cuda(signs), 128)
    bias = rng.standard_normal(N) * 0.1
    layer = dtq.QuantLinear.create(cuda(w.astype(np.float16)), wb, 8, bias=cuda(bias), balance=bal)
    y = layer.forward(xt, out_dtype=torch.float16)
    shard = M // 8
    for r in range(8):
        a, b = r * shard, (r + 1) * shard
        assert torch.equal(layer.forward(xt[a:b], out_dtype=torch.float16), y[a:b]), f"shard {r}"
    codes, s, z = layer.quantize(xt)
    acc = layer.gemm(codes, s, z, out_dtype=torch.int32)
    rows = np.sort(rng.choice(M, 256, replace=False))
    rows[:2] = [0, 1]
    x_rows = xt[torch.as_tensor(rows, device=DEV)].double().cpu().numpy()
    xr = oracle.rotate_blocks(oracle.scale_x(x_rows, smooth), signs, 128)
    c_ref, s_ref, _ = oracle.quantize_rows(xr, 8)
    c_gpu = codes.cpu().numpy()[rows]
    d = np.abs(c_gpu.astype(np.int32) - c_ref.astype(np.int32))
    assert d.max() <= 1 and (d > 0).mean() <= 1e-4, (d.max(), (d > 0).mean())
    assert np.allclose(s.cpu().numpy()[rows], s_ref, rtol=1e-6)
    wc, sw, _ = layer.export()
    zw = 1 << (wb - 1)
    z_gpu = z.cpu().numpy()[rows]
    acc_ref = oracle.qlinear_acc(c_gpu, z_gpu, wc, np.full(N, zw, np.int32))
    assert np.array_equal(acc.cpu().numpy()[rows].astype(np.int64), acc_ref)
    y_ref = oracle.qlinear_epilogue(acc_ref, s.cpu().numpy()[rows], sw, bias)
    assert rel_err(y.float().cpu().numpy()[rows], y_ref) <= REL_TOL


def test_planned_layer_dispatch_per_range():
    # a22: the device dispatch of a MixedPrecisionPlan row (toydit.cpp:113-117):
    # step t of `steps` runs bits_for(layer, t * 4 / steps); each range's
    # output equals a layer built at that width alone, bit for bit
    rng = np.random.default_rng(31)
    K, N, M = 1152, 640, 300
    w = cuda(rng.standard_normal((N, K)).astype(np.float16) / np.sqrt(K))
    signs = cuda(dtq.hadamard_signs(K, 7))
    bal = dtq.Balance(cuda(rng.uniform(0.5, 2.0, K)), signs, 128)
    bias = cuda(rng.standard_normal(N) * 0.1)
    plan = dtq.MixedPrecisionPlan({"blocks.0.mlp.fc1": (8, 4, 4, 6)})
    pl = dtq.PlannedLinear.create(w, plan, "blocks.0.mlp.fc1", bias=bias, balance=bal)
    x = cuda(activations(rng, M, K))
    alone = {b: dtq.QuantLinear.create(w, b, 8, bias=bias, balance=bal) for b in (8, 4, 6)}
    steps = 20
    for t in range(steps):
        b = plan.bits_for("blocks.0.mlp.fc1", dtq.range_index(t, steps))
        layer = pl.select(t, steps)
        assert layer.weight_bits == b
        assert torch.equal(pl.forward(x, t, steps), alone[b].forward(x)), (t, b)
    with pytest.raises(ValueError):
        pl.select(steps, steps)


def test_row_flag_path_subprocess():
    # the opt-in concurrent quantizer -> GEMM path (row flags) must stay
    # bit-identical to the two stages back to back: tests/test_gpu_rowflags.py
    # in a process of its own with the switch on
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, DTQ_ROW_FLAGS="1", PYTHONPATH=root)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        os.path.join(root, "tests", "test_gpu_rowflags.py")],
                       capture_output=True, text=True, env=env, timeout=600, cwd=root)
    print(r.stdout[-2000:])
    assert r.returncode == 0 and " passed" in r.stdout, r.stdout[-3000:] + r.stderr[-2000:]


def test_race_stress_every_tile_config():
    # race detection by repetition (compute-sanitizer is closed on this pool):
    # tools/race_stress.py, every GEMM tile config incl. W4 CTA pairs, each
    # forward repeated and interleaved with other shapes -- bit-identical
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "tools", "race_stress.py"), "30"],
                       capture_output=True, text=True, timeout=900, cwd=root)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr[-2000:]
    assert r.stdout.count('"mismatches": 0') == 5


@pytest.mark.parametrize("wb", [8, 4])
@pytest.mark.parametrize("odt", [torch.float16, torch.bfloat16])
def test_gelu_epilogue(oracle, wb, odt):
    # gelu(qlinear_forward(x)) with GELU applied in the GEMM's epilogue on the
    # fp32 y (the fc1 -> gelu of toydit.cpp:215-216): against the oracle's
    # exact-erf GELU of the reference epilogue within the output dtype's
    # tolerance, and against GELU applied to the fp32 output of the plain
    # forward (the same fp32 y) within one output rounding
    rng = np.random.default_rng(77 + wb)
    M, K, N = 1000, 1152, 4608
    x = activations(rng, M, K)
    w = (rng.standard_normal((N, K)) / np.sqrt(K)).astype(np.float16)
    bias = rng.standard_normal(N) * 0.1
    bal = dtq.Balance(cuda(rng.uniform(0.5, 2.0, K)), cuda(dtq.hadamard_signs(K, 7)), 128)
    layer = dtq.QuantLinear.create(cuda(w), wb, 8, bias=cuda(bias), balance=bal)
    xt = cuda(x)
    y = layer.forward(xt, out_dtype=odt, activation=dtq.ACT_GELU).double().cpu().numpy()
    y32 = layer.forward(xt, out_dtype=torch.float32).double().cpu().numpy()
    g32 = oracle.gelu(y32)
    tol = 2 ** -8 if odt == torch.bfloat16 else 2 ** -11
    assert np.all(np.abs(y - g32) <= tol * np.abs(g32) + 1e-6), np.abs(y - g32).max()
    codes, s, z = layer.quantize(xt)
    rows = np.sort(rng.choice(M, 128, replace=False))
    wc, sw, _ = layer.export()
    acc_ref = oracle.qlinear_acc(codes.cpu().numpy()[rows], z.cpu().numpy()[rows], wc,
                                 np.full(N, 1 << (wb - 1), np.int32))
    y_ref = oracle.gelu(oracle.qlinear_epilogue(acc_ref, s.cpu().numpy()[rows], sw, bias))
    err = rel_err(y[rows], y_ref)
    assert err <= (4e-3 if odt == torch.bfloat16 else REL_TOL), err
    with pytest.raises(dtq.DtqError):
        layer.forward(xt, out_dtype=torch.float32, activation=dtq.ACT_GELU)  # F16 / BF16 only
