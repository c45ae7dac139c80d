"""Pins the C restatement (oracle/dtq_oracle.c) before it is trusted.

1. against the golden vectors produced by the UNMODIFIED reference
   (tests/golden/make_golden.py), which travel to the GPU box;
2. against the reference library itself (oracle/_ref/libdtq_ref.so) on
   fresh seeded inputs, where that library was built;
3. against the known answers hard-coded in the reference unit tests
   (proj/tests/test_quant.cpp, test_balance.cpp, test_qgemm.cpp).
"""
import numpy as np
import pytest


def f64(a):
    return np.asarray(a, dtype=np.float64)


# ---------------------------------------------------------------- known answers
def test_known_answers_minmax(oracle, golden):
    # test_quant.cpp:31-37 / :39-45 / :47-56
    assert oracle.minmax_params(np.arange(16.0), 4) == (1.0, 0)
    s, z = oracle.minmax_params([-1.0, 1.0], 8)
    assert s == 2.0 / 255.0 and z == 128
    assert oracle.minmax_params([5.0, 5.0, 5.0], 8) == (1.0, 0)
    for name in ("ka_grid", "ka_pm1", "ka_const"):
        s, z = oracle.minmax_params(golden[f"{name}_in"], int(golden[f"{name}_bits"]))
        assert s == golden[f"{name}_s"] and z == golden[f"{name}_z"]


def test_known_answers_symmetric_and_rounding(oracle):
    # test_quant.cpp:245-258: z = 128, s = 3/127
    s, z = oracle.symmetric_params([-3.0, 1.0, 2.0], 8)
    assert z == 128 and s == 3.0 / 127.0
    # test_quant.cpp:65-75: 7.3 -> 7, 20 -> 15 at s=1 z=0 b=4
    codes = oracle.quantize_rows_static(np.array([[7.3], [20.0]]), [1.0, 1.0], [0, 0], 4)
    assert codes.ravel().tolist() == [7, 15]
    # half-to-even ties
    assert [oracle.round_even(v) for v in (0.5, 1.5, 2.5, -0.5, -1.5, 2.4999)] == \
        [0.0, 2.0, 2.0, -0.0, -2.0, 2.0]


def test_known_answers_balance(oracle):
    # test_balance.cpp:116-123: one-hot spreads to 1/4 at n=16
    e1 = np.zeros((1, 16)); e1[0, 0] = 1.0
    r = oracle.rotate_blocks(e1, np.ones(16, np.int8), 16)
    assert np.allclose(np.abs(r), 0.25)
    # test_balance.cpp:87-95: n=2 Sylvester
    r = oracle.rotate_blocks(np.eye(2), np.ones(2, np.int8), 2)
    assert np.allclose(r, np.array([[1, 1], [1, -1]]) / np.sqrt(2))
    # test_balance.cpp:97-101: non power of two rejected
    with pytest.raises(ValueError):
        oracle.rotate_blocks(np.ones((1, 3)), np.ones(3, np.int8), 3)
    # test_balance.cpp:30-41 mask formula + clamps
    assert np.allclose(oracle.scaling_mask([4.0], [1.0], 0.5), [2.0])
    s = oracle.scaling_mask([0.0, 1e30], [1.0, 1e-30], 0.5)
    assert s[0] == 1.0 and s[1] == 1e5


def test_mt19937_64_is_the_standard_engine(oracle):
    # [rand.predef]: 10000th output of a default-constructed mt19937_64
    assert oracle.mt19937_64_nth(5489, 10000) == 9981545732273789042


def test_known_answer_scalar_product(oracle):
    # test_qgemm.cpp:30-43: x=1.0 (constant group -> s=1, z=0 -> code 1?) ...
    # code 131 at z_w=128, s_w=0.1 -> 0.3
    y = oracle.qlinear_forward(np.array([[1.0]]), np.array([[131]], np.uint8), [0.1], [128], 8)
    assert abs(y[0, 0] - 0.3) < 1e-6


def test_zero_rows_give_bias(oracle, golden):
    # test_qgemm.cpp:45-54
    wc, sw, zw = oracle.make_quant_linear(f64(golden["w"][:4, :8]), 8)
    bias = np.array([1.0, -2.0, 0.5, 3.0])
    y = oracle.qlinear_forward(np.zeros((2, 8)), wc, sw, zw, 8, bias)
    assert np.allclose(y, bias[None, :])


# ---------------------------------------------------------------- golden vectors
def test_golden_quantizer(oracle, golden):
    x = f64(golden["q_x"])
    codes, s, z = oracle.quantize_rows(x, 8)
    assert np.array_equal(codes, golden["q_codes"])
    assert np.array_equal(s, golden["q_s"]) and np.array_equal(z, golden["q_z"])
    for bits in (2, 4, 6):
        c, s_, z_ = oracle.quantize_rows(x, bits)
        assert np.array_equal(c, golden[f"q{bits}_codes"])
        assert np.array_equal(s_, golden[f"q{bits}_s"]) and np.array_equal(z_, golden[f"q{bits}_z"])


@pytest.mark.parametrize("wb", [8, 4])
def test_golden_qlinear(oracle, golden, wb):
    w = f64(golden["w"])
    wc, sw, zw = oracle.make_quant_linear(w, wb)
    assert np.array_equal(wc, golden[f"w{wb}_codes"])
    assert np.array_equal(sw, golden[f"w{wb}_s"]) and np.array_equal(zw, golden[f"w{wb}_z"])
    y = oracle.qlinear_forward(f64(golden["q_x"]), wc, sw, zw, wb, golden["bias"])
    assert np.array_equal(y, golden[f"w{wb}_y"])          # bit-exact fp64
    y = oracle.qlinear_forward(f64(golden["q_x"]), wc, sw, zw, wb, None)
    assert np.array_equal(y, golden[f"w{wb}_y_nobias"])


def test_golden_w4_packing(oracle, golden):
    packed = oracle.pack_codes(golden["w4_codes"], 4)
    assert np.array_equal(packed, golden["w4_packed"])
    back = oracle.unpack_codes(packed, 4, golden["w4_codes"].size)
    assert np.array_equal(back.reshape(golden["w4_codes"].shape), golden["w4_codes"])


def test_golden_balance(oracle, golden):
    x = f64(golden["q_x"])
    w = f64(golden["w"])
    signs = oracle.hadamard_signs(x.shape[1], 7)
    assert np.array_equal(signs, golden["bal_signs"])
    xr = oracle.rotate_blocks(oracle.scale_x(x, golden["bal_smooth"]), signs, 128)
    c, s, z = oracle.quantize_rows(xr, 8)
    assert np.array_equal(c, golden["bal_codes"])
    assert np.array_equal(s, golden["bal_s"]) and np.array_equal(z, golden["bal_z"])
    wr = oracle.rotate_blocks(oracle.scale_w(w, golden["bal_smooth"]), signs, 128)
    wc, sw, zw = oracle.make_quant_linear(wr, 8)
    assert np.array_equal(wc, golden["bal_wcodes"])
    y = oracle.qlinear_forward(xr, wc, sw, zw, 8, golden["bias"])
    assert np.array_equal(y, golden["bal_y"])
    c, s, z = oracle.quantize_rows(oracle.rotate_blocks(x, signs, 128), 8)
    assert np.array_equal(c, golden["rot_codes"]) and np.array_equal(s, golden["rot_s"])


@pytest.mark.parametrize("i", [0, 1, 2])
def test_golden_ragged(oracle, golden, i):
    x, w = f64(golden[f"rag{i}_x"]), f64(golden[f"rag{i}_w"])
    wc, sw, zw = oracle.make_quant_linear(w, 8)
    assert np.array_equal(wc, golden[f"rag{i}_wc"])
    y = oracle.qlinear_forward(x, wc, sw, zw, 8, golden[f"rag{i}_b"])
    assert np.array_equal(y, golden[f"rag{i}_y"])


# ---------------------------------------------------------------- vs the reference library
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_against_reference_library(oracle, reference, seed):
    rng = np.random.default_rng(seed)
    M, K, N = 1 + seed * 17, 256 + 128 * seed, 3 + 40 * seed
    x = (rng.standard_normal((M, K)) * (1 + seed)).astype(np.float16).astype(np.float64)
    w = rng.standard_normal((N, K))
    for bits in (8, 4):
        a, b = oracle.quantize_rows(x, bits), reference.quantize_rows(x, bits)
        assert all(np.array_equal(p, q) for p, q in zip(a, b))
        wo, wr = oracle.make_quant_linear(w, bits), reference.make_quant_linear(w, bits)
        assert all(np.array_equal(p, q) for p, q in zip(wo, wr))
        bias = rng.standard_normal(N)
        yo = oracle.qlinear_forward(x, *wo, bits, bias)
        yr = reference.qlinear_forward(x, *wr, bits, bias, threads=2)
        assert np.array_equal(yo, yr)
    signs = oracle.hadamard_signs(K, seed + 3)
    assert np.array_equal(signs, reference.hadamard_signs(K, seed + 3))
    assert np.array_equal(oracle.rotate_blocks(x, signs, 128), reference.rotate_blocks(x, signs, 128))
    assert np.array_equal(oracle.rotate_blocks(x, signs, K) if (K & (K - 1)) == 0 else x,
                          reference.rotate_blocks(x, signs, K) if (K & (K - 1)) == 0 else x)


def test_int_path_matches_float_path(oracle, reference):
    # acceptance.cpp:241-270 / test_qgemm.cpp:56-77: int path == float path within 1e-3
    rng = np.random.default_rng(3)
    for trial in range(20):
        n, c_in, c_out = 1 + rng.integers(64), 1 + rng.integers(128), 1 + rng.integers(64)
        wb = 8 if trial % 2 == 0 else 4
        x = rng.standard_normal((n, c_in)) * (1 + trial % 4)
        w = rng.standard_normal((c_out, c_in))
        wc, sw, zw = oracle.make_quant_linear(w, wb)
        yi = oracle.qlinear_forward(x, wc, sw, zw, wb)
        yf = reference.qlinear_forward_float(x, wc, sw, zw, wb)
        assert np.abs(yi - yf).max() / max(np.abs(yf).max(), 1.0) <= 1e-3


def test_overflow_guard(oracle):
    # qgemm.cpp:29-34: int64 bound is never hit at realistic sizes
    assert oracle.overflow_guard(8, 8, 1 << 40) == 0
    assert oracle.overflow_guard(8, 8, 1 << 50) == 2


def test_layernorm_pinned_to_torch(oracle):
    # the reference has no LayerNorm: the oracle's restatement (used as the
    # checker of the LN-modulate prologue) is pinned against PyTorch's
    # F.layer_norm in fp64 -- biased variance, eps inside the sqrt
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(17)
    x = rng.standard_normal((64, 1152)) * np.exp(rng.standard_normal(1152)) + 3.0
    x[0] = 7.25                      # constant row: 0 / sqrt(eps)
    x[1, :] = rng.standard_normal(1152) * 1e-4 + 1e4  # large offset, tiny spread
    for eps in (1e-6, 1e-5):
        got = oracle.layernorm(x, eps)
        want = torch.nn.functional.layer_norm(torch.from_numpy(x), (1152,), eps=eps).numpy()
        d = np.abs(got - want).max(axis=1)
        # row 1 is ill-conditioned (offset / spread = 1e8): both sums cancel
        # ~1e4 * 2^-52 / 1e-4 ~ 2e-8 of a unit value; every other row agrees
        # to rounding
        assert d[1] <= 1e-7 and np.delete(d, 1).max() <= 1e-12, d.max()
