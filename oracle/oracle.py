"""numpy front-end for the parity checkers (TEST INFRASTRUCTURE ONLY).

`Oracle` wraps oracle/liboracle.so (the C restatement, dtq_oracle.c) and
`Reference` wraps oracle/_ref/libdtq_ref.so (the unmodified reference
library compiled from /root/reference/proj/core/src by oracle/Makefile).
Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this
module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libdtq_ref.so")

_p = C.c_void_p
_i64 = C.c_int64
_int = C.c_int
_dbl = C.c_double


def _ptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"], "arrays must be C-contiguous"
    return a.ctypes.data_as(_p)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


class OracleError(RuntimeError):
    pass


def _check(st: int, what: str):
    if st == 1:
        raise ValueError(f"{what}: invalid argument")
    if st == 2:
        raise OverflowError(f"{what}: accumulator could overflow")
    if st != 0:
        raise OracleError(f"{what}: status {st}")


class Oracle:
    """C restatement of the reference path (dtq_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        L = self.lib = C.CDLL(path)
        L.dtq_oracle_round_even.restype = _dbl
        L.dtq_oracle_round_even.argtypes = [_dbl]
        L.dtq_oracle_mt19937_64_nth.restype = C.c_uint64
        L.dtq_oracle_mt19937_64_nth.argtypes = [C.c_uint64, _i64]
        L.dtq_oracle_pack_codes.restype = _i64
        L.dtq_oracle_num_cpus.restype = _int
        for name in ("minmax_params", "symmetric_params"):
            getattr(L, f"dtq_oracle_{name}").argtypes = [_p, _i64, _int, _p, _p]
        L.dtq_oracle_quantize_rows.argtypes = [_p, _i64, _i64, _int, _int, _p, _p, _p]
        L.dtq_oracle_quantize_rows_static.argtypes = [_p, _i64, _i64, _int, _p, _p, _p]
        L.dtq_oracle_dequantize_rows.argtypes = [_p, _i64, _i64, _p, _p, _p]
        L.dtq_oracle_fwht.argtypes = [_p, _i64]
        L.dtq_oracle_hadamard_signs.argtypes = [_i64, _int, C.c_uint64, _p]
        L.dtq_oracle_rotate_blocks.argtypes = [_p, _i64, _i64, _i64, _p]
        L.dtq_oracle_scaling_mask.argtypes = [_p, _p, _i64, _dbl, _p]
        L.dtq_oracle_scale_x.argtypes = [_p, _i64, _i64, _p]
        L.dtq_oracle_scale_w.argtypes = [_p, _i64, _i64, _p]
        L.dtq_oracle_modulate.argtypes = [_p, _i64, _i64, _p, _p]
        L.dtq_oracle_gelu.argtypes = [_p, _i64]
        L.dtq_oracle_layernorm.argtypes = [_p, _i64, _i64, _dbl]
        L.dtq_oracle_overflow_guard.argtypes = [_int, _int, _i64]
        L.dtq_oracle_qlinear_acc.argtypes = [_p, _p, _i64, _i64, _p, _p, _i64, _p, _int]
        L.dtq_oracle_qlinear_epilogue.argtypes = [_p, _p, _i64, _p, _p, _i64, _p]
        L.dtq_oracle_qlinear_forward.argtypes = [_p, _i64, _i64, _int, _p, _p, _p, _int, _i64,
                                                 _p, _p, _int]
        L.dtq_oracle_pack_codes.argtypes = [_p, _i64, _int, _p]
        L.dtq_oracle_unpack_codes.argtypes = [_p, _i64, _int, _i64, _p]

    # quant.cpp -----------------------------------------------------------
    def round_even(self, v: float) -> float:
        return self.lib.dtq_oracle_round_even(float(v))

    def minmax_params(self, g, bits: int):
        g = _f64(g)
        s, z = np.zeros(1), np.zeros(1, np.int32)
        _check(self.lib.dtq_oracle_minmax_params(_ptr(g), g.size, bits, _ptr(s), _ptr(z)),
               "minmax_params")
        return float(s[0]), int(z[0])

    def symmetric_params(self, g, bits: int):
        g = _f64(g)
        s, z = np.zeros(1), np.zeros(1, np.int32)
        _check(self.lib.dtq_oracle_symmetric_params(_ptr(g), g.size, bits, _ptr(s), _ptr(z)),
               "symmetric_params")
        return float(s[0]), int(z[0])

    def quantize_rows(self, x, bits: int = 8, symmetric: bool = False):
        """quantize(x, per_token | per_output_channel, bits, Dynamic)."""
        x = _f64(x)
        M, K = x.shape
        codes = np.zeros((M, K), np.uint8)
        s, z = np.zeros(M), np.zeros(M, np.int32)
        _check(self.lib.dtq_oracle_quantize_rows(_ptr(x), M, K, bits, int(symmetric),
                                                 _ptr(codes), _ptr(s), _ptr(z)), "quantize")
        return codes, s, z

    def quantize_rows_static(self, x, s, z, bits: int = 8):
        x, s = _f64(x), _f64(s)
        z = np.ascontiguousarray(z, np.int32)
        M, K = x.shape
        codes = np.zeros((M, K), np.uint8)
        _check(self.lib.dtq_oracle_quantize_rows_static(_ptr(x), M, K, bits, _ptr(s), _ptr(z),
                                                        _ptr(codes)), "quantize_static")
        return codes

    def dequantize_rows(self, codes, s, z):
        codes = np.ascontiguousarray(codes, np.uint8)
        s, z = _f64(s), np.ascontiguousarray(z, np.int32)
        out = np.zeros(codes.shape)
        self.lib.dtq_oracle_dequantize_rows(_ptr(codes), codes.shape[0], codes.shape[1],
                                            _ptr(s), _ptr(z), _ptr(out))
        return out

    # balance.cpp ---------------------------------------------------------
    def hadamard_signs(self, n: int, seed: int, randomize: bool = True):
        out = np.zeros(n, np.int8)
        self.lib.dtq_oracle_hadamard_signs(n, int(randomize), seed, _ptr(out))
        return out

    def mt19937_64_nth(self, seed: int, n: int) -> int:
        return int(self.lib.dtq_oracle_mt19937_64_nth(seed, n))

    def fwht(self, v):
        v = _f64(v).copy()
        _check(self.lib.dtq_oracle_fwht(_ptr(v), v.size), "fwht")
        return v

    def rotate_blocks(self, x, signs, hblock: int = 128):
        x = _f64(x).copy()
        signs = np.ascontiguousarray(signs, np.int8)
        _check(self.lib.dtq_oracle_rotate_blocks(_ptr(x), x.shape[0], x.shape[1], hblock,
                                                 _ptr(signs)), "rotate_blocks")
        return x

    def scaling_mask(self, act_amax, w_amax, alpha: float):
        a, w = _f64(act_amax), _f64(w_amax)
        s = np.zeros(a.size)
        _check(self.lib.dtq_oracle_scaling_mask(_ptr(a), _ptr(w), a.size, alpha, _ptr(s)),
               "scaling_mask")
        return s

    def scale_x(self, x, s):
        x = _f64(x).copy()
        self.lib.dtq_oracle_scale_x(_ptr(x), x.shape[0], x.shape[1], _ptr(_f64(s)))
        return x

    def scale_w(self, w, s):
        w = _f64(w).copy()
        self.lib.dtq_oracle_scale_w(_ptr(w), w.shape[0], w.shape[1], _ptr(_f64(s)))
        return w

    def modulate(self, x, scale, shift):
        x = _f64(x).copy()
        self.lib.dtq_oracle_modulate(_ptr(x), x.shape[0], x.shape[1], _ptr(_f64(scale)),
                                     _ptr(_f64(shift)))
        return x

    def gelu(self, x):
        x = _f64(x).copy()
        self.lib.dtq_oracle_gelu(_ptr(x), x.size)
        return x

    def layernorm(self, x, eps: float = 1e-6):
        """Row LayerNorm, no affine (no reference counterpart; pinned against
        torch.nn.functional.layer_norm in fp64)."""
        x = _f64(x).copy()
        self.lib.dtq_oracle_layernorm(_ptr(x), x.shape[0], x.shape[1], float(eps))
        return x

    # qgemm.cpp -----------------------------------------------------------
    def make_quant_linear(self, w, wbits: int):
        """make_quant_linear (qgemm.cpp:9-21): symmetric per-out-channel."""
        return self.quantize_rows(w, wbits, symmetric=True)

    def qlinear_acc(self, xc, zx, wc, zw, threads: int = 0):
        xc = np.ascontiguousarray(xc, np.uint8)
        wc = np.ascontiguousarray(wc, np.uint8)
        zx = np.ascontiguousarray(zx, np.int32)
        zw = np.ascontiguousarray(zw, np.int32)
        M, K = xc.shape
        N = wc.shape[0]
        acc = np.zeros((M, N), np.int64)
        _check(self.lib.dtq_oracle_qlinear_acc(_ptr(xc), _ptr(zx), M, K, _ptr(wc), _ptr(zw), N,
                                               _ptr(acc), threads), "qlinear_acc")
        return acc

    def qlinear_epilogue(self, acc, sx, sw, bias=None):
        acc = np.ascontiguousarray(acc, np.int64)
        M, N = acc.shape
        y = np.zeros((M, N))
        self.lib.dtq_oracle_qlinear_epilogue(_ptr(acc), _ptr(_f64(sx)), M, _ptr(_f64(sw)),
                                             _ptr(None if bias is None else _f64(bias)), N,
                                             _ptr(y))
        return y

    def qlinear_forward(self, x, wc, sw, zw, wbits: int, bias=None, act_bits: int = 8,
                        threads: int = 0):
        x = _f64(x)
        M, K = x.shape
        wc = np.ascontiguousarray(wc, np.uint8)
        N = wc.shape[0]
        y = np.zeros((M, N))
        b = None if bias is None else _f64(bias)
        _check(self.lib.dtq_oracle_qlinear_forward(
            _ptr(x), M, K, act_bits, _ptr(wc), _ptr(_f64(sw)),
            _ptr(np.ascontiguousarray(zw, np.int32)), wbits, N, _ptr(b), _ptr(y), threads),
            "qlinear_forward")
        return y

    def overflow_guard(self, act_bits: int, wbits: int, c_in: int) -> int:
        return self.lib.dtq_oracle_overflow_guard(act_bits, wbits, c_in)

    # trace_io.cpp --------------------------------------------------------
    def pack_codes(self, codes, bits: int):
        codes = np.ascontiguousarray(codes, np.uint8).ravel()
        out = np.zeros((codes.size * bits + 7) // 8, np.uint8)
        n = self.lib.dtq_oracle_pack_codes(_ptr(codes), codes.size, bits, _ptr(out))
        if n < 0:
            raise ValueError("pack_codes: bad bits or code out of range")
        return out

    def unpack_codes(self, packed, bits: int, count: int):
        packed = np.ascontiguousarray(packed, np.uint8)
        out = np.zeros(count, np.uint8)
        _check(self.lib.dtq_oracle_unpack_codes(_ptr(packed), packed.size, bits, count,
                                                _ptr(out)), "unpack_codes")
        return out

    def num_cpus(self) -> int:
        return int(self.lib.dtq_oracle_num_cpus())


class Reference:
    """The unmodified reference library (oracle/_ref/libdtq_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where "
                                    "/root/reference exists")
        L = self.lib = C.CDLL(path)
        L.dtq_ref_round_even.restype = _dbl
        L.dtq_ref_round_even.argtypes = [_dbl]
        L.dtq_ref_quantize_rows.argtypes = [_p, _i64, _i64, _int, _int, _p, _p, _p]
        L.dtq_ref_minmax_params.argtypes = [_p, _i64, _int, _p, _p]
        L.dtq_ref_make_quant_linear.argtypes = [_p, _i64, _i64, _int, _int, _p, _p, _p]
        L.dtq_ref_qlinear_forward.argtypes = [_p, _i64, _i64, _p, _p, _p, _int, _i64, _p, _int,
                                              _p, _int]
        L.dtq_ref_qlinear_forward_float.argtypes = [_p, _i64, _i64, _p, _p, _p, _int, _i64, _p,
                                                    _int, _p]
        L.dtq_ref_hadamard_signs.argtypes = [_i64, _int, C.c_uint64, _p]
        L.dtq_ref_rotate_blocks.argtypes = [_p, _i64, _i64, _i64, _p]
        L.dtq_ref_scaling_mask.argtypes = [_p, _p, _i64, _dbl, _p]
        L.dtq_ref_apply_scaling.argtypes = [_p, _i64, _p, _i64, _i64, _p]
        L.dtq_ref_pack_codes.restype = _i64
        L.dtq_ref_pack_codes.argtypes = [_p, _i64, _int, _p]
        L.dtq_ref_write_checkpoint.argtypes = [C.c_char_p, _int, _p, _p, _p, _p, _p, _p, _p]
        L.dtq_ref_read_checkpoint_layer.argtypes = [C.c_char_p, _i64, _p, _p, _p, _p]

    def round_even(self, v: float) -> float:
        return self.lib.dtq_ref_round_even(float(v))

    def write_checkpoint(self, path: str, layers):
        """layers: list of (name, W [N,K] f64, bits, mask [K] f32 or None,
        rot [K] +-1 int8 or None) -> the reference's write_checkpoint."""
        n = len(layers)
        keep = []
        names = (C.c_char_p * n)(*[l[0].encode() for l in layers])
        ws = (C.c_void_p * n)()
        Ns = np.zeros(n, np.int64)
        Ks = np.zeros(n, np.int64)
        bits = np.zeros(n, np.int32)
        masks = (C.c_void_p * n)()
        rots = (C.c_void_p * n)()
        for i, (_, w, b, mask, rot) in enumerate(layers):
            w = _f64(w)
            keep.append(w)
            ws[i] = w.ctypes.data
            Ns[i], Ks[i] = w.shape
            bits[i] = b
            if mask is not None:
                m = np.ascontiguousarray(mask, np.float32)
                keep.append(m)
                masks[i] = m.ctypes.data
            if rot is not None:
                r = np.ascontiguousarray(rot, np.int8)
                keep.append(r)
                rots[i] = r.ctypes.data
        st = self.lib.dtq_ref_write_checkpoint(path.encode(), n, names, ws, Ns.ctypes.data,
                                               Ks.ctypes.data, bits.ctypes.data, masks, rots)
        if st:
            raise RuntimeError(f"reference write_checkpoint failed ({st})")

    def read_checkpoint_layer(self, path: str, i: int, N: int, K: int):
        codes = np.zeros((N, K), np.uint8)
        scale = np.zeros(N, np.float64)
        zero = np.zeros(N, np.int32)
        n = C.c_int64(0)
        st = self.lib.dtq_ref_read_checkpoint_layer(path.encode(), i, codes.ctypes.data,
                                                    scale.ctypes.data, zero.ctypes.data,
                                                    C.byref(n))
        if st:
            raise RuntimeError(f"reference read_checkpoint failed ({st})")
        return codes, scale, zero

    def quantize_rows(self, x, bits: int = 8, symmetric: bool = False):
        x = _f64(x)
        M, K = x.shape
        codes = np.zeros((M, K), np.uint8)
        s, z = np.zeros(M), np.zeros(M, np.int32)
        _check(self.lib.dtq_ref_quantize_rows(_ptr(x), M, K, bits, int(symmetric), _ptr(codes),
                                              _ptr(s), _ptr(z)), "ref quantize")
        return codes, s, z

    def minmax_params(self, g, bits: int):
        g = _f64(g)
        s, z = np.zeros(1), np.zeros(1, np.int32)
        _check(self.lib.dtq_ref_minmax_params(_ptr(g), g.size, bits, _ptr(s), _ptr(z)),
               "ref minmax_params")
        return float(s[0]), int(z[0])

    def make_quant_linear(self, w, wbits: int, act_bits: int = 8):
        w = _f64(w)
        N, K = w.shape
        codes = np.zeros((N, K), np.uint8)
        s, z = np.zeros(N), np.zeros(N, np.int32)
        _check(self.lib.dtq_ref_make_quant_linear(_ptr(w), N, K, wbits, act_bits, _ptr(codes),
                                                  _ptr(s), _ptr(z)), "ref make_quant_linear")
        return codes, s, z

    def qlinear_forward(self, x, wc, sw, zw, wbits: int, bias=None, act_bits: int = 8,
                        threads: int = 1):
        x = _f64(x)
        M, K = x.shape
        wc = np.ascontiguousarray(wc, np.uint8)
        N = wc.shape[0]
        y = np.zeros((M, N))
        b = None if bias is None else _f64(bias)
        _check(self.lib.dtq_ref_qlinear_forward(
            _ptr(x), M, K, _ptr(wc), _ptr(_f64(sw)), _ptr(np.ascontiguousarray(zw, np.int32)),
            wbits, N, _ptr(b), act_bits, _ptr(y), threads), "ref qlinear_forward")
        return y

    def qlinear_forward_float(self, x, wc, sw, zw, wbits: int, bias=None, act_bits: int = 8):
        x = _f64(x)
        M, K = x.shape
        wc = np.ascontiguousarray(wc, np.uint8)
        N = wc.shape[0]
        y = np.zeros((M, N))
        b = None if bias is None else _f64(bias)
        _check(self.lib.dtq_ref_qlinear_forward_float(
            _ptr(x), M, K, _ptr(wc), _ptr(_f64(sw)), _ptr(np.ascontiguousarray(zw, np.int32)),
            wbits, N, _ptr(b), act_bits, _ptr(y)), "ref qlinear_forward_float")
        return y

    def hadamard_signs(self, n: int, seed: int, randomize: bool = True):
        """First n sign draws of hadamard_matrix (balance.cpp:69-80).

        The reference only accepts power-of-two n; the blockwise rotation
         uses the first K draws of the same engine, which
        are the leading entries of hadamard_matrix(next_pow2(K)).sign_diag."""
        n2 = 2
        while n2 < n:
            n2 *= 2
        out = np.zeros(n2, np.int8)
        _check(self.lib.dtq_ref_hadamard_signs(n2, int(randomize), seed, _ptr(out)),
               "ref hadamard_matrix")
        return out[:n].copy()

    def rotate_blocks(self, x, signs, hblock: int = 128):
        x = _f64(x).copy()
        signs = np.ascontiguousarray(signs, np.int8)
        _check(self.lib.dtq_ref_rotate_blocks(_ptr(x), x.shape[0], x.shape[1], hblock,
                                              _ptr(signs)), "ref rotate_channels")
        return x

    def scaling_mask(self, act_amax, w_amax, alpha: float):
        a, w = _f64(act_amax), _f64(w_amax)
        s = np.zeros(a.size)
        _check(self.lib.dtq_ref_scaling_mask(_ptr(a), _ptr(w), a.size, alpha, _ptr(s)),
               "ref compute_scaling_mask")
        return s

    def apply_scaling(self, x, w, s):
        x, w = _f64(x).copy(), _f64(w).copy()
        _check(self.lib.dtq_ref_apply_scaling(_ptr(x), x.shape[0], _ptr(w), w.shape[0],
                                              x.shape[1], _ptr(_f64(s))), "ref apply_scaling")
        return x, w

    def pack_codes(self, codes, bits: int):
        codes = np.ascontiguousarray(codes, np.uint8).ravel()
        out = np.zeros((codes.size * bits + 7) // 8, np.uint8)
        n = self.lib.dtq_ref_pack_codes(_ptr(codes), codes.size, bits, _ptr(out))
        if n < 0:
            raise ValueError("ref pack_codes failed")
        return out


def reference_available() -> bool:
    return os.path.exists(REF_SO)
