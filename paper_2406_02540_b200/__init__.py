"""B200-native (sm_100a) ViDiT-Q quantized-linear path.

Python front-end over the C ABI in include/dtq_capi.h, implemented by
libdtq_b200.so (built in-tree from csrc/ by `python __graft_entry__.py` or
`make -C paper_2406_02540_b200`).  PyTorch is used only for device memory
and streams; every computation runs in the hand-written CUDA kernels.

The names mirror the reference API (/root/reference/proj/core/include/dtq):

  quantize_rows        quantize(x, per_token | per_output_channel, bits, Dynamic)
  QuantLinear.create   make_quant_linear(w, weight_bits, act_bits, bias)
                       (+ weight side of apply_balance)
  QuantLinear.forward  qlinear_forward(x, layer) with the fused quantizer
  QuantLinear.gemm     the integer GEMM + dequant epilogue on given codes
  Balance              BalanceTransform{mask, rotation} (blockwise Hadamard)

There is no CPU fallback: loading fails loudly without the built library,
and every compute call fails without an sm_100 device.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DTQ_B200_LIB") or os.path.join(HERE, "libdtq_b200.so")  # override: diagnostics builds

F16, BF16, F32, F64, S32 = 0, 1, 2, 3, 4
MODE_FAST, MODE_EXACT = 0, 1
PROLOGUE_NONE, PROLOGUE_MODULATE, PROLOGUE_GELU, PROLOGUE_LN_MODULATE = 0, 1, 2, 3
ACT_NONE, ACT_GELU = 0, 1

DTQ_OK, DTQ_ERR_INVALID_ARGUMENT, DTQ_ERR_OVERFLOW, DTQ_ERR_CUDA, DTQ_ERR_UNSUPPORTED = range(5)

#: every symbol include/dtq_capi.h declares (checked by tests/test_capi.py)
EXPORTED = (
    "dtq_last_error", "dtq_capi_version", "dtq_device_check", "dtq_quantize_rows",
    "dtq_qlinear_create", "dtq_qlinear_create_from_codes", "dtq_qlinear_destroy",
    "dtq_qlinear_info", "dtq_qlinear_export", "dtq_qgemm", "dtq_qlinear_workspace_bytes",
    "dtq_qlinear_forward", "dtq_qlinear_quantize", "dtq_qlinear_forward_host",
    "dtq_quantize_static", "dtq_dequantize", "dtq_balance_apply", "dtq_matmul_nt_f64",
    "dtq_checkpoint_open", "dtq_checkpoint_close", "dtq_checkpoint_num_layers",
    "dtq_checkpoint_layer_info", "dtq_checkpoint_load_layer",
    "dtq_planned_create", "dtq_planned_destroy", "dtq_planned_select", "dtq_planned_bits",
    "dtq_col_absmax_f64", "dtq_row_absmax_f64", "dtq_fwht_f64", "dtq_qlinear_forward_act",
)


class DtqError(RuntimeError):
    """DTQ_ERR_CUDA / DTQ_ERR_UNSUPPORTED."""


class _Prologue(C.Structure):
    _fields_ = [("kind", C.c_int32), ("scale", C.c_void_p), ("shift", C.c_void_p),
                ("eps", C.c_float)]


class _Balance(C.Structure):
    _fields_ = [("smooth", C.c_void_p), ("signs", C.c_void_p), ("hblock", C.c_int32)]


_lib = None


def lib():
    """Load libdtq_b200.so (raises if it was not built: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built; run `python __graft_entry__.py` "
                          "(nvcc, sm_100a).  There is no CPU fallback.")
    L = C.CDLL(LIB_PATH)
    p, i64, i32 = C.c_void_p, C.c_int64, C.c_int
    L.dtq_last_error.restype = C.c_char_p
    L.dtq_quantize_rows.argtypes = [p, i32, i64, i64, i64, i32, i32, i32, p, p, p, i64, p, p, p, p]
    L.dtq_qlinear_create.argtypes = [p, i32, i64, i64, i64, i32, i32, p, p, p, p]
    L.dtq_qlinear_create_from_codes.argtypes = [p, i32, i64, i32, p, i64, i64, i32, p, p, p, p]
    L.dtq_qlinear_destroy.argtypes = [p]
    L.dtq_qlinear_info.argtypes = [p, p, p, p, p]
    L.dtq_qlinear_export.argtypes = [p, p, p, p, p]
    L.dtq_qgemm.argtypes = [p, i64, p, p, i64, p, p, i32, i64, p]
    L.dtq_qlinear_workspace_bytes.restype = C.c_size_t
    L.dtq_qlinear_workspace_bytes.argtypes = [p, i64]
    L.dtq_qlinear_forward.argtypes = [p, i32, i64, i64, p, i32, p, p, i32, i64, p, C.c_size_t, p, p]
    if hasattr(L, "dtq_qlinear_forward_act"):
        L.dtq_qlinear_forward_act.argtypes = [p, i32, i64, i64, p, i32, p, i32, p, i32, i64, p,
                                              C.c_size_t, p, p]
    L.dtq_qlinear_quantize.argtypes = [p, i32, i64, i64, p, i32, p, p, i64, p, p, p, p]
    L.dtq_qlinear_forward_host.argtypes = [p, i32, i64, p, i32, p, i32, p]
    L.dtq_checkpoint_open.argtypes = [C.c_char_p, p]
    L.dtq_checkpoint_close.argtypes = [p]
    L.dtq_checkpoint_num_layers.argtypes = [p, p]
    L.dtq_checkpoint_layer_info.argtypes = [p, i64, p, p, p, p, p, p, p]
    L.dtq_checkpoint_load_layer.argtypes = [p, i64, i32, i32, p, p]
    if hasattr(L, "dtq_planned_create"):  # (an older library via DTQ_B200_LIB lacks them)
        L.dtq_planned_create.argtypes = [p, i32, i64, i64, i64, p, i32, p, p, p, p]
        L.dtq_planned_destroy.argtypes = [p]
        L.dtq_planned_select.argtypes = [p, i64, i64, p]
        L.dtq_planned_bits.argtypes = [p, i32, p]
    _lib = L
    return L


def _check(status: int):
    if status == DTQ_OK:
        return
    msg = lib().dtq_last_error().decode(errors="replace")
    if status == DTQ_ERR_INVALID_ARGUMENT:
        raise ValueError(msg)
    if status == DTQ_ERR_OVERFLOW:
        raise OverflowError(msg)
    raise DtqError(msg)


def _torch():
    import torch
    return torch


_DTYPES = None


def _dtype_code(t) -> int:
    global _DTYPES
    if _DTYPES is None:
        torch = _torch()
        _DTYPES = {torch.float16: F16, torch.bfloat16: BF16, torch.float32: F32,
                   torch.float64: F64, torch.int32: S32}
    return _DTYPES[t]


def _ptr(t) -> Optional[int]:
    return None if t is None else t.data_ptr()


_RAW_STREAM = None


def _stream(stream=None) -> int:
    """The cudaStream_t to launch on: `stream`, else torch's current stream
    of the current device (read without building a Stream object: this runs
    on every call)."""
    global _RAW_STREAM
    if stream is not None:
        return stream.cuda_stream
    torch = _torch()
    if _RAW_STREAM is None:
        _RAW_STREAM = getattr(torch._C, "_cuda_getCurrentRawStream", False)
    if _RAW_STREAM:
        return _RAW_STREAM(torch.cuda.current_device())
    return torch.cuda.current_stream().cuda_stream


@dataclass
class Balance:
    """BalanceTransform (balance.hpp:31-34) on the device.

    smooth: [K] fp64 ScalingMask.s (activations divided, weights multiplied)
    signs:  [K] int8 +-1 RotationMatrix.sign_diag (blockwise, hblock columns)
    """
    smooth: Optional[object] = None
    signs: Optional[object] = None
    hblock: int = 128

    def _c(self) -> _Balance:
        return _Balance(_ptr(self.smooth), _ptr(self.signs), int(self.hblock))


@dataclass
class Prologue:
    """Fused prologue: MODULATE x*(1+scale)+shift (toydit.cpp:339-369),
    GELU (toydit.cpp:83) or LN_MODULATE (LayerNorm then modulate; unpinned)."""
    kind: int = PROLOGUE_NONE
    scale: Optional[object] = None   # [K] fp32 cuda
    shift: Optional[object] = None   # [K] fp32 cuda
    eps: float = 1e-6

    def _c(self) -> _Prologue:
        return _Prologue(self.kind, _ptr(self.scale), _ptr(self.shift), float(self.eps))


def _ref_or_none(obj):
    return None if obj is None else C.byref(obj)


def _check_rows(t, cols: int, what: str, cuda: bool = True):
    """A 2-D row-major tensor with `cols` columns (the reference's
    'X cols != C_in' check, qgemm.cpp:26-27) on the expected side."""
    if t.dim() != 2 or t.shape[1] != cols:
        raise ValueError(f"{what}: expected [rows, {cols}], got {tuple(t.shape)}")
    if t.stride(1) != 1:
        raise ValueError(f"{what}: rows must be contiguous (stride(1) == 1)")
    if bool(t.is_cuda) != cuda:
        raise ValueError(f"{what}: expected a {'CUDA' if cuda else 'host'} tensor")


def _check_out(out, M: int, N: int, what: str, cuda: bool = True):
    if out.dim() != 2 or tuple(out.shape) != (M, N) or out.stride(1) != 1:
        raise ValueError(f"{what}: output must be [{M}, {N}] with contiguous rows, "
                         f"got {tuple(out.shape)} / strides {tuple(out.stride())}")
    if bool(out.is_cuda) != cuda:
        raise ValueError(f"{what}: output on the wrong device")


def quantize_rows(x, bits: int = 8, symmetric: bool = False, mode: int = MODE_FAST,
                  balance: Optional[Balance] = None, prologue: Optional[Prologue] = None,
                  status=None, stream=None):
    """quantize(x, per_token, bits, Dynamic) on a CUDA tensor [rows, cols].

    Returns (codes u8 [rows, cols], scale f64 [rows], zero_point i32 [rows])."""
    torch = _torch()
    if x.dim() != 2:
        raise ValueError("quantize_rows: expected a 2-D tensor")
    _check_rows(x, x.shape[1], "quantize_rows")
    rows, cols = x.shape
    ldc = (cols + 15) // 16 * 16
    codes_buf = torch.empty((rows, ldc), dtype=torch.uint8, device=x.device)
    scale = torch.empty(rows, dtype=torch.float64, device=x.device)
    zero = torch.empty(rows, dtype=torch.int32, device=x.device)
    b = balance._c() if balance is not None else None
    pr = prologue._c() if prologue is not None else None
    _check(lib().dtq_quantize_rows(x.data_ptr(), _dtype_code(x.dtype), rows, cols, x.stride(0),
                                   bits, int(symmetric), mode, _ref_or_none(b), _ref_or_none(pr),
                                   codes_buf.data_ptr(), ldc, scale.data_ptr(), zero.data_ptr(),
                                   _ptr(status), _stream(stream)))
    return codes_buf[:, :cols], scale, zero


class QuantLinear:
    """Device-resident QuantLinear (qgemm.hpp:17-24) behind an opaque handle."""

    def __init__(self, handle: int, N: int, K: int, wbits: int, abits: int, balance=None,
                 owner=None):
        self._h = C.c_void_p(handle)
        self.N, self.K, self.weight_bits, self.act_bits = N, K, wbits, abits
        self.balance = balance
        self._ws = None
        self._owner = owner  # a borrowed handle (PlannedLinear.select) is not destroyed here

    @classmethod
    def create(cls, w, weight_bits: int = 8, act_bits: int = 8, bias=None,
               balance: Optional[Balance] = None, stream=None) -> "QuantLinear":
        """make_quant_linear (qgemm.cpp:9-21) + weight-side balance, on the GPU."""
        torch = _torch()
        assert w.is_cuda and w.dim() == 2 and w.stride(1) == 1
        N, K = w.shape
        bias_t = None if bias is None else torch.as_tensor(bias, dtype=torch.float64,
                                                           device=w.device).contiguous()
        h = C.c_void_p()
        b = balance._c() if balance is not None else None
        _check(lib().dtq_qlinear_create(w.data_ptr(), _dtype_code(w.dtype), N, K, w.stride(0),
                                        weight_bits, act_bits, _ptr(bias_t), _ref_or_none(b),
                                        _stream(stream), C.byref(h)))
        return cls(h.value, N, K, weight_bits, act_bits, balance)

    @classmethod
    def from_codes(cls, codes, scale, weight_bits: int, K: int, act_bits: int = 8, bias=None,
                   packed: bool = False, balance: Optional[Balance] = None, stream=None):
        """Build from reference codes (checkpoint loader path, trace_io.cpp:263-316)."""
        torch = _torch()
        N = scale.shape[0]
        bias_t = None if bias is None else torch.as_tensor(bias, dtype=torch.float64,
                                                           device=codes.device).contiguous()
        ld = 0 if packed else codes.stride(0)
        h = C.c_void_p()
        b = balance._c() if balance is not None else None
        _check(lib().dtq_qlinear_create_from_codes(codes.data_ptr(), int(packed), ld, weight_bits,
                                                   scale.data_ptr(), N, K, act_bits, _ptr(bias_t),
                                                   _ref_or_none(b), _stream(stream), C.byref(h)))
        return cls(h.value, N, K, weight_bits, act_bits, balance)

    def close(self):
        if self._h is not None and self._h.value and self._owner is None:
            lib().dtq_qlinear_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def export(self):
        """(codes u8 [N,K], scale f64 [N], wsum i32 [N]) as numpy, reference convention."""
        import numpy as np
        codes = np.zeros((self.N, self.K), np.uint8)
        scale = np.zeros(self.N, np.float64)
        wsum = np.zeros(self.N, np.int32)
        _check(lib().dtq_qlinear_export(self._h, codes.ctypes.data, scale.ctypes.data,
                                        wsum.ctypes.data, _stream(None)))
        return codes, scale, wsum

    def workspace(self, M: int, device=None):
        """A forward workspace for up to M rows (zeroed: its row-flag
        counters must start at zero; every forward leaves them zero)."""
        torch = _torch()
        n = lib().dtq_qlinear_workspace_bytes(self._h, M)
        return torch.zeros(n, dtype=torch.uint8, device=device or "cuda")

    def gemm(self, codes, s_x, z_x, out_dtype=None, out=None, stream=None):
        """Integer GEMM + epilogue on quantized activations (qgemm.cpp:52-63)."""
        torch = _torch()
        _check_rows(codes, self.K, "gemm codes")
        if codes.dtype != torch.uint8:
            raise ValueError("gemm: codes must be uint8")
        M = codes.shape[0]
        if s_x.numel() < M or z_x.numel() < M or s_x.dtype != torch.float64 or \
                z_x.dtype != torch.int32 or not (s_x.is_cuda and z_x.is_cuda):
            raise ValueError("gemm: s_x (f64) and z_x (i32) need M entries on the device")
        if out is None:
            out = torch.empty((M, self.N), dtype=out_dtype or torch.float16, device=codes.device)
        _check_out(out, M, self.N, "gemm")
        _check(lib().dtq_qgemm(codes.data_ptr(), codes.stride(0), s_x.data_ptr(), z_x.data_ptr(),
                               M, self._h, out.data_ptr(), _dtype_code(out.dtype), out.stride(0),
                               _stream(stream)))
        return out

    def quantize(self, x, mode: int = MODE_FAST, prologue: Optional[Prologue] = None,
                 out=None, status=None, stream=None):
        """The fused-quantizer stage of forward(): (codes, s_x, z_x)."""
        torch = _torch()
        _check_rows(x, self.K, "quantize")
        M = x.shape[0]
        if out is None:
            ldc = (self.K + 15) // 16 * 16
            buf = torch.empty((M, ldc), dtype=torch.uint8, device=x.device)
            out = (buf[:, :self.K], torch.empty(M, dtype=torch.float64, device=x.device),
                   torch.empty(M, dtype=torch.int32, device=x.device))
        codes, s, z = out
        _check_out(codes, M, self.K, "quantize codes")
        if s.numel() < M or z.numel() < M:
            raise ValueError("quantize: s / z need M entries")
        pr = prologue._c() if prologue is not None else None
        _check(lib().dtq_qlinear_quantize(x.data_ptr(), _dtype_code(x.dtype), M, x.stride(0),
                                          self._h, mode, _ref_or_none(pr), codes.data_ptr(),
                                          codes.stride(0), s.data_ptr(), z.data_ptr(),
                                          _ptr(status), _stream(stream)))
        return codes, s, z

    def forward(self, x, out_dtype=None, mode: int = MODE_FAST,
                prologue: Optional[Prologue] = None, out=None, workspace=None, status=None,
                stream=None, activation: int = ACT_NONE):
        """qlinear_forward(x, layer): fused quantizer + GEMM, stream-ordered;
        `activation=ACT_GELU` applies GELU to y in the GEMM's epilogue."""
        torch = _torch()
        _check_rows(x, self.K, "qlinear_forward")
        M = x.shape[0]
        if out is None:
            out = torch.empty((M, self.N), dtype=out_dtype or torch.float16, device=x.device)
        _check_out(out, M, self.N, "qlinear_forward")
        pr = prologue._c() if prologue is not None else None
        if workspace is not None and (workspace.dtype != torch.uint8 or not workspace.is_cuda
                                      or not workspace.is_contiguous()):
            raise ValueError("qlinear_forward: workspace must be a contiguous uint8 CUDA tensor")
        ws_ptr, ws_n = (None, 0) if workspace is None else (workspace.data_ptr(), workspace.numel())
        if activation != ACT_NONE:
            _check(lib().dtq_qlinear_forward_act(x.data_ptr(), _dtype_code(x.dtype), M, x.stride(0),
                                                 self._h, mode, _ref_or_none(pr), activation,
                                                 out.data_ptr(), _dtype_code(out.dtype),
                                                 out.stride(0), ws_ptr, ws_n, _ptr(status),
                                                 _stream(stream)))
            return out
        _check(lib().dtq_qlinear_forward(x.data_ptr(), _dtype_code(x.dtype), M, x.stride(0),
                                         self._h, mode, _ref_or_none(pr), out.data_ptr(),
                                         _dtype_code(out.dtype), out.stride(0), ws_ptr, ws_n,
                                         _ptr(status), _stream(stream)))
        return out

    def forward_host(self, x_host, y_host, mode: int = MODE_FAST, stream=None):
        """Host buffers in, host buffers out (H2D + forward + D2H, synchronised)."""
        _check_rows(x_host, self.K, "forward_host", cuda=False)
        M = x_host.shape[0]
        _check_out(y_host, M, self.N, "forward_host", cuda=False)
        if not (x_host.is_contiguous() and y_host.is_contiguous()):
            raise ValueError("forward_host: host buffers must be dense")
        _check(lib().dtq_qlinear_forward_host(x_host.data_ptr(), _dtype_code(x_host.dtype), M,
                                              self._h, mode, y_host.data_ptr(),
                                              _dtype_code(y_host.dtype), _stream(stream)))
        return y_host


NUM_RANGES = 4  # plan.hpp:17 kNumRanges


def range_index(t: int, steps: int) -> int:
    """Timestep range of denoising step t of `steps` (toydit.cpp:115)."""
    if steps <= 0 or not 0 <= t < steps:
        raise ValueError(f"step {t} outside [0, {steps})")
    return t * NUM_RANGES // steps


@dataclass
class MixedPrecisionPlan:
    """MixedPrecisionPlan (plan.hpp:30-40): weight bits per (layer, range)."""
    bits: dict
    budget: float = 8.0

    def bits_for(self, layer: str, range_idx: int) -> int:
        if layer not in self.bits:
            raise ValueError(f"MixedPrecisionPlan: unknown layer {layer}")
        row = self.bits[layer]
        if not 0 <= range_idx < NUM_RANGES:
            raise IndexError("MixedPrecisionPlan: range index out of range")  # array::at
        return int(row[range_idx])


class PlannedLinear:
    """One layer of a MixedPrecisionPlan on the device (dtq_planned_*): a
    device-resident QuantLinear per distinct weight width of the layer's
    row, and the per-step dispatch of toydit.cpp:113-117."""

    def __init__(self, handle: int, name: str, N: int, K: int, bits, act_bits: int):
        self._h = C.c_void_p(handle)
        self.name, self.N, self.K, self.bits, self.act_bits = name, N, K, tuple(bits), act_bits

    @classmethod
    def create(cls, w, plan: MixedPrecisionPlan, name: str, act_bits: int = 8, bias=None,
               balance: Optional[Balance] = None, stream=None) -> "PlannedLinear":
        torch = _torch()
        _check_rows(w, w.shape[1] if w.dim() == 2 else -1, "planned weights")
        N, K = w.shape
        bits = [plan.bits_for(name, r) for r in range(NUM_RANGES)]
        arr = (C.c_int32 * NUM_RANGES)(*bits)
        bias_t = None if bias is None else torch.as_tensor(bias, dtype=torch.float64,
                                                           device=w.device).contiguous()
        h = C.c_void_p()
        b = balance._c() if balance is not None else None
        _check(lib().dtq_planned_create(w.data_ptr(), _dtype_code(w.dtype), N, K, w.stride(0), arr,
                                        act_bits, _ptr(bias_t), _ref_or_none(b), _stream(stream),
                                        C.byref(h)))
        return cls(h.value, name, N, K, bits, act_bits)

    def select(self, t: int, steps: int) -> QuantLinear:
        """The QuantLinear serving step t of `steps` (borrowed from this layer)."""
        h = C.c_void_p()
        _check(lib().dtq_planned_select(self._h, t, steps, C.byref(h)))
        return QuantLinear(h.value, self.N, self.K, self.bits[range_index(t, steps)],
                           self.act_bits, owner=self)

    def forward(self, x, t: int, steps: int, **kw):
        return self.select(t, steps).forward(x, **kw)

    def workspace_bytes(self, M: int) -> int:
        """Forward workspace bytes for up to M rows at any step (the widest
        of the row's handles: a W4A8 one also holds its unpacked s8 weights)."""
        return max(lib().dtq_qlinear_workspace_bytes(self.select(r, NUM_RANGES)._h, M)
                   for r in range(NUM_RANGES))

    def close(self):
        if self._h is not None and self._h.value:
            lib().dtq_planned_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Checkpoint:
    """A reference quantized checkpoint (trace_io.cpp:225-316) loaded onto the
    B200: `len(ck)` layers, `ck.info(i)`, `ck.load(i)` -> QuantLinear whose
    packed codes were uploaded as stored and unpacked on the device."""

    def __init__(self, path: str):
        h = C.c_void_p()
        _check(lib().dtq_checkpoint_open(os.fsencode(path), C.byref(h)))
        self._h = h

    def __len__(self) -> int:
        n = C.c_int64(0)
        _check(lib().dtq_checkpoint_num_layers(self._h, C.byref(n)))
        return n.value

    def info(self, i: int) -> dict:
        name = C.c_char_p()
        N, K, mlen, rlen = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
        bits, sym = C.c_int(), C.c_int()
        _check(lib().dtq_checkpoint_layer_info(self._h, i, C.byref(name), C.byref(N), C.byref(K),
                                               C.byref(bits), C.byref(sym), C.byref(mlen),
                                               C.byref(rlen)))
        return {"name": name.value.decode(), "N": N.value, "K": K.value, "bits": bits.value,
                "symmetric": bool(sym.value), "mask_len": mlen.value, "rot_len": rlen.value}

    def load(self, i: int, act_bits: int = 8, hblock: int = 0, stream=None) -> "QuantLinear":
        inf = self.info(i)
        h = C.c_void_p()
        _check(lib().dtq_checkpoint_load_layer(self._h, i, act_bits, hblock, _stream(stream),
                                               C.byref(h)))
        return QuantLinear(h.value, inf["N"], inf["K"], inf["bits"], act_bits, None)

    def close(self):
        if self._h is not None and self._h.value:
            lib().dtq_checkpoint_close(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def hadamard_signs(n: int, seed: int, randomize: bool = True):
    """RotationMatrix.sign_diag (balance.cpp:73-78): first n draws of
    std::mt19937_64(seed), (draw & 1) ? +1 : -1, as an int8 numpy array.
    (Host-side, one-time; the engine is the C++ standard's mt19937_64.)"""
    import numpy as np
    out = np.ones(n, np.int8)
    if not randomize:
        return out
    mt = [0] * 312
    mt[0] = seed & 0xFFFFFFFFFFFFFFFF
    for i in range(1, 312):
        mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & 0xFFFFFFFFFFFFFFFF
    idx = 312
    UM, LM = 0xFFFFFFFF80000000, 0x7FFFFFFF
    for k in range(n):
        if idx >= 312:
            for i in range(312):
                x = (mt[i] & UM) | (mt[(i + 1) % 312] & LM)
                xa = x >> 1
                if x & 1:
                    xa ^= 0xB5026F5AA96619E9
                mt[i] = mt[(i + 156) % 312] ^ xa
            idx = 0
        y = mt[idx]
        idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        out[k] = 1 if (y & 1) else -1
    return out
