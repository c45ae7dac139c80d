"""CPU-side checks of the drop-in boundary: the C-ABI library loads, exports
exactly what include/dtq_capi.h declares, and refuses to compute without a
sm_100 device (no CPU fallback)."""
import ctypes
import os
import re

import pytest

import paper_2406_02540_b200 as dtq

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "dtq_capi.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(dtq_[a-z0-9_]+)\s*\(", text)))


def test_header_matches_python_binding():
    assert declared_symbols() == sorted(dtq.EXPORTED)


def test_library_exports_every_declared_symbol():
    if not os.path.exists(dtq.LIB_PATH):
        pytest.skip("libdtq_b200.so not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(dtq.LIB_PATH)
    for name in declared_symbols():
        assert hasattr(lib, name), f"{name} missing from libdtq_b200.so"


def test_version_and_no_cpu_fallback():
    if not os.path.exists(dtq.LIB_PATH):
        pytest.skip("libdtq_b200.so not built")
    L = dtq.lib()
    assert L.dtq_capi_version() == 1
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    # without a device the boundary reports a CUDA error instead of computing
    assert L.dtq_device_check() == dtq.DTQ_ERR_CUDA
    assert b"no CUDA device" in L.dtq_last_error() or b"sm_100" in L.dtq_last_error()


def test_invalid_arguments_are_rejected_before_the_device():
    if not os.path.exists(dtq.LIB_PATH):
        pytest.skip("libdtq_b200.so not built")
    L = dtq.lib()
    # bits outside {2,4,6,8} -> DTQ_ERR_INVALID_ARGUMENT (quant.cpp:143-146)
    st = L.dtq_quantize_rows(1, dtq.F16, 4, 8, 8, 3, 0, 0, None, None, 1, 16, 1, 1, None, None)
    assert st == dtq.DTQ_ERR_INVALID_ARGUMENT
    # empty matrix
    st = L.dtq_quantize_rows(1, dtq.F16, 0, 8, 8, 8, 0, 0, None, None, 1, 16, 1, 1, None, None)
    assert st == dtq.DTQ_ERR_INVALID_ARGUMENT
    # weight bits 3 (make_quant_linear: unsupported bit width)
    h = ctypes.c_void_p()
    st = L.dtq_qlinear_create(1, dtq.F16, 4, 8, 8, 3, 8, None, None, None, ctypes.byref(h))
    assert st == dtq.DTQ_ERR_INVALID_ARGUMENT


def test_hadamard_signs_match_the_oracle_engine(oracle):
    import numpy as np
    for seed, n in [(7, 1152), (0, 64), (123, 4608)]:
        assert np.array_equal(dtq.hadamard_signs(n, seed), oracle.hadamard_signs(n, seed))


def test_mixed_precision_plan_mirror():
    # plan.hpp:30-40 bits_for (unknown layer -> std::invalid_argument) and the
    # range index of toydit.cpp:115 (t * 4 / steps)
    plan = dtq.MixedPrecisionPlan({"attn.qkv": (8, 4, 4, 4), "mlp.fc1": (4, 4, 4, 8)}, 5.0)
    assert plan.bits_for("attn.qkv", 0) == 8 and plan.bits_for("mlp.fc1", 3) == 8
    with pytest.raises(ValueError, match="unknown layer"):
        plan.bits_for("mlp.fc2", 0)
    assert [dtq.range_index(t, 20) for t in (0, 4, 5, 9, 10, 14, 15, 19)] == \
        [0, 0, 1, 1, 2, 2, 3, 3]
    assert [dtq.range_index(t, 6) for t in range(6)] == [0, 0, 1, 2, 2, 3]
    with pytest.raises(ValueError):
        dtq.range_index(20, 20)


def test_planned_layer_rejects_unquantized_widths_before_the_device():
    if not os.path.exists(dtq.LIB_PATH):
        pytest.skip("libdtq_b200.so not built")
    L = dtq.lib()
    h = ctypes.c_void_p()
    bits = (ctypes.c_int32 * 4)(8, 16, 4, 4)  # 16 = the reference's FP passthrough
    st = L.dtq_planned_create(1, dtq.F16, 4, 8, 8, bits, 8, None, None, None, ctypes.byref(h))
    assert st == dtq.DTQ_ERR_INVALID_ARGUMENT and b"range 1" in L.dtq_last_error()


def _build_c_example(tmp_path):
    import shutil
    import subprocess
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None or not os.path.exists(dtq.LIB_PATH):
        pytest.skip("no C compiler or libdtq_b200.so not built")
    libdir = os.path.dirname(dtq.LIB_PATH)
    exe = str(tmp_path / "capi_example")
    r = subprocess.run([cc, "-std=c11", "-Wall", "-Wextra", "-Werror", "-O2",
                        "-I" + os.path.join(ROOT, "include"), "-I/usr/local/cuda/include",
                        os.path.join(ROOT, "tests", "capi_example.c"), "-o", exe,
                        "-L" + libdir, "-ldtq_b200", "-L/usr/local/cuda/lib64", "-lcudart", "-lm",
                        "-Wl,-rpath," + libdir], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_caller_compiles_and_refuses_without_device(tmp_path):
    # include/dtq_capi.h is plain C11 (what cgo / JNI / N-API bind); without
    # a sm_100 device every compute entry point returns DTQ_ERR_CUDA
    import subprocess
    import torch
    exe = _build_c_example(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    if torch.cuda.is_available():
        assert r.returncode == 0 and "ok:" in r.stdout, r.stdout + r.stderr
    else:
        assert r.returncode == 3, r.stdout + r.stderr
