"""The C++ drop-in (include/dtq/*.hpp over the C ABI, libdtq_dropin.so).

CPU: the library exports every dtq:: entry point the reference's headers
declare (quant.hpp / balance.hpp / qgemm.hpp / matrix.hpp / plan.hpp) and the
reference's own unit-test binary is built against it.
GPU: that binary -- the reference's test_quant.cpp, test_qgemm.cpp and
test_balance.cpp compiled unmodified (tests/dropin/Makefile) -- passes on
the B200, i.e. the reference's own known-answer and property tests hold for
the device implementation.
"""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2406_02540_b200", "libdtq_dropin.so")
BIN = os.path.join(ROOT, "tests", "dropin", "_bin", "dtq_ref_tests")

# reference declarations (quant.hpp:20-112, balance.hpp:16-71, qgemm.hpp:17-54,
# plan.hpp) as demangled prefixes
DROPIN_API = [
    "dtq::round_even(double)",
    "dtq::bits_supported(int)",
    "dtq::GroupingScheme::group_count(",
    "dtq::GroupingScheme::group_of(",
    "dtq::compute_minmax_params(",
    "dtq::compute_symmetric_params(",
    "dtq::compute_params(",
    "dtq::quantize(",
    "dtq::dequantize(",
    "dtq::fake_quantize(",
    "dtq::error_report(",
    "dtq::incoherence(",
    "dtq::fwht(double*",
    "dtq::compute_scaling_mask(",
    "dtq::apply_scaling(",
    "dtq::hadamard_matrix(",
    "dtq::RotationMatrix::dense() const",
    "dtq::rotate_channels(",
    "dtq::apply_rotation(",
    "dtq::static_dynamic_balance(",
    "dtq::apply_balance(",
    "dtq::choose_alpha(",
    "dtq::make_quant_linear(",
    "dtq::qlinear_forward(",
    "dtq::qlinear_forward_float(",
    "dtq::weight_bytes(",
    "dtq::checkpoint_bytes(",
    "dtq::fp16_baseline_bytes(",
    "dtq::matmul_nt(",
    "dtq::partition_timesteps(",
]


def _exports():
    if not os.path.exists(LIB):
        pytest.skip("libdtq_dropin.so not built")
    nm = shutil.which("nm")
    if nm is None:
        pytest.skip("nm not available")
    out = subprocess.run([nm, "-D", "-C", "--defined-only", LIB], check=True,
                         capture_output=True, text=True).stdout
    return out


def test_dropin_exports_reference_api():
    out = _exports()
    missing = [f for f in DROPIN_API if f not in out]
    assert not missing, missing


def test_dropin_has_no_host_compute_path():
    # the drop-in runs its arithmetic through libdtq_b200 (no CPU fallback):
    # it must link the product library, not the oracle
    out = subprocess.run(["ldd", LIB], capture_output=True, text=True).stdout if os.path.exists(LIB) else ""
    if not out:
        pytest.skip("libdtq_dropin.so not built")
    assert "libdtq_b200.so" in out
    assert "dtq_oracle" not in out and "dtq_ref" not in out


@pytest.mark.gpu
def test_reference_unit_tests_pass_on_device():
    if not os.path.exists(BIN):
        pytest.skip("reference unit-test binary not built (needs /root/reference at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    print(r.stderr[-4000:])
    assert r.returncode == 0, r.stderr[-4000:]
    assert "0 failed" in r.stdout


ACC = os.path.join(ROOT, "tests", "dropin", "_bin", "dtq_ref_acceptance")


@pytest.mark.gpu
def test_reference_acceptance_suite_passes_on_device(tmp_path):
    # tests/acceptance.cpp (10 criteria: quantizer correctness over 10k trials,
    # grouping, balance invariance, incoherence, int GEMM == float path, the
    # toy-DiT ablation ordering, memory ratios, plan arithmetic, heatmap,
    # serialization) with the reference's own toydit / sensitivity / trace_io
    # sources and every core numerics call on the B200 drop-in
    if not os.path.exists(ACC):
        pytest.skip("acceptance binary not built (needs /root/reference at build time)")
    r = subprocess.run([ACC], capture_output=True, text=True, timeout=900, cwd=tmp_path)
    print(r.stdout[-3000:])
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "all criteria passed" in r.stdout


APP = os.path.join(ROOT, "tests", "dropin", "_bin", "dtq_ref_app_tests")


@pytest.mark.gpu
def test_reference_model_and_io_unit_tests_pass_on_device(tmp_path):
    # tests/test_toydit.cpp, test_sensitivity.cpp, test_trace_io.cpp compiled
    # unmodified with the reference's toydit / sensitivity / trace_io sources:
    # the toy DiT's linears, the sensitivity sweep's fake-quantization and the
    # checkpoint writer's weight quantization all run on the B200 drop-in
    if not os.path.exists(APP):
        pytest.skip("model/io test binary not built (needs /root/reference at build time)")
    env = dict(os.environ, TMPDIR=str(tmp_path))
    r = subprocess.run([APP], capture_output=True, text=True, timeout=900, env=env)
    print(r.stdout)
    print(r.stderr[-4000:])
    assert r.returncode == 0, r.stderr[-4000:]
    assert " 0 failed" in r.stdout


THREADS = os.path.join(ROOT, "tests", "dropin", "_bin", "dtq_thread_test")


@pytest.mark.gpu
def test_dropin_concurrent_forward_is_bitexact():
    # qlinear_forward on one const layer from 8 threads (first use included)
    if not os.path.exists(THREADS):
        pytest.skip("thread test binary not built")
    r = subprocess.run([THREADS], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0 and "threads ok" in r.stdout, r.stdout + r.stderr[-2000:]


FIELDS = os.path.join(ROOT, "tests", "dropin", "_bin", "dtq_fields_test")


@pytest.mark.gpu
def test_dropin_reads_current_layer_fields_and_wide_groups():
    # a layer's bias / codes / scales / act_bits changed after its first
    # forward are used (never a stale device copy), copies stay independent,
    # and per_tensor / per_channel groups of > 16384 elements quantize
    if not os.path.exists(FIELDS):
        pytest.skip("fields test binary not built")
    r = subprocess.run([FIELDS], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0 and "fields ok" in r.stdout, r.stdout + r.stderr[-2000:]
