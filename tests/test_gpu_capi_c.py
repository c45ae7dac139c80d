"""The plain-C caller of the C ABI (tests/capi_example.c) on the B200: a
balanced W8A8 layer created and run through dtq_qlinear_create /
dtq_qlinear_forward from C, output finite and non-zero."""
import subprocess

import pytest

from test_capi import _build_c_example

pytestmark = pytest.mark.gpu


def test_c_caller_runs_a_forward(tmp_path):
    exe = _build_c_example(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok:" in r.stdout, r.stdout + r.stderr
