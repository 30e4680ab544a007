"""The reference's C++ runtime API, called from a compiled C++ program exactly
as reference callers do (tests/cpp/test_runtime_api.cpp, built by build()):
optimize -> derive_versions -> compile_version_set -> execute / train_step,
OffloadDevice, ExecutionContext, HostModel's public maps, l1_loss / sgd_step,
and the dynamic-batch (VdimBinding::enable) case of test_runtime.cpp:289-303."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "test_runtime_api")


def test_cpp_test_program_builds():
    subprocess.run(["make", "-C", os.path.join(ROOT, "paper_2205_10357_b200", "csrc"), "cpptest"], check=True,
                   capture_output=True)
    assert os.access(BIN, os.X_OK)


@pytest.mark.gpu
def test_reference_cpp_api_on_the_b200():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("[PASS]") == 7
