"""The C++ drop-in (paper_2506_00225_b200/dropin/splatmap_b200.cpp): the REFERENCE's own
test files (proj/tests/test_splat_render.cpp, test_explorer.cpp) linked against the B200
render / render_entropy / refresh_candidate_scores (oracle/Makefile target `dropin`)."""
import subprocess

import pytest

from conftest import ROOT, has_gpu

BIN = ROOT / "oracle" / "_ref"
TESTS = ["dropin_test_splat_render", "dropin_test_explorer"]


def _bin(name):
    exe = BIN / name
    if not exe.exists():
        pytest.skip(f"{exe} not built (make -C oracle dropin needs /root/reference)")
    return exe


@pytest.mark.skipif(has_gpu(), reason="checks the no-GPU failure path")
def test_dropin_fails_loudly_without_gpu():
    r = subprocess.run([str(_bin(TESTS[0]))], capture_output=True, text=True, timeout=300)
    assert r.returncode != 0
    assert "no CUDA device" in r.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("name", TESTS)
def test_reference_tests_pass_on_the_gpu_dropin(name):
    r = subprocess.run([str(_bin(name))], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 failed" in r.stdout, r.stdout
