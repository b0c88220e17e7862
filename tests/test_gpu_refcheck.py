"""The reference's OWN hot-path tests (proj/tests/test_reorder.cpp,
test_pipeline_sim.cpp, test_orchestrator.cpp — 56 TEST_CASEs), compiled
unmodified and linked against the mmplan:: GPU shim
(paper_2408_04275_b200/shim/mmplan_gpu.cpp) instead of the reference's
reorder / pipeline_sim / simulate / orchestrator implementations, so every
hot-path call they make runs on the B200 through libdisttrain_b200.so
(oracle/refcheck/Makefile builds oracle/_ref/refcheck in the build
container; the binary travels to the GPU box).  One more TEST_CASE of our own
(oracle/refcheck/shim_warnings.cpp) checks that the shim forwards a
CostModel's warning sink string for string against the reference functions
linked into the same binary."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "refcheck")

pytestmark = pytest.mark.gpu


def test_reference_tests_pass_on_the_gpu_shim():
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/refcheck not built (needs /root/reference at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=1200)
    print(r.stdout)
    print(r.stderr[-4000:])
    assert "test cases:" in r.stdout, r.stderr[-2000:]
    assert r.returncode == 0, r.stdout + r.stderr[-4000:]
