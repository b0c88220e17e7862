"""Replays the golden fixtures (tests/golden/*.npz, recorded from the
compiled reference by tests/golden/make_golden.py) on the oracle port (CPU)
and on the CUDA path (GPU): bit-exact."""
import os

import numpy as np
import pytest

import golden_inputs as GI

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _check(pl, name):
    want = np.load(os.path.join(HERE, name + ".npz"))
    got = GI.CASES[name](pl)
    assert sorted(got) == sorted(want.files), name
    for k in want.files:
        a, b = np.asarray(got[k]), want[k]
        assert a.shape == b.shape and a.dtype.kind == b.dtype.kind, (name, k)
        assert np.array_equal(a, b), (name, k)


@pytest.mark.parametrize("name", sorted(GI.CASES))
def test_port_matches_fixtures(name, port):
    _check(port, name)


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(GI.CASES))
def test_gpu_matches_fixtures(name, gpu):
    _check(gpu, name)
