"""CUDA path vs the oracle (compiled reference when present, else the C
restatement), bit-exact, through the C ABI of libdisttrain_b200.so."""
import numpy as np
import pytest

import golden_cases as G
import parity_cases as P

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["intra", "select", "schedule", "exhaustive", "brute", "inter", "cost",
                                  "simulate", "disaggregated", "stream", "orchestration"])
def test_gpu_matches_oracle(name, gpu, oracle_best):
    rng = np.random.default_rng(4321 + len(name))
    getattr(P, "check_" + name)(gpu, oracle_best, rng)


@pytest.mark.parametrize("case", G.ALL, ids=lambda f: f.__name__)
def test_gpu_golden(case, gpu):
    case(gpu)
