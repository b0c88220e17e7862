"""Pins the plain-C restatement (oracle/port, `mmport_`) against the
UNMODIFIED reference compiled from /root/reference (oracle/_ref, `mmref_`):
identical inputs, bit-exact outputs.  CPU only."""
import numpy as np
import pytest

import parity_cases as P


@pytest.mark.parametrize("name", ["intra", "select", "schedule", "exhaustive", "brute", "inter", "cost",
                                  "simulate", "stats", "disaggregated", "stream", "orchestration"])
def test_port_matches_reference(name, port, ref):
    rng = np.random.default_rng(1234 + len(name))
    getattr(P, "check_" + name)(port, ref, rng)
