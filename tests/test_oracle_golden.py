"""The oracles reproduce the reference's own known answers (golden vectors
restated from proj/tests/*.cpp).  CPU only."""
import pytest

import golden_cases as G


@pytest.mark.parametrize("case", G.ALL, ids=lambda f: f.__name__)
@pytest.mark.parametrize("backend", ["ref", "port"])
def test_oracle_golden(case, backend, request):
    case(request.getfixturevalue(backend))
