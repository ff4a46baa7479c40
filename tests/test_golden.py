"""The oracle reproduces its committed golden fixtures (tests/golden/make_golden.py). CPU."""
import json
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
GOLD = json.load(open(os.path.join(HERE, "golden", "oracle_golden.json")))


@pytest.mark.parametrize("name", sorted(GOLD))
def test_oracle_reproduces_golden(name):
    import make_golden
    qp = make_golden.cases()[name]
    got = make_golden.solve_case(qp)
    want = GOLD[name]
    assert got["status"] == want["status"] and got["iter"] == want["iter"]
    assert got["objective"] == pytest.approx(want["objective"], rel=1e-12, abs=1e-14)
    assert np.allclose(got["v"], want["v"], rtol=1e-10, atol=1e-13)
    assert [r[7] for r in got["log"]] == [r[7] for r in want["log"]]
