"""Golden vectors produced by the reference library itself
(tests/golden/make_golden.py).  The oracle must reproduce them on CPU (so it
stays pinned where the reference is absent, e.g. on the GPU box) and the CUDA
product must reproduce them on the GPU, byte for byte."""
import os

import numpy as np
import pytest

import helpers
from golden_cases import GOLDEN, build

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _check(lib, name):
    g = np.load(os.path.join(HERE, f"{name}.npz"))
    cfg, painted, action = build(name)
    s = helpers.prepared(lib, cfg, painted)
    res, err = action(s)
    assert repr(err) == str(g["error"])
    assert np.array_equal(res["dts"], g["dts"])
    assert np.array_equal(np.array(res["counters"], dtype=np.float64), g["counters"])
    st = s.download()
    assert np.array_equal(np.array([st.step, st.time]), g["step_time"])
    bad = [f for f in helpers.STATE_FIELDS
           if not np.array_equal(getattr(st, f)[:cfg.nmat] if f in ("m", "e", "k") else getattr(st, f),
                                 g[f][:cfg.nmat] if f in ("m", "e", "k") else g[f])]
    assert bad == []


@pytest.mark.parametrize("name", GOLDEN)
def test_oracle_reproduces_golden(orc, name):
    _check(orc, name)


@pytest.mark.gpu
@pytest.mark.parametrize("name", GOLDEN)
def test_product_reproduces_golden(name):
    _check(helpers.product_lib(), name)
