"""tests/golden_util.random_params reproduces the reference's randomized
parameter sets (checked against the parameters stored in a fixture that was
built with them)."""

import numpy as np

from golden_util import load, random_params
from paper_2603_21090_b200.config import Dims


def test_random_params_matches_fixture_params():
    z = load("engine_k2_last_adaptive")  # make_golden: seed 5, random biases
    dims = Dims(d_s=8, d_e=4, d_t=8, d_m=8, d_k=4, heads=2, layers=2)
    p = random_params(5, dims)
    for k, v in p.tensors().items():
        np.testing.assert_array_equal(v, z["param_" + k].reshape(v.shape), err_msg=k)
