"""librnntg's host input generators against the compiled reference (no GPU):
init_model weights (model.hpp:129-169) and DetRng gaussian features
(common.hpp:86-127) must be bit-identical, so bench.py's GPU arm decodes the
reference arm's exact inputs."""
import numpy as np
import pytest

from tests import helpers as H


@pytest.mark.parametrize("cfg", [(500, 80, 512, 512, 512, 1, 0.4), (37, 11, 24, 16, 20, 99, -1.4), (2, 1, 1, 1, 1, 0, 0.0)])
def test_init_model_weights_bit_identical(cfg):
    from paper_2211_00484_b200.api import init_model_weights

    V, F, D, E, J, seed, bias = cfg
    want = H.ref().model(V, F, D, E, J, seed, bias).w.p
    got = init_model_weights(V, F, D, E, J, seed=seed, blank_bias=bias)
    assert set(got) == set(want)
    for k in want:
        assert got[k].shape == want[k].shape, k
        assert np.array_equal(got[k].view(np.uint32), want[k].view(np.uint32)), k


def test_gaussian_features_bit_identical():
    from paper_2211_00484_b200.api import gaussian_features

    B, T, F = 12, 37, 80
    got = gaussian_features(7000, B, T, F, threads=3)
    for i in range(B):
        want = H.ref().features(7000 + i, T, F)
        assert np.array_equal(got[i * T : (i + 1) * T].view(np.uint32), want.view(np.uint32)), i
    # thread count does not change the bits
    assert np.array_equal(gaussian_features(7000, B, T, F, threads=1).view(np.uint32), got.view(np.uint32))


def test_generators_validate():
    from paper_2211_00484_b200.api import ValidationError, gaussian_features, init_model_weights

    with pytest.raises(ValidationError):
        init_model_weights(1, 80, 512, 512, 512)
    with pytest.raises(ValidationError):
        gaussian_features(0, -1, 10, 80)
