"""Seeded initial factors on the device (csrc/init.cu) against the host draw
of nmf.py:115-127 (numpy default_rng PCG64): bit-identical."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,m,r,seed", [(1, 1, 1, 0), (500, 1000, 10, 0), (333, 77, 7, 123),
                                        (10000, 20000, 50, 1), (64, 129, 200, 2**40 + 5)])
@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_device_init_bit_identical(n, m, r, seed, precision):
    import torch

    from paper_1506_08938_b200 import NmfConfig
    from paper_1506_08938_b200.nmf import device_initial_factors, initial_factors_from_mean

    cfg = NmfConfig(rank=r, seed=seed, precision=precision)
    mean = 0.7312
    G, FT = device_initial_factors(n, m, mean, cfg)
    g, ft = initial_factors_from_mean(n, m, mean, cfg)
    dt = np.float32 if precision == "fp32" else np.float64
    assert np.array_equal(G.cpu().numpy(), g.astype(dt))
    assert np.array_equal(FT.cpu().numpy(), ft.astype(dt))


def test_device_init_config5_sample():
    """Config-5 size (2.4e8 draws): the tail of the stream (the last F
    column block) equals the host draw -- the jump-ahead reaches the far end."""
    from paper_1506_08938_b200 import NmfConfig
    from paper_1506_08938_b200.nmf import device_initial_factors

    n, m, r = 1000000, 200000, 200
    cfg = NmfConfig(rank=r, seed=4)
    G, FT = device_initial_factors(n, m, 2.0, cfg)
    rng = np.random.default_rng(4)
    rng.bit_generator.advance(n * r + (r - 1) * m)  # F row r-1 starts here
    tail = rng.uniform(size=m) * np.sqrt(2.0 / r)
    assert np.array_equal(FT[:, r - 1].cpu().numpy(), tail.astype(np.float32))
    head = np.random.default_rng(4).uniform(size=1000) * np.sqrt(2.0 / r)
    assert np.array_equal(G.reshape(-1)[:1000].cpu().numpy(), head.astype(np.float32))
