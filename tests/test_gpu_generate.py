"""GEN: deterministic under sharding; follows the reference synthetic law."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_1905_13746_b200 import dense  # noqa: E402


def test_sharding_reproduces_the_same_rows():
    whole = dense.generate(5000, 60, group_rows=[2000, 3000], seed=3)
    a = dense.generate(2100, 60, group_rows=[2000, 3000], seed=3)
    b = dense.generate(2900, 60, group_rows=[2000, 3000], seed=3, row_offset=2100)
    for i in range(3):
        assert torch.equal(whole[i], torch.cat([a[i], b[i]]))


def test_law():
    x, size, lab = dense.generate(200_000, 50, group_rows=[100_000, 100_000], divergence=0.8,
                                  seed=1)
    x, size, lab = x.cpu().numpy(), size.cpu().numpy(), lab.cpu().numpy()
    assert (size[:100_000] < 5120).all() and (size[100_000:] >= 5120).all()
    assert (size[100_000:] < 10240).all()
    assert abs(lab.mean() - 0.5) < 0.01
    T = 64 + size // 64
    assert abs(x.sum(1).mean() / T.mean() - 1) < 0.01
    m = x[lab == 1]
    assert m[:, :25].sum() > 3 * m[:, 25:].sum()   # malware owns the first ceil(V/2)
