"""TinyLM host side (paper_2602_12029_b200/tinylm.py) on the CPU: the
parameter init (model.ts:181-198 with rng.ts) is bit-identical to the
oracle's restatement, and the rng matches the reference's published
splitmix64 vectors (rng.test.ts:5-13)."""

import pytest
import torch

from oracle.tinylm import TinyConfig as OConfig
from oracle.tinylm import TinyLM as OTiny
from paper_2602_12029_b200.tinylm import TinyConfig, init_params, shared_prefix_length, splitmix64


def test_splitmix64_published_vectors():
    s, out = 0, []
    for _ in range(3):
        s, z = splitmix64(s)
        out.append(z)
    assert out == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]


@pytest.mark.parametrize("shape,seed", [((2, 32, 2, 32, 19), 5), ((1, 16, 4, 24, 7), 11)])
def test_init_matches_oracle(shape, seed):
    p, q = init_params(TinyConfig(*shape), seed), OTiny.init(OConfig(*shape), seed).p
    for k in ("tokEmb", "prevEmb", "posEmb", "lnFg", "lnFb", "head"):
        assert torch.equal(p[k], q[k]), k
    for a, b in zip(p["blocks"], q["blocks"], strict=True):
        for k in b:
            assert torch.equal(a[k], b[k]), k


def test_init_width_check_and_prefix_length():
    with pytest.raises(ValueError):
        init_params(TinyConfig(2, 30, 4, 32, 19), 0)
    assert [shared_prefix_length(r, 10) for r in (0, 0.3, 0.5, 1)] == [0, 3, 5, 9]
    with pytest.raises(ValueError):
        shared_prefix_length(1.5, 10)
