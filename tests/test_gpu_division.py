"""The fast kernels divide by shared divisors with a hoisted reciprocal
(hj_math.cuh div_by).  It must equal IEEE '/' bit for bit on every operand
pair -- random exponents, zeros, subnormals, huge values, infinities."""
import pytest
import torch

from paper_2411_03501_b200 import _lib
from paper_2411_03501_b200 import device as dev

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_hoisted_division_is_ieee(seed):
    lib = dev.require()
    bad = torch.zeros(1, dtype=torch.int64, device="cuda")
    _lib.check(lib.hj_check_division(200_000_000, seed, bad.data_ptr(), dev.stream()), "hj_check_division")
    assert int(bad.item()) == 0
