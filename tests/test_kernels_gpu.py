"""Device self-checks of arithmetic building blocks the bit-exact kernels rely on."""
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("max_den,seed", [(64, 1), (4096, 2), (1 << 20, 3), ((1 << 31) - 1, 4)])
def test_reciprocal_division_is_correctly_rounded(max_den, seed):
    """resolve_spec.cu div_rcp (RN(1/b) + two FMA remainder corrections) == __ddiv_rn, bit for
    bit, on 2^26 random operands per denominator range (Eq. 3/4 and the buffer mean divide by
    integer counts)."""
    from paper_2604_10060_b200.api import debug_div_check

    assert debug_div_check(1 << 26, seed, max_den) == 0
