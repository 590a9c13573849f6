"""NEXT-1 parameter derivation: oracle and C ABI against the values the
paper and SPEC print (-m "not gpu"; host-only functions, no GPU needed)."""
import pytest

from oracle import params as O
from paper_2105_13678_b200 import pa as P
from paper_2105_13678_b200._binding import PAError

BOTH = [O, P]


@pytest.mark.parametrize("impl", BOTH)
@pytest.mark.parametrize("eps,s", [
    (1e-10, 65),    # SPEC.md:203 (epsilon of Table 2, PAPER.md: "security parameter of PA 10^-10")
    (0.25, 2),      # 2^-2 = 0.25 exactly
    (0.5, 1),       # s = 0 is raised to the minimum 1
    (2.0 ** -11, 20),   # exact power: 2^(-20/2-1) = 2^-11
])
def test_security_coefficient(impl, eps, s):
    assert impl.derive_security_coefficient(eps) == s


@pytest.mark.parametrize("impl", BOTH)
@pytest.mark.parametrize("ratio,k", [(0.2957, 3), (0.0972, 10), (0.5, 2)])   # SPEC.md:212-214, Table 3
def test_block_count(impl, ratio, k):
    assert impl.select_block_count(ratio) == k


@pytest.mark.parametrize("impl", BOTH)
@pytest.mark.parametrize("target,k,gamma", [
    (260_000_000, 10, 25_964_951),   # SPEC.md:221, the abstract's 2.6e8 block
    (200_000_000, 3, 57_885_161),    # SPEC.md:222, DV-QKD n ~ 2e8
    (21, 3, 7),
])
def test_select_gamma(impl, target, k, gamma):
    g, exceeds = impl.select_gamma(target, k)
    assert (g, exceeds) == (gamma, False)


@pytest.mark.parametrize("impl", BOTH)
def test_select_gamma_exceeds(impl):
    assert impl.select_gamma(5, 3) == (3, True)          # 3 * 3 > 5: smallest exponent, flagged


@pytest.mark.parametrize("impl", BOTH)
def test_paper_params_p1(impl):
    """eps = 1e-10, r = 0.0972, target 2.6e8 -> gamma = 25,964,951, k = 10;
    with t = n - m for m = 25,237,932 (the P1 workload)."""
    n = 10 * 25_964_951
    d = impl.derive_paper_params(260_000_000, 0.0972, n - 25_237_932 - 65, 1e-10)
    assert d == {"gamma": 25_964_951, "k": 10, "n": n, "s": 65, "m": 25_237_932}


@pytest.mark.parametrize("impl", BOTH)
def test_paper_params_invariants(impl):
    err = PAError if impl is P else ValueError
    with pytest.raises(err):
        impl.derive_paper_params(260_000_000, 0.0972, 0, 1e-10)     # m + s > gamma
    with pytest.raises(err):
        impl.derive_paper_params(260_000_000, 0.0972, 10 ** 12, 1e-10)   # m <= 0
    with pytest.raises(err):
        impl.derive_security_coefficient(1.5)
    with pytest.raises(err):
        impl.select_block_count(0.0)


def test_oracle_matches_abi_on_a_grid():
    for eps in (1e-3, 1e-6, 1e-9, 1e-12, 3e-7, 0.1, 0.49):
        assert O.derive_security_coefficient(eps) == P.derive_security_coefficient(eps)
    for ratio in (0.9, 0.34, 0.2, 0.125, 0.0972, 0.01):
        assert O.select_block_count(ratio) == P.select_block_count(ratio)
    for target in (10, 1000, 10**6, 10**8, 10**9):
        for k in (1, 2, 3, 10, 31):
            assert O.select_gamma(target, k) == P.select_gamma(target, k)
