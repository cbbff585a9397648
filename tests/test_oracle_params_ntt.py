"""Pins for oracle O1 (primes), O2 (root, NTT) and O3 (RNG) -- independent of the oracle's own code.

Each check uses a route the oracle does not: sympy primality, the NTT's defining sum evaluated with
Python integers, schoolbook negacyclic convolution, closed forms.
"""
import numpy as np
import pytest
import sympy

import oracle

# SURVEY.md Appendix A (generated there with sympy.isprime from rule O1)
APPX_A = {
    12: dict(q=[1125899906826241, 1099511480321, 1099511390209], p=[1125899906629633],
             psi=[46909545429, 870088, 188538203, 12064401162]),
    16: dict(q=[1125899903827969, 1099510054913, 1099507695617, 1099506515969, 1099504549889, 1099503894529,
                1099503370241, 1099502714881, 1099500617729, 1099499569153, 1099499175937, 1099498258433],
             p=[1125899902124033, 1125899887312897, 1125899886395393, 1125899885740033],
             psi=[938640682, 7252600, 14931816, 13263982, 1356182, 16944792, 34586525, 6447889, 10819214,
                  34605531, 39932316, 3084991, 15995550378, 23906205461, 1661048488, 25140104975]),
}


def _rule_primes_sympy(log_n, L, alpha):
    """O1 rule evaluated with sympy (independent of the oracle's Miller-Rabin)."""
    two_n = 2 << log_n
    def desc(start_exclusive, count):
        c = (start_exclusive - 1) // two_n * two_n + 1
        if c >= start_exclusive:
            c -= two_n
        out = []
        while len(out) < count:
            if sympy.isprime(c):
                out.append(c)
            c -= two_n
        return out
    fifty = desc(1 << 50, 1 + alpha)
    forty = desc(1 << 40, L - 1)
    return [fifty[0]] + forty, fifty[1:]


@pytest.mark.parametrize("log_n,L,alpha", [(12, 3, 1), (16, 12, 4), (4, 2, 1), (8, 4, 2)])
def test_prime_rule_matches_sympy(log_n, L, alpha):
    q, p = oracle.gen_params(log_n, L, alpha)
    eq, ep = _rule_primes_sympy(log_n, L, alpha)
    assert q == eq and p == ep
    for v in q + p:
        assert (v - 1) % (2 << log_n) == 0
    assert len(set(q + p)) == len(q + p)


@pytest.mark.parametrize("log_n", [12, 16])
def test_appendix_a_table(log_n):
    L, alpha = (3, 1) if log_n == 12 else (12, 4)
    q, p = oracle.gen_params(log_n, L, alpha)
    assert q == APPX_A[log_n]["q"] and p == APPX_A[log_n]["p"]
    psis = [oracle.min_root(v, log_n) for v in q + p]
    assert psis == APPX_A[log_n]["psi"]


@pytest.mark.parametrize("log_n,L,alpha", [(12, 3, 1), (6, 2, 1)])
def test_min_root_is_minimal_primitive(log_n, L, alpha):
    """psi^N' = -1 and psi is the smallest of all odd powers of any primitive 2N'-th root (Python pow)."""
    n = 1 << log_n
    q, p = oracle.gen_params(log_n, L, alpha)
    for v in q + p:
        psi = oracle.min_root(v, log_n)
        assert pow(psi, n, v) == v - 1
        # independent enumeration: find a root from a sympy primitive root, take all odd powers
        g = sympy.primitive_root(v)
        r0 = pow(g, (v - 1) // (2 * n), v)
        roots = [pow(r0, k, v) for k in range(1, 2 * n, 2)]
        assert min(roots) == psi


def _brv(x, bits):
    return int(format(x, f"0{bits}b")[::-1], 2) if bits else 0


@pytest.mark.parametrize("log_n", [3, 4, 5, 6])
def test_ntt_matches_definition(log_n):
    """NTT(a)[k] = sum_i a_i psi^{(2 brv(k)+1) i} mod q, evaluated directly with Python ints."""
    n = 1 << log_n
    o = oracle.Oracle(log_n, 2, 1, 2)
    rs = np.random.default_rng(log_n)
    for limb in range(3):
        q, psi = o.moduli[limb], o.psi[limb]
        a = [int(v) for v in rs.integers(0, q, n, dtype=np.uint64)]
        want = [sum(a[i] * pow(psi, (2 * _brv(k, log_n) + 1) * i, q) for i in range(n)) % q for k in range(n)]
        got = [int(v) for v in o.ntt(limb, a)]
        assert got == want
        assert [int(v) for v in o.intt(limb, got)] == a


@pytest.mark.parametrize("log_n", [3, 4, 5])
def test_ntt_convolution_schoolbook(log_n):
    """INTT(NTT(a) * NTT(b)) == a*b mod (X^N' + 1), schoolbook negacyclic product in Python ints."""
    n = 1 << log_n
    o = oracle.Oracle(log_n, 2, 1, 2)
    rs = np.random.default_rng(100 + log_n)
    for limb in range(3):
        q = o.moduli[limb]
        a = [int(v) for v in rs.integers(0, q, n, dtype=np.uint64)]
        b = [int(v) for v in rs.integers(0, q, n, dtype=np.uint64)]
        c = [0] * n
        for i in range(n):
            for j in range(n):
                if i + j < n:
                    c[i + j] += a[i] * b[j]
                else:
                    c[i + j - n] -= a[i] * b[j]
        c = [v % q for v in c]
        A, Bv = o.ntt(limb, a), o.ntt(limb, b)
        prod = [(int(x) * int(y)) % q for x, y in zip(A, Bv)]
        assert [int(v) for v in o.intt(limb, prod)] == c


@pytest.mark.parametrize("log_n,L,alpha", [(12, 3, 1), (16, 12, 4)])
def test_ntt_closed_forms_and_roundtrip(log_n, L, alpha):
    """NTT(X)[k] = psi^{2brv(k)+1}; NTT(1) = all ones; INTT(NTT(a)) = a."""
    n = 1 << log_n
    o = oracle.Oracle(log_n, L, alpha, 3)
    rs = np.random.default_rng(7)
    for limb in [0, 1, L + alpha - 1]:
        q, psi = o.moduli[limb], o.psi[limb]
        x = np.zeros(n, np.uint64); x[1] = 1
        got = o.ntt(limb, x)
        ks = rs.integers(0, n, 64)
        for k in ks:
            assert int(got[k]) == pow(psi, 2 * _brv(int(k), log_n) + 1, q)
        one = np.zeros(n, np.uint64); one[0] = 1
        assert (o.ntt(limb, one) == 1).all()
        a = rs.integers(0, q, n, dtype=np.uint64)
        assert (o.intt(limb, o.ntt(limb, a)) == a).all()


def test_rng_determinism_and_moments():
    """O3: same seed -> same draws; uniform/ternary/CBD(eta=21) moments."""
    a = oracle.rng_fill(1234, "raw", 1000)
    b = oracle.rng_fill(1234, "raw", 1000)
    assert (a == b).all() and not (a == oracle.rng_fill(1235, "raw", 1000)).all()
    q = 1099511480321
    u = oracle.rng_fill(5, "uniform", 400000, q).astype(np.float64)
    assert u.min() >= 0 and u.max() < q
    assert abs(u.mean() / q - 0.5) < 0.005
    t = oracle.rng_fill(6, "ternary", 300000)
    assert set(np.unique(t)) == {-1, 0, 1}
    for v in (-1, 0, 1):
        assert abs(np.mean(t == v) - 1 / 3) < 0.005
    e = oracle.rng_fill(7, "cbd", 400000).astype(np.float64)
    assert abs(e.mean()) < 0.02 and abs(e.var() - 10.5) < 0.15
    assert np.abs(e).max() <= 21
