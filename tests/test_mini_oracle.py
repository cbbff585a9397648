"""The C oracle (oracle/ensi_oracle.c) against the independent big-integer mini-oracle (oracle/mini.py), word for
word, for N' <= 256 (SURVEY.md 8(c) O10 "pinned internally by agreement between two independent
implementations"): NTT, automorphism, ModUp, KIP + ModDown (R10 centred), hoisted rotations, Layout B (O11) and
rescale (O12).  The mini-oracle is itself pinned to the schoolbook negacyclic product and to exact integer
identities here, and the ModDown cross-check is shown to reject an uncentred and an exact-CRT conversion."""
import numpy as np
import pytest

import oracle
from oracle.mini import Mini


def _pair(log_n, L, alpha, dnum):
    o = oracle.Oracle(log_n, L, alpha, dnum)
    return o, Mini(log_n, o.q, o.p, dnum)


def _rand(rs, moduli, n):
    return np.stack([rs.integers(0, m, n, dtype=np.uint64) for m in moduli])


def _lst(a):
    return [[int(v) for v in row] for row in a]


def _ct_list(ct):
    return [_lst(ct[0]), _lst(ct[1])]


def _ct_np(ct):
    return np.array(ct, dtype=np.uint64)


@pytest.fixture(scope="module")
def ks64():
    # N' = 64, L = 4, alpha = 2, dnum = 2: two limbs per digit (non-trivial basis conversion) and two special primes
    return _pair(6, 4, 2, 2)


def test_mini_ntt_is_the_negacyclic_transform():
    """The mini NTT turns the schoolbook product in Z_q[X]/(X^N'+1) into the slot-wise product, and INTT inverts it."""
    mo = Mini(4, [97, 193], [], 1)                     # q = 1 mod 32
    rs = np.random.default_rng(1)
    for q in mo.q:
        a = [int(v) for v in rs.integers(0, q, 16)]
        b = [int(v) for v in rs.integers(0, q, 16)]
        c = [0] * 16
        for i in range(16):
            for j in range(16):
                k = i + j
                c[k % 16] = (c[k % 16] + (a[i] * b[j] if k < 16 else -a[i] * b[j])) % q
        A, Bn = mo.ntt(q, a), mo.ntt(q, b)
        assert mo.intt(q, [x * y % q for x, y in zip(A, Bn)]) == c
        assert mo.intt(q, A) == a


@pytest.mark.parametrize("log_n,L,alpha", [(4, 3, 1), (6, 4, 2), (8, 3, 1)])
def test_ntt_c_vs_mini(log_n, L, alpha):
    o, mo = _pair(log_n, L, alpha, -(-L // alpha))
    rs = np.random.default_rng(log_n)
    for li, m in enumerate(o.moduli):
        a = rs.integers(0, m, o.n, dtype=np.uint64)
        a[:2] = [0, m - 1]
        assert [int(v) for v in o.ntt(li, a)] == mo.ntt(m, [int(v) for v in a])
        assert [int(v) for v in o.intt(li, a)] == mo.intt(m, [int(v) for v in a])


def test_min_root_c_vs_mini():
    for log_n in (4, 6, 8):
        o, mo = _pair(log_n, 3, 1, 3)
        from oracle.mini import min_root
        assert [min_root(m, o.n) for m in o.moduli] == o.psi


def test_automorphism_c_vs_mini(ks64):
    """NTT-slot permutation of the C oracle == coefficient-domain a(X) -> a(X^g) of the mini-oracle."""
    o, mo = ks64
    rs = np.random.default_rng(2)
    rows = _rand(rs, o.q, o.n)
    for r in (1, 3, -1, 17, 31):
        g = o.galois(r)
        got = o.automorph_ntt(g, rows)
        for i in range(o.L):
            assert [int(v) for v in got[i]] == mo.automorph_ntt(o.q[i], [int(v) for v in rows[i]], g)


@pytest.mark.parametrize("level", [4, 3])
def test_modup_c_vs_mini(ks64, level):
    """ModUp (O10, no overflow correction; level 3 = a partial last digit)."""
    o, mo = ks64
    c = _rand(np.random.default_rng(3 + level), o.q[:level], o.n)
    got = o.modup(level, c)
    want = mo.modup(level, _lst(c))
    assert [[[int(v) for v in row] for row in d] for d in got] == want


@pytest.mark.parametrize("level", [4, 2])
def test_moddown_c_vs_mini_and_conventions(ks64, level):
    """ModDown (R10 centred) agrees word for word; an uncentred or exact-CRT conversion does not."""
    o, mo = ks64
    ext = o.q[:level] + o.p
    acc = _rand(np.random.default_rng(7 + level), ext, o.n)
    got = _lst(o.moddown(level, acc))
    assert got == mo.moddown(level, _lst(acc))
    assert got != mo.moddown(level, _lst(acc), variant="uncentred")
    assert got != mo.moddown(level, _lst(acc), variant="exact")


@pytest.mark.parametrize("level", [4, 3])
def test_rotation_c_vs_mini(ks64, level):
    """Rot(ct; g) = ModUp, sigma_g on the extended digits, KIP, ModDown, + sigma_g(c0): seeded uniform keys and
    ciphertext (the bits do not depend on key validity); hoisted C rotations == single mini rotations."""
    o, mo = ks64
    rs = np.random.default_rng(11 + level)
    T = o.L + o.alpha
    gs = [o.galois(r) for r in (1, 5, -3, 31)]
    keys = np.stack([np.stack([np.stack([_rand(rs, o.moduli, o.n) for _ in range(2)]) for _ in range(o.dnum)])
                     for _ in gs])
    assert keys.shape == (len(gs), o.dnum, 2, T, o.n)
    ct = np.stack([_rand(rs, o.q[:level], o.n) for _ in range(2)])
    got = o.rotate_hoisted(ct, gs, keys)
    for r, g in enumerate(gs):
        want = mo.rotate(_ct_list(ct), g, [[_lst(keys[r, t, j]) for j in range(2)] for t in range(o.dnum)])
        assert _ct_list(got[r]) == want, g
        assert (o.rotate(ct, g, keys[r]) == got[r]).all()


def test_rotation_c_vs_mini_n256():
    """The same at N' = 256 with the C1 digit shape (alpha = 1, three digits)."""
    o, mo = _pair(8, 3, 1, 3)
    rs = np.random.default_rng(21)
    g = o.galois(7)
    key = np.stack([np.stack([_rand(rs, o.moduli, o.n) for _ in range(2)]) for _ in range(o.dnum)])
    ct = np.stack([_rand(rs, o.q, o.n) for _ in range(2)])
    want = mo.rotate(_ct_list(ct), g, [[_lst(key[t, j]) for j in range(2)] for t in range(o.dnum)])
    assert _ct_list(o.rotate(ct, g, key)) == want


@pytest.mark.parametrize("B", [0, 2])
def test_layout_b_c_vs_mini(ks64, B):
    """O11 at N' = 64 (32 slots, s = 4 tokens per block, k = 8 columns per ciphertext), d = 11 (ragged), m = 3:
    B = k (baby steps only) and B = 2 (four giant steps), every output word."""
    o, mo = ks64
    s, d, m = 4, 11, 3
    k, n_in, Bq, G, rots = oracle.layout_b_plan(o.n, s, d, m, B)
    rs = np.random.default_rng(31 + B)
    x = np.stack([np.stack([_rand(rs, o.q, o.n) for _ in range(2)]) for _ in range(n_in)])
    W = rs.integers(-1, 2, (d, m)).astype(np.int8)
    gk = oracle.layout_b_galois(o.n, o.log_n, s, Bq, G)
    keys = np.stack([np.stack([np.stack([_rand(rs, o.moduli, o.n) for _ in range(2)]) for _ in range(o.dnum)])
                     for _ in gk])
    got = o.pcmm_b(x, W, s, k, Bq, gk, keys)
    kd = {g: [[_lst(keys[i, t, j]) for j in range(2)] for t in range(o.dnum)] for i, g in enumerate(gk)}
    want = mo.pcmm_b([_ct_list(c) for c in x], W.tolist(), s, k, Bq, kd)
    for i in range(m):
        assert _ct_list(got[i]) == want[i], i
    sub = o.pcmm_b(x, W, s, k, Bq, gk, keys, cols=[2, 0], nthreads=3)
    assert (sub[0] == got[2]).all() and (sub[1] == got[0]).all()


@pytest.mark.parametrize("B", [1, 2, 4])
def test_layout_b_lazy_moddown_c_vs_mini(ks64, B):
    """R19 lazy ModDown at N' = 64 (k = 8, so G = 8, 4, 2 giant steps): the C oracle's lazy form == the mini-oracle's
    (its own ModUp / KIP / centred ModDown, summed over Q_l u P by Python integers) word for word; at G = 2 (one
    giant rotation per output) lazy == eager exactly, while at G > 2 the two differ (a single ModDown of the sum is
    not the sum of the ModDowns) -- so a lazy path that silently ran the eager one would fail here."""
    o, mo = ks64
    s, d, m = 4, 11, 3
    k, n_in, Bq, G, rots = oracle.layout_b_plan(o.n, s, d, m, B)
    rs = np.random.default_rng(61 + B)
    x = np.stack([np.stack([_rand(rs, o.q, o.n) for _ in range(2)]) for _ in range(n_in)])
    W = rs.integers(-1, 2, (d, m)).astype(np.int8)
    gk = oracle.layout_b_galois(o.n, o.log_n, s, Bq, G)
    keys = np.stack([np.stack([np.stack([_rand(rs, o.moduli, o.n) for _ in range(2)]) for _ in range(o.dnum)])
                     for _ in gk])
    lazy = o.pcmm_b(x, W, s, k, Bq, gk, keys, lazy=True)
    eager = o.pcmm_b(x, W, s, k, Bq, gk, keys)
    kd = {g: [[_lst(keys[i, t, j]) for j in range(2)] for t in range(o.dnum)] for i, g in enumerate(gk)}
    want = mo.pcmm_b([_ct_list(c) for c in x], W.tolist(), s, k, Bq, kd, lazy=True)
    for i in range(m):
        assert _ct_list(lazy[i]) == want[i], i
    if G <= 2:
        assert (lazy == eager).all()
    else:
        assert not (lazy == eager).all()
    sub = o.pcmm_b(x, W, s, k, Bq, gk, keys, cols=[1], nthreads=2, lazy=True)
    assert (sub[0] == lazy[1]).all()


def test_pcmm_a_c_vs_mini(ks64):
    o, mo = ks64
    rs = np.random.default_rng(41)
    x = np.stack([np.stack([_rand(rs, o.q, o.n) for _ in range(2)]) for _ in range(6)])
    W = rs.integers(-1, 2, (6, 5)).astype(np.int8)
    got = o.pcmm_a(x, W)
    want = mo.pcmm_a([_ct_list(c) for c in x], W.tolist())
    assert [_ct_list(c) for c in got] == want


@pytest.mark.parametrize("level", [4, 2])
def test_rescale_c_vs_mini(ks64, level):
    o, mo = ks64
    ct = np.stack([_rand(np.random.default_rng(51 + level + j), o.q[:level], o.n) for j in range(2)])
    assert _ct_list(o.rescale(ct)) == mo.rescale(_ct_list(ct))


@pytest.mark.parametrize("form,s,d,m", [(2, 8, 4, 2), (1, 8, 3, 4), (2, 4, 1, 2)])
def test_ccmm_c_vs_mini(form, s, d, m):
    """R18 CCMM at N' = 64 (32 slots, s-slot head blocks; L = 4 so two levels are left for the mask and the product):
    the oracle's CCMM (a Python driver over the C oracle's rotations, products, relinearisation and rescale) == the
    mini-oracle's own step-by-step R18 with Python integers, every output word -- both forms with alignments that
    need a giant AND a baby step (Ba = 2: form 2 element j = 3, form 1 column i = 3), d = 1.  (The final rescale
    divides the relinearisation's ModDown rounding away, so this pins the R18 step order, amounts, mask and
    products; the ModDown convention itself is pinned by the rotation and Layout-B cross-checks.)  Ciphertexts, keys and the mask are seeded uniform words (the arithmetic is
    data-oblivious)."""
    o, mo = _pair(6, 4, 2, 2)
    rs = np.random.default_rng(70 + 10 * form + d)
    level = 4
    pi, amounts, per_out, Ba = oracle.ccmm_plan(form, s, d, m)
    nsrc = m if form == 2 else d
    a = np.stack([np.stack([_rand(rs, o.q, o.n) for _ in range(2)]) for _ in range(d)])
    src = np.stack([np.stack([_rand(rs, o.q, o.n) for _ in range(2)]) for _ in range(nsrc)])
    mask = _rand(rs, o.q, o.n)
    keys = {o.galois(r): np.stack([np.stack([_rand(rs, o.moduli, o.n) for _ in range(2)]) for _ in range(o.dnum)])
            for r in amounts}
    rlk = np.stack([np.stack([_rand(rs, o.moduli, o.n) for _ in range(2)]) for _ in range(o.dnum)])
    got = o.ccmm(a, src, form, s, d, m, mask, keys, rlk)
    kd = {g: [[_lst(k[t, j]) for j in range(2)] for t in range(o.dnum)] for g, k in keys.items()}
    want = mo.ccmm([_ct_list(c) for c in a], [_ct_list(c) for c in src], form, s, d, m, _lst(mask), kd,
                   [[_lst(rlk[t, j]) for j in range(2)] for t in range(o.dnum)], Ba)
    assert len(want) == m
    for i in range(m):
        assert _ct_list(got[i]) == want[i], i
