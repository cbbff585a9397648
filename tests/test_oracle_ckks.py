"""Pins for oracle O4-O12 against the paper and the mathematics (closed forms, invariants, decryption).

All parameters here are the C1 toy set (N'=2^12, L=3) or tinier rings; full-size checks live in the
GPU parity tests.
"""
import json
import os

import numpy as np
import pytest

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")
DELTA = 2.0 ** 40


def _enc_cols(o, pk, X, level, seed):
    """Encrypt every column of X (s x d) as one ciphertext (column-wise packing)."""
    d = X.shape[1]
    m_res = np.stack([o.encode(X[:, j], level, DELTA) for j in range(d)])
    seeds = np.arange(d, dtype=np.uint64) + np.uint64(seed)
    return o.encrypt_batch(seeds, pk, level, m_res)


# ---------------------------------------------------------------- O5 encode / decode

def test_encode_constant_closed_form():
    """A constant slot vector c encodes to the constant polynomial round(Delta*c)."""
    n = 1 << 12
    c = oracle.encode_coeffs(np.full(n // 2, 0.3), n, DELTA)
    assert c[0] == int(np.floor(0.3 * DELTA + 0.5))
    assert all(v == 0 for v in c[1:])


def test_encode_decode_roundtrip_and_padding():
    n = 1 << 12
    z = np.random.default_rng(0).uniform(-1, 1, 100)
    got = oracle.decode_coeffs(oracle.encode_coeffs(z, n, DELTA), n, DELTA)
    assert np.max(np.abs(got[:100] - z)) < 2 ** -30
    assert np.max(np.abs(got[100:])) < 2 ** -30      # zero padding


def test_encode_single_slot_evaluation():
    """Slot u is the evaluation at zeta^{5^u}: check m(zeta^{5^u}) directly with a Python sum."""
    n = 64
    z = np.random.default_rng(1).uniform(-1, 1, n // 2)
    c = oracle.encode_coeffs(z, n, DELTA)
    zeta = np.exp(1j * np.pi / n)
    for u in [0, 1, 5, 31]:
        e = pow(5, u, 2 * n)
        val = sum(c[i] * zeta ** (e * i) for i in range(n)) / DELTA
        assert abs(val.real - z[u]) < 1e-9 and abs(val.imag) < 1e-9


# ---------------------------------------------------------------- O4, O6, O7

def test_encrypt_decrypt_identity(c1):
    o, skc, sk, pk = c1
    z = np.random.default_rng(2).uniform(-1, 1, 2048)
    for level in (3, 2, 1):
        ct = o.encrypt(99, pk, level, o.encode(z, level, DELTA))
        got = o.decrypt(sk, ct, DELTA)
        assert np.max(np.abs(got - z)) < 2e-6


def test_keygen_deterministic_and_pk_relation(c1):
    """pk0 + pk1*s is the small error e (centred |e| <= 21) -- checked via INTT, coefficientwise."""
    o, skc, sk, pk = c1
    skc2, sk2, pk2 = o.keygen(0x454E5349 + 1)
    assert (sk2 == sk).all() and (pk2 == pk).all() and (skc2 == skc).all()
    for i in range(o.L):
        q = o.q[i]
        e_ntt = [(int(a) + int(b) * int(s)) % q for a, b, s in zip(pk[0, i], pk[1, i], sk[i])]
        e = o.intt(i, e_ntt)
        ec = [(int(v) if int(v) <= q // 2 else int(v) - q) for v in e]
        assert max(abs(v) for v in ec) <= 21
    # secret is ternary and sk is its NTT in every limb (Q and P)
    assert set(np.unique(skc)) <= {-1, 0, 1}
    for i in range(o.L + o.alpha):
        q = o.moduli[i]
        assert [int(v) for v in o.intt(i, sk[i])] == [int(v) % q for v in skc.astype(np.int64)]


def test_crt_limb_consistency_invariant(c1):
    """O7: for a PCMM output the CRT over limbs {0,1} equals the full CRT (|mu| << q0 q1 / 2)."""
    o, skc, sk, pk = c1
    X = synth.gen_X(3, 16, 16)
    W = synth.gen_W(4, 16, 16)
    x = _enc_cols(o, pk, X, 3, 500)
    y = o.pcmm_a(x, W)
    mu = o.decrypt_residues(sk, y[5])
    full = oracle.crt_centered(mu, o.q[:3])
    two = oracle.crt_centered(mu[:2], o.q[:2])
    assert full == two


# ---------------------------------------------------------------- O8 PCMM Layout A (Algorithm 1)

def test_toy_example_word_identity(c1):
    """y0 = x0 - x2, y1 = x1 - x0 + x3 (mod q), every RNS word."""
    o, skc, sk, pk = c1
    g = json.load(open(os.path.join(GOLD, "toy_example.json")))
    W = np.array(g["W"], np.int8)
    x = synth.gen_words(11, o.q, 4, 3, o.n)
    y = o.pcmm_a(x, W)
    for i, spec in enumerate(g["Y"]):
        for r in range(3):
            q = o.q[r]
            want = np.zeros((2, o.n), dtype=object)
            for j in spec["plus"]:
                want = want + x[j, :, r, :].astype(object)
            for j in spec["minus"]:
                want = want - x[j, :, r, :].astype(object)
            want = np.mod(want, q).astype(np.uint64)
            assert (y[i, :, r, :] == want).all()


@pytest.mark.parametrize("kind", ["zero", "identity", "neg_identity", "permutation", "plus", "minus"])
def test_edge_weights(c1, kind):
    o = c1[0]
    d = m = 8
    x = synth.gen_words(12, o.q, d, 3, o.n)
    x[0, 0, 0, :5] = 0                                     # edge words 0
    x[1, 1, 1, :5] = np.uint64(o.q[1] - 1)                 # and q-1
    W = synth.edge_W(kind, d, m, seed=3)
    y = o.pcmm_a(x, W)
    qv = np.array(o.q[:3], np.uint64)[None, :, None]
    if kind == "zero":
        assert (y == 0).all()
    elif kind in ("identity", "permutation"):
        for i in range(m):
            j = int(np.nonzero(W[:, i])[0][0])
            assert (y[i] == x[j]).all()                     # bitwise copy
    elif kind == "neg_identity":
        want = np.where(x == 0, np.uint64(0), qv - x)
        assert (y == want).all()
    else:
        tot = np.mod(np.sum(x.astype(object), axis=0), np.array(o.q[:3], dtype=object)[None, :, None])
        if kind == "minus":
            tot = np.mod(-tot, np.array(o.q[:3], dtype=object)[None, :, None])
        for i in range(m):
            assert (y[i] == tot.astype(np.uint64)).all()


def test_pcmm_linearity_and_ntt_commutation(c1):
    o = c1[0]
    d, m = 12, 10
    x = synth.gen_words(13, o.q, d, 3, o.n)
    rs = np.random.default_rng(5)
    W1 = rs.integers(-1, 2, (d, m)).astype(np.int8)
    W2 = np.where(rs.random((d, m)) < 0.5, 0, -W1).astype(np.int8)   # W1+W2 stays ternary
    y1, y2, y12 = o.pcmm_a(x, W1), o.pcmm_a(x, W2), o.pcmm_a(x, (W1 + W2).astype(np.int8))
    qv = np.array(o.q[:3], np.uint64)[None, None, :, None]
    assert (((y1 + y2) % qv) == y12).all()
    # INTT(sum) == sum(INTT): accumulate in coefficient form and compare limb 1 of output 3
    xi = np.stack([o.intt(1, x[j, 0, 1]) for j in range(d)]).astype(object)
    want = np.mod(sum(int(W1[j, 3]) * xi[j] for j in range(d)), o.q[1]).astype(np.uint64)
    assert (o.intt(1, y1[3, 0, 1]) == want).all()


def test_pcmm_threads_and_sampled_columns(c1):
    o = c1[0]
    x = synth.gen_words(14, o.q, 16, 3, o.n)
    W = synth.gen_W(15, 16, 16)
    y1 = o.pcmm_a(x, W, nthreads=1)
    y4 = o.pcmm_a(x, W, nthreads=4)
    ys = o.pcmm_a(x, W, cols=[3, 7, 15], nthreads=2)
    assert (y1 == y4).all() and (ys == y1[[3, 7, 15]]).all()


def test_pcmm_decrypts_to_float_product(c1):
    """North-star tolerance: decrypt(PCMM) vs float64 X.W, max-abs <= 1e-4 at scale 2^40 (C1 shape)."""
    o, skc, sk, pk = c1
    X = synth.gen_X(synth.SEED_BASE + 1, 16, 16)
    W = synth.gen_W(synth.SEED_BASE + 101, 16, 16)
    x = _enc_cols(o, pk, X, 3, 1000)
    y = o.pcmm_a(x, W)
    ref = X @ W.astype(np.float64)
    err = 0.0
    for i in range(16):
        z = o.decrypt(sk, y[i], DELTA)
        err = max(err, np.max(np.abs(z[:16] - ref[:, i])), np.max(np.abs(z[16:])))
    assert err < 1e-4


# ---------------------------------------------------------------- O9 automorphism

def test_automorphism_coeff_closed_form_python():
    """a(X^g) mod (X^N'+1) computed with Python ints matches the coefficient-form oracle,
    and NTT(sigma_g(INTT(x))) equals the NTT-domain permutation bitwise."""
    o = oracle.Oracle(5, 2, 1, 2)
    n = o.n
    rs = np.random.default_rng(8)
    for g in [5, 25, 2 * n - 1, 3, 125 % (2 * n)]:
        q = o.q[0]
        a = [int(v) for v in rs.integers(0, q, n, dtype=np.uint64)]
        want = [0] * n
        for i in range(n):
            e = i * g % (2 * n)
            if e < n:
                want[e] = (want[e] + a[i]) % q
            else:
                want[e - n] = (want[e - n] - a[i]) % q
        assert [int(v) for v in o.automorph_coeff(0, g, a)] == want
        xt = o.ntt(0, a)
        assert (o.automorph_ntt(g, xt) == o.ntt(0, want)).all()


def test_galois_identity_element():
    n = 1 << 12
    assert oracle.galois_elt(12, n // 2) == 1
    assert oracle.galois_elt(12, 0) == 1
    assert oracle.galois_elt(12, 1) == 5
    assert oracle.galois_elt(12, -1) == pow(5, n // 2 - 1, 2 * n)


# ---------------------------------------------------------------- O10 key switching / rotation

def test_rotkey_gadget_identity(c1):
    """b_t + a_t s - e_t == [r in D_t] (P mod q_r) sigma_g(s), limb by limb (O4)."""
    o, skc, sk, pk = c1
    g = o.galois(3)
    key, e = o.rotkey(77, g, sk, want_e=True)
    sg = o.automorph_ntt(g, sk)
    P = 1
    for p in o.p:
        P *= p
    for t in range(o.dnum):
        for i in range(o.L + o.alpha):
            r = o.moduli[i]
            e_ntt = o.ntt(i, [int(v) % r for v in e[t]])
            lhs = [(int(b) + int(a) * int(s) - int(ee)) % r for b, a, s, ee in zip(key[t, 0, i], key[t, 1, i], sk[i], e_ntt)]
            in_digit = i < o.L and t * o.alpha <= i < (t + 1) * o.alpha
            want = [(P % r) * int(v) % r if in_digit else 0 for v in sg[i]]
            assert lhs == want


def _tiny_ks_ctx():
    # two limbs per digit so the basis conversion is non-trivial: L=4, alpha=2, dnum=2, N'=32
    return oracle.Oracle(5, 4, 2, 2)


def test_modup_crt_identity():
    """ModUp: per digit the extension is x + u*Q_t with 0 <= u < |D_t| (exact big-integer identity)."""
    o = _tiny_ks_ctx()
    level = 4
    rs = np.random.default_rng(9)
    c = np.stack([rs.integers(0, o.q[i], o.n, dtype=np.uint64) for i in range(level)])
    ext = o.modup(level, c)
    coef = np.stack([o.intt(i, c[i]) for i in range(level)])
    ext_limbs = list(range(level)) + [o.L + k for k in range(o.alpha)]
    for t in range(2):
        D = [t * 2, t * 2 + 1]
        Qt = o.q[D[0]] * o.q[D[1]]
        x = oracle.crt_centered(coef[D], [o.q[i] for i in D])
        x = [v % Qt for v in x]                    # the canonical digit value in [0, Q_t)
        ext_coef = np.stack([o.intt(li, ext[t, e]) for e, li in enumerate(ext_limbs)])
        for k in range(o.n):
            us = set()
            for e, li in enumerate(ext_limbs):
                r = o.moduli[li]
                v = int(ext_coef[e, k])
                if li in D:
                    assert v == x[k] % r
                    continue
                # v == x + u Q_t mod r for some u in [0, |D_t|)
                cand = [u for u in range(len(D)) if (x[k] + u * Qt) % r == v]
                assert cand, (t, k, li)
                us.add(cand[0])
            assert len(us) == 1                    # one u shared by all target limbs


def test_moddown_exact_identity():
    """ModDown(acc) * P + v == acc over Q_l (exact big-integer identity) with v the fast-converted P-residue of R10:
    v = sum_k y_k (P/p_k), y_k = [acc_{p_k} (P/p_k)^{-1}]_{p_k} CENTRED in (-p_k/2, p_k/2], no overflow correction.
    Pinned to that v exactly, so an exact-CRT ModDown (v = the centred residue of acc mod P) or an uncentred
    conversion (y_k in [0, p_k)) fails; the overflow u = (v - [acc]_P) / P must also take more than one value."""
    o = _tiny_ks_ctx()
    level = 3
    rs = np.random.default_rng(10)
    ext_limbs = list(range(level)) + [o.L + k for k in range(o.alpha)]
    acc = np.stack([rs.integers(0, o.moduli[li], o.n, dtype=np.uint64) for li in ext_limbs])
    out = o.moddown(level, acc)
    P = o.p[0] * o.p[1]
    acc_c = np.stack([o.intt(li, acc[e]) for e, li in enumerate(ext_limbs)])
    out_c = np.stack([o.intt(i, out[i]) for i in range(level)])
    xp = [v % P for v in oracle.crt_centered(acc_c[level:], o.p)]      # [acc]_P in [0, P)
    us = set()
    for k in range(o.n):
        v = 0
        for kk, pk in enumerate(o.p):
            y = int(acc_c[level + kk, k]) * pow(P // pk, -1, pk) % pk
            v += (y - pk if y > pk // 2 else y) * (P // pk)
        assert (v - xp[k]) % P == 0
        us.add((v - xp[k]) // P)
        for i in range(level):
            q = o.q[i]
            assert (int(out_c[i, k]) * P + v - int(acc_c[i, k])) % q == 0, (i, k)
    assert len(us) > 1 and max(abs(u) for u in us) <= o.alpha


def test_rotation_decrypts_to_cyclic_shift(c1):
    """decrypt(Rot(ct; r)) == cyclic left shift by r; r<0 shifts right."""
    o, skc, sk, pk = c1
    gold = json.load(open(os.path.join(GOLD, "rotation_example.json")))
    z = np.zeros(o.n // 2)
    z[:4] = gold["input"]
    ct = o.encrypt(5, pk, 3, o.encode(z, 3, DELTA))
    g = o.galois(gold["k"])
    key = o.rotkey(6, g, sk)
    got = o.decrypt(sk, o.rotate(ct, g, key), DELTA)
    want = np.roll(z, -gold["k"])
    assert np.allclose(got[:3], gold["expected"][:3], atol=1e-5)
    assert np.max(np.abs(got - want)) < 1e-5
    # random vector, several shifts incl. negative, and Rot(Rot(ct,r),-r) ~ ct
    z = np.random.default_rng(11).uniform(-1, 1, o.n // 2)
    ct = o.encrypt(7, pk, 3, o.encode(z, 3, DELTA))
    for r in (1, 17, -5, 1000):
        g = o.galois(r)
        key = o.rotkey(100 + r, g, sk)
        rot = o.rotate(ct, g, key)
        assert np.max(np.abs(o.decrypt(sk, rot, DELTA) - np.roll(z, -r))) < 1e-5
        gi = o.galois(-r)
        back = o.rotate(rot, gi, o.rotkey(200 + r, gi, sk))
        assert np.max(np.abs(o.decrypt(sk, back, DELTA) - z)) < 1e-5


def test_rotation_noise_has_no_slot0_spike():
    """R10: ModDown converts centred P-residues, so the conversion overflow is zero-mean and the v*s term does
    not pile up in the lowest-frequency slot.  Rotation noise stays at the fresh-encryption level (N'=2^14)."""
    o = oracle.Oracle(14, 12, 4, 3)
    skc, sk, pk = o.keygen(5)
    ct = o.encrypt(5, pk, 12, o.encode(np.zeros(o.n // 2), 12, DELTA))
    fresh = np.max(np.abs(o.decrypt(sk, ct, DELTA)))
    g = o.galois(1)
    rot = o.rotate(ct, g, o.rotkey(777, g, sk))
    err = np.abs(o.decrypt(sk, rot, DELTA))
    assert err.max() < 2 * fresh
    assert err[0] < 5 * np.median(err) + fresh


def test_hoisted_equals_single_rotations(c1):
    o, skc, sk, pk = c1
    ct = synth.gen_words(21, o.q, 1, 2, o.n)[0]
    gs = [o.galois(r) for r in (1, 2, 33)]
    keys = np.stack([o.rotkey(300 + i, g, sk) for i, g in enumerate(gs)])
    hoisted = o.rotate_hoisted(ct, gs, keys)
    for i, g in enumerate(gs):
        assert (hoisted[i] == o.rotate(ct, g, keys[i])).all()


# ---------------------------------------------------------------- O11 Layout B

def test_layout_b_plan_counts():
    # C2 765 rotations with B=256, G=1; C1 15 rotations
    assert oracle.layout_b_plan(1 << 16, 128, 768, 768) == (256, 3, 256, 1, 765)
    assert oracle.layout_b_plan(1 << 12, 16, 16, 16) == (16, 1, 16, 1, 15)
    k, n_in, B, G, rots = oracle.layout_b_plan(1 << 16, 128, 3072, 768)
    assert rots == (B - 1) * n_in + (G - 1) * 768


def _layout_b_setup(o, sk, pk, X, s, k, seed):
    d = X.shape[1]
    n_in = -(-d // k)
    slots = o.n // 2
    cts = []
    for c in range(n_in):
        z = np.zeros(slots)
        for b in range(k):
            col = c * k + b
            if col < d:
                z[b * s:(b + 1) * s] = X[:, col]
        cts.append(o.encrypt(seed + c, pk, 3, o.encode(z, 3, DELTA)))
    return np.stack(cts)


@pytest.mark.parametrize("d,m,s,B", [(16, 16, 16, 0), (16, 16, 16, 1), (16, 16, 16, 4), (20, 6, 16, 4)])
def test_layout_b_decrypts_block0(c1, d, m, s, B):
    """Block 0 of y_i decrypts to (X.W)[:, i] within 1e-4; B=k and B=1 agree after decryption."""
    o, skc, sk, pk = c1
    k, n_in, B, G, rots = oracle.layout_b_plan(o.n, s, d, m, B)
    X = synth.gen_X(31 + d, s, d)
    W = synth.gen_W(32 + d, d, m)
    x = _layout_b_setup(o, sk, pk, X, s, k, 4000)
    gk = oracle.layout_b_galois(o.n, o.log_n, s, B, G)
    keys = np.stack([o.rotkey(5000 + i, g, sk) for i, g in enumerate(gk)])
    y = o.pcmm_b(x, W, s, k, B, gk, keys)
    ref = X @ W.astype(np.float64)
    for i in range(m):
        z = o.decrypt(sk, y[i], DELTA)
        assert np.max(np.abs(z[:s] - ref[:, i])) < 1e-4


@pytest.mark.parametrize("d,m,s,B", [(16, 16, 16, 1), (20, 6, 16, 4), (16, 16, 16, 8)])
def test_layout_b_lazy_moddown_decrypts_block0(c1, d, m, s, B):
    """R19: the lazy-ModDown Layout B (giant steps summed over Q_l u P, one ModDown per output) decrypts to the same
    (X.W)[:, i] within 1e-4 -- with G = 16, 4 and 2 giant steps -- and its noise is no larger than the eager
    form's plus one fresh-rotation error (one ModDown rounding instead of G - 1)."""
    o, skc, sk, pk = c1
    k, n_in, B, G, rots = oracle.layout_b_plan(o.n, s, d, m, B)
    X = synth.gen_X(41 + d, s, d)
    W = synth.gen_W(42 + d, d, m)
    x = _layout_b_setup(o, sk, pk, X, s, k, 4100)
    gk = oracle.layout_b_galois(o.n, o.log_n, s, B, G)
    keys = np.stack([o.rotkey(5100 + i, g, sk) for i, g in enumerate(gk)])
    y = o.pcmm_b(x, W, s, k, B, gk, keys, lazy=True)
    ye = o.pcmm_b(x, W, s, k, B, gk, keys)
    ref = X @ W.astype(np.float64)
    for i in range(m):
        z = o.decrypt(sk, y[i], DELTA)
        ze = o.decrypt(sk, ye[i], DELTA)
        assert np.max(np.abs(z[:s] - ref[:, i])) < 1e-4
        assert np.max(np.abs(z - ze)) < 1e-5
    if G <= 2:
        assert (y == ye).all()


# ---------------------------------------------------------------- O12 rescale

def test_rescale_is_rounded_division(c1):
    """CRT(rescale(c)) == round(CRT(c) / q_last) coefficientwise (centred remainder), exact."""
    o = c1[0]
    ct = synth.gen_words(41, o.q, 1, 3, o.n)[0]
    out = o.rescale(ct)
    ql = o.q[2]
    for poly in range(2):
        cin = np.stack([o.intt(i, ct[poly, i]) for i in range(3)])
        cout = np.stack([o.intt(i, out[poly, i]) for i in range(2)])
        Qin = o.q[0] * o.q[1] * ql
        xin = [v % Qin for v in oracle.crt_centered(cin, o.q[:3])]
        xout = [v % (o.q[0] * o.q[1]) for v in oracle.crt_centered(cout, o.q[:2])]
        for k in range(0, o.n, 7):
            rem = xin[k] % ql
            if rem > ql // 2:
                rem -= ql
            want = ((xin[k] - rem) // ql) % (o.q[0] * o.q[1])
            assert xout[k] == want


def test_rescale_preserves_values_at_delta_squared(c1):
    o, skc, sk, pk = c1
    z = np.random.default_rng(12).uniform(-1, 1, o.n // 2)
    scale2 = DELTA * DELTA
    ct = o.encrypt(8, pk, 3, o.encode(z, 3, scale2))
    out = o.rescale(ct)
    got = o.decrypt(sk, out, scale2 / o.q[2])
    assert np.max(np.abs(got - z)) < 1e-6
