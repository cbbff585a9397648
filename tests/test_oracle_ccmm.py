"""Pins for the CCMM oracle primitives and composition (R18).

What the mathematics fixes, checked by routes that do not reuse the oracle's own arithmetic:
* the relinearisation key is a gadget towards s^2, with s^2 formed by a schoolbook negacyclic square of the
  ternary coefficient vector (numpy convolution), not by the oracle's NTT-domain square;
* the plaintext product in NTT form is the negacyclic polynomial product (schoolbook, Python integers);
* a ciphertext tensor product decrypts (under s, s^2) to the slot-wise product of the messages (CKKS Mult,
  PAPER.md:124-126), relinearisation keeps the decryption, rescale divides the scale;
* CCMM decrypts, head block by head block, to the float64 matrix product, in both forms
  (A.B with B column-encoded, and A.K^T with K column-encoded).
"""
import numpy as np
import pytest

import oracle

DELTA = 2.0 ** 40


def _negacyclic(a, b, n):
    full = np.convolve(np.asarray(a, dtype=object), np.asarray(b, dtype=object))
    out = [0] * n
    for k, v in enumerate(full):
        if k < n:
            out[k] += v
        else:
            out[k - n] -= v
    return out


def test_relinkey_gadget_identity(c1):
    """b_t + a_t s - e_t == [r in D_t] (P mod q_r) s^2 limb by limb; s^2 from a schoolbook negacyclic square."""
    o, skc, sk, pk = c1
    key, e = o.relinkey(4242, sk, want_e=True)
    sq = np.convolve(skc.astype(np.int64), skc.astype(np.int64))       # |coeff| <= N', exact in int64
    s2c = sq[:o.n].copy()
    s2c[:o.n - 1] -= sq[o.n:]
    P = 1
    for p in o.p:
        P *= p
    for t in range(o.dnum):
        for i in range(o.L + o.alpha):
            r = o.moduli[i]
            s2 = o.ntt(i, [int(v) % r for v in s2c])
            e_ntt = o.ntt(i, [int(v) % r for v in e[t]])
            lhs = [(int(b) + int(a) * int(s) - int(ee)) % r
                   for b, a, s, ee in zip(key[t, 0, i], key[t, 1, i], sk[i], e_ntt)]
            in_digit = i < o.L and t * o.alpha <= i < (t + 1) * o.alpha
            want = [(P % r) * int(v) % r if in_digit else 0 for v in s2]
            assert lhs == want


def test_mul_plain_is_negacyclic_product():
    """INTT(ct (.) pt) == INTT(ct) * INTT(pt) mod (X^N' + 1, q) per limb (schoolbook, N' = 32)."""
    o = oracle.Oracle(5, 4, 2, 2)
    rs = np.random.default_rng(21)
    level = 3
    ct = np.stack([np.stack([rs.integers(0, o.q[i], o.n, dtype=np.uint64) for i in range(level)]) for _ in range(2)])
    pt = np.stack([rs.integers(0, o.q[i], o.n, dtype=np.uint64) for i in range(level)])
    out = o.mul_plain(ct, pt)
    for p in range(2):
        for i in range(level):
            q = o.q[i]
            a = [int(v) for v in o.intt(i, ct[p, i])]
            b = [int(v) for v in o.intt(i, pt[i])]
            want = [v % q for v in _negacyclic(a, b, o.n)]
            assert [int(v) for v in o.intt(i, out[p, i])] == want


def test_mul_ct_relin_rescale_decrypt_to_slot_product(c1):
    """Tensor product -> slot-wise product at scale Delta^2; relinearisation keeps it; rescale divides by q_last."""
    o, skc, sk, pk = c1
    rs = np.random.default_rng(22)
    x, y = rs.uniform(-1, 1, o.n // 2), rs.uniform(-1, 1, o.n // 2)
    cx = o.encrypt(31, pk, 3, o.encode(x, 3, DELTA))
    cy = o.encrypt(32, pk, 3, o.encode(y, 3, DELTA))
    d3 = o.mul_ct(cx, cy)
    assert np.max(np.abs(o.decrypt3(sk, d3, DELTA * DELTA) - x * y)) < 1e-6
    rlk = o.relinkey(33, sk)
    r = o.relin(d3, rlk)
    assert np.max(np.abs(o.decrypt(sk, r, DELTA * DELTA) - x * y)) < 1e-6
    out = o.rescale(r)
    assert np.max(np.abs(o.decrypt(sk, out, DELTA * DELTA / o.q[2]) - x * y)) < 1e-6


def _ccmm_setup(o, sk, pk, form, s, d, m, seed):
    """Per head h (H = (N'/2)/s blocks): A_h (s x d) and B_h (d x m) [form 2] or K_h (m x d) [form 1]."""
    H = (o.n // 2) // s
    rs = np.random.default_rng(seed)
    A = rs.uniform(-1, 1, (H, s, d))
    level = 3

    def enc(cols, sd):
        m_res = np.stack([o.encode(z, level, DELTA) for z in cols])
        return o.encrypt_batch(np.arange(len(cols), dtype=np.uint64) + np.uint64(sd), pk, level, m_res)

    def slots(mat_cols):                        # mat_cols [H][rows][ncols] -> one slot vector per column
        Hh, rows, nc = mat_cols.shape
        out = np.zeros((nc, o.n // 2))
        for h in range(Hh):
            out[:, h * s:h * s + rows] = mat_cols[h].T
        return out

    a = enc(slots(A), seed)
    if form == 2:
        Bm = rs.uniform(-1, 1, (H, d, m))
        src = enc(slots(Bm), seed + 1000)
        ref = np.einsum("hsd,hdm->hsm", A, Bm)
    else:
        K = rs.uniform(-1, 1, (H, m, d))
        src = enc(slots(K), seed + 1000)
        ref = np.einsum("hsd,hmd->hsm", A, K)
    pi, amounts, per_out, _ = oracle.ccmm_plan(form, s, d, m)
    z = np.zeros(o.n // 2)
    for h in range(H):
        z[h * s:h * s + s:pi] = 1.0
    coeffs = o.encode(z, level, float(o.q[level - 1]))
    mask = np.stack([o.ntt(i, coeffs[i]) for i in range(level)])
    keys = {o.galois(r): o.rotkey(5000 + k, o.galois(r), sk) for k, r in enumerate(amounts)}
    rlk = o.relinkey(6000, sk)
    return a, src, mask, keys, rlk, ref


@pytest.mark.parametrize("form,s,d,m", [(2, 16, 4, 3), (2, 16, 3, 2), (2, 4, 1, 2), (2, 16, 11, 2), (1, 16, 4, 3),
                                        (1, 8, 2, 8), (1, 16, 3, 11)])
def test_ccmm_decrypts_to_matrix_product(c1, form, s, d, m):
    o, skc, sk, pk = c1
    a, src, mask, keys, rlk, ref = _ccmm_setup(o, sk, pk, form, s, d, m, 900 + 10 * form + d)
    y = o.ccmm(a, src, form, s, d, m, mask, keys, rlk)
    assert y.shape == (m, 2, 1, o.n)
    scale = DELTA * DELTA / o.q[1]
    H = (o.n // 2) // s
    for i in range(m):
        z = o.decrypt(sk, y[i], scale)
        got = z.reshape(H, s)
        assert np.max(np.abs(got - ref[:, :, i])) < 1e-4, (i, np.max(np.abs(got - ref[:, :, i])))


def test_ccmm_plan_counts():
    """Table III shapes: 105 keys instead of ~2060 with the baby-step giant-step alignment."""
    pi, amounts, per, Ba = oracle.ccmm_plan(2, 2048, 96, 96)
    assert pi == 128 and Ba == 16 and per == 4 + 15 + 80 + 96 * 7
    assert set(amounts) == set(range(1, 16)) | {16 * g for g in range(1, 6)} | {-(1 << u) for u in range(7)} \
        | {-128 * (1 << u) for u in range(4)}
    pi, amounts, per, Ba = oracle.ccmm_plan(2, 2048, 2048, 96)         # S (2048 x 2048) . V (2048 x 96)
    assert pi == 2048 and Ba == 64 and len(amounts) == 63 + 31 + 11 and per == 2047 + 2048 * 11
    pi, amounts, per, Ba = oracle.ccmm_plan(1, 2048, 96, 2048)         # Q (2048 x 96) . K^T
    assert pi == 2048 and Ba == 64 and len(amounts) == 63 + 31 + 11 and per == 96 * 2 + 96 * 11
