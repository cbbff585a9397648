"""CPU oracle for the ENSI ternary-PCMM hot path (arXiv 2509.09424).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package.  It shares no code with the CUDA path
(paper_2509_09424_b200/); neither imports the other.

The arithmetic lives in ``ensi_oracle.c`` (plain loops, ``%``-reduced 128-bit products); this module
is ctypes marshalling plus the float64 encode/decode and big-integer CRT that the paper's client
performs:

* ``encode``  -- O5: slot u <-> evaluation at zeta^{5^u mod 2N'}, m = round_half_away(Delta * tau^{-1}(z)),
  tau^{-1} evaluated with numpy's FFT (a library primitive used as one step).
* ``decode``  -- O7: z_u = Re m(zeta^{5^u}) / Delta.
* ``crt_centered`` -- O7: CRT over all l limbs with Python integers, centred lift.
* ``Oracle.ccmm``  -- R18: the ciphertext-ciphertext matrix product of PAPER.md:343-360
  (c_i = sum_j a_j (x) rep(B_ji)), element extraction by mask + rotations, composed step by step from
  the C primitives (rotation, plaintext product, tensor product, relinearisation, rescale).

Parity status per function is listed in DESIGN.md section "Oracle pins"; key switching bit patterns
(O10) are pinned by exact CRT identities and decryption, not by external vectors.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import build as _build

_LIB = None

u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
i8p = np.ctypeslib.ndpointer(dtype=np.int8, flags="C_CONTIGUOUS")
u32p = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")


def lib():
    global _LIB
    if _LIB is None:
        path = _build.build()
        L = C.CDLL(path)
        L.or_ctx_create.restype = C.c_void_p
        L.or_ctx_create.argtypes = [C.c_uint32] * 4 + [C.c_void_p, C.c_void_p]
        L.or_ctx_destroy.argtypes = [C.c_void_p]
        L.or_ctx_moduli.argtypes = [C.c_void_p, u64p, u64p]
        L.or_min_root.restype = C.c_uint64
        L.or_min_root.argtypes = [C.c_uint64, C.c_uint32]
        L.or_gen_params.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, u64p, u64p]
        L.or_ntt.argtypes = [C.c_void_p, C.c_uint32, u64p]
        L.or_intt.argtypes = [C.c_void_p, C.c_uint32, u64p]
        L.or_rng_fill.argtypes = [C.c_uint64, C.c_int, C.c_uint64, C.c_uint64, i64p]
        L.or_keygen.argtypes = [C.c_void_p, C.c_uint64, i8p, u64p, u64p]
        L.or_rotkey.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, u64p, u64p, C.c_void_p]
        L.or_encrypt.argtypes = [C.c_void_p, C.c_uint64, u64p, C.c_uint32, u64p, u64p]
        L.or_encrypt_batch.argtypes = [C.c_void_p, u64p, C.c_uint32, u64p, C.c_uint32, u64p, u64p, C.c_uint32]
        L.or_decrypt.argtypes = [C.c_void_p, u64p, C.c_uint32, u64p, u64p]
        L.or_pcmm_a.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_void_p, i8p,
                                C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint32]
        L.or_automorph_ntt.argtypes = [C.c_uint32, C.c_uint64, C.c_uint32, u64p, u64p]
        L.or_automorph_coeff.argtypes = [C.c_void_p, C.c_uint32, C.c_uint64, u64p, u64p]
        L.or_modup.argtypes = [C.c_void_p, C.c_uint32, u64p, u64p]
        L.or_moddown.argtypes = [C.c_void_p, C.c_uint32, u64p, u64p]
        L.or_rotate_hoisted.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, u64p, u64p, u64p, u64p]
        L.or_rotate.argtypes = [C.c_void_p, C.c_uint32, C.c_uint64, u64p, u64p, u64p]
        L.or_galois_elt.restype = C.c_uint64
        L.or_galois_elt.argtypes = [C.c_uint32, C.c_int64]
        L.or_pcmm_b.restype = C.c_int
        L.or_pcmm_b.argtypes = [C.c_void_p] + [C.c_uint32] * 8 + [u64p, i8p, C.c_uint32, u64p, u64p, C.c_void_p,
                                                                 C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32]
        L.or_rescale.argtypes = [C.c_void_p, C.c_uint32, u64p, u64p]
        L.or_relinkey.argtypes = [C.c_void_p, C.c_uint64, u64p, u64p, C.c_void_p]
        L.or_mul_plain.argtypes = [C.c_void_p, C.c_uint32, u64p, u64p, u64p]
        L.or_mul_ct.argtypes = [C.c_void_p, C.c_uint32, u64p, u64p, u64p]
        L.or_relin.argtypes = [C.c_void_p, C.c_uint32, u64p, u64p, u64p]
        _LIB = L
    return _LIB


def gen_params(log_n: int, L: int, alpha: int):
    """O1 prime rule -> (q list, p list)."""
    q = np.zeros(L, np.uint64)
    p = np.zeros(max(alpha, 1), np.uint64)
    lib().or_gen_params(log_n, L, alpha, q, p)
    return [int(v) for v in q], [int(v) for v in p[:alpha]]


def min_root(q: int, log_n: int) -> int:
    """O2: minimal primitive 2N'-th root of unity mod q."""
    return int(lib().or_min_root(q, log_n))


def galois_elt(log_n: int, r: int) -> int:
    """O9: g = 5^r mod 2N' (left rotation by r)."""
    return int(lib().or_galois_elt(log_n, r))


def rng_fill(seed: int, kind: str, n: int, q: int = 0) -> np.ndarray:
    kinds = {"raw": 0, "uniform": 1, "ternary": 2, "cbd": 3}
    out = np.zeros(n, np.int64)
    lib().or_rng_fill(seed, kinds[kind], q, n, out)
    return out


# ---------------------------------------------------------------- encoding (O5) / decoding (O7)

def _slot_exponents(n: int) -> np.ndarray:
    """5^u mod 2N' for u in [0, N'/2)."""
    two_n = 2 * n
    e = np.empty(n // 2, np.int64)
    v = 1
    for u in range(n // 2):
        e[u] = v
        v = (v * 5) % two_n
    return e


def encode_coeffs(z, n: int, scale: float) -> list:
    """O5: real slot vector z (len <= N'/2, zero padded) -> integer coefficients (Python ints).

    m_j = (Delta/N') zeta^{-j} sum_t Z_{2t+1} e^{-2 pi i t j / N'} with Z at exponent 5^u = z_u and at
    -5^u = conj(z_u); round half away from zero in float64.
    """
    z = np.asarray(z, dtype=np.float64)
    slots = n // 2
    if z.shape[0] > slots:
        raise ValueError("more values than slots")
    zz = np.zeros(slots, np.complex128)
    zz[: z.shape[0]] = z
    e = _slot_exponents(n)
    Z = np.zeros(n, np.complex128)
    Z[(e - 1) // 2] = zz
    Z[((2 * n - e) - 1) // 2] = np.conj(zz)
    j = np.arange(n)
    m = np.fft.fft(Z) * np.exp(-1j * np.pi * j / n) / n
    v = m.real * scale
    r = np.sign(v) * np.floor(np.abs(v) + 0.5)
    return [int(x) for x in r]


def coeffs_to_residues(coeffs, moduli) -> np.ndarray:
    """Python-int coefficients -> [len(moduli)][N'] uint64 residues (c mod q, canonical)."""
    out = np.empty((len(moduli), len(coeffs)), np.uint64)
    if all(-(1 << 62) < c < (1 << 62) for c in coeffs):
        a = np.array(coeffs, dtype=np.int64)
        for i, q in enumerate(moduli):
            out[i] = np.mod(a, np.int64(q)).astype(np.uint64)
        return out
    for i, q in enumerate(moduli):
        out[i] = np.array([c % q for c in coeffs], dtype=np.uint64)
    return out


def crt_centered(res: np.ndarray, moduli) -> list:
    """O7: residues [l][N'] -> centred integers in (-Q/2, Q/2] (Python ints)."""
    moduli = [int(q) for q in moduli]
    Q = 1
    for q in moduli:
        Q *= q
    basis = []
    for q in moduli:
        qh = Q // q
        basis.append(qh * pow(qh % q, -1, q))
    n = res.shape[1]
    cols = [[int(v) for v in res[i]] for i in range(len(moduli))]
    out = []
    half = Q // 2
    for k in range(n):
        x = 0
        for i in range(len(moduli)):
            x += cols[i][k] * basis[i]
        x %= Q
        if x > half:
            x -= Q
        out.append(x)
    return out


def decode_coeffs(coeffs, n: int, scale: float) -> np.ndarray:
    """O7: z_u = Re sum_j m_j zeta^{5^u j} / Delta, evaluated as N' * ifft(m_j zeta^j) at t = (5^u-1)/2."""
    m = np.array([float(c) for c in coeffs], dtype=np.float64)
    j = np.arange(n)
    vals = np.fft.ifft(m * np.exp(1j * np.pi * j / n)) * n
    e = _slot_exponents(n)
    return vals[(e - 1) // 2].real / scale


# ---------------------------------------------------------------- context

class Oracle:
    """One CKKS parameter set (O1).  Limb order everywhere: q_0..q_{L-1}, p_0..p_{alpha-1}."""

    def __init__(self, log_n: int, L: int, alpha: int, dnum: int, q=None, p=None):
        self.log_n, self.n, self.L, self.alpha, self.dnum = log_n, 1 << log_n, L, alpha, dnum
        qa = np.ascontiguousarray(q, np.uint64) if q is not None else None
        pa = np.ascontiguousarray(p, np.uint64) if p is not None else None
        self._keep = (qa, pa)
        h = lib().or_ctx_create(log_n, L, alpha, dnum,
                                qa.ctypes.data if qa is not None else None,
                                pa.ctypes.data if pa is not None else None)
        if not h:
            raise ValueError("invalid oracle parameters")
        self.h = C.c_void_p(h)
        mods = np.zeros(L + alpha, np.uint64)
        psis = np.zeros(L + alpha, np.uint64)
        lib().or_ctx_moduli(self.h, mods, psis)
        self.moduli = [int(v) for v in mods]
        self.psi = [int(v) for v in psis]
        self.q = self.moduli[:L]
        self.p = self.moduli[L:]

    def __del__(self):
        try:
            lib().or_ctx_destroy(self.h)
        except Exception:
            pass

    # -- NTT (O2)
    def ntt(self, limb: int, a) -> np.ndarray:
        a = np.array(a, dtype=np.uint64, copy=True)
        lib().or_ntt(self.h, limb, a)
        return a

    def intt(self, limb: int, a) -> np.ndarray:
        a = np.array(a, dtype=np.uint64, copy=True)
        lib().or_intt(self.h, limb, a)
        return a

    # -- keys (O4)
    def keygen(self, seed: int):
        n, T = self.n, self.L + self.alpha
        skc = np.zeros(n, np.int8)
        sk = np.zeros((T, n), np.uint64)
        pk = np.zeros((2, self.L, n), np.uint64)
        lib().or_keygen(self.h, seed, skc, sk, pk)
        return skc, sk, pk

    def rotkey(self, seed: int, g: int, sk_ntt: np.ndarray, want_e: bool = False):
        n, T = self.n, self.L + self.alpha
        key = np.zeros((self.dnum, 2, T, n), np.uint64)
        e = np.zeros((self.dnum, n), np.int64) if want_e else None
        lib().or_rotkey(self.h, seed, g, np.ascontiguousarray(sk_ntt), key, e.ctypes.data if want_e else None)
        return (key, e) if want_e else key

    # -- encode / encrypt / decrypt (O5-O7)
    def encode(self, z, level: int, scale: float) -> np.ndarray:
        return coeffs_to_residues(encode_coeffs(z, self.n, scale), self.q[:level])

    def encrypt(self, seed: int, pk: np.ndarray, level: int, m_res: np.ndarray) -> np.ndarray:
        ct = np.zeros((2, level, self.n), np.uint64)
        lib().or_encrypt(self.h, seed, np.ascontiguousarray(pk), level, np.ascontiguousarray(m_res, np.uint64), ct)
        return ct

    def encrypt_batch(self, seeds, pk, level: int, m_res: np.ndarray, nthreads: int = 0) -> np.ndarray:
        seeds = np.ascontiguousarray(seeds, np.uint64)
        cnt = seeds.shape[0]
        ct = np.zeros((cnt, 2, level, self.n), np.uint64)
        nth = nthreads or min(cnt, os.cpu_count() or 1)
        lib().or_encrypt_batch(self.h, seeds, cnt, np.ascontiguousarray(pk), level,
                               np.ascontiguousarray(m_res, np.uint64), ct, nth)
        return ct

    def decrypt_residues(self, sk_ntt, ct: np.ndarray) -> np.ndarray:
        level = ct.shape[1]
        mu = np.zeros((level, self.n), np.uint64)
        lib().or_decrypt(self.h, np.ascontiguousarray(sk_ntt), level, np.ascontiguousarray(ct), mu)
        return mu

    def decrypt(self, sk_ntt, ct: np.ndarray, scale: float, limbs=None) -> np.ndarray:
        mu = self.decrypt_residues(sk_ntt, ct)
        level = ct.shape[1]
        use = list(range(level)) if limbs is None else list(limbs)
        coeffs = crt_centered(mu[use], [self.q[i] for i in use])
        return decode_coeffs(coeffs, self.n, scale)

    # -- PCMM Layout A (O8, Algorithm 1)
    def pcmm_a(self, x: np.ndarray, W: np.ndarray, cols=None, nthreads: int = 1) -> np.ndarray:
        x = np.ascontiguousarray(x, np.uint64)
        W = np.ascontiguousarray(W, np.int8)
        d, m = W.shape
        level = x.shape[2]
        assert x.shape[0] == d and x.shape[1] == 2 and x.shape[3] == self.n
        if cols is None:
            y = np.zeros((m, 2, level, self.n), np.uint64)
            lib().or_pcmm_a(self.h, level, d, m, m, x.ctypes.data, W, y.ctypes.data, None, 0, nthreads)
        else:
            ca = np.ascontiguousarray(cols, np.uint32)
            y = np.zeros((ca.shape[0], 2, level, self.n), np.uint64)
            lib().or_pcmm_a(self.h, level, d, m, m, x.ctypes.data, W, y.ctypes.data, ca.ctypes.data, ca.shape[0], nthreads)
        return y

    # -- automorphism / key switching / rotation (O9, O10)
    def automorph_ntt(self, g: int, rows: np.ndarray) -> np.ndarray:
        rows = np.ascontiguousarray(rows, np.uint64)
        out = np.zeros_like(rows)
        r = rows.reshape(-1, self.n)
        lib().or_automorph_ntt(self.log_n, g, r.shape[0], r, out.reshape(-1, self.n))
        return out

    def automorph_coeff(self, limb: int, g: int, a) -> np.ndarray:
        a = np.ascontiguousarray(a, np.uint64)
        out = np.zeros_like(a)
        lib().or_automorph_coeff(self.h, limb, g, a, out)
        return out

    def galois(self, r: int) -> int:
        return galois_elt(self.log_n, r)

    def modup(self, level: int, c: np.ndarray) -> np.ndarray:
        beta = -(-level // self.alpha)
        out = np.zeros((beta, level + self.alpha, self.n), np.uint64)
        lib().or_modup(self.h, level, np.ascontiguousarray(c, np.uint64), out)
        return out

    def moddown(self, level: int, acc: np.ndarray) -> np.ndarray:
        out = np.zeros((level, self.n), np.uint64)
        lib().or_moddown(self.h, level, np.ascontiguousarray(acc, np.uint64), out)
        return out

    def rotate(self, ct: np.ndarray, g: int, key: np.ndarray) -> np.ndarray:
        out = np.zeros_like(ct)
        lib().or_rotate(self.h, ct.shape[1], g, np.ascontiguousarray(key), np.ascontiguousarray(ct), out)
        return out

    def rotate_hoisted(self, ct: np.ndarray, gs, keys: np.ndarray) -> np.ndarray:
        ga = np.ascontiguousarray(gs, np.uint64)
        out = np.zeros((ga.shape[0],) + ct.shape, np.uint64)
        lib().or_rotate_hoisted(self.h, ct.shape[1], ga.shape[0], ga, np.ascontiguousarray(keys),
                                np.ascontiguousarray(ct), out)
        return out

    # -- PCMM Layout B (O11)
    def pcmm_b(self, x: np.ndarray, W: np.ndarray, s: int, k: int, B: int, gkeys, keys: np.ndarray, cols=None,
               nthreads: int = 1, lazy: bool = False) -> np.ndarray:
        """O11.  cols: compute only these output columns (returns one ciphertext per listed column).
        lazy (R19): the giant steps' key inner products are summed over Q_l u P and ModDown'ed once per
        output (y_i = T_{i,0} + sum_gam (sigma(T_{i,gam}.c0), 0) + ModDown(sum_gam KIP_gam)) -- identical words to
        the eager form when there is at most one giant rotation per output (G <= 2)."""
        W = np.ascontiguousarray(W, np.int8)
        d, m = W.shape
        n_in, _, level, _ = x.shape
        ca = None if cols is None else np.ascontiguousarray(cols, np.uint32)
        ncols = m if ca is None else ca.shape[0]
        y = np.zeros((ncols, 2, level, self.n), np.uint64)
        ga = np.ascontiguousarray(gkeys, np.uint64)
        rc = lib().or_pcmm_b(self.h, level, s, k, B, d, m, m, n_in, np.ascontiguousarray(x, np.uint64), W,
                             ga.shape[0], ga, np.ascontiguousarray(keys), y.ctypes.data,
                             ca.ctypes.data if ca is not None else None, ncols, nthreads, 1 if lazy else 0)
        if rc != 0:
            raise KeyError("missing rotation key")
        return y

    # -- rescale (O12)
    def rescale(self, ct: np.ndarray) -> np.ndarray:
        level = ct.shape[1]
        out = np.zeros((2, level - 1, self.n), np.uint64)
        lib().or_rescale(self.h, level, np.ascontiguousarray(ct, np.uint64), out)
        return out

    # -- CCMM primitives (R18)
    def relinkey(self, seed: int, sk_ntt: np.ndarray, want_e: bool = False):
        n, T = self.n, self.L + self.alpha
        key = np.zeros((self.dnum, 2, T, n), np.uint64)
        e = np.zeros((self.dnum, n), np.int64) if want_e else None
        lib().or_relinkey(self.h, seed, np.ascontiguousarray(sk_ntt), key, e.ctypes.data if want_e else None)
        return (key, e) if want_e else key

    def add(self, a: np.ndarray, b: np.ndarray) -> np.ndarray:
        """ciphertext addition (PAPER.md:124 Add): word-wise (a + b) mod q_r; a, b [..][l][N']"""
        level = a.shape[-2]
        q = np.array(self.q[:level], np.uint64).reshape(level, 1)
        return (a + b) % q

    def mul_plain(self, ct: np.ndarray, pt: np.ndarray) -> np.ndarray:
        out = np.zeros_like(ct)
        lib().or_mul_plain(self.h, ct.shape[1], np.ascontiguousarray(ct), np.ascontiguousarray(pt, np.uint64), out)
        return out

    def mul_ct(self, a: np.ndarray, b: np.ndarray) -> np.ndarray:
        level = a.shape[1]
        out = np.zeros((3, level, self.n), np.uint64)
        lib().or_mul_ct(self.h, level, np.ascontiguousarray(a), np.ascontiguousarray(b), out)
        return out

    def relin(self, d3: np.ndarray, key: np.ndarray) -> np.ndarray:
        level = d3.shape[1]
        out = np.zeros((2, level, self.n), np.uint64)
        lib().or_relin(self.h, level, np.ascontiguousarray(d3), np.ascontiguousarray(key), out)
        return out

    def ccmm(self, a: np.ndarray, src: np.ndarray, form: int, s: int, d: int, m: int, mask_pt: np.ndarray,
             rot_keys: dict, relin_key: np.ndarray, outputs=None) -> np.ndarray:
        """R18: C = A . B (form 2, ``src`` = the m column ciphertexts of B, d <= s) or C = A . K^T (form 1,
        ``src`` = the d column ciphertexts of K, m <= s), every head block of s slots in SIMD.
        a [d][2][l][N'] (level l >= 3), mask_pt [l][N'] = encode(1 at slots h s + u, u = 0 mod pi) at scale
        q_{l-1}; rot_keys {g: key}.  Returns the output columns ``outputs`` (default all m) at level l - 2.
        Steps per output column i, in this order (PAPER.md:354-359 c_i = sum_j a_j (x) b_i^(j)):
          1. form 2: periodic copy P_i = b_i; for u < log2(s/pi): P_i += Rot(P_i, -pi 2^u)
          2. align   R_j = Rot(P_i, j) (form 2) or Rot(k_j, i) (form 1), every amount r = gam B + b (B = the
                     baby count of ccmm_plan) taken as Rot(Rot(., gam B), b) -- giant step first (baby-step
                     giant-step: B + R/B keys instead of R; Rot(., 0) = identity).  Form 2: the giant steps of P_i
                     share one ModUp and the babies of each giant step share one (hoisted); form 1: contiguous
                     output columns of one giant step share Rot(k_j, gam B)
          3. mask    M_j = Rescale(R_j (.) mask)                       -> level l-1, scale Delta
          4. replicate: for u < log2(pi): M_j += Rot(M_j, -2^u)        -> rep(B_ji) on every slot of the block
          5. D_i = sum_j a_j|_{l-1} (x) M_j  (tensor products)
          6. c_i = Rescale(Relin(D_i))                                   -> level l-2"""
        level = a.shape[2]
        pi, _, _, Ba = ccmm_plan(form, s, d, m)
        lg = lambda v: v.bit_length() - 1
        key = lambda r: rot_keys[self.galois(r)]
        rot = lambda x, r: x if r == 0 else self.rotate(x, self.galois(r), key(r))
        outs = list(range(m)) if outputs is None else list(outputs)
        res = []
        for i in outs:
            if form == 2:
                P = src[i]
                for u in range(lg(s // pi)):
                    r = -pi * (1 << u)
                    P = self.add(P, self.rotate(P, self.galois(r), key(r)))
                zero = np.zeros_like(relin_key)
                G = -(-d // Ba)
                Gs = self.rotate_hoisted(P, [self.galois(g * Ba) for g in range(G)],
                                         np.stack([key(g * Ba) if g else zero for g in range(G)]))
                R = []
                for g in range(G):
                    nb = min(Ba, d - g * Ba)
                    R += list(self.rotate_hoisted(Gs[g], [self.galois(b) for b in range(nb)],
                                                  np.stack([key(b) if b else zero for b in range(nb)])))
                R = np.stack(R)
            else:
                b, gam = i % Ba, i // Ba
                R = np.stack([rot(rot(src[j], gam * Ba), b) for j in range(d)])
            D = None
            for j in range(d):
                M = self.rescale(self.mul_plain(R[j], mask_pt))
                for u in range(lg(pi)):
                    r = -(1 << u)
                    M = self.add(M, self.rotate(M, self.galois(r), key(r)))
                t = self.mul_ct(np.ascontiguousarray(a[j][:, :level - 1]), M)
                D = t if D is None else self.add(D, t)
            res.append(self.rescale(self.relin(D, relin_key)))
        return np.stack(res)

    def decrypt3(self, sk_ntt, d3: np.ndarray, scale: float) -> np.ndarray:
        """decrypt a 3-component product: mu = d0 + d1 s + d2 s^2 (NTT), INTT, CRT, decode"""
        level = d3.shape[1]
        s2 = self.mul_plain(np.stack([sk_ntt[:level], sk_ntt[:level]]), sk_ntt[:level])[0]
        ct2 = np.stack([self.add(d3[0], self.mul_plain(np.stack([d3[2], d3[2]]), s2)[0]), d3[1]])
        return self.decrypt(sk_ntt, ct2, scale)


def ccmm_plan(form: int, s: int, d: int, m: int):
    """R18 schedule: (period pi, rotation amounts that need keys, rotations per output column (form 1: the
    largest over the columns), baby count B).  Alignment amounts r < R (R = d for form 2, m for form 1) are
    r = gam B + b with B = 2^ceil(ceil(log2 R) / 2)."""
    pi = s if form == 1 else 1 << max(0, (d - 1).bit_length())
    lg = lambda v: v.bit_length() - 1
    R = d if form == 2 else m
    Ba = 1 << (((R - 1).bit_length() + 1) // 2)
    amounts = [-(1 << u) for u in range(lg(pi))]
    amounts += [b for b in range(1, min(Ba, R))] + [g * Ba for g in range(1, -(-R // Ba))]
    if form == 2:
        amounts += [-pi * (1 << u) for u in range(lg(s // pi))]
        per_out = lg(s // pi) + (min(Ba, d) - 1) + (d - min(Ba, d)) + d * lg(pi)
    else:
        per_out = d * ((1 if R > 1 else 0) + (1 if R > Ba else 0)) + d * lg(pi)
    return pi, sorted(set(amounts)), per_out, Ba


def layout_b_plan(n: int, s: int, d: int, m: int, B: int = 0):
    """O11 schedule: k = min((N'/2)/s, 2^ceil(log2 d)), n_in = ceil(d/k), B | k power of two,
    default B = argmin (B-1) n_in + (k/B - 1) m.  Returns (k, n_in, B, G, rotations)."""
    k = min((n // 2) // s, 1 << max(0, (d - 1).bit_length()))
    n_in = -(-d // k)
    if B == 0:
        best = None
        b = 1
        while b <= k:
            cost = (b - 1) * n_in + (k // b - 1) * m
            if best is None or cost < best[0]:
                best = (cost, b)
            b *= 2
        B = best[1]
    G = k // B
    return k, n_in, B, G, (B - 1) * n_in + (G - 1) * m


def layout_b_galois(n: int, log_n: int, s: int, B: int, G: int):
    """Galois elements Layout B needs: 5^{s b} (b in [1,B)) and 5^{s B gam} (gam in [1,G))."""
    gs = [galois_elt(log_n, s * b) for b in range(1, B)]
    gs += [galois_elt(log_n, s * B * g) for g in range(1, G)]
    out = []
    for g in gs:
        if g not in out:
            out.append(g)
    return out
