"""Independent big-integer mini-oracle for N' <= 256 ("an independent Python big-integer
mini-oracle for N' <= 256 cross-checks the C oracle word for word").

TEST INFRASTRUCTURE ONLY (like the rest of oracle/): only tests/ import it.  It shares no code with
``ensi_oracle.c`` nor with the CUDA path: every step is written from its definition with Python integers,
by a different route wherever one exists, so that a slip in the C oracle's index algebra, digit handling or
rounding convention shows up as a word mismatch:

* NTT      -- the defining sum NTT(a)[k] = sum_i a_i psi^{(2 brv(k)+1) i} (O2), O(N'^2); INTT solves it back
              with the explicit inverse sum (N'^{-1} sum_k A_k psi^{-(2 brv(k)+1) i}).
* sigma_g  -- in the COEFFICIENT domain, a(X) -> a(X^g) with X^{N'} = -1 (O9), then the NTT (the C oracle
              permutes NTT slots by index algebra instead).
* ModUp    -- per digit the exact integer sum_i y_i (Q_t/q_i) reduced mod every target r (O10: "no overflow
              correction", so ext = x + u Q_t with 0 <= u < |D_t|), instead of per-target modular sums.
* ModDown  -- the exact signed integer v = sum_k y_k (P/p_k) with y_k centred in (-p_k/2, p_k/2] (R10),
              reduced mod q_i, then (acc - NTT(v)) P^{-1}.
* Rot      -- ModUp first, then sigma_g on every extended digit (O10), KIP, ModDown, + sigma_g(c0).
* Layout B -- O11 step by step (baby rotations, Algorithm-1 partial sums, giant rotations, sum).
* rescale  -- O12 in the coefficient domain: (c_i - t) q_{l-1}^{-1} with t the centred last limb, then NTT.
* CCMM     -- R18 step by step (periodic copy, giant-then-baby alignment, mask + rescale, doubling replication,
              tensor products summed, relinearisation = the key switch of d2 with no automorphism, rescale), with
              rotations taken one at a time (hoisted rotations are the same words by the O10 definition).

Ciphertexts are lists of polynomials: ct[poly][limb] = list of N' Python ints (NTT form, canonical).
"""
from __future__ import annotations


def _brv(x: int, bits: int) -> int:
    r = 0
    for _ in range(bits):
        r = (r << 1) | (x & 1)
        x >>= 1
    return r


def min_root(q: int, n: int) -> int:
    """O2: the smallest x in [1, q) with x^{N'} = -1 mod q (a primitive 2N'-th root); every primitive 2N'-th root is
    an odd power of any one of them."""
    assert (q - 1) % (2 * n) == 0
    for base in range(2, 1000):
        r = pow(base, (q - 1) // (2 * n), q)
        if pow(r, n, q) == q - 1:
            break
    else:
        raise ValueError("no 2N'-th root found")
    return min(pow(r, 2 * j + 1, q) for j in range(n))


class Mini:
    """One parameter set: moduli q_0..q_{L-1}, p_0..p_{alpha-1} (given, e.g. the O1 rule's), dnum digits."""

    def __init__(self, log_n: int, q: list, p: list, dnum: int):
        self.log_n, self.n = log_n, 1 << log_n
        self.q, self.p = [int(v) for v in q], [int(v) for v in p]
        self.L, self.alpha, self.dnum = len(self.q), len(self.p), dnum
        self.moduli = self.q + self.p
        self._pw = {}
        for m in self.moduli:
            psi = min_root(m, self.n)
            pw = [1] * (2 * self.n)
            for e in range(1, 2 * self.n):
                pw[e] = pw[e - 1] * psi % m
            self._pw[m] = pw

    # ---------------------------------------------------------------- O2
    def ntt(self, m: int, a: list) -> list:
        n, lg, pw = self.n, self.log_n, self._pw[m]
        out = []
        for k in range(n):
            e = 2 * _brv(k, lg) + 1
            out.append(sum(a[i] * pw[(e * i) % (2 * n)] for i in range(n)) % m)
        return out

    def intt(self, m: int, A: list) -> list:
        n, lg, pw = self.n, self.log_n, self._pw[m]
        ninv = pow(n, -1, m)
        out = []
        for i in range(n):
            s = 0
            for k in range(n):
                e = (2 * _brv(k, lg) + 1) * i % (2 * n)
                s += A[k] * pw[(2 * n - e) % (2 * n)]
            out.append(s * ninv % m)
        return out

    # ---------------------------------------------------------------- O9
    def automorph_coeff(self, m: int, a: list, g: int) -> list:
        """a(X) -> a(X^g) in Z_m[X]/(X^{N'}+1)."""
        n = self.n
        out = [0] * n
        for i, c in enumerate(a):
            e = i * g % (2 * n)
            if e < n:
                out[e] = (out[e] + c) % m
            else:
                out[e - n] = (out[e - n] - c) % m
        return out

    def automorph_ntt(self, m: int, A: list, g: int) -> list:
        return self.ntt(m, self.automorph_coeff(m, self.intt(m, A), g))

    def galois(self, r: int) -> int:
        return pow(5, r % (self.n // 2), 2 * self.n)

    # ---------------------------------------------------------------- O10
    def _ext_moduli(self, level: int) -> list:
        return self.q[:level] + self.p

    def _digits(self, level: int) -> list:
        a = self.alpha
        return [list(range(t * a, min((t + 1) * a, level))) for t in range(-(-level // a))]

    def modup(self, level: int, c: list) -> list:
        """c [level][N'] NTT form -> [beta][level + alpha][N'] NTT form over Q_l u P."""
        ext_mod = self._ext_moduli(level)
        out = []
        for D in self._digits(level):
            Qt = 1
            for i in D:
                Qt *= self.q[i]
            coef = {i: self.intt(self.q[i], c[i]) for i in D}
            # y_i = [c_i (Q_t/q_i)^{-1}]_{q_i}; the exact integer X = sum_i y_i (Q_t/q_i) (no correction: X = x + u Q_t)
            ys = {i: [v * pow(Qt // self.q[i], -1, self.q[i]) % self.q[i] for v in coef[i]] for i in D}
            X = [sum(ys[i][k] * (Qt // self.q[i]) for i in D) for k in range(self.n)]
            rows = []
            for e, r in enumerate(ext_mod):
                if e < level and e in D:
                    rows.append(list(c[e]))                       # the digit's own limbs: the input's NTT words
                else:
                    rows.append(self.ntt(r, [v % r for v in X]))
            out.append(rows)
        return out

    def moddown(self, level: int, acc: list, variant: str = "centred") -> list:
        """acc [level + alpha][N'] NTT form over Q_l u P -> [level][N'] NTT form over Q_l.  variant "centred" is
        R10 (the definition); "uncentred" (y_k in [0, p_k)) and "exact" (v = the centred residue of acc mod P,
        an exact CRT) exist only so tests can show the cross-check tells the conventions apart."""
        P = 1
        for pk in self.p:
            P *= pk
        pc = [self.intt(pk, acc[level + k]) for k, pk in enumerate(self.p)]
        v = [0] * self.n
        for k, pk in enumerate(self.p):
            w = pow(P // pk, -1, pk)
            for j in range(self.n):
                y = pc[k][j] * w % pk
                if y > pk // 2 and variant == "centred":
                    y -= pk                                        # centred in (-p_k/2, p_k/2]
                v[j] += y * (P // pk)
        if variant == "exact":
            v = [x % P - (P if x % P > P // 2 else 0) for x in v]
        out = []
        for i in range(level):
            qi = self.q[i]
            z = self.ntt(qi, [x % qi for x in v])
            pinv = pow(P, -1, qi)
            out.append([(acc[i][j] - z[j]) * pinv % qi for j in range(self.n)])
        return out

    def rotate(self, ct: list, g: int, key: list) -> list:
        """Rot(ct; g) (O9 + O10).  key [dnum][2][L + alpha][N'] (key[t][0] = b_t, key[t][1] = a_t)."""
        level = len(ct[0])
        if g % (2 * self.n) == 1:
            return [[list(r) for r in ct[0]], [list(r) for r in ct[1]]]
        ext_mod = self._ext_moduli(level)
        ext_idx = list(range(level)) + [self.L + k for k in range(self.alpha)]
        dig = self.modup(level, ct[1])                              # ModUp first ...
        dig = [[self.automorph_ntt(ext_mod[e], row, g) for e, row in enumerate(d)] for d in dig]   # ... then sigma_g
        ks = []
        for j in range(2):
            acc = []
            for e, r in enumerate(ext_mod):
                acc.append([sum(dig[t][e][k] * key[t][j][ext_idx[e]][k] for t in range(len(dig))) % r
                            for k in range(self.n)])
            ks.append(self.moddown(level, acc))
        c0g = [self.automorph_ntt(self.q[i], ct[0][i], g) for i in range(level)]
        out0 = [[(c0g[i][k] + ks[0][i][k]) % self.q[i] for k in range(self.n)] for i in range(level)]
        return [out0, ks[1]]

    def rotate_parts(self, ct: list, g: int, key: list):
        """Rot(ct; g) before its ModDown (R19): (sigma_g(c0), [acc_0, acc_1]) with acc_j over Q_l u P, so that
        Rot = (sigma_g(c0) + ModDown(acc_0), ModDown(acc_1))."""
        level = len(ct[0])
        ext_mod = self._ext_moduli(level)
        ext_idx = list(range(level)) + [self.L + k for k in range(self.alpha)]
        dig = self.modup(level, ct[1])
        dig = [[self.automorph_ntt(ext_mod[e], row, g) for e, row in enumerate(d)] for d in dig]
        accs = [[[sum(dig[t][e][k] * key[t][j][ext_idx[e]][k] for t in range(len(dig))) % r for k in range(self.n)]
                 for e, r in enumerate(ext_mod)] for j in range(2)]
        return [self.automorph_ntt(self.q[i], ct[0][i], g) for i in range(level)], accs

    # ---------------------------------------------------------------- O8 / O11
    def add(self, a: list, b: list, sign: int = 1) -> list:
        return [[[(x + sign * y) % self.q[i] for x, y in zip(a[p][i], b[p][i])] for i in range(len(a[p]))]
                for p in range(2)]

    def zero(self, level: int) -> list:
        return [[[0] * self.n for _ in range(level)] for _ in range(2)]

    def pcmm_a(self, x: list, W) -> list:
        """Algorithm 1: y_i = sum_j W[j][i] x_j from the trivial ciphertext (0, 0)."""
        d, m = len(W), len(W[0])
        level = len(x[0][0])
        ys = []
        for i in range(m):
            y = self.zero(level)
            for j in range(d):
                if W[j][i]:
                    y = self.add(y, x[j], int(W[j][i]))
            ys.append(y)
        return ys

    def pcmm_b(self, x: list, W, s: int, k: int, B: int, keys: dict, lazy: bool = False) -> list:
        """O11: R_{c,b} = Rot(ct_c; s b), T_{i,gam} = sum_{c,b} W[c k + gam B + b][i] R_{c,b},
        y_i = T_{i,0} + sum_{gam >= 1} Rot(T_{i,gam}; s B gam).  keys: {galois element: key}.
        lazy (R19): the giant rotations' KIP outputs are summed over Q_l u P and ModDown'ed once per output."""
        d, m = len(W), len(W[0])
        level = len(x[0][0])
        G = k // B
        R = {}
        for c in range(len(x)):
            for b in range(B):
                g = self.galois(s * b)
                R[c, b] = x[c] if b == 0 else self.rotate(x[c], g, keys[g])
        ext_mod = self._ext_moduli(level)
        ys = []
        for i in range(m):
            y = self.zero(level)
            la = [[[0] * self.n for _ in ext_mod] for _ in range(2)]
            for gam in range(G):
                T = self.zero(level)
                for c in range(len(x)):
                    for b in range(B):
                        col = c * k + gam * B + b
                        if col < d and W[col][i]:
                            T = self.add(T, R[c, b], int(W[col][i]))
                if gam:
                    g = self.galois(s * B * gam)
                    if lazy:
                        c0g, accs = self.rotate_parts(T, g, keys[g])
                        y[0] = [[(a + b) % self.q[r] for a, b in zip(y[0][r], c0g[r])] for r in range(level)]
                        la = [[[(a + b) % ext_mod[e] for a, b in zip(la[j][e], accs[j][e])] for e in range(len(ext_mod))]
                              for j in range(2)]
                        continue
                    T = self.rotate(T, g, keys[g])
                y = self.add(y, T)
            if lazy and G > 1:
                y = self.add(y, [self.moddown(level, la[0]), self.moddown(level, la[1])])
            ys.append(y)
        return ys

    # ---------------------------------------------------------------- R18 (CCMM)
    def mul_plain(self, ct: list, pt: list) -> list:
        """slot-wise (NTT-domain) product of both polynomials with the plaintext pt [level][N']."""
        return [[[x * y % self.q[i] for x, y in zip(ct[p][i], pt[i])] for i in range(len(ct[p]))] for p in range(2)]

    def mul_ct(self, a: list, b: list) -> list:
        """(a0 b0, a0 b1 + a1 b0, a1 b1), NTT domain."""
        level = len(a[0])
        d0 = [[x * y % self.q[i] for x, y in zip(a[0][i], b[0][i])] for i in range(level)]
        d1 = [[(x * y + u * v) % self.q[i] for x, y, u, v in zip(a[0][i], b[1][i], a[1][i], b[0][i])]
              for i in range(level)]
        d2 = [[x * y % self.q[i] for x, y in zip(a[1][i], b[1][i])] for i in range(level)]
        return [d0, d1, d2]

    def relin(self, d: list, key: list) -> list:
        """(d0 + ModDown(KIP_0), d1 + ModDown(KIP_1)) with KIP over ModUp(d2) and the relinearisation key (no
        automorphism)."""
        level = len(d[0])
        ext_mod = self._ext_moduli(level)
        ext_idx = list(range(level)) + [self.L + k for k in range(self.alpha)]
        dig = self.modup(level, d[2])
        ks = []
        for j in range(2):
            acc = [[sum(dig[t][e][k] * key[t][j][ext_idx[e]][k] for t in range(len(dig))) % r for k in range(self.n)]
                   for e, r in enumerate(ext_mod)]
            ks.append(self.moddown(level, acc))
        return [[[(x + y) % self.q[i] for x, y in zip(d[j][i], ks[j][i])] for i in range(level)] for j in range(2)]

    def ccmm(self, a: list, src: list, form: int, s: int, d: int, m: int, mask: list, keys: dict, rlk: list,
             Ba: int) -> list:
        """R18: per output column i -- form 2: P_i = b_i, P_i += Rot(P_i, -pi 2^u) (u < log2(s/pi));
        R_j = Rot(Rot(P_i, gam Ba), b) for j = gam Ba + b < d; form 1: R_j = Rot(Rot(k_j, gam Ba), b) for
        i = gam Ba + b; M_j = Rescale(R_j (.) mask); M_j += Rot(M_j, -2^u) (u < log2 pi); D_i = sum_j
        a_j|_{l-1} (x) M_j; c_i = Rescale(Relin(D_i)).  Rot(., 0) is the identity."""
        pi = s if form == 1 else 1 << max(0, (d - 1).bit_length())
        lg = lambda v: v.bit_length() - 1

        def rot(x, r):
            if r == 0:
                return x
            g = self.galois(r)
            return self.rotate(x, g, keys[g])

        out = []
        for i in range(m):
            if form == 2:
                P = src[i]
                for u in range(lg(s // pi)):
                    P = self.add(P, rot(P, -pi * (1 << u)))
                R = [rot(rot(P, (j // Ba) * Ba), j % Ba) for j in range(d)]
            else:
                R = [rot(rot(src[j], (i // Ba) * Ba), i % Ba) for j in range(d)]
            D = None
            for j in range(d):
                M = self.rescale(self.mul_plain(R[j], mask))
                for u in range(lg(pi)):
                    M = self.add(M, rot(M, -(1 << u)))
                aj = [[list(r) for r in a[j][p][:len(M[0])]] for p in range(2)]
                t = self.mul_ct(aj, M)
                D = t if D is None else [[[(x + y) % self.q[r] for x, y in zip(D[c][r], t[c][r])]
                                          for r in range(len(t[c]))] for c in range(3)]
            out.append(self.rescale(self.relin(D, rlk)))
        return out

    # ---------------------------------------------------------------- O12
    def rescale(self, ct: list) -> list:
        level = len(ct[0])
        ql = self.q[level - 1]
        out = []
        for p in range(2):
            t = self.intt(ql, ct[p][level - 1])
            t = [v - ql if v > ql // 2 else v for v in t]            # centred last limb
            rows = []
            for i in range(level - 1):
                qi = self.q[i]
                ci = self.intt(qi, ct[p][i])
                inv = pow(ql, -1, qi)
                rows.append(self.ntt(qi, [(a - b) * inv % qi for a, b in zip(ci, t)]))
            out.append(rows)
        return out
