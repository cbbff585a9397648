/*
 * oracle/ensi_oracle.c -- plain, slow CPU oracle for the ENSI ternary-PCMM hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or constant generator with paper_2509_09424_b200/csrc (the CUDA path).
 *
 * Every routine is written as the textbook definition or the step-by-step algorithm,
 * with 128-bit products reduced by the C '%' operator (no Barrett, no Shoup, no lazy
 * reduction).  Citations: PAPER.md = /root/reference/PAPER.md (arXiv 2509.09424 LaTeX),
 * SURVEY.md section 8(c) rows O1..O12 give the readings used where the paper is silent.
 *
 * Function -> passage -> pin (tests/test_oracle_*.py):
 *   or_ctx_create   O1 prime rule (paper silent)   pinned: SURVEY App. A table + sympy
 *   or_min_root     O2 minimal primitive 2N'-th root                    pinned: App. A psi column, x^N' = -1
 *   or_ntt/or_intt  O2 NTT(a)[k] = sum_i a_i psi^{(2brv(k)+1) i}        pinned: direct sum, schoolbook conv.
 *   or_keygen       O4 ("Random sampling")                 pinned: decrypt identity
 *   or_rotkey       O4 gadget b_t + a_t s = e_t + [r in D_t] P s'(g)    pinned: gadget identity test
 *   or_encrypt      O6 Enc_pk                            pinned: encrypt->decrypt identity
 *   or_decrypt      O7 Dec_sk                            pinned: identity + CRT invariant
 *   or_pcmm_a       O8 Algorithm 1                    pinned: toy example, X.W float, perms
 *   or_automorph    O9 sigma_g (PAPER.md:134-138 Rot)                    pinned: coeff closed form, slot shift
 *   or_modup/...    O10 hybrid key switching (paper silent: evk only)    pinned: CRT identities, decrypt
 *   or_rotate*      O9+O10                                              pinned: decrypt == cyclic shift
 *   or_pcmm_b       O11 Layout B (our construction)         pinned: decrypt block 0 == X.W
 *                   lazy = 1: R19 lazy ModDown of the giant steps        pinned: == eager at G <= 2, mini-oracle,
 *                                                                          decrypt block 0 == X.W
 *   or_rescale      O12                                   pinned: == round(c/q_last) (big int)
 *   or_relinkey     O4 gadget towards s^2 (CCMM, R18)                    pinned: gadget identity test
 *   or_mul_plain    pt x ct in NTT form (R18)                            pinned: schoolbook negacyclic product
 *   or_mul_ct       tensor product (PAPER.md:124-126 Mult)                pinned: d0+d1 s+d2 s^2 == m_a m_b (big int)
 *   or_relin        O10 with the relinearisation key                     pinned: decrypt(relin(d)) ~ decrypt3(d)
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

typedef unsigned __int128 u128;

/* ------------------------------------------------------------------ modular arithmetic */
static uint64_t mulmod(uint64_t a, uint64_t b, uint64_t q) { return (uint64_t)(((u128)a * b) % q); }
/* a, b canonical in [0, q): the sum/difference reduced by one conditional correction (q < 2^62). */
static uint64_t addmod(uint64_t a, uint64_t b, uint64_t q) { uint64_t s = a + b; return s >= q ? s - q : s; }
static uint64_t submod(uint64_t a, uint64_t b, uint64_t q) { return a >= b ? a - b : a + q - b; }
static uint64_t powmod(uint64_t a, uint64_t e, uint64_t q) {
    uint64_t r = 1 % q; a %= q;
    while (e) { if (e & 1) r = mulmod(r, a, q); a = mulmod(a, a, q); e >>= 1; }
    return r;
}
/* q prime: Fermat inverse */
static uint64_t invmod(uint64_t a, uint64_t q) { return powmod(a % q, q - 2, q); }
/* signed int64 -> [0,q) */
static uint64_t smod(int64_t v, uint64_t q) {
    int64_t r = v % (int64_t)q;
    return (uint64_t)(r < 0 ? r + (int64_t)q : r);
}

/* deterministic Miller-Rabin, valid for all n < 2^64 with these bases */
static int is_prime_u64(uint64_t n) {
    static const uint64_t bases[12] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    if (n < 2) return 0;
    for (int i = 0; i < 12; i++) { if (n % bases[i] == 0) return n == bases[i]; }
    uint64_t d = n - 1; int s = 0;
    while ((d & 1) == 0) { d >>= 1; s++; }
    for (int i = 0; i < 12; i++) {
        uint64_t x = powmod(bases[i], d, n);
        if (x == 1 || x == n - 1) continue;
        int comp = 1;
        for (int r = 1; r < s; r++) { x = mulmod(x, x, n); if (x == n - 1) { comp = 0; break; } }
        if (comp) return 0;
    }
    return 1;
}

static uint32_t brv(uint32_t x, uint32_t bits) {
    uint32_t r = 0;
    for (uint32_t i = 0; i < bits; i++) { r = (r << 1) | (x & 1); x >>= 1; }
    return r;
}

/* ------------------------------------------------------------------ RNG (O3) */
/* xoshiro256** seeded through SplitMix64.  Draw order is documented per function. */
typedef struct { uint64_t s[4]; } rng_t;
static uint64_t splitmix64(uint64_t* x) {
    uint64_t z = (*x += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
static void rng_seed(rng_t* r, uint64_t seed) { uint64_t x = seed; for (int i = 0; i < 4; i++) r->s[i] = splitmix64(&x); }
static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
static uint64_t rng_next(rng_t* r) {
    uint64_t* s = r->s;
    uint64_t result = rotl(s[1] * 5, 7) * 9;
    uint64_t t = s[1] << 17;
    s[2] ^= s[0]; s[3] ^= s[1]; s[1] ^= s[2]; s[0] ^= s[3];
    s[2] ^= t; s[3] = rotl(s[3], 45);
    return result;
}
/* uniform in [0,q) by rejection of u >= floor(2^64/q)*q */
static uint64_t rng_uniform(rng_t* r, uint64_t q) {
    uint64_t lim = (uint64_t)((((u128)1) << 64) / q * q);   /* floor(2^64/q)*q  (< 2^64 as q is not a power of 2) */
    for (;;) { uint64_t u = rng_next(r); if (u < lim) return u % q; }
}
/* ternary {-1,0,1}: reject u >= 3*floor(2^64/3), then (u mod 3) - 1 */
static int64_t rng_ternary(rng_t* r) {
    const uint64_t lim = 3ULL * (UINT64_MAX / 3ULL);  /* 3*floor((2^64-1)/3) == 3*floor(2^64/3) since 3 does not divide 2^64 */
    for (;;) { uint64_t u = rng_next(r); if (u < lim) return (int64_t)(u % 3) - 1; }
}
/* centred binomial, eta = 21: popcnt(u & (2^21-1)) - popcnt((u>>21) & (2^21-1)) */
static int64_t rng_cbd(rng_t* r) {
    uint64_t u = rng_next(r);
    return (int64_t)__builtin_popcountll(u & 0x1FFFFFULL) - (int64_t)__builtin_popcountll((u >> 21) & 0x1FFFFFULL);
}

/* exported for the RNG self-test (O3): kind 0 = raw u64, 1 = uniform mod q, 2 = ternary, 3 = cbd */
void or_rng_fill(uint64_t seed, int kind, uint64_t q, uint64_t n, int64_t* out) {
    rng_t r; rng_seed(&r, seed);
    for (uint64_t i = 0; i < n; i++) {
        if (kind == 0) out[i] = (int64_t)rng_next(&r);
        else if (kind == 1) out[i] = (int64_t)rng_uniform(&r, q);
        else if (kind == 2) out[i] = rng_ternary(&r);
        else out[i] = rng_cbd(&r);
    }
}

/* ------------------------------------------------------------------ context (O1, O2) */
#define OR_MAXLIMB 64
typedef struct {
    uint32_t log_n, n, L, alpha, dnum;
    uint64_t mod[OR_MAXLIMB];       /* limbs 0..L-1 = q_i, L..L+alpha-1 = p_k */
    uint64_t psi[OR_MAXLIMB];       /* minimal primitive 2N'-th root per limb */
    uint64_t* psi_rev[OR_MAXLIMB];  /* psi^{brv(i)}    i in [0,N') */
    uint64_t* ipsi_rev[OR_MAXLIMB]; /* psi^{-brv(i)}   i in [0,N') */
    uint64_t ninv[OR_MAXLIMB];
} or_ctx;

/* O2: the minimal x in [1,q) with x^{N'} == -1 (mod q), i.e. the smallest primitive 2N'-th root.
 * All primitive 2N'-th roots are the odd powers of one of them. */
uint64_t or_min_root(uint64_t q, uint32_t log_n) {
    uint64_t two_n = 2ULL << log_n, n = 1ULL << log_n;
    uint64_t root = 0;
    for (uint64_t h = 2; h < q; h++) {
        uint64_t c = powmod(h, (q - 1) / two_n, q);
        if (powmod(c, n, q) == q - 1) { root = c; break; }
    }
    uint64_t best = root, c2 = mulmod(root, root, q), cur = root;
    for (uint64_t k = 1; k < two_n; k += 2) {   /* cur = root^k */
        if (cur < best) best = cur;
        cur = mulmod(cur, c2, q);
    }
    return best;
}

/* O1 prime rule.  q_0 = the largest prime < 2^50 with q == 1 (mod 2N').  q_1..q_{L-1} = the L-1
 * largest primes < 2^40 with q == 1 (mod 2N'), descending.  p_0..p_{alpha-1} = the next alpha primes
 * below q_0 in the 50-bit sequence.  Returns 0 on success. */
int or_gen_params(uint32_t log_n, uint32_t L, uint32_t alpha, uint64_t* q, uint64_t* p) {
    uint64_t two_n = 2ULL << log_n;
    uint64_t c = ((1ULL << 50) - 1) / two_n * two_n + 1;    /* largest value == 1 mod 2N' below 2^50 */
    if (c >= (1ULL << 50)) c -= two_n;
    uint32_t got = 0;
    for (; got < 1 + alpha; c -= two_n) {
        if (is_prime_u64(c)) { if (got == 0) q[0] = c; else p[got - 1] = c; got++; }
    }
    c = ((1ULL << 40) - 1) / two_n * two_n + 1;
    if (c >= (1ULL << 40)) c -= two_n;
    for (got = 1; got < L; c -= two_n) if (is_prime_u64(c)) q[got++] = c;
    return 0;
}

static void ctx_tables(or_ctx* cx, uint32_t i) {
    uint64_t q = cx->mod[i], n = cx->n;
    cx->psi[i] = or_min_root(q, cx->log_n);
    uint64_t ipsi = invmod(cx->psi[i], q);
    cx->psi_rev[i] = (uint64_t*)malloc(n * sizeof(uint64_t));
    cx->ipsi_rev[i] = (uint64_t*)malloc(n * sizeof(uint64_t));
    for (uint64_t k = 0; k < n; k++) {
        uint32_t e = brv((uint32_t)k, cx->log_n);
        cx->psi_rev[i][k] = powmod(cx->psi[i], e, q);
        cx->ipsi_rev[i][k] = powmod(ipsi, e, q);
    }
    cx->ninv[i] = invmod(n % q, q);
}

/* q/p may be NULL (=> O1 rule).  dnum digits, alpha = ceil(L/dnum) expected (not enforced here). */
or_ctx* or_ctx_create(uint32_t log_n, uint32_t L, uint32_t alpha, uint32_t dnum, const uint64_t* q, const uint64_t* p) {
    if (L + alpha > OR_MAXLIMB || log_n < 2 || log_n > 17) return NULL;
    or_ctx* cx = (or_ctx*)calloc(1, sizeof(or_ctx));
    cx->log_n = log_n; cx->n = 1u << log_n; cx->L = L; cx->alpha = alpha; cx->dnum = dnum;
    uint64_t qq[OR_MAXLIMB], pp[OR_MAXLIMB];
    if (!q || !p) or_gen_params(log_n, L, alpha, qq, pp);
    for (uint32_t i = 0; i < L; i++) cx->mod[i] = q ? q[i] : qq[i];
    for (uint32_t k = 0; k < alpha; k++) cx->mod[L + k] = p ? p[k] : pp[k];
    for (uint32_t i = 0; i < L + alpha; i++) ctx_tables(cx, i);
    return cx;
}
void or_ctx_destroy(or_ctx* cx) {
    if (!cx) return;
    for (uint32_t i = 0; i < cx->L + cx->alpha; i++) { free(cx->psi_rev[i]); free(cx->ipsi_rev[i]); }
    free(cx);
}
void or_ctx_moduli(const or_ctx* cx, uint64_t* mod_out, uint64_t* psi_out) {
    for (uint32_t i = 0; i < cx->L + cx->alpha; i++) { mod_out[i] = cx->mod[i]; psi_out[i] = cx->psi[i]; }
}

/* ------------------------------------------------------------------ NTT (O2) */
/* In-place merged-psi Cooley-Tukey: output a[k] = sum_i a_i psi^{(2 brv(k)+1) i} (bit-reversed order). */
void or_ntt(const or_ctx* cx, uint32_t limb, uint64_t* a) {
    uint64_t q = cx->mod[limb]; const uint64_t* w = cx->psi_rev[limb];
    uint32_t n = cx->n, t = n;
    for (uint32_t m = 1; m < n; m <<= 1) {
        t >>= 1;
        for (uint32_t i = 0; i < m; i++) {
            uint32_t j1 = 2 * i * t;
            uint64_t S = w[m + i];
            for (uint32_t j = j1; j < j1 + t; j++) {
                uint64_t U = a[j], V = mulmod(a[j + t], S, q);
                a[j] = addmod(U, V, q);
                a[j + t] = submod(U, V, q);
            }
        }
    }
}
/* Gentleman-Sande inverse of or_ntt, including the N'^{-1} factor. */
void or_intt(const or_ctx* cx, uint32_t limb, uint64_t* a) {
    uint64_t q = cx->mod[limb]; const uint64_t* w = cx->ipsi_rev[limb];
    uint32_t n = cx->n, t = 1;
    for (uint32_t m = n; m > 1; m >>= 1) {
        uint32_t h = m >> 1, j1 = 0;
        for (uint32_t i = 0; i < h; i++) {
            uint64_t S = w[h + i];
            for (uint32_t j = j1; j < j1 + t; j++) {
                uint64_t U = a[j], V = a[j + t];
                a[j] = addmod(U, V, q);
                a[j + t] = mulmod(submod(U, V, q), S, q);
            }
            j1 += 2 * t;
        }
        t <<= 1;
    }
    for (uint32_t j = 0; j < n; j++) a[j] = mulmod(a[j], cx->ninv[limb], q);
}

/* ------------------------------------------------------------------ keys (O4) */
/* Secret key: N' ternary draws (coefficient order) from seed.  sk_coeff[N'] int8 (may be NULL),
 * sk_ntt[(L+alpha)][N'] (NTT form over every limb of Q u P).
 * Public key over Q (L limbs): draw a limb-major uniform (already NTT form: a uniform element of
 * R_q is uniform in either form), then N' CBD draws for e.  pk0 = -a*s + e, pk1 = a. */
void or_keygen(const or_ctx* cx, uint64_t seed, int8_t* sk_coeff, uint64_t* sk_ntt, uint64_t* pk) {
    uint32_t n = cx->n, L = cx->L, T = cx->L + cx->alpha;
    rng_t r; rng_seed(&r, seed);
    int64_t* s = (int64_t*)malloc(n * sizeof(int64_t));
    int64_t* e = (int64_t*)malloc(n * sizeof(int64_t));
    for (uint32_t k = 0; k < n; k++) s[k] = rng_ternary(&r);
    if (sk_coeff) for (uint32_t k = 0; k < n; k++) sk_coeff[k] = (int8_t)s[k];
    for (uint32_t i = 0; i < T; i++) {
        for (uint32_t k = 0; k < n; k++) sk_ntt[(size_t)i * n + k] = smod(s[k], cx->mod[i]);
        or_ntt(cx, i, sk_ntt + (size_t)i * n);
    }
    uint64_t* a = pk + (size_t)L * n;          /* pk1 */
    for (uint32_t i = 0; i < L; i++)
        for (uint32_t k = 0; k < n; k++) a[(size_t)i * n + k] = rng_uniform(&r, cx->mod[i]);
    for (uint32_t k = 0; k < n; k++) e[k] = rng_cbd(&r);
    uint64_t* tmp = (uint64_t*)malloc(n * sizeof(uint64_t));
    for (uint32_t i = 0; i < L; i++) {
        uint64_t q = cx->mod[i];
        for (uint32_t k = 0; k < n; k++) tmp[k] = smod(e[k], q);
        or_ntt(cx, i, tmp);
        for (uint32_t k = 0; k < n; k++) {
            uint64_t as = mulmod(a[(size_t)i * n + k], sk_ntt[(size_t)i * n + k], q);
            pk[(size_t)i * n + k] = submod(tmp[k], as, q);
        }
    }
    free(tmp); free(s); free(e);
}

/* ------------------------------------------------------------------ automorphism (O9) */
/* NTT form: out[k] = in[k'] with 2 brv(k')+1 == (2 brv(k)+1) g (mod 2N').  rows x N' words. */
void or_automorph_ntt(uint32_t log_n, uint64_t g, uint32_t rows, const uint64_t* in, uint64_t* out) {
    uint32_t n = 1u << log_n; uint64_t two_n = 2ULL * n;
    for (uint32_t k = 0; k < n; k++) {
        uint64_t e = (2ULL * brv(k, log_n) + 1) * (g % two_n) % two_n;
        uint32_t kp = brv((uint32_t)((e - 1) / 2), log_n);
        for (uint32_t r = 0; r < rows; r++) out[(size_t)r * n + k] = in[(size_t)r * n + kp];
    }
}
/* coefficient form (used only by tests as a second route): a_i X^i -> (-1)^{floor(i g / N')} a_i X^{i g mod N'} */
void or_automorph_coeff(const or_ctx* cx, uint32_t limb, uint64_t g, const uint64_t* in, uint64_t* out) {
    uint32_t n = cx->n; uint64_t q = cx->mod[limb];
    for (uint32_t i = 0; i < n; i++) {
        uint64_t e = (uint64_t)i * (g % (2ULL * n)) % (2ULL * n);
        if (e < n) out[e] = in[i];
        else out[e - n] = submod(0, in[i], q);
    }
}

/* Switching key towards a target key s' (O4), seed-driven.  Draw order: for t in [0,dnum):
 * a_t limb-major uniform over all L+alpha limbs, then N' CBD draws e_t.
 * key[t][0][limb][k] = b_t = -a_t*s + e_t + [limb in D_t] * (P mod q_limb) * s',  key[t][1] = a_t.
 * D_t = Q-limbs [t*alpha, (t+1)*alpha) cap [0,L).  target [(L+alpha)][N'] = s' in NTT form.
 * e_out (optional) = int64 [dnum][N'] the e_t. */
static void gadget_key(const or_ctx* cx, uint64_t seed, const uint64_t* sk_ntt, const uint64_t* target, uint64_t* key,
                       int64_t* e_out) {
    uint32_t n = cx->n, L = cx->L, A = cx->alpha, T = L + A;
    rng_t r; rng_seed(&r, seed);
    int64_t* e = (int64_t*)malloc(n * sizeof(int64_t));
    uint64_t* tmp = (uint64_t*)malloc(n * sizeof(uint64_t));
    for (uint32_t t = 0; t < cx->dnum; t++) {
        uint64_t* b = key + ((size_t)t * 2 + 0) * T * n;
        uint64_t* a = key + ((size_t)t * 2 + 1) * T * n;
        for (uint32_t i = 0; i < T; i++)
            for (uint32_t k = 0; k < n; k++) a[(size_t)i * n + k] = rng_uniform(&r, cx->mod[i]);
        for (uint32_t k = 0; k < n; k++) e[k] = rng_cbd(&r);
        if (e_out) memcpy(e_out + (size_t)t * n, e, n * sizeof(int64_t));
        for (uint32_t i = 0; i < T; i++) {
            uint64_t q = cx->mod[i];
            uint64_t Pq = 1;      /* P mod q_i */
            for (uint32_t kk = 0; kk < A; kk++) Pq = mulmod(Pq, cx->mod[L + kk] % q, q);
            int in_digit = (i < L) && (i >= t * A) && (i < (t + 1) * A);
            for (uint32_t k = 0; k < n; k++) tmp[k] = smod(e[k], q);
            or_ntt(cx, i, tmp);
            for (uint32_t k = 0; k < n; k++) {
                uint64_t v = submod(tmp[k], mulmod(a[(size_t)i * n + k], sk_ntt[(size_t)i * n + k], q), q);
                if (in_digit) v = addmod(v, mulmod(Pq, target[(size_t)i * n + k], q), q);
                b[(size_t)i * n + k] = v;
            }
        }
    }
    free(e); free(tmp);
}

/* Rotation key for Galois element g: the switching key towards s' = sigma_g(s). */
void or_rotkey(const or_ctx* cx, uint64_t seed, uint64_t g, const uint64_t* sk_ntt, uint64_t* key, int64_t* e_out) {
    uint32_t T = cx->L + cx->alpha;
    uint64_t* sg = (uint64_t*)malloc((size_t)T * cx->n * sizeof(uint64_t));
    or_automorph_ntt(cx->log_n, g, T, sk_ntt, sg);
    gadget_key(cx, seed, sk_ntt, sg, key, e_out);
    free(sg);
}

/* Relinearisation key (CCMM, R18): the switching key towards s' = s^2 (pointwise square in NTT form =
 * negacyclic square of the coefficient polynomial).  Same draw order as or_rotkey. */
void or_relinkey(const or_ctx* cx, uint64_t seed, const uint64_t* sk_ntt, uint64_t* key, int64_t* e_out) {
    uint32_t n = cx->n, T = cx->L + cx->alpha;
    uint64_t* s2 = (uint64_t*)malloc((size_t)T * n * sizeof(uint64_t));
    for (uint32_t i = 0; i < T; i++)
        for (uint32_t k = 0; k < n; k++)
            s2[(size_t)i * n + k] = mulmod(sk_ntt[(size_t)i * n + k], sk_ntt[(size_t)i * n + k], cx->mod[i]);
    gadget_key(cx, seed, sk_ntt, s2, key, e_out);
    free(s2);
}

/* ------------------------------------------------------------------ encrypt / decrypt (O6, O7) */
/* Public-key encryption at level l (first l limbs).  m_res [l][N'] = message residues, coefficient form.
 * Draw order: N' ternary (v), N' CBD (e0), N' CBD (e1).
 * c0 = v*pk0 + e0 + m,  c1 = v*pk1 + e1, NTT form, out [2][l][N']. */
void or_encrypt(const or_ctx* cx, uint64_t seed, const uint64_t* pk, uint32_t level, const uint64_t* m_res, uint64_t* ct) {
    uint32_t n = cx->n, L = cx->L;
    rng_t r; rng_seed(&r, seed);
    int64_t* v = (int64_t*)malloc(n * sizeof(int64_t));
    int64_t* e0 = (int64_t*)malloc(n * sizeof(int64_t));
    int64_t* e1 = (int64_t*)malloc(n * sizeof(int64_t));
    for (uint32_t k = 0; k < n; k++) v[k] = rng_ternary(&r);
    for (uint32_t k = 0; k < n; k++) e0[k] = rng_cbd(&r);
    for (uint32_t k = 0; k < n; k++) e1[k] = rng_cbd(&r);
    uint64_t* tv = (uint64_t*)malloc(n * 8), * t0 = (uint64_t*)malloc(n * 8), * t1 = (uint64_t*)malloc(n * 8);
    for (uint32_t i = 0; i < level; i++) {
        uint64_t q = cx->mod[i];
        for (uint32_t k = 0; k < n; k++) {
            tv[k] = smod(v[k], q);
            t0[k] = addmod(smod(e0[k], q), m_res[(size_t)i * n + k] % q, q);
            t1[k] = smod(e1[k], q);
        }
        or_ntt(cx, i, tv); or_ntt(cx, i, t0); or_ntt(cx, i, t1);
        for (uint32_t k = 0; k < n; k++) {
            ct[(size_t)i * n + k] = addmod(mulmod(tv[k], pk[(size_t)i * n + k], q), t0[k], q);
            ct[((size_t)level + i) * n + k] = addmod(mulmod(tv[k], pk[((size_t)L + i) * n + k], q), t1[k], q);
        }
    }
    free(v); free(e0); free(e1); free(tv); free(t0); free(t1);
}

typedef struct { const or_ctx* cx; const uint64_t* seeds; const uint64_t* pk; uint32_t level; const uint64_t* m; uint64_t* ct; uint32_t count, tid, nth; } enc_job;
static void* enc_worker(void* p) {
    enc_job* j = (enc_job*)p; size_t w = (size_t)j->level * j->cx->n;
    for (uint32_t c = j->tid; c < j->count; c += j->nth) or_encrypt(j->cx, j->seeds[c], j->pk, j->level, j->m + c * w, j->ct + c * 2 * w);
    return NULL;
}
/* count independent encryptions (one seed each) on nthreads threads; m [count][l][N'], ct [count][2][l][N'] */
void or_encrypt_batch(const or_ctx* cx, const uint64_t* seeds, uint32_t count, const uint64_t* pk, uint32_t level,
                      const uint64_t* m_res, uint64_t* ct, uint32_t nthreads) {
    if (nthreads < 1) nthreads = 1;
    pthread_t th[256]; enc_job jobs[256]; if (nthreads > 256) nthreads = 256;
    for (uint32_t t = 0; t < nthreads; t++) {
        jobs[t] = (enc_job){cx, seeds, pk, level, m_res, ct, count, t, nthreads};
        pthread_create(&th[t], NULL, enc_worker, &jobs[t]);
    }
    for (uint32_t t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
}

/* mu = c0 + c1*s (NTT), then INTT: out [l][N'] residues in coefficient form (CRT/decode in Python). */
void or_decrypt(const or_ctx* cx, const uint64_t* sk_ntt, uint32_t level, const uint64_t* ct, uint64_t* mu) {
    uint32_t n = cx->n;
    for (uint32_t i = 0; i < level; i++) {
        uint64_t q = cx->mod[i];
        for (uint32_t k = 0; k < n; k++)
            mu[(size_t)i * n + k] = addmod(ct[(size_t)i * n + k],
                                           mulmod(ct[((size_t)level + i) * n + k], sk_ntt[(size_t)i * n + k], q), q);
        or_intt(cx, i, mu + (size_t)i * n);
    }
}

/* ------------------------------------------------------------------ PCMM Layout A (O8, Algorithm 1) */
/* PAPER.md:307-327.  W is d x m row-major with row stride ldw (W[j*ldw+i]), entries in {-1,0,1}.
 * x: d ciphertexts [d][2][l][N'] (NTT form), y: m ciphertexts [m][2][l][N'].
 * for i: y_i <- (0,0); for j: W=+1 -> y_i (+)= x_j ; W=-1 -> y_i (-)= x_j ; W=0 -> skip.
 * Threads split the output columns i (each column is independent). */
typedef struct { const or_ctx* cx; uint32_t level, d, m, ldw; const uint64_t* x; const int8_t* W; uint64_t* y;
                 const uint32_t* cols; uint32_t ncols, tid, nth; } pcmm_job;
static void pcmm_column(const or_ctx* cx, uint32_t level, uint32_t d, uint32_t ldw, const uint64_t* x, const int8_t* W,
                        uint32_t i, uint64_t* yi) {
    uint32_t n = cx->n; size_t w = (size_t)2 * level * n;
    memset(yi, 0, w * sizeof(uint64_t));                               /* line 2: y_i <- 0 (trivial ciphertext) */
    for (uint32_t j = 0; j < d; j++) {                                  /* line 3 */
        int8_t s = W[(size_t)j * ldw + i];
        if (s == 0) continue;
        const uint64_t* xj = x + (size_t)j * w;
        for (uint32_t poly = 0; poly < 2; poly++)
            for (uint32_t r = 0; r < level; r++) {
                uint64_t q = cx->mod[r]; size_t off = ((size_t)poly * level + r) * n;
                if (s == 1) for (uint32_t k = 0; k < n; k++) yi[off + k] = addmod(yi[off + k], xj[off + k], q);   /* line 5 */
                else        for (uint32_t k = 0; k < n; k++) yi[off + k] = submod(yi[off + k], xj[off + k], q);   /* line 7 */
            }
    }
}
static void* pcmm_worker(void* p) {
    pcmm_job* j = (pcmm_job*)p; size_t w = (size_t)2 * j->level * j->cx->n;
    for (uint32_t c = j->tid; c < j->ncols; c += j->nth) {
        uint32_t i = j->cols ? j->cols[c] : c;
        pcmm_column(j->cx, j->level, j->d, j->ldw, j->x, j->W, i, j->y + (size_t)c * w);
    }
    return NULL;
}
/* cols == NULL: all m columns, y holds m cts.  cols != NULL: only the ncols listed columns, y holds ncols cts
 * (the sampled-column mode used by bench.py's cpu_baseline). */
void or_pcmm_a(const or_ctx* cx, uint32_t level, uint32_t d, uint32_t m, uint32_t ldw, const uint64_t* x, const int8_t* W,
               uint64_t* y, const uint32_t* cols, uint32_t ncols, uint32_t nthreads) {
    if (!cols) ncols = m;
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    pthread_t th[256]; pcmm_job jobs[256];
    for (uint32_t t = 0; t < nthreads; t++) {
        jobs[t] = (pcmm_job){cx, level, d, m, ldw, x, W, y, cols, ncols, t, nthreads};
        pthread_create(&th[t], NULL, pcmm_worker, &jobs[t]);
    }
    for (uint32_t t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
}

/* ------------------------------------------------------------------ hybrid key switching (O10) */
/* number of digits at level l: beta = ceil(l / alpha); digit t covers Q-limbs [t*alpha, min((t+1)alpha, l)) */
static uint32_t n_digits(const or_ctx* cx, uint32_t level) { return (level + cx->alpha - 1) / cx->alpha; }

/* Extended limb index list at level l: Q-limbs 0..l-1 then P-limbs L..L+alpha-1 (ctx indices). */
static uint32_t ext_limb(const or_ctx* cx, uint32_t level, uint32_t e) { return e < level ? e : cx->L + (e - level); }

/* ModUp of one NTT-form polynomial c [l][N'] into out [beta][l+alpha][N'] (NTT form).
 * Per digit t: (i) INTT of the D_t limbs; (ii) y_i = [c_i (Q_t/q_i)^{-1}]_{q_i};
 * (iii) every target limb r outside D_t: ext_r = sum_{i in D_t} y_i [Q_t/q_i]_r mod r (no correction);
 * (iv) NTT;  (v) the D_t limbs are the input's own NTT limbs. */
void or_modup(const or_ctx* cx, uint32_t level, const uint64_t* c, uint64_t* out) {
    uint32_t n = cx->n, A = cx->alpha, E = level + A, beta = n_digits(cx, level);
    uint64_t* coef = (uint64_t*)malloc((size_t)A * n * 8);
    for (uint32_t t = 0; t < beta; t++) {
        uint32_t lo = t * A, hi = (t + 1) * A < level ? (t + 1) * A : level, cnt = hi - lo;
        uint64_t* o = out + (size_t)t * E * n;
        for (uint32_t a = 0; a < cnt; a++) {
            uint32_t i = lo + a; uint64_t q = cx->mod[i];
            uint64_t qhat = 1;                                   /* Q_t / q_i mod q_i */
            for (uint32_t b = lo; b < hi; b++) if (b != i) qhat = mulmod(qhat, cx->mod[b] % q, q);
            uint64_t qhat_inv = invmod(qhat, q);
            memcpy(coef + (size_t)a * n, c + (size_t)i * n, (size_t)n * 8);
            or_intt(cx, i, coef + (size_t)a * n);
            for (uint32_t k = 0; k < n; k++) coef[(size_t)a * n + k] = mulmod(coef[(size_t)a * n + k], qhat_inv, q);
        }
        for (uint32_t e = 0; e < E; e++) {
            uint32_t li = ext_limb(cx, level, e); uint64_t r = cx->mod[li];
            if (li >= lo && li < hi) { memcpy(o + (size_t)e * n, c + (size_t)li * n, (size_t)n * 8); continue; }
            for (uint32_t k = 0; k < n; k++) {
                uint64_t acc = 0;
                for (uint32_t a = 0; a < cnt; a++) {
                    uint64_t qh = 1;                              /* [Q_t / q_{lo+a}]_r */
                    for (uint32_t b = lo; b < hi; b++) if (b != lo + a) qh = mulmod(qh, cx->mod[b] % r, r);
                    acc = addmod(acc, mulmod(coef[(size_t)a * n + k] % r, qh, r), r);
                }
                o[(size_t)e * n + k] = acc;
            }
            or_ntt(cx, li, o + (size_t)e * n);
        }
    }
    free(coef);
}

/* ModDown of acc [l+alpha][N'] (NTT form over Q_l u P) -> out [l][N'] (NTT form over Q_l).
 * INTT of the P limbs; y_k = [acc_{p_k} (P/p_k)^{-1}]_{p_k} taken centred in (-p_k/2, p_k/2];
 * z_i = sum_k y_k [P/p_k]_{q_i} mod q_i (no overflow correction; the centred lift makes the overflow
 * zero-mean, R10 -- an uncentred lift leaves a bias v in [0,alpha) whose v*s term concentrates
 * ~alpha/2 |s(zeta)| / |1-zeta| / Delta of error in slot 0, measured 1.6e-5 per rotation at N'=2^16);
 * NTT; out_i = (acc_i - z_i) * [P^{-1}]_{q_i}. */
void or_moddown(const or_ctx* cx, uint32_t level, const uint64_t* acc, uint64_t* out) {
    uint32_t n = cx->n, L = cx->L, A = cx->alpha;
    uint64_t* pc = (uint64_t*)malloc((size_t)A * n * 8);
    uint64_t* z = (uint64_t*)malloc((size_t)n * 8);
    for (uint32_t k = 0; k < A; k++) {
        uint64_t p = cx->mod[L + k], phat = 1;
        for (uint32_t b = 0; b < A; b++) if (b != k) phat = mulmod(phat, cx->mod[L + b] % p, p);
        uint64_t phat_inv = invmod(phat, p);
        memcpy(pc + (size_t)k * n, acc + ((size_t)level + k) * n, (size_t)n * 8);
        or_intt(cx, L + k, pc + (size_t)k * n);
        for (uint32_t j = 0; j < n; j++) pc[(size_t)k * n + j] = mulmod(pc[(size_t)k * n + j], phat_inv, p);
    }
    for (uint32_t i = 0; i < level; i++) {
        uint64_t q = cx->mod[i], Pinv = 1;
        for (uint32_t b = 0; b < A; b++) Pinv = mulmod(Pinv, cx->mod[L + b] % q, q);
        Pinv = invmod(Pinv, q);
        for (uint32_t j = 0; j < n; j++) {
            uint64_t s = 0;
            for (uint32_t k = 0; k < A; k++) {
                uint64_t ph = 1;                                  /* [P / p_k]_{q_i} */
                for (uint32_t b = 0; b < A; b++) if (b != k) ph = mulmod(ph, cx->mod[L + b] % q, q);
                /* centred residue y in (-p_k/2, p_k/2]: the conversion overflow is then zero-mean (R10) */
                uint64_t y = pc[(size_t)k * n + j], pk = cx->mod[L + k];
                uint64_t yq = (y > pk / 2) ? submod(y % q, pk % q, q) : y % q;
                s = addmod(s, mulmod(yq, ph, q), q);
            }
            z[j] = s;
        }
        or_ntt(cx, i, z);
        for (uint32_t j = 0; j < n; j++)
            out[(size_t)i * n + j] = mulmod(submod(acc[(size_t)i * n + j], z[j], q), Pinv, q);
    }
    free(pc); free(z);
}

/* Key inner product for one Galois element applied to already-ModUp'ed, already-permuted digits (O10):
 * acc_j[e] = sum_t dig[t][e] key[t][j][e] mod r_e over the extended basis Q_l u P.
 * dig [beta][l+alpha][N'], key [dnum][2][L+alpha][N'] -> acc [2][l+alpha][N'] */
static void kip(const or_ctx* cx, uint32_t level, const uint64_t* dig, const uint64_t* key, uint64_t* acc) {
    uint32_t n = cx->n, A = cx->alpha, E = level + A, T = cx->L + A, beta = n_digits(cx, level);
    for (uint32_t j = 0; j < 2; j++)
        for (uint32_t e = 0; e < E; e++) {
            uint32_t li = ext_limb(cx, level, e); uint64_t r = cx->mod[li];
            for (uint32_t k = 0; k < n; k++) {
                uint64_t s = 0;
                for (uint32_t t = 0; t < beta; t++)
                    s = addmod(s, mulmod(dig[((size_t)t * E + e) * n + k], key[(((size_t)t * 2 + j) * T + li) * n + k], r), r);
                acc[((size_t)j * E + e) * n + k] = s;
            }
        }
}
/* Key inner product + ModDown: ks_j = ModDown(acc_j), ks [2][l][N'] */
static void kip_moddown(const or_ctx* cx, uint32_t level, const uint64_t* dig, const uint64_t* key, uint64_t* ks) {
    uint32_t n = cx->n, E = level + cx->alpha;
    uint64_t* acc = (uint64_t*)malloc((size_t)2 * E * n * 8);
    kip(cx, level, dig, key, acc);
    for (uint32_t j = 0; j < 2; j++) or_moddown(cx, level, acc + (size_t)j * E * n, ks + (size_t)j * level * n);
    free(acc);
}

/* Hoisted rotations (O9 + O10): one ModUp of c1, then per Galois element g_r:
 * sigma_g on every limb of every extended digit (ModUp first, then sigma_g), KIP with key_r, ModDown,
 * out_r = (sigma_g(c0) + ks0, ks1).  keys [n_g][dnum][2][L+alpha][N'], out [n_g][2][l][N'].
 * g == 1 gives the identity copy (no key switch). */
void or_rotate_hoisted(const or_ctx* cx, uint32_t level, uint32_t n_g, const uint64_t* gs, const uint64_t* keys,
                       const uint64_t* ct, uint64_t* out) {
    uint32_t n = cx->n, A = cx->alpha, E = level + A, T = cx->L + A, beta = n_digits(cx, level);
    size_t keyw = (size_t)cx->dnum * 2 * T * n, ctw = (size_t)2 * level * n;
    uint64_t* dig = (uint64_t*)malloc((size_t)beta * E * n * 8);
    uint64_t* dperm = (uint64_t*)malloc((size_t)beta * E * n * 8);
    uint64_t* ks = (uint64_t*)malloc(ctw * 8);
    uint64_t* c0g = (uint64_t*)malloc((size_t)level * n * 8);
    or_modup(cx, level, ct + (size_t)level * n, dig);
    for (uint32_t r = 0; r < n_g; r++) {
        uint64_t* o = out + r * ctw;
        if (gs[r] % (2ULL * n) == 1) { memcpy(o, ct, ctw * 8); continue; }
        or_automorph_ntt(cx->log_n, gs[r], beta * E, dig, dperm);
        kip_moddown(cx, level, dperm, keys + r * keyw, ks);
        or_automorph_ntt(cx->log_n, gs[r], level, ct, c0g);
        for (uint32_t i = 0; i < level; i++) {
            uint64_t q = cx->mod[i];
            for (uint32_t k = 0; k < n; k++) {
                o[(size_t)i * n + k] = addmod(c0g[(size_t)i * n + k], ks[(size_t)i * n + k], q);
                o[((size_t)level + i) * n + k] = ks[((size_t)level + i) * n + k];
            }
        }
    }
    free(dig); free(dperm); free(ks); free(c0g);
}

/* non-hoisted rotation = hoisted with a single element (identical bits by the O10 definition) */
void or_rotate(const or_ctx* cx, uint32_t level, uint64_t g, const uint64_t* key, const uint64_t* ct, uint64_t* out) {
    or_rotate_hoisted(cx, level, 1, &g, key, ct, out);
}

/* The parts of Rot(ct; g) before the ModDown (R19, lazy ModDown): c0g = sigma_g(c0) [l][N'] and
 * acc [2][l+alpha][N'] = KIP(sigma_g(ModUp(c1)), key) over Q_l u P, so that Rot(ct; g) = (c0g + ModDown(acc_0),
 * ModDown(acc_1)). */
static void rot_parts(const or_ctx* cx, uint32_t level, uint64_t g, const uint64_t* key, const uint64_t* ct,
                      uint64_t* c0g, uint64_t* acc) {
    uint32_t n = cx->n, E = level + cx->alpha, beta = n_digits(cx, level);
    uint64_t* dig = (uint64_t*)malloc((size_t)beta * E * n * 8);
    uint64_t* dperm = (uint64_t*)malloc((size_t)beta * E * n * 8);
    or_modup(cx, level, ct + (size_t)level * n, dig);
    or_automorph_ntt(cx->log_n, g, beta * E, dig, dperm);
    kip(cx, level, dperm, key, acc);
    or_automorph_ntt(cx->log_n, g, level, ct, c0g);
    free(dig); free(dperm);
}

/* g = 5^r mod 2N' (left rotation by r slots, r taken mod N'/2) */
uint64_t or_galois_elt(uint32_t log_n, int64_t r) {
    uint64_t two_n = 2ULL << log_n, half = 1ULL << (log_n - 1);
    int64_t rr = r % (int64_t)half; if (rr < 0) rr += (int64_t)half;
    return powmod(5, (uint64_t)rr, two_n);
}

/* ------------------------------------------------------------------ PCMM Layout B (O11) */
/* Inputs: n_in cts, block b of ct c (slots [b*s,(b+1)*s)) holds column c*k+b.  B | k, G = k/B.
 * Baby: R_{c,b} = Rot(ct_c; s*b), b in [0,B) (b=0 identity; one ModUp per c, hoisted).
 * T_{i,gam} = sum_c sum_b W[c*k + gam*B + b, i] R_{c,b}   (Algorithm-1 arithmetic, indices >= d skipped).
 * y_i = T_{i,0} + sum_{gam>=1} Rot(T_{i,gam}; s*B*gam).
 * keys: n_keys keys for Galois elements gkeys[] (must contain 5^{s b} for b in [1,B) and 5^{s B gam} for gam in [1,G)). */
static const uint64_t* find_key(const or_ctx* cx, uint32_t n_keys, const uint64_t* gkeys, const uint64_t* keys, uint64_t g) {
    size_t keyw = (size_t)cx->dnum * 2 * (cx->L + cx->alpha) * cx->n;
    for (uint32_t i = 0; i < n_keys; i++) if (gkeys[i] == g) return keys + i * keyw;
    return NULL;
}
/* Baby-step rotations R[c][b] = Rot(ct_c; s*b) for b in [b0, b1) of one input c: one worker job (the hoisted
 * rotations of one input are split into chunks so every host thread has work; bits are identical by O10). */
typedef struct { const or_ctx* cx; uint32_t level, B, n_in, nchunk; const uint64_t* gb; const uint64_t* kb; const uint64_t* x;
                 uint64_t* R; uint32_t tid, nth; } baby_job;
static void* baby_worker(void* p) {
    baby_job* j = (baby_job*)p;
    size_t ctw = (size_t)2 * j->level * j->cx->n, keyw = (size_t)j->cx->dnum * 2 * (j->cx->L + j->cx->alpha) * j->cx->n;
    uint32_t per = (j->B + j->nchunk - 1) / j->nchunk;
    for (uint32_t t = j->tid; t < j->n_in * j->nchunk; t += j->nth) {
        uint32_t c = t / j->nchunk, b0 = (t % j->nchunk) * per, b1 = b0 + per < j->B ? b0 + per : j->B;
        if (b0 >= b1) continue;
        or_rotate_hoisted(j->cx, j->level, b1 - b0, j->gb + b0, j->kb + (size_t)b0 * keyw, j->x + c * ctw,
                          j->R + ((size_t)c * j->B + b0) * ctw);
    }
    return NULL;
}
/* Output columns cols[0..ncols) (all m when cols == NULL); y holds one ciphertext per computed column. */
typedef struct { const or_ctx* cx; uint32_t level, s, k, B, d, ldw, n_in, n_keys; const int8_t* W; const uint64_t* gkeys;
                 const uint64_t* keys; const uint64_t* R; uint64_t* y; const uint32_t* cols; uint32_t ncols, tid, nth;
                 int rc; uint32_t lazy; } bcol_job;
static void* bcol_worker(void* p) {
    bcol_job* j = (bcol_job*)p;
    const or_ctx* cx = j->cx;
    uint32_t n = cx->n, level = j->level, G = j->k / j->B;
    size_t ctw = (size_t)2 * level * n;
    uint32_t E = level + cx->alpha;
    uint64_t* Tt = (uint64_t*)malloc(ctw * 8);
    uint64_t* rot = (uint64_t*)malloc(ctw * 8);
    uint64_t* la = (uint64_t*)malloc((size_t)2 * E * n * 8);      /* lazy: sum of the giant steps' KIP outputs */
    uint64_t* acc = (uint64_t*)malloc((size_t)2 * E * n * 8);
    uint64_t* c0g = (uint64_t*)malloc((size_t)level * n * 8);
    for (uint32_t ci = j->tid; ci < j->ncols; ci += j->nth) {
        uint32_t i = j->cols ? j->cols[ci] : ci;
        uint64_t* yi = j->y + (size_t)ci * ctw;
        memset(yi, 0, ctw * 8);
        memset(la, 0, (size_t)2 * E * n * 8);
        for (uint32_t gam = 0; gam < G; gam++) {
            memset(Tt, 0, ctw * 8);
            for (uint32_t c = 0; c < j->n_in; c++)
                for (uint32_t b = 0; b < j->B; b++) {
                    uint32_t col = c * j->k + gam * j->B + b;
                    if (col >= j->d) continue;
                    int8_t w = j->W[(size_t)col * j->ldw + i];
                    if (w == 0) continue;
                    const uint64_t* rc = j->R + ((size_t)c * j->B + b) * ctw;
                    for (uint32_t poly = 0; poly < 2; poly++)
                        for (uint32_t rr = 0; rr < level; rr++) {
                            uint64_t q = cx->mod[rr]; size_t off = ((size_t)poly * level + rr) * n;
                            for (uint32_t kk = 0; kk < n; kk++)
                                Tt[off + kk] = (w == 1) ? addmod(Tt[off + kk], rc[off + kk], q) : submod(Tt[off + kk], rc[off + kk], q);
                        }
                }
            const uint64_t* src = Tt;
            if (gam > 0) {
                uint64_t g = or_galois_elt(cx->log_n, (int64_t)j->s * j->B * gam);
                const uint64_t* kk = find_key(cx, j->n_keys, j->gkeys, j->keys, g);
                if (!kk) { j->rc = 5; break; }
                if (j->lazy) {
                    /* R19: y_i += (sigma_g(T.c0), 0) now; la += KIP(...) over Q_l u P, one ModDown at the end */
                    rot_parts(cx, level, g, kk, Tt, c0g, acc);
                    for (uint32_t e = 0; e < E; e++) {
                        uint64_t r = cx->mod[ext_limb(cx, level, e)];
                        for (uint32_t poly = 0; poly < 2; poly++)
                            for (uint32_t kk2 = 0; kk2 < n; kk2++) {
                                size_t o = ((size_t)poly * E + e) * n + kk2;
                                la[o] = addmod(la[o], acc[o], r);
                            }
                    }
                    for (uint32_t rr = 0; rr < level; rr++) {
                        uint64_t q = cx->mod[rr];
                        for (uint32_t kk2 = 0; kk2 < n; kk2++) {
                            size_t o = (size_t)rr * n + kk2;
                            yi[o] = addmod(yi[o], c0g[o], q);
                        }
                    }
                    continue;
                }
                or_rotate(cx, level, g, kk, Tt, rot);
                src = rot;
            }
            for (uint32_t poly = 0; poly < 2; poly++)
                for (uint32_t rr = 0; rr < level; rr++) {
                    uint64_t q = cx->mod[rr]; size_t off = ((size_t)poly * level + rr) * n;
                    for (uint32_t kk = 0; kk < n; kk++) yi[off + kk] = addmod(yi[off + kk], src[off + kk], q);
                }
        }
        if (j->rc) break;
        if (j->lazy && G > 1) {
            for (uint32_t poly = 0; poly < 2; poly++) {
                or_moddown(cx, level, la + (size_t)poly * E * n, rot);
                for (uint32_t rr = 0; rr < level; rr++) {
                    uint64_t q = cx->mod[rr]; size_t off = ((size_t)poly * level + rr) * n;
                    for (uint32_t kk = 0; kk < n; kk++) yi[off + kk] = addmod(yi[off + kk], rot[(size_t)rr * n + kk], q);
                }
            }
        }
    }
    free(Tt); free(rot); free(la); free(acc); free(c0g);
    return NULL;
}
/* Threads (nthreads >= 1) split the baby rotations and then the output columns; the arithmetic of every word is the
 * sequence written above (threading changes no result). */
int or_pcmm_b(const or_ctx* cx, uint32_t level, uint32_t s, uint32_t k, uint32_t B, uint32_t d, uint32_t m, uint32_t ldw,
              uint32_t n_in, const uint64_t* x, const int8_t* W, uint32_t n_keys, const uint64_t* gkeys, const uint64_t* keys,
              uint64_t* y, const uint32_t* cols, uint32_t ncols, uint32_t nthreads, uint32_t lazy) {
    uint32_t n = cx->n;
    size_t ctw = (size_t)2 * level * n;
    if (!cols) ncols = m;
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    uint64_t* R = (uint64_t*)malloc((size_t)n_in * B * ctw * 8);     /* R[c][b] */
    uint64_t* gb = (uint64_t*)malloc((size_t)B * 8);
    size_t keyw = (size_t)cx->dnum * 2 * (cx->L + cx->alpha) * n;
    uint64_t* kb = (uint64_t*)calloc((size_t)B * keyw, 8);
    for (uint32_t b = 0; b < B; b++) {
        gb[b] = or_galois_elt(cx->log_n, (int64_t)s * b);
        if (b == 0) continue;
        const uint64_t* kk = find_key(cx, n_keys, gkeys, keys, gb[b]);
        if (!kk) { free(R); free(gb); free(kb); return 5; }
        memcpy(kb + b * keyw, kk, keyw * 8);
    }
    pthread_t th[256];
    uint32_t nchunk = (nthreads + n_in - 1) / n_in;
    if (nchunk > B) nchunk = B;
    baby_job bj[256];
    for (uint32_t t = 0; t < nthreads; t++) {
        bj[t] = (baby_job){cx, level, B, n_in, nchunk, gb, kb, x, R, t, nthreads};
        pthread_create(&th[t], NULL, baby_worker, &bj[t]);
    }
    for (uint32_t t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
    bcol_job cj[256];
    int rc = 0;
    for (uint32_t t = 0; t < nthreads; t++) {
        cj[t] = (bcol_job){cx, level, s, k, B, d, ldw, n_in, n_keys, W, gkeys, keys, R, y, cols, ncols, t, nthreads, 0,
                           lazy};
        pthread_create(&th[t], NULL, bcol_worker, &cj[t]);
    }
    for (uint32_t t = 0; t < nthreads; t++) {
        pthread_join(th[t], NULL);
        if (cj[t].rc) rc = cj[t].rc;
    }
    free(R); free(gb); free(kb);
    return rc;
}

/* ------------------------------------------------------------------ rescale (O12) */
/* Per poly: t = INTT_{q_{l-1}}(c[q_{l-1}]) taken centred in (-q/2, q/2]; for i < l-1:
 * c'[q_i] = (c[q_i] - NTT_{q_i}(t mod q_i)) * [q_{l-1}^{-1}]_{q_i}.  in [2][l][N'] -> out [2][l-1][N']. */
void or_rescale(const or_ctx* cx, uint32_t level, const uint64_t* ct, uint64_t* out) {
    uint32_t n = cx->n, last = level - 1;
    uint64_t ql = cx->mod[last];
    uint64_t* t = (uint64_t*)malloc((size_t)n * 8);
    uint64_t* ti = (uint64_t*)malloc((size_t)n * 8);
    for (uint32_t poly = 0; poly < 2; poly++) {
        memcpy(t, ct + ((size_t)poly * level + last) * n, (size_t)n * 8);
        or_intt(cx, last, t);
        for (uint32_t i = 0; i < last; i++) {
            uint64_t q = cx->mod[i], qinv = invmod(ql % q, q);
            for (uint32_t k = 0; k < n; k++) {
                int64_t centred = t[k] > ql / 2 ? (int64_t)t[k] - (int64_t)ql : (int64_t)t[k];
                ti[k] = smod(centred, q);
            }
            or_ntt(cx, i, ti);
            for (uint32_t k = 0; k < n; k++)
                out[((size_t)poly * last + i) * n + k] =
                    mulmod(submod(ct[((size_t)poly * level + i) * n + k], ti[k], q), qinv, q);
        }
    }
    free(t); free(ti);
}

/* ------------------------------------------------------------------ CCMM primitives */
/* Plaintext-ciphertext product in NTT form (both polys), PAPER.md:124 ring arithmetic:
 * out_p[r][k] = ct_p[r][k] * pt[r][k] mod q_r.  ct/out [2][l][N'], pt [l][N']. */
void or_mul_plain(const or_ctx* cx, uint32_t level, const uint64_t* ct, const uint64_t* pt, uint64_t* out) {
    uint32_t n = cx->n;
    for (uint32_t p = 0; p < 2; p++)
        for (uint32_t i = 0; i < level; i++)
            for (uint32_t k = 0; k < n; k++) {
                size_t o = ((size_t)p * level + i) * n + k;
                out[o] = mulmod(ct[o], pt[(size_t)i * n + k], cx->mod[i]);
            }
}

/* Ciphertext-ciphertext tensor product (the Mult of PAPER.md:124-126 before relinearisation):
 * (a0, a1) x (b0, b1) -> (d0, d1, d2) = (a0 b0, a0 b1 + a1 b0, a1 b1), so that
 * d0 + d1 s + d2 s^2 = (a0 + a1 s)(b0 + b1 s).  a, b [2][l][N'] -> out [3][l][N']. */
void or_mul_ct(const or_ctx* cx, uint32_t level, const uint64_t* a, const uint64_t* b, uint64_t* out) {
    uint32_t n = cx->n;
    size_t P = (size_t)level * n;
    for (uint32_t i = 0; i < level; i++) {
        uint64_t q = cx->mod[i];
        for (uint32_t k = 0; k < n; k++) {
            size_t o = (size_t)i * n + k;
            out[o] = mulmod(a[o], b[o], q);
            out[P + o] = addmod(mulmod(a[o], b[P + o], q), mulmod(a[P + o], b[o], q), q);
            out[2 * P + o] = mulmod(a[P + o], b[P + o], q);
        }
    }
}

/* Relinearisation: key switching of d2 from s^2 to s (O10 with the relinearisation key, no automorphism):
 * ks = ModDown(KIP(ModUp(d2), rlk)); out = (d0 + ks0, d1 + ks1).  d [3][l][N'] -> out [2][l][N']. */
void or_relin(const or_ctx* cx, uint32_t level, const uint64_t* d, const uint64_t* key, uint64_t* out) {
    uint32_t n = cx->n, A = cx->alpha, E = level + A, beta = n_digits(cx, level);
    size_t P = (size_t)level * n;
    uint64_t* dig = (uint64_t*)malloc((size_t)beta * E * n * 8);
    uint64_t* ks = (uint64_t*)malloc(2 * P * 8);
    or_modup(cx, level, d + 2 * P, dig);
    kip_moddown(cx, level, dig, key, ks);
    for (uint32_t i = 0; i < level; i++) {
        uint64_t q = cx->mod[i];
        for (uint32_t k = 0; k < n; k++) {
            size_t o = (size_t)i * n + k;
            out[o] = addmod(d[o], ks[o], q);
            out[P + o] = addmod(d[P + o], ks[P + o], q);
        }
    }
    free(dig); free(ks);
}
