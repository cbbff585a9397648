// host_math.cpp -- host-side number theory for context setup (primes, roots, Shoup/Barrett constants).
// Independent of oracle/ (no shared code): min_root / is_prime_u64 here and their counterparts in
// the C oracle (oracle/) are two separate transcriptions of the same textbook rules (R1 prime rule,
// R2 minimal root).  The oracle's side is pinned to SURVEY.md Appendix A (tests/test_oracle_params_ntt.py);
// this side is pinned only transitively, to the oracle, by tests/test_gpu_parity.py
// test_moduli_and_roots_match_oracle.
#include "ensi_internal.h"

namespace ensi {

typedef unsigned __int128 u128;

uint64_t mulmod_h(uint64_t a, uint64_t b, uint64_t q) { return (uint64_t)(((u128)a * b) % q); }

uint64_t powmod_h(uint64_t a, uint64_t e, uint64_t q) {
    uint64_t r = 1 % q;
    a %= q;
    while (e) {
        if (e & 1) r = mulmod_h(r, a, q);
        a = mulmod_h(a, a, q);
        e >>= 1;
    }
    return r;
}

uint64_t invmod_h(uint64_t a, uint64_t q) { return powmod_h(a % q, q - 2, q); }

uint64_t shoup_h(uint64_t w, uint64_t q) { return (uint64_t)((((u128)w) << 64) / q); }

Barrett barrett_h(uint64_t q) {
    Barrett b;
    b.q = q;
    b.w = 64 - __builtin_clzll(q);
    b.mu = (uint64_t)((((u128)1) << (2 * b.w + 2)) / q);
    return b;
}

bool is_prime_u64(uint64_t n) {
    if (n < 2) return false;
    static const uint64_t small[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    for (uint64_t p : small)
        if (n % p == 0) return n == p;
    uint64_t d = n - 1;
    int s = 0;
    while (!(d & 1)) {
        d >>= 1;
        s++;
    }
    for (uint64_t a : small) {
        uint64_t x = powmod_h(a, d, n);
        if (x == 1 || x == n - 1) continue;
        bool composite = true;
        for (int r = 1; r < s; r++) {
            x = mulmod_h(x, x, n);
            if (x == n - 1) {
                composite = false;
                break;
            }
        }
        if (composite) return false;
    }
    return true;
}

// Largest candidate == 1 (mod 2N') strictly below 2^bits, walking down.
static uint64_t top_candidate(uint32_t bits, uint64_t two_n) {
    uint64_t lim = 1ull << bits;
    uint64_t c = (lim - 1) / two_n * two_n + 1;
    if (c >= lim) c -= two_n;
    return c;
}

void gen_primes(uint32_t log_n, uint32_t L, uint32_t alpha, uint64_t* q, uint64_t* p) {
    const uint64_t two_n = 2ull << log_n;
    uint64_t c = top_candidate(50, two_n);
    for (uint32_t got = 0; got < 1 + alpha; c -= two_n) {
        if (!is_prime_u64(c)) continue;
        if (got == 0) q[0] = c;
        else p[got - 1] = c;
        got++;
    }
    c = top_candidate(40, two_n);
    for (uint32_t got = 1; got < L; c -= two_n)
        if (is_prime_u64(c)) q[got++] = c;
}

uint64_t min_root(uint64_t q, uint32_t log_n) {
    const uint64_t two_n = 2ull << log_n, n = 1ull << log_n;
    uint64_t root = 0;
    for (uint64_t h = 2; h < q; h++) {
        uint64_t c = powmod_h(h, (q - 1) / two_n, q);
        if (powmod_h(c, n, q) == q - 1) {
            root = c;
            break;
        }
    }
    uint64_t best = root, sq = mulmod_h(root, root, q), cur = root;
    for (uint64_t k = 1; k < two_n; k += 2) {
        if (cur < best) best = cur;
        cur = mulmod_h(cur, sq, q);
    }
    return best;
}

uint64_t galois_of_rotation(uint32_t log_n, int64_t r) {
    const int64_t half = 1ll << (log_n - 1);
    int64_t rr = r % half;
    if (rr < 0) rr += half;
    return powmod_h(5, (uint64_t)rr, 2ull << log_n);
}

}  // namespace ensi
