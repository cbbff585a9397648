// ccmm.cu -- ciphertext-ciphertext matrix multiplication (R18), PAPER.md:343-360:
//     c_i = sum_j a_j (x) rep(B_ji)
// with rep(B_ji) = a ciphertext holding the element B_ji on every slot of its head block, extracted by a mask
// product and rotations.  Per output column i (form 2: C = A.B, B column-encoded; form 1: C = A.K^T):
//   1. form 2: periodic copy P_i = b_i + Rot(., -pi 2^u) ...   (log2(s/pi) rotations; pi = 2^ceil(log2 d))
//   2. align   R_j = Rot(P_i, j) | form 1: R_j = Rot(k_j, i), amount r = gam B + b as Rot(Rot(., gam B), b)
//              (baby-step giant-step: B + R/B keys; form 2: the giant steps share one ModUp, the babies of each
//              giant step share one; form 1: Rot(k_j, gam B) is shared by B contiguous output columns)
//   3. mask    M_j = Rescale(R_j (.) mask)                    -> level l-1, scale Delta
//   4. replicate M_j += Rot(M_j, -2^u), u < log2(pi)          (key-stationary batches over j, add fused in ModDown)
//   5. D_i = sum_j a_j|_{l-1} (x) M_j                          (one pass: three 64-bit products per word and j)
//   6. c_i = Rescale(Relin(D_i))                               -> level l-2
// Every step is an exact integer map, so the output words equal the oracle's (oracle/__init__.py Oracle.ccmm).
#include "ensi_internal.h"

namespace ensi {

static constexpr uint32_t kT = 256;

// out[c][p][i][k] = x[c][p][i][k] * pt[i][k] mod q_i   (x, out: count ciphertexts at `level`, contiguous)
__global__ void __launch_bounds__(kT) k_mul_plain(const uint64_t* __restrict__ x, const uint64_t* __restrict__ pt,
                                                  uint64_t* __restrict__ out, uint32_t log_n, uint32_t level,
                                                  ModTab tab) {
    const uint32_t n = 1u << log_n, i = blockIdx.y, cp = blockIdx.z;
    const uint32_t k = blockIdx.x * kT + threadIdx.x;
    const size_t o = ((size_t)cp * level + i) * n + k;
    out[o] = mul_mod(x[o], pt[(size_t)i * n + k], tab.br(i));
}

// D[3][lv][n] (+)= sum_{j < cnt} a_j (x) e_j on the first lv limbs:
//   (a0 e0, a0 e1 + a1 e0, a1 e1); a_j at a + j a_stride with limb stride per poly la*n, e_j contiguous at level lv.
__global__ void __launch_bounds__(kT) k_tensor_acc(const uint64_t* __restrict__ a, uint64_t a_stride, uint32_t la,
                                                   const uint64_t* __restrict__ e, uint32_t cnt,
                                                   uint64_t* __restrict__ D, uint32_t log_n, uint32_t lv, ModTab tab,
                                                   uint32_t init) {
    const uint32_t n = 1u << log_n, i = blockIdx.y;
    const uint32_t k = blockIdx.x * kT + threadIdx.x;
    const Barrett br = tab.br(i);
    const uint64_t q = br.q;
    const size_t P = (size_t)lv * n, o = (size_t)i * n + k;
    uint64_t s0 = 0, s1 = 0, s2 = 0;
    if (!init) {
        s0 = D[o];
        s1 = D[P + o];
        s2 = D[2 * P + o];
    }
    const uint64_t* ap = a + (size_t)i * n + k;
    const uint64_t* ep = e + o;
    const size_t aP = (size_t)la * n, eS = 2 * P;
    for (uint32_t j = 0; j < cnt; j++) {
        const uint64_t a0 = __ldg(ap + j * a_stride), a1 = __ldg(ap + j * a_stride + aP);
        const uint64_t e0 = __ldg(ep + j * eS), e1 = __ldg(ep + j * eS + P);
        s0 = add_mod(s0, mul_mod(a0, e0, br), q);
        s1 = add_mod(s1, add_mod(mul_mod(a0, e1, br), mul_mod(a1, e0, br), q), q);
        s2 = add_mod(s2, mul_mod(a1, e1, br), q);
    }
    D[o] = s0;
    D[P + o] = s1;
    D[2 * P + o] = s2;
}

int mul_plain(ensi_ctx* ctx, const uint64_t* x, uint32_t count, uint32_t level, const uint64_t* pt, uint64_t* out,
              cudaStream_t st) {
    if (count == 0) return ENSI_OK;
    dim3 g(ctx->n / kT, level, count * 2);
    k_mul_plain<<<g, kT, 0, st>>>(x, pt, out, ctx->log_n, level, ctx->tab);
    ENSI_LAUNCH_CHECK(ctx);
    return ENSI_OK;
}

int tensor_acc(ensi_ctx* ctx, const uint64_t* a, uint64_t a_stride, uint32_t la, const uint64_t* e, uint32_t cnt,
               uint64_t* D, uint32_t lv, bool init, cudaStream_t st) {
    dim3 g(ctx->n / kT, lv);
    k_tensor_acc<<<g, kT, 0, st>>>(a, a_stride, la, e, cnt, D, ctx->log_n, lv, ctx->tab, init ? 1u : 0u);
    ENSI_LAUNCH_CHECK(ctx);
    return ENSI_OK;
}

// Relinearisation of cnt three-component products d [cnt][3][lv][n] -> out [cnt][2][lv][n]:
// (d0 + ks0(d2), d1 + ks1(d2)) with the relinearisation key (key switching of d2 from s^2 to s, O10).
int relinearize(ensi_ctx* ctx, const uint64_t* d, uint32_t cnt, uint32_t lv, uint64_t* out, cudaStream_t st) {
    if (!ctx->d_relin) return set_err(ctx, ENSI_ENOKEY, "no relinearisation key loaded");
    const uint64_t one = 1, P = (uint64_t)lv * ctx->n;
    KsOpts ko;
    ko.key_base = ctx->d_relin;
    ko.switch_identity = true;
    ko.c1_off = 2 * P;      // d2
    ko.add_mask = 2;        // out1 += d1
    ko.add1_off = P;
    for (uint32_t c0 = 0; c0 < cnt; c0 += 96) {
        const uint32_t nc = std::min<uint32_t>(96, cnt - c0);
        int rc = rotate_hoisted_multi(ctx, d + (size_t)c0 * 3 * P, nc, 3 * P, lv, 1, &one, out + (size_t)c0 * 2 * P, 1,
                                      st, &ko);
        if (rc) return rc;
    }
    return ENSI_OK;
}

int cc_scratch(ensi_ctx* ctx, size_t words) {
    if (ctx->cc_words >= words) return ENSI_OK;
    cudaFree(ctx->cc_buf);     // synchronises: no queued kernel still uses the old buffer
    ctx->cc_buf = nullptr;
    ctx->cc_words = 0;
    cudaError_t e = cudaMalloc(&ctx->cc_buf, words * 8);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return set_err(ctx, ENSI_ENOMEM, "CCMM scratch allocation failed");
    }
    ctx->cc_words = words;
    return ENSI_OK;
}

static uint32_t ilog2(uint32_t v) {
    uint32_t r = 0;
    while ((1u << (r + 1)) <= v) r++;
    return r;
}

// out[c] = x[c] + Rot(x[c], r) for cnt ciphertexts (one key: the batch is key-stationary), add fused into ModDown
static int add_rotated(ensi_ctx* ctx, const uint64_t* x, uint32_t cnt, uint32_t level, int64_t r, uint64_t* out,
                       cudaStream_t st) {
    const uint64_t g = galois_of_rotation(ctx->log_n, r), ctw = (uint64_t)2 * level * ctx->n;
    KsOpts ko;
    ko.add_mask = 3;
    for (uint32_t c0 = 0; c0 < cnt; c0 += 96) {
        const uint32_t nc = std::min<uint32_t>(96, cnt - c0);
        int rc = rotate_hoisted_multi(ctx, x + c0 * ctw, nc, ctw, level, 1, &g, out + c0 * ctw, 1, st, &ko);
        if (rc) return rc;
    }
    return ENSI_OK;
}

// alignment baby count: B = 2^ceil(ceil(log2 R) / 2) for alignment amounts r < R (oracle.ccmm_plan)
static uint32_t baby_count(uint32_t R) {
    uint32_t c = 0;
    while ((1u << c) < R) c++;   // ceil(log2 R)
    return 1u << ((c + 1) / 2);
}

// out[c] = Rot(x[c], r) for cnt ciphertexts (key-stationary), or a copy when r == 0
static int rotate_all(ensi_ctx* ctx, const uint64_t* x, uint32_t cnt, uint32_t level, int64_t r, uint64_t* out,
                      cudaStream_t st) {
    const uint64_t ctw = (uint64_t)2 * level * ctx->n;
    if (r == 0) {
        cudaError_t e = cudaMemcpyAsync(out, x, cnt * ctw * 8, cudaMemcpyDeviceToDevice, st);
        return e == cudaSuccess ? ENSI_OK : cuda_err(ctx, e, "ccmm copy");
    }
    const uint64_t g = galois_of_rotation(ctx->log_n, r);
    for (uint32_t c0 = 0; c0 < cnt; c0 += 96) {
        const uint32_t nc = std::min<uint32_t>(96, cnt - c0);
        int rc = rotate_hoisted_multi(ctx, x + c0 * ctw, nc, ctw, level, 1, &g, out + c0 * ctw, 1, st);
        if (rc) return rc;
    }
    return ENSI_OK;
}

int ccmm(ensi_ctx* ctx, const uint64_t* a, const uint64_t* src, uint32_t form, uint32_t s, uint32_t d, uint32_t m,
         uint32_t level, const uint64_t* mask, uint64_t* y, uint32_t i0, uint32_t i1, cudaStream_t st) {
    NvtxRange nvtx_("ccmm.columns");
    const uint32_t n = ctx->n, l1 = level - 1, l2 = level - 2;
    const uint32_t pi = form == 1 ? s : (1u << ilog2(2 * d - 1));     // 2^ceil(log2 d)
    const uint32_t Ba = baby_count(form == 2 ? d : m);
    const uint32_t G2 = form == 2 ? (d + Ba - 1) / Ba : 0;           // form 2: giant steps per column
    const uint64_t ctw = (uint64_t)2 * level * n, ctw1 = (uint64_t)2 * l1 * n, ctw2 = (uint64_t)2 * l2 * n;
    // j chunks: whole baby groups of Ba (form 2), at most ~96 ciphertexts
    const uint32_t chunk = std::min<uint32_t>(d, Ba <= 96 ? (96 / Ba) * Ba : Ba);
    // form 1: Rot(k_j, gam B) for all j is kept across the contiguous output columns of one giant step (d <= 256)
    const bool cache1 = form == 1 && d <= 256;
    const size_t g_cts = form == 2 ? G2 : (cache1 ? d : chunk);
    // buffers: P, P' [2][ctw] | Gs [g_cts][ctw] | R [chunk][ctw] | M, M' [2][chunk][ctw1] | D | Cr
    const size_t need = (2 + g_cts + (size_t)chunk) * ctw + 2 * (size_t)chunk * ctw1 + 3 * (size_t)l1 * n + ctw1;
    int rc = cc_scratch(ctx, need);
    if (rc) return rc;
    uint64_t* Pb[2] = {ctx->cc_buf, ctx->cc_buf + ctw};
    uint64_t* Gs = Pb[1] + ctw;
    uint64_t* R = Gs + g_cts * ctw;
    uint64_t* Mb[2] = {R + (size_t)chunk * ctw, R + (size_t)chunk * ctw + (size_t)chunk * ctw1};
    uint64_t* D = Mb[1] + (size_t)chunk * ctw1;
    uint64_t* Cr = D + 3 * (size_t)l1 * n;
    std::vector<uint64_t> gs;
    uint32_t cached_gam = 0xFFFFFFFFu;
    for (uint32_t i = i0; i < i1 && !rc; i++) {
        const uint64_t* G1 = src;                  // form 1: Rot(k_., gam B) for this column's giant step
        if (form == 2) {
            // 1. periodic copy of column i across the block, period pi
            const uint64_t* cur = src + (size_t)i * ctw;
            for (uint32_t u = 0; (pi << u) < s && !rc; u++) {
                uint64_t* nxt = Pb[u & 1];
                rc = add_rotated(ctx, cur, 1, level, -(int64_t)pi * (1ll << u), nxt, st);
                cur = nxt;
            }
            // 2a. giant steps Rot(P_i, gam B), gam < G: one ModUp (hoisted)
            gs.resize(G2);
            for (uint32_t g = 0; g < G2; g++) gs[g] = galois_of_rotation(ctx->log_n, (int64_t)g * Ba);
            if (!rc) rc = rotate_hoisted_multi(ctx, cur, 1, 0, level, G2, gs.data(), Gs, G2, st);
        } else if (i / Ba != 0 && cache1) {
            // 2a. giant step Rot(k_j, gam B) for every j, shared by the columns gam B .. gam B + B - 1
            if (i / Ba != cached_gam) {
                rc = rotate_all(ctx, src, d, level, (int64_t)(i / Ba) * Ba, Gs, st);
                cached_gam = i / Ba;
            }
            G1 = Gs;
        }
        for (uint32_t j0 = 0; j0 < d && !rc; j0 += chunk) {
            const uint32_t jc = std::min<uint32_t>(chunk, d - j0);
            // 2. align element (j, i) to slot 0 of every period: amount r = gam B + b as Rot(Rot(., gam B), b)
            if (form == 2) {
                for (uint32_t g = j0 / Ba; g * Ba < j0 + jc && !rc; g++) {    // 2b. babies of giant step g, hoisted
                    const uint32_t nb = std::min(Ba, d - g * Ba);
                    gs.resize(nb);
                    for (uint32_t b = 0; b < nb; b++) gs[b] = galois_of_rotation(ctx->log_n, (int64_t)b);
                    rc = rotate_hoisted_multi(ctx, Gs + (size_t)g * ctw, 1, 0, level, nb, gs.data(),
                                              R + (size_t)(g * Ba - j0) * ctw, nb, st);
                }
            } else {
                const uint32_t b = i % Ba, gam = i / Ba;
                const uint64_t* x = G1 + (size_t)j0 * ctw;
                if (gam && !cache1) {                  // large d: giant step per chunk into R, then babies in place
                    rc = rotate_all(ctx, src + (size_t)j0 * ctw, jc, level, (int64_t)gam * Ba, Gs, st);
                    x = Gs;
                }
                if (!rc) rc = rotate_all(ctx, x, jc, level, (int64_t)b, R, st);
            }
            if (rc) break;
            // 3. mask (scale q_{l-1}) and rescale: exactly scale Delta at level l-1
            rc = mul_plain(ctx, R, jc, level, mask, R, st);
            if (!rc) rc = rescale(ctx, R, jc, level, Mb[0], st);
            // 4. replicate over the pi slots of each period (doubling)
            uint32_t cur = 0;
            for (uint32_t u = 0; (1u << u) < pi && !rc; u++, cur ^= 1)
                rc = add_rotated(ctx, Mb[cur], jc, l1, -(int64_t)(1ll << u), Mb[cur ^ 1], st);
            if (rc) break;
            // 5. D_i (+)= sum_j a_j (x) rep(B_ji)
            rc = tensor_acc(ctx, a + (size_t)j0 * ctw, ctw, level, Mb[cur], jc, D, l1, j0 == 0, st);
        }
        // 6. relinearise and rescale
        if (!rc) rc = relinearize(ctx, D, 1, l1, Cr, st);
        if (!rc) rc = rescale(ctx, Cr, 1, l1, y + (size_t)(i - i0) * ctw2, st);
    }
    if (!rc) {
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_err(ctx, e, "ccmm");
    }
    return rc;
}

}  // namespace ensi
