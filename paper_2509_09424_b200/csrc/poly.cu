// poly.cu -- rescale (row a4), decrypt pointwise (row a10) and ciphertext add (Layout-B giant steps).
#include <cmath>

#include "ensi_internal.h"

namespace ensi {

static constexpr uint32_t kT = 256;

struct RescaleConst {
    uint64_t qlinv[ENSI_MAXT], qlinv_sh[ENSI_MAXT];   // [q_{l-1}^{-1}]_{q_i}
    uint64_t ql_mod[ENSI_MAXT];                        // q_{l-1} mod q_i
};

// t = INTT'd last limb (coefficient form) rows [count*2][n].  For i < l-1 write the centred value mod q_i:
// tc = t if t <= q_last/2 else t - q_last  ->  [tc]_{q_i}.
__global__ void __launch_bounds__(kT) k_rescale_convert(const uint64_t* __restrict__ tl, uint64_t* __restrict__ out,
                                                        uint32_t log_n, uint32_t level, ModTab tab, RescaleConst rc) {
    const uint32_t n = 1u << log_n, lm1 = level - 1;
    const uint32_t i = blockIdx.y, cp = blockIdx.z;
    const uint32_t k = blockIdx.x * kT + threadIdx.x;
    const uint64_t ql = tab.q[lm1], q = tab.q[i];
    uint64_t t = tl[(size_t)cp * n + k];
    uint64_t v = reduce64(t, tab.br(i));
    if (t > (ql >> 1)) v = sub_mod(v, rc.ql_mod[i], q);
    out[((size_t)cp * lm1 + i) * n + k] = v;
}

// out[c][poly][i] = (in[c][poly][i] - tconv[c][poly][i]) * q_last^{-1}
__global__ void __launch_bounds__(kT) k_rescale_final(const uint64_t* __restrict__ in, const uint64_t* __restrict__ tc,
                                                      uint64_t* __restrict__ out, uint32_t log_n, uint32_t level,
                                                      ModTab tab, RescaleConst rc) {
    const uint32_t n = 1u << log_n, lm1 = level - 1;
    const uint32_t i = blockIdx.y, cp = blockIdx.z;
    const uint32_t k = blockIdx.x * kT + threadIdx.x;
    const uint64_t q = tab.q[i];
    uint64_t v = sub_mod(in[((size_t)cp * level + i) * n + k], tc[((size_t)cp * lm1 + i) * n + k], q);
    out[((size_t)cp * lm1 + i) * n + k] = mul_shoup(v, rc.qlinv[i], rc.qlinv_sh[i], q);
}

__global__ void __launch_bounds__(kT) k_copy_last_limb(const uint64_t* __restrict__ in, uint64_t* __restrict__ out,
                                                       uint32_t log_n, uint32_t level) {
    const uint32_t n = 1u << log_n, cp = blockIdx.y;
    const uint32_t k = blockIdx.x * kT + threadIdx.x;
    out[(size_t)cp * n + k] = in[((size_t)cp * level + level - 1) * n + k];
}

int rescale(ensi_ctx* ctx, const uint64_t* in, uint32_t count, uint32_t level, uint64_t* out, cudaStream_t st) {
    const uint32_t n = ctx->n, lm1 = level - 1;
    if (count == 0) return ENSI_OK;
    RescaleConst rc{};
    const uint64_t ql = ctx->mod[lm1];
    for (uint32_t i = 0; i < lm1; i++) {
        uint64_t q = ctx->mod[i];
        rc.qlinv[i] = invmod_h(ql % q, q);
        rc.qlinv_sh[i] = shoup_h(rc.qlinv[i], q);
        rc.ql_mod[i] = ql % q;
    }
    const size_t w_t = (size_t)count * 2 * n, w_c = (size_t)count * 2 * lm1 * n;
    int r = ensure_scratch(ctx, (w_t + w_c) * 8);
    if (r) return r;
    uint64_t* tl = (uint64_t*)ctx->scratch;
    uint64_t* tc = tl + w_t;
    k_copy_last_limb<<<dim3(n / kT, count * 2), kT, 0, st>>>(in, tl, ctx->log_n, level);
    ENSI_LAUNCH_CHECK(ctx);
    LimbMap lm = identity_map(1);
    lm.limb[0] = (uint8_t)lm1;
    ntt_inverse(ctx, tl, count * 2, lm, st);
    k_rescale_convert<<<dim3(n / kT, lm1, count * 2), kT, 0, st>>>(tl, tc, ctx->log_n, level, ctx->tab, rc);
    ENSI_LAUNCH_CHECK(ctx);
    ntt_forward(ctx, tc, count * 2 * lm1, identity_map(lm1), st);
    k_rescale_final<<<dim3(n / kT, lm1, count * 2), kT, 0, st>>>(in, tc, out, ctx->log_n, level, ctx->tab, rc);
    ENSI_LAUNCH_CHECK(ctx);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? ENSI_OK : cuda_err(ctx, e, "rescale");
}

// mu[i][k] = c0[i][k] + c1[i][k] * s[i][k] mod q_i   (NTT form)
__global__ void __launch_bounds__(kT) k_decrypt_mu(const uint64_t* __restrict__ ct, const uint64_t* __restrict__ sk,
                                                   uint64_t* __restrict__ mu, uint32_t log_n, uint32_t level,
                                                   ModTab tab) {
    const uint32_t n = 1u << log_n, i = blockIdx.y;
    const uint32_t k = blockIdx.x * kT + threadIdx.x;
    const Barrett br = tab.br(i);
    uint64_t v = mul_mod(ct[((size_t)level + i) * n + k], sk[(size_t)i * n + k], br);
    mu[(size_t)i * n + k] = add_mod(v, ct[(size_t)i * n + k], br.q);
}

int decrypt_mu(ensi_ctx* ctx, const uint64_t* ct, uint32_t level, uint64_t* mu, cudaStream_t st) {
    k_decrypt_mu<<<dim3(ctx->n / kT, level), kT, 0, st>>>(ct, ctx->d_sk, mu, ctx->log_n, level, ctx->tab);
    ENSI_LAUNCH_CHECK(ctx);
    ntt_inverse(ctx, mu, level, identity_map(level), st);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? ENSI_OK : cuda_err(ctx, e, "decrypt");
}

// y += x over count ciphertexts (flat grid-stride; limb of word w = (w / n) % level)
__global__ void __launch_bounds__(kT) k_add_into(uint64_t* __restrict__ y, const uint64_t* __restrict__ x,
                                                 uint64_t words, uint32_t log_n, uint32_t level, ModTab tab) {
    for (uint64_t w = (uint64_t)blockIdx.x * kT + threadIdx.x; w < words; w += (uint64_t)gridDim.x * kT) {
        const uint64_t q = tab.q[(w >> log_n) % level];
        y[w] = add_mod(y[w], x[w], q);
    }
}

void add_into(ensi_ctx* ctx, uint64_t* y, const uint64_t* x, uint32_t count, uint32_t level, cudaStream_t st) {
    if (count == 0) return;
    const uint64_t words = (uint64_t)count * 2 * level * ctx->n;
    k_add_into<<<148 * 8, kT, 0, st>>>(y, x, words, ctx->log_n, level, ctx->tab);
    ENSI_LAUNCH_CHECK(ctx);
}

}  // namespace ensi
