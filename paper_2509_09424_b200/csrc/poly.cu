// poly.cu -- rescale (row a4), decrypt pointwise (row a10) and ciphertext add (Layout-B giant steps).
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "ensi_internal.h"
#include "ntt_fp.cuh"

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

// FP64-NTT rescale with the conversion fused into the first forward pass (load) and the final combine into the
// last pass (store): no converted-limb or transformed-limb round trip through HBM.  Row r of the transform = (cp =
// r / (l-1) ciphertext-poly, limb i = r % (l-1)).
struct RescaleInFp {
    const uint64_t* tl;                 // INTT'd last limb, [count*2][n]
    uint64_t ql;
    uint32_t lm1;
    double qd[ENSI_MAXT];
    __device__ __forceinline__ uint64_t load(const uint64_t*, uint32_t row, uint32_t i, uint32_t k) const {
        const uint32_t cp = row / lm1;
        const uint64_t t = tl[(size_t)cp * 65536 + k];
        const long long vc = t > (ql >> 1) ? (long long)t - (long long)ql : (long long)t;   // centred, R12
        const double q = qd[i];
        return nttfp::canon(nttfp::red(nttfp::i2d(vc), q, 1.0 / q), (uint64_t)q);
    }
};
struct RescaleOutFp {
    static constexpr bool kFused = true;
    const uint64_t* in;                 // [count*2][level][n]
    uint64_t* out;                      // [count*2][level-1][n]
    uint32_t level, lm1;
    double qd[ENSI_MAXT], c[ENSI_MAXT], cq[ENSI_MAXT];   // q_i, [q_last^-1]_{q_i} centred, RN(c / q_i)
    __device__ __forceinline__ void store(uint64_t*, uint32_t row, uint32_t i, uint32_t k, uint64_t tt) const {
        const uint32_t cp = row / lm1;
        const uint64_t x = in[((size_t)cp * level + i) * 65536 + k];
        const double V = (double)(long long)x - (double)(long long)tt;       // exact, |V| < q_i
        const double q = qd[i];
        out[((size_t)cp * lm1 + i) * 65536 + k] = nttfp::canon(nttfp::mulmod(V, c[i], cq[i], q), (uint64_t)q);
    }
};

static int rescale_chunk(ensi_ctx* ctx, const uint64_t* in, uint32_t count, uint32_t level, uint64_t* out,
                         cudaStream_t st) {
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
    if (ctx->log_n == 16 && ctx->ntt_fp_ok) {
        // conversion fused into the first NTT pass, the final combine into the last (other rings / moduli >= 2^50:
        // the separate convert / NTT / final kernels below)
        RescaleInFp fin{};
        RescaleOutFp fout{};
        fin.tl = tl;
        fin.ql = ql;
        fin.lm1 = lm1;
        fout.in = in;
        fout.out = out;
        fout.level = level;
        fout.lm1 = lm1;
        for (uint32_t i = 0; i < lm1; i++) {
            const uint64_t q = ctx->mod[i];
            fin.qd[i] = fout.qd[i] = (double)q;
            fout.c[i] = rc.qlinv[i] > q / 2 ? -(double)(q - rc.qlinv[i]) : (double)rc.qlinv[i];
            fout.cq[i] = fout.c[i] / (double)q;
        }
        const double2* tw = reinterpret_cast<const double2*>(ctx->d_tw3);
        const double2* ninv = tw + (size_t)ctx->T * 2 * n;
        const LimbMap zm = identity_map(lm1);
        dim3 g(16, count * 2 * lm1);
        nttfp::k_ntt256<nttfp::FWD_A, RescaleInFp><<<g, 256, 0, st>>>(tc, zm, ctx->tab, tw, ninv, fin);
        nttfp::k_ntt256<nttfp::FWD_B, nttfp::PlainIn, RescaleOutFp><<<g, 256, 0, st>>>(tc, zm, ctx->tab, tw, ninv,
                                                                                    nttfp::PlainIn(), fout);
        ctx->launches += 2;
        cudaError_t e = cudaGetLastError();
        return e == cudaSuccess ? ENSI_OK : cuda_err(ctx, e, "rescale");
    }
    k_rescale_convert<<<dim3(n / kT, lm1, count * 2), kT, 0, st>>>(tl, tc, ctx->log_n, level, ctx->tab, rc);
    ENSI_LAUNCH_CHECK(ctx);
    ntt_forward(ctx, tc, count * 2 * lm1, identity_map(lm1), st);
    k_rescale_final<<<dim3(n / kT, lm1, count * 2), kT, 0, st>>>(in, tc, out, ctx->log_n, level, ctx->tab, rc);
    ENSI_LAUNCH_CHECK(ctx);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? ENSI_OK : cuda_err(ctx, e, "rescale");
}

// Chunks of at most 256 ciphertexts: bounded scratch (256 x 2 x level limbs) and transform grids far below the
// 65535-row launch limit, whatever the layer width (a 5504-output rescale epilogue is 121k limb rows).
int rescale(ensi_ctx* ctx, const uint64_t* in, uint32_t count, uint32_t level, uint64_t* out, cudaStream_t st) {
    const uint64_t ci = (uint64_t)2 * level * ctx->n, co = (uint64_t)2 * (level - 1) * ctx->n;
    for (uint32_t c0 = 0; c0 < count; c0 += 256) {
        const int r = rescale_chunk(ctx, in + c0 * ci, std::min<uint32_t>(256, count - c0), level, out + c0 * co, st);
        if (r) return r;
    }
    return ENSI_OK;
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

// ---------------------------------------------------------------- wire format (compact host transfers)
// Each thread moves 4 consecutive words = wb 32-bit words of wire bytes (4 wb bytes, 4-byte aligned).
template <uint32_t WB>
__global__ void __launch_bounds__(kT) k_wire_unpack(const uint32_t* __restrict__ in, uint64_t* __restrict__ out,
                                                    size_t groups, size_t in_rs, size_t out_rs) {
    // blockIdx.y: row (one (ciphertext, poly) slice of one limb); in_rs / out_rs: row strides in 32-bit / 64-bit words
    const size_t gi = (size_t)blockIdx.x * kT + threadIdx.x;
    if (gi >= groups) return;
    in += blockIdx.y * in_rs;
    out += blockIdx.y * out_rs;
    uint32_t u[WB + 1];
#pragma unroll
    for (uint32_t i = 0; i < WB; i++) u[i] = __ldcs(in + gi * WB + i);
    u[WB] = 0;
#pragma unroll
    for (uint32_t k = 0; k < 4; k++) {
        const uint32_t bit = k * WB * 8, wi = bit / 32, sh = bit % 32;   // compile-time after unrolling
        const uint64_t lo = (uint64_t)__funnelshift_r(u[wi], u[wi + 1], sh);
        const uint64_t hi = (uint64_t)__funnelshift_r(u[wi + 1], WB > wi + 2 ? u[wi + 2] : 0u, sh);
        uint64_t v = lo | (hi << 32);
        if (WB < 8) v &= (1ull << (8 * WB)) - 1;
        out[gi * 4 + k] = v;
    }
}
template <uint32_t WB>
__global__ void __launch_bounds__(kT) k_wire_pack(const uint64_t* __restrict__ in, uint32_t* __restrict__ out,
                                                  size_t groups, size_t in_rs, size_t out_rs) {
    const size_t gi = (size_t)blockIdx.x * kT + threadIdx.x;
    if (gi >= groups) return;
    in += blockIdx.y * in_rs;
    out += blockIdx.y * out_rs;
    uint32_t u[WB + 2];
#pragma unroll
    for (uint32_t i = 0; i < WB + 2; i++) u[i] = 0;
#pragma unroll
    for (uint32_t k = 0; k < 4; k++) {
        const uint64_t v = __ldcs(in + gi * 4 + k);
        const uint32_t bit = k * WB * 8, wi = bit / 32, sh = bit % 32;
        // place the low 8 WB bytes of v at bit offset `bit`
        const uint64_t vlo = (uint64_t)(uint32_t)v << sh;             // bits of word wi / wi+1
        const uint64_t vhi = (v >> 32) << sh;
        u[wi] |= (uint32_t)vlo;
        u[wi + 1] |= (uint32_t)(vlo >> 32) | (uint32_t)vhi;
        u[wi + 2] |= (uint32_t)(vhi >> 32);
    }
#pragma unroll
    for (uint32_t i = 0; i < WB; i++) out[gi * WB + i] = u[i];
}

template <uint32_t WB>
static void wire_launch(bool unpack, const void* in, void* out, size_t groups, uint32_t rows, size_t in_rs,
                        size_t out_rs, cudaStream_t st) {
    const dim3 g((uint32_t)((groups + kT - 1) / kT), rows);
    if (unpack) k_wire_unpack<WB><<<g, kT, 0, st>>>((const uint32_t*)in, (uint64_t*)out, groups, in_rs, out_rs);
    else k_wire_pack<WB><<<g, kT, 0, st>>>((const uint64_t*)in, (uint32_t*)out, groups, in_rs, out_rs);
}

// rows x `words` words of one limb (width wb): row i of the wire side at +i*wire_rs bytes, of the word side at
// +i*word_rs words (wire_rs a multiple of 4, word_rs of 1) -- one launch for all rows (<= 65535 per launch)
static int wire_dispatch(ensi_ctx* ctx, bool unpack, const void* in, void* out, size_t words, uint32_t wb,
                         uint32_t rows, size_t wire_rs, size_t word_rs, cudaStream_t st) {
    if (words % 4) return set_err(ctx, ENSI_EINVAL, "wire transfers move multiples of 4 words");
    if (wire_rs % 4) return set_err(ctx, ENSI_EINVAL, "wire rows must start 4-byte aligned");
    const size_t groups = words / 4;
    for (uint32_t r0 = 0; r0 < rows; r0 += 65535) {
        const uint32_t nr = std::min<uint32_t>(65535, rows - r0);
        const uint8_t* wi = (const uint8_t*)(unpack ? in : out) + (size_t)r0 * wire_rs;
        const uint64_t* wo = (const uint64_t*)(unpack ? out : in) + (size_t)r0 * word_rs;
        const void* src = unpack ? (const void*)wi : (const void*)wo;
        void* dst = unpack ? (void*)wo : (void*)wi;
        const size_t in_rs = unpack ? wire_rs / 4 : word_rs, out_rs = unpack ? word_rs : wire_rs / 4;
        switch (wb) {
            case 1: wire_launch<1>(unpack, src, dst, groups, nr, in_rs, out_rs, st); break;
            case 2: wire_launch<2>(unpack, src, dst, groups, nr, in_rs, out_rs, st); break;
            case 3: wire_launch<3>(unpack, src, dst, groups, nr, in_rs, out_rs, st); break;
            case 4: wire_launch<4>(unpack, src, dst, groups, nr, in_rs, out_rs, st); break;
            case 5: wire_launch<5>(unpack, src, dst, groups, nr, in_rs, out_rs, st); break;
            case 6: wire_launch<6>(unpack, src, dst, groups, nr, in_rs, out_rs, st); break;
            case 7: wire_launch<7>(unpack, src, dst, groups, nr, in_rs, out_rs, st); break;
            case 8: {
                const size_t dp = unpack ? word_rs * 8 : wire_rs, sp = unpack ? wire_rs : word_rs * 8;
                cudaError_t e = cudaMemcpy2DAsync(dst, dp, src, sp, words * 8, nr, cudaMemcpyDeviceToDevice, st);
                if (e != cudaSuccess) return cuda_err(ctx, e, "wire copy");
                continue;
            }
            default: return set_err(ctx, ENSI_EINVAL, "wire width must be 1..8 bytes");
        }
        ctx->launches += 1;
    }
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? ENSI_OK : cuda_err(ctx, e, "wire");
}

int wire_unpack(ensi_ctx* ctx, const uint8_t* in, uint64_t* out, size_t words, uint32_t wb, cudaStream_t st) {
    return wire_dispatch(ctx, true, in, out, words, wb, 1, 0, 0, st);
}
int wire_pack(ensi_ctx* ctx, const uint64_t* in, uint8_t* out, size_t words, uint32_t wb, cudaStream_t st) {
    return wire_dispatch(ctx, false, in, out, words, wb, 1, 0, 0, st);
}
int wire_unpack_rows(ensi_ctx* ctx, const uint8_t* in, size_t wire_rs, uint64_t* out, size_t word_rs, uint32_t rows,
                     size_t words, uint32_t wb, cudaStream_t st) {
    return wire_dispatch(ctx, true, in, out, words, wb, rows, wire_rs, word_rs, st);
}
int wire_pack_rows(ensi_ctx* ctx, const uint64_t* in, size_t word_rs, uint8_t* out, size_t wire_rs, uint32_t rows,
                   size_t words, uint32_t wb, cudaStream_t st) {
    return wire_dispatch(ctx, false, in, out, words, wb, rows, wire_rs, word_rs, st);
}

}  // namespace ensi
