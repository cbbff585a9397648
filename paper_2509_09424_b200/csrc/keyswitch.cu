// keyswitch.cu -- Galois automorphism + hybrid key switching + hoisted rotations (rows a6, a7, a8).
//
// DESIGN.md R9/R10 (= SURVEY.md 8(c) O9/O10; the paper defines Rot only as a slot shift, PAPER.md:134-138,
// and names evk in KeyGen):
//   ModUp per digit t (D_t = Q-limbs [t alpha, (t+1) alpha) cap [0,l)): INTT, y_i = [c_i (Q_t/q_i)^-1]_{q_i},
//   ext_r = sum_i y_i [Q_t/q_i]_r mod r (no overflow correction), NTT.  Rot(ct; g): sigma_g applied to the
//   ModUp'ed digits (ModUp first, then sigma_g), key inner product over the digits, ModDown
//   (INTT of the P limbs, fast conversion to Q_l, NTT, (acc - z) P^-1), plus sigma_g(c0).
// Hoisting: one ModUp per input ciphertext serves every Galois element of a batch.  The automorphism is
// fused into the key-inner-product load (a gather through the NTT-domain index permutation).
#include <algorithm>

#include "ensi_internal.h"
#include "ntt_fp.cuh"

namespace ensi {

static constexpr uint32_t kT = 256;
static constexpr uint32_t kMaxBatch = 64;

// A batch of cnt Galois elements applied to n_ct input ciphertexts (key-stationary: each key word is read once
// for all n_ct inputs).  Rotation (c, gi) reads input c at c0 + c * in_stride and writes output ciphertext
// c * out_c_stride + oidx[gi].  Key-switch rows are indexed gj = (c * cnt + gi) * 2 + j.
struct GBatch {
    uint64_t g[kMaxBatch];
    uint32_t key[kMaxBatch];   // index of the Galois key in ctx->galois / d_keys
    uint32_t oidx[kMaxBatch];  // output ciphertext slot (per input)
    uint32_t cnt, n_ct, out_c_stride;
    uint64_t in_stride;        // words between consecutive input ciphertexts
    __host__ __device__ uint32_t c_of(uint32_t r) const { return r / cnt; }
    __host__ __device__ uint32_t gi_of(uint32_t r) const { return r % cnt; }
};

// ---------------------------------------------------------------- conversion tables

int conv_tables(ensi_ctx* ctx, uint32_t level, ConvTables** out) {
    if (ctx->conv.size() < ctx->L + 1) ctx->conv.resize(ctx->L + 1);
    ConvTables& ct = ctx->conv[level];
    if (ct.d_modup) {
        *out = &ct;
        return ENSI_OK;
    }
    const uint32_t A = ctx->A, L = ctx->L, E = level + A;
    const uint32_t beta = (level + A - 1) / A;
    std::vector<uint64_t> mu((size_t)beta * A * 2 + (size_t)beta * E * A * 2, 0);
    size_t off1 = (size_t)beta * A * 2;
    for (uint32_t t = 0; t < beta; t++) {
        uint32_t lo = t * A, hi = std::min((t + 1) * A, level);
        for (uint32_t a = 0; a < hi - lo; a++) {
            uint32_t i = lo + a;
            uint64_t q = ctx->mod[i], qh = 1;
            for (uint32_t b = lo; b < hi; b++)
                if (b != i) qh = mulmod_h(qh, ctx->mod[b] % q, q);
            uint64_t inv = invmod_h(qh, q);
            mu[(t * A + a) * 2] = inv;
            mu[(t * A + a) * 2 + 1] = shoup_h(inv, q);
        }
        for (uint32_t e = 0; e < E; e++) {
            uint64_t r = ctx->mod[ext_limb(ctx, level, e)];
            for (uint32_t a = 0; a < hi - lo; a++) {
                uint64_t v = 1;
                for (uint32_t b = lo; b < hi; b++)
                    if (b != lo + a) v = mulmod_h(v, ctx->mod[b] % r, r);
                size_t idx = off1 + (((size_t)t * E + e) * A + a) * 2;
                mu[idx] = v;
                mu[idx + 1] = shoup_h(v, r);
            }
        }
    }
    // moddown: phinv [A][2], ph [level][A][2], Pinv [level][2], p_k mod q_i [level][A]
    std::vector<uint64_t> md((size_t)A * 2 + (size_t)level * A * 2 + (size_t)level * 2 + (size_t)level * A, 0);
    for (uint32_t k = 0; k < A; k++) {
        uint64_t p = ctx->mod[L + k], ph = 1;
        for (uint32_t b = 0; b < A; b++)
            if (b != k) ph = mulmod_h(ph, ctx->mod[L + b] % p, p);
        uint64_t inv = invmod_h(ph, p);
        md[k * 2] = inv;
        md[k * 2 + 1] = shoup_h(inv, p);
    }
    for (uint32_t i = 0; i < level; i++) {
        uint64_t q = ctx->mod[i], P = 1;
        for (uint32_t k = 0; k < A; k++) {
            uint64_t v = 1;
            for (uint32_t b = 0; b < A; b++)
                if (b != k) v = mulmod_h(v, ctx->mod[L + b] % q, q);
            size_t idx = (size_t)A * 2 + ((size_t)i * A + k) * 2;
            md[idx] = v;
            md[idx + 1] = shoup_h(v, q);
            P = mulmod_h(P, ctx->mod[L + k] % q, q);
        }
        uint64_t pinv = invmod_h(P, q);
        size_t idx = (size_t)A * 2 + (size_t)level * A * 2 + (size_t)i * 2;
        ct.h_pinv.push_back(pinv);
        md[idx] = pinv;
        md[idx + 1] = shoup_h(pinv, q);
        for (uint32_t k = 0; k < A; k++)
            md[(size_t)A * 2 + (size_t)level * A * 2 + (size_t)level * 2 + (size_t)i * A + k] = ctx->mod[L + k] % q;
    }
    // moddown v2 constants [level][A][3]: ph, ph shoup, q - (p * ph mod q)
    std::vector<uint64_t> md2((size_t)level * A * 3);
    for (uint32_t i = 0; i < level; i++) {
        const uint64_t q = ctx->mod[i];
        for (uint32_t k = 0; k < A; k++) {
            const uint64_t ph = md[(size_t)A * 2 + ((size_t)i * A + k) * 2];
            const uint64_t pph = mulmod_h(ctx->mod[L + k] % q, ph, q);
            md2[((size_t)i * A + k) * 3 + 0] = ph;
            md2[((size_t)i * A + k) * 3 + 1] = shoup_h(ph, q);
            md2[((size_t)i * A + k) * 3 + 2] = pph ? q - pph : 0;
        }
    }
    if (cudaMalloc(&ct.d_moddown2, md2.size() * 8) != cudaSuccess ||
        cudaMemcpy(ct.d_moddown2, md2.data(), md2.size() * 8, cudaMemcpyHostToDevice) != cudaSuccess)
        return cuda_err(ctx, cudaGetLastError(), "conv_tables md2");
    if (ctx->ntt_fp_ok) {
        // ModUp, FP64 copy of mu with every constant centred and paired with RN(c / modulus)
        std::vector<double> uf(mu.size());
        auto centred_ = [](uint64_t w, uint64_t q) -> double { return w > q / 2 ? -(double)(q - w) : (double)w; };
        for (uint32_t t = 0; t < beta; t++) {
            const uint32_t lo = t * A, hi = std::min((t + 1) * A, level);
            for (uint32_t a = 0; a < hi - lo; a++) {
                const uint64_t q = ctx->mod[lo + a];
                const size_t i0 = ((size_t)t * A + a) * 2;
                uf[i0] = centred_(mu[i0], q);
                uf[i0 + 1] = uf[i0] / (double)q;
                for (uint32_t e = 0; e < E; e++) {
                    const uint64_t r = ctx->mod[ext_limb(ctx, level, e)];
                    const size_t i1 = off1 + (((size_t)t * E + e) * A + a) * 2;
                    uf[i1] = centred_(mu[i1], r);
                    uf[i1 + 1] = uf[i1] / (double)r;
                }
            }
        }
        ct.h_modup_fp = uf;
        if (cudaMalloc(&ct.d_modup_fp, uf.size() * 8) != cudaSuccess ||
            cudaMemcpy(ct.d_modup_fp, uf.data(), uf.size() * 8, cudaMemcpyHostToDevice) != cudaSuccess)
            return cuda_err(ctx, cudaGetLastError(), "conv_tables modup fp");
        std::vector<double> mf((size_t)A * 2 + (size_t)level * A * 2);
        auto centred = [](uint64_t w, uint64_t q) -> double { return w > q / 2 ? -(double)(q - w) : (double)w; };
        for (uint32_t k = 0; k < A; k++) {
            const uint64_t p = ctx->mod[L + k];
            mf[k * 2] = centred(md[k * 2], p);
            mf[k * 2 + 1] = mf[k * 2] / (double)p;
        }
        for (uint32_t i = 0; i < level; i++)
            for (uint32_t k = 0; k < A; k++) {
                const size_t o = (size_t)A * 2 + ((size_t)i * A + k) * 2;
                mf[o] = centred(md[o], ctx->mod[i]);
                mf[o + 1] = mf[o] / (double)ctx->mod[i];
            }
        ct.h_moddown_fp = mf;
        if (cudaMalloc(&ct.d_moddown_fp, mf.size() * 8) != cudaSuccess ||
            cudaMemcpy(ct.d_moddown_fp, mf.data(), mf.size() * 8, cudaMemcpyHostToDevice) != cudaSuccess)
            return cuda_err(ctx, cudaGetLastError(), "conv_tables fp");
    }
    cudaError_t e1 = cudaMalloc(&ct.d_modup, mu.size() * 8);
    if (e1 != cudaSuccess) return cuda_err(ctx, e1, "conv_tables malloc");
    e1 = cudaMalloc(&ct.d_moddown, md.size() * 8);
    if (e1 != cudaSuccess) return cuda_err(ctx, e1, "conv_tables malloc");
    cudaMemcpy(ct.d_modup, mu.data(), mu.size() * 8, cudaMemcpyHostToDevice);
    e1 = cudaMemcpy(ct.d_moddown, md.data(), md.size() * 8, cudaMemcpyHostToDevice);
    if (e1 != cudaSuccess) return cuda_err(ctx, e1, "conv_tables copy");
    ct.level = level;
    ct.beta = beta;
    *out = &ct;
    return ENSI_OK;
}

// ---------------------------------------------------------------- kernels

// ModUp conversion.  coef = INTT(c1) [l][N'] (coefficient form).  ext [beta][E][N']:
//   e in D_t -> coef (NTT brings it back to c1's own limb bit-exactly), else the fast conversion.
__global__ void __launch_bounds__(kT) k_modup_convert(const uint64_t* __restrict__ coef, uint64_t* __restrict__ ext,
                                                      uint32_t log_n, uint32_t level, uint32_t L, uint32_t A,
                                                      ModTab tab, const uint64_t* __restrict__ cm) {
    const uint32_t n = 1u << log_n, E = level + A;
    const uint32_t row = blockIdx.y, t = row / E, e = row % E;
    const uint32_t beta_ = (level + A - 1) / A;
    coef += (size_t)blockIdx.z * level * n;                // input ciphertext blockIdx.z of a batched ModUp
    ext += (size_t)blockIdx.z * beta_ * E * n;
    const uint32_t li = e < level ? e : L + (e - level);
    const uint32_t lo = t * A, hi = min((t + 1) * A, level), cnt = hi - lo;
    const uint32_t k = blockIdx.x * kT + threadIdx.x;
    uint64_t out;
    if (li >= lo && li < hi) {
        out = coef[(size_t)li * n + k];
    } else {
        const uint64_t beta = (level + A - 1) / A;
        const uint64_t* qhinv = cm + (size_t)t * A * 2;
        const uint64_t* qh = cm + beta * A * 2 + (((size_t)t * E + e) * A) * 2;
        const uint64_t r = tab.q[li];
        uint64_t sum = 0;
        for (uint32_t a = 0; a < cnt; a++) {
            const uint64_t qi = tab.q[lo + a];
            uint64_t y = mul_shoup(coef[(size_t)(lo + a) * n + k], qhinv[2 * a], qhinv[2 * a + 1], qi);
            sum += mul_shoup_lazy(y, qh[2 * a], qh[2 * a + 1], r);
        }
        out = reduce64(sum, tab.br(li));
    }
    ext[(size_t)row * n + k] = out;
}

// Extended-digit row order.  perm == 0: row = e (limbs in Q_l u P order).  perm != 0: the E - c_t converted limbs
// first, then the digit's own c_t limbs (c_t = A, fewer in a partial last digit when A does not divide the level),
// which are copied in NTT form from the input instead of being INTT'ed, converted and NTT'ed again -- the ModUp
// NTT then runs on E - c_t rows per digit.
__device__ __forceinline__ uint32_t ext_row(uint32_t perm, uint32_t t, uint32_t e, uint32_t A, uint32_t E,
                                            uint32_t level) {
    if (!perm) return e;
    const uint32_t lo = t * A, hi = min(lo + A, level), c = hi - lo;   // the last digit may hold fewer limbs
    return e < lo ? e : (e >= hi ? e - c : (E - c) + (e - lo));
}

// FP64 ModUp conversion, one thread per (input, digit t, position k) producing all E extended limbs: the digit's
// y_i = [c_i (Q_t/q_i)^-1]_{q_i} (canonical, as the oracle's uncorrected fast conversion requires, R10) are computed
// once; ext_r = sum_i y_i [Q_t/q_i]_r with |partial sums| <= 2.5 r, one centred reduction, canonical store.
// The digit's own limbs are copied (the NTT that follows restores the input's NTT words).
__global__ void __launch_bounds__(kT) k_modup_convert_fp(const uint64_t* __restrict__ coef, uint64_t* __restrict__ ext,
                                                         uint32_t log_n, uint32_t level, uint32_t L, uint32_t A,
                                                         ModTab tab, const double* __restrict__ cf, uint32_t perm) {
    const uint32_t n = 1u << log_n, E = level + A, beta = (level + A - 1) / A;
    const uint32_t t = blockIdx.y;
    const uint32_t k = blockIdx.x * kT + threadIdx.x;
    coef += (size_t)blockIdx.z * level * n;
    ext += ((size_t)blockIdx.z * beta + t) * E * n;
    const uint32_t lo = t * A, hi = min((t + 1) * A, level), cnt = hi - lo;
    const double* cinv = cf + (size_t)t * A * 2;
    const double* cq = cf + (size_t)beta * A * 2 + (size_t)t * E * A * 2;
    uint64_t own[8];
    double y[8];
#pragma unroll
    for (uint32_t a = 0; a < 8; a++) {
        if (a < cnt) {
            const uint64_t qa = tab.q[lo + a];
            own[a] = coef[(size_t)(lo + a) * n + k];
            double r = nttfp::mulmod(nttfp::i2d((long long)own[a]), __ldg(cinv + 2 * a), __ldg(cinv + 2 * a + 1),
                                     (double)qa);
            y[a] = r < 0.0 ? r + (double)qa : r;                     // canonical [0, q_a)
        }
    }
    for (uint32_t e = 0; e < E; e++) {
        const uint32_t li = e < level ? e : L + (e - level);
        uint64_t out;
        if (li >= lo && li < hi) {
            if (perm) continue;                  // copied from the input's NTT-form limbs by the host
            out = 0;
#pragma unroll
            for (uint32_t a = 0; a < 8; a++)
                if (a < cnt && lo + a == li) out = own[a];
        } else {
            const uint64_t r = tab.q[li];
            const double rd = (double)r;
            const double* c = cq + (size_t)e * A * 2;
            double sum = 0.0;
#pragma unroll
            for (uint32_t a = 0; a < 8; a++)
                if (a < cnt) sum += nttfp::mulmod(y[a], __ldg(c + 2 * a), __ldg(c + 2 * a + 1), rd);
            out = nttfp::canon(nttfp::red(sum, rd, 1.0 / rd), r);
        }
        ext[(size_t)ext_row(perm, t, e, A, E, level) * n + k] = out;
    }
}

// Same conversion with the constants in the kernel-parameter bank and the target/source loops unrolled to fixed
// bounds (alpha <= 4, beta <= 4, E <= 16): no per-position constant loads or divisions.
struct MUConstFp {
    double cinv[4][4], cinvq[4][4];       // [t][a]: (Q_t/q_i)^-1 mod q_i centred, RN(./q_i)
    double c[4][16][4], cq[4][16][4];     // [t][e][a]: [Q_t/q_i]_{r_e} centred, RN(./r_e)
    double qs[16], r[16], rinv[16];       // q of the source limbs (Q order), r_e, RN(1/r_e)
};
// The digit index is a template parameter so every constant (Q_t/q_i)^-1, [Q_t/q_i]_{r_e} is a compile-time offset
// into the parameter bank (ncu: the runtime-indexed version spent 150 of 1331 warp instructions per position on
// LDC constant loads plus their address arithmetic).
template <uint32_t TT>
__device__ __forceinline__ void modup_fpc_body(const uint64_t* __restrict__ coef, uint64_t* __restrict__ ext,
                                               uint32_t n, uint32_t level, uint32_t L, uint32_t A,
                                               const MUConstFp& mc, uint32_t perm, uint32_t k) {
    const uint32_t E = level + A;
    const uint32_t lo = TT * A, hi = min(lo + A, level), cnt = hi - lo;
    uint64_t own[4];
    double y[4];
#pragma unroll
    for (uint32_t a = 0; a < 4; a++) {
        if (a < cnt) {
            const double qa = mc.qs[lo + a];
            own[a] = coef[(size_t)(lo + a) * n + k];
            const double rr = nttfp::mulmod(nttfp::i2d((long long)own[a]), mc.cinv[TT][a], mc.cinvq[TT][a], qa);
            y[a] = rr < 0.0 ? rr + qa : rr;                           // canonical [0, q_a)
        }
    }
#pragma unroll
    for (uint32_t e = 0; e < 16; e++) {
        if (e < E) {
            const uint32_t li = e < level ? e : L + (e - level);
            if (li >= lo && li < hi) {
                if (perm) continue;
                uint64_t out = 0;
#pragma unroll
                for (uint32_t a = 0; a < 4; a++)
                    if (a < cnt && lo + a == li) out = own[a];
                ext[(size_t)e * n + k] = out;
            } else {
                double sum = 0.0;
#pragma unroll
                for (uint32_t a = 0; a < 4; a++)
                    if (a < cnt) sum += nttfp::mulmod(y[a], mc.c[TT][e][a], mc.cq[TT][e][a], mc.r[e]);
                ext[(size_t)ext_row(perm, TT, e, A, E, level) * n + k] =
                    nttfp::canon(nttfp::red(sum, mc.r[e], mc.rinv[e]), (uint64_t)mc.r[e]);
            }
        }
    }
}
__global__ void __launch_bounds__(kT) k_modup_convert_fpc(const uint64_t* __restrict__ coef, uint64_t* __restrict__ ext,
                                                          uint32_t log_n, uint32_t level, uint32_t L, uint32_t A,
                                                          const __grid_constant__ MUConstFp mc, uint32_t perm) {
    const uint32_t n = 1u << log_n, E = level + A, beta = (level + A - 1) / A;
    const uint32_t t = blockIdx.y;
    const uint32_t k = blockIdx.x * kT + threadIdx.x;
    coef += (size_t)blockIdx.z * level * n;
    ext += ((size_t)blockIdx.z * beta + t) * E * n;
    switch (t) {
        case 0: modup_fpc_body<0>(coef, ext, n, level, L, A, mc, perm, k); break;
        case 1: modup_fpc_body<1>(coef, ext, n, level, L, A, mc, perm, k); break;
        case 2: modup_fpc_body<2>(coef, ext, n, level, L, A, mc, perm, k); break;
        default: modup_fpc_body<3>(coef, ext, n, level, L, A, mc, perm, k); break;
    }
}

// two consecutive positions per thread (16-byte loads and stores)
template <uint32_t TT>
__device__ __forceinline__ void modup_fpc_body2(const uint64_t* __restrict__ coef, uint64_t* __restrict__ ext,
                                                uint32_t n, uint32_t level, uint32_t L, uint32_t A,
                                                const MUConstFp& mc, uint32_t perm, uint32_t k) {
    const uint32_t E = level + A;
    const uint32_t lo = TT * A, hi = min(lo + A, level), cnt = hi - lo;
    ulonglong2 own[4];
    double ya[4], yb[4];
#pragma unroll
    for (uint32_t a = 0; a < 4; a++) {
        if (a < cnt) {
            const double qa = mc.qs[lo + a];
            own[a] = *reinterpret_cast<const ulonglong2*>(coef + (size_t)(lo + a) * n + k);
            const double ra = nttfp::mulmod(nttfp::i2d((long long)own[a].x), mc.cinv[TT][a], mc.cinvq[TT][a], qa);
            const double rb = nttfp::mulmod(nttfp::i2d((long long)own[a].y), mc.cinv[TT][a], mc.cinvq[TT][a], qa);
            ya[a] = ra < 0.0 ? ra + qa : ra;                          // canonical [0, q_a)
            yb[a] = rb < 0.0 ? rb + qa : rb;
        }
    }
#pragma unroll
    for (uint32_t e = 0; e < 16; e++) {
        if (e < E) {
            const uint32_t li = e < level ? e : L + (e - level);
            if (li >= lo && li < hi) {
                if (perm) continue;
                ulonglong2 out = make_ulonglong2(0, 0);
#pragma unroll
                for (uint32_t a = 0; a < 4; a++)
                    if (a < cnt && lo + a == li) out = own[a];
                *reinterpret_cast<ulonglong2*>(ext + (size_t)e * n + k) = out;
            } else {
                double sa = 0.0, sb = 0.0;
#pragma unroll
                for (uint32_t a = 0; a < 4; a++)
                    if (a < cnt) {
                        sa += nttfp::mulmod(ya[a], mc.c[TT][e][a], mc.cq[TT][e][a], mc.r[e]);
                        sb += nttfp::mulmod(yb[a], mc.c[TT][e][a], mc.cq[TT][e][a], mc.r[e]);
                    }
                const uint64_t r = (uint64_t)mc.r[e];
                *reinterpret_cast<ulonglong2*>(ext + (size_t)ext_row(perm, TT, e, A, E, level) * n + k) =
                    make_ulonglong2(nttfp::canon(nttfp::red(sa, mc.r[e], mc.rinv[e]), r),
                                    nttfp::canon(nttfp::red(sb, mc.r[e], mc.rinv[e]), r));
            }
        }
    }
}
__global__ void __launch_bounds__(kT) k_modup_convert_fpc2(const uint64_t* __restrict__ coef, uint64_t* __restrict__ ext,
                                                           uint32_t log_n, uint32_t level, uint32_t L, uint32_t A,
                                                           const __grid_constant__ MUConstFp mc, uint32_t perm) {
    const uint32_t n = 1u << log_n, E = level + A, beta = (level + A - 1) / A;
    const uint32_t t = blockIdx.y;
    const uint32_t k = 2 * (blockIdx.x * kT + threadIdx.x);
    coef += (size_t)blockIdx.z * level * n;
    ext += ((size_t)blockIdx.z * beta + t) * E * n;
    switch (t) {
        case 0: modup_fpc_body2<0>(coef, ext, n, level, L, A, mc, perm, k); break;
        case 1: modup_fpc_body2<1>(coef, ext, n, level, L, A, mc, perm, k); break;
        case 2: modup_fpc_body2<2>(coef, ext, n, level, L, A, mc, perm, k); break;
        default: modup_fpc_body2<3>(coef, ext, n, level, L, A, mc, perm, k); break;
    }
}

// FP64 key inner product, lean (<= 32 registers, 8 CTAs/SM: the kernel is memory-latency sensitive): per digit one
// exact FP64 product per key polynomial (a, b < q < 2^50: h = ab, l = fma(a, b, -h), t = rint(h / q),
// r = fma(-t, q, h) + l, |r| <= 0.75 q), beta partial products summed (|s| < 6 q), one centred reduction, canonical
// store -- the same words as k_kip2 at ~1/3 of its integer instructions (128-bit products + Barrett).
__device__ __forceinline__ double kip_mul(double a, double b, double q, double qinv) {
    const double h = a * b;
    const double l = fma(a, b, -h);
    const double t = fma(h, qinv, nttfp::kM) - nttfp::kM;
    return fma(-t, q, h) + l;
}
__global__ void __launch_bounds__(kT, 8) k_kip_fp(const uint64_t* __restrict__ ext, const uint64_t* __restrict__ keys,
                                                  uint64_t* __restrict__ acc, GBatch gb, uint32_t log_n, uint32_t level,
                                                  uint32_t L, uint32_t A, uint32_t dnum, uint32_t beta, ModTab tab,
                                                  uint64_t ext_stride, uint32_t perm, uint32_t limb_major,
                                                  const uint64_t* __restrict__ c1p, uint64_t in_stride) {
    const uint32_t n = 1u << log_n, E = level + A, T = L + A;
    // limb_major: grid (k blocks, rotations, limbs) -- all rotations of one extended limb run back to back, so the
    // gathered digit rows of that limb (beta x N' words per input) stay in L2 across the batch's rotations
    const uint32_t e = limb_major ? blockIdx.z : blockIdx.y, gi = limb_major ? blockIdx.y : blockIdx.z;
    const uint32_t li = e < level ? e : L + (e - level);
    const uint32_t k = blockIdx.x * kT + threadIdx.x;
    const uint32_t src = galois_src_index(k, gb.g[gi], log_n);
    const uint64_t* key = keys + (size_t)gb.key[gi] * dnum * 2 * T * n + (size_t)li * n + k;
    const uint64_t q = tab.q[li];
    const double qd = (double)q, qinv = 1.0 / qd;
    for (uint32_t c = 0; c < gb.n_ct; c++) {
        const uint64_t* ex = ext + (size_t)c * ext_stride + src;
        double s0 = 0.0, s1 = 0.0;
        for (uint32_t t = 0; t < beta; t++) {
            // perm == 2: a digit's own limbs are read straight from the input's c1 (NTT form), never copied
            const bool own = perm == 2 && e >= t * A && e < t * A + A && e < level;
            const uint64_t* dp = own ? c1p + (size_t)c * in_stride + (size_t)e * n + src
                                     : ex + ((size_t)t * E + ext_row(perm, t, e, A, E, level)) * n;
            const double dv = nttfp::i2d((long long)*dp);
            const uint64_t* kp = key + (size_t)t * 2 * T * n;
            s0 += kip_mul(dv, nttfp::i2d((long long)__ldg(kp)), qd, qinv);
            s1 += kip_mul(dv, nttfp::i2d((long long)__ldg(kp + (size_t)T * n)), qd, qinv);
        }
        const size_t r = (size_t)c * gb.cnt + gi;
        acc[((r * 2 + 0) * E + e) * n + k] = nttfp::canon(nttfp::red(s0, qd, qinv), q);
        acc[((r * 2 + 1) * E + e) * n + k] = nttfp::canon(nttfp::red(s1, qd, qinv), q);
    }
}

// Same key inner product specialised on the digit count (BETA <= 4): the digit row offsets are resolved once per
// thread, both key words of every digit are loaded once and reused for every input of the batch, and the digit loops
// are unrolled.  ncu had the generic kernel issue-bound (85 % issue active, 519 warp instructions per 32 words and
// limb, 45 % of them uniform-datapath index arithmetic re-evaluated inside the input and digit loops).
template <uint32_t BETA>
__global__ void __launch_bounds__(kT, 6) k_kip_fpt(const uint64_t* __restrict__ ext,
                                                   const uint64_t* __restrict__ keys,
                                                   uint64_t* __restrict__ acc, GBatch gb, uint32_t log_n,
                                                   uint32_t level, uint32_t L, uint32_t A, uint32_t dnum, ModTab tab,
                                                   uint64_t ext_stride, uint32_t perm, uint32_t limb_major,
                                                   const uint64_t* __restrict__ c1p, uint64_t in_stride) {
    const uint32_t n = 1u << log_n, E = level + A, T = L + A;
    const uint32_t e = limb_major ? blockIdx.z : blockIdx.y, gi = limb_major ? blockIdx.y : blockIdx.z;
    const uint32_t li = e < level ? e : L + (e - level);
    const uint32_t k = blockIdx.x * kT + threadIdx.x;
    const uint32_t src = galois_src_index(k, gb.g[gi], log_n);
    const size_t TN = (size_t)T * n;
    const uint64_t* key = keys + (size_t)gb.key[gi] * dnum * 2 * TN + (size_t)li * n + k;
    const uint64_t q = tab.q[li];
    const double qd = (double)q, qinv = 1.0 / qd;
    // per digit: a pointer walking the inputs (own limbs read in place from c1, the rest from the extended digits)
    const uint64_t* p[BETA];
    size_t str[BETA];
    double kb0[BETA], kb1[BETA];
#pragma unroll
    for (uint32_t t = 0; t < BETA; t++) {
        const bool own = perm == 2 && e >= t * A && e < t * A + A && e < level;
        p[t] = own ? c1p + (size_t)e * n + src : ext + ((size_t)t * E + ext_row(perm, t, e, A, E, level)) * n + src;
        str[t] = own ? in_stride : ext_stride;
        kb0[t] = nttfp::i2d((long long)__ldg(key + (size_t)t * 2 * TN));
        kb1[t] = nttfp::i2d((long long)__ldg(key + (size_t)t * 2 * TN + TN));
    }
    uint64_t* o = acc + ((size_t)gi * 2 * E + e) * n + k;
    const size_t ostep = (size_t)gb.cnt * 2 * E * n, en = (size_t)E * n;
    for (uint32_t c = 0; c < gb.n_ct; c++) {
        double s0 = 0.0, s1 = 0.0;
#pragma unroll
        for (uint32_t t = 0; t < BETA; t++) {
            const double dv = nttfp::i2d((long long)*p[t]);
            p[t] += str[t];
            s0 += kip_mul(dv, kb0[t], qd, qinv);
            s1 += kip_mul(dv, kb1[t], qd, qinv);
        }
        o[0] = nttfp::canon(nttfp::red(s0, qd, qinv), q);
        o[en] = nttfp::canon(nttfp::red(s1, qd, qinv), q);
        o += ostep;
    }
}

// Two consecutive positions per thread: the key words of both come with one 16-byte load per digit and key
// polynomial, the outputs go out as 16-byte stores, and the per-thread setup is shared (ENSI_KIP_PAIR=0: one
// position per thread).
template <uint32_t BETA>
__global__ void __launch_bounds__(kT, 4) k_kip_fpt2(const uint64_t* __restrict__ ext,
                                                    const uint64_t* __restrict__ keys,
                                                    uint64_t* __restrict__ acc, GBatch gb, uint32_t log_n,
                                                    uint32_t level, uint32_t L, uint32_t A, uint32_t dnum, ModTab tab,
                                                    uint64_t ext_stride, uint32_t perm, uint32_t limb_major,
                                                    const uint64_t* __restrict__ c1p, uint64_t in_stride,
                                                    uint32_t accum_out) {
    // accum_out (R19 lazy ModDown): acc already holds canonical partial sums over Q_l u P; add them (in place)
    const uint32_t n = 1u << log_n, E = level + A, T = L + A;
    const uint32_t e = limb_major ? blockIdx.z : blockIdx.y, gi = limb_major ? blockIdx.y : blockIdx.z;
    const uint32_t li = e < level ? e : L + (e - level);
    const uint32_t k = 2 * (blockIdx.x * kT + threadIdx.x);
    const uint64_t g = gb.g[gi];
    const uint32_t srcA = galois_src_index(k, g, log_n), srcB = galois_src_index(k + 1, g, log_n);
    const size_t TN = (size_t)T * n;
    const uint64_t* key = keys + (size_t)gb.key[gi] * dnum * 2 * TN + (size_t)li * n + k;
    const uint64_t q = tab.q[li];
    const double qd = (double)q, qinv = 1.0 / qd;
    const uint64_t* p[BETA];
    size_t str[BETA];
    double k0a[BETA], k0b[BETA], k1a[BETA], k1b[BETA];
#pragma unroll
    for (uint32_t t = 0; t < BETA; t++) {
        const bool own = perm == 2 && e >= t * A && e < t * A + A && e < level;
        p[t] = own ? c1p + (size_t)e * n : ext + ((size_t)t * E + ext_row(perm, t, e, A, E, level)) * n;
        str[t] = own ? in_stride : ext_stride;
        const ulonglong2 w0 = __ldg(reinterpret_cast<const ulonglong2*>(key + (size_t)t * 2 * TN));
        const ulonglong2 w1 = __ldg(reinterpret_cast<const ulonglong2*>(key + (size_t)t * 2 * TN + TN));
        k0a[t] = nttfp::i2d((long long)w0.x), k0b[t] = nttfp::i2d((long long)w0.y);
        k1a[t] = nttfp::i2d((long long)w1.x), k1b[t] = nttfp::i2d((long long)w1.y);
    }
    uint64_t* o = acc + ((size_t)gi * 2 * E + e) * n + k;
    const size_t ostep = (size_t)gb.cnt * 2 * E * n, en = (size_t)E * n;
    for (uint32_t c = 0; c < gb.n_ct; c++) {
        double s0a = 0.0, s1a = 0.0, s0b = 0.0, s1b = 0.0;
#pragma unroll
        for (uint32_t t = 0; t < BETA; t++) {
            const double da = nttfp::i2d((long long)p[t][srcA]), db = nttfp::i2d((long long)p[t][srcB]);
            p[t] += str[t];
            s0a += kip_mul(da, k0a[t], qd, qinv);
            s1a += kip_mul(da, k1a[t], qd, qinv);
            s0b += kip_mul(db, k0b[t], qd, qinv);
            s1b += kip_mul(db, k1b[t], qd, qinv);
        }
        if (accum_out) {
            const ulonglong2 p0 = *reinterpret_cast<const ulonglong2*>(o), p1 = *reinterpret_cast<const ulonglong2*>(o + en);
            s0a += nttfp::i2d((long long)p0.x), s0b += nttfp::i2d((long long)p0.y);
            s1a += nttfp::i2d((long long)p1.x), s1b += nttfp::i2d((long long)p1.y);
        }
        *reinterpret_cast<ulonglong2*>(o) = make_ulonglong2(nttfp::canon(nttfp::red(s0a, qd, qinv), q),
                                                             nttfp::canon(nttfp::red(s0b, qd, qinv), q));
        *reinterpret_cast<ulonglong2*>(o + en) = make_ulonglong2(nttfp::canon(nttfp::red(s1a, qd, qinv), q),
                                                                  nttfp::canon(nttfp::red(s1b, qd, qinv), q));
        o += ostep;
    }
}

// Key inner product with the automorphism fused on load, both key polynomials per thread (the digit gathers are
// shared): acc[gi][j][e][k] = sum_t ext[t][e][src_g(k)] * key[gi][t][j][limb(e)][k]  (mod r), j = 0, 1.
__global__ void __launch_bounds__(kT) k_kip2(const uint64_t* __restrict__ ext, const uint64_t* __restrict__ keys,
                                             uint64_t* __restrict__ acc, GBatch gb, uint32_t log_n, uint32_t level,
                                             uint32_t L, uint32_t A, uint32_t dnum, uint32_t beta, ModTab tab,
                                             uint64_t ext_stride, uint32_t perm) {
    const uint32_t n = 1u << log_n, E = level + A, T = L + A;
    const uint32_t e = blockIdx.y, gi = blockIdx.z;
    const uint32_t li = e < level ? e : L + (e - level);
    const uint32_t k = blockIdx.x * kT + threadIdx.x;
    const uint32_t src = galois_src_index(k, gb.g[gi], log_n);
    const uint64_t* key = keys + (size_t)gb.key[gi] * dnum * 2 * T * n + (size_t)li * n + k;
    const Barrett br = tab.br(li);
    // key-stationary: the key words of this position are fetched from HBM for the first input and served from L1
    // for the others (same addresses, same thread)
    for (uint32_t c = 0; c < gb.n_ct; c++) {
        const uint64_t* ex = ext + (size_t)c * ext_stride;
        U128 s0{0, 0}, s1{0, 0};
        for (uint32_t t = 0; t < beta; t++) {
            uint64_t dv = ex[((size_t)t * E + ext_row(perm, t, e, A, E, level)) * n + src];
            mac128(s0, dv, __ldg(key + ((size_t)t * 2 + 0) * T * n));
            mac128(s1, dv, __ldg(key + ((size_t)t * 2 + 1) * T * n));
            if ((t & 3) == 3 && t + 1 < beta) {
                s0.lo = barrett128(s0.hi, s0.lo, br);
                s0.hi = 0;
                s1.lo = barrett128(s1.hi, s1.lo, br);
                s1.hi = 0;
            }
        }
        const size_t r = (size_t)c * gb.cnt + gi;
        acc[((r * 2 + 0) * E + e) * n + k] = barrett128(s0.hi, s0.lo, br);
        acc[((r * 2 + 1) * E + e) * n + k] = barrett128(s1.hi, s1.lo, br);
    }
}

// ModDown conversion: z[gi][j][i][k] = sum_k' y_k' [P/p_k']_{q_i}  (mod q_i), y_k' = [pc_k' (P/p_k')^-1]_{p_k'}
// taken centred in (-p/2, p/2] (R10: zero-mean conversion overflow), pc = INTT'ed P limbs of acc.
__global__ void __launch_bounds__(kT) k_moddown_convert(const uint64_t* __restrict__ acc, uint64_t* __restrict__ z,
                                                        uint32_t log_n, uint32_t level, uint32_t L, uint32_t A,
                                                        ModTab tab, const uint64_t* __restrict__ cm) {
    const uint32_t n = 1u << log_n, E = level + A;
    const uint32_t i = blockIdx.y, gj = blockIdx.z;
    const uint32_t k = blockIdx.x * kT + threadIdx.x;
    const uint64_t* phinv = cm;
    const uint64_t* ph = cm + (size_t)A * 2 + (size_t)i * A * 2;
    const uint64_t q = tab.q[i];
    const uint64_t* pc = acc + ((size_t)gj * E + level) * n;
    const uint64_t* pmodq = cm + (size_t)A * 2 + (size_t)level * A * 2 + (size_t)level * 2 + (size_t)i * A;
    const Barrett bq = tab.br(i);
    uint64_t sum = 0;
    for (uint32_t a = 0; a < A; a++) {
        const uint64_t p = tab.q[L + a];
        uint64_t y = mul_shoup(pc[(size_t)a * n + k], phinv[2 * a], phinv[2 * a + 1], p);
        uint64_t yq = reduce64(y, bq);
        if (y > (p >> 1)) yq = sub_mod(yq, pmodq[a], q);
        sum += mul_shoup_lazy(yq, ph[2 * a], ph[2 * a + 1], q);
    }
    z[((size_t)gj * level + i) * n + k] = reduce64(sum, bq);
}

// Same conversion, one thread per word position producing all `level` target limbs: the alpha centred residues
// y_k' are computed once (not once per target limb), and y_k' [P/p_k']_{q_i} is a lazy Shoup product of the
// un-reduced y (< p < 2^64 is a valid Shoup input); the centring adds the precomputed -[p_k' P/p_k']_{q_i}.
// Constants per (i, k'): [P/p_k']_{q_i}, its Shoup companion, q_i - [p_k' (P/p_k')]_{q_i}  (md2, [level][A][3]).
__global__ void __launch_bounds__(kT) k_moddown_convert2(const uint64_t* __restrict__ acc, uint64_t* __restrict__ z,
                                                         uint32_t log_n, uint32_t level, uint32_t L, uint32_t A,
                                                         ModTab tab, const uint64_t* __restrict__ cm,
                                                         const uint64_t* __restrict__ md2) {
    const uint32_t n = 1u << log_n, E = level + A;
    const uint32_t gj = blockIdx.y;
    const uint32_t k = blockIdx.x * kT + threadIdx.x;
    const uint64_t* pc = acc + ((size_t)gj * E + level) * n + k;
    uint64_t y[8];
    bool neg[8];
#pragma unroll
    for (uint32_t a = 0; a < 8; a++) {
        if (a < A) {
            const uint64_t p = tab.q[L + a];
            y[a] = mul_shoup(pc[(size_t)a * n], cm[2 * a], cm[2 * a + 1], p);
            neg[a] = y[a] > (p >> 1);
        }
    }
    for (uint32_t i = 0; i < level; i++) {
        const uint64_t q = tab.q[i];
        const uint64_t* c = md2 + (size_t)i * A * 3;
        uint64_t sum = 0;
#pragma unroll
        for (uint32_t a = 0; a < 8; a++) {
            if (a < A) {
                sum += mul_shoup_lazy(y[a], c[3 * a], c[3 * a + 1], q);   // [0, 2q)
                if (neg[a]) sum += c[3 * a + 2];                          // [0, q)
            }
        }
        z[((size_t)gj * level + i) * n + k] = reduce64(sum, tab.br(i));   // sum < 3 A q < 2^(2w+2)
    }
}

// FP64 version (all moduli < 2^50, ntt_fp.cuh arithmetic): y_k' = [pc_k' (P/p_k')^-1]_{p_k'} as the exact centred
// representative in [-(p-1)/2, (p-1)/2] (R10), then z_i = sum_k' y_k' [P/p_k']_{q_i} with |sum| <= 2.5 q_i,
// one centred reduction, canonical store -- the same words as k_moddown_convert2.
__device__ __forceinline__ double y_centred(double x, double p, double hp, double w, double wq) {
    double r = nttfp::mulmod(x, w, wq, p);      // |r| <= 0.625 p, r == x w mod p
    r = r > hp ? r - p : r;
    return r < -hp ? r + p : r;
}
__global__ void __launch_bounds__(kT) k_moddown_convert_fp(const uint64_t* __restrict__ acc, uint64_t* __restrict__ z,
                                                           uint32_t log_n, uint32_t level, uint32_t L, uint32_t A,
                                                           ModTab tab, const double* __restrict__ mf) {
    const uint32_t n = 1u << log_n, E = level + A;
    const uint32_t gj = blockIdx.y;
    const uint32_t k = blockIdx.x * kT + threadIdx.x;
    const uint64_t* pc = acc + ((size_t)gj * E + level) * n + k;
    double y[8];
#pragma unroll
    for (uint32_t a = 0; a < 8; a++) {
        if (a < A) {
            const uint64_t p = tab.q[L + a];
            y[a] = y_centred(nttfp::i2d((long long)pc[(size_t)a * n]), (double)p, (double)(p >> 1),
                             __ldg(mf + 2 * a), __ldg(mf + 2 * a + 1));
        }
    }
    const double* c = mf + (size_t)A * 2;
    for (uint32_t i = 0; i < level; i++) {
        const uint64_t q = tab.q[i];
        const double qd = (double)q;
        double s = 0.0;
#pragma unroll
        for (uint32_t a = 0; a < 8; a++)
            if (a < A) s += nttfp::mulmod(y[a], __ldg(c + ((size_t)i * A + a) * 2), __ldg(c + ((size_t)i * A + a) * 2 + 1), qd);
        z[((size_t)gj * level + i) * n + k] = nttfp::canon(nttfp::red(s, qd, 1.0 / qd), q);
    }
}

// Same conversion with every constant in the kernel-parameter (constant) bank and the target / source loops fully
// unrolled to fixed bounds: the products read their constants as instruction operands instead of ~100 uniform
// global loads and 12 double divisions per position (level <= 16, alpha <= 8).
struct MDConstFp {
    double yw[8], ywq[8], p[8], hp[8];    // (P/p_k)^-1 mod p_k centred, RN(./p_k), p_k, floor(p_k / 2)
    double c[16][8], cq[16][8];           // [P/p_k]_{q_i} centred, RN(./q_i)
    double q[16], qinv[16];               // q_i, RN(1/q_i)
};
__global__ void __launch_bounds__(kT) k_moddown_convert_fpc(const uint64_t* __restrict__ acc, uint64_t* __restrict__ z,
                                                            uint32_t log_n, uint32_t level, uint32_t A,
                                                            const __grid_constant__ MDConstFp mc) {
    const uint32_t n = 1u << log_n, E = level + A;
    const uint32_t gj = blockIdx.y;
    const uint32_t k = blockIdx.x * kT + threadIdx.x;
    const uint64_t* pc = acc + ((size_t)gj * E + level) * n + k;
    double y[8];
#pragma unroll
    for (uint32_t a = 0; a < 8; a++)
        if (a < A) y[a] = y_centred(nttfp::i2d((long long)pc[(size_t)a * n]), mc.p[a], mc.hp[a], mc.yw[a], mc.ywq[a]);
#pragma unroll
    for (uint32_t i = 0; i < 16; i++) {
        if (i < level) {
            double s = 0.0;
#pragma unroll
            for (uint32_t a = 0; a < 8; a++)
                if (a < A) s += nttfp::mulmod(y[a], mc.c[i][a], mc.cq[i][a], mc.q[i]);
            z[((size_t)gj * level + i) * n + k] = nttfp::canon(nttfp::red(s, mc.q[i], mc.qinv[i]), (uint64_t)mc.q[i]);
        }
    }
}

// two consecutive positions per thread (16-byte loads and stores)
__global__ void __launch_bounds__(kT) k_moddown_convert_fpc2(const uint64_t* __restrict__ acc, uint64_t* __restrict__ z,
                                                             uint32_t log_n, uint32_t level, uint32_t A,
                                                             const __grid_constant__ MDConstFp mc) {
    const uint32_t n = 1u << log_n, E = level + A;
    const uint32_t gj = blockIdx.y;
    const uint32_t k = 2 * (blockIdx.x * kT + threadIdx.x);
    const uint64_t* pc = acc + ((size_t)gj * E + level) * n + k;
    double ya[4], yb[4];
#pragma unroll
    for (uint32_t a = 0; a < 4; a++)
        if (a < A) {
            const ulonglong2 w = *reinterpret_cast<const ulonglong2*>(pc + (size_t)a * n);
            ya[a] = y_centred(nttfp::i2d((long long)w.x), mc.p[a], mc.hp[a], mc.yw[a], mc.ywq[a]);
            yb[a] = y_centred(nttfp::i2d((long long)w.y), mc.p[a], mc.hp[a], mc.yw[a], mc.ywq[a]);
        }
#pragma unroll
    for (uint32_t i = 0; i < 16; i++) {
        if (i < level) {
            double sa = 0.0, sb = 0.0;
#pragma unroll
            for (uint32_t a = 0; a < 4; a++)
                if (a < A) {
                    sa += nttfp::mulmod(ya[a], mc.c[i][a], mc.cq[i][a], mc.q[i]);
                    sb += nttfp::mulmod(yb[a], mc.c[i][a], mc.cq[i][a], mc.q[i]);
                }
            const uint64_t q = (uint64_t)mc.q[i];
            *reinterpret_cast<ulonglong2*>(z + ((size_t)gj * level + i) * n + k) =
                make_ulonglong2(nttfp::canon(nttfp::red(sa, mc.q[i], mc.qinv[i]), q),
                                nttfp::canon(nttfp::red(sb, mc.q[i], mc.qinv[i]), q));
        }
    }
}

// out[gi][j][i][k] = (acc_q_i - z) * P^-1 (+ c0[i][src_g(k)] when j == 0)
__global__ void __launch_bounds__(kT) k_moddown_final(const uint64_t* __restrict__ acc, const uint64_t* __restrict__ z,
                                                      const uint64_t* __restrict__ c0, uint64_t* __restrict__ out,
                                                      GBatch gb, uint32_t log_n, uint32_t level, uint32_t A,
                                                      ModTab tab, const uint64_t* __restrict__ cm,
                                                      uint32_t add_mask, uint64_t add1_off, uint32_t gj0,
                                                      const uint64_t* __restrict__ add_src, uint64_t add_stride) {
    const uint32_t n = 1u << log_n, E = level + A;
    // gj: rotation-polynomial index in the batch; z holds the rows of this launch's sub-batch [gj0, gj0 + gridDim.z)
    const uint32_t i = blockIdx.y, gj = gj0 + blockIdx.z, j = gj & 1;
    const uint32_t c = gb.c_of(gj >> 1), gi = gb.gi_of(gj >> 1);
    const uint32_t k = blockIdx.x * kT + threadIdx.x;
    const uint64_t q = tab.q[i];
    const uint64_t* pinv = cm + (size_t)A * 2 + (size_t)level * A * 2 + (size_t)i * 2;
    uint64_t v = sub_mod(acc[((size_t)gj * E + i) * n + k], z[((size_t)blockIdx.z * level + i) * n + k], q);
    v = mul_shoup(v, pinv[0], pinv[1], q);
    if (j == 0 && c0) v = add_mod(v, c0[c * gb.in_stride + (size_t)i * n + galois_src_index(k, gb.g[gi], log_n)], q);
    if ((add_mask >> j) & 1) {
        const uint64_t* ab = add_src ? add_src + c * add_stride : c0 + c * gb.in_stride;
        v = add_mod(v, ab[(j ? add1_off : 0) + (size_t)i * n + k], q);
    }
    out[((((size_t)c * gb.out_c_stride + gb.oidx[gi]) * 2 + j) * level + i) * n + k] = v;
}

// FP64 final combine: out = (acc_{q_i} - z) P^{-1} (+ sigma_g(c0)) (+ added input) with one exact FP64 product
// (ncu had the integer kernel issue-bound at 74 %, 35 % IMAD from the 64-bit Shoup product and a runtime
// division for (input, element)); the FP64 pipe is otherwise idle here.
struct MDFinConst {
    double pinv[16], pinvq[16], q[16], qinv[16];   // [P^-1]_{q_i} centred, RN(./q_i), q_i, RN(1/q_i)
};
__global__ void __launch_bounds__(kT) k_moddown_final_fp(const uint64_t* __restrict__ acc, const uint64_t* __restrict__ z,
                                                         const uint64_t* __restrict__ c0, uint64_t* __restrict__ out,
                                                         GBatch gb, uint32_t log_n, uint32_t level, uint32_t A,
                                                         const __grid_constant__ MDFinConst fc, uint32_t add_mask,
                                                         uint64_t add1_off, uint32_t gj0,
                                                         const uint64_t* __restrict__ add_src, uint64_t add_stride) {
    const uint32_t n = 1u << log_n, E = level + A;
    const uint32_t i = blockIdx.y, gj = gj0 + blockIdx.z, j = gj & 1, r = gj >> 1;
    const uint32_t c = gb.n_ct == 1 ? 0u : r / gb.cnt, gi = r - c * gb.cnt;
    const uint32_t k = blockIdx.x * kT + threadIdx.x;
    const double qd = fc.q[i], qinv = fc.qinv[i];
    const long long dv = (long long)acc[((size_t)gj * E + i) * n + k] - (long long)z[((size_t)blockIdx.z * level + i) * n + k];
    double v = nttfp::mulmod(nttfp::i2d(dv), fc.pinv[i], fc.pinvq[i], qd);          // |v| <= 0.625 q
    const uint64_t* cb = c0 + c * gb.in_stride + (size_t)i * n;
    if (j == 0 && c0) v += nttfp::i2d((long long)cb[galois_src_index(k, gb.g[gi], log_n)]);
    if ((add_mask >> j) & 1) {
        const uint64_t* ab = (add_src ? add_src + c * add_stride : c0 + c * gb.in_stride) + (size_t)i * n;
        v += nttfp::i2d((long long)ab[(j ? add1_off : 0) + k]);
    }
    out[((((size_t)c * gb.out_c_stride + gb.oidx[gi]) * 2 + j) * level + i) * n + k] =
        nttfp::canon(nttfp::red(v, qd, qinv), (uint64_t)qd);
}

// Same combine for two consecutive positions per thread (16-byte loads of acc / z / the added input and 16-byte
// stores; the per-thread setup is shared).
__global__ void __launch_bounds__(kT) k_moddown_final_fp2(const uint64_t* __restrict__ acc, const uint64_t* __restrict__ z,
                                                          const uint64_t* __restrict__ c0, uint64_t* __restrict__ out,
                                                          GBatch gb, uint32_t log_n, uint32_t level, uint32_t A,
                                                          const __grid_constant__ MDFinConst fc, uint32_t add_mask,
                                                          uint64_t add1_off, uint32_t gj0,
                                                          const uint64_t* __restrict__ add_src, uint64_t add_stride) {
    const uint32_t n = 1u << log_n, E = level + A;
    const uint32_t i = blockIdx.y, gj = gj0 + blockIdx.z, j = gj & 1, r = gj >> 1;
    const uint32_t c = gb.n_ct == 1 ? 0u : r / gb.cnt, gi = r - c * gb.cnt;
    const uint32_t k = 2 * (blockIdx.x * kT + threadIdx.x);
    const double qd = fc.q[i], qinv = fc.qinv[i], pw = fc.pinv[i], pq = fc.pinvq[i];
    const ulonglong2 av = *reinterpret_cast<const ulonglong2*>(acc + ((size_t)gj * E + i) * n + k);
    const ulonglong2 zv = *reinterpret_cast<const ulonglong2*>(z + ((size_t)blockIdx.z * level + i) * n + k);
    double va = nttfp::mulmod(nttfp::i2d((long long)av.x - (long long)zv.x), pw, pq, qd);
    double vb = nttfp::mulmod(nttfp::i2d((long long)av.y - (long long)zv.y), pw, pq, qd);
    const uint64_t* cb = c0 + c * gb.in_stride + (size_t)i * n;
    if (j == 0 && c0) {
        const uint64_t g = gb.g[gi];
        va += nttfp::i2d((long long)cb[galois_src_index(k, g, log_n)]);
        vb += nttfp::i2d((long long)cb[galois_src_index(k + 1, g, log_n)]);
    }
    if ((add_mask >> j) & 1) {
        const uint64_t* ab = (add_src ? add_src + c * add_stride : c0 + c * gb.in_stride) + (size_t)i * n;
        const ulonglong2 w = *reinterpret_cast<const ulonglong2*>(ab + (j ? add1_off : 0) + k);
        va += nttfp::i2d((long long)w.x);
        vb += nttfp::i2d((long long)w.y);
    }
    const uint64_t q = (uint64_t)qd;
    *reinterpret_cast<ulonglong2*>(out + ((((size_t)c * gb.out_c_stride + gb.oidx[gi]) * 2 + j) * level + i) * n + k) =
        make_ulonglong2(nttfp::canon(nttfp::red(va, qd, qinv), q), nttfp::canon(nttfp::red(vb, qd, qinv), q));
}

// R19 (lazy ModDown of Layout-B giant steps): la[c][j][e] = (init ? 0 : la[c][j][e]) + acc[c][j][e] mod r_e over the
// extended basis Q_l u P, and out[c].c0 = add[c].c0 + sigma_g(ct[c].c0) (poly 1 of out is left to lazy_moddown).
// One Galois element per call (acc [n_ct][2][E][N'], rotation index = input index).
__global__ void __launch_bounds__(kT) k_lazy_accum(const uint64_t* __restrict__ acc, uint64_t* __restrict__ la,
                                                   const uint64_t* __restrict__ ct, uint64_t* out,
                                                   const uint64_t* add_src, uint64_t add_stride, GBatch gb,
                                                   uint32_t log_n, uint32_t level, uint32_t A, uint32_t L, ModTab tab,
                                                   uint32_t init, uint32_t c0_only) {
    // c0_only: the key inner product already summed into la (k_kip_fpt2 accum_out); only the sigma_g(c0) add is left
    const uint32_t n = 1u << log_n, E = level + A;
    const uint32_t e = blockIdx.y, gj = blockIdx.z, j = gj & 1, c = gj >> 1;
    const uint32_t k = blockIdx.x * kT + threadIdx.x;
    const uint64_t r = tab.q[e < level ? e : L + (e - level)];
    const size_t o = ((size_t)gj * E + e) * n + k;
    if (!c0_only) {
        uint64_t v = acc[o];
        if (!init) v = add_mod(v, la[o], r);
        la[o] = v;
    }
    if (j == 0 && e < level) {
        const uint64_t s = ct[c * gb.in_stride + (size_t)e * n + galois_src_index(k, gb.g[0], log_n)];
        const uint64_t* ab = (add_src ? add_src + c * add_stride : ct + c * gb.in_stride) + (size_t)e * n;
        out[(((size_t)c * gb.out_c_stride + gb.oidx[0]) * 2 * level + e) * n + k] = add_mod(ab[k], s, r);
    }
}

// ---------------------------------------------------------------- host driver

const uint64_t* find_key(const ensi_ctx* ctx, uint64_t g) {
    for (size_t i = 0; i < ctx->galois.size(); i++)
        if (ctx->galois[i] == g) return ctx->d_keys + i * (size_t)ctx->dnum * 2 * ctx->T * ctx->n;
    return nullptr;
}

static int key_index(const ensi_ctx* ctx, uint64_t g) {
    for (size_t i = 0; i < ctx->galois.size(); i++)
        if (ctx->galois[i] == g) return (int)i;
    return -1;
}

// ModDown of gcnt extended-basis polynomials acc [gcnt][E][N'] (rotation r = gj / 2, poly j = gj % 2) and the final
// combine out = (acc_Q - z) P^{-1} (+ sigma_g(c0) on poly 0 when c0 != NULL) (+ the added polynomials, add_mask):
// INTT of the P rows, conversion, NTT, combine.  The P rows of acc are transformed in place.
static void moddown_combine(ensi_ctx* ctx, ConvTables* cvt, uint64_t* acc, uint64_t* z, uint32_t gcnt, uint32_t level,
                            const uint64_t* c0, uint64_t* out, const GBatch& gb, uint32_t add_mask, uint64_t add1o,
                            const uint64_t* add_src, uint64_t add_stride, cudaStream_t st) {
    const uint32_t n = ctx->n, A = ctx->A, E = level + A;
    LimbMap pm = identity_map(A);
    for (uint32_t a = 0; a < A; a++) pm.limb[a] = (uint8_t)(ctx->L + a);
    pm.grp_rows = A;
    pm.grp_stride = E;
    pm.grp_off = level;
    // ModDown of the batch's 2 nr polynomials: INTT of the P rows, conversion, NTT, final combine
    const uint32_t g0 = 0;
    uint64_t* accs = acc;
    {
    ntt_inverse(ctx, accs, gcnt * A, pm, st);
    if (A <= 8 && ctx->ntt_fp_ok) {
        dim3 g(n / kT, gcnt);
        if (level <= 16) {
            MDConstFp mc{};
            const std::vector<double>& mf = cvt->h_moddown_fp;
            for (uint32_t a = 0; a < A; a++) {
                const uint64_t pk = ctx->mod[ctx->L + a];
                mc.yw[a] = mf[2 * a];
                mc.ywq[a] = mf[2 * a + 1];
                mc.p[a] = (double)pk;
                mc.hp[a] = (double)(pk >> 1);
            }
            for (uint32_t i = 0; i < level; i++) {
                mc.q[i] = (double)ctx->mod[i];
                mc.qinv[i] = 1.0 / mc.q[i];
                for (uint32_t a = 0; a < A; a++) {
                    mc.c[i][a] = mf[(size_t)A * 2 + ((size_t)i * A + a) * 2];
                    mc.cq[i][a] = mf[(size_t)A * 2 + ((size_t)i * A + a) * 2 + 1];
                }
            }
            if (A <= 4 && n >= 2 * kT)
                k_moddown_convert_fpc2<<<dim3(g.x / 2, g.y), kT, 0, st>>>(accs, z, ctx->log_n, level, A, mc);
            else
                k_moddown_convert_fpc<<<g, kT, 0, st>>>(accs, z, ctx->log_n, level, A, mc);
        } else
        k_moddown_convert_fp<<<g, kT, 0, st>>>(accs, z, ctx->log_n, level, ctx->L, A, ctx->tab,
                                               cvt->d_moddown_fp);
        ENSI_LAUNCH_CHECK(ctx);
    } else if (A <= 8) {
        dim3 g(n / kT, gcnt);
        k_moddown_convert2<<<g, kT, 0, st>>>(accs, z, ctx->log_n, level, ctx->L, A, ctx->tab, cvt->d_moddown,
                                             cvt->d_moddown2);
        ENSI_LAUNCH_CHECK(ctx);
    } else {
        dim3 g(n / kT, level, gcnt);
        k_moddown_convert<<<g, kT, 0, st>>>(accs, z, ctx->log_n, level, ctx->L, A, ctx->tab, cvt->d_moddown);
        ENSI_LAUNCH_CHECK(ctx);
    }
    ntt_forward(ctx, z, gcnt * level, identity_map(level), st);
    {
        dim3 g(n / kT, level, gcnt);
        if (ctx->ntt_fp_ok && level <= 16) {
            MDFinConst fc{};
            for (uint32_t i = 0; i < level; i++) {
                const uint64_t q = ctx->mod[i], w = cvt->h_pinv[i];
                fc.q[i] = (double)q;
                fc.qinv[i] = 1.0 / fc.q[i];
                fc.pinv[i] = w > q / 2 ? -(double)(q - w) : (double)w;
                fc.pinvq[i] = fc.pinv[i] / fc.q[i];
            }
            if (n >= 2 * kT) {
                dim3 g2(g.x / 2, g.y, g.z);
                k_moddown_final_fp2<<<g2, kT, 0, st>>>(acc, z, c0, out, gb, ctx->log_n, level, A, fc, add_mask,
                                                       add1o, g0, add_src, add_stride);
            } else
                k_moddown_final_fp<<<g, kT, 0, st>>>(acc, z, c0, out, gb, ctx->log_n, level, A, fc, add_mask,
                                                     add1o, g0, add_src, add_stride);
        } else
        k_moddown_final<<<g, kT, 0, st>>>(acc, z, c0, out, gb, ctx->log_n, level, A, ctx->tab, cvt->d_moddown,
                                          add_mask, add1o, g0, add_src, add_stride);
        ENSI_LAUNCH_CHECK(ctx);
    }
    }
}

// Batch sizes of the key-switching core (measured): up to 32 Galois elements and ~96
// rotations per key inner product, and at least 8 inputs before a single-element call is split over the two
// internal streams.
static constexpr uint32_t kKsBatch = 32, kKsRotCap = 96, kKsSplitMin = 8;

// Hoisted rotations of n_ct ciphertexts (input c at ct + c * in_stride words, [2][level][N']) by n_g Galois elements:
// rotation (c, r) -> out + (c * out_c_stride + r) ciphertexts.  One ModUp per input; per batch of up to 32 Galois
// elements one key-stationary KIP (each key word read once for all n_ct inputs) and one ModDown over n_ct * cnt.
int rotate_hoisted_multi(ensi_ctx* ctx, const uint64_t* ct, uint32_t n_ct, uint64_t in_stride, uint32_t level,
                         uint32_t n_g, const uint64_t* galois, uint64_t* out, uint32_t out_c_stride, cudaStream_t st,
                         const KsOpts* opts) {
    const uint32_t n = ctx->n, A = ctx->A, E = level + A;
    const KsOpts ko = opts ? *opts : KsOpts{};
    const uint64_t c1o = ko.c1_off ? ko.c1_off : (uint64_t)level * n;
    const uint64_t add1o = ko.add1_off ? ko.add1_off : (uint64_t)level * n;
    const uint64_t* keys_base = ko.key_base ? ko.key_base : ctx->d_keys;
    const uint64_t two_n_mask = 2ull * n - 1;
    const size_t ctw = (size_t)2 * level * n;
    if (A == 0) return set_err(ctx, ENSI_ENOKEY, "context has no special primes (num_p == 0): no key switching");
    if (n_ct == 0) return ENSI_OK;
    std::vector<uint32_t> idx;
    std::vector<uint64_t> gs;
    for (uint32_t r = 0; r < n_g; r++) {
        uint64_t g = galois[r] & two_n_mask;
        if (g == 1 && !ko.switch_identity) {
            if (ko.add_mask) return set_err(ctx, ENSI_EINVAL, "identity rotation with an added input");
            for (uint32_t c = 0; c < n_ct; c++)
                cudaMemcpyAsync(out + ((size_t)c * out_c_stride + r) * ctw, ct + c * in_stride, ctw * 8,
                                cudaMemcpyDeviceToDevice, st);
            continue;
        }
        int ki = ko.switch_identity ? (g == 1 ? 0 : -1) : key_index(ctx, g);
        if (ki < 0) return set_err(ctx, ENSI_ENOKEY, "no rotation key loaded for Galois element " + std::to_string(g));
        idx.push_back(r);
        gs.push_back(g);
    }
    if (idx.empty()) return ENSI_OK;
    if (ko.lazy_acc && (idx.size() != 1 || n_g != 1))
        return set_err(ctx, ENSI_EINVAL, "lazy ModDown: one (non-identity) Galois element per call");
    ConvTables* cvt = nullptr;
    int rc = conv_tables(ctx, level, &cvt);
    if (rc) return rc;
    const uint32_t beta = cvt->beta;
    if (beta > 8) return set_err(ctx, ENSI_EINVAL, "more than 8 key-switch digits");
    // One Galois element over many inputs (independent-input rotations, CCMM's replicate steps): the inputs are
    // split in two halves that run ModUp -> KIP -> ModDown on the two internal streams with disjoint scratch, so
    // one half's HBM-bound key inner product overlaps the other half's FP64-bound transforms.
    if (!ko.scratch && idx.size() == 1 && n_ct >= kKsSplitMin) {
        const uint32_t h0 = n_ct / 2, h1 = n_ct - h0;
        auto words = [&](uint32_t h) -> size_t {
            return (size_t)h * level * n + (size_t)h * beta * E * n + (size_t)h * 2 * E * n + (size_t)h * 2 * level * n;
        };
        rc = ensure_scratch(ctx, (words(h0) + words(h1)) * 8);
        if (rc) return rc;
        if (!ctx->st_ks[0]) {
            for (int i = 0; i < 2; i++) {
                cudaStreamCreateWithFlags(&ctx->st_ks[i], cudaStreamNonBlocking);
                cudaEventCreateWithFlags(&ctx->ev_ks_done[i], cudaEventDisableTiming);
            }
            cudaEventCreateWithFlags(&ctx->ev_ks_fork, cudaEventDisableTiming);
        }
        cudaEventRecord(ctx->ev_ks_fork, st);
        for (int i = 0; i < 2; i++) cudaStreamWaitEvent(ctx->st_ks[i], ctx->ev_ks_fork, 0);
        KsOpts k0 = ko, k1 = ko;
        k0.scratch = (uint64_t*)ctx->scratch;
        k1.scratch = (uint64_t*)ctx->scratch + words(h0);
        if (ko.add_src) k1.add_src = ko.add_src + (size_t)h0 * ko.add_stride;
        if (ko.lazy_acc) k1.lazy_acc = ko.lazy_acc + (size_t)h0 * 2 * E * n;
        rc = rotate_hoisted_multi(ctx, ct, h0, in_stride, level, n_g, galois, out, out_c_stride, ctx->st_ks[0], &k0);
        if (!rc)
            rc = rotate_hoisted_multi(ctx, ct + (size_t)h0 * in_stride, h1, in_stride, level, n_g, galois,
                                      out + (size_t)h0 * out_c_stride * ctw, out_c_stride, ctx->st_ks[1], &k1);
        for (int i = 0; i < 2; i++) {
            cudaEventRecord(ctx->ev_ks_done[i], ctx->st_ks[i]);
            cudaStreamWaitEvent(st, ctx->ev_ks_done[i], 0);
        }
        return rc;
    }
    // rotations per key-switch batch: up to 32 Galois elements, and at most ~96 rotations (n_ct * cnt) so the
    // (acc, z) scratch stays bounded (~2.8 GB per set at C2)
    const uint32_t nb = std::min<uint32_t>((uint32_t)idx.size(),
                                           std::max<uint32_t>(1, std::min<uint32_t>(kKsBatch, kKsRotCap / n_ct)));
    const uint32_t nbatches = (uint32_t)((idx.size() + nb - 1) / nb);
    // Batches alternate between two internal streams, each with its own (acc, z) buffers: the key inner product of
    // batch b+1 (HBM-bound) runs alongside the ModDown transforms of batch b (FP64/LSU-bound).
    const uint32_t nsets = nbatches > 1 ? 2 : 1;
    // scratch: coef [n_ct][level][n] | ext [n_ct][beta][E][n] | nsets x (acc [n_ct][nb][2][E][n] | z [n_ct][nb][2][level][n])
    const size_t w_coef = (size_t)n_ct * level * n, w_ext1 = (size_t)beta * E * n, w_acc = (size_t)n_ct * nb * 2 * E * n,
                 w_z = (size_t)n_ct * nb * 2 * level * n;
    if (!ko.scratch) {
        rc = ensure_scratch(ctx, (w_coef + n_ct * w_ext1 + nsets * (w_acc + w_z)) * 8);
        if (rc) return rc;
    }
    uint64_t* coef = ko.scratch ? ko.scratch : (uint64_t*)ctx->scratch;
    uint64_t* ext = coef + w_coef;
    uint64_t* set0 = ext + n_ct * w_ext1;
    if (nsets == 2 && !ctx->st_ks[0]) {
        for (int i = 0; i < 2; i++) {
            cudaStreamCreateWithFlags(&ctx->st_ks[i], cudaStreamNonBlocking);
            cudaEventCreateWithFlags(&ctx->ev_ks_done[i], cudaEventDisableTiming);
        }
        cudaEventCreateWithFlags(&ctx->ev_ks_fork, cudaEventDisableTiming);
    }

    // ---- ModUp (once per input; all inputs in one launch per step so small batches still fill the GPU)
    const uint32_t perm = (ctx->ntt_fp_ok && A <= 8) ? 1u : 0u;
    const bool own_direct = perm && beta <= 8;
    {
        NvtxRange nvtx_modup("ks.modup");
        const size_t row_b = (size_t)level * n * 8;
        // INTT of every input's c1 into coef: out of place (the first pass reads the input rows through a TMA
        // tensor map) when the strides allow, else copy + in place
        LimbMap sm = identity_map(level);
        sm.grp_rows = level;
        sm.grp_stride = (uint32_t)((n_ct > 1 ? in_stride : 2ull * level * n) / n);
        sm.grp_off = (uint32_t)(c1o / n);
        const bool strided_ok = in_stride % n == 0 && c1o % n == 0;
        if (!(strided_ok && ntt_inverse_from(ctx, ct, sm, coef, n_ct * level, identity_map(level), st))) {
            if (n_ct == 1)
                cudaMemcpyAsync(coef, ct + c1o, row_b, cudaMemcpyDeviceToDevice, st);
            else
                cudaMemcpy2DAsync(coef, row_b, ct + c1o, in_stride * 8, row_b, n_ct, cudaMemcpyDeviceToDevice, st);
            ntt_inverse(ctx, coef, n_ct * level, identity_map(level), st);
        }
        if (ctx->ntt_fp_ok && A <= 4 && beta <= 4 && E <= 16) {
            MUConstFp mc{};
            const std::vector<double>& uf = cvt->h_modup_fp;
            const size_t off1 = (size_t)beta * A * 2;
            for (uint32_t t = 0; t < beta; t++)
                for (uint32_t a = 0; a < A && t * A + a < level; a++) {
                    mc.cinv[t][a] = uf[((size_t)t * A + a) * 2];
                    mc.cinvq[t][a] = uf[((size_t)t * A + a) * 2 + 1];
                    for (uint32_t e = 0; e < E; e++) {
                        mc.c[t][e][a] = uf[off1 + (((size_t)t * E + e) * A + a) * 2];
                        mc.cq[t][e][a] = uf[off1 + (((size_t)t * E + e) * A + a) * 2 + 1];
                    }
                }
            for (uint32_t i = 0; i < level && i < 16; i++) mc.qs[i] = (double)ctx->mod[i];
            for (uint32_t e = 0; e < E; e++) {
                mc.r[e] = (double)ctx->mod[ext_limb(ctx, level, e)];
                mc.rinv[e] = 1.0 / mc.r[e];
            }
            dim3 g(n / kT, beta, n_ct);
            if (n >= 2 * kT)
                k_modup_convert_fpc2<<<dim3(g.x / 2, g.y, g.z), kT, 0, st>>>(coef, ext, ctx->log_n, level, ctx->L, A,
                                                                           mc, perm);
            else
                k_modup_convert_fpc<<<g, kT, 0, st>>>(coef, ext, ctx->log_n, level, ctx->L, A, mc, perm);
        } else if (ctx->ntt_fp_ok && A <= 8) {
            dim3 g(n / kT, beta, n_ct);
            k_modup_convert_fp<<<g, kT, 0, st>>>(coef, ext, ctx->log_n, level, ctx->L, A, ctx->tab,
                                                 cvt->d_modup_fp, perm);
        } else {
            dim3 g(n / kT, beta * E, n_ct);
            k_modup_convert<<<g, kT, 0, st>>>(coef, ext, ctx->log_n, level, ctx->L, A, ctx->tab, cvt->d_modup);
        }
        ENSI_LAUNCH_CHECK(ctx);
        if (perm) {
            // own limbs: the input's c1 limbs [tA, tA + c_t) in NTT form (c_t = A, or fewer in a partial last
            // digit), to rows [E - c_t, E) of every digit block -- unless the key inner product reads them straight
            // from the input (own_direct)
            for (uint32_t t = 0; t < beta && !own_direct; t++) {
                const uint32_t c_t = std::min(A, level - t * A);
                const size_t own_b = (size_t)c_t * n * 8;
                uint64_t* dst = ext + ((size_t)t * E + (E - c_t)) * n;
                const uint64_t* src = ct + c1o + (size_t)t * A * n;
                if (n_ct == 1)
                    cudaMemcpyAsync(dst, src, own_b, cudaMemcpyDeviceToDevice, st);
                else
                    cudaMemcpy2DAsync(dst, w_ext1 * 8, src, in_stride * 8, own_b, n_ct, cudaMemcpyDeviceToDevice, st);
            }
            if (level % A == 0) {          // every digit has E - A converted rows: one launch over all digits
                LimbMap em = identity_map(1);
                em.period = beta * (E - A);
                em.grp_rows = E - A;
                em.grp_stride = E;
                em.grp_off = 0;
                for (uint32_t t = 0, r = 0; t < beta; t++)
                    for (uint32_t e = 0; e < E; e++)
                        if (e < t * A || e >= (t + 1) * A) em.limb[r++] = (uint8_t)ext_limb(ctx, level, e);
                ntt_forward(ctx, ext, n_ct * beta * (E - A), em, st);
            } else {                       // partial last digit: one launch per digit (rows per block differ)
                for (uint32_t t = 0; t < beta; t++) {
                    const uint32_t lo = t * A, hi = std::min(lo + A, level), rows_t = E - (hi - lo);
                    LimbMap em = identity_map(1);
                    em.period = rows_t;
                    em.grp_rows = rows_t;
                    em.grp_stride = beta * E;
                    em.grp_off = t * E;
                    for (uint32_t e = 0, r = 0; e < E; e++)
                        if (e < lo || e >= hi) em.limb[r++] = (uint8_t)ext_limb(ctx, level, e);
                    ntt_forward(ctx, ext, n_ct * rows_t, em, st);
                }
            }
        } else {
            ntt_forward(ctx, ext, n_ct * beta * E, ext_map(ctx, level), st);
        }
    }

    if (nsets == 2) {
        cudaEventRecord(ctx->ev_ks_fork, st);
        for (int i = 0; i < 2; i++) cudaStreamWaitEvent(ctx->st_ks[i], ctx->ev_ks_fork, 0);
    }
    const cudaStream_t st_caller = st;

    // ---- per batch of Galois elements
    for (size_t b0 = 0; b0 < idx.size(); b0 += nb) {
        NvtxRange nvtx_batch("ks.kip_moddown_batch");
        const uint32_t bi = (uint32_t)(b0 / nb);
        cudaStream_t st = nsets == 2 ? ctx->st_ks[bi & 1] : st_caller;   // batches of a set run in order
        uint64_t* acc = set0 + (size_t)(bi % nsets) * (w_acc + w_z);
        uint64_t* z = acc + w_acc;
        const uint32_t cnt = (uint32_t)std::min<size_t>(nb, idx.size() - b0);
        GBatch gb{};
        for (uint32_t i = 0; i < cnt; i++) {
            gb.g[i] = gs[b0 + i];
            gb.key[i] = ko.switch_identity ? 0u : (uint32_t)key_index(ctx, gs[b0 + i]);
            gb.oidx[i] = idx[b0 + i];
        }
        gb.cnt = cnt;
        gb.n_ct = n_ct;
        gb.out_c_stride = out_c_stride;
        gb.in_stride = in_stride;
        const uint32_t nr = n_ct * cnt;   // rotations in this batch
        // R19: the two-position FP64 key inner product sums straight into the lazy accumulator (read-add-write), so
        // the batch's acc is never written and re-read; other KIP kernels keep acc and k_lazy_accum adds it
        const bool kip_lazy = ko.lazy_acc != nullptr;
        uint64_t* kip_out = kip_lazy ? ko.lazy_acc : acc;
        const uint32_t kip_accum = kip_lazy && !ko.lazy_init ? 1u : 0u;
        bool kip_fused_lazy = false;
        if (kip_lazy && !(ctx->ntt_fp_ok && beta <= 4 && n >= 2 * kT)) {
            kip_out = acc;                 // the k_kip_fpt2 path is not taken: unfused lazy accumulate below
        }
        {
            dim3 g(n / kT, E, cnt);
            if (ctx->ntt_fp_ok && beta <= 8) {
                const uint32_t lm = 1u;   // limb-major grid: a limb's gathered digit rows stay in L2 across the batch
                dim3 gk = lm ? dim3(n / kT, cnt, E) : g;
                const uint32_t pm = own_direct ? 2u : perm;
                const uint64_t* c1p = ct + c1o;
                switch (beta) {
#define ENSI_KIPT(B)                                                                                                   \
    case B:                                                                                                            \
        if (n >= 2 * kT) {                                                                                             \
            dim3 g2(gk.x / 2, gk.y, gk.z);                                                                             \
            k_kip_fpt2<B><<<g2, kT, 0, st>>>(ext, keys_base, kip_out, gb, ctx->log_n, level, ctx->L, A, ctx->dnum,     \
                                             ctx->tab, w_ext1, pm, lm, c1p, in_stride, kip_accum);                     \
            kip_fused_lazy = kip_lazy;                                                                                 \
        } else {                                                                                                       \
            k_kip_fpt<B><<<gk, kT, 0, st>>>(ext, keys_base, acc, gb, ctx->log_n, level, ctx->L, A, ctx->dnum,          \
                                            ctx->tab, w_ext1, pm, lm, c1p, in_stride);                                 \
        }                                                                                                              \
        break;
                    ENSI_KIPT(1)
                    ENSI_KIPT(2)
                    ENSI_KIPT(3)
                    ENSI_KIPT(4)
#undef ENSI_KIPT
                    default:
                        k_kip_fp<<<gk, kT, 0, st>>>(ext, keys_base, acc, gb, ctx->log_n, level, ctx->L, A, ctx->dnum,
                                                    beta, ctx->tab, w_ext1, pm, lm, c1p, in_stride);
                }
            }
            else
                k_kip2<<<g, kT, 0, st>>>(ext, keys_base, acc, gb, ctx->log_n, level, ctx->L, A, ctx->dnum, beta,
                                         ctx->tab, w_ext1, perm);
            ENSI_LAUNCH_CHECK(ctx);
        }
        if (ko.lazy_acc) {
            // R19: sum this giant step's key inner product into the lazy accumulator (Q_l u P) -- done by the KIP
            // itself when kip_fused_lazy -- and add (sigma_g(c0), 0) to the output now; the one ModDown per output
            // runs in lazy_moddown
            dim3 g(n / kT, kip_fused_lazy ? level : E, nr * 2);
            k_lazy_accum<<<g, kT, 0, st>>>(acc, ko.lazy_acc, ct, out, ko.add_src, ko.add_stride, gb, ctx->log_n, level,
                                          A, ctx->L, ctx->tab, ko.lazy_init ? 1u : 0u, kip_fused_lazy ? 1u : 0u);
            ENSI_LAUNCH_CHECK(ctx);
            continue;
        }
        moddown_combine(ctx, cvt, acc, z, nr * 2, level, ct, out, gb, ko.add_mask, add1o, ko.add_src, ko.add_stride, st);
    }
    if (nsets == 2) {
        for (int k = 0; k < 2; k++) {
            cudaEventRecord(ctx->ev_ks_done[k], ctx->st_ks[k]);
            cudaStreamWaitEvent(st, ctx->ev_ks_done[k], 0);
        }
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_err(ctx, e, "rotate_hoisted");
    return ENSI_OK;
}

int rotate_hoisted(ensi_ctx* ctx, const uint64_t* ct, uint32_t level, uint32_t n_g, const uint64_t* galois,
                   uint64_t* out, cudaStream_t st) {
    return rotate_hoisted_multi(ctx, ct, 1, 0, level, n_g, galois, out, 0, st);
}

// R19: out[c] += ModDown(la[c]) for both polynomials of n_ct outputs (la [n_ct][2][E][N'], out [n_ct][2][level][N'],
// in place), after every giant step went through rotate_hoisted_multi with KsOpts.lazy_acc.
int lazy_moddown(ensi_ctx* ctx, uint64_t* la, uint32_t n_ct, uint32_t level, uint64_t* out, cudaStream_t st) {
    if (n_ct == 0) return ENSI_OK;
    ConvTables* cvt = nullptr;
    int rc = conv_tables(ctx, level, &cvt);
    if (rc) return rc;
    const size_t ctw = (size_t)2 * level * ctx->n;
    rc = ensure_scratch(ctx, (size_t)n_ct * ctw * 8);              // z [n_ct][2][level][N']
    if (rc) return rc;
    GBatch gb{};
    gb.g[0] = 1;
    gb.key[0] = 0;
    gb.oidx[0] = 0;
    gb.cnt = 1;
    gb.n_ct = n_ct;
    gb.out_c_stride = 1;
    gb.in_stride = ctw;
    moddown_combine(ctx, cvt, la, (uint64_t*)ctx->scratch, 2 * n_ct, level, nullptr, out, gb, 3u, (uint64_t)level * ctx->n,
                    out, ctw, st);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? ENSI_OK : cuda_err(ctx, e, "lazy_moddown");
}

}  // namespace ensi
