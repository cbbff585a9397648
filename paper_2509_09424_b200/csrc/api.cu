// api.cu -- the C ABI of libensi.so (include/ensi.h).  Argument validation, key/weight management,
// Layout-A/B orchestration.  Every arithmetic step runs in the kernels of ntt.cu, accum.cu, accum_tc.cu,
// keyswitch.cu and poly.cu; the host does CRT/decode only inside ensi_decrypt_debug (debug, never timed).
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "ensi_internal.h"

using namespace ensi;

namespace ensi {

int set_err(ensi_ctx* ctx, int code, const std::string& msg) {
    if (ctx) ctx->err = msg;
    return code;
}
int cuda_err(ensi_ctx* ctx, cudaError_t e, const char* where) {
    return set_err(ctx, ENSI_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

int ensure_scratch(ensi_ctx* ctx, size_t bytes) {
    if (bytes <= ctx->scratch_bytes) return ENSI_OK;
    if (ctx->scratch) {
        cudaDeviceSynchronize();
        cudaFree(ctx->scratch);
        ctx->scratch = nullptr;
        ctx->scratch_bytes = 0;
    }
    cudaError_t e = cudaMalloc(&ctx->scratch, bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return set_err(ctx, ENSI_ENOMEM, "scratch allocation of " + std::to_string(bytes) + " bytes failed");
    }
    ctx->scratch_bytes = bytes;
    return ENSI_OK;
}

}  // namespace ensi

namespace {

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        // a non-sticky error left in the runtime's per-thread slot by earlier, unrelated CUDA calls of the process
        // (seen: "invalid device ordinal" after NCCL / torch teardown in the GPU test run) would otherwise be
        // reported by this call's cudaGetLastError() check; sticky errors (a faulted context) persist regardless
        cudaGetLastError();
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

int check_view(ensi_ctx* ctx, const ensi_ct_view* v, const char* name) {
    if (!v || !v->data) return set_err(ctx, ENSI_EINVAL, std::string(name) + ": NULL view or data");
    if (v->level < 1 || v->level > ctx->L)
        return set_err(ctx, ENSI_ELEVEL, std::string(name) + ": level " + std::to_string(v->level) +
                                             " outside [1, num_q=" + std::to_string(ctx->L) + "]");
    return ENSI_OK;
}

bool overlaps(const ensi_ct_view* a, const ensi_ct_view* b, uint32_t n) {
    const uint8_t* a0 = (const uint8_t*)a->data;
    const uint8_t* a1 = a0 + (size_t)a->count * 2 * a->level * n * 8;
    const uint8_t* b0 = (const uint8_t*)b->data;
    const uint8_t* b1 = b0 + (size_t)b->count * 2 * b->level * n * 8;
    return a0 < b1 && b0 < a1;
}

// pack a d x m ternary matrix (row stride ldw) into [rows][2][mw] planes
int pack_planes(ensi_ctx* ctx, const int8_t* W, uint32_t d, uint32_t m, uint32_t ldw, uint32_t mw,
                std::vector<uint32_t>& out, uint64_t* nnz) {
    out.assign((size_t)d * 2 * mw, 0u);
    uint64_t cnt = 0;
    for (uint32_t j = 0; j < d; j++) {
        const int8_t* row = W + (size_t)j * ldw;
        uint32_t* pos = out.data() + (size_t)j * 2 * mw;
        uint32_t* neg = pos + mw;
        for (uint32_t i = 0; i < m; i++) {
            int8_t v = row[i];
            if (v == 1) {
                pos[i >> 5] |= 1u << (i & 31);
                cnt++;
            } else if (v == -1) {
                neg[i >> 5] |= 1u << (i & 31);
                cnt++;
            } else if (v != 0) {
                return set_err(ctx, ENSI_ENOTTERNARY, "W[" + std::to_string(j) + "][" + std::to_string(i) +
                                                          "] = " + std::to_string((int)v) + " is not in {-1,0,1}");
            }
        }
    }
    if (nnz) *nnz = cnt;
    return ENSI_OK;
}

// opts.kernel -> tensor-core variant: 0/2 best, 3 single CTA, 4 pairs without multicast
int tc_variant(uint32_t kernel) { return kernel == 3 ? TC_ONE_CTA : kernel == 4 ? TC_PAIR : TC_AUTO; }

// opts.kernel -> accumulate path (*tc: tensor cores).  0 picks the tensor-core path when the device and moduli
// allow it (sm_100a, 2^32 < q < 2^60, d < 2^22 for the epilogue's 64-bit narrow combine), else the CUDA cores;
// 2..4 request a tensor-core variant and fail with EINVAL where it is unavailable.
int select_kernel(ensi_ctx* ctx, uint32_t kernel, uint32_t level, uint32_t d, bool* tc) {
    if (kernel > 4) return set_err(ctx, ENSI_EINVAL, "opts.kernel must be 0..4");
    const bool ok = tc_supported(ctx, level) && d < (1u << 22);
    if (kernel >= 2 && !ok)
        return set_err(ctx, ENSI_EINVAL,
                       "tensor-core accumulate not available for these parameters (sm_100a, 2^32 < q < 2^60, d < 2^22)");
    *tc = kernel >= 2 || (kernel == 0 && ok);
    return ENSI_OK;
}

struct LayoutBPlan {
    uint32_t k, n_in, B, G, rotations;
};

int plan_b(ensi_ctx* ctx, uint32_t d, uint32_t m, uint32_t s, uint32_t baby, LayoutBPlan* p) {
    const uint32_t slots = ctx->n / 2;
    if (s == 0 || (s & (s - 1)) || s > slots)
        return set_err(ctx, ENSI_EDIM, "block_s must be a power of two <= N'/2");
    uint32_t pow2d = 1;
    while (pow2d < d) pow2d <<= 1;
    p->k = std::min(slots / s, pow2d);
    p->n_in = (d + p->k - 1) / p->k;
    if (baby == 0) {
        uint64_t best = UINT64_MAX;
        for (uint32_t b = 1; b <= p->k; b <<= 1) {
            uint64_t cost = (uint64_t)(b - 1) * p->n_in + (uint64_t)(p->k / b - 1) * m;
            if (cost < best) {
                best = cost;
                p->B = b;
            }
        }
    } else {
        if ((baby & (baby - 1)) || baby > p->k || p->k % baby)
            return set_err(ctx, ENSI_EDIM, "baby must be a power of two dividing k");
        p->B = baby;
    }
    p->G = p->k / p->B;
    p->rotations = (p->B - 1) * p->n_in + (p->G - 1) * m;
    return ENSI_OK;
}

// Layout-B weights for (k, B): one packed weight object per giant step gam, whose row r = c*B + b holds
// W[c*k + gam*B + b] (zero rows past d).  Built once per (k, B) and cached on the weights handle.
int weights_b(ensi_ctx* ctx, ensi_weights* w, uint32_t k, uint32_t B, uint32_t n_in,
              const std::vector<ensi_weights*>** out) {
    auto key = std::make_pair(k, B);
    auto it = w->packs_b.find(key);
    if (it != w->packs_b.end()) {
        *out = &it->second;
        return ENSI_OK;
    }
    const uint32_t G = k / B, rows = n_in * B;
    std::vector<int8_t> Wg((size_t)rows * w->m);
    std::vector<ensi_weights*> subs;
    for (uint32_t gam = 0; gam < G; gam++) {
        std::fill(Wg.begin(), Wg.end(), 0);
        for (uint32_t c = 0; c < n_in; c++)
            for (uint32_t b = 0; b < B; b++) {
                uint32_t col = c * k + gam * B + b;
                if (col < w->d) std::memcpy(&Wg[((size_t)c * B + b) * w->m], &w->host[(size_t)col * w->m], w->m);
            }
        ensi_weights* sw = nullptr;
        int rc = ensi_weights_pack(ctx, Wg.data(), rows, w->m, w->m, &sw);
        if (rc) {
            for (auto* x : subs) ensi_weights_destroy(x);
            return rc;
        }
        subs.push_back(sw);
    }
    auto& slot = w->packs_b[key];
    slot = std::move(subs);
    *out = &slot;
    return ENSI_OK;
}

// Layout B (R11) after validation: hoisted baby steps of all inputs, the Algorithm-1 accumulate per giant step,
// and the giant-step rotations of the m partial sums.  The giant steps are key-stationary: one
// rotate_hoisted_multi call per chunk of outputs reads the giant key once for the whole chunk, and its final
// combine adds the running sum in place (out = acc_out, add_src = acc_out), so no per-output rotation launch, no
// rotated copy and no separate add pass.  Output words are those of O11 (modular additions are exact).
int layout_b_run(ensi_ctx* ctx, const ensi_ct_view* x, ensi_weights* w, const std::vector<ensi_weights*>& subs,
                 const LayoutBPlan& p, const ensi_pcmm_opts& o, bool tc, uint64_t* acc_out, cudaStream_t st) {
    const uint32_t m = w->m, level = x->level;
    const size_t ctw = (size_t)2 * level * ctx->n;
    const uint32_t rows = p.n_in * p.B;
    // rotated inputs R [rows] and (G > 1) the giant-step partials T [m]: ctx-owned, grown on demand (cudaMallocAsync
    // would return the 9+ GB to the OS at every synchronisation under the default pool release threshold)
    // R19 lazy ModDown (G > 2 only: with one giant rotation per output it is the eager path): the extended-basis
    // accumulators of all m outputs, la [m][2][level + A][N']
    const bool lazy = o.moddown_lazy && p.G > 2;
    const size_t law = (size_t)2 * (level + ctx->A) * ctx->n;
    const size_t need = ((size_t)rows + (p.G > 1 ? (size_t)m : 0)) * ctw + (lazy ? (size_t)m * law : 0);
    if (ctx->lb_words < need) {
        cudaStreamSynchronize(st);
        cudaFree(ctx->lb_buf);
        ctx->lb_buf = nullptr;
        ctx->lb_words = 0;
        cudaError_t ea = cudaMalloc(&ctx->lb_buf, need * 8);
        if (ea != cudaSuccess) {
            cudaGetLastError();
            return set_err(ctx, ENSI_ENOMEM, "layout B scratch allocation failed");
        }
        ctx->lb_words = need;
    }
    uint64_t* R = ctx->lb_buf;
    uint64_t* Tg = p.G > 1 ? R + (size_t)rows * ctw : nullptr;
    uint64_t* La = lazy ? Tg + (size_t)m * ctw : nullptr;
    auto accum_b = [&](uint32_t gm, uint64_t* dst) -> int {
        ensi_weights* sw = subs[gm];
        return tc ? accum_ternary_tc(ctx, R, sw->d, sw, dst, level, st, 0, 0, tc_variant(o.kernel))
                  : accum_ternary(ctx, R, sw->d, sw->d_planes, sw->mw, m, dst, level, st);
    };
    std::vector<uint64_t> gb(p.B);
    for (uint32_t b = 0; b < p.B; b++) gb[b] = galois_of_rotation(ctx->log_n, (int64_t)o.block_s * b);
    // baby steps for all inputs at once: key-stationary (each rotation key read once for the n_in inputs)
    int rc;
    {
        NvtxRange r_("layoutB.baby_rotations");
        rc = rotate_hoisted_multi(ctx, x->data, p.n_in, ctw, level, p.B, gb.data(), R, p.B, st);
    }
    if (!rc) {
        NvtxRange r_("layoutB.accumulate");
        rc = accum_b(0, acc_out);
    }
    for (uint32_t gm = 1; gm < p.G && !rc; gm++) {
        NvtxRange r_("layoutB.giant_step");
        rc = accum_b(gm, Tg);
        const uint64_t gg = galois_of_rotation(ctx->log_n, (int64_t)o.block_s * p.B * gm);
        // chunks of at most 96 outputs bound the key-switching scratch (as ensi_rotate_batch)
        for (uint32_t c0 = 0; c0 < m && !rc; c0 += 96) {
            const uint32_t nc = std::min<uint32_t>(96, m - c0);
            KsOpts ko;
            ko.add_mask = 3;
            ko.add_src = acc_out + (size_t)c0 * ctw;
            ko.add_stride = ctw;
            if (lazy) {
                ko.lazy_acc = La + (size_t)c0 * law;
                ko.lazy_init = gm == 1;
            }
            rc = rotate_hoisted_multi(ctx, Tg + (size_t)c0 * ctw, nc, ctw, level, 1, &gg, acc_out + (size_t)c0 * ctw, 1,
                                      st, &ko);
        }
    }
    // R19: one ModDown per output of the summed giant-step key inner products, added in place
    NvtxRange r_lazy(lazy ? "layoutB.lazy_moddown" : "layoutB.done");
    for (uint32_t c0 = 0; lazy && c0 < m && !rc; c0 += 96) {
        const uint32_t nc = std::min<uint32_t>(96, m - c0);
        rc = lazy_moddown(ctx, La + (size_t)c0 * law, nc, level, acc_out + (size_t)c0 * ctw, st);
    }
    return rc;
}

// iterative radix-2 complex FFT (host, debug decode only): a[k] = sum_j a_j e^{sign 2 pi i jk / n}
void fft_host(std::vector<std::complex<double>>& a, int sign) {
    const size_t n = a.size();
    for (size_t i = 1, j = 0; i < n; i++) {
        size_t bit = n >> 1;
        for (; j & bit; bit >>= 1) j ^= bit;
        j ^= bit;
        if (i < j) std::swap(a[i], a[j]);
    }
    for (size_t len = 2; len <= n; len <<= 1) {
        double ang = sign * 2 * M_PI / (double)len;
        for (size_t i = 0; i < n; i += len)
            for (size_t k = 0; k < len / 2; k++) {
                std::complex<double> w(std::cos(ang * k), std::sin(ang * k));
                std::complex<double> u = a[i + k], v = a[i + k + len / 2] * w;
                a[i + k] = u + v;
                a[i + k + len / 2] = u - v;
            }
    }
}

}  // namespace

extern "C" {

uint32_t ensi_abi_version(void) { return ENSI_ABI_VERSION; }

const char* ensi_last_error(const ensi_ctx* ctx) { return ctx ? ctx->err.c_str() : "NULL context"; }

uint64_t ensi_launch_count(const ensi_ctx* ctx) { return ctx ? ctx->launches : 0; }

int ensi_last_compact_plan(const ensi_ctx* ctx, uint32_t* cluster_pairs, uint32_t* clusters) {
    if (!ctx || !cluster_pairs || !clusters) return ENSI_EINVAL;
    *cluster_pairs = ctx->tcc_cpairs;
    *clusters = ctx->tcc_nclust;
    return ENSI_OK;
}

uint32_t ensi_pcmm_kernel(const ensi_ctx* ctx, uint32_t level, uint32_t requested) {
    if (!ctx) return 0;
    const bool tc = tc_supported(ctx, level);
    if (requested == 1) return 1;
    if (requested >= 2 && requested <= 4) return tc ? requested : 0;
    return tc ? 2 : 1;
}

int ensi_ctx_create(const ensi_params* prm, int cuda_device, ensi_ctx** out) {
    if (!out) return ENSI_EINVAL;
    *out = nullptr;
    if (!prm) return ENSI_EINVAL;
    if (prm->log_n < 8 || prm->log_n > 17) return ENSI_EINVAL;
    if (prm->num_q < 1 || prm->num_q + prm->num_p > ENSI_MAXT) return ENSI_EINVAL;
    if (prm->num_p > 0) {
        if (prm->dnum < 1 || prm->num_p != (prm->num_q + prm->dnum - 1) / prm->dnum) return ENSI_EINVAL;
    }
    ensi_ctx* ctx = new (std::nothrow) ensi_ctx();
    if (!ctx) return ENSI_ENOMEM;
    ctx->device = cuda_device;
    ctx->log_n = prm->log_n;
    ctx->n = 1u << prm->log_n;
    ctx->L = prm->num_q;
    ctx->A = prm->num_p;
    ctx->dnum = prm->num_p ? prm->dnum : 0;
    ctx->T = prm->num_q + prm->num_p;
    ctx->log2_scale = prm->log2_scale > 0 ? prm->log2_scale : 40.0;
    uint64_t qq[ENSI_MAXT], pp[ENSI_MAXT];
    if (!prm->q || (prm->num_p && !prm->p)) gen_primes(prm->log_n, prm->num_q, prm->num_p, qq, pp);
    for (uint32_t i = 0; i < ctx->L; i++) ctx->mod[i] = prm->q ? prm->q[i] : qq[i];
    for (uint32_t k = 0; k < ctx->A; k++) ctx->mod[ctx->L + k] = prm->p ? prm->p[k] : pp[k];
    const uint64_t two_n = 2ull * ctx->n;
    for (uint32_t i = 0; i < ctx->T; i++) {
        uint64_t q = ctx->mod[i];
        bool ok = q > 2 && q < (1ull << 60) && (q % two_n) == 1 && is_prime_u64(q);
        for (uint32_t j = 0; j < i && ok; j++) ok = ctx->mod[j] != q;
        if (!ok) {
            int rc = set_err(ctx, ENSI_EINVAL, "modulus " + std::to_string(q) + " rejected");
            delete ctx;
            return rc;
        }
    }
    DeviceGuard g(cuda_device);
    cudaError_t e = cudaSetDevice(cuda_device);
    if (e != cudaSuccess) {
        delete ctx;
        return ENSI_ECUDA;
    }
    // keep stream-ordered allocations (rescale epilogue temporaries) pooled instead of returning them to the OS
    {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, cuda_device) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
        cudaGetLastError();
    }
    // twiddle tables
    const uint32_t n = ctx->n;
    std::vector<uint64_t> tw((size_t)ctx->T * 4 * n + 2 * ctx->T);
    for (uint32_t i = 0; i < ctx->T; i++) {
        const uint64_t q = ctx->mod[i];
        ctx->psi[i] = min_root(q, ctx->log_n);
        const uint64_t ipsi = invmod_h(ctx->psi[i], q);
        uint64_t* base = tw.data() + (size_t)i * 4 * n;
        // psi^k and psi^-k in natural order, then scatter by bit reversal
        uint64_t p = 1, ip = 1;
        for (uint32_t k = 0; k < n; k++) {
            uint32_t r = 0;
            for (uint32_t b = 0, kk = k; b < ctx->log_n; b++, kk >>= 1) r = (r << 1) | (kk & 1);
            base[r] = p;
            base[n + r] = shoup_h(p, q);
            base[2 * n + r] = ip;
            base[3 * n + r] = shoup_h(ip, q);
            p = mulmod_h(p, ctx->psi[i], q);
            ip = mulmod_h(ip, ipsi, q);
        }
        ctx->ninv[i] = invmod_h(n % q, q);
        ctx->ninv_sh[i] = shoup_h(ctx->ninv[i], q);
        tw[(size_t)ctx->T * 4 * n + 2 * i] = ctx->ninv[i];
        tw[(size_t)ctx->T * 4 * n + 2 * i + 1] = ctx->ninv_sh[i];
        Barrett b = barrett_h(q);
        ctx->tab.q[i] = q;
        ctx->tab.mu[i] = b.mu;
        ctx->tab.w[i] = b.w;
    }
    e = cudaMalloc(&ctx->d_tw, tw.size() * 8);
    if (e == cudaSuccess) e = cudaMemcpy(ctx->d_tw, tw.data(), tw.size() * 8, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
        std::vector<uint64_t> tw2((size_t)ctx->T * 4 * n);
        for (uint32_t i = 0; i < ctx->T; i++)
            for (uint32_t dir = 0; dir < 2; dir++)
                for (uint32_t k = 0; k < n; k++) {
                    const uint64_t* base = tw.data() + (size_t)i * 4 * n + (size_t)dir * 2 * n;
                    tw2[(((size_t)i * 2 + dir) * n + k) * 2 + 0] = base[k];
                    tw2[(((size_t)i * 2 + dir) * n + k) * 2 + 1] = base[n + k];
                }
        e = cudaMalloc(&ctx->d_tw2, tw2.size() * 8);
        if (e == cudaSuccess) e = cudaMemcpy(ctx->d_tw2, tw2.data(), tw2.size() * 8, cudaMemcpyHostToDevice);
    }
    ctx->ntt_fp_ok = true;
    for (uint32_t i = 0; i < ctx->T; i++) ctx->ntt_fp_ok = ctx->ntt_fp_ok && ctx->mod[i] < (1ull << 50);

    if (e == cudaSuccess && ctx->ntt_fp_ok) {
        // centred twiddle c (|c| < q/2, exact in a double) and RN(c / q) for the FP64 NTT (ntt_fp.cuh)
        std::vector<double> tw3((size_t)ctx->T * 4 * n + (size_t)ctx->T * 2);
        auto centred = [](uint64_t w, uint64_t q) -> double {
            return w > q / 2 ? -(double)(q - w) : (double)w;
        };
        // table position of natural index k: identity, except the lane-transposed block-pass region at N'=2^16
        // (ntt_fp.cuh): stage base m = 32768 >> lt (lt <= 3), block run b = m + sub (128 >> lt), k = b + tt J + j
        // (J = 8 >> lt) -> b + j 16 + tt
        auto tpos = [&](uint32_t k) -> uint32_t {
            if (ctx->log_n != 16 || k < 4096) return k;
            uint32_t lt = 0;
            while ((32768u >> lt) > k) lt++;
            const uint32_t m = 32768u >> lt, run = 128u >> lt, J = 8u >> lt;
            const uint32_t b = m + ((k - m) / run) * run, off = k - b, tt = off / J, j = off % J;
            return b + j * 16 + tt;
        };
        for (uint32_t i = 0; i < ctx->T; i++) {
            const uint64_t q = ctx->mod[i];
            for (uint32_t dir = 0; dir < 2; dir++)
                for (uint32_t k = 0; k < n; k++) {
                    const double c = centred(tw[(size_t)i * 4 * n + (size_t)dir * 2 * n + k], q);
                    const uint32_t kp = tpos(k);
                    tw3[(((size_t)i * 2 + dir) * n + kp) * 2 + 0] = c;
                    tw3[(((size_t)i * 2 + dir) * n + kp) * 2 + 1] = c / (double)q;
                }
            const double c = centred(ctx->ninv[i], q);
            tw3[(size_t)ctx->T * 4 * n + 2 * i] = c;
            tw3[(size_t)ctx->T * 4 * n + 2 * i + 1] = c / (double)q;
        }
        e = cudaMalloc(&ctx->d_tw3, tw3.size() * 8);
        if (e == cudaSuccess) e = cudaMemcpy(ctx->d_tw3, tw3.data(), tw3.size() * 8, cudaMemcpyHostToDevice);
        // compact copy (w only) for the narrow-limb block passes: [T][fwd, inv][n] doubles, same positions
        std::vector<double> tw1((size_t)ctx->T * 2 * n);
        for (size_t i = 0; i < tw1.size(); i++) tw1[i] = tw3[2 * i];
        if (e == cudaSuccess) e = cudaMalloc(&ctx->d_tw1, tw1.size() * 8);
        if (e == cudaSuccess) e = cudaMemcpy(ctx->d_tw1, tw1.data(), tw1.size() * 8, cudaMemcpyHostToDevice);
    }
    if (e != cudaSuccess) {
        ensi_ctx_destroy(ctx);
        return ENSI_ECUDA;
    }
    *out = ctx;
    return ENSI_OK;
}

void ensi_ctx_destroy(ensi_ctx* ctx) {
    if (!ctx) return;
    DeviceGuard g(ctx->device);
    cudaDeviceSynchronize();
    cudaFree(ctx->d_tw);
    cudaFree(ctx->d_tw2);
    cudaFree(ctx->d_tw3);
    cudaFree(ctx->d_tw1);
    cudaFree(ctx->d_sk);
    if (ctx->keys_owned) cudaFree(ctx->d_keys);
    if (ctx->relin_owned) cudaFree(ctx->d_relin);
    cudaFree(ctx->cc_buf);
    for (auto& c : ctx->conv) {
        cudaFree(c.d_modup);
        cudaFree(c.d_moddown);
        cudaFree(c.d_moddown2);
        cudaFree(c.d_moddown_fp);
        cudaFree(c.d_modup_fp);
    }
    cudaFree(ctx->scratch);
    cudaFree(ctx->host_stage);
    cudaFree(ctx->lb_buf);
    if (ctx->st_h2d) {
        cudaStreamDestroy(ctx->st_h2d);
        cudaStreamDestroy(ctx->st_d2h);
        for (int b = 0; b < 2; b++) {
            cudaEventDestroy(ctx->ev_h2d[b]);
            cudaEventDestroy(ctx->ev_comp[b]);
            cudaEventDestroy(ctx->ev_d2h[b]);
        }
        cudaEventDestroy(ctx->ev_start);
    }
    if (ctx->st_ks[0]) {
        for (int i = 0; i < 2; i++) {
            cudaStreamDestroy(ctx->st_ks[i]);
            cudaEventDestroy(ctx->ev_ks_done[i]);
        }
        cudaEventDestroy(ctx->ev_ks_fork);
    }
    delete ctx;
}

int ensi_ctx_moduli(const ensi_ctx* ctx, uint64_t* moduli_out, uint64_t* psi_out) {
    if (!ctx) return ENSI_EINVAL;
    for (uint32_t i = 0; i < ctx->T; i++) {
        if (moduli_out) moduli_out[i] = ctx->mod[i];
        if (psi_out) psi_out[i] = ctx->psi[i];
    }
    return ENSI_OK;
}

int ensi_load_keys(ensi_ctx* ctx, const ensi_keys* keys) {
    if (!ctx || !keys) return ENSI_EINVAL;
    DeviceGuard g(ctx->device);
    const size_t n = ctx->n;
    cudaDeviceSynchronize();
    if (keys->sk_ntt) {
        for (size_t i = 0; i < (size_t)ctx->T * n; i++)
            if (keys->sk_ntt[i] >= ctx->mod[i / n]) return set_err(ctx, ENSI_EINVAL, "sk word not canonical");
        if (!ctx->d_sk) {
            cudaError_t e = cudaMalloc(&ctx->d_sk, (size_t)ctx->T * n * 8);
            if (e != cudaSuccess) return cuda_err(ctx, e, "sk malloc");
        }
        cudaError_t e = cudaMemcpy(ctx->d_sk, keys->sk_ntt, (size_t)ctx->T * n * 8, cudaMemcpyHostToDevice);
        if (e != cudaSuccess) return cuda_err(ctx, e, "sk copy");
    }
    if (keys->n_rot > 0) {
        if (!keys->galois || !keys->rot_keys) return set_err(ctx, ENSI_EINVAL, "NULL galois or rot_keys");
        if (ctx->A == 0) return set_err(ctx, ENSI_EINVAL, "rotation keys need num_p > 0");
        for (uint32_t r = 0; r < keys->n_rot; r++)
            if ((keys->galois[r] & 1) == 0 || keys->galois[r] >= 2ull * n)
                return set_err(ctx, ENSI_EINVAL, "galois element must be odd and < 2N'");
        if (ctx->keys_owned) cudaFree(ctx->d_keys);
        ctx->d_keys = nullptr;
        ctx->keys_owned = false;
        const size_t bytes = (size_t)keys->n_rot * ctx->dnum * 2 * ctx->T * n * 8;
        if (keys->rot_keys_mem == ENSI_MEM_DEVICE) {
            ctx->d_keys = const_cast<uint64_t*>(keys->rot_keys);
        } else {
            cudaError_t e = cudaMalloc(&ctx->d_keys, bytes);
            if (e != cudaSuccess) {
                cudaGetLastError();
                return set_err(ctx, ENSI_ENOMEM, "rotation key allocation failed");
            }
            ctx->keys_owned = true;
            e = cudaMemcpy(ctx->d_keys, keys->rot_keys, bytes, cudaMemcpyHostToDevice);
            if (e != cudaSuccess) return cuda_err(ctx, e, "rotation key copy");
        }
        ctx->galois.assign(keys->galois, keys->galois + keys->n_rot);
    }
    return ENSI_OK;
}

int ensi_weights_pack(ensi_ctx* ctx, const int8_t* W, uint32_t d, uint32_t m, uint32_t ldw, ensi_weights** out) {
    if (!ctx || !W || !out) return ctx ? set_err(ctx, ENSI_EINVAL, "NULL argument") : ENSI_EINVAL;
    *out = nullptr;
    if (d == 0 || m == 0) return set_err(ctx, ENSI_EDIM, "d and m must be positive");
    if (ldw < m) return set_err(ctx, ENSI_EDIM, "ldw < m");
    DeviceGuard g(ctx->device);
    ensi_weights* w = new (std::nothrow) ensi_weights();
    if (!w) return ENSI_ENOMEM;
    w->ctx = ctx;
    w->d = d;
    w->m = m;
    w->mw = 2 * ((m + 63) / 64);
    std::vector<uint32_t> pl;
    int rc = pack_planes(ctx, W, d, m, ldw, w->mw, pl, &w->nnz);
    if (rc) {
        delete w;
        return rc;
    }
    w->host.resize((size_t)d * m);
    for (uint32_t j = 0; j < d; j++) std::memcpy(&w->host[(size_t)j * m], W + (size_t)j * ldw, m);
    cudaError_t e = cudaMalloc(&w->d_planes, pl.size() * 4);
    if (e == cudaSuccess) e = cudaMemcpy(w->d_planes, pl.data(), pl.size() * 4, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        ensi_weights_destroy(w);
        return cuda_err(ctx, e, "weights upload");
    }
    *out = w;
    return ENSI_OK;
}

void ensi_weights_destroy(ensi_weights* w) {
    if (!w) return;
    DeviceGuard g(w->ctx->device);
    cudaDeviceSynchronize();
    cudaFree(w->d_planes);
    for (auto& kv : w->packs_b)
        for (auto* sw : kv.second) ensi_weights_destroy(sw);
    cudaFree(w->d_wt8);
    delete w;
}

int ensi_pcmm_ternary_packed(ensi_ctx* ctx, const ensi_ct_view* x, const ensi_weights* wc, ensi_ct_view* y,
                             const ensi_pcmm_opts* opts, void* stream) {
    ensi::NvtxRange nvtx_("ensi.pcmm");
    if (!ctx) return ENSI_EINVAL;
    if (!wc) return set_err(ctx, ENSI_EINVAL, "NULL weights");
    ensi_weights* w = const_cast<ensi_weights*>(wc);
    if (w->ctx != ctx) return set_err(ctx, ENSI_EINVAL, "weights belong to another context");
    int rc = check_view(ctx, x, "x");
    if (rc) return rc;
    rc = check_view(ctx, y, "y");
    if (rc) return rc;
    ensi_pcmm_opts o{};
    if (opts) o = *opts;
    const uint32_t d = w->d, m = w->m, level = x->level, n = ctx->n;
    const uint32_t out_level = o.rescale_out ? level - 1 : level;
    // ---- every check happens before any allocation or enqueue
    if (o.rescale_out && level < 2) return set_err(ctx, ENSI_ELEVEL, "rescale_out needs level >= 2");
    if (y->level != out_level) return set_err(ctx, ENSI_ELEVEL, "y.level must be x.level (-1 with rescale_out)");
    if (y->count != m) return set_err(ctx, ENSI_EDIM, "y.count != m");
    if (overlaps(x, y, n)) return set_err(ctx, ENSI_EINVAL, "y aliases x");
    if (o.layout > 1) return set_err(ctx, ENSI_EINVAL, "layout must be 0 (A) or 1 (B)");
    if (o.moddown_lazy > 1 || (o.moddown_lazy && o.layout != 1))
        return set_err(ctx, ENSI_EINVAL, "moddown_lazy must be 0, or 1 with Layout B");
    bool tc = false;
    rc = select_kernel(ctx, o.kernel, level, d, &tc);
    if (rc) return rc;
    LayoutBPlan p{};
    const std::vector<ensi_weights*>* subs = nullptr;
    if (o.layout == 0) {
        if (x->count != d) return set_err(ctx, ENSI_EDIM, "Layout A: x.count must equal d");
    } else {
        rc = plan_b(ctx, d, m, o.block_s, o.baby, &p);
        if (rc) return rc;
        if (x->count != p.n_in) return set_err(ctx, ENSI_EDIM, "Layout B: x.count must be ceil(d/k)");
        if (ctx->A == 0 && p.rotations > 0)
            return set_err(ctx, ENSI_ENOKEY, "context has no special primes (num_p == 0): no key switching");
        for (uint32_t b = 1; b < p.B; b++)
            if (!find_key(ctx, galois_of_rotation(ctx->log_n, (int64_t)o.block_s * b)))
                return set_err(ctx, ENSI_ENOKEY, "missing baby-step key for rotation " + std::to_string(o.block_s * b));
        for (uint32_t gm = 1; gm < p.G; gm++)
            if (!find_key(ctx, galois_of_rotation(ctx->log_n, (int64_t)o.block_s * p.B * gm)))
                return set_err(ctx, ENSI_ENOKEY, "missing giant-step key for rotation " +
                                                     std::to_string(o.block_s * p.B * gm));
        rc = weights_b(ctx, w, p.k, p.B, p.n_in, &subs);
        if (rc) return rc;
    }
    cudaStream_t st = (cudaStream_t)stream;
    DeviceGuard g(ctx->device);
    const size_t ctw = (size_t)2 * level * n;
    // output of the accumulate goes to y directly unless a rescale epilogue follows (then into a stream-ordered
    // temporary that every exit path below returns)
    uint64_t* acc_out = y->data;
    struct StreamBuf {
        uint64_t* p = nullptr;
        cudaStream_t st = nullptr;
        ~StreamBuf() {
            if (p) cudaFreeAsync(p, st);
        }
    } owned;
    if (o.rescale_out) {
        owned.st = st;
        cudaError_t e = cudaMallocAsync((void**)&owned.p, (size_t)m * ctw * 8, st);
        if (e != cudaSuccess) {
            owned.p = nullptr;
            cudaGetLastError();
            return set_err(ctx, ENSI_ENOMEM, "pcmm rescale temporary");
        }
        acc_out = owned.p;
    }
    if (o.layout == 0) {
        rc = tc ? accum_ternary_tc(ctx, x->data, d, w, acc_out, level, st, 0, 0, tc_variant(o.kernel))
                : accum_ternary(ctx, x->data, d, w->d_planes, w->mw, m, acc_out, level, st);
    } else {
        rc = layout_b_run(ctx, x, w, *subs, p, o, tc, acc_out, st);
    }
    if (!rc && o.rescale_out) {
        rc = ensi::rescale(ctx, acc_out, m, level, y->data, st);
        if (!rc) y->log2_scale = x->log2_scale - std::log2((double)ctx->mod[level - 1]);
    } else if (!rc) {
        y->log2_scale = x->log2_scale;
    }
    if (!rc) {
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) rc = cuda_err(ctx, e, "pcmm");
    }
    return rc;
}

int ensi_pcmm_ternary(ensi_ctx* ctx, const ensi_ct_view* x, const int8_t* W, uint32_t d, uint32_t m, uint32_t ldw,
                      ensi_ct_view* y, const ensi_pcmm_opts* opts, void* stream) {
    ensi_weights* w = nullptr;
    int rc = ensi_weights_pack(ctx, W, d, m, ldw, &w);
    if (rc) return rc;
    rc = ensi_pcmm_ternary_packed(ctx, x, w, y, opts, stream);
    if (!rc) {
        cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
        if (e != cudaSuccess) rc = cuda_err(ctx, e, "pcmm sync");
    }
    ensi_weights_destroy(w);
    return rc;
}

// Wire format: limb r of a polynomial is N' words of w_r = ceil(bitlen(q_r) / 8) bytes,
// little-endian; a ciphertext is [poly 0: limb 0 .. level-1][poly 1: ...].
static uint32_t wire_width(const ensi_ctx* ctx, uint32_t limb) {
    uint32_t b = 0;
    while (b < 64 && (ctx->mod[limb] >> b)) b++;
    return (b + 7) / 8;
}
static size_t wire_poly_bytes(const ensi_ctx* ctx, uint32_t level) {
    size_t s = 0;
    for (uint32_t r = 0; r < level; r++) s += (size_t)ctx->n * wire_width(ctx, r);
    return s;
}

uint64_t ensi_wire_bytes(const ensi_ctx* ctx, uint32_t level) {
    if (!ctx || level < 1 || level > ctx->L) return 0;
    return 2 * wire_poly_bytes(ctx, level);
}

// one (poly, limb) slice of every input (and output) ciphertext moves per pipeline step: host -> device (wire
// bytes unpacked on the device when wire), accumulate, device -> host (packed on the device when wire)
static int pcmm_host_impl(ensi_ctx* ctx, const void* x_host, uint32_t level, const ensi_weights* wc, void* y_host,
                          uint32_t kernel, void* stream, bool wire) {
    if (!ctx) return ENSI_EINVAL;
    if (!x_host || !y_host || !wc) return set_err(ctx, ENSI_EINVAL, "NULL argument");
    ensi_weights* w = const_cast<ensi_weights*>(wc);
    if (w->ctx != ctx) return set_err(ctx, ENSI_EINVAL, "weights belong to another context");
    if (level < 1 || level > ctx->L) return set_err(ctx, ENSI_ELEVEL, "level out of range");
    DeviceGuard g(ctx->device);
    const uint32_t d = w->d, m = w->m, n = ctx->n, slices = 2 * level;
    bool tc = false;
    int rc = select_kernel(ctx, kernel, level, d, &tc);
    if (rc) return rc;
    // wire slices go straight through the compact kernel where it applies (default or tcgen05 pairs requested)
    const bool compact = wire && tc && (kernel == 0 || kernel == 2) && tcc_supported(ctx, level);
    const size_t ctb = wire ? 2 * wire_poly_bytes(ctx, level) : (size_t)2 * level * n * 8;
    const size_t stage_words = (size_t)(d + m) * n;          // one slice of every input and output
    // per buffer: the u64 slice stage, plus (wire) the same slice in wire bytes (<= 8 bytes per word)
    const size_t buf_words = wire ? 2 * stage_words : stage_words;
    if (!ctx->host_stage || ctx->host_stage_words < 2 * buf_words) {
        if (ctx->host_stage) {
            cudaDeviceSynchronize();
            cudaFree(ctx->host_stage);
        }
        ctx->host_stage = nullptr;
        cudaError_t e = cudaMalloc(&ctx->host_stage, 2 * buf_words * 8);
        if (e != cudaSuccess) {
            cudaGetLastError();
            ctx->host_stage_words = 0;
            return set_err(ctx, ENSI_ENOMEM, "staging allocation failed");
        }
        ctx->host_stage_words = 2 * buf_words;
    }
    if (!ctx->st_h2d) {
        cudaStreamCreateWithFlags(&ctx->st_h2d, cudaStreamNonBlocking);
        cudaStreamCreateWithFlags(&ctx->st_d2h, cudaStreamNonBlocking);
        for (int b = 0; b < 2; b++) {
            cudaEventCreateWithFlags(&ctx->ev_h2d[b], cudaEventDisableTiming);
            cudaEventCreateWithFlags(&ctx->ev_comp[b], cudaEventDisableTiming);
            cudaEventCreateWithFlags(&ctx->ev_d2h[b], cudaEventDisableTiming);
        }
        cudaEventCreateWithFlags(&ctx->ev_start, cudaEventDisableTiming);
    }
    cudaStream_t st = (cudaStream_t)stream;
    const uint8_t* xh = (const uint8_t*)x_host;
    uint8_t* yh = (uint8_t*)y_host;
    // start: the copy streams wait for everything already queued on the caller's stream
    cudaEventRecord(ctx->ev_start, st);
    cudaStreamWaitEvent(ctx->st_h2d, ctx->ev_start, 0);
    cudaStreamWaitEvent(ctx->st_d2h, ctx->ev_start, 0);
    for (uint32_t s = 0; s < slices && !rc; s++) {
        const int b = s & 1;
        uint64_t* xs = ctx->host_stage + (size_t)b * buf_words;
        uint64_t* ys = xs + (size_t)d * n;
        uint8_t* xw = (uint8_t*)(xs + stage_words);                        // wire stage (wire only)
        uint8_t* yw = xw + (size_t)d * n * 8;
        const uint32_t poly = s / level, limb = s % level;
        const uint32_t wb = wire ? wire_width(ctx, limb) : 8;
        const size_t rowb = (size_t)n * wb;
        // byte offset of this slice inside a ciphertext
        size_t off = 0;
        if (wire) {
            off = (size_t)poly * wire_poly_bytes(ctx, level);
            for (uint32_t r = 0; r < limb; r++) off += (size_t)n * wire_width(ctx, r);
        } else {
            off = ((size_t)poly * level + limb) * n * 8;
        }
        if (s >= 2) cudaStreamWaitEvent(ctx->st_h2d, ctx->ev_comp[b], 0);   // x stage b free again
        cudaMemcpy2DAsync(wire ? (void*)xw : (void*)xs, rowb, xh + off, ctb, rowb, d, cudaMemcpyHostToDevice,
                          ctx->st_h2d);
        cudaEventRecord(ctx->ev_h2d[b], ctx->st_h2d);
        cudaStreamWaitEvent(st, ctx->ev_h2d[b], 0);
        if (s >= 2) cudaStreamWaitEvent(st, ctx->ev_d2h[b], 0);             // y stage b drained
        if (compact) {
            // the wire slice is a compact slice: the compact tensor-core kernel reads and writes it directly
            rc = accum_ternary_tcc(ctx, xw, d, w, yw, level, st, (int)limb);
        } else {
            if (wire) rc = wire_unpack(ctx, xw, xs, (size_t)d * n, wb, st);
            if (!rc)
                rc = tc ? accum_ternary_tc(ctx, xs, d, w, ys, level, st, n, limb, tc_variant(kernel))
                        : accum_ternary(ctx, xs, d, w->d_planes, w->mw, m, ys, level, st, n, limb);
            if (!rc && wire) rc = wire_pack(ctx, ys, yw, (size_t)m * n, wb, st);
        }
        cudaEventRecord(ctx->ev_comp[b], st);
        cudaStreamWaitEvent(ctx->st_d2h, ctx->ev_comp[b], 0);
        cudaMemcpy2DAsync(yh + off, ctb, wire ? (const void*)yw : (const void*)ys, rowb, rowb, m,
                          cudaMemcpyDeviceToHost, ctx->st_d2h);
        cudaEventRecord(ctx->ev_d2h[b], ctx->st_d2h);
    }
    // the caller's stream completes only after the last device->host copy
    cudaStreamWaitEvent(st, ctx->ev_d2h[(slices - 1) & 1], 0);
    if (slices >= 2) cudaStreamWaitEvent(st, ctx->ev_d2h[(slices - 2) & 1], 0);
    if (!rc) {
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) rc = cuda_err(ctx, e, "pcmm_host");
    }
    return rc;
}

int ensi_pcmm_ternary_host(ensi_ctx* ctx, const uint64_t* x_host, uint32_t level, double log2_scale,
                           const ensi_weights* wc, uint64_t* y_host, uint32_t kernel, void* stream) {
    ensi::NvtxRange nvtx_("ensi.pcmm_host");
    (void)log2_scale;
    return pcmm_host_impl(ctx, x_host, level, wc, y_host, kernel, stream, false);
}

int ensi_pcmm_ternary_host_wire(ensi_ctx* ctx, const uint8_t* x_wire, uint32_t level, double log2_scale,
                                const ensi_weights* wc, uint8_t* y_wire, uint32_t kernel, void* stream) {
    ensi::NvtxRange nvtx_("ensi.pcmm_host_wire");
    (void)log2_scale;
    return pcmm_host_impl(ctx, x_wire, level, wc, y_wire, kernel, stream, true);
}

namespace {
// shared validation of the compact-layout accumulate calls (plain and fused gather)
int check_compact(ensi_ctx* ctx, const ensi_compact_view* x, const ensi_weights* wc, const ensi_pcmm_opts* opts) {
    if (!wc) return set_err(ctx, ENSI_EINVAL, "NULL weights");
    if (wc->ctx != ctx) return set_err(ctx, ENSI_EINVAL, "weights belong to another context");
    if (!x || !x->data) return set_err(ctx, ENSI_EINVAL, "NULL view or data");
    if (x->level < 1 || x->level > ctx->L) return set_err(ctx, ENSI_ELEVEL, "x.level outside [1, num_q]");
    ensi_pcmm_opts o{};
    if (opts) o = *opts;
    if (o.layout != 0) return set_err(ctx, ENSI_EINVAL, "compact ciphertexts: Layout A only");
    if (o.rescale_out) return set_err(ctx, ENSI_EINVAL, "compact ciphertexts: no rescale epilogue");
    if (o.moddown_lazy) return set_err(ctx, ENSI_EINVAL, "moddown_lazy: Layout B only");
    if (o.kernel != 0 && o.kernel != 2) return set_err(ctx, ENSI_EINVAL, "compact ciphertexts: kernel must be 0 or 2");
    if (o.cluster_pairs > 8) return set_err(ctx, ENSI_EINVAL, "cluster_pairs must be 0..8");
    if (x->count != wc->d) return set_err(ctx, ENSI_EDIM, "x.count must equal d");
    if (!tcc_supported(ctx, x->level) || wc->d >= (1u << 22))
        return set_err(ctx, ENSI_EINVAL, "compact tensor-core accumulate unavailable (sm_100a, 5..8-byte words, N' >= 256)");
    return ENSI_OK;
}
}  // namespace

int ensi_pcmm_ternary_compact(ensi_ctx* ctx, const ensi_compact_view* x, const ensi_weights* wc, ensi_compact_view* y,
                              const ensi_pcmm_opts* opts, void* stream) {
    ensi::NvtxRange nvtx_("ensi.pcmm_compact");
    if (!ctx) return ENSI_EINVAL;
    if (!y || !y->data) return set_err(ctx, ENSI_EINVAL, "NULL view or data");
    int rc = check_compact(ctx, x, wc, opts);
    if (rc) return rc;
    ensi_weights* w = const_cast<ensi_weights*>(wc);
    if (y->level != x->level) return set_err(ctx, ENSI_ELEVEL, "y.level must equal x.level");
    if (y->count != w->m) return set_err(ctx, ENSI_EDIM, "y.count != m");
    const uint64_t cb = 2 * wire_poly_bytes(ctx, x->level);
    const uint8_t *x0 = x->data, *x1 = x0 + (size_t)x->count * cb, *y0 = y->data, *y1 = y0 + (size_t)y->count * cb;
    if (x0 < y1 && y0 < x1) return set_err(ctx, ENSI_EINVAL, "y aliases x");
    DeviceGuard g(ctx->device);
    rc = accum_ternary_tcc(ctx, x->data, w->d, w, y->data, x->level, (cudaStream_t)stream, -1,
                           opts ? opts->cluster_pairs : 0);
    if (!rc) y->log2_scale = x->log2_scale;
    return rc;
}

int ensi_pcmm_ternary_compact_gather(ensi_ctx* ctx, const ensi_compact_view* x, const ensi_weights* wc,
                                     uint8_t* const* y_dst, uint32_t n_dst, uint32_t rows_total, uint32_t row0,
                                     const ensi_pcmm_opts* opts, void* stream) {
    ensi::NvtxRange nvtx_("ensi.pcmm_compact_gather");
    if (!ctx) return ENSI_EINVAL;
    int rc = check_compact(ctx, x, wc, opts);
    if (rc) return rc;
    ensi_weights* w = const_cast<ensi_weights*>(wc);
    if (!y_dst || n_dst < 1 || n_dst > 8) return set_err(ctx, ENSI_EINVAL, "y_dst: 1..8 destination buffers");
    if ((uint64_t)row0 + w->m > rows_total) return set_err(ctx, ENSI_EDIM, "row0 + m exceeds rows_total");
    const uint64_t cb = 2 * wire_poly_bytes(ctx, x->level);
    const uint8_t *x0 = x->data, *x1 = x0 + (size_t)x->count * cb;
    uint8_t* dst[8];
    for (uint32_t p = 0; p < n_dst; p++) {
        if (!y_dst[p]) return set_err(ctx, ENSI_EINVAL, "NULL destination buffer");
        const uint8_t *b0 = y_dst[p], *b1 = b0 + (size_t)rows_total * cb;
        if (x0 < b1 && b0 < x1) return set_err(ctx, ENSI_EINVAL, "a destination buffer aliases x");
        dst[p] = y_dst[p] + (size_t)row0 * cb;       // this rank's rows of destination p
    }
    DeviceGuard g(ctx->device);
    return accum_ternary_tcc_dst(ctx, x->data, w->d, w, dst, n_dst, x->level, (cudaStream_t)stream, -1,
                                 opts ? opts->cluster_pairs : 0);
}

typedef CUresult (*PFN_memGetAddressRange)(CUdeviceptr*, size_t*, CUdeviceptr);

int ensi_ipc_get_handle(ensi_ctx* ctx, const void* dev_ptr, ensi_ipc_handle* out) {
    if (!ctx) return ENSI_EINVAL;
    if (!dev_ptr || !out) return set_err(ctx, ENSI_EINVAL, "NULL argument");
    static PFN_memGetAddressRange range = nullptr;
    if (!range) {
        void* fp = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fp, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            range = (PFN_memGetAddressRange)fp;
        if (!range) return set_err(ctx, ENSI_ECUDA, "cuMemGetAddressRange unavailable");
    }
    DeviceGuard g(ctx->device);
    CUdeviceptr base = 0;
    size_t size = 0;
    if (range(&base, &size, (CUdeviceptr)dev_ptr) != CUDA_SUCCESS) return set_err(ctx, ENSI_EINVAL, "not a device allocation");
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, (void*)base);
    if (e != cudaSuccess) return cuda_err(ctx, e, "cudaIpcGetMemHandle");
    static_assert(sizeof(h) <= sizeof(out->handle), "IPC handle size");
    std::memset(out, 0, sizeof(*out));
    std::memcpy(out->handle, &h, sizeof(h));
    out->offset = (uint64_t)((CUdeviceptr)dev_ptr - base);
    return ENSI_OK;
}

int ensi_ipc_open(ensi_ctx* ctx, const ensi_ipc_handle* h, void** dev_ptr) {
    if (!ctx) return ENSI_EINVAL;
    if (!h || !dev_ptr) return set_err(ctx, ENSI_EINVAL, "NULL argument");
    DeviceGuard g(ctx->device);
    cudaIpcMemHandle_t ih;
    std::memcpy(&ih, h->handle, sizeof(ih));
    void* base = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&base, ih, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return cuda_err(ctx, e, "cudaIpcOpenMemHandle");
    *dev_ptr = (uint8_t*)base + h->offset;
    ctx->ipc_bases[*dev_ptr] = base;
    return ENSI_OK;
}

int ensi_ipc_close(ensi_ctx* ctx, void* dev_ptr) {
    if (!ctx) return ENSI_EINVAL;
    auto it = ctx->ipc_bases.find(dev_ptr);
    if (it == ctx->ipc_bases.end()) return set_err(ctx, ENSI_EINVAL, "pointer was not opened with ensi_ipc_open");
    DeviceGuard g(ctx->device);
    cudaError_t e = cudaIpcCloseMemHandle(it->second);
    ctx->ipc_bases.erase(it);
    return e == cudaSuccess ? ENSI_OK : cuda_err(ctx, e, "cudaIpcCloseMemHandle");
}

int ensi_peer_signal(ensi_ctx* ctx, uint32_t* const* flags_dst, uint32_t n_dst, uint32_t slot, uint32_t epoch,
                     void* stream) {
    ensi::NvtxRange nvtx_("ensi.peer_signal");
    if (!ctx) return ENSI_EINVAL;
    if (!flags_dst || n_dst < 1 || n_dst > 8) return set_err(ctx, ENSI_EINVAL, "flags_dst: 1..8 flag arrays");
    PeerFlags pf{};
    pf.n = n_dst;
    for (uint32_t p = 0; p < n_dst; p++) {
        if (!flags_dst[p]) return set_err(ctx, ENSI_EINVAL, "NULL flag array");
        pf.f[p] = flags_dst[p];
    }
    DeviceGuard g(ctx->device);
    k_peer_signal<<<1, 32, 0, (cudaStream_t)stream>>>(pf, slot, epoch);
    ENSI_LAUNCH_CHECK(ctx);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? ENSI_OK : cuda_err(ctx, e, "peer_signal");
}

int ensi_peer_wait(ensi_ctx* ctx, const uint32_t* flags, uint32_t n, uint32_t epoch, void* stream) {
    ensi::NvtxRange nvtx_("ensi.peer_wait");
    if (!ctx) return ENSI_EINVAL;
    if (!flags || n < 1 || n > 32) return set_err(ctx, ENSI_EINVAL, "flags: 1..32 entries");
    DeviceGuard g(ctx->device);
    k_peer_wait<<<1, 32, 0, (cudaStream_t)stream>>>(flags, n, epoch);
    ENSI_LAUNCH_CHECK(ctx);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? ENSI_OK : cuda_err(ctx, e, "peer_wait");
}

int ensi_wire_pack(ensi_ctx* ctx, const ensi_ct_view* x, uint8_t* out, void* stream) {
    if (!ctx) return ENSI_EINVAL;
    int rc = check_view(ctx, x, "x");
    if (rc) return rc;
    if (!out) return set_err(ctx, ENSI_EINVAL, "NULL output");
    DeviceGuard g(ctx->device);
    const uint32_t lv = x->level, n = ctx->n;
    const size_t pb = wire_poly_bytes(ctx, lv);
    // one launch per limb over all (ciphertext, poly) rows
    size_t off = 0;
    for (uint32_t r = 0; r < lv && !rc; r++) {
        const uint32_t wb = wire_width(ctx, r);
        rc = wire_pack_rows(ctx, x->data + (size_t)r * n, (size_t)lv * n, out + off, pb, 2 * x->count, n, wb,
                            (cudaStream_t)stream);
        off += (size_t)n * wb;
    }
    return rc;
}

int ensi_wire_unpack(ensi_ctx* ctx, const uint8_t* in, ensi_ct_view* y, void* stream) {
    if (!ctx) return ENSI_EINVAL;
    int rc = check_view(ctx, y, "y");
    if (rc) return rc;
    if (!in) return set_err(ctx, ENSI_EINVAL, "NULL input");
    DeviceGuard g(ctx->device);
    const uint32_t lv = y->level, n = ctx->n;
    const size_t pb = wire_poly_bytes(ctx, lv);
    size_t off = 0;
    for (uint32_t r = 0; r < lv && !rc; r++) {
        const uint32_t wb = wire_width(ctx, r);
        rc = wire_unpack_rows(ctx, in + off, pb, y->data + (size_t)r * n, (size_t)lv * n, 2 * y->count, n, wb,
                              (cudaStream_t)stream);
        off += (size_t)n * wb;
    }
    return rc;
}

int ensi_ntt(ensi_ctx* ctx, uint64_t* data, uint32_t rows, const uint32_t* limb_of_row, uint32_t period, int inverse,
             void* stream) {
    ensi::NvtxRange nvtx_("ensi.ntt");
    if (!ctx) return ENSI_EINVAL;
    if (!data || !limb_of_row) return set_err(ctx, ENSI_EINVAL, "NULL argument");
    if (period == 0 || period > 2 * ENSI_MAXT) return set_err(ctx, ENSI_EINVAL, "period out of range");
    if (rows > 65535) return set_err(ctx, ENSI_EDIM, "at most 65535 rows per call");
    LimbMap mp = identity_map(1);
    mp.period = period;
    for (uint32_t i = 0; i < period; i++) {
        if (limb_of_row[i] >= ctx->T) return set_err(ctx, ENSI_EINVAL, "limb index out of range");
        mp.limb[i] = (uint8_t)limb_of_row[i];
    }
    DeviceGuard g(ctx->device);
    if (inverse) ntt_inverse(ctx, data, rows, mp, (cudaStream_t)stream);
    else ntt_forward(ctx, data, rows, mp, (cudaStream_t)stream);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? ENSI_OK : cuda_err(ctx, e, "ntt");
}

int ensi_rotate_hoisted(ensi_ctx* ctx, const ensi_ct_view* x, uint32_t n_g, const uint64_t* galois, ensi_ct_view* y,
                        void* stream) {
    ensi::NvtxRange nvtx_("ensi.rotate_hoisted");
    if (!ctx) return ENSI_EINVAL;
    int rc = check_view(ctx, x, "x");
    if (rc) return rc;
    rc = check_view(ctx, y, "y");
    if (rc) return rc;
    if (!galois && n_g) return set_err(ctx, ENSI_EINVAL, "NULL galois");
    if (y->count < n_g) return set_err(ctx, ENSI_EDIM, "y.count < n_g");
    if (y->level != x->level) return set_err(ctx, ENSI_ELEVEL, "y.level != x.level");
    if (overlaps(x, y, ctx->n)) return set_err(ctx, ENSI_EINVAL, "y aliases x");
    DeviceGuard g(ctx->device);
    rc = rotate_hoisted(ctx, x->data, x->level, n_g, galois, y->data, (cudaStream_t)stream);
    if (!rc) y->log2_scale = x->log2_scale;
    return rc;
}

int ensi_rotate_batch(ensi_ctx* ctx, const ensi_ct_view* x, uint32_t n_g, const uint64_t* galois, ensi_ct_view* y,
                      void* stream) {
    ensi::NvtxRange nvtx_("ensi.rotate_batch");
    if (!ctx) return ENSI_EINVAL;
    int rc = check_view(ctx, x, "x");
    if (rc) return rc;
    rc = check_view(ctx, y, "y");
    if (rc) return rc;
    if (!galois && n_g) return set_err(ctx, ENSI_EINVAL, "NULL galois");
    if ((uint64_t)y->count < (uint64_t)x->count * n_g) return set_err(ctx, ENSI_EDIM, "y.count < x.count * n_g");
    if (y->level != x->level) return set_err(ctx, ENSI_ELEVEL, "y.level != x.level");
    if (overlaps(x, y, ctx->n)) return set_err(ctx, ENSI_EINVAL, "y aliases x");
    if (n_g == 0 || x->count == 0) return ENSI_OK;
    DeviceGuard g(ctx->device);
    const uint64_t ctw = (uint64_t)2 * x->level * ctx->n;
    // inputs in chunks of at most 96 (bounds the ModUp and key-switch scratch)
    for (uint32_t c0 = 0; c0 < x->count && !rc; c0 += 96) {
        const uint32_t nc = std::min<uint32_t>(96, x->count - c0);
        rc = rotate_hoisted_multi(ctx, x->data + (uint64_t)c0 * ctw, nc, ctw, x->level, n_g, galois,
                                  y->data + (uint64_t)c0 * n_g * ctw, n_g, (cudaStream_t)stream);
    }
    if (!rc) y->log2_scale = x->log2_scale;
    return rc;
}

int ensi_rescale(ensi_ctx* ctx, const ensi_ct_view* x, ensi_ct_view* y, void* stream) {
    ensi::NvtxRange nvtx_("ensi.rescale");
    if (!ctx) return ENSI_EINVAL;
    int rc = check_view(ctx, x, "x");
    if (rc) return rc;
    rc = check_view(ctx, y, "y");
    if (rc) return rc;
    if (x->level < 2) return set_err(ctx, ENSI_ELEVEL, "rescale needs level >= 2");
    if (y->level != x->level - 1 || y->count != x->count) return set_err(ctx, ENSI_EDIM, "y must be count x (level-1)");
    if (overlaps(x, y, ctx->n)) return set_err(ctx, ENSI_EINVAL, "y aliases x");
    DeviceGuard g(ctx->device);
    rc = ensi::rescale(ctx, x->data, x->count, x->level, y->data, (cudaStream_t)stream);
    if (!rc) y->log2_scale = x->log2_scale - std::log2((double)ctx->mod[x->level - 1]);
    return rc;
}

// ---------------------------------------------------------------------------------------------- CCMM (R18)

int ensi_load_relin_key(ensi_ctx* ctx, const uint64_t* relin_key, uint32_t mem) {
    if (!ctx) return ENSI_EINVAL;
    if (!relin_key) return set_err(ctx, ENSI_EINVAL, "NULL relinearisation key");
    if (ctx->A == 0) return set_err(ctx, ENSI_EINVAL, "relinearisation needs num_p > 0");
    if (mem != ENSI_MEM_HOST && mem != ENSI_MEM_DEVICE) return set_err(ctx, ENSI_EINVAL, "mem must be HOST or DEVICE");
    DeviceGuard g(ctx->device);
    cudaDeviceSynchronize();
    if (ctx->relin_owned) cudaFree(ctx->d_relin);
    ctx->d_relin = nullptr;
    ctx->relin_owned = false;
    if (mem == ENSI_MEM_DEVICE) {
        ctx->d_relin = const_cast<uint64_t*>(relin_key);
        return ENSI_OK;
    }
    const size_t bytes = (size_t)ctx->dnum * 2 * ctx->T * ctx->n * 8;
    cudaError_t e = cudaMalloc(&ctx->d_relin, bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        ctx->d_relin = nullptr;
        return set_err(ctx, ENSI_ENOMEM, "relinearisation key allocation failed");
    }
    ctx->relin_owned = true;
    e = cudaMemcpy(ctx->d_relin, relin_key, bytes, cudaMemcpyHostToDevice);
    return e == cudaSuccess ? ENSI_OK : cuda_err(ctx, e, "relinearisation key copy");
}

int ensi_mul_plain(ensi_ctx* ctx, const ensi_ct_view* x, const uint64_t* pt, double pt_log2_scale, ensi_ct_view* y,
                   void* stream) {
    if (!ctx) return ENSI_EINVAL;
    int rc = check_view(ctx, x, "x");
    if (rc) return rc;
    rc = check_view(ctx, y, "y");
    if (rc) return rc;
    if (!pt) return set_err(ctx, ENSI_EINVAL, "NULL plaintext");
    if (y->count != x->count) return set_err(ctx, ENSI_EDIM, "y.count != x.count");
    if (y->level != x->level) return set_err(ctx, ENSI_ELEVEL, "y.level != x.level");
    if (y->data != x->data && overlaps(x, y, ctx->n)) return set_err(ctx, ENSI_EINVAL, "y partially aliases x");
    DeviceGuard g(ctx->device);
    rc = ensi::mul_plain(ctx, x->data, x->count, x->level, pt, y->data, (cudaStream_t)stream);
    if (!rc) y->log2_scale = x->log2_scale + pt_log2_scale;
    return rc;
}

int ensi_mul_relin(ensi_ctx* ctx, const ensi_ct_view* a, const ensi_ct_view* b, ensi_ct_view* y, void* stream) {
    ensi::NvtxRange nvtx_("ensi.mul_relin");
    if (!ctx) return ENSI_EINVAL;
    int rc = check_view(ctx, a, "a");
    if (!rc) rc = check_view(ctx, b, "b");
    if (!rc) rc = check_view(ctx, y, "y");
    if (rc) return rc;
    if (a->count != b->count || y->count != a->count) return set_err(ctx, ENSI_EDIM, "a, b, y counts differ");
    if (a->level != b->level || y->level != a->level) return set_err(ctx, ENSI_ELEVEL, "a, b, y levels differ");
    if (overlaps(a, y, ctx->n) || overlaps(b, y, ctx->n)) return set_err(ctx, ENSI_EINVAL, "y aliases a or b");
    if (!ctx->d_relin) return set_err(ctx, ENSI_ENOKEY, "no relinearisation key loaded");
    if (a->count == 0) return ENSI_OK;
    DeviceGuard g(ctx->device);
    const uint32_t lv = a->level, n = ctx->n;
    const uint64_t ctw = (uint64_t)2 * lv * n, P = (uint64_t)lv * n;
    const cudaStream_t st = (cudaStream_t)stream;
    const uint32_t chunk = std::min<uint32_t>(a->count, 32);
    rc = ensi::cc_scratch(ctx, (size_t)chunk * 3 * P);
    for (uint32_t c0 = 0; c0 < a->count && !rc; c0 += chunk) {
        const uint32_t nc = std::min<uint32_t>(chunk, a->count - c0);
        for (uint32_t c = 0; c < nc && !rc; c++)
            rc = ensi::tensor_acc(ctx, a->data + (size_t)(c0 + c) * ctw, ctw, lv, b->data + (size_t)(c0 + c) * ctw, 1,
                                  ctx->cc_buf + (size_t)c * 3 * P, lv, true, st);
        if (!rc) rc = ensi::relinearize(ctx, ctx->cc_buf, nc, lv, y->data + (size_t)c0 * ctw, st);
    }
    if (!rc) y->log2_scale = a->log2_scale + b->log2_scale;
    return rc;
}

int ensi_ccmm(ensi_ctx* ctx, const ensi_ct_view* a, const ensi_ct_view* src, const uint64_t* mask_pt, ensi_ct_view* y,
              const ensi_ccmm_opts* opts, void* stream) {
    ensi::NvtxRange nvtx_("ensi.ccmm");
    if (!ctx) return ENSI_EINVAL;
    if (!opts || !mask_pt) return set_err(ctx, ENSI_EINVAL, "NULL opts or mask");
    int rc = check_view(ctx, a, "a");
    if (!rc) rc = check_view(ctx, src, "src");
    if (!rc) rc = check_view(ctx, y, "y");
    if (rc) return rc;
    const uint32_t form = opts->form, s = opts->block_s, d = opts->d, m = opts->m;
    if (form != 1 && form != 2) return set_err(ctx, ENSI_EINVAL, "form must be 1 (A.K^T) or 2 (A.B)");
    if (s < 2 || (s & (s - 1)) || s > ctx->n / 2) return set_err(ctx, ENSI_EDIM, "block_s must be a power of two in [2, N'/2]");
    if (d == 0 || m == 0) return set_err(ctx, ENSI_EDIM, "d and m must be positive");
    if (form == 2 && d > s) return set_err(ctx, ENSI_EDIM, "form 2 needs d <= block_s");
    if (form == 1 && m > s) return set_err(ctx, ENSI_EDIM, "form 1 needs m <= block_s");
    if (a->count != d) return set_err(ctx, ENSI_EDIM, "a.count != d");
    if (src->count != (form == 2 ? m : d)) return set_err(ctx, ENSI_EDIM, "src.count != (form 2 ? m : d)");
    if (opts->col0 >= m) return set_err(ctx, ENSI_EDIM, "col0 >= m");
    const uint32_t cols = opts->cols ? opts->cols : m - opts->col0;
    if (opts->col0 + (uint64_t)cols > m) return set_err(ctx, ENSI_EDIM, "col0 + cols > m");
    if (y->count != cols) return set_err(ctx, ENSI_EDIM, "y.count != cols");
    if (src->level != a->level) return set_err(ctx, ENSI_ELEVEL, "a and src levels differ");
    if (a->level < 3) return set_err(ctx, ENSI_ELEVEL, "CCMM consumes two levels: a.level >= 3 required");
    if (y->level != a->level - 2) return set_err(ctx, ENSI_ELEVEL, "y.level must be a.level - 2");
    if (overlaps(a, y, ctx->n) || overlaps(src, y, ctx->n)) return set_err(ctx, ENSI_EINVAL, "y aliases an input");
    if (ctx->A == 0) return set_err(ctx, ENSI_ENOKEY, "context has no special primes: no key switching");
    if (!ctx->d_relin) return set_err(ctx, ENSI_ENOKEY, "no relinearisation key loaded");
    DeviceGuard g(ctx->device);
    rc = ensi::ccmm(ctx, a->data, src->data, form, s, d, m, a->level, mask_pt, y->data, opts->col0, opts->col0 + cols,
                    (cudaStream_t)stream);
    if (!rc) y->log2_scale = a->log2_scale + src->log2_scale - std::log2((double)ctx->mod[a->level - 2]);
    return rc;
}

int ensi_decrypt_debug(ensi_ctx* ctx, const ensi_ct_view* ct, uint32_t index, uint64_t* coeffs_out, double* slots_out) {
    if (!ctx) return ENSI_EINVAL;
    int rc = check_view(ctx, ct, "ct");
    if (rc) return rc;
    if (index >= ct->count) return set_err(ctx, ENSI_EDIM, "index >= count");
    if (!ctx->d_sk) return set_err(ctx, ENSI_ENOKEY, "no secret key loaded");
    DeviceGuard g(ctx->device);
    const uint32_t n = ctx->n, level = ct->level;
    uint64_t* mu = nullptr;
    cudaError_t e = cudaMalloc(&mu, (size_t)level * n * 8);
    if (e != cudaSuccess) return cuda_err(ctx, e, "decrypt malloc");
    rc = decrypt_mu(ctx, ct->data + (size_t)index * 2 * level * n, level, mu, 0);
    std::vector<uint64_t> h((size_t)level * n);
    if (!rc) {
        e = cudaMemcpy(h.data(), mu, h.size() * 8, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) rc = cuda_err(ctx, e, "decrypt copy");
    }
    cudaFree(mu);
    if (rc) return rc;
    if (coeffs_out) std::memcpy(coeffs_out, h.data(), h.size() * 8);
    if (slots_out) {
        // CRT over limbs {0,1} (or limb 0 alone), centred, then decode z_u = Re sum_j m_j zeta^{5^u j} / Delta
        std::vector<std::complex<double>> a(n);
        const uint64_t q0 = ctx->mod[0];
        const double scale = std::exp2(ct->log2_scale);
        typedef unsigned __int128 u128;
        for (uint32_t j = 0; j < n; j++) {
            double v;
            if (level >= 2) {
                const uint64_t q1 = ctx->mod[1];
                uint64_t r0 = h[j], r1 = h[n + j];
                uint64_t t = mulmod_h((r1 + q1 - r0 % q1) % q1, invmod_h(q0 % q1, q1), q1);
                u128 x = (u128)t * q0 + r0, Q = (u128)q0 * q1;
                v = (x > Q / 2) ? -(double)(Q - x) : (double)x;
            } else {
                uint64_t r0 = h[j];
                v = (r0 > q0 / 2) ? -(double)(q0 - r0) : (double)r0;
            }
            double ang = M_PI * (double)j / (double)n;   // m_j zeta^j
            a[j] = std::complex<double>(v * std::cos(ang), v * std::sin(ang));
        }
        fft_host(a, +1);   // sum_j (m_j zeta^j) e^{2 pi i j t / n}
        uint64_t e5 = 1;
        const uint64_t two_n = 2ull * n;
        for (uint32_t u = 0; u < n / 2; u++) {
            slots_out[u] = a[(e5 - 1) / 2].real() / scale;
            e5 = (e5 * 5) % two_n;
        }
    }
    return ENSI_OK;
}

}  // extern "C"
