// ensi_internal.h -- context and launch helpers shared by the CUDA translation units of libensi.so.
#pragma once
#include <cuda.h>
#include <nvtx3/nvToolsExt.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "../../include/ensi.h"
#include "modarith.cuh"

#define ENSI_MAXT 64

namespace ensi {

// Per-limb modulus data passed by value to kernels (lives in the kernel-parameter constant bank).
struct ModTab {
    uint64_t q[ENSI_MAXT];
    uint64_t mu[ENSI_MAXT];
    uint32_t w[ENSI_MAXT];
    __host__ __device__ Barrett br(uint32_t i) const { return Barrett{q[i], mu[i], w[i]}; }
};

// Row -> limb map for batched polynomial kernels: logical row r uses limb[r % period] and lives at physical
// row (r / grp_rows) * grp_stride + grp_off + r % grp_rows (identity when grp_rows is huge).
struct LimbMap {
    uint32_t period;
    uint32_t grp_rows, grp_stride, grp_off;
    uint8_t limb[ENSI_MAXT * 2];
    __host__ __device__ uint64_t phys(uint32_t r) const {
        return (uint64_t)(r / grp_rows) * grp_stride + grp_off + (r % grp_rows);
    }
};

// ModUp / ModDown basis-conversion constants for one level, resident on the device.
struct ConvTables {
    uint32_t level, beta;
    // modup: per digit t, per source i in D_t: (Q_t/q_i)^{-1} mod q_i (+shoup)  -> [beta][alpha][2]
    // per digit t, per ext limb e, per source a: [Q_t/q_i]_{r_e} (+shoup)      -> [beta][E][alpha][2]
    uint64_t* d_modup = nullptr;
    // moddown: per p_k: (P/p_k)^{-1} mod p_k (+shoup) [alpha][2]; per q_i per k: [P/p_k]_{q_i} (+shoup)
    // [level][alpha][2]; per q_i: P^{-1} mod q_i (+shoup) [level][2]
    uint64_t* d_moddown = nullptr;
    // moddown v2: per (q_i, p_k): [P/p_k]_{q_i}, Shoup companion, q_i - [p_k P/p_k]_{q_i}  -> [level][alpha][3]
    uint64_t* d_moddown2 = nullptr;
    // moddown for the FP64 conversion (moduli < 2^50): (P/p_k)^-1 mod p_k centred and RN(./p_k) [alpha][2], then
    // [P/p_k]_{q_i} centred and RN(./q_i) [level][alpha][2]
    double* d_moddown_fp = nullptr;
    std::vector<double> h_moddown_fp;     // host copy (kernel-parameter constants)
    // modup for the FP64 conversion: same indexing as d_modup, (centred constant, RN(constant / modulus)) pairs
    double* d_modup_fp = nullptr;
    std::vector<double> h_modup_fp;       // host copy (kernel-parameter constants)
    std::vector<uint64_t> h_pinv;         // [level]: P^{-1} mod q_i (canonical), for the FP64 final combine
};

}  // namespace ensi

struct ensi_weights {
    ensi_ctx* ctx = nullptr;
    uint32_t d = 0, m = 0, mw = 0;        // mw = 32-bit words per sign-plane row (multiple of 2)
    std::vector<int8_t> host;             // dense d x m copy (row-major, ldw = m) for Layout-B re-packing
    uint32_t* d_planes = nullptr;         // [d][2][mw]: pos bits then neg bits (bit i%32 of word i/32)
    uint64_t nnz = 0;
    // Layout B: per (k, B), one re-ordered weight object per giant step (rows c*B + b = W[c*k + gam*B + b])
    std::map<std::pair<uint32_t, uint32_t>, std::vector<ensi_weights*>> packs_b;
    // byte-sliced tensor-core operand (W^T as int8 [m_pad][d_pad], K-major), built lazily
    int8_t* d_wt8 = nullptr;
    uint32_t wt_mpad = 0, wt_dpad = 0;
};

struct ensi_ctx {
    int device = 0;
    uint32_t log_n = 0, n = 0, L = 0, A = 0, dnum = 0, T = 0;
    double log2_scale = 40.0;
    uint64_t mod[ENSI_MAXT] = {};
    uint64_t psi[ENSI_MAXT] = {};
    ensi::ModTab tab{};
    // twiddles: [T][4][n] = psi_rev, psi_rev_shoup, ipsi_rev, ipsi_rev_shoup
    uint64_t* d_tw = nullptr;
    uint64_t* d_tw2 = nullptr;            // interleaved [T][fwd, inv][n][w, w'] for the v2 NTT passes
    // FP64 NTT (ntt_fp.cuh, all moduli < 2^50): [T][fwd, inv][n] of (w centred, RN(w/q)), then [T] of
    // (n^-1 centred, RN(n^-1/q)), as double2
    double* d_tw3 = nullptr;
    double* d_tw1 = nullptr;              // compact [T][fwd, inv][n] w-only copy (narrow-limb block passes)
    bool ntt_fp_ok = false;
    uint64_t ninv[ENSI_MAXT] = {}, ninv_sh[ENSI_MAXT] = {};
    // keys
    uint64_t* d_sk = nullptr;             // [T][n]
    std::vector<uint64_t> galois;
    uint64_t* d_keys = nullptr;
    bool keys_owned = false;
    uint64_t* d_relin = nullptr;          // relinearisation key [dnum][2][T][n] (CCMM)
    bool relin_owned = false;
    uint64_t* cc_buf = nullptr;           // CCMM scratch
    size_t cc_words = 0;
    // conversion tables per level (1..L)
    std::vector<ensi::ConvTables> conv;
    // scratch (grown on demand)
    void* scratch = nullptr;
    size_t scratch_bytes = 0;
    // Layout-B scratch (rotated inputs + giant-step partials)
    uint64_t* lb_buf = nullptr;
    size_t lb_words = 0;
    // host-staged pipeline (ensi_pcmm_ternary_host)
    uint64_t* host_stage = nullptr;
    size_t host_stage_words = 0;
    cudaStream_t st_h2d = nullptr, st_d2h = nullptr;
    cudaEvent_t ev_h2d[2] = {}, ev_comp[2] = {}, ev_d2h[2] = {}, ev_start = nullptr;
    // key switching: two internal streams for alternating rotation batches
    cudaStream_t st_ks[2] = {};
    cudaEvent_t ev_ks_done[2] = {}, ev_ks_fork = nullptr;
    std::map<void*, void*> ipc_bases;        // ensi_ipc_open: returned pointer -> opened allocation base
    std::string err;
    uint64_t launches = 0;
    uint32_t tcc_cpairs = 0, tcc_nclust = 0;   // last compact accumulate launch shape
};

namespace ensi {

// NVTX phase ranges (per-phase tracing).  Header-only NVTX v3: free when no tool is attached; under
// nsys / ncu --nvtx the host-side enqueue phases of every call are labelled (ensi.*, ks.*, layoutB.*, ccmm.*).
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

// error helpers (api.cu)
int set_err(ensi_ctx* ctx, int code, const std::string& msg);
int cuda_err(ensi_ctx* ctx, cudaError_t e, const char* where);

// host math (host_math.cpp)
bool is_prime_u64(uint64_t n);
uint64_t powmod_h(uint64_t a, uint64_t e, uint64_t q);
uint64_t mulmod_h(uint64_t a, uint64_t b, uint64_t q);
uint64_t invmod_h(uint64_t a, uint64_t q);
uint64_t shoup_h(uint64_t w, uint64_t q);
Barrett barrett_h(uint64_t q);
void gen_primes(uint32_t log_n, uint32_t L, uint32_t alpha, uint64_t* q, uint64_t* p);
uint64_t min_root(uint64_t q, uint32_t log_n);
uint64_t galois_of_rotation(uint32_t log_n, int64_t r);

// scratch
int ensure_scratch(ensi_ctx* ctx, size_t bytes);

// NTT (ntt.cu): in-place on rows [rows][n], row r modulus = map.limb[r % map.period]
void ntt_forward(ensi_ctx* ctx, uint64_t* data, uint32_t rows, const LimbMap& map, cudaStream_t st);
// out-of-place INTT: rows of src (smap.phys) -> dst (dmap); false when the FP64/TMA path is unavailable (nothing done)
bool ntt_inverse_from(ensi_ctx* ctx, const uint64_t* src, const LimbMap& smap, uint64_t* dst, uint32_t rows,
                      const LimbMap& dmap, cudaStream_t st);
// tensor map of a row buffer for the FP64 NTT's TMA block passes (false: TMA unavailable or disabled)
bool ntt_row_tmap(const ensi_ctx* ctx, uint64_t* data, uint32_t rows, const LimbMap& map, CUtensorMap* tm);
void ntt_inverse(ensi_ctx* ctx, uint64_t* data, uint32_t rows, const LimbMap& map, cudaStream_t st);

// accumulate (accum.cu)
// x: d "ciphertexts" of ctw words each (default ctw = 2*level*N'); word w of a ct lives in limb
// (limb0 + w / N') % level.  A staged chunk holding one limb r of every ct passes ctw = N', limb0 = r.
int accum_ternary(ensi_ctx* ctx, const uint64_t* x, uint32_t d, const uint32_t* planes, uint32_t mw, uint32_t m,
                  uint64_t* y, uint32_t level, cudaStream_t st, uint64_t ctw = 0, uint32_t limb0 = 0);
uint32_t accum_rows_between_reductions(const ensi_ctx* ctx, uint32_t level);
// tensor-core variants: pairs with cluster multicast (default when 2*ceil(m/256) <= 8), pairs without
// multicast, single CTA (cta_group::1)
enum { TC_AUTO = 0, TC_PAIR_MC = 1, TC_PAIR = 2, TC_ONE_CTA = 3 };
int accum_ternary_tc(ensi_ctx* ctx, const uint64_t* x, uint32_t d, ensi_weights* w, uint64_t* y, uint32_t level,
                     cudaStream_t st, uint64_t ctw = 0, uint32_t limb0 = 0, int variant = TC_AUTO);
bool tc_supported(const ensi_ctx* ctx, uint32_t level);
// compact word layout (accum_tcc.cu): w_r = ceil(bitlen(q_r)/8) bytes per word of limb r
uint32_t compact_word_bytes(const ensi_ctx* ctx, uint32_t limb);
bool tcc_supported(const ensi_ctx* ctx, uint32_t level);
// x: d compact ciphertexts (slice_limb < 0) or d copies of one staged (poly, limb) slice of limb slice_limb
struct PeerFlags {
    uint32_t* f[8];
    uint32_t n;
};
__global__ void k_peer_signal(PeerFlags pf, uint32_t slot, uint32_t epoch);
__global__ void k_peer_wait(const uint32_t* flags, uint32_t n, uint32_t epoch);
// launch shape of the tensor-core pair kernels (accum_tcc.cu): c pairs per multicast cluster, K clusters
int tc_plan_clusters(ensi_ctx* ctx, uint32_t pgroups, uint32_t ntiles, const void* kmc, const void* kpl, size_t smem,
                     uint32_t threads, uint32_t force, uint32_t* cpairs, uint32_t* nclust);
int accum_ternary_tcc_dst(ensi_ctx* ctx, const uint8_t* x, uint32_t d, ensi_weights* w, uint8_t* const* y_dst,
                          uint32_t n_dst, uint32_t level, cudaStream_t st, int slice_limb = -1,
                          uint32_t cluster_pairs = 0);
int accum_ternary_tcc(ensi_ctx* ctx, const uint8_t* x, uint32_t d, ensi_weights* w, uint8_t* y, uint32_t level,
                      cudaStream_t st, int slice_limb = -1, uint32_t cluster_pairs = 0);

// key switching (keyswitch.cu)
int conv_tables(ensi_ctx* ctx, uint32_t level, ConvTables** out);
int rotate_hoisted(ensi_ctx* ctx, const uint64_t* ct, uint32_t level, uint32_t n_g, const uint64_t* galois,
                   uint64_t* out, cudaStream_t st);
// Key-switching core options beyond plain rotation (CCMM, R18).
struct KsOpts {
    const uint64_t* key_base = nullptr;  // switching keys [.][dnum][2][T][N'] used instead of ctx->d_keys
    bool switch_identity = false;        // g == 1 is key-switched with key_base[0] (relinearisation), not copied
    uint64_t c1_off = 0;                 // words from a ciphertext to the polynomial that is key-switched (0: level N')
    uint32_t add_mask = 0;               // bit j: output poly j += an unpermuted polynomial of the input ciphertext
    uint64_t add1_off = 0;               // words from a ciphertext to the polynomial added to output poly 1 (0: level N')
    const uint64_t* add_src = nullptr;   // non-NULL: the added polynomials come from add_src + c * add_stride (input c)
    uint64_t add_stride = 0;             //   instead of the input ciphertext itself (may alias out exactly)
    uint64_t* scratch = nullptr;         // internal: caller-provided scratch region (no ensure_scratch, no splitting)
    uint64_t* lazy_acc = nullptr;        // R19: [n_ct][2][level+A][N'] -- accumulate the KIP output here (no ModDown)
    bool lazy_init = false;              //   and add (sigma_g(c0), 0) to out; lazy_init: overwrite instead of add
};
int lazy_moddown(ensi_ctx* ctx, uint64_t* la, uint32_t n_ct, uint32_t level, uint64_t* out, cudaStream_t st);
int rotate_hoisted_multi(ensi_ctx* ctx, const uint64_t* ct, uint32_t n_ct, uint64_t in_stride, uint32_t level,
                         uint32_t n_g, const uint64_t* galois, uint64_t* out, uint32_t out_c_stride, cudaStream_t st,
                         const KsOpts* opts = nullptr);
const uint64_t* find_key(const ensi_ctx* ctx, uint64_t g);

// CCMM (ccmm.cu, R18)
int mul_plain(ensi_ctx* ctx, const uint64_t* x, uint32_t count, uint32_t level, const uint64_t* pt, uint64_t* out,
              cudaStream_t st);
int tensor_acc(ensi_ctx* ctx, const uint64_t* a, uint64_t a_stride, uint32_t la, const uint64_t* e, uint32_t cnt,
               uint64_t* D, uint32_t lv, bool init, cudaStream_t st);
int relinearize(ensi_ctx* ctx, const uint64_t* d, uint32_t cnt, uint32_t lv, uint64_t* out, cudaStream_t st);
int cc_scratch(ensi_ctx* ctx, size_t words);
int ccmm(ensi_ctx* ctx, const uint64_t* a, const uint64_t* src, uint32_t form, uint32_t s, uint32_t d, uint32_t m,
         uint32_t level, const uint64_t* mask, uint64_t* y, uint32_t i0, uint32_t i1, cudaStream_t st);

// wire format (poly.cu): words <-> wb-byte little-endian packing, words a multiple of 4
int wire_unpack(ensi_ctx* ctx, const uint8_t* in, uint64_t* out, size_t words, uint32_t wb, cudaStream_t st);
int wire_pack(ensi_ctx* ctx, const uint64_t* in, uint8_t* out, size_t words, uint32_t wb, cudaStream_t st);
int wire_unpack_rows(ensi_ctx* ctx, const uint8_t* in, size_t wire_rs, uint64_t* out, size_t word_rs, uint32_t rows,
                     size_t words, uint32_t wb, cudaStream_t st);
int wire_pack_rows(ensi_ctx* ctx, const uint64_t* in, size_t word_rs, uint8_t* out, size_t wire_rs, uint32_t rows,
                   size_t words, uint32_t wb, cudaStream_t st);

// poly (poly.cu)
int rescale(ensi_ctx* ctx, const uint64_t* in, uint32_t count, uint32_t level, uint64_t* out, cudaStream_t st);
int decrypt_mu(ensi_ctx* ctx, const uint64_t* ct, uint32_t level, uint64_t* mu, cudaStream_t st);
void add_into(ensi_ctx* ctx, uint64_t* y, const uint64_t* x, uint32_t count, uint32_t level, cudaStream_t st);

inline LimbMap identity_map(uint32_t level) {
    LimbMap m{};
    m.period = level;
    m.grp_rows = 1u << 30;
    m.grp_stride = 0;
    m.grp_off = 0;
    for (uint32_t i = 0; i < level; i++) m.limb[i] = (uint8_t)i;
    return m;
}
// limbs of an extended (Q_l u P) polynomial: e < level -> q_e, else p_{e-level}
inline uint32_t ext_limb(const ensi_ctx* ctx, uint32_t level, uint32_t e) { return e < level ? e : ctx->L + (e - level); }
inline LimbMap ext_map(const ensi_ctx* ctx, uint32_t level) {
    LimbMap m = identity_map(level + ctx->A);
    for (uint32_t e = 0; e < level + ctx->A; e++) m.limb[e] = (uint8_t)ext_limb(ctx, level, e);
    return m;
}

}  // namespace ensi

#define ENSI_LAUNCH_CHECK(ctx)                                             \
    do {                                                                   \
        (ctx)->launches++;                                                 \
    } while (0)
