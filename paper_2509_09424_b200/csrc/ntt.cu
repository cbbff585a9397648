// ntt.cu -- negacyclic NTT / INTT per RNS limb (row a5; R10).
//
// Forward: merged-psi Cooley-Tukey, output a[k] = sum_i a_i psi^{(2 brv(k)+1) i} (bit-reversed order).
// Inverse: Gentleman-Sande with psi^{-brv}, times N'^{-1}.
// N' = N1 * N2.  For log_n <= 12 a single kernel keeps the whole limb in shared memory.  Otherwise two
// passes: the strided pass runs the first log N1 stages on N2 independent columns (elements c + N2 i),
// the block pass runs the remaining log N2 stages on contiguous blocks of N2 words.  Each pass stages a
// 32 KB tile in shared memory (4096 words) with coalesced loads (16+ consecutive words per column row).
// Twiddle multiplications are Shoup products; every output word is canonical.
#include "ensi_internal.h"
#include "ntt_v2.cuh"
#include "ntt_fp.cuh"

namespace ensi {

static constexpr uint32_t kTile = 4096;   // words per CTA tile (32 KB)
static constexpr uint32_t kThreads = 256;

__device__ __forceinline__ void ct_bfly(uint64_t& U, uint64_t& V, uint64_t w, uint64_t wp, uint64_t q) {
    uint64_t v = mul_shoup(V, w, wp, q);
    uint64_t u = U;
    U = add_mod(u, v, q);
    V = sub_mod(u, v, q);
}
__device__ __forceinline__ void gs_bfly(uint64_t& U, uint64_t& V, uint64_t w, uint64_t wp, uint64_t q) {
    uint64_t u = U, v = V;
    U = add_mod(u, v, q);
    V = mul_shoup(sub_mod(u, v, q), w, wp, q);
}

// ---- forward, strided pass: stages m = 1 .. N1/2 on columns c0 .. c0+cols-1
__global__ void __launch_bounds__(kThreads) k_ntt_fwd_strided(uint64_t* __restrict__ data, uint32_t log_n,
                                                               uint32_t log_n2, LimbMap map, ModTab tab,
                                                               const uint64_t* __restrict__ tw) {
    __shared__ uint64_t sm[kTile];
    const uint32_t n = 1u << log_n, N2 = 1u << log_n2, logN1 = log_n - log_n2, N1 = 1u << logN1;
    const uint32_t lcols = 12 - logN1, cols = 1u << lcols;   // N1 * cols == 4096
    const uint32_t row = blockIdx.y, limb = map.limb[row % map.period];
    const uint64_t q = tab.q[limb];
    const uint64_t* W = tw + (size_t)limb * 4 * n;
    const uint64_t* Wp = W + n;
    uint64_t* a = data + map.phys(row) * n;
    const uint32_t c0 = blockIdx.x * cols;
    for (uint32_t idx = threadIdx.x; idx < kTile; idx += kThreads) {
        uint32_t i = idx >> lcols, cc = idx & (cols - 1);
        sm[idx] = a[c0 + cc + ((size_t)i << log_n2)];
    }
    __syncthreads();
    for (uint32_t lm = 0; lm < logN1; lm++) {
        const uint32_t m = 1u << lm, lt = logN1 - 1 - lm;
        for (uint32_t bi = threadIdx.x; bi < kTile / 2; bi += kThreads) {
            uint32_t cc = bi & (cols - 1), b = bi >> lcols;
            uint32_t i1 = ((b >> lt) << (lt + 1)) | (b & ((1u << lt) - 1)), i2 = i1 + (1u << lt);
            uint32_t ti = m + (b >> lt);
            uint64_t U = sm[(i1 << lcols) | cc], V = sm[(i2 << lcols) | cc];
            ct_bfly(U, V, W[ti], Wp[ti], q);
            sm[(i1 << lcols) | cc] = U;
            sm[(i2 << lcols) | cc] = V;
        }
        __syncthreads();
    }
    for (uint32_t idx = threadIdx.x; idx < kTile; idx += kThreads) {
        uint32_t i = idx >> lcols, cc = idx & (cols - 1);
        a[c0 + cc + ((size_t)i << log_n2)] = sm[idx];
    }
}

// ---- forward, block pass: stages m = 2^lm0 .. N'/2 inside blocks of N2 = 2^log_n2 contiguous words.
// A CTA covers min(4096, N') words = nb blocks.
__global__ void __launch_bounds__(kThreads) k_ntt_fwd_block(uint64_t* __restrict__ data, uint32_t log_n,
                                                            uint32_t log_n2, uint32_t lm0, LimbMap map, ModTab tab,
                                                            const uint64_t* __restrict__ tw) {
    __shared__ uint64_t sm[kTile];
    const uint32_t n = 1u << log_n, N2 = 1u << log_n2;
    const uint32_t tile = n < kTile ? n : kTile;
    const uint32_t row = blockIdx.y, limb = map.limb[row % map.period];
    const uint64_t q = tab.q[limb];
    const uint64_t* W = tw + (size_t)limb * 4 * n;
    const uint64_t* Wp = W + n;
    uint64_t* a = data + map.phys(row) * n + (size_t)blockIdx.x * tile;
    const uint32_t B0 = blockIdx.x * (tile >> log_n2);
    for (uint32_t idx = threadIdx.x; idx < tile; idx += kThreads) sm[idx] = a[idx];
    __syncthreads();
    for (uint32_t lm = lm0; lm < log_n; lm++) {
        const uint32_t m = 1u << lm, lt = log_n - 1 - lm;
        for (uint32_t bi = threadIdx.x; bi < tile / 2; bi += kThreads) {
            uint32_t bb = bi >> (log_n2 - 1), b = bi & ((N2 >> 1) - 1);
            uint32_t i1 = ((b >> lt) << (lt + 1)) | (b & ((1u << lt) - 1)), i2 = i1 + (1u << lt);
            uint32_t ti = m + (B0 + bb) * (N2 >> (lt + 1)) + (b >> lt);
            uint32_t base = bb << log_n2;
            uint64_t U = sm[base + i1], V = sm[base + i2];
            ct_bfly(U, V, W[ti], Wp[ti], q);
            sm[base + i1] = U;
            sm[base + i2] = V;
        }
        __syncthreads();
    }
    for (uint32_t idx = threadIdx.x; idx < tile; idx += kThreads) a[idx] = sm[idx];
}

// ---- inverse, block pass: GS stages t = 1 .. N2/2 (lt = 0 .. log_n2-1) inside blocks; optional N'^{-1}
__global__ void __launch_bounds__(kThreads) k_intt_block(uint64_t* __restrict__ data, uint32_t log_n, uint32_t log_n2,
                                                         int scale, LimbMap map, ModTab tab,
                                                         const uint64_t* __restrict__ tw, const uint64_t* ninv) {
    __shared__ uint64_t sm[kTile];
    const uint32_t n = 1u << log_n, N2 = 1u << log_n2;
    const uint32_t tile = n < kTile ? n : kTile;
    const uint32_t row = blockIdx.y, limb = map.limb[row % map.period];
    const uint64_t q = tab.q[limb];
    const uint64_t* W = tw + (size_t)limb * 4 * n + 2 * (size_t)n;
    const uint64_t* Wp = W + n;
    uint64_t* a = data + map.phys(row) * n + (size_t)blockIdx.x * tile;
    const uint32_t B0 = blockIdx.x * (tile >> log_n2);
    for (uint32_t idx = threadIdx.x; idx < tile; idx += kThreads) sm[idx] = a[idx];
    __syncthreads();
    for (uint32_t lt = 0; lt < log_n2; lt++) {
        const uint32_t h = n >> (lt + 1);
        for (uint32_t bi = threadIdx.x; bi < tile / 2; bi += kThreads) {
            uint32_t bb = bi >> (log_n2 - 1), b = bi & ((N2 >> 1) - 1);
            uint32_t i1 = ((b >> lt) << (lt + 1)) | (b & ((1u << lt) - 1)), i2 = i1 + (1u << lt);
            uint32_t ti = h + (B0 + bb) * (N2 >> (lt + 1)) + (b >> lt);
            uint32_t base = bb << log_n2;
            uint64_t U = sm[base + i1], V = sm[base + i2];
            gs_bfly(U, V, W[ti], Wp[ti], q);
            sm[base + i1] = U;
            sm[base + i2] = V;
        }
        __syncthreads();
    }
    if (scale) {
        const uint64_t ni = ninv[2 * limb], nip = ninv[2 * limb + 1];
        for (uint32_t idx = threadIdx.x; idx < tile; idx += kThreads) a[idx] = mul_shoup(sm[idx], ni, nip, q);
    } else {
        for (uint32_t idx = threadIdx.x; idx < tile; idx += kThreads) a[idx] = sm[idx];
    }
}

// ---- inverse, strided pass: GS stages t = N2 .. N'/2 on columns, then N'^{-1}
__global__ void __launch_bounds__(kThreads) k_intt_strided(uint64_t* __restrict__ data, uint32_t log_n,
                                                           uint32_t log_n2, LimbMap map, ModTab tab,
                                                           const uint64_t* __restrict__ tw, const uint64_t* ninv) {
    __shared__ uint64_t sm[kTile];
    const uint32_t n = 1u << log_n, logN1 = log_n - log_n2;
    const uint32_t lcols = 12 - logN1, cols = 1u << lcols;
    const uint32_t row = blockIdx.y, limb = map.limb[row % map.period];
    const uint64_t q = tab.q[limb];
    const uint64_t* W = tw + (size_t)limb * 4 * n + 2 * (size_t)n;
    const uint64_t* Wp = W + n;
    uint64_t* a = data + map.phys(row) * n;
    const uint32_t c0 = blockIdx.x * cols;
    for (uint32_t idx = threadIdx.x; idx < kTile; idx += kThreads) {
        uint32_t i = idx >> lcols, cc = idx & (cols - 1);
        sm[idx] = a[c0 + cc + ((size_t)i << log_n2)];
    }
    __syncthreads();
    for (uint32_t ltt = 0; ltt < logN1; ltt++) {
        const uint32_t lt = ltt + log_n2, h = n >> (lt + 1);
        for (uint32_t bi = threadIdx.x; bi < kTile / 2; bi += kThreads) {
            uint32_t cc = bi & (cols - 1), b = bi >> lcols;
            uint32_t i1 = ((b >> ltt) << (ltt + 1)) | (b & ((1u << ltt) - 1)), i2 = i1 + (1u << ltt);
            uint32_t ti = h + (b >> ltt);
            uint64_t U = sm[(i1 << lcols) | cc], V = sm[(i2 << lcols) | cc];
            gs_bfly(U, V, W[ti], Wp[ti], q);
            sm[(i1 << lcols) | cc] = U;
            sm[(i2 << lcols) | cc] = V;
        }
        __syncthreads();
    }
    const uint64_t ni = ninv[2 * limb], nip = ninv[2 * limb + 1];
    for (uint32_t idx = threadIdx.x; idx < kTile; idx += kThreads) {
        uint32_t i = idx >> lcols, cc = idx & (cols - 1);
        a[c0 + cc + ((size_t)i << log_n2)] = mul_shoup(sm[idx], ni, nip, q);
    }
}


static uint32_t split_log_n2(uint32_t log_n) { return log_n <= 12 ? log_n : log_n - log_n / 2; }

// Kernel choice at N' = 2^16: the FP64 passes (ntt_fp.cuh) when every modulus is below 2^50, else the integer v2
// passes; other sizes use the generic shared-memory kernels above.  The narrow-limb FP64 block passes read the
// compact w-only twiddle table (ctx->d_tw1).
static bool use_fp(const ensi_ctx* ctx) { return ctx->log_n == 16 && ctx->ntt_fp_ok; }
static bool use_v2(const ensi_ctx* ctx) { return ctx->log_n == 16 && !ctx->ntt_fp_ok; }
static const double* tw1_of(const ensi_ctx* ctx) { return ctx->d_tw1; }

// Tensor map of a row buffer for the TMA block passes: {16 words, N'/16 chunks, physical rows}, box {16, 256, 1},
// SWIZZLE_128B (false if the driver entry point is unavailable; the callers then use the shared-memory transpose).
typedef CUresult (*PFN_tmapEncode)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static bool row_tmap(const ensi_ctx* ctx, uint64_t* data, uint32_t rows, const LimbMap& map, CUtensorMap* tm) {
    static int init = 0;
    static PFN_tmapEncode enc = nullptr;
    if (!init) {
        init = 1;
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            enc = (PFN_tmapEncode)p;
    }
    if (!enc || rows == 0) return false;
    const uint64_t n = ctx->n;
    cuuint64_t dims[3] = {16, n / 16, map.phys(rows - 1) + 1};
    cuuint64_t strides[2] = {128, n * 8};
    cuuint32_t box[3] = {16, 256, 1}, es[3] = {1, 1, 1};
    return enc(tm, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, (void*)data, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
           CUDA_SUCCESS;
}

bool ntt_row_tmap(const ensi_ctx* ctx, uint64_t* data, uint32_t rows, const LimbMap& map, CUtensorMap* tm) {
    return row_tmap(ctx, data, rows, map, tm);
}

void ntt_forward(ensi_ctx* ctx, uint64_t* data, uint32_t rows, const LimbMap& map, cudaStream_t st) {
    if (rows == 0) return;
    const uint32_t log_n = ctx->log_n, n = ctx->n;
    if (use_fp(ctx)) {
        const double2* tw = reinterpret_cast<const double2*>(ctx->d_tw3);
        dim3 g(16, rows);
        CUtensorMap tm;
        nttfp::k_ntt256<nttfp::FWD_A><<<g, 256, 0, st>>>(data, map, ctx->tab, tw, tw + (size_t)ctx->T * 2 * n);
        if (row_tmap(ctx, data, rows, map, &tm))
            nttfp::k_ntt256_tma<nttfp::FWD_B><<<g, 256, 0, st>>>(data, map, ctx->tab, tw, tw + (size_t)ctx->T * 2 * n, tm,
                                                                 nttfp::PlainOut(), LimbMap(), 0u, tw1_of(ctx));
        else
            nttfp::k_ntt256<nttfp::FWD_B><<<g, 256, 0, st>>>(data, map, ctx->tab, tw, tw + (size_t)ctx->T * 2 * n);
        ctx->launches += 2;
        return;
    }
    if (use_v2(ctx)) {
        const uint64_t* ninv = ctx->d_tw + (size_t)ctx->T * 4 * n;
        dim3 g(16, rows);
        v2::k_ntt256<v2::FWD_A><<<g, 256, 0, st>>>(data, map, ctx->tab, ctx->d_tw2, ninv);
        v2::k_ntt256<v2::FWD_B><<<g, 256, 0, st>>>(data, map, ctx->tab, ctx->d_tw2, ninv);
        ctx->launches += 2;
        return;
    }
    const uint32_t ln2 = split_log_n2(log_n);
    const uint32_t tile = n < kTile ? n : kTile;
    if (ln2 < log_n) {
        const uint32_t cols = 1u << (12 - (log_n - ln2));
        dim3 g((1u << ln2) / cols, rows);
        k_ntt_fwd_strided<<<g, kThreads, 0, st>>>(data, log_n, ln2, map, ctx->tab, ctx->d_tw);
        ENSI_LAUNCH_CHECK(ctx);
    }
    dim3 g2(n / tile, rows);
    k_ntt_fwd_block<<<g2, kThreads, 0, st>>>(data, log_n, ln2, log_n - ln2, map, ctx->tab, ctx->d_tw);
    ENSI_LAUNCH_CHECK(ctx);
}

bool ntt_inverse_from(ensi_ctx* ctx, const uint64_t* src, const LimbMap& smap, uint64_t* dst, uint32_t rows,
                      const LimbMap& dmap, cudaStream_t st) {
    if (rows == 0) return true;
    if (!use_fp(ctx)) return false;
    CUtensorMap tm;
    if (!row_tmap(ctx, const_cast<uint64_t*>(src), rows, smap, &tm)) return false;
    const double2* tw = reinterpret_cast<const double2*>(ctx->d_tw3);
    const uint32_t n = ctx->n;
    dim3 g(16, rows);
    nttfp::k_ntt256_tma<nttfp::INV_B><<<g, 256, 0, st>>>(dst, dmap, ctx->tab, tw, tw + (size_t)ctx->T * 2 * n, tm,
                                                         nttfp::PlainOut(), smap, 1u, tw1_of(ctx));
    nttfp::k_ntt256<nttfp::INV_A><<<g, 256, 0, st>>>(dst, dmap, ctx->tab, tw, tw + (size_t)ctx->T * 2 * n);
    ctx->launches += 2;
    return true;
}

void ntt_inverse(ensi_ctx* ctx, uint64_t* data, uint32_t rows, const LimbMap& map, cudaStream_t st) {
    if (rows == 0) return;
    const uint32_t log_n = ctx->log_n, n = ctx->n;
    const uint32_t ln2 = split_log_n2(log_n);
    const uint32_t tile = n < kTile ? n : kTile;
    const uint64_t* ninv = ctx->d_tw + (size_t)ctx->T * 4 * n;   // [T][2] appended after the twiddles
    if (use_fp(ctx)) {
        const double2* tw = reinterpret_cast<const double2*>(ctx->d_tw3);
        dim3 g(16, rows);
        CUtensorMap tm;
        if (row_tmap(ctx, data, rows, map, &tm))
            nttfp::k_ntt256_tma<nttfp::INV_B><<<g, 256, 0, st>>>(data, map, ctx->tab, tw, tw + (size_t)ctx->T * 2 * n, tm,
                                                                 nttfp::PlainOut(), LimbMap(), 0u, tw1_of(ctx));
        else
            nttfp::k_ntt256<nttfp::INV_B><<<g, 256, 0, st>>>(data, map, ctx->tab, tw, tw + (size_t)ctx->T * 2 * n);
        nttfp::k_ntt256<nttfp::INV_A><<<g, 256, 0, st>>>(data, map, ctx->tab, tw, tw + (size_t)ctx->T * 2 * n);
        ctx->launches += 2;
        return;
    }
    if (use_v2(ctx)) {
        dim3 g(16, rows);
        v2::k_ntt256<v2::INV_B><<<g, 256, 0, st>>>(data, map, ctx->tab, ctx->d_tw2, ninv);
        v2::k_ntt256<v2::INV_A><<<g, 256, 0, st>>>(data, map, ctx->tab, ctx->d_tw2, ninv);
        ctx->launches += 2;
        return;
    }
    dim3 g2(n / tile, rows);
    k_intt_block<<<g2, kThreads, 0, st>>>(data, log_n, ln2, ln2 == log_n ? 1 : 0, map, ctx->tab, ctx->d_tw, ninv);
    ENSI_LAUNCH_CHECK(ctx);
    if (ln2 < log_n) {
        const uint32_t cols = 1u << (12 - (log_n - ln2));
        dim3 g((1u << ln2) / cols, rows);
        k_intt_strided<<<g, kThreads, 0, st>>>(data, log_n, ln2, map, ctx->tab, ctx->d_tw, ninv);
        ENSI_LAUNCH_CHECK(ctx);
    }
}

}  // namespace ensi
