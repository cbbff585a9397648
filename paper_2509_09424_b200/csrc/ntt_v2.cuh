// ntt_v2.cuh -- N' = 2^16 negacyclic NTT passes (register radix-16 groups), shared by ntt.cu and the fused
// key-switching kernels of keyswitch.cu.
#pragma once
#include "ensi_internal.h"

namespace ensi {
// ================================================================================================================
// v2 for N' = 2^16 = 256 x 256: two passes of 8 radix-2 stages.  A CTA (256 threads) owns 16 sub-problems of 256
// points (pass A: columns c + 256 i; pass B: blocks 256 b + i); 16 threads per sub-problem, 16 points each, held
// in registers.  The 8 stages split into two register groups of 4 (strides 128..16 with points i = tt + 16k, then
// strides 8..1 with points i = 16 tt + k) separated by one shared-memory exchange, instead of a shared-memory
// round trip and a barrier per stage.  Harvey lazy butterflies keep values in [0, 4q) (CT) / [0, 2q) (GS); the
// last store reduces to canonical words.  Global accesses are 128-byte coalesced in every pass.
// ================================================================================================================
namespace v2 {

enum Pass { FWD_A = 0, FWD_B = 1, INV_B = 2, INV_A = 3 };
static constexpr uint32_t kRow = 273;   // smem row stride (words): 256 + 16 pads + 1 -> conflict-free

__device__ __forceinline__ uint32_t sidx(uint32_t sp, uint32_t i) { return sp * kRow + i + (i >> 4); }

// Plain I/O: the pass reads and writes the row in place.  Fused callers (keyswitch.cu) pass functors that compute
// the first pass's input on the fly (IN::load) or consume the last pass's canonical output (OUT::store).
struct PlainIn {
    __device__ __forceinline__ uint64_t load(const uint64_t* a, uint32_t, uint32_t, uint32_t k) const { return a[k]; }
};
struct PlainOut {
    __device__ __forceinline__ void store(uint64_t* a, uint32_t, uint32_t, uint32_t k, uint64_t v) const { a[k] = v; }
};

// tw: interleaved (w, w') table [limb][fwd/inv][N'][2] (ctx->d_tw2): one 16-byte load per butterfly twiddle.
template <int PASS, class IN = PlainIn, class OUT = PlainOut>
__global__ void __launch_bounds__(256, 3) k_ntt256(uint64_t* __restrict__ data, LimbMap map, ModTab tab,
                                                const uint64_t* __restrict__ tw, const uint64_t* __restrict__ ninv,
                                                IN in = IN(), OUT out = OUT()) {
    __shared__ uint64_t sm[16 * kRow];
    const uint32_t n = 65536;
    const uint32_t row = blockIdx.y, limb = map.limb[row % map.period];
    const uint64_t q = tab.q[limb], q2 = 2 * q;
    const bool fwd = PASS == FWD_A || PASS == FWD_B;
    const bool colp = PASS == FWD_A || PASS == INV_A;          // column (strided) pass
    const ulonglong2* W2 = reinterpret_cast<const ulonglong2*>(tw) + ((size_t)limb * 2 + (fwd ? 0 : 1)) * n;
    uint64_t* a = data + map.phys(row) * n;
    const uint32_t tid = threadIdx.x;
    // lane mapping: column passes put consecutive sub-problems (columns) on consecutive lanes; block passes put
    // consecutive points on consecutive lanes -- both give 128-byte coalesced global accesses
    const uint32_t sp = colp ? (tid & 15) : (tid >> 4);
    const uint32_t tt = colp ? (tid >> 4) : (tid & 15);
    const uint32_t sub = blockIdx.x * 16 + sp;                 // column c or block b
    auto gaddr = [&](uint32_t i) -> uint64_t { return colp ? (uint64_t)sub + 256ull * i : 256ull * sub + i; };
    uint64_t v[16];

    // twiddle index of the butterfly whose lower point is i1 at local stride 2^lt
    auto twi = [&](uint32_t lt, uint32_t i1) -> uint32_t {
        if (colp) return (128u >> lt) + (i1 >> (lt + 1));
        return (32768u >> lt) + sub * (128u >> lt) + (i1 >> (lt + 1));
    };
    auto ct = [&](uint64_t& U, uint64_t& V, uint32_t t) {   // CT, inputs/outputs in [0, 4q)
        uint64_t u = U >= q2 ? U - q2 : U;
        const ulonglong2 w = W2[t];
        uint64_t x = mul_shoup_lazy(V, w.x, w.y, q);         // [0, 2q)
        U = u + x;
        V = u + q2 - x;
    };
    auto gs = [&](uint64_t& U, uint64_t& V, uint32_t t) {   // GS, inputs/outputs in [0, 2q)
        uint64_t u = U, x = V;
        uint64_t s = u + x;
        U = s >= q2 ? s - q2 : s;
        const ulonglong2 w = W2[t];
        V = mul_shoup_lazy(u + q2 - x, w.x, w.y, q);
    };

    if (fwd) {
        // ---- load points i = tt + 16 k (coalesced for both passes)
#pragma unroll
        for (uint32_t k = 0; k < 16; k++)
            v[k] = PASS == FWD_A ? in.load(a, row, limb, (uint32_t)gaddr(tt + 16 * k)) : a[gaddr(tt + 16 * k)];
        // ---- group 1: local strides 128, 64, 32, 16 (k-stride 8, 4, 2, 1)
#pragma unroll
        for (int lt = 7; lt >= 4; lt--) {
            const uint32_t ks = 1u << (lt - 4);
#pragma unroll
            for (uint32_t k = 0; k < 16; k++)
                if (!(k & ks)) ct(v[k], v[k + ks], twi(lt, tt + 16 * k));
        }
#pragma unroll
        for (uint32_t k = 0; k < 16; k++) sm[sidx(sp, tt + 16 * k)] = v[k];
        __syncthreads();
#pragma unroll
        for (uint32_t k = 0; k < 16; k++) v[k] = sm[sidx(sp, 16 * tt + k)];
        // ---- group 2: local strides 8, 4, 2, 1 on points i = 16 tt + k
#pragma unroll
        for (int lt = 3; lt >= 0; lt--) {
            const uint32_t ks = 1u << lt;
#pragma unroll
            for (uint32_t k = 0; k < 16; k++)
                if (!(k & ks)) ct(v[k], v[k + ks], twi(lt, 16 * tt + k));
        }
        if (PASS == FWD_A) {
            // intermediate: keep [0, 4q) -> [0, 2q) is enough for the next pass's lazy butterflies
#pragma unroll
            for (uint32_t k = 0; k < 16; k++) a[gaddr(16 * tt + k)] = v[k] >= q2 ? v[k] - q2 : v[k];
        } else {
            // final: canonical, stored through smem so the block's 256 points leave as 128-byte segments
            __syncthreads();
#pragma unroll
            for (uint32_t k = 0; k < 16; k++) {
                uint64_t x = v[k] >= q2 ? v[k] - q2 : v[k];
                sm[sidx(sp, 16 * tt + k)] = x >= q ? x - q : x;
            }
            __syncthreads();
#pragma unroll
            for (uint32_t k = 0; k < 16; k++)
                out.store(a, row, limb, (uint32_t)gaddr(tt + 16 * k), sm[sidx(sp, tt + 16 * k)]);
        }
    } else {
        // ---- load points i = 16 tt + k
        if (PASS == INV_B) {
#pragma unroll
            for (uint32_t k = 0; k < 16; k++) sm[sidx(sp, tt + 16 * k)] = a[gaddr(tt + 16 * k)];
            __syncthreads();
#pragma unroll
            for (uint32_t k = 0; k < 16; k++) v[k] = sm[sidx(sp, 16 * tt + k)];
        } else {
#pragma unroll
            for (uint32_t k = 0; k < 16; k++) v[k] = a[gaddr(16 * tt + k)];
        }
        // ---- group 1: local strides 1, 2, 4, 8
#pragma unroll
        for (int lt = 0; lt <= 3; lt++) {
            const uint32_t ks = 1u << lt;
#pragma unroll
            for (uint32_t k = 0; k < 16; k++)
                if (!(k & ks)) gs(v[k], v[k + ks], twi(lt, 16 * tt + k));
        }
        if (PASS == INV_B) __syncthreads();
#pragma unroll
        for (uint32_t k = 0; k < 16; k++) sm[sidx(sp, 16 * tt + k)] = v[k];
        __syncthreads();
#pragma unroll
        for (uint32_t k = 0; k < 16; k++) v[k] = sm[sidx(sp, tt + 16 * k)];
        // ---- group 2: local strides 16, 32, 64, 128 on points i = tt + 16 k
#pragma unroll
        for (int lt = 4; lt <= 7; lt++) {
            const uint32_t ks = 1u << (lt - 4);
#pragma unroll
            for (uint32_t k = 0; k < 16; k++)
                if (!(k & ks)) gs(v[k], v[k + ks], twi(lt, tt + 16 * k));
        }
        if (PASS == INV_B) {
#pragma unroll
            for (uint32_t k = 0; k < 16; k++) a[gaddr(tt + 16 * k)] = v[k];   // [0, 2q) intermediate
        } else {
            const uint64_t ni = ninv[2 * limb], nip = ninv[2 * limb + 1];
#pragma unroll
            for (uint32_t k = 0; k < 16; k++) a[gaddr(tt + 16 * k)] = mul_shoup(v[k], ni, nip, q);
        }
    }
}

}  // namespace v2

}  // namespace ensi
