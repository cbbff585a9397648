// tc_ptx.cuh -- tcgen05 / TMA / mbarrier / cluster PTX wrappers and the byte-plane recombination shared by the
// tensor-core accumulate kernels (accum_tc.cu: uint64 words; accum_tcc.cu: compact words).
#pragma once
#include <cuda.h>

#include "ensi_internal.h"

namespace ensi {
namespace tc {

static constexpr uint32_t kIdescI8 = (2u << 4)     // D format s32
                                     | (1u << 7)   // A format: signed int8
                                     | (0u << 10)  // B format: unsigned int8
                                     | (0u << 15)  // A K-major
                                     | (1u << 16); // B MN-major
__host__ __device__ constexpr uint32_t idesc_i8(uint32_t m, uint32_t n) {
    return kIdescI8 | ((n >> 3) << 17) | ((m >> 4) << 24);
}
static constexpr uint32_t kPeerMask = 0xFEFFFFFFu;

struct EpiConst {
    uint64_t off_lo[ENSI_MAXT], off_hi[ENSI_MAXT];   // a multiple of q >= 2^80 (makes the 128-bit value non-negative)
    uint64_t off64[ENSI_MAXT];                       // narrow limbs: a multiple of q >= max |V| (64-bit path)
    uint32_t mu32[ENSI_MAXT];                        // narrow limbs: floor(2^64 / q) (< 2^32 since q > 2^32)
    uint32_t narrow_ok;                              // 64-bit path valid for this d (2 max|V| + q < 2^64)
};


__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
        "@P1 bra DONE_%=;\n\t"
        "bra WAIT_%=;\n\t"
        "DONE_%=:\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(0x989680u)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int32_t c0, int32_t c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"((uint64_t)map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int32_t c0, int32_t c1) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"((uint64_t)map),
                 "r"(smem_u32(src)), "r"(c0), "r"(c1)
                 : "memory");
}
__device__ __forceinline__ void tma_store_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void tma_store_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void tma_store_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// UMMA shared-memory descriptor, SWIZZLE_128B, Blackwell version bits.
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (2ull << 61);
}

__device__ __forceinline__ void mma_i8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(0u), "r"(0u), "r"(0u), "r"(0u));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

#define TMEM_LD_X32(taddr, r)                                                                                       \
    asm volatile(                                                                                                   \
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"   \
        "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                                          \
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),          \
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),    \
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),  \
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])   \
        : "r"(taddr))

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa_rank(uint32_t saddr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}
// Release of a TMEM accumulator to the pair leader's MMA issuer.  Relaxed: the only thing ordered before it is
// the epilogue's tcgen05.ld, already complete (tcgen05.wait::ld) and fenced (tcgen05.fence::before_thread_sync);
// a release.cluster arrive would also drain every prior store of the thread (ERRBAR), measured at 25% of the
// kernel's warp-stall samples.
__device__ __forceinline__ bool elect_one() {
    uint32_t pred;
    asm volatile(
        "{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(pred));
    return pred != 0;
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void tma_load_2d_2sm(void* dst, const CUtensorMap* map, uint64_t* bar, int32_t c0,
                                                int32_t c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
        "%4}], [%2];" ::"r"(smem_u32(dst)),
        "l"((uint64_t)map), "r"(smem_u32(bar) & kPeerMask), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void mma_i8_2sm(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                           uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, {%5, %6, %7, %8, %9, %10, %11, %12}, p;\n\t}" ::"r"(
            d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(0u), "r"(0u), "r"(0u), "r"(0u), "r"(0u), "r"(0u),
        "r"(0u), "r"(0u));
}
__device__ __forceinline__ void mma_commit_2sm_mc(uint64_t* bar, uint16_t mask) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"(mask)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d_2sm_mc(void* dst, const CUtensorMap* map, uint64_t* bar, uint16_t mask,
                                                   int32_t c0, int32_t c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
        " [%0], [%1, {%4, %5}], [%2], %3;" ::"r"(smem_u32(dst)),
        "l"((uint64_t)map), "r"(smem_u32(bar) & kPeerMask), "h"(mask), "r"(c0), "r"(c1)
        : "memory");
}

// sum_b D_b 2^{8b} (signed, |D_b| < 2^31) mod q, canonical.
__device__ __forceinline__ uint64_t combine_word(const uint32_t* r, const Barrett& br, uint64_t off_lo,
                                                 uint64_t off_hi) {
    int64_t lo = (int64_t)(int32_t)r[0] + (int64_t)(int32_t)r[1] * 256 + (int64_t)(int32_t)r[2] * 65536 +
                 (int64_t)(int32_t)r[3] * 16777216;
    int64_t hi = (int64_t)(int32_t)r[4] + (int64_t)(int32_t)r[5] * 256 + (int64_t)(int32_t)r[6] * 65536 +
                 (int64_t)(int32_t)r[7] * 16777216;
    // V = lo + hi * 2^32 as 128-bit two's complement, plus a multiple of q that makes it non-negative
    uint64_t v_lo = (uint64_t)lo + ((uint64_t)hi << 32);
    uint64_t carry = v_lo < (uint64_t)lo ? 1 : 0;
    int64_t v_hi = (hi >> 32) + (lo >> 63) + (int64_t)carry;
    uint64_t x_lo = v_lo + off_lo;
    uint64_t x_hi = (uint64_t)v_hi + off_hi + (x_lo < v_lo ? 1 : 0);
    return barrett128(x_hi, x_lo, br);
}

// planes 0..4 only (q < 2^40: bytes 5..7 of every canonical word are zero, so D_5 = D_6 = D_7 = 0).
// |V| <= 255 d (2^32 + 2^24 + 2^16 + 2^8 + 1) < 2^63 for d < 2^23, so V is a signed 64-bit value; u = V + off64
// (a multiple of q) is non-negative and u mod q = V mod q.  64-bit Barrett with mu = floor(2^64/q) < 2^32:
// qhat = floor((u_hi mu + floor(u_lo mu / 2^32)) / 2^32) = floor(u mu / 2^64) exactly, and u mu / 2^64 > u/q - 1,
// so qhat >= floor(u/q) - 1 and u - qhat q lies in [0, 2q): one conditional subtraction.
__device__ __forceinline__ uint64_t combine_word5(const uint32_t* r, uint64_t q, uint32_t mu32, uint64_t off64) {
    int64_t v = (int64_t)off64 + (int64_t)(int32_t)r[0];
    v += (int64_t)(int32_t)r[1] * 256;
    v += (int64_t)(int32_t)r[2] * 65536;
    v += (int64_t)(int32_t)r[3] * 16777216;
    const uint64_t u = (uint64_t)v + ((uint64_t)(int64_t)(int32_t)r[4] << 32);
    const uint32_t t = __umulhi((uint32_t)u, mu32);
    const uint32_t qhat = (uint32_t)(((uint64_t)(uint32_t)(u >> 32) * mu32 + t) >> 32);
    const uint64_t rr = u - (uint64_t)qhat * q;
    return rr >= q ? rr - q : rr;
}

// One cluster's walk over the (super-group sg, word tile t) work items of the pair kernels: items kc, kc + K,
// kc + 2K, ... of the list ordered tile-major (item = t nsg + sg) or super-group-major (item = sg ntiles + t),
// stepped without divisions (k_accum_tcc / k_accum_tc2).
struct WorkIter {
    uint32_t sg, t, dsg, dt, nsg, ntiles, tmajor;
    __device__ __forceinline__ WorkIter(uint32_t kc, uint32_t nclust, uint32_t nsg_, uint32_t ntiles_, uint32_t tmajor_)
        : nsg(nsg_), ntiles(ntiles_), tmajor(tmajor_) {
        if (tmajor) {
            t = kc / nsg;
            sg = kc % nsg;
            dt = nclust / nsg;
            dsg = nclust % nsg;
        } else {
            sg = kc / ntiles;
            t = kc % ntiles;
            dsg = nclust / ntiles;
            dt = nclust % ntiles;
        }
    }
    __device__ __forceinline__ bool valid() const { return tmajor ? t < ntiles : sg < nsg; }
    __device__ __forceinline__ void next() {
        sg += dsg;
        t += dt;
        if (tmajor) {
            if (sg >= nsg) {
                sg -= nsg;
                t++;
            }
        } else if (t >= ntiles) {
            t -= ntiles;
            sg++;
        }
    }
};

}  // namespace tc
}  // namespace ensi
