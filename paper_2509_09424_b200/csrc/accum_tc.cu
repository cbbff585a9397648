// accum_tc.cu -- row a3 (Algorithm 1) on the 5th-generation tensor cores.
//
// Byte-sliced exact integer contraction.  For a ciphertext word x (< 2^60) write x = sum_b x_b 2^{8b} with
// bytes x_b in [0,255].  Then for every output i and word w
//     y_i[w] = sum_j W[j][i] x_j[w] = sum_b 2^{8b} D[i][8w+b],   D[i][c] = sum_j W[j][i] * byte_c(x_j)
// and D is an int8 x uint8 -> int32 GEMM that is EXACT (|D| <= 255 d < 2^31).  Its B operand is the raw memory
// of the input ciphertexts: byte c of ciphertext j is B[j][c], i.e. B is an MN-major (N-contiguous) uint8
// matrix that TMA reads straight from the uint64 ciphertext buffers -- no repacking pass.  A = W^T (int8,
// K-major, zero padded).  The epilogue reads 8 consecutive TMEM columns (the 8 byte planes of one word) per
// thread, forms sum_b D_b 2^{8b} as a signed 128-bit value and reduces it to the canonical word in [0, q) --
// the same unique value Algorithm 1 defines, so the output is bit-identical to the oracle and to accum.cu.
//
// Kernel structure (persistent, one CTA per SM, 320 threads):
//   warp 0      TMA producer: W^T slice (resident in smem when 128*d_pad <= 96 KB, else streamed per stage) and
//               the X byte tiles (128 K-rows x 256 bytes, two SWIZZLE_128B boxes) into a 3-stage mbarrier ring.
//   warp 1      TMEM allocation (512 columns = 2 accumulators x 256) and the single-thread tcgen05.mma issue:
//               M = 128 outputs, N = 256 bytes (32 words), K = 32 per instruction, kind::i8 (s8 x u8 -> s32).
//   warps 2..9  epilogue: tcgen05.ld 32x32b.x32, byte-plane recombination + Barrett, SWIZZLE_128B smem
//               staging, TMA bulk-tensor store of 32 outputs x 16 words per warp.
// CTA b owns output group g = b % G (128 outputs) and walks the word tiles t = b / G, b / G + P, ...; the G CTAs
// that share a word tile run at the same time, so each X tile is read from HBM once and served to the others
// from L2.
#include <cuda.h>

#include <cstring>

#include "ensi_internal.h"
#include "tc_ptx.cuh"

#ifndef ENSI_EPI_EARLY_RELEASE
#define ENSI_EPI_EARLY_RELEASE 1
#endif

namespace ensi {

namespace tc {

static constexpr uint32_t kThreads = 320;
static constexpr uint32_t kStages = 3;
static constexpr uint32_t kBoxK = 128;                  // K rows per stage / A box inner bytes
static constexpr uint32_t kABox = 128 * 128;            // 16 KB: 128 outputs x 128 K
static constexpr uint32_t kBStage = 2 * 128 * 128;      // 32 KB: 128 K x 256 bytes (two 128-byte boxes)
static constexpr uint32_t kYWarp = 32 * 128;            // 4 KB: 32 outputs x 16 words
static constexpr uint32_t kAResMax = 96 * 1024;         // resident W^T slice budget
static constexpr uint32_t kIdesc = (2u << 4)            // D format s32
                                   | (1u << 7)          // A format: signed int8
                                   | (0u << 10)         // B format: unsigned int8
                                   | (0u << 15)         // A K-major
                                   | (1u << 16)         // B MN-major
                                   | ((256u >> 3) << 17)  // N = 256
                                   | ((128u >> 4) << 24); // M = 128


template <bool A_RES>
__global__ void __launch_bounds__(kThreads, 1)
    k_accum_tc(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
               const __grid_constant__ CUtensorMap map_y, uint32_t kblocks, uint32_t groups, uint32_t per_group,
               uint32_t ntiles, uint32_t log_n, uint32_t level, uint32_t limb0, ModTab tab, EpiConst ec) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    const uint32_t a_bytes = A_RES ? kblocks * kABox : kStages * kABox;
    uint8_t* sA = smem;
    uint8_t* sB = sA + a_bytes;
    uint8_t* sY = sB + kStages * kBStage;
    uint64_t* bars = (uint64_t*)(sY + 8 * kYWarp);
    uint64_t* full = bars;                    // [kStages]
    uint64_t* empty = bars + kStages;         // [kStages]
    uint64_t* tfull = bars + 2 * kStages;     // [2]
    uint64_t* tempty = tfull + 2;             // [2]
    uint64_t* afull = tempty + 2;             // [1]
    uint32_t* tmem_slot = (uint32_t*)(afull + 1);

    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t g = blockIdx.x % groups;   // output group (128 outputs)
    const uint32_t p = blockIdx.x / groups;   // position in the group's tile walk
    if (p >= per_group) return;

    if (threadIdx.x == 0) {
        for (uint32_t s = 0; s < kStages; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; a++) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 8);
        }
        mbar_init(afull, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ------------------------------------------------------------------ TMA producer
        if (lane == 0) {
            if (A_RES) {
                mbar_expect_tx(afull, kblocks * kABox);
                for (uint32_t kb = 0; kb < kblocks; kb++)
                    tma_load_2d(sA + kb * kABox, &map_a, afull, (int32_t)(kb * kBoxK), (int32_t)(g * 128));
            }
            uint32_t s = 0, ph = 0;
            for (uint32_t t = p; t < ntiles; t += per_group) {
                for (uint32_t kb = 0; kb < kblocks; kb++) {
                    mbar_wait(&empty[s], ph ^ 1);
                    mbar_expect_tx(&full[s], kBStage + (A_RES ? 0 : kABox));
                    uint8_t* b = sB + s * kBStage;
                    tma_load_2d(b, &map_b, &full[s], (int32_t)(t * 256), (int32_t)(kb * kBoxK));
                    tma_load_2d(b + kBStage / 2, &map_b, &full[s], (int32_t)(t * 256 + 128), (int32_t)(kb * kBoxK));
                    if (!A_RES)
                        tma_load_2d(sA + s * kABox, &map_a, &full[s], (int32_t)(kb * kBoxK), (int32_t)(g * 128));
                    if (++s == kStages) {
                        s = 0;
                        ph ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------------ MMA issuer
        if (lane == 0) {
            if (A_RES) mbar_wait(afull, 0);
            uint32_t s = 0, ph = 0, it = 0;
            for (uint32_t t = p; t < ntiles; t += per_group, it++) {
                const uint32_t acc = it & 1, use = it >> 1;
                mbar_wait(&tempty[acc], (use & 1) ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * 256;
                for (uint32_t kb = 0; kb < kblocks; kb++) {
                    mbar_wait(&full[s], ph);
                    tc_fence_after();
                    const uint32_t a_base = smem_u32(sA + (A_RES ? kb : s) * kABox);
                    const uint32_t b_base = smem_u32(sB + s * kBStage);
#pragma unroll
                    for (uint32_t kk = 0; kk < kBoxK / 32; kk++) {
                        uint64_t ad = umma_desc(a_base + kk * 32, 16, 1024);
                        uint64_t bd = umma_desc(b_base + kk * 32 * 128, kBStage / 2, 1024);
                        mma_i8(d_tmem, ad, bd, kIdesc, (kb | kk) != 0);
                    }
                    mma_commit(&empty[s]);
                    if (++s == kStages) {
                        s = 0;
                        ph ^= 1;
                    }
                }
                mma_commit(&tfull[acc]);
            }
        }
    } else {
        // ------------------------------------------------------------------ epilogue (8 warps)
        const uint32_t e = warp - 2;                 // 0..7
        const uint32_t quarter = warp & 3;           // TMEM lane quarter this warp may access
        const uint32_t half = e >> 2;                // words [16 half, 16 half + 16) of the tile
        uint8_t* ys = sY + e * kYWarp;
        const uint32_t row = lane;                   // output g*128 + 32*quarter + lane
        const uint32_t words_per_limb = 1u << log_n;
        uint32_t it = 0;
        for (uint32_t t = p; t < ntiles; t += per_group, it++) {
            const uint32_t acc = it & 1, use = it >> 1;
            const uint32_t word0 = t * 32;
            const uint32_t limb = (limb0 + word0 / words_per_limb) % level;
            const Barrett br = tab.br(limb);
            const uint64_t olo = ec.off_lo[limb], ohi = ec.off_hi[limb];
            mbar_wait(&tfull[acc], use & 1);
            tc_fence_after();
            // the previous TMA store from this warp's staging buffer must have finished reading it
            if (lane == 0) tma_store_wait_read0();
            __syncwarp();
#pragma unroll 1
            for (uint32_t c = 0; c < 4; c++) {   // 4 chunks of 4 words (32 TMEM columns)
                uint32_t r[32];
                const uint32_t taddr = tmem_base + ((quarter * 32) << 16) + acc * 256 + half * 128 + c * 32;
                TMEM_LD_X32(taddr, r);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (uint32_t wv = 0; wv < 4; wv += 2) {
                    uint64_t v0 = combine_word(r + 8 * wv, br, olo, ohi);
                    uint64_t v1 = combine_word(r + 8 * (wv + 1), br, olo, ohi);
                    const uint32_t wl = c * 4 + wv;             // word within this warp's 16 (even)
                    const uint32_t chunk = (wl >> 1) ^ (row & 7);  // SWIZZLE_128B: 16-byte chunk XOR row
                    uint64_t* dst = (uint64_t*)(ys + row * 128 + chunk * 16);
                    asm volatile("st.shared.v2.u64 [%0], {%1, %2};" ::"r"(smem_u32(dst)), "l"(v0), "l"(v1) : "memory");
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) {
                tma_store_2d(&map_y, ys, (int32_t)(word0 + half * 16), (int32_t)(g * 128 + quarter * 32));
                tma_store_commit();
            }
        }
        if (lane == 0) tma_store_wait0();
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
    }
}

// ================================================================================================================
// 2-CTA variant (cta_group::2, cluster of 2 on a TPC).  The pair computes M = 256 outputs x N = 256 bytes per tile:
// CTA r holds W^T rows [128 r, 128 r + 128) of the pair's 256 outputs (resident A) and the N-half [128 r, 128 r + 128)
// of every X byte tile, so each SM pulls half as many X bytes per MMA cycle as the 1-CTA kernel, and the freed
// shared memory deepens the TMA ring to 6 stages.  The leader (rank 0) issues the MMAs; both CTAs' TMA loads
// complete on the leader's barriers, the MMA commits multicast to both CTAs' barriers, and the epilogues
// (one per CTA, on its own TMEM lanes) release the accumulator through the leader's tempty barrier.
// ================================================================================================================

static constexpr uint32_t kStages2 = 6;
static constexpr uint32_t kThreads2 = 64 + 8 * 32;     // producer, MMA, 8 epilogue warps
static constexpr uint32_t kBStage2 = 128 * 128;         // 16 KB: 128 K rows x this CTA's 128-byte N half
static constexpr uint32_t kIdesc2 = (2u << 4) | (1u << 7) | (0u << 10) | (0u << 15) | (1u << 16) |
                                    ((256u >> 3) << 17) | ((256u >> 4) << 24);   // M = 256, N = 256

// MC = false: clusters of one pair (2 CTAs), each pair loads its own X tiles; the pairs of the pgroups output
//             groups that share a word tile meet only in L2.
// MC = true:  clusters of cpairs pairs (2*cpairs <= 8 CTAs).  The cpairs pairs of a cluster cover consecutive
//             output groups (a super-group) of the same word tile in lockstep; every X sub-box (32 K-rows x 128
//             bytes) is loaded once by one pair and multicast to the same N-half of every pair of the cluster, so
//             each X byte leaves L2/HBM once per cluster.  The stage ring is released only when all cpairs MMA
//             issuers have consumed it.
// Work items (super-group, word tile) are dealt round-robin to the nclust co-resident clusters, in the order and
// with the resident-W^T reloads of k_accum_tcc (accum_tcc.cu); tc_plan_clusters picks cpairs and nclust.
template <bool A_RES, bool MC>
__global__ void __launch_bounds__(kThreads2, 1)
    k_accum_tc2(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                const __grid_constant__ CUtensorMap map_y, uint32_t kblocks, uint32_t ntiles, uint32_t nsg,
                uint32_t tmajor, uint32_t nclust, uint32_t log_n, uint32_t level, uint32_t limb0, ModTab tab,
                EpiConst ec, uint32_t cpairs) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    const uint32_t a_bytes = A_RES ? kblocks * kABox : kStages2 * kABox;
    uint8_t* sA = smem;
    uint8_t* sB = sA + a_bytes;
    uint8_t* sY = sB + kStages2 * kBStage2;
    uint64_t* bars = (uint64_t*)(sY + 8 * kYWarp);
    uint64_t* full = bars;                     // [kStages2]  (leader's are the live ones)
    uint64_t* empty = bars + kStages2;         // [kStages2]  (per CTA, multicast commits)
    uint64_t* tfull = bars + 2 * kStages2;     // [2]         (per CTA, multicast commits)
    uint64_t* tempty = tfull + 2;              // [2]         (leader's: 16 arrivals)
    uint64_t* afull = tempty + 2;              // [1]         (leader's)
    uint64_t* adone = afull + 1;               // [1]         (per CTA: the MMAs reading the resident A completed)
    uint32_t* tmem_slot = (uint32_t*)(adone + 1);

    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t crank = cluster_rank();
    const uint32_t rank = crank & 1;           // rank inside the CTA pair (0 = leader, issues the MMAs)
    const uint32_t lead = crank & ~1u;         // cluster rank of this pair's leader
    const uint32_t pin = crank >> 1;           // pair inside the cluster
    const uint32_t kc = blockIdx.x / (2 * cpairs);
    // pair group (sg cpairs + pin): outputs [256 pg, 256 pg + 256); this CTA's 128-output group
    auto grp = [&](uint32_t sg) -> uint32_t { return (sg * cpairs + pin) * 2 + rank; };
    const uint16_t pair_mask = (uint16_t)(0x3u << lead);
    const uint16_t all_mask = MC ? (uint16_t)((1u << (2 * cpairs)) - 1) : pair_mask;

    if (threadIdx.x == 0) {
        for (uint32_t s = 0; s < kStages2; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], MC ? cpairs : 1);
        }
        for (int a = 0; a < 2; a++) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 16);
        }
        mbar_init(afull, 1);
        mbar_init(adone, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ------------------------------------------------------------------ TMA producer (both CTAs)
        if (lane == 0) {
            uint32_t s = 0, ph = 0, cur = ~0u, adph = 0;
            for (WorkIter wi(kc, nclust, nsg, ntiles, tmajor); wi.valid(); wi.next()) {
                const uint32_t sg = wi.sg, t = wi.t;
                const uint32_t g = grp(sg);
                if (A_RES && sg != cur) {
                    if (cur != ~0u) {           // every MMA on the previous W^T has completed (MMA issuer's commit)
                        mbar_wait(adone, adph);
                        adph ^= 1;
                    }
                    if (rank == 0) mbar_expect_tx(afull, 2 * kblocks * kABox);
                    for (uint32_t kb = 0; kb < kblocks; kb++)
                        tma_load_2d_2sm(sA + kb * kABox, &map_a, afull, (int32_t)(kb * kBoxK), (int32_t)(g * 128));
                    cur = sg;
                }
                for (uint32_t kb = 0; kb < kblocks; kb++) {
                    mbar_wait(&empty[s], ph ^ 1);
                    if (rank == 0) mbar_expect_tx(&full[s], 2 * (kBStage2 + (A_RES ? 0 : kABox)));
                    if (MC) {
                        // sub-box j (32 K-rows) of this N-half: issued by the pair with j % cpairs == its rank in the
                        // cluster, multicast to the same N-half (cluster ranks rank, rank + 2, ...) of every pair
                        const uint16_t half_mask = (uint16_t)(all_mask & (rank ? 0xAAAAu : 0x5555u));
                        for (uint32_t j = lead >> 1; j < kBoxK / 32; j += cpairs)
                            tma_load_2d_2sm_mc(sB + s * kBStage2 + j * 4096, &map_b, &full[s], half_mask,
                                               (int32_t)(t * 256 + rank * 128), (int32_t)(kb * kBoxK + j * 32));
                    } else {
                        tma_load_2d_2sm(sB + s * kBStage2, &map_b, &full[s], (int32_t)(t * 256 + rank * 128),
                                        (int32_t)(kb * kBoxK));
                    }
                    if (!A_RES)
                        tma_load_2d_2sm(sA + s * kABox, &map_a, &full[s], (int32_t)(kb * kBoxK), (int32_t)(g * 128));
                    if (++s == kStages2) {
                        s = 0;
                        ph ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------------ MMA issuer (leader CTA only)
        // The whole warp runs the loop (warp-uniform control flow and operands, so descriptors live in uniform
        // registers); one elected lane -- always lane 0, which therefore also owns the commits -- issues the MMAs.
        // A single-lane loop made the compiler rebuild every descriptor through an ELECT/R2UR.BROADCAST loop
        // (~23 instructions per MMA), and the issuer warp was busy 94% of its samples.
        if (rank == 0) {
            const uint64_t adesc0 = umma_desc(smem_u32(sA), 16, 1024);
            const uint64_t bdesc0 = umma_desc(smem_u32(sB), kBStage2, 1024);
            uint32_t s = 0, ph = 0, j = 0, cur = ~0u, aph = 0;
            for (WorkIter wi(kc, nclust, nsg, ntiles, tmajor); wi.valid(); wi.next(), j++) {
                const uint32_t sg = wi.sg, t = wi.t;
                if (A_RES && sg != cur) {
                    if (cur != ~0u) {           // release the resident W^T once the MMAs issued on it complete
                        if (elect_one()) mma_commit_2sm_mc(adone, pair_mask);
                        __syncwarp();
                    }
                    mbar_wait(afull, aph);
                    aph ^= 1;
                    tc_fence_after();
                    cur = sg;
                }
                const uint32_t acc = j & 1, use = j >> 1;
                mbar_wait(&tempty[acc], (use & 1) ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * 256;
                for (uint32_t kb = 0; kb < kblocks; kb++) {
                    mbar_wait(&full[s], ph);
                    tc_fence_after();
                    // descriptor start-address field is (smem address >> 4): K step of 32 bytes in A is +2, K step of
                    // 32 rows x 128 bytes in B is +256
                    const uint64_t ad = adesc0 + (uint64_t)(((A_RES ? kb : s) * kABox) >> 4);
                    const uint64_t bd = bdesc0 + (uint64_t)((s * kBStage2) >> 4);
                    if (elect_one()) {
#pragma unroll
                        for (uint32_t kk = 0; kk < kBoxK / 32; kk++)
                            mma_i8_2sm(d_tmem, ad + 2 * kk, bd + 256 * kk, kIdesc2, (kb | kk) != 0);
                        mma_commit_2sm_mc(&empty[s], all_mask);
                    }
                    __syncwarp();
                    if (++s == kStages2) {
                        s = 0;
                        ph ^= 1;
                    }
                }
                if (elect_one()) mma_commit_2sm_mc(&tfull[acc], pair_mask);
                __syncwarp();
            }
        }
    } else {
        // ------------------------------------------------------------------ epilogue (8 warps per CTA)
        // warp (quarter q = warp % 4, half h = (warp-2) / 4): TMEM lanes [32q, 32q+32) = outputs, words
        // [16 h, 16 h + 16) of the 32-word tile.
        const uint32_t e = warp - 2;
        const uint32_t quarter = warp & 3;
        const uint32_t half = e >> 2;
        uint8_t* ys = sY + e * kYWarp;
        const uint32_t row = lane;
        const uint32_t words_per_limb = 1u << log_n;
        const uint32_t tempty_leader0 = mapa_rank(smem_u32(&tempty[0]), lead);
        uint32_t j = 0;
        for (WorkIter wi(kc, nclust, nsg, ntiles, tmajor); wi.valid(); wi.next(), j++) {
            const uint32_t sg = wi.sg, t = wi.t;
            const uint32_t g = grp(sg);
            const uint32_t acc = j & 1, use = j >> 1;
            const uint32_t word0 = t * 32;
            const uint32_t limb = (limb0 + word0 / words_per_limb) % level;
            const Barrett br = tab.br(limb);
            const uint64_t olo = ec.off_lo[limb], ohi = ec.off_hi[limb];
            const bool narrow = ec.narrow_ok && br.w <= 40;   // bytes 5..7 of every word are zero
            const uint64_t off64 = ec.off64[limb];
            const uint32_t mu32 = ec.mu32[limb];
            mbar_wait(&tfull[acc], use & 1);
            tc_fence_after();
            if (lane == 0) tma_store_wait_read0();
            __syncwarp();
            // Software-pipelined TMEM drain: the 32-column load of chunk c+1 is in flight while chunk c's four
            // words are combined (four independent reduction chains per thread).
            const uint32_t tbase = tmem_base + ((quarter * 32) << 16) + acc * 256 + half * 128;
            uint32_t ra[32], rb[32];
            auto combine4 = [&](const uint32_t* r, uint32_t c) {
                uint64_t v[4];
                if (narrow) {
#pragma unroll
                    for (uint32_t wv = 0; wv < 4; wv++) v[wv] = combine_word5(r + 8 * wv, br.q, mu32, off64);
                } else {
#pragma unroll
                    for (uint32_t wv = 0; wv < 4; wv++) v[wv] = combine_word(r + 8 * wv, br, olo, ohi);
                }
#pragma unroll
                for (uint32_t wv = 0; wv < 4; wv += 2) {
                    const uint32_t wl = c * 4 + wv;
                    const uint32_t chunk = (wl >> 1) ^ (row & 7);
                    uint64_t* dst = (uint64_t*)(ys + row * 128 + chunk * 16);
                    asm volatile("st.shared.v2.u64 [%0], {%1, %2};" ::"r"(smem_u32(dst)), "l"(v[wv]), "l"(v[wv + 1])
                                 : "memory");
                }
            };
#if ENSI_EPI_EARLY_RELEASE
            // Drain the whole 128-column slice into registers (4 x 32 columns, one wait) and hand the accumulator
            // back before any combine: the MMA issuer's wait for a free accumulator no longer includes the
            // epilogue's arithmetic.
            uint32_t rc[32], rd[32];
            TMEM_LD_X32(tbase, ra);
            TMEM_LD_X32(tbase + 32, rb);
            TMEM_LD_X32(tbase + 64, rc);
            TMEM_LD_X32(tbase + 96, rd);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_remote(tempty_leader0 + acc * 8);
            combine4(ra, 0);
            combine4(rb, 1);
            combine4(rc, 2);
            combine4(rd, 3);
#else
            TMEM_LD_X32(tbase, ra);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            TMEM_LD_X32(tbase + 32, rb);
            combine4(ra, 0);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            TMEM_LD_X32(tbase + 64, ra);
            combine4(rb, 1);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            TMEM_LD_X32(tbase + 96, rb);
            combine4(ra, 2);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            // every TMEM read of this accumulator slice is done: hand it back to the MMA issuer
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_remote(tempty_leader0 + acc * 8);
            combine4(rb, 3);
#endif
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) {
                tma_store_2d(&map_y, ys, (int32_t)(word0 + half * 16), (int32_t)(g * 128 + quarter * 32));
                tma_store_commit();
            }
        }
        if (lane == 0) tma_store_wait0();
    }
    tc_fence_before();
    cluster_sync_all();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
    }
}

}  // namespace tc

// ---------------------------------------------------------------------------------------------- host side

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
    static PFN_encodeTiled fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_encodeTiled)p;
    }
    return fn;
}

bool tc_supported(const ensi_ctx* ctx, uint32_t level) {
    (void)level;
    if (ctx->n < 32) return false;
    int dev = ctx->device, major = 0, minor = 0;
    if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess) return false;
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    if (major != 10 || minor != 0) return false;   // built for sm_100a only
    // epilogue ranges: the 64-bit narrow combine needs 2^32 < q (mu32 = floor(2^64/q) < 2^32), the 128-bit combine
    // needs V + off < 2^(2w+2) with off ~ 2^80 (w >= 40, i.e. every limb that is not narrow), and q < 2^60
    for (uint32_t i = 0; i < ctx->L; i++)
        if (ctx->mod[i] >= (1ull << 60) || ctx->mod[i] <= (1ull << 32)) return false;
    return get_encode() != nullptr;
}

int build_wt8(ensi_ctx* ctx, ensi_weights* w) {
    if (w->d_wt8) return ENSI_OK;
    const uint32_t mpad = (w->m + 255) / 256 * 256, dpad = (w->d + 127) / 128 * 128;
    std::vector<int8_t> wt((size_t)mpad * dpad, 0);
    for (uint32_t j = 0; j < w->d; j++)
        for (uint32_t i = 0; i < w->m; i++) wt[(size_t)i * dpad + j] = w->host[(size_t)j * w->m + i];
    cudaError_t e = cudaMalloc(&w->d_wt8, wt.size());
    if (e == cudaSuccess) e = cudaMemcpy(w->d_wt8, wt.data(), wt.size(), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cuda_err(ctx, e, "W^T upload");
    w->wt_mpad = mpad;
    w->wt_dpad = dpad;
    return ENSI_OK;
}

// Epilogue constants per limb: off = a multiple of q >= 2^80 (128-bit path), off64 = a multiple of q >= max|V| and
// mu32 = floor(2^64 / q) (64-bit path of words below 2^40), narrow_ok = the 64-bit path is exact for this d.
void fill_epi_const(const ensi_ctx* ctx, const ensi_weights* w, tc::EpiConst* ecp) {
    tc::EpiConst& ec = *ecp;
    std::memset(&ec, 0, sizeof(ec));
    for (uint32_t i = 0; i < ctx->L; i++) {
        // off = q * ceil(2^80 / q) as 128-bit
        typedef unsigned __int128 u128;
        const u128 q = ctx->mod[i];
        const u128 two80 = ((u128)1) << 80;
        const u128 off = ((two80 + q - 1) / q) * q;
        ec.off_lo[i] = (uint64_t)off;
        ec.off_hi[i] = (uint64_t)(off >> 64);
        // narrow 64-bit path: Vmax = 255 d_pad (2^32 + 2^24 + 2^16 + 2^8 + 1)
        const u128 vmax = (u128)255 * w->wt_dpad * ((((u128)1) << 32) + (1u << 24) + (1u << 16) + (1u << 8) + 1);
        const u128 off64 = ((vmax + q - 1) / q) * q;
        ec.off64[i] = (uint64_t)off64;
        ec.mu32[i] = (q > (((u128)1) << 32)) ? (uint32_t)((((u128)1) << 64) / q) : 0;
        if (i == 0) ec.narrow_ok = (2 * vmax + q < (((u128)1) << 64)) ? 1 : 0;
        if (!(q > (((u128)1) << 32))) ec.narrow_ok = 0;
    }
}

int accum_ternary_tc(ensi_ctx* ctx, const uint64_t* x, uint32_t d, ensi_weights* w, uint64_t* y, uint32_t level,
                     cudaStream_t st, uint64_t ctw, uint32_t limb0, int variant) {
    if (ctw == 0) ctw = (uint64_t)2 * level * ctx->n;
    if (ctw % 32) return set_err(ctx, ENSI_EINVAL, "ciphertext too small for the tensor-core tile");
    if (d != w->d) return set_err(ctx, ENSI_EDIM, "d mismatch");
    int rc = build_wt8(ctx, w);
    if (rc) return rc;
    PFN_encodeTiled enc = get_encode();
    if (!enc) return set_err(ctx, ENSI_ECUDA, "cuTensorMapEncodeTiled unavailable");
    CUtensorMap ma, mb, my;
    {   // A = W^T int8 [mpad][dpad], box 128 (K) x 128 (M)
        cuuint64_t dims[2] = {w->wt_dpad, w->wt_mpad};
        cuuint64_t strides[1] = {w->wt_dpad};
        cuuint32_t box[2] = {128, 128}, es[2] = {1, 1};
        if (enc(&ma, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void*)w->d_wt8, dims, strides, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return set_err(ctx, ENSI_ECUDA, "tensor map A");
    }
    const uint32_t pgroups = w->wt_mpad / 256;
    tc::EpiConst ec;
    fill_epi_const(ctx, w, &ec);
    const uint32_t kblocks = w->wt_dpad / 128;
    const uint32_t ntiles = (uint32_t)(ctw / 32);
    const bool ares = (size_t)kblocks * tc::kABox <= tc::kAResMax;
    typedef void (*Kern2)(CUtensorMap, CUtensorMap, CUtensorMap, uint32_t, uint32_t, uint32_t, uint32_t, uint32_t,
                          uint32_t, uint32_t, uint32_t, ModTab, tc::EpiConst, uint32_t);
    const Kern2 kmc = ares ? tc::k_accum_tc2<true, true> : tc::k_accum_tc2<false, true>;
    const Kern2 kpl = ares ? tc::k_accum_tc2<true, false> : tc::k_accum_tc2<false, false>;
    const size_t smem2 = 1024 + (ares ? (size_t)kblocks * tc::kABox : (size_t)tc::kStages2 * tc::kABox) +
                         tc::kStages2 * tc::kBStage2 + 8 * tc::kYWarp + 256;
    uint32_t cpairs = 1, nclust = 1;           // pairs per multicast cluster, co-resident clusters
    if (variant != TC_ONE_CTA) {
        // TC_AUTO / TC_PAIR_MC: the per-layer launch shape; TC_PAIR: plain pairs (no multicast)
        rc = tc_plan_clusters(ctx, pgroups, ntiles, (const void*)kmc, (const void*)kpl, smem2, tc::kThreads2,
                              variant == TC_PAIR ? 1u : 0u, &cpairs, &nclust);
        if (rc) return rc;
        variant = cpairs >= 2 ? TC_PAIR_MC : TC_PAIR;
    }
    {   // B = raw ciphertext bytes [d][ctw*8], box 128 bytes x 128 rows (x 32 rows: multicast sub-boxes)
        cuuint64_t dims[2] = {ctw * 8, d};
        cuuint64_t strides[1] = {ctw * 8};
        cuuint32_t box[2] = {128, variant == TC_PAIR_MC ? 32u : 128u}, es[2] = {1, 1};
        if (enc(&mb, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void*)x, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return set_err(ctx, ENSI_ECUDA, "tensor map B");
    }
    {   // Y = uint64 [m][ctw], box 16 words x 32 rows (SWIZZLE_128B; pair kernels: 8 words, SWIZZLE_64B)
        cuuint64_t dims[2] = {ctw, w->m};
        cuuint64_t strides[1] = {ctw * 8};
        cuuint32_t box[2] = {16u, 32}, es[2] = {1, 1};
        if (enc(&my, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, (void*)y, dims, strides, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return set_err(ctx, ENSI_ECUDA, "tensor map Y");
    }
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
    cudaError_t e;
    if (variant != TC_ONE_CTA) {
        // CTA pairs (cta_group::2) in clusters of cpairs pairs, items dealt round-robin (see k_accum_tc2)
        const uint32_t nsg = (pgroups + cpairs - 1) / cpairs;
        nclust = std::min(nclust, nsg * ntiles);
        const uint32_t tmajor = (!ares || nclust % nsg == 0) ? 1u : 0u;
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2 * cpairs;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(2 * cpairs * nclust, 1, 1);
        cfg.blockDim = dim3(tc::kThreads2, 1, 1);
        cfg.dynamicSmemBytes = smem2;
        cfg.stream = st;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        e = cudaLaunchKernelEx(&cfg, cpairs >= 2 ? kmc : kpl, ma, mb, my, kblocks, ntiles, nsg, tmajor, nclust,
                               ctx->log_n, level, limb0, ctx->tab, ec, cpairs);
        ENSI_LAUNCH_CHECK(ctx);
        if (e == cudaSuccess) e = cudaGetLastError();
        return e == cudaSuccess ? ENSI_OK : cuda_err(ctx, e, "accum_tc2 launch");
    }
    const uint32_t groups = (w->m + 127) / 128;
    uint32_t per_group = std::max<uint32_t>(1, (uint32_t)sms / groups);
    per_group = std::min(per_group, ntiles);
    const size_t a_bytes = ares ? (size_t)kblocks * tc::kABox : (size_t)tc::kStages * tc::kABox;
    const size_t smem = 1024 + a_bytes + tc::kStages * tc::kBStage + 8 * tc::kYWarp + 256;
    const uint32_t grid = groups * per_group;
    if (ares) {
        e = cudaFuncSetAttribute(tc::k_accum_tc<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e == cudaSuccess)
            tc::k_accum_tc<true><<<grid, tc::kThreads, smem, st>>>(ma, mb, my, kblocks, groups, per_group, ntiles,
                                                                   ctx->log_n, level, limb0, ctx->tab, ec);
    } else {
        e = cudaFuncSetAttribute(tc::k_accum_tc<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e == cudaSuccess)
            tc::k_accum_tc<false><<<grid, tc::kThreads, smem, st>>>(ma, mb, my, kblocks, groups, per_group, ntiles,
                                                                    ctx->log_n, level, limb0, ctx->tab, ec);
    }
    ENSI_LAUNCH_CHECK(ctx);
    if (e == cudaSuccess) e = cudaGetLastError();
    return e == cudaSuccess ? ENSI_OK : cuda_err(ctx, e, "accum_tc launch");
}

}  // namespace ensi
