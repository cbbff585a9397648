// accum_tcc.cu -- row a3 (Algorithm 1) on the tensor cores for ciphertexts stored in the COMPACT
// word layout: limb r of a polynomial is N' words of w_r = ceil(bitlen(q_r)/8) bytes,
// little-endian, limbs of poly 0 then poly 1 -- the bytes a canonical word can occupy and nothing else.
//
// Same exact byte-sliced contraction as accum_tc.cu (D[i][c] = sum_j W[j][i] byte_c(x_j), int8 x uint8 -> int32,
// y_i[w] = sum_b 2^{8b} D[i][w_r w + b] mod q), but the B operand holds only the w_r non-zero byte planes of every
// word: at the O1 primes 62 of the 96 planes of the uint64 layout (5 on each 40-bit limb, 7 on the 50-bit one), so
// the layer moves 62/96 of the HBM bytes and issues 62/96 of the MMAs.  Its outputs are compact words too.
//
// Tiles: a word tile of one (poly, limb) slice is 48 words (w = 5, N = 240 bytes), 40 (w = 6, N = 240), 32 (w = 7,
// N = 224; w = 8, N = 256); the last tile of a slice may be shorter (N' mod 48 or mod 40 words).  CTA pairs
// (cta_group::2, M = 256 outputs): each CTA holds its half of every K row of the tile (half_cols) in a 128-byte SWIZZLE_128B
// atom (a 128-byte TMA box, the few bytes past N/2 belong to the next tile and are ignored), W^T resident; clusters
// of pairs over consecutive output groups share every X sub-box by TMA multicast, as in k_accum_tc2.  Epilogue:
// the two warps of a TMEM lane quarter each drain half the tile's words (tcgen05.ld x8 pieces), recombine the
// w planes of each word (64-bit Barrett for w = 5, 128-bit otherwise), pack the canonical words back to w bytes,
// and stage one [32 outputs][N bytes] row block that a single TMA store writes.
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>

#include "tc_ptx.cuh"

namespace ensi {
namespace tcc {

using namespace tc;

static constexpr uint32_t kStages = 6;
static constexpr uint32_t kThreads = 64 + 8 * 32;      // producer, MMA issuer, 8 epilogue warps
static constexpr uint32_t kBoxK = 128;                  // K rows per stage
static constexpr uint32_t kABox = 128 * 128;            // 16 KB: 128 outputs x 128 K (W^T, K-major)
static constexpr uint32_t kBStage = 128 * 128;          // 16 KB: 128 K rows x one 128-byte atom (this CTA's N half)
static constexpr uint32_t kYQuarter = 32 * 256;         // staging per TMEM lane quarter: 32 outputs x <= 256 bytes
static constexpr uint32_t kAResMax = 96 * 1024;
static constexpr uint32_t kMaxSlices = 96;
static constexpr uint32_t kMaxMaps = 8;

// Tile table (kernel-parameter bank): slice s = (poly, limb) of a ciphertext (or the one staged slice).
struct Tiles {
    uint32_t nslices, words;                  // slices; words per slice (N')
    uint32_t tile0[kMaxSlices + 1];           // first tile of slice s; tile0[nslices] = tiles per ciphertext
    uint32_t byte0[kMaxSlices];               // byte offset of slice s inside a ciphertext
    uint8_t wb[kMaxSlices], limb[kMaxSlices], wpt[kMaxSlices], map_full[kMaxSlices], map_tail[kMaxSlices];
};
static constexpr uint32_t kMaxPeers = 8;
struct StoreMaps {
    // Y store maps [destination][tile width N] (box {N, 32}).  One destination: the output buffer.  Several (the fused
    // gather epilogue): every GPU's gathered buffer, this rank's rows of it (row0 * ct bytes on)
    CUtensorMap m[kMaxPeers][kMaxMaps];
    uint32_t n_dst;
};

struct TileInfo {
    uint32_t byte, n, nw, wb, limb, map;
};
// t must not decrease between calls with the same s (every role walks its tiles in increasing order)
__device__ __forceinline__ TileInfo tile_info(const Tiles& tl, uint32_t t, uint32_t& s) {
    while (t >= tl.tile0[s + 1]) s++;
    const uint32_t wpt = tl.wpt[s], wb = tl.wb[s];
    const uint32_t w0 = (t - tl.tile0[s]) * wpt;
    const uint32_t nw = min(wpt, tl.words - w0);
    TileInfo ti;
    ti.byte = tl.byte0[s] + w0 * wb;
    ti.nw = nw;
    ti.wb = wb;
    ti.n = nw * wb;
    ti.limb = tl.limb[s];
    ti.map = nw == wpt ? tl.map_full[s] : tl.map_tail[s];
    return ti;
}

// Tile halves.  A tile of n = 2 hb bytes is split between the pair: CTA 0 loads its 128-byte box from the tile's
// first byte, CTA 1 from byte (hb & ~15) -- TMA box starts stay 16-byte aligned (hb = 120 or 40 at w = 5, 120 / 72
// / 24 at w = 6 are not; a misaligned start is an illegal instruction on sm_100a, measured).  The MMA takes P
// columns from each CTA (N = 2P, P a multiple of 16 as cta_group::2 needs): CTA 0's bytes [0, hb) are columns
// [0, hb), CTA 1's bytes [hb, n) are columns [P + (hb & 15), P + (hb & 15) + hb).  Columns outside those hold
// neighbouring bytes (or TMA zero fill) that the epilogue never reads.
__host__ __device__ constexpr uint32_t half_cols(uint32_t hb) { return (hb + (hb & 15) + 15) & ~15u; }
__host__ __device__ constexpr uint32_t half1_col(uint32_t hb) { return half_cols(hb) + (hb & 15); }

#define TMEM_LD_X8(taddr, r)                                                                                        \
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"                         \
                 : "=r"((r)[0]), "=r"((r)[1]), "=r"((r)[2]), "=r"((r)[3]), "=r"((r)[4]), "=r"((r)[5]),              \
                   "=r"((r)[6]), "=r"((r)[7])                                                                        \
                 : "r"(taddr))

// 128-bit recombination of W >= 6 byte planes (|D_b| < 2^31), canonical result.
template <uint32_t W>
__device__ __forceinline__ uint64_t combine_w(const uint32_t* r, const Barrett& br, uint64_t off_lo, uint64_t off_hi) {
    int64_t lo = (int64_t)(int32_t)r[0] + (int64_t)(int32_t)r[1] * 256 + (int64_t)(int32_t)r[2] * 65536 +
                 (int64_t)(int32_t)r[3] * 16777216;
    int64_t hi = (int64_t)(int32_t)r[4];
    if (W > 5) hi += (int64_t)(int32_t)r[5] * 256;
    if (W > 6) hi += (int64_t)(int32_t)r[6] * 65536;
    if (W > 7) hi += (int64_t)(int32_t)r[7] * 16777216;
    const uint64_t v_lo = (uint64_t)lo + ((uint64_t)hi << 32);
    const uint64_t carry = v_lo < (uint64_t)lo ? 1 : 0;
    const int64_t v_hi = (hi >> 32) + (lo >> 63) + (int64_t)carry;
    const uint64_t x_lo = v_lo + off_lo;
    const uint64_t x_hi = (uint64_t)v_hi + off_hi + (x_lo < v_lo ? 1 : 0);
    return barrett128(x_hi, x_lo, br);
}

struct EpiArgs {
    Barrett br;
    uint64_t off_lo, off_hi, off64;
    uint32_t mu32;
};

// CW words (W bytes each) of one output row from their TMEM planes r[0, CW W) -> canonical words, packed into
// CW W / 8 little-endian u64 and written to the staging row at dst.
template <uint32_t W, uint32_t CW>
__device__ __forceinline__ void epi_chunk(const uint32_t* r, const EpiArgs& ea, uint8_t* dst) {
    static_assert((CW * W) % 8 == 0, "a chunk ends on a u64");
    uint64_t u[CW * W / 8];
#pragma unroll
    for (uint32_t j = 0; j < CW * W / 8; j++) u[j] = 0;
#pragma unroll
    for (uint32_t i = 0; i < CW; i++) {
        uint64_t v;
#ifdef ENSI_ABL_NOCOMBINE   // timing-only ablation build (wrong words; profiles/r02_tcc_ablations.md)
        v = r[W * i];
#else
        if constexpr (W == 5) v = combine_word5(r + 5 * i, ea.br.q, ea.mu32, ea.off64);
        else v = combine_w<W>(r + W * i, ea.br, ea.off_lo, ea.off_hi);
#endif
        constexpr uint32_t bits = 8 * W;
        const uint32_t bit = i * bits, j = bit / 64, sh = bit % 64;
        u[j] |= v << sh;
        if (sh + bits > 64) u[j + 1] |= v >> (64 - sh);
    }
#pragma unroll
    for (uint32_t j = 0; j < CW * W / 8; j++)
        asm volatile("st.shared.u64 [%0], %1;" ::"r"(smem_u32(dst + 8 * j)), "l"(u[j]) : "memory");
}

// The whole epilogue of one tile for a warp (quarter q, half h): drain this warp's HW words (W TMEM columns each) and
// hand the accumulator back, then both warps of the quarter stage their halves of one [32][N] row block -- in chunks
// of 8 words, each written as soon as it is combined (staging everything after the last combine measured 2-7 %
// slower: the burst of shared-memory writes stalls the MMA operand reads) -- and the half-0 warp issues the TMA store.
template <uint32_t W, uint32_t HW>
__device__ __forceinline__ void epi_tile(uint32_t tbase_q, uint32_t release_addr, uint32_t lane, uint32_t half,
                                         uint32_t quarter, uint8_t* ys, const EpiArgs& ea, const CUtensorMap* map,
                                         uint32_t byte, uint32_t row0, uint32_t n_dst) {
    constexpr uint32_t NB = W * HW;             // bytes (and TMEM columns) of this warp's half row segment
    constexpr uint32_t CH = 8;                  // words per staged chunk
    static_assert(NB % 8 == 0, "TMEM pieces are 8 columns");
#ifdef ENSI_ABL_NOEPI       // timing-only ablation build (no outputs): release the accumulator at once
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive_remote(release_addr);
    return;
#endif
    uint32_t r[NB];
#pragma unroll
    for (uint32_t c = 0; c < NB; c += 8) TMEM_LD_X8(tbase_q + half * half1_col(NB) + c, r + c);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive_remote(release_addr);
    // staging free: the previous TMA store of this quarter has read it
    if (half == 0 && lane == 0) tma_store_wait_read0();
    asm volatile("bar.sync %0, 64;" ::"r"(1 + quarter) : "memory");
    uint8_t* dst = ys + lane * (2 * NB) + half * NB;
#pragma unroll
    for (uint32_t c0 = 0; c0 < HW; c0 += CH) {
        if constexpr (HW % CH == 0) {
            epi_chunk<W, CH>(r + W * c0, ea, dst + W * c0);
        } else {
            if (c0 + CH <= HW) epi_chunk<W, CH>(r + W * c0, ea, dst + W * c0);
            else epi_chunk<W, (HW % CH)>(r + W * c0, ea, dst + W * c0);
        }
    }
    fence_proxy_async();
    asm volatile("bar.sync %0, 64;" ::"r"(1 + quarter) : "memory");
    if (half == 0 && lane == 0) {
        for (uint32_t dd = 0; dd < n_dst; dd++) tma_store_2d(map + dd * kMaxMaps, ys, (int32_t)byte, (int32_t)row0);
        tma_store_commit();
    }
}

template <bool A_RES, bool MC>
__global__ void __launch_bounds__(kThreads, 1)
    k_accum_tcc(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                const __grid_constant__ StoreMaps maps, const __grid_constant__ Tiles tl, uint32_t kblocks,
                uint32_t ntiles, uint32_t nsg, uint32_t tmajor, uint32_t nclust, ModTab tab, tc::EpiConst ec,
                uint32_t cpairs) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    const uint32_t a_bytes = A_RES ? kblocks * kABox : kStages * kABox;
    uint8_t* sA = smem;
    uint8_t* sB = sA + a_bytes;
    uint8_t* sY = sB + kStages * kBStage;
    uint64_t* bars = (uint64_t*)(sY + 4 * kYQuarter);
    uint64_t* full = bars;                     // [kStages]  (leader's are the live ones)
    uint64_t* empty = bars + kStages;          // [kStages]  (per CTA, multicast commits)
    uint64_t* tfull = bars + 2 * kStages;      // [2]        (per CTA, multicast commits)
    uint64_t* tempty = tfull + 2;              // [2]        (leader's: 16 arrivals)
    uint64_t* afull = tempty + 2;              // [1]        (leader's)
    uint64_t* adone = afull + 1;               // [1]        (per CTA: the MMAs reading the resident A completed)
    uint32_t* tmem_slot = (uint32_t*)(adone + 1);

    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t crank = cluster_rank();
    const uint32_t rank = crank & 1;
    const uint32_t lead = crank & ~1u;
    // Work items (super-group sg, word tile t): super-group sg = the cpairs consecutive pair groups
    // [sg cpairs, (sg + 1) cpairs) of 256 outputs each (one per pair of the cluster; groups past the padded W^T are
    // TMA zero fill, their stores clipped).  Cluster kc takes items kc, kc + K, kc + 2K, ... of the list ordered
    // tile-major (tmajor: item = t nsg + sg -- every super-group's clusters read the same X tiles at about the same
    // time, so each is fetched from DRAM once; a resident W^T needs K to be a multiple of nsg) or super-group-major
    // (item = sg ntiles + t: a cluster's super-group changes at most nsg - 1 times, its resident W^T reloaded then).
    // Either way the K clusters of a round take K consecutive items: neighbouring tiles, DRAM-page friendly.
    const uint32_t pin = crank >> 1;
    const uint32_t kc = blockIdx.x / (2 * cpairs);
    auto grp = [&](uint32_t sg) -> uint32_t { return (sg * cpairs + pin) * 2 + rank; };   // 128-row block
    const uint16_t pair_mask = (uint16_t)(0x3u << lead);
    const uint16_t all_mask = MC ? (uint16_t)((1u << (2 * cpairs)) - 1) : pair_mask;

    if (threadIdx.x == 0) {
        for (uint32_t s = 0; s < kStages; s++) {
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
            uint32_t s = 0, ph = 0, sl = 0, cur = ~0u, adph = 0;
            for (WorkIter wi(kc, nclust, nsg, ntiles, tmajor); wi.valid(); wi.next()) {
                const uint32_t sg = wi.sg, t = wi.t;
                const uint32_t g = grp(sg);
                if (sg != cur) {
                    if (!tmajor) sl = 0;
                    if (A_RES) {
                        if (cur != ~0u) {       // every MMA on the previous W^T has completed (MMA issuer's commit)
                            mbar_wait(adone, adph);
                            adph ^= 1;
                        }
                        if (rank == 0) mbar_expect_tx(afull, 2 * kblocks * kABox);
                        for (uint32_t kb = 0; kb < kblocks; kb++)
                            tma_load_2d_2sm(sA + kb * kABox, &map_a, afull, (int32_t)(kb * kBoxK), (int32_t)(g * 128));
                    }
                    cur = sg;
                }
                const TileInfo ti = tile_info(tl, t, sl);
                const int32_t x0 = (int32_t)(ti.byte + rank * ((ti.n >> 1) & ~15u));   // this CTA's half (half_cols)
                for (uint32_t kb = 0; kb < kblocks; kb++) {
                    mbar_wait(&empty[s], ph ^ 1);
                    if (rank == 0) mbar_expect_tx(&full[s], 2 * (kBStage + (A_RES ? 0 : kABox)));
                    if (MC) {
                        const uint16_t half_mask = (uint16_t)(all_mask & (rank ? 0xAAAAu : 0x5555u));
                        for (uint32_t j = lead >> 1; j < kBoxK / 32; j += cpairs)
                            tma_load_2d_2sm_mc(sB + s * kBStage + j * 4096, &map_b, &full[s], half_mask, x0,
                                               (int32_t)(kb * kBoxK + j * 32));
                    } else {
                        tma_load_2d_2sm(sB + s * kBStage, &map_b, &full[s], x0, (int32_t)(kb * kBoxK));
                    }
                    if (!A_RES)
                        tma_load_2d_2sm(sA + s * kABox, &map_a, &full[s], (int32_t)(kb * kBoxK), (int32_t)(g * 128));
                    if (++s == kStages) {
                        s = 0;
                        ph ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------------ MMA issuer (leader CTA only)
        if (rank == 0) {
            const uint64_t adesc0 = umma_desc(smem_u32(sA), 16, 1024);
            const uint64_t bdesc0 = umma_desc(smem_u32(sB), kBStage, 1024);
            uint32_t s = 0, ph = 0, sl = 0, cur = ~0u, aph = 0, j = 0;
            for (WorkIter wi(kc, nclust, nsg, ntiles, tmajor); wi.valid(); wi.next(), j++) {
                const uint32_t sg = wi.sg, t = wi.t;
                if (sg != cur) {
                    if (!tmajor) sl = 0;
                    if (A_RES) {
                        if (cur != ~0u) {       // release the resident W^T once the MMAs issued on it complete
                            if (elect_one()) mma_commit_2sm_mc(adone, pair_mask);
                            __syncwarp();
                        }
                        mbar_wait(afull, aph);
                        aph ^= 1;
                        tc_fence_after();
                    }
                    cur = sg;
                }
                const TileInfo ti = tile_info(tl, t, sl);
                const uint32_t idesc = idesc_i8(256, 2 * half_cols(ti.n >> 1));   // see half_cols
                const uint32_t acc = j & 1, use = j >> 1;
                mbar_wait(&tempty[acc], (use & 1) ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * 256;
                for (uint32_t kb = 0; kb < kblocks; kb++) {
                    mbar_wait(&full[s], ph);
                    tc_fence_after();
                    const uint64_t ad = adesc0 + (uint64_t)(((A_RES ? kb : s) * kABox) >> 4);
                    const uint64_t bd = bdesc0 + (uint64_t)((s * kBStage) >> 4);
                    if (elect_one()) {
#pragma unroll
                        for (uint32_t kk = 0; kk < kBoxK / 32; kk++)
                            mma_i8_2sm(d_tmem, ad + 2 * kk, bd + 256 * kk, idesc, (kb | kk) != 0);
                        mma_commit_2sm_mc(&empty[s], all_mask);
                    }
                    __syncwarp();
                    if (++s == kStages) {
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
        const uint32_t e = warp - 2;
        const uint32_t quarter = warp & 3;
        const uint32_t half = e >> 2;
        uint8_t* ys = sY + quarter * kYQuarter;
        const uint32_t tempty_leader0 = mapa_rank(smem_u32(&tempty[0]), lead);
        uint32_t sl = 0, cur = ~0u, j = 0;
        for (WorkIter wi(kc, nclust, nsg, ntiles, tmajor); wi.valid(); wi.next(), j++) {
            const uint32_t sg = wi.sg, t = wi.t;
            if (sg != cur && !tmajor) sl = 0;
            cur = sg;
            const uint32_t g = grp(sg);
            const TileInfo ti = tile_info(tl, t, sl);
            const uint32_t acc = j & 1, use = j >> 1;
            EpiArgs ea;
            ea.br = tab.br(ti.limb);
            ea.off_lo = ec.off_lo[ti.limb];
            ea.off_hi = ec.off_hi[ti.limb];
            ea.off64 = ec.off64[ti.limb];
            ea.mu32 = ec.mu32[ti.limb];
            const CUtensorMap* map = &maps.m[0][ti.map];
            const uint32_t row0 = g * 128 + quarter * 32;
            const uint32_t tq = tmem_base + ((quarter * 32) << 16) + acc * 256;
            const uint32_t rel = tempty_leader0 + acc * 8;
            mbar_wait(&tfull[acc], use & 1);
            tc_fence_after();
            switch (ti.wb * 64 + ti.nw / 2) {
                // full tiles: 48 / 40 / 32 / 32 words; tails: N' mod 48 (16, 32) and N' mod 40 (8, 16, 24, 32)
                case 5 * 64 + 24: epi_tile<5, 24>(tq, rel, lane, half, quarter, ys, ea, map, ti.byte, row0, maps.n_dst); break;
                case 5 * 64 + 8: epi_tile<5, 8>(tq, rel, lane, half, quarter, ys, ea, map, ti.byte, row0, maps.n_dst); break;
                case 5 * 64 + 16: epi_tile<5, 16>(tq, rel, lane, half, quarter, ys, ea, map, ti.byte, row0, maps.n_dst); break;
                case 6 * 64 + 20: epi_tile<6, 20>(tq, rel, lane, half, quarter, ys, ea, map, ti.byte, row0, maps.n_dst); break;
                case 6 * 64 + 4: epi_tile<6, 4>(tq, rel, lane, half, quarter, ys, ea, map, ti.byte, row0, maps.n_dst); break;
                case 6 * 64 + 8: epi_tile<6, 8>(tq, rel, lane, half, quarter, ys, ea, map, ti.byte, row0, maps.n_dst); break;
                case 6 * 64 + 12: epi_tile<6, 12>(tq, rel, lane, half, quarter, ys, ea, map, ti.byte, row0, maps.n_dst); break;
                case 6 * 64 + 16: epi_tile<6, 16>(tq, rel, lane, half, quarter, ys, ea, map, ti.byte, row0, maps.n_dst); break;
                case 7 * 64 + 16: epi_tile<7, 16>(tq, rel, lane, half, quarter, ys, ea, map, ti.byte, row0, maps.n_dst); break;
                default: epi_tile<8, 16>(tq, rel, lane, half, quarter, ys, ea, map, ti.byte, row0, maps.n_dst); break;
            }
        }
        if (half == 0 && lane == 0) tma_store_wait0();
    }
    tc_fence_before();
    cluster_sync_all();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
    }
}

}  // namespace tcc

// ---------------------------------------------------------------------------------------------- host side

uint32_t compact_word_bytes(const ensi_ctx* ctx, uint32_t limb) {
    uint32_t b = 0;
    while (b < 64 && (ctx->mod[limb] >> b)) b++;
    return (b + 7) / 8;
}

// words per full tile for a w-byte word (N = words * w <= 256, a multiple of 16)
static uint32_t words_per_tile(uint32_t wb) { return wb == 5 ? 48 : wb == 6 ? 40 : 32; }

bool tcc_supported(const ensi_ctx* ctx, uint32_t level) {
    if (!tc_supported(ctx, level)) return false;            // sm_100a, 2^32 < q < 2^60 (w in 5..8)
    if (ctx->n < 256) return false;
    for (uint32_t r = 0; r < level; r++) {
        const uint32_t wb = compact_word_bytes(ctx, r), tail = ctx->n % words_per_tile(wb);
        if (wb < 5 || wb > 8) return false;
        if (tail && !((wb == 5 && (tail == 16 || tail == 32)) || (wb == 6 && tail % 8 == 0))) return false;
    }
    return true;
}

typedef CUresult (*PFN_encodeTiledC)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                     const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                     CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiledC get_encode_c() {
    static PFN_encodeTiledC fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_encodeTiledC)p;
    }
    return fn;
}

namespace tcc {
typedef void (*KernFn)(CUtensorMap, CUtensorMap, StoreMaps, Tiles, uint32_t, uint32_t, uint32_t, uint32_t, uint32_t,
                       ModTab, tc::EpiConst, uint32_t);

// Relative per-SM rate of a cluster of c pairs sharing every X sub-box by multicast (c = 1: plain pairs, each
// X tile read through L2 by every pair) -- measured at 2048x2048 with every c forced (tools/bench_cluster.py,
// profiles/r02_tcc_ablations.md).
static constexpr double kFeed[9] = {0, 0.52, 0.85, 0.90, 1.0, 1.0, 1.0, 1.0, 1.0};

// Co-resident clusters of c pairs (cudaOccupancyMaxActiveClusters; cached per device, kernel and smem size).
static int max_clusters(int dev, const void* k, size_t smem, uint32_t threads, uint32_t c) {
    static std::mutex mu;
    static std::map<std::tuple<int, const void*, size_t, uint32_t>, int> cache;
    const auto key = std::make_tuple(dev, k, smem, c);
    {
        std::lock_guard<std::mutex> g(mu);
        auto it = cache.find(key);
        if (it != cache.end()) return it->second;
    }
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2 * c;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(2 * c * 64, 1, 1);
    cfg.blockDim = dim3(threads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, (void*)k, &cfg) != cudaSuccess) {
        cudaGetLastError();
        n = 0;
    }
    std::lock_guard<std::mutex> g(mu);
    cache[key] = n;
    return n;
}

}  // namespace tcc

// Cluster shape: c pairs per cluster (2c CTAs, c <= 8) and K co-resident clusters, minimising the estimated time
// ceil(I_c / K_c) / kFeed[c] with I_c = ceil(pgroups / c) word-tile items (a super-group that overhangs the padded
// W^T computes zero rows); force = 1..8 takes that c (ensi_pcmm_opts.cluster_pairs).  Shared by the compact
// (k_accum_tcc) and the uint64-word (k_accum_tc2) pair kernels: kmc / kpl are the multicast / plain-pair variants.

int tc_plan_clusters(ensi_ctx* ctx, uint32_t pgroups, uint32_t ntiles, const void* kmc, const void* kpl, size_t smem,
                     uint32_t threads, uint32_t force, uint32_t* cpairs, uint32_t* nclust) {
    for (const void* k : {kmc, kpl}) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return cuda_err(ctx, e, "accumulate smem attribute");
    }
    // clusters of up to 16 CTAs (8 pairs) are a non-portable size
    const bool big = cudaFuncSetAttribute(kmc, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess;
    if (!big) cudaGetLastError();
    const uint32_t cmax = big ? 8 : 4;
    if (force > cmax) return set_err(ctx, ENSI_EINVAL, "cluster_pairs larger than this device allows");
    double best = 0;
    for (uint32_t c = force ? force : 1; c <= (force ? force : cmax); c++) {
        const int kc = tcc::max_clusters(ctx->device, c == 1 ? kpl : kmc, smem, threads, c);
        if (kc < 1) continue;
        const uint64_t items = (uint64_t)((pgroups + c - 1) / c) * ntiles;
        const double est = (double)((items + kc - 1) / kc) / tcc::kFeed[c];
        if (best == 0 || est < best * 0.999) {
            best = est;
            *cpairs = c;
            *nclust = (uint32_t)kc;
        }
    }
    if (best == 0) return set_err(ctx, ENSI_ECUDA, "tensor-core accumulate: no cluster shape fits on this device");
    return ENSI_OK;
}

int build_wt8(ensi_ctx* ctx, ensi_weights* w);
void fill_epi_const(const ensi_ctx* ctx, const ensi_weights* w, tc::EpiConst* ec);

// x: d compact ciphertexts of ct_bytes each; y: m of them.  A whole ciphertext (slice_limb < 0: 2 level slices)
// or one staged (poly, limb) slice of every ciphertext (slice_limb = r: ct_bytes = N' w_r).
// y_dst[0..n_dst): output buffers, each [m][ct_bytes] from its pointer on (one for the plain call; every GPU's
// gathered buffer, offset to this rank's rows, for the fused gather epilogue) -- every tile is TMA-stored to each.
int accum_ternary_tcc_dst(ensi_ctx* ctx, const uint8_t* x, uint32_t d, ensi_weights* w, uint8_t* const* y_dst,
                          uint32_t n_dst, uint32_t level, cudaStream_t st, int slice_limb, uint32_t cluster_pairs) {
    if (n_dst < 1 || n_dst > tcc::kMaxPeers) return set_err(ctx, ENSI_EINVAL, "1..8 output destinations");
    if (d != w->d) return set_err(ctx, ENSI_EDIM, "d mismatch");
    if (!tcc_supported(ctx, level)) return set_err(ctx, ENSI_EINVAL, "compact tensor-core accumulate unavailable");
    int rc = build_wt8(ctx, w);
    if (rc) return rc;
    PFN_encodeTiledC enc = get_encode_c();
    if (!enc) return set_err(ctx, ENSI_ECUDA, "cuTensorMapEncodeTiled unavailable");
    tcc::Tiles tl{};
    tl.words = ctx->n;
    tl.nslices = slice_limb < 0 ? 2 * level : 1;
    uint32_t ns[tcc::kMaxMaps] = {}, nmaps = 0;
    auto map_of = [&](uint32_t nbytes) -> int {
        for (uint32_t i = 0; i < nmaps; i++)
            if (ns[i] == nbytes) return (int)i;
        if (nmaps == tcc::kMaxMaps) return -1;
        ns[nmaps] = nbytes;
        return (int)nmaps++;
    };
    uint64_t off = 0, tiles = 0;
    for (uint32_t s = 0; s < tl.nslices; s++) {
        const uint32_t limb = slice_limb < 0 ? s % level : (uint32_t)slice_limb;
        const uint32_t wb = compact_word_bytes(ctx, limb), wpt = words_per_tile(wb);
        const uint32_t tail = ctx->n % wpt;
        const int mf = map_of(wpt * wb), mt = tail ? map_of(tail * wb) : mf;
        if (mf < 0 || mt < 0) return set_err(ctx, ENSI_EINVAL, "too many distinct compact tile widths");
        tl.tile0[s] = (uint32_t)tiles;
        tl.byte0[s] = (uint32_t)off;
        tl.wb[s] = (uint8_t)wb;
        tl.limb[s] = (uint8_t)limb;
        tl.wpt[s] = (uint8_t)wpt;
        tl.map_full[s] = (uint8_t)mf;
        tl.map_tail[s] = (uint8_t)mt;
        tiles += (ctx->n + wpt - 1) / wpt;
        off += (uint64_t)ctx->n * wb;
    }
    tl.tile0[tl.nslices] = (uint32_t)tiles;
    const uint64_t ct_bytes = off;
    if (ct_bytes >= (1ull << 32)) return set_err(ctx, ENSI_EINVAL, "ciphertext too large for the compact tile table");
    CUtensorMap ma, mb;
    tcc::StoreMaps maps;
    std::memset(&maps, 0, sizeof(maps));
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
    if (!ec.narrow_ok) return set_err(ctx, ENSI_EINVAL, "d too large for the compact tensor-core epilogue");
    const uint32_t kblocks = w->wt_dpad / 128;
    const bool ares = (size_t)kblocks * tcc::kABox <= tcc::kAResMax;
    const size_t a_bytes = ares ? (size_t)kblocks * tcc::kABox : (size_t)tcc::kStages * tcc::kABox;
    const size_t smem = 1024 + a_bytes + tcc::kStages * tcc::kBStage + 4 * tcc::kYQuarter + 256;
    const uint32_t ntiles = (uint32_t)tiles;
    tcc::KernFn kmc = ares ? tcc::k_accum_tcc<true, true> : tcc::k_accum_tcc<false, true>;
    tcc::KernFn kpl = ares ? tcc::k_accum_tcc<true, false> : tcc::k_accum_tcc<false, false>;
    uint32_t cpairs = 1, nclust = 1;
    rc = tc_plan_clusters(ctx, pgroups, ntiles, (const void*)kmc, (const void*)kpl, smem, tcc::kThreads, cluster_pairs,
                          &cpairs, &nclust);
    if (rc) return rc;
    const bool mc = cpairs >= 2;
    const tcc::KernFn kern = mc ? kmc : kpl;
    {   // B = compact ciphertext bytes [d][ct_bytes], box 128 bytes x 32 (multicast sub-boxes) or 128 rows
        cuuint64_t dims[2] = {ct_bytes, d};
        cuuint64_t strides[1] = {ct_bytes};
        cuuint32_t box[2] = {128, mc ? 32u : 128u}, es[2] = {1, 1};
        if (enc(&mb, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void*)x, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return set_err(ctx, ENSI_ECUDA, "tensor map B (compact)");
    }
    maps.n_dst = n_dst;
    for (uint32_t dd = 0; dd < n_dst; dd++)
        for (uint32_t i = 0; i < nmaps; i++) {   // Y = [m][ct_bytes], box {N, 32}, no swizzle (packed staging rows)
            cuuint64_t dims[2] = {ct_bytes, w->m};
            cuuint64_t strides[1] = {ct_bytes};
            cuuint32_t box[2] = {ns[i], 32}, es[2] = {1, 1};
            if (enc(&maps.m[dd][i], CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void*)y_dst[dd], dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
                return set_err(ctx, ENSI_ECUDA, "tensor map Y (compact)");
        }
    const uint32_t nsg = (pgroups + cpairs - 1) / cpairs;
    nclust = std::min(nclust, nsg * ntiles);
    // tile-major unless a resident W^T would be reloaded at every item (K not a multiple of the super-groups)
    const uint32_t tmajor = (!ares || nclust % nsg == 0) ? 1u : 0u;
    ctx->tcc_cpairs = cpairs;
    ctx->tcc_nclust = nclust;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2 * cpairs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(2 * cpairs * nclust, 1, 1);
    cfg.blockDim = dim3(tcc::kThreads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, ma, mb, maps, tl, kblocks, ntiles, nsg, tmajor, nclust, ctx->tab,
                                       ec, cpairs);
    ENSI_LAUNCH_CHECK(ctx);
    if (e == cudaSuccess) e = cudaGetLastError();
    return e == cudaSuccess ? ENSI_OK : cuda_err(ctx, e, "accum_tcc launch");
}

int accum_ternary_tcc(ensi_ctx* ctx, const uint8_t* x, uint32_t d, ensi_weights* w, uint8_t* y, uint32_t level,
                      cudaStream_t st, int slice_limb, uint32_t cluster_pairs) {
    uint8_t* dst[1] = {y};
    return accum_ternary_tcc_dst(ctx, x, d, w, dst, 1, level, st, slice_limb, cluster_pairs);
}

// ---------------------------------------------------------------------------------------------- peer signalling
// After the fused gather epilogue every rank's output rows have been TMA-stored into every GPU's gathered buffer.
// k_peer_signal (stream-ordered after that kernel, so its stores are complete) makes them visible system-wide and
// publishes `epoch` in slot `slot` of every destination's flag array; k_peer_wait spins until all n flags of this
// GPU's array reached `epoch` (release / acquire at system scope: the flags may live in another GPU's memory).
__global__ void k_peer_signal(PeerFlags pf, uint32_t slot, uint32_t epoch) {
    const uint32_t p = threadIdx.x;
    if (p < pf.n) {
        __threadfence_system();
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(pf.f[p] + slot), "r"(epoch) : "memory");
    }
}
__global__ void k_peer_wait(const uint32_t* flags, uint32_t n, uint32_t epoch) {
    const uint32_t p = threadIdx.x;
    if (p < n) {
        uint32_t v;
        // bounded: a peer that never signals (a crashed rank) faults this context after ~30 s instead of hanging
        // the GPU forever
        const long long t0 = clock64();
        for (;;) {
            asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + p) : "memory");
            if ((int32_t)(v - epoch) >= 0) break;
            __nanosleep(200);
            if (clock64() - t0 > 60000000000ll) __trap();
        }
    }
    __syncthreads();
}

}  // namespace ensi
