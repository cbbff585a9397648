// ntt_fp.cuh -- N' = 2^16 negacyclic NTT passes with the modular arithmetic on the FP64 pipe (sm_100a).
//
// Why: the integer Shoup butterfly costs ~32 instructions (a 64x64 high product is ~8 IMADs on the 32-bit integer
// multiplier) and the v2 kernel is integer-issue bound (profiles/r01_ncu_ntt_keyswitch.md).  B200 keeps a full
// FP64 unit (64 DFMA/SM/clk, half the FP32 rate), and for moduli q < 2^50 every word, twiddle and remainder is an
// integer below 2^53, i.e. an exact double.  A butterfly becomes 8 DP instructions, measured 2.4x the integer
// butterfly throughput in registers (tools/mb_modmul.cu).
//
// Exact modular product (centred residues, all values are integers held in doubles):
//   h = V*w,  l = fma(V, w, -h)                 (h + l == V*w exactly: TwoProduct)
//   t = fma(V, wq, M) - M,   wq = RN(w / q), M = 1.5*2^52    (t = rint(V*wq): the add to M rounds to an integer
//                                                             while |V*wq| < 2^51)
//   r = fma(-t, q, h) + l                        (= V*w - t*q exactly: h - t*q is an integer < 2^53 because
//                                                 ulp(h) <= 2^49 when |V*w| < 2^101)
//   |V*w/q - t| <= 1/2 + |V| 2^-55   ->   |r| <= 0.625 q   for |V| < 2^52.
// Bounds (b = max |value| / q): CT (forward) outputs U +- r grow by 0.625 per stage; GS (inverse) sums U + V
// double per stage.  Preconditions of the product: |V| < 2^52 and every sum < 2^53.
//  * narrow limbs (q < 2^41, bmax = 2^52/q >= 2048): forward runs both passes unreduced (b <= 1 + 16*0.625 = 11);
//    inverse reduces the sums every 4 stages (b <= 16).
//  * wide limbs (2^41 <= q < 2^50, bmax > 4): forward reduces every 4 stages (b <= 1 + 4*0.625 = 3.5); inverse
//    centres its input and reduces the sums every 2 stages (product inputs b <= 2.5).
// Centred reduction red(v) = v - rint(v/q) q (3 DP), |red(v)| <= q/2 + tiny.  The last store maps the centred
// result to the canonical word in [0, q), so the output is bit-identical to the integer kernels (and the oracle).
// The pass-A -> pass-B intermediate is stored as the double's bit pattern (private to the two launches).
#pragma once
#include <cuda.h>

#include "ensi_internal.h"

namespace ensi {
#ifndef ENSI_NTTFP_MINB
#define ENSI_NTTFP_MINB 4
#endif
namespace nttfp {

enum Pass { FWD_A = 0, FWD_B = 1, INV_B = 2, INV_A = 3 };
static constexpr uint32_t kRow = 273;          // smem row stride (words): 256 + 16 pads + 1 -> conflict-free
static constexpr double kM = 6755399441055744.0;   // 1.5 * 2^52
static constexpr long long kMbits = 0x4338000000000000ll;

__device__ __forceinline__ uint32_t sidx(uint32_t sp, uint32_t i) { return sp * kRow + i + (i >> 4); }

// signed integer |x| < 2^51 <-> double, through the 1.5*2^52 binade (one integer add + one DADD)
__device__ __forceinline__ double i2d(long long x) { return __longlong_as_double(kMbits + x) - kM; }
__device__ __forceinline__ long long d2i(double v) { return __double_as_longlong(v + kM) - kMbits; }
// centred integer-valued double (|v| < q) -> canonical word in [0, q)
__device__ __forceinline__ uint64_t canon(double v, uint64_t q) {
    long long x = d2i(v);
    return (uint64_t)(x + ((x >> 63) & (long long)q));
}
__device__ __forceinline__ double red(double v, double q, double qinv) {
    const double t = fma(v, qinv, kM) - kM;
    return fma(-t, q, v);
}
__device__ __forceinline__ double mulmod(double V, double w, double wq, double q) {
    const double h = V * w;
    const double l = fma(V, w, -h);
    const double t = fma(V, wq, kM) - kM;
    return fma(-t, q, h) + l;
}

struct PlainIn {
    __device__ __forceinline__ uint64_t load(const uint64_t* a, uint32_t, uint32_t, uint32_t k) const { return a[k]; }
};
struct PlainOut {
    static constexpr bool kFused = false;   // true: the TMA block pass hands every word to store() (lane-consecutive)
    __device__ __forceinline__ void store(uint64_t* a, uint32_t, uint32_t, uint32_t k, uint64_t v) const { a[k] = v; }
};

// tw: [limb][fwd/inv][N'] of (w centred, RN(w/q)) as double2, then [limb] of (n^-1 centred, RN(n^-1/q)).
// Lane-transposed region: for the block-pass stages with local stride 2^lt <= 8 (table indices >= 4096), each
// (stage, block) run of 128 >> lt twiddles is stored as [j][tt] instead of [tt][j] (tt < 16, j < 8 >> lt), so the
// 16 lanes that need entry j of their own tt read 16 consecutive entries (was one 128-byte line per lane).
// Same CTA geometry as the integer v2 passes (ntt_v2.cuh): 16 sub-problems of 256 points, 16 points per thread.
// ---- TMA helpers for the block passes (tile = 16 consecutive 256-point blocks = 32 KB, SWIZZLE_128B)
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void tile_load(void* dst, const CUtensorMap* map, uint64_t* bar, int32_t c1, int32_t c2) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(32768u) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::
            "r"(su32(dst)),
        "l"((uint64_t)map), "r"(su32(bar)), "r"(0), "r"(c1), "r"(c2)
        : "memory");
}
__device__ __forceinline__ void tile_wait(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}" ::"r"(su32(bar)),
        "r"(0u)
        : "memory");
}
__device__ __forceinline__ void tile_store(const CUtensorMap* map, const void* src, int32_t c1, int32_t c2) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"((uint64_t)map),
                 "r"(su32(src)), "r"(0), "r"(c1), "r"(c2)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
// 16-byte unit j (words 2j, 2j+1) of tile row r (128 bytes) under SWIZZLE_128B
__device__ __forceinline__ uint32_t tile_off(uint32_t r, uint32_t j) { return r * 128 + ((j ^ (r & 7)) << 4); }

template <int PASS, bool WIDE, class IN, class OUT, bool TMA = false>
__device__ __forceinline__ void ntt256_body(uint64_t* __restrict__ a, uint32_t row, uint32_t limb, uint64_t q,
                                            const double2* __restrict__ W2, const double2* __restrict__ ninv,
                                            double* sm, const IN& in, const OUT& out,
                                            const CUtensorMap* tmap = nullptr, uint32_t prow = 0,
                                            uint64_t* bar = nullptr, const double* __restrict__ W1 = nullptr) {
    const double qd = (double)q, qinv = 1.0 / qd;
    const bool fwd = PASS == FWD_A || PASS == FWD_B;
    const bool colp = PASS == FWD_A || PASS == INV_A;
    // block-pass twiddles of the narrow limbs come from the compact table (w only, 8 bytes) with the quotient
    // companion formed here: RN(w RN(1/q)) is within 2^-52 relative of w/q, and for |V| < 2^44 (narrow limbs)
    // the quotient estimate moves by < 2^-9, so the |r| <= 0.625 q bound of mulmod holds -- this halves the
    // per-block twiddle bytes the block passes pull from L2 (twice their data bytes with the double2 table)
    const bool compact = !colp && !WIDE && W1 != nullptr;
    auto twf = [&](uint32_t idx) -> double2 {
        if (compact) {
            const double w = __ldg(W1 + idx);
            return make_double2(w, w * qinv);
        }
        return W2[idx];
    };
    const uint32_t tid = threadIdx.x;
    const uint32_t sp = colp ? (tid & 15) : (tid >> 4);
    const uint32_t tt = colp ? (tid >> 4) : (tid & 15);
    const uint32_t sub = blockIdx.x * 16 + sp;
    auto gaddr = [&](uint32_t i) -> uint64_t { return colp ? (uint64_t)sub + 256ull * i : 256ull * sub + i; };
    // twiddle index of the butterfly with lower point i1 at local stride 2^lt is pre(lt) + (i1 >> (lt + 1)).  For
    // points i1 = tt + 16 k (lt >= 4) that is pre(lt) + (k >> (lt - 3)); for i1 = 16 tt + k (lt <= 3) it is
    // pre(lt) + (tt << (3 - lt)) + (k >> (lt + 1)): each distinct twiddle is loaded once per thread and stage
    // (15 + 15 loads per pass instead of one per butterfly -- the L1/LSU wavefronts were the limiter).
    auto pre = [&](uint32_t lt) -> uint32_t {
#ifdef ENSI_ABL_TW
        return colp ? (128u >> lt) : (32768u >> lt) + (sub & 1) * (128u >> lt);   // ablation: timing only
#else
        return colp ? (128u >> lt) : (32768u >> lt) + sub * (128u >> lt);
#endif
    };
    auto ct = [&](double& U, double& V, const double2 w) {
        const double r = mulmod(V, w.x, w.y, qd);
        V = U - r;
        U = U + r;
    };
    auto gs = [&](double& U, double& V, const double2 w, bool reduce) {
        const double s = U + V;
        V = mulmod(U - V, w.x, w.y, qd);
        U = reduce ? red(s, qd, qinv) : s;
    };
    double v[16];

    if (fwd) {
#pragma unroll
        for (uint32_t k = 0; k < 16; k++) {
            const uint32_t i = tt + 16 * k;
            if (PASS == FWD_A) v[k] = i2d((long long)in.load(a, row, limb, (uint32_t)gaddr(i)));
            else v[k] = __longlong_as_double((long long)__ldcg(a + gaddr(i)));
        }
        {
            // the group's 15 distinct twiddles are fetched up front (one batch of loads in flight instead of
            // a dependent load before every stage)
            double2 tw[15];
#pragma unroll
            for (int lt = 7; lt >= 4; lt--) {
                const uint32_t sh = lt - 3, base = pre(lt);
#pragma unroll
                for (uint32_t j = 0; j < (16u >> sh); j++) tw[((1u << (7 - lt)) - 1) + j] = twf(base + j);
            }
#pragma unroll
            for (int lt = 7; lt >= 4; lt--) {
                const uint32_t ks = 1u << (lt - 4), sh = lt - 3;
#pragma unroll
                for (uint32_t k = 0; k < 16; k++)
                    if (!(k & ks)) ct(v[k], v[k + ks], tw[((1u << (7 - lt)) - 1) + (k >> sh)]);
            }
        }
#pragma unroll
        for (uint32_t k = 0; k < 16; k++) sm[sidx(sp, tt + 16 * k)] = WIDE ? red(v[k], qd, qinv) : v[k];
        __syncthreads();
#pragma unroll
        for (uint32_t k = 0; k < 16; k++) v[k] = sm[sidx(sp, 16 * tt + k)];
        {
            // the group's 15 distinct twiddles are fetched up front (one batch of loads in flight instead of
            // a dependent load before every stage)
            double2 tw[15];
#pragma unroll
            for (int lt = 3; lt >= 0; lt--) {
                // block passes read the lane-transposed table region (twi_step = 16: the 16 lanes of a j are
                // consecutive entries, one 256-byte coalesced load); column passes the natural order
                const uint32_t sh = lt + 1, base = colp ? pre(lt) + (tt << (3 - lt)) : pre(lt) + tt;
                const uint32_t step = colp ? 1u : 16u;
#pragma unroll
                for (uint32_t j = 0; j < (16u >> sh); j++) tw[((1u << (3 - lt)) - 1) + j] = twf(base + step * j);
            }
#pragma unroll
            for (int lt = 3; lt >= 0; lt--) {
                const uint32_t ks = 1u << lt, sh = lt + 1;
#pragma unroll
                for (uint32_t k = 0; k < 16; k++)
                    if (!(k & ks)) ct(v[k], v[k + ks], tw[((1u << (3 - lt)) - 1) + (k >> sh)]);
            }
        }
        if (PASS == FWD_A) {
#pragma unroll
            for (uint32_t k = 0; k < 16; k++)
                a[gaddr(16 * tt + k)] = (uint64_t)__double_as_longlong(WIDE ? red(v[k], qd, qinv) : v[k]);
        } else if (TMA) {
            // final canonical words straight from registers into the swizzled tile, one TMA bulk store per CTA
            __syncthreads();
            uint8_t* tile = reinterpret_cast<uint8_t*>(sm);
            const uint32_t r = sp * 16 + tt;
#pragma unroll
            for (uint32_t j = 0; j < 8; j++)
                *reinterpret_cast<ulonglong2*>(tile + tile_off(r, j)) =
                    make_ulonglong2(canon(red(v[2 * j], qd, qinv), q), canon(red(v[2 * j + 1], qd, qinv), q));
            if constexpr (OUT::kFused) {
                // fused epilogue: lane-consecutive words of the tile (coalesced global traffic in out.store)
                __syncthreads();
#pragma unroll 4
                for (uint32_t k = 0; k < 16; k++) {
                    const uint32_t w = threadIdx.x + 256 * k, r2 = w >> 4;
                    const uint64_t zt =
                        *reinterpret_cast<const uint64_t*>(tile + tile_off(r2, (w >> 1) & 7) + 8 * (w & 1));
                    out.store(a, row, limb, 4096 * blockIdx.x + w, zt);
                }
            } else {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncthreads();
                if (threadIdx.x == 0) tile_store(tmap, tile, (int32_t)(256 * blockIdx.x), (int32_t)prow);
            }
        } else {
            __syncthreads();
#pragma unroll
            for (uint32_t k = 0; k < 16; k++) sm[sidx(sp, 16 * tt + k)] = red(v[k], qd, qinv);
            __syncthreads();
#pragma unroll
            for (uint32_t k = 0; k < 16; k++)
                out.store(a, row, limb, (uint32_t)gaddr(tt + 16 * k), canon(sm[sidx(sp, tt + 16 * k)], q));
        }
    } else {
        // wide limbs centre the canonical input (b = 1/2) so that two doubling stages stay below b = 2
        auto load_in = [&](uint64_t x) -> double {
            long long s = (long long)x;
            if (WIDE) s -= (s > (long long)(q >> 1)) ? (long long)q : 0;
            return i2d(s);
        };
        if (PASS == INV_B && TMA) {
            if (threadIdx.x == 0) tile_load(sm, tmap, bar, (int32_t)(256 * blockIdx.x), (int32_t)prow);
            tile_wait(bar);
            const uint8_t* tile = reinterpret_cast<const uint8_t*>(sm);
            const uint32_t r = sp * 16 + tt;
#pragma unroll
            for (uint32_t j = 0; j < 8; j++) {
                const ulonglong2 x = *reinterpret_cast<const ulonglong2*>(tile + tile_off(r, j));
                v[2 * j] = load_in(x.x);
                v[2 * j + 1] = load_in(x.y);
            }
        } else if (PASS == INV_B) {
#pragma unroll
            for (uint32_t k = 0; k < 16; k++) sm[sidx(sp, tt + 16 * k)] = load_in(a[gaddr(tt + 16 * k)]);
            __syncthreads();
#pragma unroll
            for (uint32_t k = 0; k < 16; k++) v[k] = sm[sidx(sp, 16 * tt + k)];
        } else {
#pragma unroll
            for (uint32_t k = 0; k < 16; k++) v[k] = __longlong_as_double((long long)__ldcg(a + gaddr(16 * tt + k)));
        }
#pragma unroll
        for (int lt = 0; lt <= 3; lt++) {
            const uint32_t ks = 1u << lt, sh = lt + 1;
            const uint32_t base = colp ? pre(lt) + (tt << (3 - lt)) : pre(lt) + tt, step = colp ? 1u : 16u;
            const bool rd = WIDE ? (lt & 1) : (lt == 3);
            double2 w;
#pragma unroll
            for (uint32_t k = 0; k < 16; k++) {
                if (!(k & ((1u << sh) - 1))) w = twf(base + step * (k >> sh));
                if (!(k & ks)) gs(v[k], v[k + ks], w, rd);
            }
        }
        if (PASS == INV_B) __syncthreads();
#pragma unroll
        for (uint32_t k = 0; k < 16; k++) sm[sidx(sp, 16 * tt + k)] = v[k];
        __syncthreads();
#pragma unroll
        for (uint32_t k = 0; k < 16; k++) v[k] = sm[sidx(sp, tt + 16 * k)];
#pragma unroll
        for (int lt = 4; lt <= 7; lt++) {
            const uint32_t ks = 1u << (lt - 4), sh = lt - 3, base = pre(lt);
            const bool rd = WIDE ? (lt & 1) : (lt == 7);
            double2 w;
#pragma unroll
            for (uint32_t k = 0; k < 16; k++) {
                if (!(k & ((1u << sh) - 1))) w = twf(base + (k >> sh));
                if (!(k & ks)) gs(v[k], v[k + ks], w, rd);
            }
        }
        if (PASS == INV_B) {
#pragma unroll
            for (uint32_t k = 0; k < 16; k++) a[gaddr(tt + 16 * k)] = (uint64_t)__double_as_longlong(v[k]);
        } else {
            const double2 ni = ninv[limb];
#pragma unroll
            for (uint32_t k = 0; k < 16; k++) a[gaddr(tt + 16 * k)] = canon(mulmod(v[k], ni.x, ni.y, qd), q);
        }
    }
}

template <int PASS, class IN = PlainIn, class OUT = PlainOut>
__global__ void __launch_bounds__(256, ENSI_NTTFP_MINB) k_ntt256(uint64_t* __restrict__ data, LimbMap map, ModTab tab,
                                                const double2* __restrict__ tw, const double2* __restrict__ ninv,
                                                IN in = IN(), OUT out = OUT()) {
    __shared__ double sm[16 * kRow];
    const uint32_t n = 65536;
    const uint32_t row = blockIdx.y, limb = map.limb[row % map.period];
    const uint64_t q = tab.q[limb];
    const bool fwd = PASS == FWD_A || PASS == FWD_B;
    const double2* W2 = tw + ((size_t)limb * 2 + (fwd ? 0 : 1)) * n;
    uint64_t* a = data + map.phys(row) * n;
    if (q >= (1ull << 41)) ntt256_body<PASS, true>(a, row, limb, q, W2, ninv, sm, in, out);
    else ntt256_body<PASS, false>(a, row, limb, q, W2, ninv, sm, in, out);
}

// Block passes with TMA tile I/O (PlainIn / PlainOut only): INV_B loads its 16 blocks with one bulk-tensor load,
// FWD_B stores them with one bulk-tensor store, instead of a shared-memory transpose around coalesced
// per-thread accesses.  tmap: the data buffer as a 3D tensor {16 words, N'/16 chunks, physical rows}.
template <int PASS, class OUT = PlainOut>
__global__ void __launch_bounds__(256, ENSI_NTTFP_MINB) k_ntt256_tma(uint64_t* __restrict__ data, LimbMap map, ModTab tab,
                                                    const double2* __restrict__ tw, const double2* __restrict__ ninv,
                                                    const __grid_constant__ CUtensorMap tmap, OUT out = OUT(),
                                                    LimbMap smap = LimbMap(), uint32_t oop = 0,
                                                    const double* __restrict__ tw1 = nullptr) {
    __shared__ __align__(1024) double sm[16 * kRow];
    __shared__ __align__(8) uint64_t bar;
    const uint32_t n = 65536;
    const uint32_t row = blockIdx.y, limb = map.limb[row % map.period];
    const uint64_t q = tab.q[limb];
    const bool fwd = PASS == FWD_A || PASS == FWD_B;
    const double2* W2 = tw + ((size_t)limb * 2 + (fwd ? 0 : 1)) * n;
    // oop (INV_B only): tile loaded from row smap.phys(row) of tmap's buffer, results written to data (map)
    const uint32_t prow = oop ? (uint32_t)smap.phys(row) : (uint32_t)map.phys(row);
    uint64_t* a = data + map.phys(row) * n;
    if (PASS == INV_B) {
        if (threadIdx.x == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
    }
    const PlainIn in;
    const double* W1 = tw1 ? tw1 + ((size_t)limb * 2 + (fwd ? 0 : 1)) * n : nullptr;
    if (q >= (1ull << 41)) ntt256_body<PASS, true, PlainIn, OUT, true>(a, row, limb, q, W2, ninv, sm, in, out, &tmap, prow, &bar);
    else ntt256_body<PASS, false, PlainIn, OUT, true>(a, row, limb, q, W2, ninv, sm, in, out, &tmap, prow, &bar, W1);
}

}  // namespace nttfp
}  // namespace ensi
