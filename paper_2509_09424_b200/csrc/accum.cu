// accum.cu -- row a3, the ternary accumulate of Algorithm 1 on the CUDA-core integer pipes.
//
// y_i[w] = sum_{j : W[j][i] != 0} W[j][i] x_j[w]  mod q(w),  for every word w of the 2*l*N' words of a ciphertext.
// This is a d -> m integer contraction over M = 2 l N' word positions.  Tiling:
//   CTA = 8 warps = 64 outputs x 32*AP word positions (one limb, so q is CTA-uniform); AP = 4: 2 CTAs per SM.
//   warp w owns outputs i0 + 8w .. +8; lane owns positions lane + 32p, p < AP  ->  8*AP int64 accumulators.
//   x_j tiles (8 rows of 256 words) are staged in shared memory with cp.async, double buffered, and read by
//   all 8 warps (each x word is fetched from L2/HBM once per 64 outputs).
//   The weight sign is warp-uniform: one branch per (j, output) covers 8 words per lane, and zeros are
//   skipped exactly as Alg. 1 lines 4-8 skip W = 0.
// Accumulation is signed and lazy: on the FP64 pipe for limbs below 2^51 (acc_u2d), in 64-bit integers otherwise.
// Integer path: the host derives `ared`, the number of rows between intermediate
// reductions, from the widest active modulus (accum_rows_between_reductions) so that |acc| never leaves the
// int64 range nor the Barrett input range: 8191 rows for the O1 primes (< 2^50), 7 for a modulus near 2^60.
// The epilogue maps acc to the canonical word in [0, q) (Barrett), so the output is the unique canonical value
// and equals the oracle bit for bit.
#include <algorithm>

#include "ensi_internal.h"

#ifndef ENSI_ACC_AP
#define ENSI_ACC_AP 4
#endif

namespace ensi {

#ifndef ENSI_ACC_AO
#define ENSI_ACC_AO 8
#endif
#ifndef ENSI_ACC_RUNROLL
#define ENSI_ACC_RUNROLL 4
#endif
static constexpr int AO = ENSI_ACC_AO;  // outputs per warp
// FP64 path: rows of a stage unrolled (the next row's shared loads issue under this row's DFMAs; measured
// C2 88.0 / 86.6 / 85.5 ms at 1 / 2 / 4; 16 outputs per warp: 86.0-86.5 / 85.5 ms at 1 / 2 (224 registers))
static constexpr int kRunroll = ENSI_ACC_RUNROLL;
static constexpr int AP = ENSI_ACC_AP;  // positions per lane
static constexpr int AW = 8;          // warps per CTA
static constexpr int ATI = AO * AW;   // 64 outputs per CTA
static constexpr int ATW = 32 * AP;   // 256 positions per CTA
static constexpr int NPW = ATI / 32;  // sign-plane words per sign and row of the CTA's output tile
#ifndef ENSI_ACC_AKC
#define ENSI_ACC_AKC 32
#endif
static constexpr int AKC = ENSI_ACC_AKC;   // x rows per pipeline stage (32: 160 KB of dynamic shared memory, 1 CTA/SM; measured 86 ms vs 89 at 16 and 94 at 8 rows)

// dynamic shared memory layout: sx [2][AKC][ATW] uint64 | swd [2][AKC][ATI] double | ssg [2][AKC][2 NPW] uint32
static constexpr size_t kAccSmem =
    (size_t)2 * AKC * ATW * 8 + (size_t)2 * AKC * ATI * 8 + (size_t)2 * AKC * 2 * NPW * 4;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
    uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// FP64-pipe accumulation for limbs q < 2^51 (every limb at the O1 primes).  Every canonical word and every partial sum
// of up to `ared_fp` signed terms is an integer below 2^53, i.e. an exact double: one DFMA acc += w x (w in {-1,0,1})
// per term-word on the FP64 pipe (64 lanes/clk/SM on B200) instead of the 64-bit IADD3 + IADD3.X pair and the per-
// output sign branch on the integer pipe (3.86 instructions per term-word, profiles/r01_ncu_accum_cudacore.md).
// A word enters as a double through the 2^52 binade (x < 2^52: OR its high half into 0x43300000, subtract 2^52) and
// leaves through the centred reduction v - rint(v/q) q (exact) and the 1.5*2^52 round trip; the result is the same
// canonical word the integer path produces.
__device__ __forceinline__ double acc_u2d(uint64_t x) {
    return __longlong_as_double((long long)(x | 0x4330000000000000ull)) - 4503599627370496.0;   // x < 2^52
}
__device__ __forceinline__ double acc_red(double v, double q, double qinv) {
    const double t = fma(v, qinv, 6755399441055744.0) - 6755399441055744.0;   // rint(v / q), |v / q| < 2^51
    return fma(-t, q, v);                                                       // exact: |v - t q| <= q/2 + tiny
}
__device__ __forceinline__ uint64_t acc_canon(double v, uint64_t q, double qd, double qinv) {
    const long long r = __double_as_longlong(acc_red(v, qd, qinv) + 6755399441055744.0) - 0x4338000000000000ll;
    return (uint64_t)(r + ((r >> 63) & (long long)q));
}

// planes: [d][2][mw] uint32 (pos bits, neg bits); bit (i % 32) of word i / 32; mw even, zero padded.
__global__ void __launch_bounds__(256, AO * AP > 32 ? 1 : 8 / AP)
    k_accum_ternary(const uint64_t* __restrict__ x, uint32_t d, uint64_t ctw, const uint32_t* __restrict__ planes,
                    uint32_t mw, uint32_t m, uint64_t* __restrict__ y, uint32_t log_n, uint32_t level, uint32_t limb0,
                    ModTab tab, uint32_t ared) {
    extern __shared__ __align__(16) uint8_t acc_smem[];
    uint64_t (*sx)[AKC][ATW] = reinterpret_cast<uint64_t (*)[AKC][ATW]>(acc_smem);
    double (*swd)[AKC][ATI] = reinterpret_cast<double (*)[AKC][ATI]>(acc_smem + (size_t)2 * AKC * ATW * 8);
    // sign words of the tile: pos [0, NPW), neg [NPW, 2 NPW)
    uint32_t (*ssg)[AKC][2 * NPW] = reinterpret_cast<uint32_t (*)[AKC][2 * NPW]>(
        acc_smem + (size_t)2 * AKC * ATW * 8 + (size_t)2 * AKC * ATI * 8);
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t i0 = blockIdx.x * ATI;
    const uint64_t pos0 = (uint64_t)blockIdx.y * ATW;
    const uint32_t limb = (uint32_t)((limb0 + (pos0 >> log_n)) % level);
    const Barrett br = tab.br(limb);
    const uint32_t wsel = (warp * AO) >> 5, wsh = (warp * AO) & 31;   // this warp's AO sign bits
    const uint32_t pw0 = i0 >> 5;   // first plane word of this output tile

    int64_t acc[AO][AP];
#pragma unroll
    for (int o = 0; o < AO; o++)
#pragma unroll
        for (int p = 0; p < AP; p++) acc[o][p] = 0;

    const uint32_t nstages = (d + AKC - 1) / AKC;
    uint32_t since = 0;   // rows accumulated since the last reduction (every acc is then canonical, in [0, q))
    auto load_stage = [&](uint32_t s, int buf) {
        const uint32_t j0 = s * AKC;
        // x: AKC rows x ATW words in 16-byte chunks, AKC * ATW / 512 per thread
#pragma unroll
        for (int c = 0; c < AKC * ATW / 512; c++) {
            uint32_t chunk = tid + c * 256;
            uint32_t r = chunk / (ATW / 2), col = (chunk % (ATW / 2)) * 2;
            uint32_t j = j0 + r;
            if (j < d) cp_async16(&sx[buf][r][col], x + (uint64_t)j * ctw + pos0 + col);
        }
        if (tid < AKC * 2 * NPW) {
            const uint32_t r = tid / (2 * NPW), which = tid % (2 * NPW), j = j0 + r;
            const uint32_t sign = which / NPW, word = pw0 + which % NPW;
            if (j < d && word < mw) {
                const uint32_t* src = planes + ((uint64_t)j * 2 + sign) * mw + word;
                cp_async4(&ssg[buf][r][which], src);
            } else {
                ssg[buf][r][which] = 0;
            }
        }
    };

    load_stage(0, 0);
    cp_commit();
    if (br.q < (1ull << 51)) {   // >= 2 rows between reductions (see ared_fp)
        // ---- narrow limb: the FP64 pipe (see acc_u2d); CTA-uniform branch (one limb per CTA).  Each landed stage is
        // converted in shared memory once (x words -> doubles, sign bits -> w in {-1, 0, +1}), then every (row,
        // output) is AP exact DFMAs acc += w x with no per-output branch (the branchy add/sub/skip form spent ~3 of
        // its ~4 instructions per term-word on control: 152 ms for the C2 layer).
        const double qd = (double)br.q, qinv = 1.0 / qd;
        // rows between reductions for THIS limb: (n + 1/2) q < 2^53 (8189 at 2^40, 6 at 2^50; -2 absorbs the rounding
        // of the quotient)
        const uint32_t ared_fp = (uint32_t)(9007199254740991.0 / (double)(br.q - 1)) - 2;
        double* sxd = reinterpret_cast<double*>(&sx[0][0][0]);
        double acd[AO][AP];
#pragma unroll
        for (int o = 0; o < AO; o++)
#pragma unroll
            for (int p = 0; p < AP; p++) acd[o][p] = 0.0;
        uint32_t sincef = 0;
        for (uint32_t s = 0; s < nstages; s++) {
            const int buf = s & 1;
            if (s + 1 < nstages) load_stage(s + 1, buf ^ 1);
            cp_commit();
            cp_wait<1>();
            __syncthreads();
            {   // convert this stage in place: AKC x ATW words, AKC x ATI weights
                const uint32_t rows = min((uint32_t)AKC, d - s * AKC);
#pragma unroll
                for (int c = 0; c < AKC * ATW / 256; c++) {
                    const uint32_t e = tid + 256 * c, r = e / ATW;
                    uint64_t* px = &sx[buf][0][0] + e;
                    sxd[buf * AKC * ATW + e] = r < rows ? acc_u2d(*px) : 0.0;
                }
#pragma unroll
                for (int c = 0; c < AKC * ATI / 256; c++) {
                    const uint32_t e = tid + 256 * c, r = e / ATI, o = e % ATI;
                    const uint32_t pw = ssg[buf][r][o >> 5], nw = ssg[buf][r][NPW + (o >> 5)];
                    swd[buf][r][o] = (double)(int)((pw >> (o & 31)) & 1u) - (double)(int)((nw >> (o & 31)) & 1u);
                }
            }
            __syncthreads();
#pragma unroll kRunroll
            for (int r = 0; r < AKC; r++) {
                if (sincef == ared_fp) {   // |acd| <= (ared_fp + 1/2) q < 2^53 between reductions
#pragma unroll
                    for (int o = 0; o < AO; o++)
#pragma unroll
                        for (int p = 0; p < AP; p++) acd[o][p] = acc_red(acd[o][p], qd, qinv);
                    sincef = 0;
                }
                sincef++;
                // 16-byte shared loads: lane holds positions 2 lane + {0, 1} + 64 j (j < AP / 2); the warp's 8 weights
                // are 4 broadcast double2 loads
                double xv[AP];
#pragma unroll
                for (int j = 0; j < AP / 2; j++) {
                    const double2 t2 =
                        *reinterpret_cast<const double2*>(&sxd[(buf * AKC + r) * ATW + 2 * lane + 64 * j]);
                    xv[2 * j] = t2.x;
                    xv[2 * j + 1] = t2.y;
                }
#pragma unroll
                for (int o = 0; o < AO; o += 2) {
                    const double2 w2 = *reinterpret_cast<const double2*>(&swd[buf][r][warp * AO + o]);
#pragma unroll
                    for (int p = 0; p < AP; p++) {
                        acd[o][p] = fma(w2.x, xv[p], acd[o][p]);
                        acd[o + 1][p] = fma(w2.y, xv[p], acd[o + 1][p]);
                    }
                }
            }
            __syncthreads();
        }
#pragma unroll
        for (int o = 0; o < AO; o++) {
            const uint32_t i = i0 + warp * AO + o;
            if (i < m) {
                uint64_t* yo = y + (uint64_t)i * ctw + pos0;
#pragma unroll
                for (int j = 0; j < AP / 2; j++)
                    *reinterpret_cast<ulonglong2*>(yo + 2 * lane + 64 * j) =
                        make_ulonglong2(acc_canon(acd[o][2 * j], br.q, qd, qinv),
                                        acc_canon(acd[o][2 * j + 1], br.q, qd, qinv));
            }
        }
        return;
    }
    for (uint32_t s = 0; s < nstages; s++) {
        const int buf = s & 1;
        if (s + 1 < nstages) load_stage(s + 1, buf ^ 1);
        cp_commit();
        cp_wait<1>();
        __syncthreads();
#pragma unroll 1
        for (int r = 0; r < AKC; r++) {
            if (since == ared) {   // CTA-uniform: |acc| <= (ared + 1)(q - 1) stays inside int64 and Barrett's range
#pragma unroll
                for (int o = 0; o < AO; o++)
#pragma unroll
                    for (int p = 0; p < AP; p++) acc[o][p] = (int64_t)reduce_signed(acc[o][p], br);
                since = 0;
            }
            since++;
            constexpr uint32_t omask = AO >= 32 ? 0xFFFFFFFFu : (1u << AO) - 1;
            const uint32_t pb = (ssg[buf][r][wsel] >> wsh) & omask;
            const uint32_t nb = (ssg[buf][r][NPW + wsel] >> wsh) & omask;
            if ((pb | nb) == 0) continue;
            int64_t xv[AP];
#pragma unroll
            for (int p = 0; p < AP; p++) xv[p] = (int64_t)sx[buf][r][lane + 32 * p];
#pragma unroll
            for (int o = 0; o < AO; o++) {
                if (pb & (1u << o)) {
#pragma unroll
                    for (int p = 0; p < AP; p++) acc[o][p] += xv[p];
                } else if (nb & (1u << o)) {
#pragma unroll
                    for (int p = 0; p < AP; p++) acc[o][p] -= xv[p];
                }
            }
        }
        __syncthreads();
    }
    // epilogue: canonical words, coalesced stores (32 consecutive positions per warp store)
#pragma unroll
    for (int o = 0; o < AO; o++) {
        const uint32_t i = i0 + warp * AO + o;
        if (i < m) {
            uint64_t* yo = y + (uint64_t)i * ctw + pos0;
#pragma unroll
            for (int p = 0; p < AP; p++) yo[lane + 32 * p] = reduce_signed(acc[o][p], br);
        }
    }
}

// Rows between intermediate reductions: after a reduction every accumulator is canonical, and n further signed
// terms of magnitude <= q - 1 keep it in [-n (q-1), (n+1)(q-1)].  That must stay below 2^63 (int64) and below
// 2^(2w+2) (the Barrett input bound of reduce64, w = bitlen(q)), for every active limb.
uint32_t accum_rows_between_reductions(const ensi_ctx* ctx, uint32_t level) {
    uint64_t best = UINT32_MAX;
    for (uint32_t r = 0; r < level; r++) {
        const uint64_t q = ctx->mod[r];
        const uint32_t w = ctx->tab.w[r];
        const uint64_t bound = (2 * w + 2 >= 64) ? (uint64_t)INT64_MAX : ((1ull << (2 * w + 2)) - 1);
        const uint64_t n = bound / (q - 1) - 1;
        best = std::min<uint64_t>(best, n);
    }
    return (uint32_t)std::max<uint64_t>(1, best);
}

int accum_ternary(ensi_ctx* ctx, const uint64_t* x, uint32_t d, const uint32_t* planes, uint32_t mw, uint32_t m,
                  uint64_t* y, uint32_t level, cudaStream_t st, uint64_t ctw, uint32_t limb0) {
    if (ctw == 0) ctw = (uint64_t)2 * level * ctx->n;
    if (ctw % ATW) return set_err(ctx, ENSI_EINVAL, "ring too small for the accumulate tile");
    dim3 grid((m + ATI - 1) / ATI, (uint32_t)(ctw / ATW));
    cudaError_t ea = cudaFuncSetAttribute(k_accum_ternary, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kAccSmem);
    if (ea != cudaSuccess) return cuda_err(ctx, ea, "accum_ternary smem attribute");
    k_accum_ternary<<<grid, 256, kAccSmem, st>>>(x, d, ctw, planes, mw, m, y, ctx->log_n, level, limb0, ctx->tab,
                                          accum_rows_between_reductions(ctx, level));
    ENSI_LAUNCH_CHECK(ctx);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? ENSI_OK : cuda_err(ctx, e, "accum_ternary");
}

}  // namespace ensi
