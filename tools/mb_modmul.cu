// Microbenchmark: NTT butterfly throughput in registers on one B200, integer Shoup (current ntt_v2) vs an
// FP64 (DFMA) modular multiplication with centred residues.  Standalone: nvcc -O3 -gencode
// arch=compute_100a,code=sm_100a tools/mb_modmul.cu -o tools/mb_modmul && tools/mb_modmul
// Each thread holds 16 points and runs radix-2 stages (span 8,4,2,1) repeatedly; a "pass" = 8 stages, then a
// reduction (as at a pass end).  Correctness: both variants run the same stages on the same inputs and the
// canonicalised results are compared.
#include <cstdint>
#include <cstdio>
#include <cmath>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

struct TW { uint64_t w[8], wp[8]; double wd[8], wq[8]; };

__device__ __forceinline__ void bfly_int(uint64_t& U, uint64_t& V, uint64_t w, uint64_t wp, uint64_t q, uint64_t q2) {
    uint64_t u = U >= q2 ? U - q2 : U;
    uint64_t hi = __umul64hi(V, wp);
    uint64_t t = V * w - hi * q;
    U = u + t;
    V = u + q2 - t;
}

__device__ __forceinline__ void bfly_fp(double& U, double& V, double w, double wq, double q) {
    const double M = 6755399441055744.0;  // 1.5 * 2^52
    double h = V * w;
    double l = fma(V, w, -h);
    double t = fma(V, wq, M) - M;        // rint(V w / q)
    double r = fma(-t, q, h) + l;        // V w - t q, exact, |r| <= ~q/2
    U = U + r;
    V = U - 2.0 * r;                     // (U + r) - 2r = U - r
}

// Hybrid butterfly: the quotient estimate on the FP64 pipe, the exact remainder V w - t q in 64-bit integers (IMAD on
// the FMA pipe), the butterfly adds back in FP64 -- moves ~half of the FP64 work to the idle integer pipes.
__device__ __forceinline__ void bfly_hyb(double& U, double& V, long long wi, double wq, long long qi) {
    const double M = 6755399441055744.0;
    const long long Mb = 0x4338000000000000ll;
    const long long ti = __double_as_longlong(fma(V, wq, M)) - Mb;       // rint(V w / q) as an integer
    const long long vi = __double_as_longlong(V + M) - Mb;               // V as an integer (|V| < 2^51)
    const long long ri = vi * wi - ti * qi;                               // exact in 64 bits (|r| < 2^62)
    const double r = __longlong_as_double(Mb + ri) - M;
    U = U + r;
    V = U - 2.0 * r;
}

template <int MODE>
__global__ void k_bench(uint64_t* io, const TW* tw, uint64_t q, int passes, int check) {
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    const TW T = *tw;
    if (MODE == 0) {
        uint64_t v[16];
        for (int k = 0; k < 16; k++) v[k] = io[tid * 16 + k];
        const uint64_t q2 = 2 * q;
        for (int p = 0; p < passes; p++) {
#pragma unroll
            for (int rep = 0; rep < 2; rep++)
#pragma unroll
                for (int s = 0; s < 4; s++) {
                    const int span = 8 >> s;
#pragma unroll
                    for (int k = 0; k < 16; k++)
                        if (!(k & span)) bfly_int(v[k], v[k + span], T.w[(s + 4 * rep + k) & 7], T.wp[(s + 4 * rep + k) & 7], q, q2);
                }
#pragma unroll
            for (int k = 0; k < 16; k++) { uint64_t x = v[k] >= q2 ? v[k] - q2 : v[k]; v[k] = x >= q2 ? x - q2 : x; }
        }
        for (int k = 0; k < 16; k++) { uint64_t x = v[k] % q; io[tid * 16 + k] = x; }
    } else if (MODE == 2) {
        // alternate stages: pure FP64 on even k-groups, hybrid on odd (both kinds of work in flight)
        double v[16];
        const double qd = (double)q, qinv = 1.0 / qd, M = 6755399441055744.0;
        long long wi[8];
        for (int i = 0; i < 8; i++) wi[i] = (long long)T.wd[i];
        for (int k = 0; k < 16; k++) v[k] = (double)io[tid * 16 + k];
        for (int p = 0; p < passes; p++) {
#pragma unroll
            for (int rep = 0; rep < 2; rep++)
#pragma unroll
                for (int s = 0; s < 4; s++) {
                    const int span = 8 >> s;
#pragma unroll
                    for (int k = 0; k < 16; k++)
                        if (!(k & span)) {
                            const int ti = (s + 4 * rep + k) & 7;
                            if (k & 1) bfly_hyb(v[k], v[k + span], wi[ti], T.wq[ti], (long long)q);
                            else bfly_fp(v[k], v[k + span], T.wd[ti], T.wq[ti], qd);
                        }
                }
#pragma unroll
            for (int k = 0; k < 16; k++) { double t = fma(v[k], qinv, M) - M; v[k] = fma(-t, qd, v[k]); }
        }
        for (int k = 0; k < 16; k++) {
            double x = v[k];
            long long xi = (long long)x;
            long long r = xi % (long long)q;
            if (r < 0) r += q;
            io[tid * 16 + k] = (uint64_t)r;
        }
    } else {
        double v[16];
        const double qd = (double)q, qinv = 1.0 / qd, M = 6755399441055744.0;
        for (int k = 0; k < 16; k++) v[k] = (double)io[tid * 16 + k];
        for (int p = 0; p < passes; p++) {
#pragma unroll
            for (int rep = 0; rep < 2; rep++)
#pragma unroll
                for (int s = 0; s < 4; s++) {
                    const int span = 8 >> s;
#pragma unroll
                    for (int k = 0; k < 16; k++)
                        if (!(k & span)) bfly_fp(v[k], v[k + span], T.wd[(s + 4 * rep + k) & 7], T.wq[(s + 4 * rep + k) & 7], qd);
                }
#pragma unroll
            for (int k = 0; k < 16; k++) { double t = fma(v[k], qinv, M) - M; v[k] = fma(-t, qd, v[k]); }
        }
        for (int k = 0; k < 16; k++) {
            double x = v[k];
            long long xi = (long long)x;
            long long r = xi % (long long)q;
            if (r < 0) r += q;
            io[tid * 16 + k] = (uint64_t)r;
        }
    }
}

static uint64_t mulmod_h(uint64_t a, uint64_t b, uint64_t q) { return (unsigned __int128)a * b % q; }

int main() {
    const uint64_t primes[2] = {1099511480321ull /* < 2^40, 1 mod 2^17 */, 1125899906826241ull /* < 2^50 */};
    const int threads = 148 * 4 * 256;
    for (int pi = 0; pi < 2; pi++) {
        const uint64_t q = primes[pi];
        TW T;
        uint64_t x = 0x9E3779B97F4A7C15ull;
        for (int i = 0; i < 8; i++) {
            x = x * 6364136223846793005ull + 1442695040888963407ull;
            T.w[i] = (x >> 5) % q;
            T.wp[i] = (uint64_t)(((unsigned __int128)T.w[i] << 64) / q);
            int64_t wc = T.w[i] > q / 2 ? (int64_t)T.w[i] - (int64_t)q : (int64_t)T.w[i];
            T.wd[i] = (double)wc;
            T.wq[i] = (double)wc / (double)q;
        }
        std::vector<uint64_t> h(threads * 16);
        for (auto& e : h) { x = x * 6364136223846793005ull + 1442695040888963407ull; e = (x >> 3) % q; }
        uint64_t *d0, *d1; TW* dt;
        CK(cudaMalloc(&d0, h.size() * 8)); CK(cudaMalloc(&d1, h.size() * 8)); CK(cudaMalloc(&dt, sizeof(TW)));
        CK(cudaMemcpy(dt, &T, sizeof(TW), cudaMemcpyHostToDevice));
        // correctness: 2 passes
        CK(cudaMemcpy(d0, h.data(), h.size() * 8, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(d1, h.data(), h.size() * 8, cudaMemcpyHostToDevice));
        k_bench<0><<<threads / 256, 256>>>(d0, dt, q, 2, 1);
        k_bench<1><<<threads / 256, 256>>>(d1, dt, q, 2, 1);
        CK(cudaDeviceSynchronize());
        std::vector<uint64_t> a(h.size()), b(h.size());
        CK(cudaMemcpy(a.data(), d0, h.size() * 8, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(b.data(), d1, h.size() * 8, cudaMemcpyDeviceToHost));
        size_t bad = 0;
        for (size_t i = 0; i < a.size(); i++) bad += a[i] != b[i];
        // host check of thread 0 (int variant) against plain modular arithmetic
        uint64_t v[16];
        for (int k = 0; k < 16; k++) v[k] = h[k];
        for (int p = 0; p < 2; p++)
            for (int rep = 0; rep < 2; rep++)
                for (int s = 0; s < 4; s++) {
                    int span = 8 >> s;
                    for (int k = 0; k < 16; k++)
                        if (!(k & span)) {
                            uint64_t t = mulmod_h(v[k + span], T.w[(s + 4 * rep + k) & 7], q);
                            uint64_t u = v[k];
                            v[k] = (u + t) % q;
                            v[k + span] = (u + q - t) % q;
                        }
                }
        size_t badh = 0;
        for (int k = 0; k < 16; k++) badh += v[k] != a[k];
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        const int passes = 64;
        float ms[3];
        {   // hybrid correctness (2 passes) against the FP64 variant
            uint64_t* d2; CK(cudaMalloc(&d2, h.size() * 8));
            CK(cudaMemcpy(d2, h.data(), h.size() * 8, cudaMemcpyHostToDevice));
            k_bench<2><<<threads / 256, 256>>>(d2, dt, q, 2, 1);
            CK(cudaDeviceSynchronize());
            std::vector<uint64_t> c(h.size());
            CK(cudaMemcpy(c.data(), d2, h.size() * 8, cudaMemcpyDeviceToHost));
            size_t bad2 = 0;
            for (size_t i = 0; i < c.size(); i++) bad2 += c[i] != b[i];
            printf("hybrid vs fp64 mismatches: %zu\n", bad2);
            cudaFree(d2);
        }
        for (int mode = 0; mode < 3; mode++) {
            for (int it = 0; it < 2; it++) {
                cudaEventRecord(e0);
                if (mode == 0) k_bench<0><<<threads / 256, 256>>>(d0, dt, q, passes, 0);
                else if (mode == 1) k_bench<1><<<threads / 256, 256>>>(d1, dt, q, passes, 0);
                else k_bench<2><<<threads / 256, 256>>>(d1, dt, q, passes, 0);
                cudaEventRecord(e1);
                CK(cudaEventSynchronize(e1));
                cudaEventElapsedTime(&ms[mode], e0, e1);
            }
        }
        double bfly = (double)threads * passes * 8 * 8;
        printf("q=%llu (%d-bit): mismatches int-vs-fp %zu, int-vs-host %zu | int %.3f ms %.1f Gbfly/s | fp64 %.3f ms %.1f Gbfly/s | hybrid %.3f ms %.1f Gbfly/s\n",
               (unsigned long long)q, pi ? 50 : 40, bad, badh, ms[0], bfly / ms[0] / 1e6, ms[1], bfly / ms[1] / 1e6,
               ms[2], bfly / ms[2] / 1e6);
        cudaFree(d0); cudaFree(d1); cudaFree(dt);
    }
    return 0;
}
