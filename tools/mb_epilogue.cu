// Microbenchmark: the tcgen05-accumulate epilogue recombination (combine_word5: 5 int32 byte-plane sums -> one
// canonical 40-bit RNS word) in registers, 8 warps per CTA, one CTA per SM, cycles per 16 words per warp.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/mb_epilogue.cu -o tools/mb_epilogue
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint64_t cw5(const uint32_t* r, uint64_t q, uint32_t mu32, uint64_t off64) {
    const int32_t s1 = (int32_t)r[0] + (int32_t)(r[1] << 8);
    const int32_t s2 = (int32_t)r[2] + (int32_t)(r[3] << 8);
    const uint64_t u = off64 + (uint64_t)(int64_t)s1 + ((uint64_t)(int64_t)s2 << 16) +
                       ((uint64_t)(int64_t)(int32_t)r[4] << 32);
    const uint32_t t = __umulhi((uint32_t)u, mu32);
    const uint32_t qhat = (uint32_t)(((uint64_t)(uint32_t)(u >> 32) * mu32 + t) >> 32);
    const uint64_t rr = u - (uint64_t)qhat * q;
    return rr >= q ? rr - q : rr;
}

__global__ void __launch_bounds__(256, 1) k(const uint32_t* in, uint64_t* out, uint64_t q, uint32_t mu, uint64_t off,
                                            int iters, long long* cyc) {
    uint32_t r[128];
#pragma unroll
    for (int i = 0; i < 128; i++) r[i] = in[(threadIdx.x * 128 + i) & 4095];
    uint64_t acc = 0;
    long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
        uint64_t v[16];
#pragma unroll
        for (int w = 0; w < 16; w++) v[w] = cw5(r + 8 * w, q, mu, off);
#pragma unroll
        for (int w = 0; w < 16; w++) acc ^= v[w];
#pragma unroll
        for (int i = 0; i < 128; i += 8) r[i] += (uint32_t)acc;   // dependency so the loop is not hoisted
    }
    long long t1 = clock64();
    out[blockIdx.x * 256 + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
    uint32_t *in; uint64_t* out; long long* cyc;
    cudaMalloc(&in, 4096 * 4); cudaMemset(in, 1, 4096 * 4);
    cudaMalloc(&out, 148 * 256 * 8); cudaMalloc(&cyc, 148 * 8);
    const uint64_t q = 1099511480321ull;
    const uint32_t mu = (uint32_t)(((unsigned __int128)1 << 64) / q);
    const int iters = 1000;
    k<<<148, 256>>>(in, out, q, mu, q * 300000ull, iters, cyc);
    k<<<148, 256>>>(in, out, q, mu, q * 300000ull, iters, cyc);
    long long h[148];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    printf("cycles per 16-word combine per warp (8 warps/SM): %.1f\n", (double)h[0] / iters);
    return 0;
}
