// Microbenchmark: ChaCha20 block throughput on B200 with R of the 4 quarter-round rotations
// issued on the FMA pipe as two multiply-adds (x * 2^k gives x << k in the low word,
// mad.hi(x, 2^k, x << k) adds x >> (32-k)), the multipliers runtime values so ptxas keeps
// them as IMAD / IMAD.HI; the other rotations stay SHF / PRMT on the ALU pipe.  The adds are
// on the FMA pipe in every variant (ptxas' choice, as in the library).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t rotl(uint32_t x, int n) { return __funnelshift_l(x, x, n); }
__device__ __forceinline__ uint32_t rotm(uint32_t x, uint32_t m) {   // m = 2^k (runtime)
    uint32_t lo, r;
    asm("mul.lo.u32 %0, %1, %2;" : "=r"(lo) : "r"(x), "r"(m));
    asm("mad.hi.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(x), "r"(m), "r"(lo));
    return r;
}

__device__ __forceinline__ uint32_t rotw(uint32_t x, uint32_t m, uint32_t one) {   // mul.wide + mad.lo
    unsigned long long w;
    uint32_t r;
    asm("mul.wide.u32 %0, %1, %2;" : "=l"(w) : "r"(x), "r"(m));
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"((uint32_t)w), "r"(one), "r"((uint32_t)(w >> 32)));
    return r;
}
#ifndef ROTW
#define ROTW 0
#endif
__device__ uint32_t g_one = 1;
template <int R>
__device__ __forceinline__ void qr(uint32_t &a, uint32_t &b, uint32_t &c, uint32_t &d, uint32_t m16, uint32_t m12,
                                   uint32_t m8, uint32_t m7) {
    a += b; d ^= a; d = R >= 4 ? (ROTW ? rotw(d, m16, g_one) : rotm(d, m16)) : rotl(d, 16);
    c += d; b ^= c; b = R >= 3 ? (ROTW ? rotw(b, m12, g_one) : rotm(b, m12)) : rotl(b, 12);
    a += b; d ^= a; d = R >= 2 ? (ROTW ? rotw(d, m8, g_one) : rotm(d, m8)) : rotl(d, 8);
    c += d; b ^= c; b = R >= 1 ? (ROTW ? rotw(b, m7, g_one) : rotm(b, m7)) : rotl(b, 7);
}

// H: rotations on the FMA pipe in every other quarter round only (R for odd columns, 0 for even)
template <int R, bool HALF>
__global__ void __launch_bounds__(256) bench(uint32_t *out, int iters, uint32_t m16, uint32_t m12, uint32_t m8,
                                             uint32_t m7, uint32_t seed) {
    uint32_t acc = 0;
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    for (int it = 0; it < iters; it++) {
        uint32_t x0 = 0x61707865u, x1 = 0x3320646eu, x2 = 0x79622d32u, x3 = 0x6b206574u;
        uint32_t x4 = seed, x5 = t, x6 = it, x7 = 7, x8 = 8, x9 = 9, x10 = 10, x11 = 11;
        uint32_t x12 = it * 977 + t, x13 = 0, x14 = 0, x15 = 0;
        constexpr int R2 = HALF ? 0 : R;
#pragma unroll
        for (int i = 0; i < 10; i++) {
            qr<R>(x0, x4, x8, x12, m16, m12, m8, m7); qr<R2>(x1, x5, x9, x13, m16, m12, m8, m7);
            qr<R>(x2, x6, x10, x14, m16, m12, m8, m7); qr<R2>(x3, x7, x11, x15, m16, m12, m8, m7);
            qr<R>(x0, x5, x10, x15, m16, m12, m8, m7); qr<R2>(x1, x6, x11, x12, m16, m12, m8, m7);
            qr<R>(x2, x7, x8, x13, m16, m12, m8, m7); qr<R2>(x3, x4, x9, x14, m16, m12, m8, m7);
        }
        acc ^= x0 ^ x1 ^ x2 ^ x3 ^ x4 ^ x5 ^ x6 ^ x7 ^ x8 ^ x9 ^ x10 ^ x11 ^ x12 ^ x13 ^ x14 ^ x15;
    }
    out[t] = acc;
}

template <int R, bool HALF>
static void run(uint32_t *d, int blocks, int iters) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    bench<R, HALF><<<blocks, 256>>>(d, iters, 1u << 16, 1u << 12, 1u << 8, 1u << 7, 1);
    cudaEventRecord(a);
    bench<R, HALF><<<blocks, 256>>>(d, iters, 1u << 16, 1u << 12, 1u << 8, 1u << 7, 2);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double blocks_total = (double)blocks * 256 * iters;
    printf("R=%d%s rotations on the FMA pipe: %.3f ms, %.2f G blocks/s, %.3f TB/s keystream\n", R,
           HALF ? " (every other QR)" : "", ms, blocks_total / ms / 1e6, blocks_total * 64 / ms / 1e9);
}

int main() {
    uint32_t *d;
    const int blocks = 148 * 8 * 4, iters = 64;
    cudaMalloc(&d, (size_t)blocks * 256 * 4);
    run<0, false>(d, blocks, iters); run<1, true>(d, blocks, iters); run<1, false>(d, blocks, iters);
    run<2, true>(d, blocks, iters); run<2, false>(d, blocks, iters); run<3, false>(d, blocks, iters);
    run<0, false>(d, blocks, iters);
    return 0;
}
