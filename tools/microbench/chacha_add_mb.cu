// Microbenchmark: ChaCha20 block throughput on B200 with A of the 4 quarter-round additions
// issued as IMAD (x * one + y, `one` a runtime 1 so ptxas keeps the multiply-add on the FMA
// pipe) instead of IADD3 on the ALU pipe.  The XORs and rotates stay on the ALU pipe.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t rotl(uint32_t x, int n) { return __funnelshift_l(x, x, n); }
__device__ __forceinline__ uint32_t madd(uint32_t x, uint32_t one, uint32_t y) {
    uint32_t d;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(x), "r"(one), "r"(y));
    return d;
}

template <int A>
__device__ __forceinline__ void qr(uint32_t &a, uint32_t &b, uint32_t &c, uint32_t &d, uint32_t one) {
    a = A >= 1 ? madd(b, one, a) : a + b; d ^= a; d = rotl(d, 16);
    c = A >= 3 ? madd(d, one, c) : c + d; b ^= c; b = rotl(b, 12);
    a = A >= 2 ? madd(b, one, a) : a + b; d ^= a; d = rotl(d, 8);
    c = A >= 4 ? madd(d, one, c) : c + d; b ^= c; b = rotl(b, 7);
}

template <int A>
__global__ void __launch_bounds__(256) bench(uint32_t *out, int iters, uint32_t one, uint32_t seed) {
    uint32_t acc = 0;
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    for (int it = 0; it < iters; it++) {
        uint32_t x0 = 0x61707865u, x1 = 0x3320646eu, x2 = 0x79622d32u, x3 = 0x6b206574u;
        uint32_t x4 = seed, x5 = t, x6 = it, x7 = 7, x8 = 8, x9 = 9, x10 = 10, x11 = 11;
        uint32_t x12 = it * 977 + t, x13 = 0, x14 = 0, x15 = 0;
#pragma unroll
        for (int i = 0; i < 10; i++) {
            qr<A>(x0, x4, x8, x12, one); qr<A>(x1, x5, x9, x13, one); qr<A>(x2, x6, x10, x14, one); qr<A>(x3, x7, x11, x15, one);
            qr<A>(x0, x5, x10, x15, one); qr<A>(x1, x6, x11, x12, one); qr<A>(x2, x7, x8, x13, one); qr<A>(x3, x4, x9, x14, one);
        }
        acc ^= x0 ^ x1 ^ x2 ^ x3 ^ x4 ^ x5 ^ x6 ^ x7 ^ x8 ^ x9 ^ x10 ^ x11 ^ x12 ^ x13 ^ x14 ^ x15;
    }
    out[t] = acc;
}

template <int A>
static void run(uint32_t *d, int blocks, int iters) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    bench<A><<<blocks, 256>>>(d, iters, 1u, 1);
    cudaEventRecord(a);
    bench<A><<<blocks, 256>>>(d, iters, 1u, 2);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double blocks_total = (double)blocks * 256 * iters;
    printf("A=%d adds on the FMA pipe: %.3f ms, %.2f TB/s keystream\n", A, ms, blocks_total * 64 / ms / 1e9);
}

int main() {
    uint32_t *d;
    const int blocks = 148 * 8 * 4, iters = 64;
    cudaMalloc(&d, (size_t)blocks * 256 * 4);
    run<0>(d, blocks, iters); run<1>(d, blocks, iters); run<2>(d, blocks, iters);
    run<3>(d, blocks, iters); run<4>(d, blocks, iters); run<0>(d, blocks, iters);
    return 0;
}
