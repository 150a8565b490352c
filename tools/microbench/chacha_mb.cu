// Microbenchmark: ChaCha20 block throughput on B200 with the quarter-round rotates on the ALU
// pipe (SHF) or partly moved to the FMA pipe (IMAD.WIDE + IMAD with runtime multipliers, which
// ptxas cannot strength-reduce back to shifts).  V = number of rotates per quarter round moved.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

struct Mul { uint32_t m16, m12, m8, m7, one; };

__device__ __forceinline__ uint32_t rotl_alu(uint32_t x, int n) { return __funnelshift_l(x, x, n); }
__device__ __forceinline__ uint32_t rotl_fma(uint32_t x, uint32_t mul, uint32_t one) {
    const unsigned long long p = (unsigned long long)x * mul;       // IMAD.WIDE.U32
    return (uint32_t)(p >> 32) * one + (uint32_t)p;                 // IMAD (hi * 1 + lo)
}

template <int V>
__device__ __forceinline__ void qr(uint32_t &a, uint32_t &b, uint32_t &c, uint32_t &d, const Mul &M) {
    a += b; d ^= a; d = rotl_alu(d, 16);
    c += d; b ^= c; b = V >= 2 ? rotl_fma(b, M.m12, M.one) : rotl_alu(b, 12);
    a += b; d ^= a; d = V >= 3 ? rotl_fma(d, M.m8, M.one) : rotl_alu(d, 8);
    c += d; b ^= c; b = V >= 1 ? rotl_fma(b, M.m7, M.one) : rotl_alu(b, 7);
}

template <int V>
__global__ void __launch_bounds__(256) bench(uint32_t *out, int iters, Mul M, uint32_t seed) {
    uint32_t acc = 0;
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    for (int it = 0; it < iters; it++) {
        uint32_t x0 = 0x61707865u, x1 = 0x3320646eu, x2 = 0x79622d32u, x3 = 0x6b206574u;
        uint32_t x4 = seed, x5 = t, x6 = it, x7 = 7, x8 = 8, x9 = 9, x10 = 10, x11 = 11;
        uint32_t x12 = it * 977 + t, x13 = 0, x14 = 0, x15 = 0;
#pragma unroll
        for (int i = 0; i < 10; i++) {
            qr<V>(x0, x4, x8, x12, M); qr<V>(x1, x5, x9, x13, M); qr<V>(x2, x6, x10, x14, M); qr<V>(x3, x7, x11, x15, M);
            qr<V>(x0, x5, x10, x15, M); qr<V>(x1, x6, x11, x12, M); qr<V>(x2, x7, x8, x13, M); qr<V>(x3, x4, x9, x14, M);
        }
        acc ^= x0 ^ x1 ^ x2 ^ x3 ^ x4 ^ x5 ^ x6 ^ x7 ^ x8 ^ x9 ^ x10 ^ x11 ^ x12 ^ x13 ^ x14 ^ x15;
    }
    out[t] = acc;
}

template <int V>
static void run(uint32_t *d, int blocks, int iters) {
    Mul M{1u << 16, 1u << 12, 1u << 8, 1u << 7, 1u};
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    bench<V><<<blocks, 256>>>(d, iters, M, 1);
    cudaEventRecord(a);
    bench<V><<<blocks, 256>>>(d, iters, M, 2);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double blocks_total = (double)blocks * 256 * iters;
    printf("V=%d: %.3f ms, %.1f G blocks/s = %.2f TB/s keystream\n", V, ms, blocks_total / ms / 1e6,
           blocks_total * 64 / ms / 1e9);
}

int main() {
    uint32_t *d;
    const int blocks = 148 * 8 * 4, iters = 64;
    cudaMalloc(&d, (size_t)blocks * 256 * 4);
    run<0>(d, blocks, iters);
    run<1>(d, blocks, iters);
    run<2>(d, blocks, iters);
    run<3>(d, blocks, iters);
    run<0>(d, blocks, iters);
    return 0;
}
