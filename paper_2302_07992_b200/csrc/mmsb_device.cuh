// mmsb_device.cuh -- device-side building blocks of the B200 hot path (sm_100a).
//
// Product code only: nothing here is shared with oracle/ (the CPU oracle re-derives every
// step from the paper independently).  Citations: P:<line> = /root/reference/PAPER.md.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "mmsb_geo.h"

namespace mmsb {

// --------------------------------------------------------------------------------------
// ChaCha20 block function (RFC 8439 §2.3).  The paper requires only "a cryptographically
// secure stream cipher"; reading Q12 fixes ChaCha20 with nonce 0 and counter 0, so
// byte r of the keystream is byte r%64 of block r/64: the stream is in counter form and any
// position is reachable without generating the prefix ("jump-ahead" = block counter).
// --------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t rotl32(uint32_t x, int n) { return __funnelshift_l(x, x, n); }

#define MMSB_QR(a, b, c, d)                                                     \
    a += b; d ^= a; d = rotl32(d, 16); c += d; b ^= c; b = rotl32(b, 12);       \
    a += b; d ^= a; d = rotl32(d, 8);  c += d; b ^= c; b = rotl32(b, 7);

// dr = double rounds: 10 (ChaCha20: fully unrolled, branch-free) or 6 / 4 (the reduced-round
// format option: a uniform loop)
__device__ __forceinline__ void chacha20_block(const uint32_t k[8], uint32_t counter, uint32_t o[16], int dr = 10) {
    uint32_t x0 = 0x61707865u, x1 = 0x3320646eu, x2 = 0x79622d32u, x3 = 0x6b206574u;
    uint32_t x4 = k[0], x5 = k[1], x6 = k[2], x7 = k[3], x8 = k[4], x9 = k[5], x10 = k[6], x11 = k[7];
    uint32_t x12 = counter, x13 = 0, x14 = 0, x15 = 0;
    if (dr == 10) {
#pragma unroll
        for (int i = 0; i < 10; i++) {
            MMSB_QR(x0, x4, x8, x12) MMSB_QR(x1, x5, x9, x13) MMSB_QR(x2, x6, x10, x14) MMSB_QR(x3, x7, x11, x15)
            MMSB_QR(x0, x5, x10, x15) MMSB_QR(x1, x6, x11, x12) MMSB_QR(x2, x7, x8, x13) MMSB_QR(x3, x4, x9, x14)
        }
    } else {
#pragma unroll 2
        for (int i = 0; i < dr; i++) {
            MMSB_QR(x0, x4, x8, x12) MMSB_QR(x1, x5, x9, x13) MMSB_QR(x2, x6, x10, x14) MMSB_QR(x3, x7, x11, x15)
            MMSB_QR(x0, x5, x10, x15) MMSB_QR(x1, x6, x11, x12) MMSB_QR(x2, x7, x8, x13) MMSB_QR(x3, x4, x9, x14)
        }
    }
    o[0] = x0 + 0x61707865u; o[1] = x1 + 0x3320646eu; o[2] = x2 + 0x79622d32u; o[3] = x3 + 0x6b206574u;
    o[4] = x4 + k[0]; o[5] = x5 + k[1]; o[6] = x6 + k[2]; o[7] = x7 + k[3];
    o[8] = x8 + k[4]; o[9] = x9 + k[5]; o[10] = x10 + k[6]; o[11] = x11 + k[7];
    o[12] = x12 + counter; o[13] = x13; o[14] = x14; o[15] = x15;
}

__device__ __forceinline__ void load_key(const uint8_t *keys, int img, uint32_t k[8]) {
    const uint4 *p = reinterpret_cast<const uint4 *>(keys + (size_t)img * 32);
    uint4 a = __ldg(p), b = __ldg(p + 1);
    k[0] = a.x; k[1] = a.y; k[2] = a.z; k[3] = a.w; k[4] = b.x; k[5] = b.y; k[6] = b.z; k[7] = b.w;
}

__device__ __forceinline__ uint32_t bswap32(uint32_t v) { return __byte_perm(v, 0, 0x0123); }

// PRMT with a runtime selector whose nibbles are already 0..7 (from a table or built that way):
// __byte_perm would mask the selector with 0x7777 first (one more ALU op per use)
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t s) {
    uint32_t r;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(s));
    return r;
}

// --------------------------------------------------------------------------------------
// Multi-scale block rotation (eq. roration; de-rotation P:819-835).
//
// The forward pass at level e rotates each 2^e block clockwise by 90 deg * angle; a
// one-turn clockwise rotation of an n-block sends offset (y, x) to (x, n-1-y).  Because
// levels below e keep a pixel inside its 2^e block, every aligned 2^k sub-block with k <= e
// moves rigidly: the composition over all levels maps aligned tiles onto aligned tiles
// (DESIGN.md §5.2).  The kernels exploit this at two granularities: 2^tp tiles (upper
// levels, one walk per tile) and 4x4 "cells" (levels 3..tp, one walk per cell); levels 1
// and 2 act inside a cell on bytes held in registers (PRMT).
// --------------------------------------------------------------------------------------

// destination offset -> source offset under `a` clockwise turns of an (m1+1)-block,
// m1 = 2^k - 1 so that m1 - v == v ^ m1.  Branch-free: a = 1: (m1-x, y), 2: (m1-y, m1-x),
// 3: (x, m1-y).
__device__ __forceinline__ void inv_turn(int a, int m1, int &y, int &x) {
    const int sw = a & 1, fy = (a ^ (a >> 1)) & 1, fx = (a >> 1) & 1;
    const int t = sw ? x : y, u = sw ? y : x;
    y = t ^ (-fy & m1);
    x = u ^ (-fx & m1);
}
// source offset -> destination offset under `a` clockwise turns: a = 1: (x, m1-y),
// 2: (m1-y, m1-x), 3: (m1-x, y)
__device__ __forceinline__ void fwd_turn(int a, int m1, int &y, int &x) {
    const int sw = a & 1, fy = (a >> 1) & 1, fx = (a ^ (a >> 1)) & 1;
    const int t = sw ? x : y, u = sw ? y : x;
    y = t ^ (-fy & m1);
    x = u ^ (-fx & m1);
}

// A 4x4 cell of bytes: r[i] = row i, byte j = column j (little-endian).
struct Cell { uint32_t r0, r1, r2, r3; };

// transpose: out[i][j] = in[j][i]
__device__ __forceinline__ Cell cell_transpose(Cell c) {
    uint32_t u0 = __byte_perm(c.r0, c.r1, 0x5140);   // [r0.0 r1.0 r0.1 r1.1]
    uint32_t u1 = __byte_perm(c.r2, c.r3, 0x5140);   // [r2.0 r3.0 r2.1 r3.1]
    uint32_t v0 = __byte_perm(c.r0, c.r1, 0x7362);   // [r0.2 r1.2 r0.3 r1.3]
    uint32_t v1 = __byte_perm(c.r2, c.r3, 0x7362);
    Cell o;
    o.r0 = __byte_perm(u0, u1, 0x5410);
    o.r1 = __byte_perm(u0, u1, 0x7632);
    o.r2 = __byte_perm(v0, v1, 0x5410);
    o.r3 = __byte_perm(v0, v1, 0x7632);
    return o;
}

// rotate the cell clockwise by 90 deg * r, branch-free (r differs between lanes):
//   r=0: out_i = in_i            r=1: out_i = rev(T_i)      (out[i][j] = in[3-j][i])
//   r=2: out_i = rev(in_{3-i})   r=3: out_i = T_{3-i}       (out[i][j] = in[j][3-i])
// with T = transpose(in) and rev = byte reversal.
__device__ __forceinline__ Cell cell_rot_cw(Cell c, int r) {
    const Cell t = cell_transpose(c);
    const bool odd = r & 1;
    // out_i = PRMT(a_i, a_{3-i}, S): S = 0x3210 (a_i), 0x0123 (rev a_i), 0x4567 (rev a_{3-i}),
    // 0x7654 (a_{3-i}) for r = 0..3, itself picked from a two-word table by one PRMT
    const uint32_t S = prmt(0x01233210u, 0x76544567u, (uint32_t)r * 0x22u + 0x10u);
    const uint32_t a0 = odd ? t.r0 : c.r0, a1 = odd ? t.r1 : c.r1, a2 = odd ? t.r2 : c.r2, a3 = odd ? t.r3 : c.r3;
    Cell o;
    o.r0 = prmt(a0, a3, S);
    o.r1 = prmt(a1, a2, S);
    o.r2 = prmt(a2, a1, S);
    o.r3 = prmt(a3, a0, S);
    return o;
}

// Level-1 (2x2) clockwise rotations of the two 2x2 blocks held in a row pair (top, bot):
// left block = bytes 0,1, right block = bytes 2,3; angles aL, aR.  PRMT indices: top row
// bytes 0..3, bottom row bytes 4..7.  A 2x2 block [[a,b],[c,d]] turned clockwise once is
// [[c,a],[d,b]].
__device__ __forceinline__ void pair_rot_cw(uint32_t &top, uint32_t &bot, int aL, int aR) {
    // nibble tables indexed by angle: (byte0 src, byte1 src) for the left block
    const uint32_t TOPS = 0x51450410u;   // a0: 0,1  a1: 4,0  a2: 5,4  a3: 1,5
    const uint32_t BOTS = 0x40011554u;   // a0: 4,5  a1: 5,1  a2: 1,0  a3: 0,4
    // the two selector bytes picked from the tables by one PRMT each: byte 0 = left table entry
    // aL, byte 1 = the right block's entry aR (the same entry + 0x22: byte offsets 2, 3)
    const uint32_t idx = (uint32_t)aL | ((uint32_t)(aR + 4) << 4);
    uint32_t nt = prmt(top, bot, prmt(TOPS, TOPS + 0x22222222u, idx));
    uint32_t nb = prmt(top, bot, prmt(BOTS, BOTS + 0x22222222u, idx));
    top = nt;
    bot = nb;
}

// angle of block (by, bx) of level e in a tile's angle record (2-bit fields, one u64 per row)
__device__ __forceinline__ int rec_angle(const uint64_t *rec, const Geo &g, int e, int by, int bx) {
    // the 32-bit half holding field bx (little-endian u64): one 32-bit load and shift
    const uint32_t *w = reinterpret_cast<const uint32_t *>(rec + g.lvl_off[e] + by);
    return (int)((w[bx >> 4] >> ((2 * bx) & 31)) & 3);
}

// 2-bit-field addition mod 4 (SWAR): per field (a + b) mod 4
__device__ __forceinline__ uint64_t add2(uint64_t a, uint64_t b) {
    return a ^ b ^ ((a & b & 0x5555555555555555ull) << 1);
}

// ------------------------------------------------------------------- bulk copies (TMA, 1-D)
// cp.async.bulk global -> shared with an mbarrier transaction count: one thread issues the
// copy of a whole contiguous chunk (no register staging, the copy engine keeps it in flight).
__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned phase) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra W;\n}" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}
// the same with a long suspend-time hint: the waiting warp sleeps in the barrier until the phase
// completes instead of re-polling (pipeline waits of worker warps that share the SM with ALU-bound
// keystream warps)
__device__ __forceinline__ void mbar_wait_sleep(uint64_t *bar, unsigned phase) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        " @!p bra W;\n}" ::"r"(smem_u32(bar)),
        "r"(phase), "r"(1000000u)
        : "memory");
}

// consumer release of a pipeline stage: one arrival (count = consumer warps) on its "empty" barrier
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// generic-proxy global writes (st.global) <-> async-proxy reads (cp.async.bulk) of the same data by
// CTAs of one launch: a proxy fence on both sides of the release / acquire
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

// shared -> global bulk copy (generic-proxy smem writes must be fenced first)
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void bulk_s2g(void *dst, const void *src, unsigned bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }

// drop an L2 line (128 B, aligned) without writing it back: transient scratch that exactly one
// consumer reads (keystream tiles, angle records) never costs HBM write bandwidth
__device__ __forceinline__ void discard_l2(const void *p) {
    asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
}

// ------------------------------------------------------------------- L2 residency hints
// scratch that a later CTA of the same launch reads once: keep it in L2 (evict_last) until the
// reader discards it; streamed inputs / outputs: evict first (ld/st .cs)
__device__ __forceinline__ uint64_t l2_evict_last_policy() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void st_keep(void *a, uint4 v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v4.b32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(a), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w), "l"(pol)
                 : "memory");
}

// ------------------------------------------------------------------- memory ordering
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u32(unsigned *p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_release_add_u32(unsigned *p, unsigned v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// relaxed (but coherent at gpu scope) accesses for self-contained flag|value words: no L1
// invalidation (CCTL.IVALL) per probe, unlike ld.acquire
__device__ __forceinline__ void st_relaxed(unsigned long long *p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ int ld_relaxed_s32(const int *p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

}  // namespace mmsb
