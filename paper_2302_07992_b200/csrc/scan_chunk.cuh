// scan_chunk.cuh -- the capacity prefix scan fused with embed / extract over one raster chunk
// (a7-a9): the body of the chunk kernels of k_scan.cu.  Citations:
// P:<line> = /root/reference/PAPER.md.
//
// Frame (reading Q17): F = BE32(n) || message, n in bits; E_F = F XOR KS2 (K2 keystream,
// counter form: bit k lives in ChaCha20 block k/512).  Redundant pixels (map bit 0) of the
// rotated domain, in raster order (Q18), carry b' bits each: EMR b' = b at bit positions
// 1..b, LMR b' = b-1 at positions 2..b.  Zero pixel j carries frame bits
// [j b', (j+1) b'); only bits < |F| are written (Q19).
//
// One CTA (256 threads) per 16384-pixel raster chunk, in chunk order within an image.  The
// chunk arrives in shared memory by one bulk copy (cp.async.bulk + mbarrier), so the whole
// chunk is in flight before any thread computes; thread t owns the 16-pixel groups t, t+256,
// t+512, t+768 of the chunk.  A chunk publishes its zero count (aggregate) and, once the
// look-back has found its prefix, its inclusive count; the K2 keystream of the chunk's frame
// bits is one ChaCha20 block per thread.  The per-image epilogue (capacity and integrity
// checks, boundary words of the extracted string) runs in a second small kernel, so the chunk
// CTAs retire without a grid-wide completion counter.
#pragma once
#include "mmsb_device.cuh"
#include "mmsb_kernels.h"

namespace mmsb {

constexpr unsigned long long kFlagAgg = 1ull << 62, kFlagInc = 2ull << 62, kValMask = (1ull << 62) - 1;
constexpr int kMaxBlk = kChunk * 7 / 512 + 2;          // ChaCha blocks a chunk's bits can touch
constexpr int kKbufWords = kMaxBlk * 16 + 4;     // + 3 words of alignment offset (extract)

// 16 zero-pixel flags of the pixels [p, p+16) of the chunk (bit i = pixel p+i is redundant)
template <int METHOD>
__device__ __forceinline__ uint32_t zero_mask16(const uint4 &u, bool first, const uint32_t *smap, int p_rel) {
    if constexpr (METHOD == 0) {
        // LSB == 0 -> redundant.  Two words at a time: their byte LSBs interleaved as nibble bits
        // (word a at bits 8k, word b at bits 8k + 4, one bit-select), inverted, and gathered into
        // the top byte by one multiply: l * (2^3 + 2^10 + 2^17 + 2^24) moves bit 8k to 24 + k and
        // bit 8k + 4 to 28 + k, and no two terms meet (no carries)
        auto pair = [](uint32_t a, uint32_t b) -> uint32_t {
            const uint32_t x = (a & 0x0F0F0F0Fu) | ((b << 4) & 0xF0F0F0F0u);
            return ((~x & 0x11111111u) * 0x01020408u) >> 24;
        };
        uint32_t m = pair(u.x, u.y) | (pair(u.z, u.w) << 8);
        if (first) m &= ~7u;                                     // image pixels 0..2 hold the header (Q14)
        return m;
    } else {
        return ~(smap[p_rel >> 5] >> (p_rel & 31)) & 0xFFFFu;
    }
}

// ---- per-thread bit streams of 16 pixels, specialised on b' (BP, bits per redundant pixel)
// and on the bit position of the carried field (SHIFT = 8 - b for EMR, 7 - b' for LMR).
// Both directions work on one 32-bit word (4 pixels) at a time with byte permutes: the
// fields of the set pixels of a word are consecutive in the frame stream, so a word needs
// one 32-bit window of the stream and one PRMT whose selector depends only on the word's
// 4-bit zero mask m4 (tables esel / csel in shared memory).  Between the stream window and
// the bytes, fields are held "left-aligned, MSB-first": stream field k in byte 3-k, at bits
// [8-BP, 8) of the byte, so both conversions are two halving steps (a shift and a
// select, or an add-multiply) instead of one shift and mask per field.
//   esel[m4] nibble i = 3 - (number of set bits of m4 below i)   (stream field -> pixel byte) for a
//                       set bit i, 4 + i (the pixel's own byte, second PRMT operand) otherwise
//   csel[m4] nibble 3-k = index of the k-th set bit, 4 (zero byte) past popc(m4)

// 4 consecutive BP-bit fields, MSB-first at the top of x -> field k at bits [8-BP, 8) of
// byte 3-k (the other bits of every byte are don't-care: callers mask them)
template <int BP>
__device__ __forceinline__ uint32_t fields_to_bytes(uint32_t x) {
    // fields 2, 3 to the top of the low half-word, then the second field of each half to the
    // top of its low byte
    const uint32_t x1 = __byte_perm(x, x >> (16 - 2 * BP), 0x3254);
    const uint32_t sh = x1 >> (8 - BP);
    return (x1 & 0xFF00FF00u) | (sh & 0x00FF00FFu);
}
// inverse: field k left-aligned in byte 3-k (other bits 0) -> 4 BP-bit fields MSB-first at
// the top; a low byte / half-word is moved up onto its neighbour by t + lo * (2^s - 1)
template <int BP>
__device__ __forceinline__ uint32_t bytes_to_fields(uint32_t c) {
    const uint32_t x = c + (c & 0x00FF00FFu) * ((1u << (8 - BP)) - 1u);
    return x + (x & 0xFFFFu) * ((1u << (16 - 2 * BP)) - 1u);
}

// embed (fast path: every field of the group lies below the frame end): the set pixels of
// the 16-pixel group receive consecutive BP-bit fields of the stream in kbuf from bit `rel`
template <int BP, int SHIFT>
__device__ __forceinline__ void embed16(uint32_t w[4], uint32_t mm, const uint32_t *kbuf, int rel,
                                        const uint32_t *esel) {
    constexpr uint32_t FMB = ((1u << BP) - 1u) << SHIFT;
    int o = rel;
#pragma unroll
    for (int j = 0; j < 4; j++) {
        const uint32_t m4 = (mm >> (4 * j)) & 0xFu;
        const int wi = o >> 5;
        const uint32_t x = __funnelshift_l(kbuf[wi + 1], kbuf[wi], o);   // stream bits [o, o+32)
        uint32_t e = fields_to_bytes<BP>(x);
        if constexpr (SHIFT != 8 - BP) e >>= (8 - BP - SHIFT);             // LMR: one bit lower
        // esel picks the field byte for a set pixel and the pixel's own byte otherwise, so one
        // constant-mask merge writes exactly the set pixels' fields
        const uint32_t v = prmt(e, w[j], esel[m4]);
        w[j] = (w[j] & ~(FMB * 0x01010101u)) | (v & (FMB * 0x01010101u));
        o += BP * __popc(m4);
    }
}

// embed, general path (the group reaches the frame end `fend`): bit by bit, bits at or past
// fend untouched (a partially filled last pixel keeps its remaining bits, reading Q19)
template <int BP, int SHIFT>
__device__ __noinline__ uint4 embed16_tail(uint4 u, uint32_t mm, const uint32_t *kbuf, long long rel, long long fend) {
    uint32_t w[4] = {u.x, u.y, u.z, u.w};
    long long k = rel;
    for (int i = 0; i < 16; i++) {
        if (!((mm >> i) & 1u)) continue;
        for (int t = 0; t < BP; t++, k++) {
            if (k >= fend) return make_uint4(w[0], w[1], w[2], w[3]);
            const uint32_t bit = (kbuf[k >> 5] >> (31 - (k & 31))) & 1u;
            const int pos = 8 * (i & 3) + SHIFT + BP - 1 - t;
            w[i >> 2] = (w[i >> 2] & ~(1u << pos)) | (bit << pos);
        }
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
}

// extract: the set pixels' BP-bit fields appended in raster order, XORed into kbuf (which holds
// the keystream) from bit `rel`; the first and last (partial) words can be shared with the
// neighbouring threads, so every word goes in by a shared-memory atomic XOR.
template <int BP, int SHIFT>
__device__ __forceinline__ void extract16(const uint32_t w[4], uint32_t mm, uint32_t *kbuf, int rel,
                                          const uint32_t *csel) {
    constexpr uint32_t FB = (((1u << BP) - 1u) << (8 - BP)) * 0x01010101u;
    int wi = rel >> 5;
    int nacc = rel & 31;                        // valid bits at the top of acc (leading pad = 0)
    unsigned long long acc = 0;
#pragma unroll
    for (int j = 0; j < 4; j++) {
        const uint32_t m4 = (mm >> (4 * j)) & 0xFu;
        const uint32_t t = (w[j] << (8 - BP - SHIFT)) & FB;       // byte i = field of pixel i, left-aligned
        const uint32_t c = prmt(t, 0, csel[m4]);           // set pixels' fields, bytes 3, 2, ..
        const uint32_t p = bytes_to_fields<BP>(c);
        acc |= ((unsigned long long)p << 32) >> nacc;
        nacc += BP * __popc(m4);
        if (nacc >= 32) {                       // XOR commutes: every word by one shared-memory atomic
            atomicXor(&kbuf[wi], (uint32_t)(acc >> 32));
            wi++;
            acc <<= 32;
            nacc -= 32;
        }
    }
    if (nacc > 0) atomicXor(&kbuf[wi], (uint32_t)(acc >> 32));
}

#define MMSB_BP_SWITCH(bp, METHOD, BODY)                                                   \
    switch (bp) {                                                                          \
        case 1: { constexpr int BP = 1, SH = (METHOD == 0 ? 8 : 7) - 1; BODY; } break;     \
        case 2: { constexpr int BP = 2, SH = (METHOD == 0 ? 8 : 7) - 2; BODY; } break;     \
        case 3: { constexpr int BP = 3, SH = (METHOD == 0 ? 8 : 7) - 3; BODY; } break;     \
        case 4: { constexpr int BP = 4, SH = (METHOD == 0 ? 8 : 7) - 4; BODY; } break;     \
        case 5: { constexpr int BP = 5, SH = (METHOD == 0 ? 8 : 7) - 5; BODY; } break;     \
        case 6: { constexpr int BP = 6, SH = (METHOD == 0 ? 8 : 7) - 6; BODY; } break;     \
        default: { constexpr int BP = 7, SH = (METHOD == 0 ? 8 : 7) - 7; BODY; } break;    \
    }

// b of an image as the hider / K2 receiver sees it: EMR from the 3 header LSBs (Q14; FORMAT
// if > 5 -> 0), LMR from the decoded MSB-plane header (0 on BADCASE / FORMAT)
template <int METHOD>
__device__ __forceinline__ int image_b(const uint8_t *img0, const int32_t *lmr_b, int img) {
    if constexpr (METHOD == 0) {
        const int field = ((img0[0] & 1) << 2) | ((img0[1] & 1) << 1) | (img0[2] & 1);
        return field > 5 ? 0 : field + 2;
    } else {
        return lmr_b[img];
    }
}

// embed's counting pass: zero pixels of every chunk and of the image, so that the chunk kernel
// knows its prefix and the image's capacity before it writes (the hider may embed in place)
template <int METHOD>
__device__ __forceinline__ void count_chunk(const Geo &g, const uint8_t *__restrict__ in,
                                            const uint32_t *__restrict__ map_bits, const ScanWS &ws, int cidx) {
    __shared__ uint32_t red[kScanThreads / 32];
    const int tid = threadIdx.x;
    const int img = cidx / g.nchunks, chunk = cidx % g.nchunks;
    const int cpx = g.HW < kChunk ? (int)g.HW : kChunk;
    const long long p0 = (long long)chunk * cpx;
    const uint4 *src = reinterpret_cast<const uint4 *>(in + (size_t)img * g.HW + p0);
    uint32_t c = 0;
    if constexpr (METHOD == 0) {
        // zero pixels = LSB 0: byte-lane sums of ~w & 0x01..01 over the thread's 64 pixels (<= 16
        // per lane), then one multiply adds the four lanes; the header pixels r = 0..2 (Q14) are
        // taken out by the thread that holds them
        uint32_t lanes = 0;
#pragma unroll
        for (int r = 0; r < kScanRounds; r++) {
            const int q = r * kScanThreads + tid;
            if (16 * q >= cpx) continue;
            const uint4 u = __ldg(src + q);
            lanes += (~u.x & 0x01010101u) + (~u.y & 0x01010101u) + (~u.z & 0x01010101u) + (~u.w & 0x01010101u);
            if (p0 + 16 * q == 0) lanes -= (~u.x & 0x00010101u);
        }
        c = (lanes * 0x01010101u) >> 24;
    } else {
#pragma unroll
        for (int r = 0; r < kScanRounds; r++) {
            const int q = r * kScanThreads + tid;
            if (16 * q >= cpx) continue;
            const long long pb = (long long)img * g.HW + p0 + 16 * q;
            c += __popc(~(__ldg(map_bits + (pb >> 5)) >> (pb & 31)) & 0xFFFFu);
        }
    }
    c = __reduce_add_sync(0xffffffffu, c);
    if ((tid & 31) == 0) red[tid >> 5] = c;
    __syncthreads();
    if (tid == 0) {
        uint32_t t = 0;
        for (int w = 0; w < kScanThreads / 32; w++) t += red[w];
        ws.counts[cidx] = t;
        if (t) atomicAdd(ws.ztot + img, (unsigned long long)t);
    }
}

template <int METHOD, bool EMBED>
struct ScanSmem {
    __align__(128) uint4 spx[kChunk / 16];
    __align__(16) uint32_t smap[METHOD == 1 ? kChunk / 32 : 4];
    __align__(16) uint32_t kbuf[kKbufWords];
    __align__(8) uint64_t bar, bar_ef;
    uint32_t wtot[kScanRounds][kScanThreads / 32], woff[kScanRounds][kScanThreads / 32];
    long long sh_prefix;
    uint32_t sh_agg;
    uint32_t wpre[kScanThreads / 32];
    uint32_t esel[16], csel[16];
};

// one chunk of image img (CTA of 256 threads; S in shared memory)
template <int METHOD, bool EMBED>
__device__ __forceinline__ void scan_chunk(ScanSmem<METHOD, EMBED> &S, const Geo &g, int img, int chunk,
                                           const uint8_t *__restrict__ in, uint8_t *__restrict__ out,
                                           const uint8_t *__restrict__ keys, const uint8_t *__restrict__ msg,
                                           const int64_t *__restrict__ msg_bits, long long stride,
                                           uint8_t *__restrict__ msg_out, const ScanWS &ws,
                                           const uint32_t *__restrict__ map_bits, const int32_t *__restrict__ lmr_b) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int cpx = g.HW < kChunk ? (int)g.HW : kChunk;      // pixels of this chunk
    const long long p0 = (long long)chunk * cpx;
    const uint8_t *src = in + (size_t)img * g.HW;

    if (tid == 0) {
        mbar_init(&S.bar, 1);
        if constexpr (EMBED) mbar_init(&S.bar_ef, 1);
        const unsigned bytes = (unsigned)cpx + (METHOD == 1 ? (unsigned)cpx / 8 : 0u);
        mbar_expect_tx(&S.bar, bytes);
        bulk_g2s(S.spx, src + p0, (unsigned)cpx, &S.bar);
        if constexpr (METHOD == 1)
            bulk_g2s(S.smap, map_bits + ((size_t)img * g.HW + p0) / 32, (unsigned)cpx / 8, &S.bar);
    }
    if (tid < 16) {                                          // PRMT selector tables (see embed16)
        uint32_t e = 0, c = 0;
        int k = 0;
        for (int i = 0; i < 4; i++) {
            e |= (uint32_t)(((tid >> i) & 1) ? 3 - __popc(tid & ((1 << i) - 1)) : 4 + i) << (4 * i);
            if ((tid >> i) & 1) c |= (uint32_t)i << (4 * (3 - k++));
        }
        for (; k < 4; k++) c |= 4u << (4 * (3 - k));
        S.esel[tid] = e;
        S.csel[tid] = c;
    }
    const int b = image_b<METHOD>(src, lmr_b, img);
    const int bp = METHOD == 0 ? b : b - 1;
    uint32_t key[8];
    load_key(keys, img, key);
    long long n = 0;
    if constexpr (EMBED) {
        n = msg_bits[img];
        // this chunk's prefix: the zero counts of the image's earlier chunks (embed_prep_kernel)
        uint32_t part = 0;
        for (int c = tid; c < chunk; c += kScanThreads) part += __ldg(ws.counts + (size_t)img * g.nchunks + c);
        part = __reduce_add_sync(0xffffffffu, part);
        if (lane == 0) S.wpre[wid] = part;
    }
    __syncthreads();                                         // barrier initialised (and S.wpre written)
    if constexpr (EMBED) {
        // the chunk's frame range is known from the counts already (prefix = earlier chunks,
        // aggregate = this chunk's count): its E_F blocks are fetched by one more bulk copy
        // that lands while the chunk is scanned
        if (tid == 0) {
            long long pre = 0;
            for (int w = 0; w < kScanThreads / 32; w++) pre += S.wpre[w];
            const long long agg0 = __ldg(ws.counts + (size_t)img * g.nchunks + chunk);
            const long long C = (long long)__ldcg(ws.ztot + img) * bp;
            const bool n_ok = n >= 0 && n <= 8 * stride && n <= 0xFFFFFFFFll && 32 + n <= C;
            const long long F = n_ok ? 32 + n : 0, lo = pre * bp, hi = (pre + agg0) * bp;
            const long long hie = hi < F ? hi : F, blk0 = lo >> 9;
            const int nblk = (b >= 2 && lo < hie) ? (int)(((hie - 1) >> 9) - blk0 + 1) : 0;
            mbar_expect_tx(&S.bar_ef, (unsigned)nblk * 64u);
            if (nblk) bulk_g2s(S.kbuf, ws.ef + (size_t)img * ws.ef_words + blk0 * 16, (unsigned)nblk * 64u, &S.bar_ef);
        }
    }
    mbar_wait(&S.bar, 0);

    if (b < 2) {                                             // FORMAT (EMR) / BADCASE, FORMAT (LMR)
        if constexpr (EMBED) {
            for (int q = tid; q < cpx / 16; q += kScanThreads)
                *reinterpret_cast<uint4 *>(out + (size_t)img * g.HW + p0 + 16 * q) = S.spx[q];
        }
        return;                                              // statuses: scan_finish_kernel
    }

    // ---- per-thread zero masks and counts, round r = 16-pixel group tid + 256 r
    // (the pixels stay in shared memory; they are re-read after the keystream phase)
    uint32_t m[kScanRounds];
#pragma unroll
    for (int r = 0; r < kScanRounds; r++) {
        const int q = r * kScanThreads + tid;
        m[r] = 16 * q < cpx ? zero_mask16<METHOD>(S.spx[q], r == 0 && tid == 0 && chunk == 0, S.smap, 16 * q) : 0u;
    }
    // warp-inclusive scans of the 4 round counts, two per packed u32 (counts <= 512 per warp)
    uint32_t c01 = __popc(m[0]) | ((uint32_t)__popc(m[1]) << 16);
    uint32_t c23 = __popc(m[2]) | ((uint32_t)__popc(m[3]) << 16);
    uint32_t i01 = c01, i23 = c23;
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
        const uint32_t t01 = __shfl_up_sync(0xffffffffu, i01, s), t23 = __shfl_up_sync(0xffffffffu, i23, s);
        if (lane >= s) { i01 += t01; i23 += t23; }
    }
    if (lane == 31) {
        S.wtot[0][wid] = i01 & 0xFFFFu; S.wtot[1][wid] = i01 >> 16;
        S.wtot[2][wid] = i23 & 0xFFFFu; S.wtot[3][wid] = i23 >> 16;
    }
    __syncthreads();
    // warp 0: exclusive scan of the 32 warp totals in raster order (round-major), which also
    // gives the chunk's aggregate for the look-back below; the offsets are read back after it
    uint32_t agg = 0;
    if (wid == 0) {
        const uint32_t v = (&S.wtot[0][0])[lane];
        uint32_t incl = v;
#pragma unroll
        for (int s2 = 1; s2 < 32; s2 <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, incl, s2);
            if (lane >= s2) incl += t;
        }
        (&S.woff[0][0])[lane] = incl - v;
        agg = __shfl_sync(0xffffffffu, incl, 31);
    }

    // ---- extract: single-pass decoupled look-back over the image's chunks (blockIdx order).
    // Warp 0 publishes the aggregate, then inspects 32 predecessors per probe: each lane spins
    // on its own predecessor until it has published; the nearest inclusive prefix ends the walk
    // and the aggregates in front of it are summed.  (Embed has its prefix from the counts.)
    if constexpr (EMBED) {
        if (wid == 0 && lane == 0) {
            long long pre = 0;
            for (int w = 0; w < kScanThreads / 32; w++) pre += S.wpre[w];
            S.sh_prefix = pre;
        }
    } else if (wid == 0) {
        unsigned long long *st = ws.states + (size_t)img * g.nchunks;
        unsigned long long prefix = 0;
        if (chunk == 0) {
            if (lane == 0) st_relaxed(st, kFlagInc | agg);
        } else {
            if (lane == 0) st_relaxed(st + chunk, kFlagAgg | agg);
            int base = chunk - 1;
            while (true) {
                const int k = base - lane;
                unsigned long long v = kFlagInc;                 // before chunk 0: inclusive 0
                if (k >= 0) {
                    // bounded: a predecessor that never publishes (no in-order dispatch) ends the
                    // walk with status E_CUDA for the image instead of a hang
                    unsigned spins = 0;
                    while (((v = ld_relaxed(st + k)) & ~kValMask) == 0) {
                        if (++spins > (1u << 22)) { atomicOr(ws.err + img, 1u); v = kFlagInc; break; }
                        if (spins > 64) __nanosleep(256);
                    }
                }
                const unsigned inc = __ballot_sync(0xffffffffu, (v & ~kValMask) == kFlagInc);
                const int last = inc ? __ffs(inc) - 1 : 31;
                unsigned long long val = lane <= last ? (v & kValMask) : 0ull;
#pragma unroll
                for (int s2 = 16; s2 > 0; s2 >>= 1) val += __shfl_xor_sync(0xffffffffu, val, s2);
                prefix += val;
                if (inc) break;
                base -= 32;
            }
            if (lane == 0) st_relaxed(st + chunk, kFlagInc | (prefix + agg));
        }
        if (lane == 0) S.sh_prefix = (long long)prefix;
    }
    if (wid == 0 && lane == 0) S.sh_agg = agg;
    __syncthreads();
    const long long prefix = S.sh_prefix;
    agg = S.sh_agg;
    uint32_t excl[kScanRounds];                              // this thread's groups inside the chunk
    {
        const uint32_t e01 = i01 - c01, e23 = i23 - c23;
        excl[0] = S.woff[0][wid] + (e01 & 0xFFFFu);
        excl[1] = S.woff[1][wid] + (e01 >> 16);
        excl[2] = S.woff[2][wid] + (e23 & 0xFFFFu);
        excl[3] = S.woff[3][wid] + (e23 >> 16);
    }
    const long long lo = prefix * bp, hi = (prefix + (long long)agg) * bp;

    if constexpr (EMBED) {
        // the frame is written only when it fits the image's capacity (else the chunk is copied
        // through unchanged: CAPACITY), so embedding in place needs no restore
        const long long C = (long long)__ldcg(ws.ztot + img) * bp;
        const bool n_ok = n >= 0 && n <= 8 * stride && n <= 0xFFFFFFFFll && 32 + n <= C;
        const long long F = n_ok ? 32 + n : 0;
        const long long hie = hi < F ? hi : F;
        const long long blk0 = lo >> 9;
        const int nblk = lo < hie ? (int)(((hie - 1) >> 9) - blk0 + 1) : 0;
        // E_F words of the chunk's frame blocks (embed_prep_kernel): the bulk copy issued at the start
        (void)nblk;
        mbar_wait(&S.bar_ef, 0);
        const long long base = blk0 * 512;
        // chunk-relative bit offsets fit 32 bits (lo - base < 512, a chunk holds < 2^17 frame bits):
        // the per-group arithmetic below is 32-bit; a frame end before / far past the chunk clamps
        const int rel0 = (int)(lo - base);
        const long long fend64 = hie - base;
        const int fend = fend64 < 0 ? 0 : fend64 > 0x3FFFFFFFll ? 0x3FFFFFFF : (int)fend64;
        uint8_t *dst = out + (size_t)img * g.HW + p0;
        MMSB_BP_SWITCH(bp, METHOD, ({
            _Pragma("unroll")
            for (int r = 0; r < kScanRounds; r++) {
                const int q = r * kScanThreads + tid;
                if (16 * q >= cpx) continue;
                const uint4 u = S.spx[q];
                uint32_t w[4] = {u.x, u.y, u.z, u.w};
                const int rel = rel0 + (int)excl[r] * BP;
                const int cnt = __popc(m[r]);
                if (cnt && rel < fend) {
                    if (rel + cnt * BP <= fend) embed16<BP, SH>(w, m[r], S.kbuf, rel, S.esel);
                    else {
                        const uint4 t = embed16_tail<BP, SH>(make_uint4(w[0], w[1], w[2], w[3]), m[r], S.kbuf, rel, fend);
                        w[0] = t.x; w[1] = t.y; w[2] = t.z; w[3] = t.w;
                    }
                }
                *reinterpret_cast<uint4 *>(dst + 16 * q) = make_uint4(w[0], w[1], w[2], w[3]);
            }
        }))
    } else {
        // ---- extract: gather the chunk's bit string G[lo, hi) into smem, XOR KS2, write words.
        // kx = S.kbuf + 3 so that frame word W sits at kx[W - basew] and the message words
        // W - 1 = 0 mod 4 start 16-byte aligned groups (basew is a multiple of 16).
        uint32_t *kx = S.kbuf + 3;
        const long long blk0 = lo >> 9;
        const long long base = blk0 * 512, basew = blk0 * 16;
        const int nblk = lo < hi ? (int)(((hi - 1) >> 9) - blk0 + 1) : 0;
        // the chunk's K2 keystream blocks go into kx first; every frame bit of [lo, hi) belongs to
        // exactly one 16-pixel group, which XORs its fields onto them (shared boundary words by
        // shared-memory atomics), so kx ends as G XOR KS2 with no zeroing or separate XOR pass
        if (tid < nblk) {
            uint32_t ks[16];
            chacha20_block(key, (uint32_t)(blk0 + tid), ks, g.dr);
#pragma unroll
            for (int j = 0; j < 16; j++) kx[tid * 16 + j] = bswap32(ks[j]);
        }
        __syncthreads();
        MMSB_BP_SWITCH(bp, METHOD, ({
            _Pragma("unroll")
            for (int r = 0; r < kScanRounds; r++) {
                if (!m[r]) continue;
                const uint4 u = S.spx[r * kScanThreads + tid];
                const uint32_t w[4] = {u.x, u.y, u.z, u.w};
                extract16<BP, SH>(w, m[r], kx, (int)((prefix + excl[r]) * BP - base), S.csel);
            }
        }))
        __syncthreads();
        uint32_t *mo = reinterpret_cast<uint32_t *>(msg_out + (size_t)img * stride);
        unsigned long long *parts = ws.parts + ((size_t)img * g.nchunks + chunk) * 2;
        if (lo < hi) {
            // frame words [w0, w1] (word indices < 7 HW / 32 fit 32 bits); the first and last
            // may be shared with the neighbouring chunks (merged by scan_finish), the ones in
            // between are this chunk's: the header word (W = 0) and message words W - 1 < wlim
            const int w0 = (int)(lo >> 5), w1 = (int)((hi - 1) >> 5), nw = w1 - w0 + 1;
            const bool hp = (lo & 31) != 0, tp = (hi & 31) != 0;
            const int wlim = (int)(stride / 4);
            const uint32_t *kb = kx - basew;                      // kb[W] = frame word W
            if (tid < 2 && (tid == 0 ? hp : (tp && !(nw == 1 && hp)))) {
                const int W = tid == 0 ? w0 : w1;
                const uint32_t v = kb[W];
                const long long s0 = (long long)W * 32 > lo ? (long long)W * 32 : lo;
                const long long e0 = (long long)W * 32 + 32 < hi ? (long long)W * 32 + 32 : hi;
                const int len = (int)(e0 - s0), st0 = (int)(s0 - (long long)W * 32);
                const uint32_t msk = (len == 32 ? 0xFFFFFFFFu : ((1u << len) - 1u)) << (32 - st0 - len);
                parts[W == w0 ? 0 : 1] = ((unsigned long long)(W + 1) << 32) | (v & msk);
            }
            const int o0 = w0 + (hp ? 1 : 0), o1 = w1 - (tp ? 1 : 0);   // own words [o0, o1]
            if (o0 == 0 && o1 >= 0 && tid == 0) ws.hdr[img] = kb[0];
            const int m0 = o0 > 1 ? o0 : 1, m1 = o1 < wlim ? o1 : wlim;   // own message words
            if (m0 <= m1) {
                // 16-byte groups W = a + 4 t (W - 1 = 0 mod 4) inside [m0, m1]; scalar words around
                const bool vec = (stride & 15) == 0 && (reinterpret_cast<uintptr_t>(mo) & 15) == 0;
                const int a = vec ? ((m0 + 2) & ~3) + 1 : m1 + 1;
                const int ng = a + 3 <= m1 ? (m1 - a + 1) >> 2 : 0;
                const int gend = ng ? a + 4 * ng : m0;              // first word after the groups
                for (int t = tid; t < ng; t += kScanThreads) {
                    const int W = a + 4 * t;
                    const uint4 v = *reinterpret_cast<const uint4 *>(kb + W);
                    *reinterpret_cast<uint4 *>(mo + W - 1) =
                        make_uint4(bswap32(v.x), bswap32(v.y), bswap32(v.z), bswap32(v.w));
                }
                // scalar words: [m0, min(a, m1 + 1)) before the groups, [gend, m1] after them
                const int hend = ng ? a : m1 + 1;
                const int nh = hend - m0, nt = ng ? m1 - gend + 1 : 0;
                for (int t = tid; t < nh + nt; t += kScanThreads) {
                    const int W = t < nh ? m0 + t : gend + (t - nh);
                    mo[W - 1] = bswap32(kb[W]);
                }
            }
        }
    }
}

}  // namespace mmsb
