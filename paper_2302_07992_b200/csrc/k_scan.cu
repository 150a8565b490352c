// k_scan.cu -- data hiding and extraction (a7-a9): capacity prefix scan by single-pass
// decoupled look-back over raster chunks, fused with the K2 keystream and the bit
// scatter (embed) / gather (extract).  Citations: P:<line> = /root/reference/PAPER.md.
//
// Frame (reading Q17): F = BE32(n) || message, n in bits; E_F = F XOR KS2 (K2 keystream,
// counter form: bit k lives in ChaCha20 block k/512).  Redundant pixels (map bit 0) of the
// rotated domain, in raster order (Q18), carry b' bits each: EMR b' = b at bit positions
// 1..b, LMR b' = b-1 at positions 2..b.  Zero pixel j carries frame bits
// [j b', (j+1) b'); only bits < |F| are written (Q19).
#include "mmsb_device.cuh"
#include "mmsb_kernels.h"

namespace mmsb {

constexpr unsigned long long kFlagAgg = 1ull << 62, kFlagInc = 2ull << 62, kValMask = (1ull << 62) - 1;
constexpr int kKbufWords = kChunk * 7 / 32 + 64;   // bits of one chunk + block alignment + pad

__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t x, uint32_t *wsum, uint32_t &total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t v = x;
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
        uint32_t t = __shfl_up_sync(0xffffffffu, v, s);
        if (lane >= s) v += t;
    }
    if (lane == 31) wsum[wid] = v;
    __syncthreads();
    uint32_t off = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < kScanThreads / 32; w++) {
        const uint32_t ws = wsum[w];
        if (w < wid) off += ws;
        tot += ws;
    }
    __syncthreads();
    total = tot;
    return off + v - x;
}

// 16 zero-pixel flags of the pixels [p, p+16) of image img (bit i = pixel p+i is redundant)
template <int METHOD>
__device__ __forceinline__ uint32_t zero_mask16(const uint4 &u, long long p, long long bitbase,
                                                const uint32_t *__restrict__ map_bits) {
    if constexpr (METHOD == 0) {
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
        uint32_t m = 0;
#pragma unroll
        for (int i = 0; i < 4; i++) {
            const uint32_t l = ~w[i] & 0x01010101u;              // LSB == 0 -> redundant
            m |= ((l | (l >> 7) | (l >> 14) | (l >> 21)) & 0xFu) << (4 * i);
        }
        if (p == 0) m &= ~7u;                                    // r = 0..2 hold the header (Q14)
        return m;
    } else {
        const long long bit = bitbase + p;
        return ~(__ldg(map_bits + (bit >> 5)) >> (bit & 31)) & 0xFFFFu;
    }
}

// ---- per-thread bit streams of 16 pixels, specialised on b' (bits per redundant pixel) and
// on the bit position of the carried field (SHIFT = 8 - b for EMR, 7 - b' for LMR).

// embed: the zero pixels of mm receive consecutive b'-bit groups of the frame bits held in
// kbuf (big-endian bit order), starting at relative bit `rel`; bits at or past `fend` are
// not written (a partially filled last pixel keeps its remaining bits, reading Q19).
template <int BP, int SHIFT>
__device__ __forceinline__ void embed16(uint32_t w[4], uint32_t mm, const uint32_t *kbuf, long long rel,
                                        long long fend) {
    const int cnt = __popc(mm);
    if (!cnt || rel >= fend) return;
    constexpr uint32_t FM = ((1u << BP) - 1u) << SHIFT;
    if (rel + (long long)cnt * BP <= fend) {
        int wi = (int)(rel >> 5);
        const int off = (int)(rel & 31);
        unsigned long long win = (((unsigned long long)kbuf[wi] << 32) | kbuf[wi + 1]) << off;
        int avail = 64 - off;
        wi += 2;
#pragma unroll
        for (int i = 0; i < 16; i++) {
            if ((mm >> i) & 1u) {
                if (avail < BP) {
                    win |= (unsigned long long)kbuf[wi++] << (32 - avail);
                    avail += 32;
                }
                const uint32_t val = (uint32_t)(win >> (64 - BP));
                w[i >> 2] = (w[i >> 2] & ~(FM << (8 * (i & 3)))) | (val << (SHIFT + 8 * (i & 3)));
                win <<= BP;
                avail -= BP;
            }
        }
    } else {
        long long k = rel;
#pragma unroll
        for (int i = 0; i < 16; i++) {
            if (((mm >> i) & 1u) && k < fend) {
                const int nb = (fend - k) < BP ? (int)(fend - k) : BP;
                const int wv = (int)(k >> 5), off = (int)(k & 31);
                const unsigned long long win = ((unsigned long long)kbuf[wv] << 32) | kbuf[wv + 1];
                const uint32_t val = (uint32_t)(win >> (64 - off - BP)) & ((1u << BP) - 1u);
                const uint32_t msk = (((1u << nb) - 1u) << (BP - nb)) << SHIFT;
                w[i >> 2] = (w[i >> 2] & ~(msk << (8 * (i & 3)))) | (((val << SHIFT) & msk) << (8 * (i & 3)));
            }
            if ((mm >> i) & 1u) k += BP;
        }
    }
}

// extract: the zero pixels' b'-bit fields are appended in raster order and ORed into kbuf at
// relative bit `rel`; the first and the last (partial) words are shared with the neighbouring
// threads (shared-memory atomics), the words in between belong to this thread alone.
template <int BP, int SHIFT>
__device__ __forceinline__ void extract16(const uint32_t w[4], uint32_t mm, uint32_t *kbuf, long long rel) {
    if (!mm) return;
    int wi = (int)(rel >> 5);
    int nacc = (int)(rel & 31);                 // leading pad (zeros) up to the word boundary
    unsigned long long acc = 0;
    bool first = true;
#pragma unroll
    for (int i = 0; i < 16; i++) {
        if ((mm >> i) & 1u) {
            const uint32_t val = (w[i >> 2] >> (8 * (i & 3) + SHIFT)) & ((1u << BP) - 1u);
            acc = (acc << BP) | val;
            nacc += BP;
            if (nacc >= 32) {
                const uint32_t word = (uint32_t)(acc >> (nacc - 32));
                if (first) atomicOr(&kbuf[wi], word);
                else kbuf[wi] = word;
                first = false;
                wi++;
                nacc -= 32;
            }
        }
    }
    if (nacc > 0) atomicOr(&kbuf[wi], (uint32_t)(acc & ((1ull << nacc) - 1ull)) << (32 - nacc));
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

template <int METHOD, bool EMBED>
__global__ void __launch_bounds__(kScanThreads, 8) scan_kernel(Geo g, const uint8_t *__restrict__ in,
                                                            uint8_t *__restrict__ out, const uint8_t *__restrict__ keys,
                                                            const uint8_t *__restrict__ msg,
                                                            const int64_t *__restrict__ msg_bits, long long stride,
                                                            uint8_t *__restrict__ msg_out,
                                                            int64_t *__restrict__ msg_bits_out,
                                                            int32_t *__restrict__ status, ScanWS ws,
                                                            const uint32_t *__restrict__ map_bits,
                                                            const int32_t *__restrict__ lmr_b) {
    __shared__ uint32_t wsum[kScanThreads / 32];
    __shared__ uint32_t kbuf[kKbufWords];
    __shared__ long long sh_ll[4];
    __shared__ int sh_i[4];

    const int tid = threadIdx.x;
    if (tid == 0) sh_i[0] = (int)atomicAdd(ws.ticket, 1u);
    __syncthreads();
    const int ticket = sh_i[0];
    const int img = ticket / g.nchunks, chunk = ticket % g.nchunks;
    const uint8_t *src = in + (size_t)img * g.HW;

    int b, bp;
    if constexpr (METHOD == 0) {
        const int field = ((src[0] & 1) << 2) | ((src[1] & 1) << 1) | (src[2] & 1);
        b = field > 5 ? 0 : field + 2;
        bp = b;
    } else {
        b = lmr_b[img];
        bp = b - 1;
    }
    const long long p0 = (long long)chunk * kChunk;
    if (b < 2) {                                            // FORMAT (EMR) / BADCASE, FORMAT (LMR)
        if constexpr (EMBED) {
            for (long long p = p0 + tid * 16; p < p0 + kChunk && p < g.HW; p += kScanThreads * 16)
                *reinterpret_cast<uint4 *>(out + (size_t)img * g.HW + p) =
                    __ldg(reinterpret_cast<const uint4 *>(src + p));
        }
        if (chunk == 0 && tid == 0) {
            if constexpr (METHOD == 0) status[img] = 8;
            if constexpr (!EMBED) msg_bits_out[img] = -1;
        }
        return;
    }

    // ---- per-thread zero masks (2 rounds x 16 px) and the block-local exclusive scan
    uint4 pix[2];
    uint32_t m[2], cnt[2], excl[2], tot[2];
#pragma unroll
    for (int r = 0; r < 2; r++) {
        const long long p = p0 + r * (kScanThreads * 16) + tid * 16;
        if (p < g.HW) {
            pix[r] = __ldg(reinterpret_cast<const uint4 *>(src + p));
            m[r] = zero_mask16<METHOD>(pix[r], p, (long long)img * g.HW, map_bits);
        } else {
            pix[r] = make_uint4(0, 0, 0, 0);
            m[r] = 0;
        }
        cnt[r] = __popc(m[r]);
    }
    excl[0] = block_exclusive_scan(cnt[0], wsum, tot[0]);
    excl[1] = block_exclusive_scan(cnt[1], wsum, tot[1]) + tot[0];
    const unsigned long long agg = (unsigned long long)tot[0] + tot[1];

    // ---- single-pass decoupled look-back over the image's chunks (ticket order = issue order).
    // Warp 0 publishes this chunk's aggregate, then inspects 32 predecessors per probe: every
    // lane spins on its own predecessor until that one has published, the nearest inclusive
    // prefix ends the walk, aggregates in front of it are summed (warp reduction).
    if (tid < 32) {
        unsigned long long *st = ws.states + (size_t)img * g.nchunks;
        unsigned long long prefix = 0;
        if (chunk == 0) {
            if (tid == 0) st_release(st, kFlagInc | agg);
        } else {
            if (tid == 0) st_release(st + chunk, kFlagAgg | agg);
            int base = chunk - 1;
            while (true) {
                const int k = base - tid;
                unsigned long long v = kFlagInc;                 // before chunk 0: inclusive 0
                if (k >= 0) {
                    do { v = ld_acquire(st + k); } while ((v & ~kValMask) == 0);
                }
                const unsigned inc = __ballot_sync(0xffffffffu, (v & ~kValMask) == kFlagInc);
                const int last = inc ? __ffs(inc) - 1 : 31;
                unsigned long long val = tid <= last ? (v & kValMask) : 0ull;
#pragma unroll
                for (int s2 = 16; s2 > 0; s2 >>= 1) val += __shfl_xor_sync(0xffffffffu, val, s2);
                prefix += val;
                if (inc) break;
                base -= 32;
            }
            if (tid == 0) st_release(st + chunk, kFlagInc | (prefix + agg));
        }
        if (tid == 0) sh_ll[0] = (long long)prefix;
    }
    __syncthreads();
    const long long prefix = sh_ll[0];
    const long long lo = prefix * bp, hi = (prefix + (long long)agg) * bp;

    uint32_t key[8];
    load_key(keys, img, key);

    if constexpr (EMBED) {
        const long long n = msg_bits[img];
        const bool n_ok = n >= 0 && n <= 8 * stride && n <= 0xFFFFFFFFll;
        const long long F = n_ok ? 32 + n : 0;
        const long long hie = hi < F ? hi : F;
        const long long blk0 = lo >> 9;
        if (lo < hie) {
            const int nblk = (int)(((hie - 1) >> 9) - blk0 + 1);
            const uint8_t *mimg = msg + (size_t)img * stride;
            for (int t0 = 0; t0 < nblk; t0 += kScanThreads / 4) {       // 4 lanes per ChaCha block
                const int t = t0 + (tid >> 2), cl = tid & 3;
                uint32_t ks[4];
                chacha20_block_x4(key, (uint32_t)(blk0 + t), ks);
                if (t < nblk) {
#pragma unroll
                    for (int j = 0; j < 4; j++) {
                        const long long wi = (blk0 + t) * 16 + 4 * j + cl;   // frame word index (BE)
                        uint32_t fw;
                        if (wi == 0) fw = (uint32_t)n;
                        else if (4 * wi <= stride) fw = bswap32(__ldg(reinterpret_cast<const uint32_t *>(mimg) + (wi - 1)));
                        else fw = 0;
                        kbuf[t * 16 + 4 * j + cl] = fw ^ bswap32(ks[j]);
                    }
                }
            }
            if (tid == 0) kbuf[nblk * 16] = 0;
        }
        __syncthreads();
        const long long base = blk0 * 512;
#pragma unroll
        for (int r = 0; r < 2; r++) {
            const long long p = p0 + r * (kScanThreads * 16) + tid * 16;
            if (p >= g.HW) continue;
            uint32_t w[4] = {pix[r].x, pix[r].y, pix[r].z, pix[r].w};
            const long long rel = (prefix + excl[r]) * bp - base;
            MMSB_BP_SWITCH(bp, METHOD, (embed16<BP, SH>(w, m[r], kbuf, rel, hie - base)))
            *reinterpret_cast<uint4 *>(out + (size_t)img * g.HW + p) = make_uint4(w[0], w[1], w[2], w[3]);
        }
        // ---- the image's last CTA decides the capacity outcome (32 + n <= C)
        __syncthreads();
        if (tid == 0) {
            __threadfence();
            sh_i[1] = atomicAdd(ws.done + img, 1u) == (unsigned)(g.nchunks - 1);
        }
        __syncthreads();
        if (sh_i[1]) {
            __threadfence();
            const unsigned long long last = ld_acquire(ws.states + (size_t)img * g.nchunks + g.nchunks - 1);
            const long long C = (long long)(last & kValMask) * bp;
            const bool fits = n_ok && 32 + n <= C;
            if (!fits) {                                         // CAPACITY: marked = encrypted
                for (long long p = tid * 16; p < g.HW; p += kScanThreads * 16)
                    *reinterpret_cast<uint4 *>(out + (size_t)img * g.HW + p) =
                        __ldg(reinterpret_cast<const uint4 *>(src + p));
            }
            if (tid == 0) status[img] = fits ? 0 : (n_ok ? 3 : 2);
        }
    } else {
        // ---- extract: gather the chunk's bit string G[lo, hi) into smem, XOR KS2, write words
        const long long blk0 = lo >> 9;
        const long long base = blk0 * 512, basew = blk0 * 16;
        int nblk = 0;
        if (lo < hi) {
            nblk = (int)(((hi - 1) >> 9) - blk0 + 1);
            for (int t = tid; t < nblk * 16 + 1; t += kScanThreads) kbuf[t] = 0;
        }
        __syncthreads();
        if (lo < hi) {
#pragma unroll
            for (int r = 0; r < 2; r++) {
                const uint32_t w[4] = {pix[r].x, pix[r].y, pix[r].z, pix[r].w};
                const long long rel = (prefix + excl[r]) * bp - base;
                MMSB_BP_SWITCH(bp, METHOD, (extract16<BP, SH>(w, m[r], kbuf, rel)))
            }
        }
        __syncthreads();
        for (int t0 = 0; t0 < nblk; t0 += kScanThreads / 4) {           // 4 lanes per ChaCha block
            const int t = t0 + (tid >> 2), cl = tid & 3;
            uint32_t ks[4];
            chacha20_block_x4(key, (uint32_t)(blk0 + t), ks);
            if (t < nblk) {
#pragma unroll
                for (int j = 0; j < 4; j++) kbuf[t * 16 + 4 * j + cl] ^= bswap32(ks[j]);
            }
        }
        __syncthreads();
        uint32_t *mo = reinterpret_cast<uint32_t *>(msg_out + (size_t)img * stride);
        unsigned long long *parts = ws.parts + ((size_t)img * g.nchunks + chunk) * 2;
        if (lo < hi) {
            const long long w0 = lo >> 5, w1 = (hi - 1) >> 5;
            for (long long W = w0 + tid; W <= w1; W += kScanThreads) {
                const long long s0 = W * 32 > lo ? W * 32 : lo;
                const long long e0 = W * 32 + 32 < hi ? W * 32 + 32 : hi;
                uint32_t v = kbuf[W - basew];
                if (s0 == W * 32 && e0 == W * 32 + 32) {
                    if (W == 0) ws.hdr[img] = v;
                    else if (4 * W <= stride) mo[W - 1] = bswap32(v);
                } else {
                    const int len = (int)(e0 - s0), st0 = (int)(s0 - W * 32);
                    const uint32_t msk = (len == 32 ? 0xFFFFFFFFu : ((1u << len) - 1u)) << (32 - st0 - len);
                    parts[W == w0 ? 0 : 1] = ((unsigned long long)(W + 1) << 32) | (v & msk);
                }
            }
        }
        // ---- the image's last CTA: combine boundary words, check the length, zero the tail
        __syncthreads();
        if (tid == 0) {
            __threadfence();
            sh_i[1] = atomicAdd(ws.done + img, 1u) == (unsigned)(g.nchunks - 1);
        }
        __syncthreads();
        if (!sh_i[1]) return;
        __threadfence();
        if (tid == 0) {
            const unsigned long long *pp = ws.parts + (size_t)img * g.nchunks * 2;
            long long cw = -1;
            uint32_t cv = 0;
            for (int k = 0; k < 2 * g.nchunks; k++) {
                const unsigned long long v = __ldcg(pp + k);
                if (!v) continue;
                const long long W = (long long)(v >> 32) - 1;
                if (W == cw) {
                    cv |= (uint32_t)v;
                } else {
                    if (cw == 0) ws.hdr[img] = cv;
                    else if (cw > 0 && 4 * cw <= stride) mo[cw - 1] = bswap32(cv);
                    cw = W;
                    cv = (uint32_t)v;
                }
            }
            if (cw == 0) ws.hdr[img] = cv;
            else if (cw > 0 && 4 * cw <= stride) mo[cw - 1] = bswap32(cv);
            __threadfence_block();
            const unsigned long long last = ld_acquire(ws.states + (size_t)img * g.nchunks + g.nchunks - 1);
            const long long C = (long long)(last & kValMask) * bp;
            const long long rw = C > 32 ? (C - 32 + 31) / 32 : 0;
            const bool fits = 4 * rw <= stride;
            const long long n = C >= 32 ? (long long)__ldcg(ws.hdr + img) : -1;
            const bool ok = fits && C >= 32 && n <= C - 32;
            sh_ll[1] = fits ? C : 0;
            sh_ll[2] = ok ? n : -1;
            msg_bits_out[img] = ok ? n : -1;
            status[img] = ok ? 0 : (fits ? 4 : 2);           // region beyond the caller's rows: E_INVAL
        }
        __syncthreads();
        const long long C = sh_ll[1], n = sh_ll[2];
        const long long region_w = C > 32 ? (C - 32 + 31) / 32 : 0;
        const long long keep = n < 0 ? 0 : n;                  // INTEGRITY -> zero everything
        for (long long W = keep / 32 + tid; W < region_w; W += kScanThreads) {
            uint32_t v = 0;
            if (W == keep / 32 && (keep & 31)) v = bswap32(__ldcg(mo + W)) & ~(0xFFFFFFFFu >> (keep & 31));
            mo[W] = bswap32(v);
        }
    }
}

template <int METHOD, bool EMBED>
static void launch_scan_t(const Geo &g, const uint8_t *in, uint8_t *out, const uint8_t *keys, const uint8_t *msg,
                          const int64_t *msg_bits, long long stride, uint8_t *msg_out, int64_t *msg_bits_out,
                          int32_t *status, const ScanWS &ws, const uint32_t *map_bits, const int32_t *lmr_b,
                          cudaStream_t st) {
    const unsigned grid = (unsigned)((long long)g.B * g.nchunks);
    scan_kernel<METHOD, EMBED><<<grid, kScanThreads, 0, st>>>(g, in, out, keys, msg, msg_bits, stride, msg_out,
                                                              msg_bits_out, status, ws, map_bits, lmr_b);
}

void launch_scan(const Geo &g, bool embed, const uint8_t *in, uint8_t *out, const uint8_t *keys, const uint8_t *msg,
                 const int64_t *msg_bits, long long stride, uint8_t *msg_out, int64_t *msg_bits_out, int32_t *status,
                 const ScanWS &ws, const uint32_t *map_bits, const int32_t *lmr_b, cudaStream_t st) {
    if (g.method == 0) {
        if (embed) launch_scan_t<0, true>(g, in, out, keys, msg, msg_bits, stride, msg_out, msg_bits_out, status, ws, map_bits, lmr_b, st);
        else launch_scan_t<0, false>(g, in, out, keys, msg, msg_bits, stride, msg_out, msg_bits_out, status, ws, map_bits, lmr_b, st);
    } else {
        if (embed) launch_scan_t<1, true>(g, in, out, keys, msg, msg_bits, stride, msg_out, msg_bits_out, status, ws, map_bits, lmr_b, st);
        else launch_scan_t<1, false>(g, in, out, keys, msg, msg_bits, stride, msg_out, msg_bits_out, status, ws, map_bits, lmr_b, st);
    }
}

// ======================================================================================
// stats_kernel: per-image sum of squared differences, int64 via block reduction.
// ======================================================================================
__global__ void __launch_bounds__(256) stats_kernel(long long HW, const uint8_t *__restrict__ a,
                                                    const uint8_t *__restrict__ b, unsigned long long *__restrict__ sse) {
    __shared__ unsigned long long red[8];
    const int img = blockIdx.y;
    const uint4 *pa = reinterpret_cast<const uint4 *>(a + (size_t)img * HW);
    const uint4 *pb = reinterpret_cast<const uint4 *>(b + (size_t)img * HW);
    const long long n16 = HW / 16;
    unsigned long long acc = 0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (long long)gridDim.x * blockDim.x) {
        const uint4 u = __ldg(pa + i), v = __ldg(pb + i);
        const uint32_t x[4] = {u.x, u.y, u.z, u.w}, y[4] = {v.x, v.y, v.z, v.w};
        uint32_t s = 0;
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const uint32_t d = __vabsdiffu4(x[k], y[k]);
#pragma unroll
            for (int j = 0; j < 4; j++) {
                const uint32_t dj = (d >> (8 * j)) & 0xFFu;
                s += dj * dj;
            }
        }
        acc += s;
    }
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t = 0;
        for (int w = 0; w < 8; w++) t += red[w];
        if (t) atomicAdd(sse + img, t);
    }
}

void launch_stats(long long HW, int B, const uint8_t *a, const uint8_t *b, int64_t *sse, cudaStream_t st) {
    const long long n16 = HW / 16;
    int bx = (int)((n16 + 256 * 8 - 1) / (256 * 8));
    if (bx < 1) bx = 1;
    dim3 grid(bx, B);
    stats_kernel<<<grid, 256, 0, st>>>(HW, a, b, reinterpret_cast<unsigned long long *>(sse));
}

}  // namespace mmsb
