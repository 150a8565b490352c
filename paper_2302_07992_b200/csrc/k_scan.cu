// k_scan.cu -- data hiding and extraction (a7-a9): capacity prefix scan by single-pass
// decoupled look-back over raster chunks, fused with the K2 keystream and the bit
// scatter (embed) / gather (extract).  Citations: P:<line> = /root/reference/PAPER.md.
//
// Frame (reading Q17): F = BE32(n) || message, n in bits; E_F = F XOR KS2 (K2 keystream,
// counter form: bit k lives in ChaCha20 block k/512).  Redundant pixels (map bit 0) of the
// rotated domain, in raster order (Q18), carry b' bits each: EMR b' = b at bit positions
// 1..b, LMR b' = b-1 at positions 2..b.  Zero pixel j carries frame bits
// [j b', (j+1) b'); only bits < |F| are written (Q19).
//
// One CTA (256 threads) per 16384-pixel raster chunk, in blockIdx order (chunk-major within
// an image).  The chunk arrives in shared memory by one bulk copy (cp.async.bulk + mbarrier),
// so the whole chunk is in flight before any thread computes; thread t owns the 16-pixel
// groups t, t+256, t+512, t+768 of the chunk.  A chunk publishes its zero count (aggregate)
// and, once the look-back has found its prefix, its inclusive count; the K2 keystream of the
// chunk's frame bits is one ChaCha20 block per thread.  The per-image epilogue (capacity and
// integrity checks, boundary words of the extracted string) runs in a second small kernel, so
// the chunk CTAs retire without a grid-wide completion counter.
#include "scan_chunk.cuh"

namespace mmsb {

template <int METHOD, bool EMBED>
__global__ void __launch_bounds__(kScanThreads, EMBED ? 5 : 6) scan_kernel(Geo g, const uint8_t *__restrict__ in,
                                                            uint8_t *__restrict__ out, const uint8_t *__restrict__ keys,
                                                            const uint8_t *__restrict__ msg,
                                                            const int64_t *__restrict__ msg_bits, long long stride,
                                                            uint8_t *__restrict__ msg_out, ScanWS ws,
                                                            const uint32_t *__restrict__ map_bits,
                                                            const int32_t *__restrict__ lmr_b) {
    __shared__ ScanSmem<METHOD, EMBED> S;
    scan_chunk<METHOD, EMBED>(S, g, blockIdx.x / g.nchunks, blockIdx.x % g.nchunks, in, out, keys, msg, msg_bits,
                              stride, msg_out, ws, map_bits, lmr_b);
}

// ======================================================================================
// frame_block: E_F = F XOR KS2 for one ChaCha20 block of the frame (reading Q17):
// F = BE32(n) || message, block k = frame words [16k, 16k+16).  Independent of the pixels,
// so it runs at full occupancy before the chunk kernel, which copies the words it needs.
// ======================================================================================
__device__ __forceinline__ void frame_block(const Geo &g, const uint8_t *__restrict__ keys,
                                            const uint8_t *__restrict__ msg, const int64_t *__restrict__ msg_bits,
                                            long long stride, const ScanWS &ws, int img, long long k) {
    const long long n = msg_bits[img];
    const bool n_ok = n >= 0 && n <= 8 * stride && n <= 0xFFFFFFFFll;
    const long long F = n_ok ? 32 + n : 0;
    const long long nblk = (F + 511) / 512 < ws.ef_words / 16 ? (F + 511) / 512 : ws.ef_words / 16;
    if (k >= nblk) return;
    uint32_t key[8];
    load_key(keys, img, key);
    uint32_t ks[16];
    chacha20_block(key, (uint32_t)k, ks, g.dr);
    const uint32_t *mw = reinterpret_cast<const uint32_t *>(msg + (size_t)img * stride);
    const long long nmw = stride / 4;                            // message words in the row
    uint32_t o[16];
    if (k > 0 && k * 16 + 15 < nmw && (reinterpret_cast<uintptr_t>(mw) & 15) == 0) {
        // a block inside the message row: frame words 16k .. 16k+15 = message words 16k-1 .. 16k+14, one
        // scalar and four 16-byte loads; bswap(m) ^ bswap(ks) = bswap(m ^ ks)
        const uint4 *mv = reinterpret_cast<const uint4 *>(mw + k * 16);
        const uint32_t m0 = __ldg(mw + k * 16 - 1);
        const uint4 v0 = __ldg(mv), v1 = __ldg(mv + 1), v2 = __ldg(mv + 2), v3 = __ldg(mv + 3);
        const uint32_t m[16] = {m0, v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w, v2.x, v2.y, v2.z, v2.w, v3.x, v3.y, v3.z};
#pragma unroll
        for (int j = 0; j < 16; j++) o[j] = bswap32(m[j] ^ ks[j]);
    } else {
#pragma unroll
        for (int j = 0; j < 16; j++) {
            const long long wi = k * 16 + j;
            uint32_t fw;
            if (wi == 0) fw = (uint32_t)n;
            else if (wi - 1 < nmw) fw = bswap32(__ldg(mw + (wi - 1)));
            else fw = 0;
            o[j] = fw ^ bswap32(ks[j]);
        }
    }
    uint4 *dst = reinterpret_cast<uint4 *>(ws.ef + (size_t)img * ws.ef_words + k * 16);
#pragma unroll
    for (int j = 0; j < 4; j++) dst[j] = make_uint4(o[4 * j], o[4 * j + 1], o[4 * j + 2], o[4 * j + 3]);
}

// embed_prep_kernel: embed's two pre-passes in one launch, their CTAs interleaved so that the
// memory-bound counting (one CTA per chunk) overlaps the ALU-bound frame encryption (256
// ChaCha blocks per CTA): even CTAs count while both kinds remain, odd ones encrypt.
template <int METHOD>
__global__ void __launch_bounds__(kScanThreads) embed_prep_kernel(Geo g, const uint8_t *__restrict__ in,
                                                                  const uint32_t *__restrict__ map_bits,
                                                                  const uint8_t *__restrict__ keys,
                                                                  const uint8_t *__restrict__ msg,
                                                                  const int64_t *__restrict__ msg_bits,
                                                                  long long stride, ScanWS ws, int ncount, int fpi) {
    const int nframe = g.B * fpi, both = ncount < nframe ? ncount : nframe;
    const int i = blockIdx.x;
    bool count;
    int idx;
    if (i < 2 * both) { count = (i & 1) == 0; idx = i >> 1; }
    else { count = ncount > nframe; idx = both + (i - 2 * both); }
    if (count) {
        count_chunk<METHOD>(g, in, map_bits, ws, idx);
    } else {
        const int img = idx / fpi;
        frame_block(g, keys, msg, msg_bits, stride, ws, img, (long long)(idx % fpi) * kScanThreads + threadIdx.x);
    }
}

// ======================================================================================
// scan_finish_kernel: one CTA per image, after the chunk kernel.
//   embed:   C = b' * (inclusive zero count of the last chunk); status OK if 32 + n <= C
//            (P:750), else CAPACITY (E_INVAL for an invalid n) and the marked image is reset
//            to the encrypted one; EMR FORMAT (b-field > 5) -> status FORMAT.
//   extract: merges the boundary words of the extracted string (several chunks can share a
//            word), checks n = BE32 header <= C - 32 (else INTEGRITY, nothing kept), zeroes
//            the capacity region past n.
// ======================================================================================
template <int METHOD, bool EMBED>
__global__ void __launch_bounds__(256) scan_finish_kernel(Geo g, const uint8_t *__restrict__ in,
                                                          uint8_t *__restrict__ out,
                                                          const int64_t *__restrict__ msg_bits, long long stride,
                                                          uint8_t *__restrict__ msg_out,
                                                          int64_t *__restrict__ msg_bits_out,
                                                          int32_t *__restrict__ status, ScanWS ws,
                                                          const int32_t *__restrict__ lmr_b) {
    __shared__ long long sh[2];
    const int img = blockIdx.x, tid = threadIdx.x;
    const uint8_t *src = in + (size_t)img * g.HW;
    const int b = image_b<METHOD>(src, lmr_b, img);
    if (b < 2) {
        if (tid == 0) {
            if constexpr (METHOD == 0) status[img] = 8;      // FORMAT; LMR: set by the decoder
            if constexpr (!EMBED) msg_bits_out[img] = -1;
        }
        return;
    }
    const int bp = METHOD == 0 ? b : b - 1;
    if constexpr (EMBED) {
        // the chunk kernel embedded nothing unless the frame fits: CAPACITY leaves marked ==
        // encrypted without a copy here
        const long long C = (long long)__ldcg(ws.ztot + img) * bp;
        const long long n = msg_bits[img];
        const bool n_ok = n >= 0 && n <= 8 * stride && n <= 0xFFFFFFFFll;
        const bool fits = n_ok && 32 + n <= C;
        if (tid == 0) status[img] = fits ? 0 : (n_ok ? 3 : 2);
    } else {
        const unsigned long long last = ld_acquire(ws.states + (size_t)img * g.nchunks + g.nchunks - 1);
        const long long C = (long long)(last & kValMask) * bp;
        uint32_t *mo = reinterpret_cast<uint32_t *>(msg_out + (size_t)img * stride);
        const unsigned long long *pp = ws.parts + (size_t)img * g.nchunks * 2;
        const long long rw = C > 32 ? (C - 32 + 31) / 32 : 0;
        const bool fits = 4 * rw <= stride;
        // shared words: zero them, then OR every part in (byte order commutes with OR)
        for (int k = tid; k < 2 * g.nchunks; k += 256) {
            const unsigned long long v = __ldcg(pp + k);
            if (!v) continue;
            const long long W = (long long)(v >> 32) - 1;
            if (W == 0) ws.hdr[img] = 0;
            else if (4 * W <= stride) mo[W - 1] = 0;
        }
        __syncthreads();
        for (int k = tid; k < 2 * g.nchunks; k += 256) {
            const unsigned long long v = __ldcg(pp + k);
            if (!v) continue;
            const long long W = (long long)(v >> 32) - 1;
            if (W == 0) atomicOr(ws.hdr + img, (uint32_t)v);
            else if (4 * W <= stride) atomicOr(mo + (W - 1), bswap32((uint32_t)v));
        }
        __syncthreads();
        if (tid == 0) {
            const bool lost = __ldcg(ws.err + img) != 0;     // a look-back wait timed out
            const long long n = C >= 32 ? (long long)__ldcg(ws.hdr + img) : -1;
            const bool ok = !lost && fits && C >= 32 && n <= C - 32;
            sh[0] = fits ? C : 0;
            sh[1] = ok ? n : -1;
            msg_bits_out[img] = ok ? n : -1;
            status[img] = lost ? 6 : ok ? 0 : (fits ? 4 : 2);  // region beyond the caller's rows: E_INVAL
        }
        __syncthreads();
        const long long Cf = sh[0], nn = sh[1];
        const long long region_w = Cf > 32 ? (Cf - 32 + 31) / 32 : 0;
        const long long keep = nn < 0 ? 0 : nn;                // INTEGRITY -> zero everything
        for (long long W = keep / 32 + tid; W < region_w; W += 256) {
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
    if constexpr (EMBED) {
        const long long fb = (32 + 8 * stride + 511) / 512;     // frame blocks (capped by ef_words in the kernel)
        const long long nb = fb < ws.ef_words / 16 ? fb : ws.ef_words / 16;
        const int fpi = (int)((nb + kScanThreads - 1) / kScanThreads);       // frame CTAs per image
        embed_prep_kernel<METHOD><<<grid + (unsigned)(g.B * fpi), kScanThreads, 0, st>>>(
            g, in, map_bits, keys, msg, msg_bits, stride, ws, (int)grid, fpi);
    }
    scan_kernel<METHOD, EMBED><<<grid, kScanThreads, 0, st>>>(g, in, out, keys, msg, msg_bits, stride, msg_out, ws,
                                                              map_bits, lmr_b);
    scan_finish_kernel<METHOD, EMBED><<<g.B, 256, 0, st>>>(g, in, out, msg_bits, stride, msg_out, msg_bits_out,
                                                           status, ws, lmr_b);
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
// capacity_kernel: the capacity an encrypted / marked image offers (the
// SPEC's capacity query), as the hider and the K2 receiver derive it: b from the header (EMR:
// 3 LSBs, Q14; LMR: the decoded MSB-plane header) and C = b' * (redundant pixels of the
// location map).  One CTA per image.
// ======================================================================================
template <int METHOD>
__global__ void __launch_bounds__(256) capacity_kernel(Geo g, const uint8_t *__restrict__ in,
                                                       const uint32_t *__restrict__ map_bits,
                                                       const int32_t *__restrict__ lmr_b, int32_t *__restrict__ b_out,
                                                       int64_t *__restrict__ cap_out, int32_t *__restrict__ status) {
    __shared__ unsigned long long red[8];
    const int img = blockIdx.x, tid = threadIdx.x;
    const uint8_t *src = in + (size_t)img * g.HW;
    const int b = image_b<METHOD>(src, lmr_b, img);
    if (b < 2) {                                              // EMR FORMAT; LMR status from the header kernel
        if (tid == 0) {
            b_out[img] = 0;
            cap_out[img] = 0;
            if constexpr (METHOD == 0) status[img] = 8;
        }
        return;
    }
    unsigned long long z = 0;
    for (long long q = tid; q < g.HW / 16; q += 256) {
        if constexpr (METHOD == 0) {
            z += __popc(zero_mask16<0>(__ldg(reinterpret_cast<const uint4 *>(src) + q), q == 0, nullptr, 0));
        } else {
            const long long pb = (long long)img * g.HW + 16 * q;
            z += __popc(~(__ldg(map_bits + (pb >> 5)) >> (pb & 31)) & 0xFFFFu);
        }
    }
#pragma unroll
    for (int s2 = 16; s2 > 0; s2 >>= 1) z += __shfl_xor_sync(0xffffffffu, z, s2);
    if ((tid & 31) == 0) red[tid >> 5] = z;
    __syncthreads();
    if (tid == 0) {
        unsigned long long t = 0;
        for (int w = 0; w < 8; w++) t += red[w];
        b_out[img] = b;
        cap_out[img] = (long long)(METHOD == 0 ? b : b - 1) * (long long)t;
        status[img] = 0;
    }
}

void launch_capacity(const Geo &g, const uint8_t *in, const uint32_t *map_bits, const int32_t *lmr_b,
                     int32_t *b_out, int64_t *cap_out, int32_t *status, cudaStream_t st) {
    if (g.method == 0) capacity_kernel<0><<<g.B, 256, 0, st>>>(g, in, map_bits, lmr_b, b_out, cap_out, status);
    else capacity_kernel<1><<<g.B, 256, 0, st>>>(g, in, map_bits, lmr_b, b_out, cap_out, status);
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

// both-keys receiver: the image's status is the extraction's unless that was OK
__global__ void status_merge_kernel(int B, const int32_t *__restrict__ second, int32_t *__restrict__ status) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < B && status[i] == 0) status[i] = second[i];
}

void launch_status_merge(int B, const int32_t *second, int32_t *status, cudaStream_t st) {
    status_merge_kernel<<<(B + 255) / 256, 256, 0, st>>>(B, second, status);
}

void launch_stats(long long HW, int B, const uint8_t *a, const uint8_t *b, int64_t *sse, cudaStream_t st) {
    const long long n16 = HW / 16;
    int bx = (int)((n16 + 256 * 8 - 1) / (256 * 8));
    if (bx < 1) bx = 1;
    dim3 grid(bx, B);
    stats_kernel<<<grid, 256, 0, st>>>(HW, a, b, reinterpret_cast<unsigned long long *>(sse));
}

}  // namespace mmsb
