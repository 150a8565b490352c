// k_lmr.cu -- LMR-RDHEI specific kernels: the bi-level tile coder that stands in
// for JBIG-KIT (builder-defined, reading Q16), the candidate walk until the coded maps
// fit the first-MSB plane, the MSB-plane writer and the decoders used by
// the hider, the K2 receiver and the K1 receiver.
//
// Coder (O15): tiles of side min(2^t, dim) coded independently in tile raster
// order; 9-pixel causal tile-local context (Q16), MSB->LSB (0,-1) (-1,-2) (-1,-1)
// (-1,0) (-1,+1) (-1,+2) (-2,-1) (-2,0) (-2,+1), out-of-tile pixels 0; per context a 16-bit
// probability of a 0, p0 = 32768 initially, p0 += (65536-p0)>>4 after a 0, p0 -= p0>>4 after
// a 1; carry-propagating range coder, 32-bit range, bound = (range>>16)*p0, renormalise below
// 2^24 one byte at a time through a cache byte + 0xFF run, flush = 5 byte shifts; the
// decoder reads bytes past the end of the tile's stream as 0.
//
// One GPU thread codes one tile (the coder is serial within a tile); its model (512 x u16)
// lives in shared memory.  The fast kernels (tiles 32, 64 or 128 wide: every configured shape)
// run 112-thread CTAs with a branch-free symbol step; the reference kernels
// (coder_encode_kernel / coder_decode_kernel, one warp per CTA, model entry ctx of lane l at u16
// index ctx*32 + l) serve narrower tiles.  Candidate maps are coded in waves (mmsb_kernels.h).
#include <algorithm>

#include "mmsb_device.cuh"
#include "mmsb_kernels.h"

namespace mmsb {

constexpr int kCoderThreads = 32;                 // one warp per CTA (smem-bound: 32 KB of models)
constexpr int kNCtx = 512;                        // 9-pixel template
constexpr int kRowWords = 6;                      // padded MSB-first row: 2 lead bits + <= 128 + pad

__host__ __device__ inline int lmr_tile_side(int t, int dim) { return (1 << t) < dim ? (1 << t) : dim; }
__host__ __device__ inline int lmr_tile_count(int H, int W, int t) {
    const int th = lmr_tile_side(t, H), tw = lmr_tile_side(t, W);
    return ((H + th - 1) / th) * ((W + tw - 1) / tw);
}
__host__ __device__ inline int lmr_tile_cap(int t, int H, int W) {   // >= 1.1 * raw + 64 bytes
    const int n = lmr_tile_side(t, H) * lmr_tile_side(t, W);
    return n / 8 + n / 64 + 64;
}
// stream slot stride: cap + slack for the fast encoder's unchecked digit stores (<= 32 per half-word)
__host__ __device__ inline int lmr_tile_stride(int t, int H, int W) { return lmr_tile_cap(t, H, W) + 48; }

// context bits from the two previous rows: rows are MSB-first with pixel x at padded bit x+2
__device__ __forceinline__ uint32_t row_window(const uint32_t *row, int pos, int nbits) {
    const uint64_t w = ((uint64_t)row[pos >> 5] << 32) | row[(pos >> 5) + 1];
    return (uint32_t)((w << (pos & 31)) >> (64 - nbits));
}

struct RcEnc {
    uint64_t low;
    uint32_t range;
    uint32_t cache;
    uint32_t cache_size;
    uint8_t *out;
    int n, cap;
    __device__ __forceinline__ void put(uint32_t v) {
        if (n < cap) out[n] = (uint8_t)v;
        n++;
    }
    __device__ __forceinline__ void shift_low() {
        if ((uint32_t)low < 0xFF000000u || (low >> 32) != 0) {
            const uint32_t carry = (uint32_t)(low >> 32);
            uint32_t temp = cache;
#pragma unroll 1
            do {                                      // (a pending 0xFF run is rare: keep it a plain loop)
                put((temp + carry) & 0xFFu);
                temp = 0xFFu;
            } while (--cache_size != 0);
            cache = ((uint32_t)low >> 24) & 0xFFu;
        }
        cache_size++;
        low = (uint64_t)((uint32_t)low << 8);
    }
};

// work item gid of candidate wave `wave` (mmsb_kernels.h): image, stream slot (0 = eta,
// 1 + c = candidate c), candidate index (-1 for eta) and tile; false past the wave's work
struct WaveItem { int img, slot, cand, tile; };
__device__ __forceinline__ bool wave_item(const Geo &g, int wave, int R, long long gid, const LmrEncWS &e, WaveItem &it) {
    const int Tc = lmr_tile_count(g.H, g.W, g.tile_log2);
    const int A = wave == 0 ? g.B : e.ctl->count[wave];
    const int nc = wave == 0 ? 0 : e.ctl->nc[wave];
    const int k = lmr_wave_k(wave, A, Tc, g.B, R, nc);
    const int per = (wave == 0 ? 1 : 0) + k;                     // slots per image in this wave
    if (gid >= (long long)A * per * Tc) return false;
    if (wave == 0) {                                              // image-major: eta, candidates
        const int i = (int)(gid / ((long long)per * Tc)), r = (int)(gid % ((long long)per * Tc));
        it.tile = r % Tc;
        it.img = i;
        it.cand = r / Tc - 1;
    } else {                                                      // candidate-major
        const int j = (int)(gid / ((long long)A * Tc)), r = (int)(gid % ((long long)A * Tc));
        it.tile = r % Tc;
        it.img = e.lists[(size_t)wave * g.B + r / Tc];
        it.cand = nc + j;
    }
    it.slot = it.cand + 1;
    return true;
}

// ======================================================================================
// coder_encode_kernel (tiles narrower than 32): one thread per work item of the wave
// (wave_item): slot 0 = rotated eta (MSB of I_r, eq. MSB_map) -- wave 0 only; slot 1 + c =
// rotated location map L_b = [c_r < b] of candidate c, b = order[c].
// ======================================================================================
__global__ void __launch_bounds__(kCoderThreads) coder_encode_kernel(Geo g, int wave, int round_tiles, const uint8_t *__restrict__ ceta,
                                                                     LmrEncWS ew) {
    extern __shared__ uint16_t p0s[];                                  // [kNCtx][32]
    __shared__ uint32_t rows[kCoderThreads][3][kRowWords];
    const int lane = threadIdx.x;
    const int Tc = lmr_tile_count(g.H, g.W, g.tile_log2);
    WaveItem it{0, 0, -1, 0};
    const bool active = wave_item(g, wave, round_tiles, (long long)blockIdx.x * kCoderThreads + lane, ew, it);
    if (!__any_sync(0xffffffffu, active)) return;
    const int img = it.img, slot = it.slot, tile = it.tile;
    const LmrPlan pl = ew.plan[img];
    uint8_t *streams = ew.streams;
    int32_t *sizes = ew.sizes;

    const int th = lmr_tile_side(g.tile_log2, g.H), tw = lmr_tile_side(g.tile_log2, g.W);
    const int TN = (g.W + tw - 1) / tw;
    const int y0 = (tile / TN) * th, x0 = (tile % TN) * tw;
    const int h = g.H - y0 < th ? g.H - y0 : th, w = g.W - x0 < tw ? g.W - x0 : tw;
    const int b = slot == 0 ? 0 : pl.order[it.cand < 0 ? 0 : it.cand];
    const int cap = lmr_tile_cap(g.tile_log2, g.H, g.W);

    for (int c = 0; c < kNCtx; c++) p0s[c * 32 + lane] = 32768;
    uint32_t(*R)[kRowWords] = rows[lane];
    for (int r = 0; r < 3; r++)
        for (int k = 0; k < kRowWords; k++) R[r][k] = 0;

    RcEnc e{0, 0xFFFFFFFFu, 0, 1, streams + (((size_t)img * kLmrSlots + slot) * Tc + tile) * lmr_tile_stride(g.tile_log2, g.H, g.W), 0, cap};
    const uint8_t *src = ceta + (size_t)img * g.HW;
    if (active) {
        for (int y = 0; y < h; y++) {
            uint32_t *cur = R[y % 3];
            const uint32_t *p1 = R[(y + 2) % 3], *p2 = R[(y + 1) % 3];     // rows y-1, y-2 (zero when absent)
            for (int k = 0; k < kRowWords; k++) cur[k] = 0;
            uint32_t left = 0;                                             // bit (0,-1)
            const uint8_t *rowp = src + (size_t)(y0 + y) * g.W + x0;
            for (int x = 0; x < w; x++) {
                const uint8_t v = rowp[x];
                const uint32_t bit = slot == 0 ? (uint32_t)(v >> 7) : (uint32_t)((v >> (8 - b)) & 1u);   // [c < b]
                const uint32_t ctx = (left << 8) | (row_window(p1, x, 5) << 3) | row_window(p2, x + 1, 3);
                uint16_t *pp = &p0s[ctx * 32 + lane];
                const uint32_t p = *pp;
                const uint32_t bound = (e.range >> 16) * p;
                if (bit == 0) {
                    e.range = bound;
                    *pp = (uint16_t)(p + ((65536u - p) >> 4));
                } else {
                    e.low += bound;
                    e.range -= bound;
                    *pp = (uint16_t)(p - (p >> 4));
                }
                while (e.range < (1u << 24)) {
                    e.range <<= 8;
                    e.shift_low();
                }
                left = bit;
                if (bit) cur[(x + 2) >> 5] |= 0x80000000u >> ((x + 2) & 31);
            }
            // keep the two padding words beyond the row zero for the next rows' windows
        }
        for (int i = 0; i < 5; i++) e.shift_low();
        sizes[((size_t)img * kLmrSlots + slot) * Tc + tile] = (e.n <= cap && e.n <= 65535) ? e.n : -1;
    }
}

// ======================================================================================
// lmr_plan_kernel: candidate order per image from the label histogram: b in [2,8] ordered by
// (b-1) * zeros(b) descending, ties -> smaller b (readings Q5, Q22).
// ======================================================================================
__global__ void lmr_plan_kernel(Geo g, const uint32_t *__restrict__ hist, LmrPlan *__restrict__ plan,
                                LmrWaveCtl *__restrict__ ctl, int32_t *__restrict__ mapbytes) {
    const int img = blockIdx.x * blockDim.x + threadIdx.x;
    if (img == 0) {
        for (int w = 0; w < 8; w++) { ctl->count[w] = w == 0 ? g.B : 0; ctl->nc[w] = 0; }
    }
    if (img >= g.B) return;
    for (int c = 0; c < kMapStats; c++) mapbytes[(size_t)img * kMapStats + c] = c == 16 ? 127 : 0;
    LmrPlan p{};
    long long val[9];
    for (int b = 2; b <= 8; b++) val[b] = (long long)(b - 1) * (g.HW - (long long)hist[img * kHistStride + b]);
    int ord[7];
    for (int k = 0; k < 7; k++) ord[k] = k + 2;
    for (int k = 1; k < 7; k++) {
        const int b = ord[k];
        int j = k - 1;
        while (j >= 0 && val[ord[j]] < val[b]) { ord[j + 1] = ord[j]; j--; }
        ord[j + 1] = b;
    }
    for (int k = 0; k < 7; k++) p.order[k] = (int8_t)ord[k];
    p.state = 0;
    p.b = 0;
    p.dslot = 0;
    p.eta_bytes = 0;
    p.K = 0;
    plan[img] = p;
}

// ======================================================================================
// lmr_fit_kernel: one warp per image after wave `wave`: among the candidates the wave coded, in
// order, the first for which 7 + 16 (T_eta + T_L) + 8 (bytes_eta + bytes_L) <= M N decides b
// (P:985); otherwise the image joins the next wave's list, and after the last candidate it is a
// bad case.  Also produces the decided streams' sizes and exclusive byte offsets (eta
// tiles, then map tiles).
// ======================================================================================
__global__ void lmr_fit_kernel(Geo g, int wave, int R, LmrEncWS e) {
    const int img = blockIdx.x, lane = threadIdx.x;
    const int Tc = lmr_tile_count(g.H, g.W, g.tile_log2);
    const int A = wave == 0 ? g.B : e.ctl->count[wave];
    const int nc = wave == 0 ? 0 : e.ctl->nc[wave];
    const int k = lmr_wave_k(wave, A, Tc, g.B, R, nc);
    if (img == 0 && lane == 0 && wave < 7) e.ctl->nc[wave + 1] = nc + k;
    if (e.plan[img].state != 0) return;
    const int32_t *sz = e.sizes + (size_t)img * kLmrSlots * Tc;       // slot 0: eta, slot 1 + c: candidate c
    long long teta = 0;
    int bad_eta = 0;
    for (int t = lane; t < Tc; t += 32) {
        const int v = sz[t];
        bad_eta |= v < 0;
        teta += v;
    }
#pragma unroll
    for (int s2 = 16; s2 > 0; s2 >>= 1) {
        teta += __shfl_xor_sync(0xffffffffu, teta, s2);
        bad_eta |= __shfl_xor_sync(0xffffffffu, bad_eta, s2);
    }
    int chosen = -1;
    long long K = 0;
    for (int c = nc; c < nc + k && chosen < 0; c++) {                  // candidates in order
        const int32_t *sm = sz + (size_t)(1 + c) * Tc;
        long long tot = 0;
        int bad = bad_eta;
        for (int t = lane; t < Tc; t += 32) {
            const int v = sm[t];
            bad |= v < 0;
            tot += v;
        }
#pragma unroll
        for (int s2 = 16; s2 > 0; s2 >>= 1) {
            tot += __shfl_xor_sync(0xffffffffu, tot, s2);
            bad |= __shfl_xor_sync(0xffffffffu, bad, s2);
        }
        const long long Kc = 7 + 32ll * Tc + 8 * (teta + tot);
        if (!bad && Kc <= g.HW) { chosen = c; K = Kc; }
    }
    if (chosen >= 0) {
        // sizes of the decided streams (eta tiles, then map tiles) and their exclusive prefix
        int32_t *ds = e.dsizes + (size_t)img * 2 * Tc, *off = e.offsets + (size_t)img * 2 * Tc;
        int run = 0;
        for (int k0 = 0; k0 < 2 * Tc; k0 += 32) {
            const int q = k0 + lane;
            const int v = q < 2 * Tc ? (q < Tc ? sz[q] : sz[(size_t)(1 + chosen) * Tc + (q - Tc)]) : 0;
            int x = v;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, x, d);
                if (lane >= d) x += t;
            }
            if (q < 2 * Tc) { ds[q] = v; off[q] = run + x - v; }
            run += __shfl_sync(0xffffffffu, x, 31);
        }
    }
    if (lane == 0) {
        LmrPlan p = e.plan[img];
        p.eta_bytes = bad_eta ? -1 : (int32_t)teta;
        // a bad eta (a tile over cap) fits with no candidate: the walk's outcome is the bad case
        if (chosen >= 0) { p.state = 1; p.b = p.order[chosen]; p.dslot = 1 + chosen; p.K = K; }
        else if (nc + k >= 7 || bad_eta) { p.state = 2; p.b = 0; p.K = 0; }
        else e.lists[(size_t)(wave + 1) * g.B + atomicAdd(&e.ctl->count[wave + 1], 1)] = img;
        e.plan[img] = p;
    }
}

// ======================================================================================
// lmr_concat_kernel: the decided eta and map streams of an image, concatenated in order (tile
// raster, eta first) into one byte string at their exclusive offsets: one warp per stream (a
// 4096^2 image has 2 x 1024 of them), coalesced byte copies, 8 loads in flight per lane.
// ======================================================================================
__global__ void __launch_bounds__(256) lmr_concat_kernel(Geo g, LmrEncWS ew) {
    const int img = blockIdx.y;
    const LmrPlan pl = ew.plan[img];
    if (pl.state != 1) return;
    const int Tc = lmr_tile_count(g.H, g.W, g.tile_log2);
    const int stride = lmr_tile_stride(g.tile_log2, g.H, g.W);
    const int lane = threadIdx.x & 31;
    uint8_t *dst = ew.cat + (size_t)img * (g.HW / 8);           // (a string never exceeds the plane: K <= HW)
    for (int k = blockIdx.x * 8 + (threadIdx.x >> 5); k < 2 * Tc; k += gridDim.x * 8) {
        const int n = ew.dsizes[(size_t)img * 2 * Tc + k], o = ew.offsets[(size_t)img * 2 * Tc + k];
        const int slot = k < Tc ? 0 : pl.dslot, tile = k < Tc ? k : k - Tc;
        const uint8_t *src = ew.streams + (((size_t)img * kLmrSlots + slot) * Tc + tile) * stride;
        for (int i0 = 0; i0 < n; i0 += 256) {                  // 8 coalesced byte loads in flight per lane
            uint8_t v[8];
#pragma unroll
            for (int j = 0; j < 8; j++) {
                const int i = i0 + 32 * j + lane;
                v[j] = i < n ? src[i] : 0;
            }
#pragma unroll
            for (int j = 0; j < 8; j++) {
                const int i = i0 + 32 * j + lane;
                if (i < n) dst[o + i] = v[j];
            }
        }
    }
}

// ======================================================================================
// lmr_msb_write_kernel: writes the first-MSB plane of I_e (layout reading Q15):
//   [b-2: 3 bits][t: 4 bits][16-bit byte lengths of the eta tiles][... of the map tiles]
//   [eta tile bytes][map tile bytes], MSB first, pixel r <- stream bit r for r < K; the
//   remaining MSBs keep I_r XOR s.  Bad case: the b-field 7 (bits r = 0..2 set).
// One thread per 32 pixels; the stream bits come from the concatenated string (5 bytes).
// ======================================================================================
__global__ void __launch_bounds__(256) lmr_msb_write_kernel(Geo g, LmrEncWS ew,
                                                            const uint32_t *__restrict__ hist,
                                                            uint8_t *__restrict__ enc, int32_t *__restrict__ b_out,
                                                            int64_t *__restrict__ cap_out,
                                                            int32_t *__restrict__ status) {
    const int img = blockIdx.y;
    const LmrPlan pl = ew.plan[img];
    const int Tc = lmr_tile_count(g.H, g.W, g.tile_log2);
    uint8_t *E = enc + (size_t)img * g.HW;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (pl.state == 1) {
            b_out[img] = pl.b;
            cap_out[img] = (long long)(pl.b - 1) * (g.HW - (long long)hist[img * kHistStride + pl.b]);
            status[img] = 0;
        } else {
            b_out[img] = 0;
            cap_out[img] = 0;
            status[img] = 5;
            E[0] |= 0x80; E[1] |= 0x80; E[2] |= 0x80;           // b-field 7: bad case
        }
    }
    if (pl.state != 1) return;
    const int32_t *sz = ew.dsizes + (size_t)img * 2 * Tc;
    const uint8_t *cat = ew.cat + (size_t)img * (g.HW / 8);
    const long long hdr = 7 + 32ll * Tc;                        // header bits before the stream bytes
    const long long total = (pl.K - hdr) / 8;                   // stream bytes
    for (long long p = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * 32; p < pl.K;
         p += (long long)gridDim.x * blockDim.x * 32) {
        // 32 pixels per thread (two 16-byte words in flight; HW is a power of two >= 256)
        const uint4 u0 = *reinterpret_cast<const uint4 *>(E + p);
        const uint4 u1 = *reinterpret_cast<const uint4 *>(E + p + 16);
        // the 32 plane bits of pixels [p, p+32), MSB first
        uint32_t bits32 = 0;
        if (p >= hdr) {
            const long long q = p - hdr, q0 = q >> 3;
            const int sh = (int)(q & 7);                        // bit offset inside byte q0
            unsigned long long b5 = 0;
#pragma unroll
            for (int i = 0; i < 5; i++)
                b5 = (b5 << 8) | (q0 + i < total ? (unsigned long long)cat[q0 + i] : 0ull);
            bits32 = (uint32_t)(b5 >> (8 - sh));
        } else {
            for (int i = 0; i < 32; i++) {
                const long long r = p + i;
                uint32_t bit = 0;
                if (r < 3) bit = ((uint32_t)(pl.b - 2) >> (2 - r)) & 1u;
                else if (r < 7) bit = ((uint32_t)g.tile_log2 >> (6 - r)) & 1u;
                else if (r < hdr) bit = ((uint32_t)sz[(r - 7) >> 4] >> (15 - ((r - 7) & 15))) & 1u;
                else {
                    const long long q = r - hdr;
                    const uint32_t by = q >> 3 < total ? (uint32_t)cat[q >> 3] : 0u;
                    bit = (by >> (7 - (q & 7))) & 1u;
                }
                bits32 |= bit << (31 - i);
            }
        }
        uint32_t wv[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
#pragma unroll
        for (int i = 0; i < 8; i++) {
            // the word's 4 plane bits (first pixel = nibble bit 3) to the byte MSBs: nib << (9k + 4)
            // puts nibble bit 3-k at bit 8k+7, the four terms do not overlap
            const uint32_t nib = (bits32 >> (28 - 4 * i)) & 0xFu;
            const uint32_t msb = (nib * 0x80402010u) & 0x80808080u;
            const long long nv = pl.K - (p + 4 * i);            // pixels of the word below K
            const uint32_t bm = nv >= 4 ? 0xFFFFFFFFu : (nv <= 0 ? 0u : (1u << (8 * (int)nv)) - 1u);
            wv[i] = (wv[i] & ~(bm & 0x80808080u)) | (msb & bm);
        }
        *reinterpret_cast<uint4 *>(E + p) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
        *reinterpret_cast<uint4 *>(E + p + 16) = make_uint4(wv[4], wv[5], wv[6], wv[7]);
    }
}

// ======================================================================================
// Decoding side.
// lmr_pack_kernel: MSB plane of the marked image -> bytes (stream bit r = MSB of pixel r).
// ======================================================================================
__global__ void __launch_bounds__(256) lmr_pack_kernel(long long HW, int B, const uint8_t *__restrict__ in,
                                                       uint8_t *__restrict__ mbuf) {
    const long long n16 = (long long)B * HW / 16;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (long long)gridDim.x * blockDim.x) {
        const uint4 u = __ldg(reinterpret_cast<const uint4 *>(in) + i);
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
        uint32_t out = 0;
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const uint32_t m = (w[k] >> 7) & 0x01010101u;                 // MSB of each byte
            const uint32_t b4 = ((m * 0x08040201u) >> 24) & 0xFu;           // pixel 0 -> bit 3
            out |= b4 << (12 - 4 * k);
        }
        // out: 16 bits, pixel 0 at bit 15 -> two stream bytes
        reinterpret_cast<uint16_t *>(mbuf)[i] = (uint16_t)(((out >> 8) & 0xFFu) | ((out & 0xFFu) << 8));
    }
}

// lmr_header_kernel: one warp per image parses b, t and the 2 T tile lengths; validates the
// layout (FORMAT) or the bad-case marker (BADCASE); exclusive offsets of the streams.
__device__ __forceinline__ uint32_t mbuf_bits(const uint8_t *m, long long pos, int n) {
    uint32_t v = 0;
    for (int i = 0; i < n; i++) v = (v << 1) | ((m[(pos + i) >> 3] >> (7 - ((pos + i) & 7))) & 1u);
    return v;
}

__global__ void lmr_header_kernel(Geo g, const uint8_t *__restrict__ mbuf, int32_t *__restrict__ lmr_b,
                                  int32_t *__restrict__ lmr_t, int32_t *__restrict__ offsets,
                                  int32_t *__restrict__ sizes, int32_t *__restrict__ status,
                                  int64_t *__restrict__ msg_bits_out) {
    const int img = blockIdx.x, lane = threadIdx.x;
    const uint8_t *m = mbuf + (size_t)img * (g.HW / 8);
    const int field = (int)mbuf_bits(m, 0, 3), t = (int)mbuf_bits(m, 3, 4);
    int st = 0;
    if (field == 7) st = 5;
    else if (t != g.tile_log2) st = 8;           // t is shared protocol knowledge (reading Q15)
    int Tc = 0;
    if (!st) {
        Tc = lmr_tile_count(g.H, g.W, t);
        if (7 + 32ll * Tc > g.HW) st = 8;
    }
    long long run = 0;
    if (!st) {
        for (int k0 = 0; k0 < 2 * Tc; k0 += 32) {
            const int k = k0 + lane;
            const int s = k < 2 * Tc ? (int)mbuf_bits(m, 7 + 16ll * k, 16) : 0;
            int v = s;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int tt = __shfl_up_sync(0xffffffffu, v, d);
                if (lane >= d) v += tt;
            }
            if (k < 2 * Tc) {
                offsets[(size_t)img * 2 * g.ntiles_coder + k] = (int)run + v - s;
                sizes[(size_t)img * 2 * g.ntiles_coder + k] = s;
            }
            run += __shfl_sync(0xffffffffu, v, 31);
        }
        if (7 + 32ll * Tc + 8 * run > g.HW) st = 8;
    }
    if (lane == 0) {
        lmr_b[img] = st ? 0 : field + 2;
        lmr_t[img] = st ? 0 : t;
        if (st) {
            status[img] = st;
            if (msg_bits_out) msg_bits_out[img] = -1;
        }
    }
}

// coder_decode_kernel: one thread per (image, plane, tile); plane 0 = eta (recover only),
// plane 1 = map.  Decoded bits go to packed planes (bit x&31 of word (y W + x) >> 5).
__global__ void __launch_bounds__(kCoderThreads) coder_decode_kernel(Geo g, int want_eta, const uint8_t *__restrict__ mbuf,
                                                                     const int32_t *__restrict__ lmr_b,
                                                                     const int32_t *__restrict__ lmr_t,
                                                                     const int32_t *__restrict__ offsets,
                                                                     const int32_t *__restrict__ sizes,
                                                                     uint32_t *__restrict__ eta_bits,
                                                                     uint32_t *__restrict__ map_bits) {
    extern __shared__ uint16_t p0s[];
    __shared__ uint32_t rows[kCoderThreads][3][kRowWords];
    const int lane = threadIdx.x;
    const int TcM = g.ntiles_coder;
    const int nplanes = want_eta ? 2 : 1;
    const long long gid = (long long)blockIdx.x * kCoderThreads + lane;
    const long long total = (long long)g.B * nplanes * TcM;
    bool active = gid < total;
    const int img = active ? (int)(gid / ((long long)nplanes * TcM)) : 0;
    const int rem = active ? (int)(gid % ((long long)nplanes * TcM)) : 0;
    const int plane = want_eta ? rem / TcM : 1;
    const int tile = rem % TcM;
    const int b = lmr_b[img], t = lmr_t[img];
    int Tc = 0;
    if (active && b >= 2) Tc = lmr_tile_count(g.H, g.W, t);
    active = active && b >= 2 && tile < Tc;
    if (!__any_sync(0xffffffffu, active)) return;

    const int th = lmr_tile_side(t > 0 ? t : 7, g.H), tw = lmr_tile_side(t > 0 ? t : 7, g.W);
    const int TN = (g.W + tw - 1) / tw;
    const int y0 = (tile / TN) * th, x0 = (tile % TN) * tw;
    const int h = g.H - y0 < th ? g.H - y0 : th, w = g.W - x0 < tw ? g.W - x0 : tw;

    for (int c = 0; c < kNCtx; c++) p0s[c * 32 + lane] = 32768;
    uint32_t(*R)[kRowWords] = rows[lane];
    for (int r = 0; r < 3; r++)
        for (int k = 0; k < kRowWords; k++) R[r][k] = 0;
    if (!active) return;

    const int k = (plane == 0 ? 0 : Tc) + tile;
    const int nbytes = sizes[(size_t)img * 2 * TcM + k];
    const long long bit0 = 7 + 32ll * Tc + 8ll * offsets[(size_t)img * 2 * TcM + k];
    const uint8_t *m = mbuf + (size_t)img * (g.HW / 8);
    int pos = 0;
    auto next = [&]() -> uint32_t {
        uint32_t v = 0;
        if (pos < nbytes) {
            const long long bb = bit0 + 8ll * pos;
            const uint32_t hi = m[bb >> 3], lo = m[(bb >> 3) + 1];
            v = (((hi << 8) | lo) >> (8 - (bb & 7))) & 0xFFu;
        }
        pos++;
        return v;
    };
    uint32_t range = 0xFFFFFFFFu, code = 0;
    for (int i = 0; i < 5; i++) code = (code << 8) | next();
    uint32_t *plane_out = plane == 0 ? eta_bits : map_bits;
    for (int y = 0; y < h; y++) {
        uint32_t *cur = R[y % 3];
        const uint32_t *p1 = R[(y + 2) % 3], *p2 = R[(y + 1) % 3];
        for (int kk = 0; kk < kRowWords; kk++) cur[kk] = 0;
        uint32_t left = 0, acc = 0;
        const long long rowbit = (long long)img * g.HW + (long long)(y0 + y) * g.W + x0;
        for (int x = 0; x < w; x++) {
            const uint32_t ctx = (left << 8) | (row_window(p1, x, 5) << 3) | row_window(p2, x + 1, 3);
            uint16_t *pp = &p0s[ctx * 32 + lane];
            const uint32_t p = *pp;
            const uint32_t bound = (range >> 16) * p;
            uint32_t bit;
            if (code < bound) {
                range = bound;
                bit = 0;
                *pp = (uint16_t)(p + ((65536u - p) >> 4));
            } else {
                code -= bound;
                range -= bound;
                bit = 1;
                *pp = (uint16_t)(p - (p >> 4));
            }
            while (range < (1u << 24)) {
                range <<= 8;
                code = (code << 8) | next();
            }
            left = bit;
            if (bit) cur[(x + 2) >> 5] |= 0x80000000u >> ((x + 2) & 31);
            acc |= bit << (x & 31);
            if ((x & 31) == 31 || x == w - 1) {
                const long long wb = rowbit + (x & ~31);
                if ((w & 31) == 0) plane_out[wb >> 5] = acc;
                else atomicOr(plane_out + (wb >> 5), acc << (wb & 31));
                acc = 0;
            }
        }
    }
}

// ======================================================================================
// Fast coder kernels for tiles at least 32 pixels wide (every configured shape).  Same bit
// stream as coder_encode_kernel / coder_decode_kernel, restructured for a
// serial chain that has only a few warps per SM to hide its latency (the models, 1 KB per
// tile, bound residency at ~224 tiles per SM):
//  * CTAs of kFastThreads = 112 threads (3.5 warps: all four SM sub-partitions busy) holding
//    112 KB of models, kFastCtas = 2 CTAs per SM;
//  * the row is walked in half-words of 16 pixels with the 16 symbols fully unrolled: the
//    9-pixel context of every symbol comes from two pre-aligned 32-bit slices of the rows
//    above with immediate shifts (only its (0,-1) bit depends on the symbol before);
//  * the next symbol's probability is loaded while the current one is coded -- the decoder
//    loads both candidates (their address does not depend on the bit being decoded) and
//    forwards the freshly updated probability when the contexts coincide, so after the bit
//    is known only one select remains;
//  * renormalisation is branch-free: the number of bytes to shift is clz(range) >> 3 (0..2:
//    range >= 3840 after any symbol), the decoder reads through a 160-bit MSB-aligned bit
//    buffer refilled from funnel-shifted stream words (bytes past the end read as 0) and
//    shifted once per symbol pair, the encoder's byte output is predicated (only a carry into
//    already written digits takes a branch);
//  * the step is ALU-pipe bound, so bit-dependent updates are multiply-adds with the bit as a
//    0/1 factor on the FMA pipe wherever that does not lengthen the decoder's loop-carried
//    chain.
// ======================================================================================
constexpr int kFastThreads = 112;
constexpr int kFastCtas = 2;                                   // resident CTAs per SM
constexpr int kHalfCtx = kNCtx / 2;                            // contexts with (0,-1) = 0; the rest at +kHiOff
constexpr uint32_t kHiOff = kFastThreads * kHalfCtx * 2;      // bytes: models of contexts 256..511
static constexpr size_t fast_smem() { return 2 * (size_t)kHiOff; }

// Model layout (112 KB): context ctx of thread tid at byte
//   (ctx >> 8) * kHiOff + warp * 256 * 64 + (ctx & 255) * sbytes + lane * 2,
// sbytes = 2 * (lanes of the warp): warp-interleaved (<= 2-way bank conflicts), and the two
// contexts that differ only in the (0,-1) bit a fixed immediate offset apart.
__device__ __forceinline__ void fast_model_init(uint16_t *p0s) {
    uint4 *q = reinterpret_cast<uint4 *>(p0s);
    const uint4 v = make_uint4(0x80008000u, 0x80008000u, 0x80008000u, 0x80008000u);   // p0 = 32768
    for (int i = threadIdx.x; i < (int)(fast_smem() / 16); i += kFastThreads) q[i] = v;
    __syncthreads();
}
__device__ __forceinline__ uint32_t fast_model_base(const uint16_t *p0s, int tid, uint32_t &sbytes) {
    const int w = tid >> 5;
    sbytes = 2u * ((w == kFastThreads / 32) ? (kFastThreads & 31) : 32);
    return (uint32_t)__cvta_generic_to_shared(p0s) + w * kHalfCtx * 64 + (tid & 31) * 2;
}
// shared-memory model accesses keep program order (asm volatile): a probability loaded for the
// next symbol is read before the current symbol's update, which is forwarded explicitly
__device__ __forceinline__ uint32_t lds_u16(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts_u16(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"((unsigned short)v));
}

// a * b + c as an integer multiply-add (FMA pipe); asm so that a 0/1 factor is not turned back
// into a select or mask on the ALU pipe
__device__ __forceinline__ uint32_t imad(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

__device__ __forceinline__ uint32_t nib4(uint32_t t) { return ((t * 0x08040201u) >> 24) & 0xFu; }   // bytes' bit 0 -> MSB-first nibble

template <int NW>
__device__ __forceinline__ uint32_t pick(const uint32_t (&r)[NW], int k) {       // r[k], 0 outside the row
    uint32_t v = 0;
#pragma unroll
    for (int i = 0; i < NW; i++) v = k == i ? r[i] : v;
    return v;
}

// context slices of a half-word (pixels 16h .. 16h+15 of word K of the tile row; MSB-first
// words): s1 = row y-1 from pixel 16h-2, s2 = row y-2 from pixel 16h-1 (pixels outside the tile
// are 0), i.e. funnel shifts of words K-1, K (h = 0) or K, K+1 (h = 1).
// the words K-1, K, K+1 of the two rows above, rolled along the row: the slices of the next
// half-word need no search of the row arrays, only a word entering at each word boundary
template <int NW>
struct RowWin {
    uint32_t a1, c1, n1, a2, c2, n2;
    __device__ __forceinline__ void start(const uint32_t (&p1)[NW], const uint32_t (&p2)[NW], uint32_t &s1, uint32_t &s2) {
        a1 = 0; c1 = p1[0]; n1 = NW > 1 ? p1[NW > 1 ? 1 : 0] : 0u;
        a2 = 0; c2 = p2[0]; n2 = NW > 1 ? p2[NW > 1 ? 1 : 0] : 0u;
        s1 = __funnelshift_l(c1, a1, 30);
        s2 = __funnelshift_l(c2, a2, 31);
    }
    // slices of the half-word after half h of the current word (h = 1: half 0 of the next word)
    __device__ __forceinline__ void next(int h, uint32_t &t1, uint32_t &t2) const {
        t1 = __funnelshift_l(n1, c1, h ? 30 : 14);
        t2 = __funnelshift_l(n2, c2, h ? 31 : 15);
    }
    __device__ __forceinline__ void advance(const uint32_t (&p1)[NW], const uint32_t (&p2)[NW], int K) {
        a1 = c1; c1 = n1; n1 = pick(p1, K + 2);
        a2 = c2; c2 = n2; n2 = pick(p2, K + 2);
    }
};

// rows part (bits 7..0) of the context of symbol J of a half: 5 pixels x-2..x+2 of row y-1,
// 3 pixels x-1..x+1 of row y-2 (J is a constant after unrolling)
__device__ __forceinline__ uint32_t slice_ctx(uint32_t s1, uint32_t s2, int J) {
    return ((s1 >> (24 - J)) & 0xF8u) | ((s2 >> (29 - J)) & 7u);
}
// number of bits to shift in after a symbol: clz(range) & 24 (0, 8 or 16) as one LOP3 on the
// highest set bit's index (31 - f = ~f for f in [0, 31])
__device__ __forceinline__ int renorm_shift(uint32_t range) {
    uint32_t f;
    asm("bfind.u32 %0, %1;" : "=r"(f) : "r"(range));
    return (int)(~f & 24u);
}

__device__ __forceinline__ void st_u8_if(bool c, uint8_t *p, uint32_t v) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %0, 0;\n\t@q st.global.u8 [%1], %2;\n\t}" ::"r"((uint32_t)c), "l"(p),
                 "r"(v));
}

// Encoder output as exact base-256 digits.  The reference coder (coder_encode_kernel) keeps a
// cache byte and a count of pending 0xFF bytes so that a carry out of low can still reach them;
// its output is the digit string of the exact code value (a carry never reaches a byte it has
// already written -- the nested intervals never leave the initial one), one digit per shift.
// Here the window [hi = cache digit (+ carry in bit 8) | lo = low] shifts its top digits straight
// to memory with predicated stores, branch-free; a carry out of the window is recorded in a
// per-half-word mask (bit k: into the digit before the k-th digit of the half) and added into
// the written bytes after the half (0xFF -> 0x00 backwards, +1 on the first byte below 0xFF).
// Stores go to the tile's slot while n <= cap at the half's start, else into the slot's slack
// (the stream is then over cap and discarded), so none needs a bound check.
struct FastEnc {
    uint32_t hi, lo, range;
    uint8_t *out, *obase;                     // slot; this half's stores at obase + k (obase = slot + n0, or in the slack)
    int n, cap, n0;                           // digits before this half; k = digits in this half
    int k;
    uint32_t cm;                              // carries of this half
    __device__ __forceinline__ void begin_half() {
        n += k;
        obase = n <= cap ? out + n : out + cap;
        n0 = n;
        k = 0;
        cm = 0;
    }
    // s = 0..2 digits out; p1 = (s >= 1), p2 = (s >= 2)
    __device__ __forceinline__ void emit(bool p1, bool p2, int s8) {
        cm |= (hi >> 8) << k;
        const uint32_t h8 = hi & 0xFFu;
        uint8_t *op;                              // obase + k as a wide multiply-add (FMA pipe)
        asm("mad.wide.u32 %0, %1, 1, %2;" : "=l"(op) : "r"((uint32_t)k), "l"(obase));
        st_u8_if(p1, op, h8);
        st_u8_if(p2, op + 1, lo >> 24);
        hi = __funnelshift_l(lo, h8, s8) & 0xFFu;
        lo <<= s8;
        k += s8 >> 3;
    }
    __device__ __forceinline__ void end_half(unsigned am) {
        if (__any_sync(am, cm != 0)) {
#pragma unroll 1
            while (cm) {
                const int j = __ffs(cm) - 1;
                cm &= cm - 1;
                uint32_t c = 1;
#pragma unroll 1
                for (int i = n0 + j - 1; i >= 0 && c && i < cap; i--) {      // (asm: ordered after the stores)
                    uint32_t v;
                    asm volatile("ld.global.u8 %0, [%1];" : "=r"(v) : "l"(out + i));
                    v += c;
                    st_u8_if(true, out + i, v);
                    c = v >> 8;
                }
            }
        }
    }
};

template <int NW>
__global__ void __launch_bounds__(kFastThreads, kFastCtas) coder_encode_fast_kernel(Geo g, int wave, int R,
                                                                         const uint8_t *__restrict__ ceta, LmrEncWS ew,
                                                                         unsigned long long *__restrict__ sym_count) {
    extern __shared__ __align__(16) uint16_t p0s[];
    const int tid = threadIdx.x;
    const int Tc = lmr_tile_count(g.H, g.W, g.tile_log2);
    WaveItem it{0, 0, -1, 0};
    const bool active = wave_item(g, wave, R, (long long)blockIdx.x * kFastThreads + tid, ew, it);
    if (!__syncthreads_or(active)) return;
    const int img = it.img, slot = it.slot, tile = it.tile;
    fast_model_init(p0s);
    if (!active) return;
    const unsigned am = __activemask();
    uint32_t sbytes;
    const uint32_t mbase = fast_model_base(p0s, tid, sbytes);

    const int th = lmr_tile_side(g.tile_log2, g.H);
    constexpr int w = 32 * NW;
    const int TN = g.W / w;
    const int y0 = (tile / TN) * th, x0 = (tile % TN) * w;
    const int h = g.H - y0 < th ? g.H - y0 : th;
    if (sym_count) {                                                   // profiling: coded symbols
        const unsigned v = __reduce_add_sync(am, (unsigned)(h * w));
        if ((tid & 31) == __ffs(am) - 1) atomicAdd(sym_count, (unsigned long long)v);
    }
    const int bsh = slot == 0 ? 7 : 8 - ew.plan[img].order[it.cand];      // eta: bit 7; map of b: bit 8-b
    const int cap = lmr_tile_cap(g.tile_log2, g.H, g.W);

    // early abort (waves >= 1, eta known): the candidate's map can no longer fit once its tiles'
    // running byte counts exceed the room left by eta (sizes only grow, so the walk's choice is
    // unchanged); each tile publishes its count once per row and reads the total a row later
    int32_t *abort_cnt = nullptr;
    long long room = 0;
    if (wave > 0 && it.cand >= 0) {
        abort_cnt = ew.mapbytes + (size_t)img * kMapStats + it.cand;
        room = (g.HW - 7 - 32ll * Tc) / 8 - ew.plan[img].eta_bytes;
    }
    int published = 0, seen = 0;
    bool aborted = false;
    uint8_t *slot_out = ew.streams + (((size_t)img * kLmrSlots + slot) * Tc + tile) * lmr_tile_stride(g.tile_log2, g.H, g.W);
    FastEnc e{0, 0, 0xFFFFFFFFu, slot_out, slot_out, 0, cap, 0, 0, 0};
    const uint8_t *src = ceta + (size_t)img * g.HW + x0;
    uint32_t p1[NW], p2[NW];
#pragma unroll
    for (int k = 0; k < NW; k++) { p1[k] = 0; p2[k] = 0; }
    // the row's bits, MSB-first: eta = bit 7 of the byte (eq. MSB_map), map = [c < b] = bit 8-b;
    // the next row's bytes are loaded while the current row is coded
    uint4 raw[2 * NW];
    auto load_row = [&](int y) {
        const uint4 *rp = reinterpret_cast<const uint4 *>(src + (size_t)(y0 + y) * g.W);
#pragma unroll
        for (int q = 0; q < 2 * NW; q++) raw[q] = __ldg(rp + q);
    };
    load_row(0);
#pragma unroll 1
    for (int y = 0; y < h; y++) {
        uint32_t cw[NW];
#pragma unroll
        for (int k = 0; k < NW; k++) {
            uint32_t wv = 0;
#pragma unroll
            for (int q = 0; q < 2; q++) {
                const uint32_t v[4] = {raw[2 * k + q].x, raw[2 * k + q].y, raw[2 * k + q].z, raw[2 * k + q].w};
#pragma unroll
                for (int i = 0; i < 4; i++) {
                    const uint32_t t = (v[i] >> bsh) & 0x01010101u;
                    wv |= nib4(t) << (28 - 4 * (4 * q + i));
                }
            }
            cw[k] = wv;
        }
        if (y + 1 < h) load_row(y + 1);
        uint32_t s1, s2;
        RowWin<NW> win;
        win.start(p1, p2, s1, s2);
        uint32_t actx = mbase + slice_ctx(s1, s2, 0) * sbytes;         // (0,-1) = 0 at the row start
        uint32_t p = lds_u16(actx);
        const uint32_t two = g.one + g.one, neg1 = 0u - g.one;        // opaque 2 and -1: FMA-pipe multiplies
#pragma unroll 1
        for (int q = 0; q < 2 * NW; q++) {
            uint32_t t1, t2;
            win.next(q & 1, t1, t2);                                   // next half (unused past the row)
            uint32_t cb = pick(cw, q >> 1) << (16 * (q & 1));          // the half's bits from the MSB, rolled
            e.begin_half();
#pragma unroll
            for (int J = 0; J < 16; J++) {
                // The bit is kept as an integer bv in {0, 1} and the bit-dependent selects are
                // written as multiply-adds: they issue on the FMA pipe, which the ALU-bound
                // step otherwise leaves idle (same values as the select form).
                const uint32_t bv = cb >> 31;
                cb = imad(cb, two, 0u);
                const uint32_t nrows = J < 15 ? slice_ctx(s1, s2, J + 1) : slice_ctx(t1, t2, 0);
                const uint32_t anctx = imad(bv, kHiOff, imad(nrows, sbytes, mbase));
                const uint32_t np = lds_u16(anctx);
                const uint32_t bound = (e.range >> 16) * p;
                const uint32_t tb = imad(bv, bound, 0u);                      // low += bound if 1
                asm("add.cc.u32 %0, %0, %2;\n\taddc.u32 %1, %1, 0;" : "+r"(e.lo), "+r"(e.hi) : "r"(tb));
                e.range = imad(bv, imad(bound, 0xFFFFFFFEu, e.range), bound);   // bound + bv (range - 2 bound)
                // p0 update: 1 -> p - (p >> 4) = p + floor((15 - p) / 16); 0 -> p + ((65536 - p) >> 4)
                const int32_t dp = (int32_t)imad(bv, 15u - 65536u, imad(p, neg1, 65536u));
                const uint32_t pu = p + (uint32_t)(dp >> 4);
                sts_u16(actx, pu);
                const bool r24 = e.range < (1u << 24), r16 = e.range < (1u << 16);   // 1 / 2 digits out
                const int s8 = (r24 ? 8 : 0) + (r16 ? 8 : 0);
                e.emit(r24, r16, s8);
                e.range <<= s8;
                p = anctx == actx ? pu : np;
                actx = anctx;
            }
            e.end_half(am);
            s1 = t1;
            s2 = t2;
            if (q & 1) win.advance(p1, p2, q >> 1);
        }
#pragma unroll
        for (int k = 0; k < NW; k++) { p2[k] = p1[k]; p1[k] = cw[k]; }
        if (abort_cnt) {
            // stop once the map can no longer fit, or once an earlier candidate of the walk is
            // known to fit (this one can then never be chosen)
            if (seen > room || ld_relaxed_s32(abort_cnt + 16 - it.cand) < it.cand) { aborted = true; break; }
            const int cur = e.n + e.k;
            seen = atomicAdd(abort_cnt, cur - published) + (cur - published);
            published = cur;
        }
    }
    if (aborted) {                                                     // does not fit / cannot be chosen
        ew.sizes[((size_t)img * kLmrSlots + slot) * Tc + tile] = -1;
        return;
    }
    e.begin_half();                                                    // flush: the window's 5 digits
#pragma unroll 1
    for (int i = 0; i < 5; i++) e.emit(true, false, 8);
    e.end_half(am);
    e.n += e.k;
    const bool ok = e.n <= cap && e.n <= 65535;
    ew.sizes[((size_t)img * kLmrSlots + slot) * Tc + tile] = ok ? e.n : -1;
    if (abort_cnt) {
        // the candidate's exact total once its last tile is in (a tile over its cap poisons it);
        // the last tile decides whether it fits and publishes the first fitting candidate
        atomicAdd(abort_cnt, (ok ? e.n : (1 << 28)) - published);
        __threadfence();
        if (atomicAdd(abort_cnt + 8, 1) == Tc - 1) {
            const long long tot = atomicAdd(abort_cnt, 0);
            if (tot <= room) atomicMin(abort_cnt + 16 - it.cand, it.cand);
        }
    }
}

// decoder input: the tile's stream as a 160-bit MSB-aligned bit buffer b0..b4 (nb valid bits),
// refilled from stream words funnel-shifted out of the big-endian words of the MSB-plane bytes
// (the stream starts at an arbitrary bit); stream bytes past nbytes read as 0.  A symbol takes
// at most 16 bits, so the buffer is topped up to >= 128 bits once per 8 symbols: the common
// top-up (nb in [96, 128]: one word into b3:b4) is branch-free, any other case (a group that
// took more than 32 bits) runs behind a warp vote.
struct FastIn {
    const uint32_t *w;                        // aligned word holding the next stream word's first bit
    uint32_t wa, wb, wc, wd;                  // w[0], w[1] (big-endian), w[2], w[3] (raw: loads in flight)
    int sh;                                   // stream bit 0 = bit sh of the first word
    int valid;                                // stream bits left to deliver (8 nbytes - delivered)
    uint32_t b0, b1, b2, b3, b4;
    int nb;
    __device__ __forceinline__ uint32_t keep() const {             // top min(valid, 32) bits
        const int vc = valid < 0 ? 0 : (valid > 32 ? 32 : valid);
        return ~__funnelshift_rc(0xFFFFFFFFu, 0u, vc);
    }
    // the next stream word when `take` (else 0); the word queue advances only then.  The load of
    // the queue's new last word is unconditional (the same word again when the queue stands).
    __device__ __forceinline__ uint32_t next_word(bool take) {
        const uint32_t v = take ? __funnelshift_l(wb, wa, sh) & keep() : 0u;
        valid -= take ? 32 : 0;
        wa = take ? wb : wa;
        wb = take ? bswap32(wc) : wb;
        wc = take ? wd : wc;
        w += take ? 1 : 0;
        wd = take ? __ldg(w + 3) : wd;
        return v;
    }
    __device__ __forceinline__ void init(const uint8_t *m, long long bit0, int nbytes) {
        w = reinterpret_cast<const uint32_t *>(m) + (bit0 >> 5);
        sh = (int)(bit0 & 31);
        valid = 8 * nbytes;
        wa = bswap32(__ldg(w));
        wb = bswap32(__ldg(w + 1));
        wc = __ldg(w + 2);
        wd = __ldg(w + 3);
        b0 = next_word(true);
        b1 = next_word(true);
        b2 = next_word(true);
        b3 = next_word(true);
        b4 = next_word(true);
        nb = 160;
    }
    // n in [0, 32] bits (two symbols' worth)
    __device__ __forceinline__ void consume2(int n) {
        b0 = __funnelshift_lc(b1, b0, n);
        b1 = __funnelshift_lc(b2, b1, n);
        b2 = __funnelshift_lc(b3, b2, n);
        b3 = __funnelshift_lc(b4, b3, n);
        b4 = __funnelshift_lc(0u, b4, n);
        nb -= n;
    }
    __device__ __forceinline__ void consume(int s8) {                // s8 = 0, 8 or 16 bits
        b0 = __funnelshift_l(b1, b0, s8);
        b1 = __funnelshift_l(b2, b1, s8);
        b2 = __funnelshift_l(b3, b2, s8);
        b3 = __funnelshift_l(b4, b3, s8);
        b4 <<= s8;
        nb -= s8;
    }
    // any position: one word at bit offset nb < 160 (rare path)
    __device__ __forceinline__ void add_word_any(bool need) {
        const uint32_t v = next_word(need);
        const int k = nb >> 5, r = nb & 31;
        const uint32_t hi = v >> r, lo = __funnelshift_lc(0u, v, 32 - r);
        b0 |= k == 0 ? hi : 0u;
        b1 |= k == 0 ? lo : (k == 1 ? hi : 0u);
        b2 |= k == 1 ? lo : (k == 2 ? hi : 0u);
        b3 |= k == 2 ? lo : (k == 3 ? hi : 0u);
        b4 |= k == 3 ? lo : (k == 4 ? hi : 0u);
        nb += need ? 32 : 0;
    }
    // before each group of 8 symbols (<= 128 bits): nb -> [128, 160]
    __device__ __forceinline__ void refill(unsigned am) {
        const bool mid = nb >= 96 && nb <= 128;                       // the common case: into b3:b4
        const uint32_t v = next_word(mid);
        const int r = nb & 31;
        b3 |= mid && nb < 128 ? v >> r : 0u;
        b4 |= mid ? (nb < 128 ? __funnelshift_lc(0u, v, 32 - r) : v) : 0u;
        nb += mid ? 32 : 0;
#pragma unroll 1
        while (__any_sync(am, nb < 128)) add_word_any(nb < 128);   // rare: only as many words as the neediest lane
    }
};

template <int NW>
__global__ void __launch_bounds__(kFastThreads, kFastCtas) coder_decode_fast_kernel(Geo g, int want_eta, const uint8_t *__restrict__ mbuf,
                                                                         const int32_t *__restrict__ lmr_b,
                                                                         const int32_t *__restrict__ lmr_t,
                                                                         const int32_t *__restrict__ offsets,
                                                                         const int32_t *__restrict__ sizes,
                                                                         uint32_t *__restrict__ eta_bits,
                                                                         uint32_t *__restrict__ map_bits,
                                                                         unsigned long long *__restrict__ sym_count) {
    extern __shared__ __align__(16) uint16_t p0s[];
    const int tid = threadIdx.x;
    const int TcM = g.ntiles_coder;
    const int nplanes = want_eta ? 2 : 1;
    const long long gid = (long long)blockIdx.x * kFastThreads + tid;
    const long long total = (long long)g.B * nplanes * TcM;
    bool active = gid < total;
    const int img = active ? (int)(gid / ((long long)nplanes * TcM)) : 0;
    const int rem = active ? (int)(gid % ((long long)nplanes * TcM)) : 0;
    const int plane = want_eta ? rem / TcM : 1;
    const int tile = rem % TcM;
    const int b = lmr_b[img];
    const int Tc = TcM;                                       // header t == g.tile_log2 (else FORMAT)
    active = active && b >= 2;
    if (!__syncthreads_or(active)) return;
    fast_model_init(p0s);
    if (!active) return;
    const unsigned am = __activemask();
    uint32_t sbytes;
    const uint32_t mbase = fast_model_base(p0s, tid, sbytes);

    const int th = lmr_tile_side(g.tile_log2, g.H);
    constexpr int w = 32 * NW;
    const int TN = g.W / w;
    const int y0 = (tile / TN) * th, x0 = (tile % TN) * w;
    const int h = g.H - y0 < th ? g.H - y0 : th;
    if (sym_count) {                                                   // profiling: decoded symbols
        const unsigned v = __reduce_add_sync(am, (unsigned)(h * w));
        if ((tid & 31) == __ffs(am) - 1) atomicAdd(sym_count, (unsigned long long)v);
    }

    const int k = (plane == 0 ? 0 : Tc) + tile;
    FastIn in;
    in.init(mbuf + (size_t)img * (g.HW / 8), 7 + 32ll * Tc + 8ll * offsets[(size_t)img * 2 * TcM + k],
            sizes[(size_t)img * 2 * TcM + k]);
    // the encoder's first byte is the initial cache byte: code = stream bytes 1..4
    uint32_t range = 0xFFFFFFFFu, code = __funnelshift_l(in.b1, in.b0, 8);
    in.b0 = in.b1;
    in.b1 = in.b2;
    in.b2 = in.b3;
    in.b3 = in.b4;
    in.b4 = 0;
    in.nb = 128;
    in.consume(8);
    in.refill(am);
    uint32_t *plane_out = plane == 0 ? eta_bits : map_bits;
    uint32_t p1[NW], p2[NW];
#pragma unroll
    for (int q = 0; q < NW; q++) { p1[q] = 0; p2[q] = 0; }
#pragma unroll 1
    for (int y = 0; y < h; y++) {
        uint32_t cw[NW];
#pragma unroll
        for (int q = 0; q < NW; q++) cw[q] = 0;
        uint32_t s1, s2;
        RowWin<NW> win;
        win.start(p1, p2, s1, s2);
        uint32_t actx = mbase + slice_ctx(s1, s2, 0) * sbytes;
        uint32_t p = lds_u16(actx);
        uint32_t word = 0, acc = 0;
        uint32_t *orow = plane_out + (((size_t)img * g.HW + (size_t)(y0 + y) * g.W + x0) >> 5);
#pragma unroll 1
        for (int q = 0; q < 2 * NW; q++) {
            uint32_t t1, t2;
            win.next(q & 1, t1, t2);
            uint32_t hw = 0;
            int u = 0;                                                 // bits the even symbol took
#pragma unroll
            for (int J = 0; J < 16; J++) {
                if ((J & 7) == 0) in.refill(am);                       // >= 128 bits for 8 symbols
                // both candidate contexts of the next symbol (its (0,-1) bit is the one decoded now)
                // as in the encoder, the decoded bit is an integer bv in {0, 1} and the
                // bit-dependent selects are multiply-adds on the FMA pipe
                const uint32_t nrows = J < 15 ? slice_ctx(s1, s2, J + 1) : slice_ctx(t1, t2, 0);
                const uint32_t a0 = imad(nrows, sbytes, mbase);
                const uint32_t np0 = lds_u16(a0), np1 = lds_u16(a0 + kHiOff);
                const uint32_t bound = (range >> 16) * p;
                const bool bit = code >= bound;
                const uint32_t bv = bit ? 1u : 0u;
                range = bit ? range - bound : bound;                            // the serial chain: selects
                code = imad(bv, 0u - bound, code);
                const int32_t dp = (int32_t)imad(bv, 15u - 65536u, imad(p, 0xFFFFFFFFu, 65536u));
                const uint32_t pu = p + (uint32_t)(dp >> 4);                  // the encoder's p0 update
                sts_u16(actx, pu);
                const int s8 = renorm_shift(range);                   // 0, 8 or 16 bits to shift in
                // the bit buffer is shifted once per symbol pair: the even symbol takes its bits
                // from the buffer's top, the odd one from bit u (the even symbol's shift) on
                if ((J & 1) == 0) {
                    code = __funnelshift_l(in.b0, code, s8);
                    u = s8;
                } else {
                    code = __funnelshift_l(__funnelshift_lc(in.b1, in.b0, u), code, s8);
                    in.consume2(u + s8);
                }
                range <<= s8;
                hw = imad(bv, 1u << (15 - J), hw);
                const uint32_t anctx = imad(bv, kHiOff, a0);
                const uint32_t np = imad(bv, np1 - np0, np0);
                p = anctx == actx ? pu : np;
                actx = anctx;
            }
            const uint32_t lw = __brev(hw) >> 16;                      // the half's bits, pixel order
            s1 = t1;
            s2 = t2;
            if (q & 1) {
                const int K = q >> 1;
                win.advance(p1, p2, K);
                word |= hw;
                acc |= lw << 16;
#pragma unroll
                for (int i = 0; i < NW; i++) cw[i] = i == K ? word : cw[i];
                orow[K] = acc;                                          // plane words: bit x & 31 = pixel x
            } else {
                word = hw << 16;
                acc = lw;
            }
        }
#pragma unroll
        for (int q = 0; q < NW; q++) { p2[q] = p1[q]; p1[q] = cw[q]; }
    }
}

// ---------------------------------------------------------------------------- launchers
int lmr_tile_cap_host(int t, int H, int W) { return lmr_tile_cap(t, H, W); }
int lmr_tile_stride_host(int t, int H, int W) { return lmr_tile_stride(t, H, W); }

static size_t coder_smem() { return kNCtx * 32 * sizeof(uint16_t); }

void lmr_set_smem_attrs() {
    static bool done = false;
    if (done) return;
    cudaFuncSetAttribute(coder_encode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)coder_smem());
    cudaFuncSetAttribute(coder_decode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)coder_smem());
    cudaFuncSetAttribute(coder_encode_fast_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fast_smem());
    cudaFuncSetAttribute(coder_encode_fast_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fast_smem());
    cudaFuncSetAttribute(coder_encode_fast_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fast_smem());
    cudaFuncSetAttribute(coder_decode_fast_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fast_smem());
    cudaFuncSetAttribute(coder_decode_fast_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fast_smem());
    cudaFuncSetAttribute(coder_decode_fast_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fast_smem());
    done = true;
}

void launch_lmr_plan(const Geo &g, const uint32_t *hist, const LmrEncWS &e, cudaStream_t st) {
    lmr_plan_kernel<<<(g.B + 127) / 128, 128, 0, st>>>(g, hist, e.plan, e.ctl, e.mapbytes);
}

static int sm_count() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}
// resident coder tiles per round: fast kernel kFastCtas CTAs of kFastThreads per SM, legacy 3 warps per SM
static int coder_round(const Geo &g) {
    const int tw = lmr_tile_side(g.tile_log2, g.W);
    return tw == 32 || tw == 64 || tw == 128 ? sm_count() * kFastCtas * kFastThreads : sm_count() * 3 * kCoderThreads;
}

void launch_coder_encode(const Geo &g, int wave, const uint8_t *ceta, const LmrEncWS &e,
                         unsigned long long *sym_count, cudaStream_t st) {
    lmr_set_smem_attrs();
    const int Tc = lmr_tile_count(g.H, g.W, g.tile_log2);
    const int R = coder_round(g);
    // most work items of this wave: wave 0 = B (1 + k0) Tc; later waves A k Tc <= max(kLmrWaveRounds R, B Tc)
    const long long total = wave == 0 ? (long long)g.B * (1 + lmr_wave_k(0, g.B, Tc, g.B, R, 0)) * Tc
                                      : std::max<long long>((long long)kLmrWaveRounds * R, (long long)g.B * Tc);
    const unsigned grid = (unsigned)((total + kCoderThreads - 1) / kCoderThreads);
    const unsigned fgrid = (unsigned)((total + kFastThreads - 1) / kFastThreads);
    switch (lmr_tile_side(g.tile_log2, g.W)) {
        case 32: coder_encode_fast_kernel<1><<<fgrid, kFastThreads, fast_smem(), st>>>(g, wave, R, ceta, e, sym_count); break;
        case 64: coder_encode_fast_kernel<2><<<fgrid, kFastThreads, fast_smem(), st>>>(g, wave, R, ceta, e, sym_count); break;
        case 128: coder_encode_fast_kernel<4><<<fgrid, kFastThreads, fast_smem(), st>>>(g, wave, R, ceta, e, sym_count); break;
        default: coder_encode_kernel<<<grid, kCoderThreads, coder_smem(), st>>>(g, wave, R, ceta, e);
    }
}

void launch_lmr_fit(const Geo &g, int wave, const LmrEncWS &e, cudaStream_t st) {
    lmr_fit_kernel<<<g.B, 32, 0, st>>>(g, wave, coder_round(g), e);
}

void launch_lmr_msb_write(const Geo &g, const LmrEncWS &e, const uint32_t *hist, uint8_t *enc, int32_t *b_out,
                          int64_t *cap_out, int32_t *status, cudaStream_t st) {
    const long long n32 = g.HW / 32;
    int bx = (int)((n32 + 255) / 256);
    if (bx > 16) bx = 16;
    dim3 grid(bx, g.B);
    const int Tc = lmr_tile_count(g.H, g.W, g.tile_log2);
    const int cx = (2 * Tc + 7) / 8 < 32 ? (2 * Tc + 7) / 8 : 32;
    lmr_concat_kernel<<<dim3(cx, g.B), 256, 0, st>>>(g, e);
    lmr_msb_write_kernel<<<grid, 256, 0, st>>>(g, e, hist, enc, b_out, cap_out, status);
}

void launch_lmr_decode(const Geo &g, bool want_eta, const uint8_t *marked, uint8_t *mbuf, int32_t *lmr_b,
                       int32_t *lmr_t, int32_t *offsets, int32_t *sizes, uint32_t *eta_bits, uint32_t *map_bits,
                       int32_t *status, int64_t *msg_bits_out, unsigned long long *sym_count, cudaStream_t st) {
    lmr_set_smem_attrs();
    const long long n16 = (long long)g.B * g.HW / 16;
    lmr_pack_kernel<<<(unsigned)((n16 + 255) / 256 < 148 * 16 ? (n16 + 255) / 256 : 148 * 16), 256, 0, st>>>(
        g.HW, g.B, marked, mbuf);
    lmr_header_kernel<<<g.B, 32, 0, st>>>(g, mbuf, lmr_b, lmr_t, offsets, sizes, status, msg_bits_out);
    const long long total = (long long)g.B * (want_eta ? 2 : 1) * g.ntiles_coder;
    const unsigned dgrid = (unsigned)((total + kCoderThreads - 1) / kCoderThreads);
    const unsigned fgrid = (unsigned)((total + kFastThreads - 1) / kFastThreads);
    switch (lmr_tile_side(g.tile_log2, g.W)) {
        case 32: coder_decode_fast_kernel<1><<<fgrid, kFastThreads, fast_smem(), st>>>(
                     g, want_eta ? 1 : 0, mbuf, lmr_b, lmr_t, offsets, sizes, eta_bits, map_bits, sym_count); break;
        case 64: coder_decode_fast_kernel<2><<<fgrid, kFastThreads, fast_smem(), st>>>(
                     g, want_eta ? 1 : 0, mbuf, lmr_b, lmr_t, offsets, sizes, eta_bits, map_bits, sym_count); break;
        case 128: coder_decode_fast_kernel<4><<<fgrid, kFastThreads, fast_smem(), st>>>(
                     g, want_eta ? 1 : 0, mbuf, lmr_b, lmr_t, offsets, sizes, eta_bits, map_bits, sym_count); break;
        default: coder_decode_kernel<<<dgrid, kCoderThreads, coder_smem(), st>>>(
                     g, want_eta ? 1 : 0, mbuf, lmr_b, lmr_t, offsets, sizes, eta_bits, map_bits);
    }
}

}  // namespace mmsb
