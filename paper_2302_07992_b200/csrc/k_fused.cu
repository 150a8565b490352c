// k_fused.cu -- the content owner's encode and the K1 receiver's recovery, each ONE launch
// over the whole batch (sm_100a).  Citations: P:<line> = /root/reference/PAPER.md; design
// and roofline: DESIGN.md §5.
//
// Each launch mixes two CTA roles, scheduled by blockIdx in image groups:
//   K (keystream) CTAs  -- a4: ChaCha20(K1) for TPC tiles (one 64-byte block per tile row,
//       P:656, Q12), the tile's in-tile angles (levels 1..tp, eq. roration) turned into
//       a worker record (group table + cell table), the tile total into the upper angle pyramid,
//       and a copy of the call's input tile.  Encode also derives, per pixel, the thermometer code
//       of p ^ left (EMR; its bit 8-b is the location map l = [c < b]) or eta | the thermometer code's bits 0..6
//       (LMR), and the per-image label histogram (eq. gliding1/2 P:604-625 reduce to the left
//       neighbour).  The scratch planes are tile blocks (TileBlock).
//   W (worker) CTAs -- one per strip of tiles, after the image's K CTAs have signalled.  One thread
//       per 4x4 cell; the tiles of the strip stream through a 2-stage shared-memory ring filled by
//       bulk copies (one elected thread, mbarrier transaction counts; consumers release a stage
//       per warp).
//       encode (perm_role): a3 + a5, destination cell <- rotated source cell, location map into
//       the LSB (EMR) or label plane for the coder (LMR), XOR s.
//       recover (rec_role): a10, original cell <- de-rotated destination cell, decrypted; the
//       copy-forward of P:837 / P:1061 is a scan along each row: per cell row a summary byte,
//       a shuffle scan across the tile row, the carry passed from tile to tile.
// Grid order: K(0) | K(1) W(0) | K(2) W(1) | ... | W(n-1): the keystream of group g+1 runs
// while group g is permuted; a W CTA only ever waits for K CTAs dispatched before it.
// The consumed scratch lines are dropped from L2 (discard.global.L2), so the scratch never
// costs HBM bandwidth.
#include "mmsb_device.cuh"
#include "mmsb_kernels.h"

namespace mmsb {

struct Role {
    int key, img, idx;
};

// grid (SK + SW, ngroups + L): row p holds the keystream CTAs of group p and the worker CTAs
// of group p - L, so a worker CTA is dispatched L rows after the keystream CTAs it waits for
__device__ __forceinline__ Role role_of(const FusedSched &sc) {
    const int x = blockIdx.x, p = blockIdx.y, SK = sc.GI << sc.lgK;
    Role r;
    if (x < SK) {
        r.key = 1;
        r.img = p < sc.ngroups ? p * sc.GI + (x >> sc.lgK) : 1 << 30;
        r.idx = x & ((1 << sc.lgK) - 1);
    } else {
        const int loc = x - SK;
        r.key = 0;
        r.img = p >= sc.L ? (p - sc.L) * sc.GI + (loc >> sc.lgW) : 1 << 30;
        r.idx = loc & ((1 << sc.lgW) - 1);
    }
    return r;
}

// Scratch block of a tile: three T x T planes (keystream | input image | label), each row-major
// with the rows of odd cell rows swapped in pairs (row r at position r ^ ((r >> 2) & 1)).  A
// keystream CTA thread writes its tile row as 16-byte stores; a worker thread reads the four rows
// of a 4x4 cell as 4-byte loads from two row pointers, and the 32 cells of a warp (two cell rows,
// rows 4cy + i and 4cy + 4 + i fall in different bank halves) read its own cells without bank
// conflicts.
template <int T> struct TileBlock {
    static constexpr int PLANE = T * T, BLOCK = 3 * T * T;
    static __device__ __forceinline__ int row_pos(int r) { return r ^ ((r >> 2) & 1); }
    static __device__ __forceinline__ uint4 load_cell(const uint8_t *P, int py, int px) {
        const int p = py & 1;
        const uint8_t *ae = P + (4 * py + p) * T + 4 * px, *ao = P + (4 * py + 1 - p) * T + 4 * px;
        return make_uint4(*reinterpret_cast<const uint32_t *>(ae), *reinterpret_cast<const uint32_t *>(ao),
                          *reinterpret_cast<const uint32_t *>(ae + 2 * T), *reinterpret_cast<const uint32_t *>(ao + 2 * T));
    }
};

// one counter of an image's upper pyramid: from the worker's shared-memory copy, or (pyr_glob(g))
// from the workspace in global memory (L2; written by the keystream CTAs' atomics)
template <bool GLOB>
__device__ __forceinline__ uint32_t pyr_at(const uint32_t *pyr_img, int i) {
    if constexpr (GLOB) return __ldcg(pyr_img + i);
    else return pyr_img[i];
}

// destination tile -> source tile under the levels above the tile (walk e = emax .. tp+1)
template <bool GLOB>
__device__ __forceinline__ void upper_walk_inverse(const Geo &g, const uint32_t *pyr_img, int dty, int dtx,
                                                   int &sty, int &stx, int &q) {
    int y = dty, x = dtx;
    q = 0;
    for (int e = g.emax; e > g.tp; e--) {
        const int k = e - g.tp, m1 = (1 << k) - 1;
        const int by = y >> k, bx = x >> k;
        const int a = (int)(pyr_at<GLOB>(pyr_img, g.pyr_off[e] + by * (g.W >> e) + bx) & 3u);
        int oy = y & m1, ox = x & m1;
        inv_turn(a, m1, oy, ox);
        y = (by << k) | oy;
        x = (bx << k) | ox;
        q += a;
    }
    sty = y; stx = x; q &= 3;
}

// original tile -> destination tile (walk e = tp+1 .. emax)
template <bool GLOB>
__device__ __forceinline__ void upper_walk_forward(const Geo &g, const uint32_t *pyr_img, int oty, int otx,
                                                   int &dty, int &dtx, int &q) {
    int y = oty, x = otx;
    q = 0;
    for (int e = g.tp + 1; e <= g.emax; e++) {
        const int k = e - g.tp, m1 = (1 << k) - 1;
        const int by = y >> k, bx = x >> k;
        const int a = (int)(pyr_at<GLOB>(pyr_img, g.pyr_off[e] + by * (g.W >> e) + bx) & 3u);
        int oy = y & m1, ox = x & m1;
        fwd_turn(a, m1, oy, ox);
        y = (by << k) | oy;
        x = (bx << k) | ox;
        q += a;
    }
    dty = y; dtx = x; q &= 3;
}

// EMR optimal b from the non-redundant counts (eq. optimial_b; ties -> smaller b)
__device__ __forceinline__ int emr_select_b(const uint32_t *hist_img, long long HW) {
    int best = 2;
    long long bestv = 2 * (HW - (long long)__ldcg(hist_img + 2));
    for (int b = 3; b <= 7; b++) {
        const long long v = (long long)b * (HW - (long long)__ldcg(hist_img + b));
        if (v > bestv) { best = b; bestv = v; }
    }
    return best;
}

// Cross-CTA wait of a worker on its image's keystream CTAs.  It relies on in-order CTA dispatch
// (the keystream CTAs sit L grid rows earlier); the wait is bounded (~2 s) so that a launch that
// cannot make progress (e.g. an SM partition that holds back earlier CTAs) ends with status
// E_CUDA for the image instead of hanging.
constexpr unsigned kWaitSpins = 1u << 22;
__device__ __forceinline__ bool wait_keys(const TileWS &ws, int img, int nK) {
#if defined(MMSB_PROBE_ROLES)
    if (!(MMSB_PROBE_ROLES & 1)) return true;       // keystream CTAs disabled: nothing to wait for
#endif
    for (unsigned i = 0; i < kWaitSpins; i++) {
        if (ld_acquire_u32(ws.kdone + img) >= (unsigned)nK) return true;
        __nanosleep(512);
    }
    return false;
}

// Warp 0 of a worker CTA: wait for the image's keystream CTAs, then make the upper angle
// pyramid walkable -- copied into shared memory (spyr, sized at launch) in one parallel load.
// Returns false (every lane) if the wait timed out.
template <bool XL>
__device__ __forceinline__ bool warp0_ready(const Geo &g, const TileWS &ws, int img, int nK, uint32_t *spyr) {
    const int lane = threadIdx.x & 31;
    int ok = 1;
    if (lane == 0) ok = wait_keys(ws, img, nK) ? 1 : 0;
    ok = __shfl_sync(0xffffffffu, ok, 0);
    if (!ok) return false;
    fence_proxy_async_global();                      // the scratch the bulk copies will read
    if constexpr (!XL) {
        const uint32_t *pyr_img = ws.pyr + (size_t)img * g.npyr;
        for (int i = lane; i < g.npyr; i += 32) spyr[i] = __ldcg(pyr_img + i);
    }
    __syncwarp();
    return true;
}

// ======================================================================================
// Label histogram helpers (encode K role).
// ======================================================================================
// byte-wise thermometer code of x: every byte becomes 2^bitlen - 1 (bit k set iff byte >= 2^k).
// The right shifts go through the opaque g.one as multiply-high so that they issue on the FMA
// pipe (the ALU pipe is busy with ChaCha).
__device__ __forceinline__ uint32_t smear_bytes(uint32_t x, uint32_t one) {
    uint32_t y = x | (__umulhi(x, one << 31) & 0x7F7F7F7Fu);
    y |= __umulhi(y, one << 30) & 0x3F3F3F3Fu;
    y |= __umulhi(y, one << 28) & 0x0F0F0F0Fu;
    return y;
}
// carry-save adder: (h, l) = (majority, parity) of three bit vectors
__device__ __forceinline__ void csa(uint32_t &h, uint32_t &l, uint32_t a, uint32_t b, uint32_t c) {
    const uint32_t u = a ^ b;
    h = (a & b) | (u & c);
    l = u ^ c;
}
// Harley-Seal vertical counter over 16 words (missing words are 0): every bit lane's count
// = ones + 2 twos + 4 fours + 8 eights + 16 sixteens
template <int N>
__device__ __forceinline__ void hs16(const uint32_t (&y)[N], uint32_t p[5]) {
    auto Y = [&](int i) -> uint32_t { return i < N ? y[i < N ? i : 0] : 0u; };
    uint32_t ones = 0, twos = 0, fours = 0, eights = 0, twosA, twosB, foursA, foursB, eightsA, eightsB;
    csa(twosA, ones, ones, Y(0), Y(1));
    csa(twosB, ones, ones, Y(2), Y(3));
    csa(foursA, twos, twos, twosA, twosB);
    csa(twosA, ones, ones, Y(4), Y(5));
    csa(twosB, ones, ones, Y(6), Y(7));
    csa(foursB, twos, twos, twosA, twosB);
    csa(eightsA, fours, fours, foursA, foursB);
    csa(twosA, ones, ones, Y(8), Y(9));
    csa(twosB, ones, ones, Y(10), Y(11));
    csa(foursA, twos, twos, twosA, twosB);
    csa(twosA, ones, ones, Y(12), Y(13));
    csa(twosB, ones, ones, Y(14), Y(15));
    csa(foursB, twos, twos, twosA, twosB);
    csa(eightsB, fours, fours, foursA, foursB);
    uint32_t sixteens;
    csa(sixteens, eights, eights, eightsA, eightsB);
    p[0] = ones; p[1] = twos; p[2] = fours; p[3] = eights; p[4] = sixteens;
}

// ======================================================================================
// K role: one thread per tile row, TPC = 256 / T tiles per CTA.
//   ENC: encode (copy I, label plane, histogram, inverse group table); else recover (copy I_e',
//   forward group table).
// ======================================================================================
template <int TP>
struct KSmem {
    static constexpr int T = 1 << TP, TPC = 256 / T;
    uint64_t rec[TPC][kRecSlots];                   // in-tile angles, levels 1..tp (slots lvl_off[e] + row)
    __align__(16) uint8_t wrec[TPC][kWRecBytes];    // worker records being built
    uint32_t hsum[8][4];
};

template <int TP, bool ENC, int METHOD>
__device__ __forceinline__ void key_role(const Geo &g, int img, int kidx, const uint8_t *__restrict__ keys,
                                         const uint8_t *__restrict__ src_img, const TileWS &ws, uint8_t *smem) {
    constexpr int T = 1 << TP, NW = T / 4, TPC = 256 / T, NG = T / 8;
    KSmem<TP> &S = *reinterpret_cast<KSmem<TP> *>(smem);

    const int tid = threadIdx.x, lt = tid / T, row = tid % T;
    const int tile = kidx * TPC + lt;
    const bool valid = tile < g.ntiles;
    const int ty = valid ? (tile >> g.tlog) : 0, tx = valid ? (tile & (g.tilesX - 1)) : 0;
    const long long o = (long long)(ty * T + row) * g.W + (long long)tx * T;
    using TB = TileBlock<T>;
    // this thread's row in the tile's scratch block
    uint8_t *rowp = ws.s + ((size_t)img * g.ntiles + tile) * TB::BLOCK + TB::row_pos(row) * T;

    uint32_t key[8];
    load_key(keys, img, key);
    uint32_t blk[16];
    chacha20_block(key, (uint32_t)(o >> 6), blk, g.dr);
    uint32_t w[NW];
    if constexpr (NW == 16) {
#pragma unroll
        for (int i = 0; i < 16; i++) w[i] = blk[i];
    } else {
        const int boff = (int)((o & 63) >> 2);
#pragma unroll
        for (int i = 0; i < NW; i++) w[i] = blk[boff + i];
    }
    // keystream row -> cell-layout scratch (per word, 32 lanes write 128 contiguous bytes), kept
    // in L2 until its worker has read it
    const uint64_t keep = l2_evict_last_policy();
    if (valid) {
#pragma unroll
        for (int c = 0; c < NW; c += 4) st_keep(rowp + 4 * c, make_uint4(w[c], w[c + 1], w[c + 2], w[c + 3]), keep);
    }

    // level 1: 2x2 block sums mod 4 -- horizontal pair sums per row, then the partner row
    uint64_t h1 = 0;
#pragma unroll
    for (int i = 0; i < NW; i++) {
        const uint32_t v = w[i] & 0x03030303u;
        const uint32_t p = (v + (v >> 8)) & 0x00030003u;
        const uint32_t q = (p & 3u) | ((p >> 14) & 0xCu);
        h1 |= (uint64_t)q << (4 * i);
    }
    const uint64_t partner = __shfl_xor_sync(0xffffffffu, h1, 1);
    if ((row & 1) == 0) S.rec[lt][g.lvl_off[1] + row / 2] = add2(h1, partner);

    // the tile row of the call's input image (one 16-byte load per 16 pixels) -> cell-layout scratch
    uint32_t iw[NW];
    {
        const uint8_t *src = src_img + (size_t)img * g.HW + o;
#pragma unroll
        for (int i = 0; i < NW; i += 4) {
            const uint4 u = valid ? __ldcs(reinterpret_cast<const uint4 *>(src) + i / 4) : make_uint4(0, 0, 0, 0);
            iw[i] = u.x; iw[i + 1] = u.y; iw[i + 2] = u.z; iw[i + 3] = u.w;
        }
        if (valid) {
#pragma unroll
            for (int c = 0; c < NW; c += 4)
                st_keep(rowp + TB::PLANE + 4 * c, make_uint4(iw[c], iw[c + 1], iw[c + 2], iw[c + 3]), keep);
        }
    }

    if constexpr (ENC) {
        // per pixel x = p ^ left neighbour (column 0 forced non-redundant) and its
        // thermometer code y (bit k set iff x >= 2^k, i.e. c = # leading equal bits < 8 - k).
        // The label plane for the worker: EMR y itself (l = bit 8-b); LMR eta in bit 7 and bits
        // 0..6 of y (the coder's map bit [c < b] of candidate b = bit 8-b of y, b = 2..8).
        const uint8_t *src = src_img + (size_t)img * g.HW + o;
        uint32_t prev = (valid && tx > 0) ? ((uint32_t)__ldg(src - 1) << 24) : 0u;
        uint32_t yv[NW], lv[NW];
#pragma unroll
        for (int i = 0; i < NW; i++) {
            const uint32_t left = __byte_perm(prev, iw[i], 0x6543);   // [prev.b3, w.b0, w.b1, w.b2]
            uint32_t x = iw[i] ^ left;
            if (i == 0 && tx == 0) x |= 0xFFu;
            prev = iw[i];
            const uint32_t y = smear_bytes(x, g.one);
            yv[i] = y;
            uint32_t lab;
            if constexpr (METHOD == 0) lab = y;
            else lab = (y & 0x7F7F7F7Fu) | (iw[i] & 0x80808080u);
            lv[i] = lab;
        }
        if (valid) {
#pragma unroll
            for (int c = 0; c < NW; c += 4)
                st_keep(rowp + 2 * TB::PLANE + 4 * c, make_uint4(lv[c], lv[c + 1], lv[c + 2], lv[c + 3]), keep);
        }
        // label histogram: for b = 2..8 the non-redundant pixels (c < b) = bit 8-b of y.  The
        // bit lanes of the row's words are counted by a carry-save (Harley-Seal) network, then
        // threshold k = 8 - b is the sum over the 4 byte lanes of bit k of every plane.
        uint32_t pl[5];
        hs16<NW>(yv, pl);
        uint32_t cnt[7];
#pragma unroll
        for (int k = 0; k < 7; k++) {
            const uint32_t mk = 0x01010101u << k;
            if (METHOD == 0 && k == 0) { cnt[k] = 0; continue; }        // b = 8: LMR only
            cnt[k] = __popc(pl[0] & mk) + 2 * __popc(pl[1] & mk) + 4 * __popc(pl[2] & mk) + 8 * __popc(pl[3] & mk) +
                     16 * __popc(pl[4] & mk);
        }
        // threshold bit k <-> b = 8 - k; per-thread counts <= 64, warp sums <= 2048: two counts
        // per 32-bit word for the warp reduction
        uint32_t pk[4] = {cnt[0] | (cnt[1] << 16), cnt[2] | (cnt[3] << 16), cnt[4] | (cnt[5] << 16), cnt[6]};
        if (!valid) pk[0] = pk[1] = pk[2] = pk[3] = 0;               // a row past the image's tiles counts nothing
#pragma unroll
        for (int j = 0; j < 4; j++) pk[j] = __reduce_add_sync(0xffffffffu, pk[j]);   // REDUX: one instruction per word
        // per-CTA sum, then one atomic per count (a 4096^2 image has 1024 keystream CTAs)
        if ((tid & 31) == 0) {
#pragma unroll
            for (int j = 0; j < 4; j++) S.hsum[tid >> 5][j] = pk[j];
        }
        __syncthreads();
        if (tid < 7 && (METHOD == 1 || tid > 0)) {                  // b = 8 (k = 0): LMR only
            uint32_t v = 0;
            for (int w8 = 0; w8 < 8; w8++) v += (S.hsum[w8][tid >> 1] >> (16 * (tid & 1))) & 0xFFFFu;
            if (v) atomicAdd(&ws.hist[img * kHistStride + 8 - tid], v);
        }
    }
    __syncthreads();

    // levels 2..tp: quad-tree sums mod 4 of the level below
#pragma unroll
    for (int e = 2; e <= TP; e++) {
        const int R = T >> e;
        for (int t = tid; t < TPC * R; t += 256) {
            const int l2 = t / R, r = t % R;
            const uint64_t v = add2(S.rec[l2][g.lvl_off[e - 1] + 2 * r], S.rec[l2][g.lvl_off[e - 1] + 2 * r + 1]);
            const uint64_t pe = v & 0x3333333333333333ull, po = (v >> 2) & 0x3333333333333333ull;
            uint64_t s = (pe + po) & 0x3333333333333333ull;
            s = (s | (s >> 2)) & 0x0F0F0F0F0F0F0F0Full;
            s = (s | (s >> 4)) & 0x00FF00FF00FF00FFull;
            s = (s | (s >> 8)) & 0x0000FFFF0000FFFFull;
            s = (s | (s >> 16)) & 0x00000000FFFFFFFFull;
            S.rec[l2][g.lvl_off[e] + r] = s;
        }
        __syncthreads();
    }

    // Worker record.  Group table: levels 4..tp move 2x2-cell groups rigidly; the level-3 turn of
    // the original group (a rotation of its 2x2 cells, applied first) is folded into the entry's
    // turn count.  Forward (recover): entry[original group] = group after those levels << 2 | turns;
    // inverse (encode): entry[group after those levels] = original group << 2 | turns (3-bit
    // coordinates).  Then the level-1 rows (u64, 2-bit angle per 2x2 block) and the level-2 rows
    // (u32, one angle per 4x4 cell) for the cells' own turns; levels below e_min are 0.
    {
        constexpr int NGG = NG * NG;
        for (int t = tid; t < TPC * NGG; t += 256) {
            const int l2 = t / NGG, gi = t % NGG;
            int gy = gi / NG, gx = gi % NG, q = 0;
            for (int e = (g.emin > 4 ? g.emin : 4); e <= TP; e++) {
                const int k = e - 3, m1 = (1 << k) - 1;
                const int by = gy >> k, bx = gx >> k;
                const int a = rec_angle(S.rec[l2], g, e, by, bx);
                int oy = gy & m1, ox = gx & m1;
                fwd_turn(a, m1, oy, ox);
                gy = (by << k) | oy;
                gx = (bx << k) | ox;
                q += a;
            }
            if (g.emin <= 3) q += rec_angle(S.rec[l2], g, 3, gi / NG, gi % NG);
            uint8_t *tab = S.wrec[l2];
            if constexpr (ENC) tab[gy * NG + gx] = (uint8_t)((((gi / NG) << 5) | ((gi % NG) << 2)) | (q & 3));
            else tab[gi] = (uint8_t)((gy << 5) | (gx << 2) | (q & 3));
        }
        for (int t = tid; t < TPC * (T / 2 + T / 4); t += 256) {
            const int l2 = t / (T / 2 + T / 4), r = t % (T / 2 + T / 4);
            if (r < T / 2)
                reinterpret_cast<uint64_t *>(S.wrec[l2] + kWRecL1)[r] = g.emin <= 1 ? S.rec[l2][g.lvl_off[1] + r] : 0ull;
            else
                reinterpret_cast<uint32_t *>(S.wrec[l2] + kWRecL2)[r - T / 2] =
                    g.emin <= 2 ? (uint32_t)S.rec[l2][g.lvl_off[2] + r - T / 2] : 0u;
        }
        __syncthreads();
    }
    // upper pyramid: the tile totals (= level-tp angles) into every enclosing block, summed over
    // the CTA's tiles first (neighbouring tiles share the upper blocks: fewer contended atomics)
    if (tid < 32) {
        for (int e = TP + 1 + tid; e <= g.emax; e += 32) {
            const int k = e - TP;
            int cur = -1;
            uint32_t acc = 0;
            for (int l2 = 0; l2 < TPC; l2++) {
                const int tl = kidx * TPC + l2;
                if (tl >= g.ntiles) break;
                const int blk = ((tl >> g.tlog) >> k) * (g.W >> e) + ((tl & (g.tilesX - 1)) >> k);
                if (blk != cur) {
                    if (acc) atomicAdd(&ws.pyr[(size_t)img * g.npyr + g.pyr_off[e] + cur], acc);
                    cur = blk;
                    acc = 0;
                }
                acc += (uint32_t)(S.rec[l2][g.lvl_off[TP]] & 3u);
            }
            if (acc) atomicAdd(&ws.pyr[(size_t)img * g.npyr + g.pyr_off[e] + cur], acc);
        }
    }
    // worker records out (16-byte stores)
    for (int t = tid; t < TPC * (kWRecBytes / 16); t += 256) {
        const int l2 = t / (kWRecBytes / 16), c = t % (kWRecBytes / 16);
        const int tl = kidx * TPC + l2;
        if (tl < g.ntiles)
            reinterpret_cast<uint4 *>(ws.rec + ((size_t)img * g.ntiles + tl) * kRecSlots)[c] =
                reinterpret_cast<const uint4 *>(S.wrec[l2])[c];
    }
    // publish: the proxy fence and the barrier order the CTA's scratch writes before thread 0's
    // release arrival on the image's counter (release is cumulative); workers read them by bulk copy
    fence_proxy_async_global();
    __syncthreads();
    if (tid == 0) red_release_add_u32(ws.kdone + img, 1u);
}

// ======================================================================================
// Worker roles.  One worker CTA per strip of tiles (one tile row of the image), walking the
// strip left to right.  Stage ring of kStages tiles: thread 0 issues the bulk copies of tile
// j + kStages once the 8 warps have released tile j (empty barrier, one arrival per warp).
// ======================================================================================
#ifndef MMSB_STAGES
#define MMSB_STAGES 2
#endif
constexpr int kStages = MMSB_STAGES;

__device__ __forceinline__ uint32_t bits4_to_bytes(uint32_t m4) { return ((m4 & 0xFu) * 0x00204081u) & 0x01010101u; }
// byte LSBs (bits 0, 8, 16, 24) -> bits 0..3: one multiply puts them at bits 21..24 (no other term lands there)
// (l * (2^7 + 2^14 + 2^21 + 2^28)) moves bit 8k to 28 + k with no other term at or above bit 28
__device__ __forceinline__ uint32_t bytes_to_bits4(uint32_t l) { return (l * 0x10204080u) >> 28; }

// a cell's own turns from the worker record: level-2 angle (bits 0-1), level-1 angles of its
// upper (bits 2-5) and lower (bits 6-9) 2x2 block pairs
__device__ __forceinline__ uint32_t cell_turns(const uint8_t *wrec, int py, int px) {
    const uint32_t *l1 = reinterpret_cast<const uint32_t *>(wrec + kWRecL1);
    const uint32_t *l2 = reinterpret_cast<const uint32_t *>(wrec + kWRecL2);
    const int sh = 4 * (px & 7), wi = 4 * py + (px >> 3);
    return ((l2[py] >> (2 * px)) & 3u) | (((l1[wi] >> sh) & 0xFu) << 2) | (((l1[wi + 2] >> sh) & 0xFu) << 6);
}

constexpr int kMapInline = 512;                  // strip tiles held in the struct (W <= 32768 at 64-pixel tiles)
template <int TP, bool ENC>
struct WSmem {
    static constexpr int T = 1 << TP;
    struct Stage {
        uint4 ks[ENC ? T * T / 16 : 1];      // encode: keystream of the destination tile
        uint4 src[2 * T * T / 16];           // encode: source tile's image | label planes;
                                             // recover: destination tile's keystream | image planes
        uint4 rec[kWRecBytes / 16];          // worker record (encode: source tile; recover: original tile)
    } st[kStages];
    uint64_t full[kStages], empty[kStages];
    int map[kMapInline];                     // per tile of the strip: other tile << 2 | upper turns
                                             // (longer strips: the dynamic tail, fused_smem)
    uint32_t fsel[16];                       // copy-forward PRMT selectors by 4-bit map
    int sh[4];
};

// copy-forward selector: nibble i = index of the last set bit of m at or below i, else 4
__device__ __forceinline__ uint32_t fsel_of(int m) {
    uint32_t v = 0;
    int last = 4;
    for (int i = 0; i < 4; i++) {
        if ((m >> i) & 1) last = i;
        v |= (uint32_t)last << (4 * i);
    }
    return v;
}

// the consumed scratch leaves L2 unwritten (its bulk copies have completed): lines [0, n) of a
// region, dropped by the 32 lanes of one warp
__device__ __forceinline__ void discard_lines(const void *p, int n, int lane) {
    for (int i = lane; i < n; i += 32) discard_l2(static_cast<const uint8_t *>(p) + 128 * i);
}

// ======================================================================================
// W role, encode (a3, a5): destination strip dty, tiles left to right, thread = destination cell.
//   EMR: carrier v = (I & 0xFE) | l with l = [c < b] (location map), permuted as a
//        whole byte; E = v_r XOR (s & 0xFE) (eq. image_encryption P:739 + LSB map P:744);
//        header b-2 in the LSBs of r = 0..2 (Q14).
//   LMR: E = I_r XOR s; second plane ceta = (I & 0x80) | (y & 0x7F) permuted alongside (for the
//        coder: eta = bit 7, the map bit [c < b] = bit 8-b).
// ======================================================================================
template <int TP, int METHOD, bool SPLIT, bool XL>
__device__ __forceinline__ void perm_role(const Geo &g, int img, int dty, int seg, int lgS, int nK, const TileWS &ws,
                                          uint8_t *__restrict__ enc, uint8_t *__restrict__ ceta_out,
                                          int32_t *__restrict__ b_out, int64_t *__restrict__ cap_out,
                                          int32_t *__restrict__ status, uint8_t *smem) {
    constexpr int T = 1 << TP, NC = T / 4, NG = NC / 2;
    using TB = TileBlock<T>;
    using SM = WSmem<TP, true>;
    SM &S = *reinterpret_cast<SM *>(smem);
    uint32_t *spyr = reinterpret_cast<uint32_t *>(smem + sizeof(SM));
    // XL (images above 8192^2 or strips longer than kMapInline tiles, a separate instantiation):
    // the upper pyramid is walked in global memory and the strip map lives in the dynamic tail
    int *smap = XL ? reinterpret_cast<int *>(spyr) : S.map;
    const uint32_t *gpyr = ws.pyr + (size_t)img * g.npyr;
    const int tid = threadIdx.x, lane = tid & 31;
    if constexpr (!SPLIT) { seg = 0; lgS = 0; }

    if (tid == 0) {
        for (int s = 0; s < kStages; s++) {
            mbar_init(&S.full[s], 1);
            mbar_init(&S.empty[s], 8);
        }
    }
    if (tid < 32) {
        const bool ok = warp0_ready<XL>(g, ws, img, nK, spyr);
        if (ok) {
            for (int j = tid; j < (g.tilesX >> lgS); j += 32) {
                int sty, stx, q;
                upper_walk_inverse<XL>(g, XL ? gpyr : spyr, dty, (seg << (g.tlog - lgS)) + j, sty, stx, q);
                smap[j] = (((sty << g.tlog) + stx) << 2) | q;
            }
        }
        if (tid == 0) {
            S.sh[0] = METHOD == 0 && ok ? emr_select_b(ws.hist + img * kHistStride, g.HW) : 0;
            S.sh[1] = ok;
            if (!ok) status[img] = 6;                       // MMSB_E_CUDA: keystream CTAs never arrived
        }
    }
    __syncthreads();
    if (!S.sh[1]) return;
    const int b = S.sh[0];
    const int ntx = g.tilesX >> lgS, j0 = seg * ntx;                // this worker's tiles [j0, j0 + ntx) of the strip
    const uint8_t *blk0 = ws.s + (size_t)img * g.ntiles * TB::BLOCK;      // the image's scratch blocks
    const uint64_t *rec0 = ws.rec + (size_t)img * g.ntiles * kRecSlots;

    auto issue = [&](int j) {
        const int s = j % kStages;
        if (j >= kStages) mbar_wait(&S.empty[s], ((j / kStages) - 1) & 1);
        const int stile = smap[j] >> 2, dtile = (dty << g.tlog) + j0 + j;
        mbar_expect_tx(&S.full[s], 3 * T * T + kWRecBytes);
        bulk_g2s(S.st[s].ks, blk0 + (size_t)dtile * TB::BLOCK, T * T, &S.full[s]);
        bulk_g2s(S.st[s].src, blk0 + (size_t)stile * TB::BLOCK + TB::PLANE, 2 * T * T, &S.full[s]);
        bulk_g2s(S.st[s].rec, rec0 + (size_t)stile * kRecSlots, kWRecBytes, &S.full[s]);
    };
    if (tid == 0)
        for (int j = 0; j < kStages && j < ntx; j++) issue(j);

    // this thread's destination cell and its candidate group / sub-cell positions for the 4
    // possible upper turns of the tile (undo the tile's own turn first)
    const bool act = NC * NC >= 256 || tid < NC * NC;    // 64-pixel tiles: every thread has a cell
    const int cy = act ? tid / NC : 0, cx = act ? tid % NC : 0;
    uint32_t gpos = 0, spos = 0;
#pragma unroll
    for (int q = 0; q < 4; q++) {
        int gy = cy >> 1, gx = cx >> 1, sy = cy & 1, sx = cx & 1;
        inv_turn(q, NG - 1, gy, gx);
        inv_turn(q, 1, sy, sx);
        gpos |= (uint32_t)(gy * NG + gx) << (8 * q);
        spos |= (uint32_t)(sy * 2 + sx) << (2 * q);
    }
    // opaque from here on: under the 40-register cap ptxas otherwise recomputes both tables from
    // tid in every tile iteration (ncu source page: 14 + ~30 instructions per tile and warp)
    asm volatile("" : "+r"(gpos), "+r"(spos));
    const int lsh = 8 - b;                                   // EMR: map bit l = bit 8 - b of the thermometer code
    // output rows of this thread's cell in the worker's first tile (the tile advances by T bytes)
    const size_t W = (size_t)g.W;
    uint8_t *eo = enc + (size_t)img * g.HW + (size_t)(dty * T + 4 * cy) * W + (size_t)j0 * T + 4 * cx;
    uint8_t *co = METHOD == 1 ? ceta_out + (size_t)img * g.HW + (size_t)(dty * T + 4 * cy) * W + (size_t)j0 * T + 4 * cx
                              : nullptr;

    int s = 0;
    unsigned ph = 0;
    for (int j = 0; j < ntx; j++) {
        mbar_wait_sleep(&S.full[s], ph);
        const typename SM::Stage &st = S.st[s];
        const int mp = smap[j];
        if (tid >= 224) {                                    // warp 7: drop the consumed scratch from L2
            const int dtile = (dty << g.tlog) + j0 + j;
            discard_lines(blk0 + (size_t)dtile * TB::BLOCK, T * T / 128, lane);
            discard_lines(blk0 + (size_t)(mp >> 2) * TB::BLOCK + TB::PLANE, 2 * T * T / 128, lane);
            discard_lines(rec0 + (size_t)(mp >> 2) * kRecSlots, kRecSlots * 8 / 128, lane);
        }
        if (act) {
            const int q_up = mp & 3;
            const uint8_t *wrec = reinterpret_cast<const uint8_t *>(st.rec);
            const uint32_t ge = wrec[(gpos >> (8 * q_up)) & 0xFFu];
            const int q = q_up + (int)ge;
            const int s2 = (int)(spos >> (2 * (q & 3))) & 3;
            const int py = 2 * (int)(ge >> 5) + (s2 >> 1), px = 2 * (int)((ge >> 2) & 7) + (s2 & 1);
            const uint32_t ce = cell_turns(wrec, py, px);
            const int r = (q + (int)ce) & 3;
            const uint8_t *src = reinterpret_cast<const uint8_t *>(st.src);
            const uint4 wv = TB::load_cell(src, py, px), yv = TB::load_cell(src + TB::PLANE, py, px);
            Cell v, cl;
            if constexpr (METHOD == 0) {
                v.r0 = (wv.x & 0xFEFEFEFEu) | ((yv.x >> lsh) & 0x01010101u);
                v.r1 = (wv.y & 0xFEFEFEFEu) | ((yv.y >> lsh) & 0x01010101u);
                v.r2 = (wv.z & 0xFEFEFEFEu) | ((yv.z >> lsh) & 0x01010101u);
                v.r3 = (wv.w & 0xFEFEFEFEu) | ((yv.w >> lsh) & 0x01010101u);
            } else {
                v = {wv.x, wv.y, wv.z, wv.w};
                cl = {yv.x, yv.y, yv.z, yv.w};
            }
            if (g.emin <= 1) {
                const uint32_t a01 = (ce >> 2) & 0xFu, a23 = (ce >> 6) & 0xFu;
                pair_rot_cw(v.r0, v.r1, a01 & 3, a01 >> 2);
                pair_rot_cw(v.r2, v.r3, a23 & 3, a23 >> 2);
                if constexpr (METHOD == 1) {
                    pair_rot_cw(cl.r0, cl.r1, a01 & 3, a01 >> 2);
                    pair_rot_cw(cl.r2, cl.r3, a23 & 3, a23 >> 2);
                }
            }
            v = cell_rot_cw(v, r);
            if constexpr (METHOD == 1) cl = cell_rot_cw(cl, r);

            const uint4 sv = TB::load_cell(reinterpret_cast<const uint8_t *>(st.ks), cy, cx);
            uint32_t e0, e1, e2, e3;
            if constexpr (METHOD == 0) {
                e0 = v.r0 ^ (sv.x & 0xFEFEFEFEu); e1 = v.r1 ^ (sv.y & 0xFEFEFEFEu);
                e2 = v.r2 ^ (sv.z & 0xFEFEFEFEu); e3 = v.r3 ^ (sv.w & 0xFEFEFEFEu);
                if (dty == 0 && j0 + j == 0 && tid == 0) {
                    // header: LSB(E[r]) = bit (2 - r) of b - 2 for r = 0..2; the map there is
                    // forced to 1, so capacity counts zeros after forcing (Q14)
                    const uint32_t m = v.r0 & 0x00010101u;
                    const int forced = (int)(m & 1u) + (int)((m >> 8) & 1u) + (int)((m >> 16) & 1u);
                    const uint32_t hb = (uint32_t)(b - 2);
                    const uint32_t hdr = ((hb >> 2) & 1u) | (((hb >> 1) & 1u) << 8) | ((hb & 1u) << 16);
                    e0 = (e0 & 0xFFFEFEFEu) | hdr;
                    const long long zeros = g.HW - (long long)__ldcg(ws.hist + img * kHistStride + b);
                    b_out[img] = b;
                    cap_out[img] = (long long)b * (zeros - (3 - forced));
                    status[img] = 0;
                }
            } else {
                e0 = v.r0 ^ sv.x; e1 = v.r1 ^ sv.y; e2 = v.r2 ^ sv.z; e3 = v.r3 ^ sv.w;
                __stcs(reinterpret_cast<unsigned *>(co), cl.r0);
                __stcs(reinterpret_cast<unsigned *>(co + W), cl.r1);
                __stcs(reinterpret_cast<unsigned *>(co + 2 * W), cl.r2);
                __stcs(reinterpret_cast<unsigned *>(co + 3 * W), cl.r3);
                co += T;
            }
            __stcs(reinterpret_cast<unsigned *>(eo), e0);
            __stcs(reinterpret_cast<unsigned *>(eo + W), e1);
            __stcs(reinterpret_cast<unsigned *>(eo + 2 * W), e2);
            __stcs(reinterpret_cast<unsigned *>(eo + 3 * W), e3);
            eo += T;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.empty[s]);               // this warp is done with stage s
        if (tid == 0 && j + kStages < ntx) issue(j + kStages);
        if (++s == kStages) { s = 0; ph ^= 1u; }
    }
}

// ======================================================================================
// W role, recover (a10): original strip ty, tiles left to right, thread = original cell.
//   X = I_e' XOR s (every bit, Q20); EMR: map bit = raw LSB of I_e' (r < 3 forced to 1);
//   LMR: MSB := eta_r and the map come from the decoded planes.  Inverse cell transform into
//   the original domain in registers, then per row omega := masked bits of the last
//   non-redundant pixel, replaced into the redundant ones:
//     * per cell row, xf = (X & mask) | flag for the non-redundant pixels (the flag bit lies
//       outside the mask: EMR bit 0, b <= 7; LMR bit 7, restored from eta), and
//       om = PRMT(xf, carry, fsel[m4]) gives every pixel the flagged value of the last
//       non-redundant pixel at or before it (byte 3 = the cell row's summary);
//     * the 4 summaries of a cell are one word; an inclusive shuffle scan over the cells of the
//       tile row (combine = "right if flagged else left", per byte) gives each cell its carry,
//       the tile's carry moves on to the next tile of the strip in a register.
// ======================================================================================
template <int TP, int METHOD, bool SSE, bool XL>
__device__ __forceinline__ void rec_role(const Geo &g, int img, int ty, int nK, const uint8_t *__restrict__ marked,
                                         const TileWS &ws, const uint32_t *__restrict__ eta_bits,
                                         const uint32_t *__restrict__ map_bits, const int32_t *__restrict__ lmr_b,
                                         uint8_t *__restrict__ out, int32_t *__restrict__ status,
                                         const uint8_t *__restrict__ orig, unsigned long long *__restrict__ sse,
                                         uint8_t *smem) {
    constexpr int T = 1 << TP, NC = T / 4, NG = NC / 2;
    using TB = TileBlock<T>;
    using SM = WSmem<TP, false>;
    SM &S = *reinterpret_cast<SM *>(smem);
    uint32_t *spyr = reinterpret_cast<uint32_t *>(smem + sizeof(SM));
    // XL (images above 8192^2 or strips longer than kMapInline tiles, a separate instantiation):
    // the upper pyramid is walked in global memory and the strip map lives in the dynamic tail
    int *smap = XL ? reinterpret_cast<int *>(spyr) : S.map;
    const uint32_t *gpyr = ws.pyr + (size_t)img * g.npyr;
    const int tid = threadIdx.x, lane = tid & 31;
    const uint8_t *Em = marked + (size_t)img * g.HW;
    uint8_t *O = out + (size_t)img * g.HW;

    if (tid >= 32 && tid < 48) S.fsel[tid - 32] = fsel_of(tid - 32);
    if (tid < 32) {
        int b = 0;
        if (tid == 0) {
            for (int s = 0; s < kStages; s++) {
                mbar_init(&S.full[s], 1);
                mbar_init(&S.empty[s], 8);
            }
            if constexpr (METHOD == 0) {
                const int field = ((Em[0] & 1) << 2) | ((Em[1] & 1) << 1) | (Em[2] & 1);
                b = field > 5 ? -1 : field + 2;
                if (ty == 0) status[img] = b < 0 ? 8 : 0;
            } else {
                b = __ldcg(lmr_b + img);                // <= 0: status already set by the decoder
                if (ty == 0 && b > 0) status[img] = 0;
            }
            S.sh[0] = b;
        }
        b = __shfl_sync(0xffffffffu, b, 0);
        if (b > 0) {
            if (warp0_ready<XL>(g, ws, img, nK, spyr)) {
                for (int j = tid; j < g.tilesX; j += 32) {
                    int dty, dtx, q;
                    upper_walk_forward<XL>(g, XL ? gpyr : spyr, ty, j, dty, dtx, q);
                    smap[j] = (((dty << g.tlog) + dtx) << 2) | q;
                }
            } else if (tid == 0) {
                S.sh[0] = 0;
                status[img] = 6;                            // MMSB_E_CUDA: keystream CTAs never arrived
            }
        }
    }
    __syncthreads();
    const int b = S.sh[0];
    if (b <= 0) {                                       // FORMAT / BADCASE: zero-filled output
        uint32_t sq0 = 0;
        for (int c = tid; c < T * g.W / 16; c += 256) {
            const int r = c / (g.W / 16), col = c % (g.W / 16);
            const size_t off = (size_t)(ty * T + r) * g.W + col * 16;
            *reinterpret_cast<uint4 *>(O + off) = make_uint4(0, 0, 0, 0);
            if constexpr (SSE) {                         // (I - 0)^2
                const uint4 v = __ldcs(reinterpret_cast<const uint4 *>(orig + (size_t)img * g.HW + off));
                sq0 = __dp4a(v.x, v.x, __dp4a(v.y, v.y, __dp4a(v.z, v.z, __dp4a(v.w, v.w, sq0))));
            }
        }
        if constexpr (SSE) {
            unsigned long long v = sq0;
#pragma unroll
            for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
            if (lane == 0 && v) atomicAdd(sse + img, v);
        }
        return;
    }
    const uint32_t mask = METHOD == 0 ? ((0xFFu << (8 - b)) & 0xFFu) : (0x7Fu & ~(0xFFu >> b));
    const uint32_t maskb = mask * 0x01010101u;
    const int ntx = g.tilesX;
    const uint8_t *blk0 = ws.s + (size_t)img * g.ntiles * TB::BLOCK;
    const uint64_t *rec0 = ws.rec + ((size_t)img * g.ntiles + ((size_t)ty << g.tlog)) * kRecSlots;

    auto issue = [&](int j) {
        const int s = j % kStages;
        if (j >= kStages) mbar_wait(&S.empty[s], ((j / kStages) - 1) & 1);
        const int dt = smap[j] >> 2;
        mbar_expect_tx(&S.full[s], 2 * T * T + kWRecBytes);
        bulk_g2s(S.st[s].src, blk0 + (size_t)dt * TB::BLOCK, 2 * T * T, &S.full[s]);
        bulk_g2s(S.st[s].rec, rec0 + (size_t)j * kRecSlots, kWRecBytes, &S.full[s]);
    };
    if (tid == 0)
        for (int j = 0; j < kStages && j < ntx; j++) issue(j);

    const bool act = NC * NC >= 256 || tid < NC * NC;    // 64-pixel tiles: every thread has a cell
    const int cy = act ? tid / NC : 0, cx = act ? tid % NC : 0;
    uint32_t spos = 0;                                   // sub-cell position after q turns (forward)
#pragma unroll
    for (int q = 0; q < 4; q++) {
        int sy = cy & 1, sx = cx & 1;
        fwd_turn(q, 1, sy, sx);
        spos |= (uint32_t)(sy * 2 + sx) << (2 * q);
    }
    asm volatile("" : "+r"(spos));                       // kept, not recomputed per tile (see perm_role)
    constexpr uint32_t HB = METHOD == 0 ? 0x01u : 0x80u;            // flag bit, outside the mask
    constexpr uint32_t HBW = HB * 0x01010101u;
    // combine(a, b) per byte: b if flagged else a
    auto combine = [&](uint32_t a, uint32_t bb) -> uint32_t {
        const uint32_t f = bb & HBW;
        const uint32_t m = (METHOD == 0 ? f : (f >> 7)) * 0xFFu;
        return (bb & m) | (a & ~m);
    };
    const int cw = NC < 32 ? NC : 32;                    // lanes holding one tile row's cells
    const int hlast = (lane & ~(cw - 1)) + cw - 1;       // the last of them
    uint32_t carry = 0;                                  // summaries leaving the previous tile (4 rows)
    const size_t W = (size_t)g.W;
    uint8_t *op = O + (size_t)(ty * T + 4 * cy) * W + 4 * cx;   // this cell's rows in tile 0 of the strip
    const uint8_t *ip = SSE ? orig + (size_t)img * g.HW + (size_t)(ty * T + 4 * cy) * W + 4 * cx : nullptr;
    uint32_t sq = 0;                                     // SSE of this thread's cells (<= 2^31 per strip)

    int s = 0;
    unsigned ph = 0;
    for (int j = 0; j < ntx; j++) {
        mbar_wait_sleep(&S.full[s], ph);
        const int mp = smap[j], dt = mp >> 2, q_up = mp & 3;
        if (tid >= 224)                                      // warp 7: drop the consumed scratch from L2
        {
            discard_lines(blk0 + (size_t)dt * TB::BLOCK, 2 * T * T / 128, lane);
            discard_lines(rec0 + (size_t)j * kRecSlots, kRecSlots * 8 / 128, lane);
        }
        const typename SM::Stage &st = S.st[s];
        uint32_t xw[4] = {0, 0, 0, 0}, xf[4] = {0, 0, 0, 0}, sel[4] = {0x4444u, 0x4444u, 0x4444u, 0x4444u};
        uint32_t summ = 0;
        if (act) {
            const uint8_t *wrec = reinterpret_cast<const uint8_t *>(st.rec);
            const uint32_t ge = wrec[(cy >> 1) * NG + (cx >> 1)];
            int dgy = (int)(ge >> 5), dgx = (int)((ge >> 2) & 7);
            fwd_turn(q_up, NG - 1, dgy, dgx);                // then the tile's own turn
            const int q = q_up + (int)ge;
            const int s2 = (int)(spos >> (2 * (q & 3))) & 3;
            const int py = 2 * dgy + (s2 >> 1), px = 2 * dgx + (s2 & 1);
            const uint32_t ce = cell_turns(wrec, cy, cx);
            const uint8_t *src = reinterpret_cast<const uint8_t *>(st.src);
            const uint4 sv = TB::load_cell(src, py, px), ev = TB::load_cell(src + TB::PLANE, py, px);
            Cell x = {ev.x ^ sv.x, ev.y ^ sv.y, ev.z ^ sv.z, ev.w ^ sv.w};
            Cell l;
            if constexpr (METHOD == 0) {
                l = {ev.x & 0x01010101u, ev.y & 0x01010101u, ev.z & 0x01010101u, ev.w & 0x01010101u};
                if (dt == 0 && py == 0 && px == 0) l.r0 |= 0x00010101u;   // header pixels, map 1
            } else {
                const int dty = dt >> g.tlog, dtx = dt & (g.tilesX - 1);
                const size_t bit0 = (size_t)img * g.HW + (size_t)(dty * T + 4 * py) * g.W + (size_t)dtx * T + 4 * px;
                uint32_t lr[4], er[4];
#pragma unroll
                for (int i = 0; i < 4; i++) {
                    const size_t bit = bit0 + (size_t)i * g.W;
                    lr[i] = bits4_to_bytes(__ldg(map_bits + (bit >> 5)) >> (bit & 31));
                    er[i] = bits4_to_bytes(__ldg(eta_bits + (bit >> 5)) >> (bit & 31)) << 7;   // MSB <- eta
                }
                l = {lr[0], lr[1], lr[2], lr[3]};
                x = {(x.r0 & 0x7F7F7F7Fu) | er[0], (x.r1 & 0x7F7F7F7Fu) | er[1], (x.r2 & 0x7F7F7F7Fu) | er[2],
                     (x.r3 & 0x7F7F7F7Fu) | er[3]};
            }
            const int rinv = (4 - ((q + (int)ce) & 3)) & 3;
            x = cell_rot_cw(x, rinv);
            l = cell_rot_cw(l, rinv);
            if (g.emin <= 1) {
                const uint32_t a01 = (ce >> 2) & 0xFu, a23 = (ce >> 6) & 0xFu;
                const int aL0 = (4 - (a01 & 3)) & 3, aR0 = (4 - (a01 >> 2)) & 3;
                const int aL1 = (4 - (a23 & 3)) & 3, aR1 = (4 - (a23 >> 2)) & 3;
                pair_rot_cw(x.r0, x.r1, aL0, aR0);
                pair_rot_cw(x.r2, x.r3, aL1, aR1);
                pair_rot_cw(l.r0, l.r1, aL0, aR0);
                pair_rot_cw(l.r2, l.r3, aL1, aR1);
            }
            xw[0] = x.r0; xw[1] = x.r1; xw[2] = x.r2; xw[3] = x.r3;
            const uint32_t lw[4] = {l.r0, l.r1, l.r2, l.r3};
            const bool col0 = j == 0 && cx == 0;             // column 0: omega starts at its bits
            uint32_t om0[4];
#pragma unroll
            for (int i = 0; i < 4; i++) {
                const uint32_t lf = lw[i] | (col0 ? 1u : 0u);
                sel[i] = S.fsel[bytes_to_bits4(lf)];
                xf[i] = (xw[i] & maskb) | (METHOD == 0 ? lf : (lf << 7));
                om0[i] = prmt(xf[i], 0, sel[i]);
            }
            // the cell's 4 row summaries (byte 3 of each om0) in one word
            summ = __byte_perm(__byte_perm(om0[0], om0[1], 0x0073), __byte_perm(om0[2], om0[3], 0x7300), 0x7610);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.empty[s]);             // the stage's data is in registers
        if (tid == 0 && j + kStages < ntx) issue(j + kStages);
        // inclusive scan of the summaries over the cells of the tile row (cw lanes per row)
        uint32_t v = summ;
#pragma unroll
        for (int d = 1; d < cw; d <<= 1) {
            const uint32_t u = __shfl_up_sync(0xffffffffu, v, d, cw);
            if (cx >= d) v = combine(u, v);
        }
        const uint32_t left = __shfl_up_sync(0xffffffffu, v, 1, cw);
        const uint32_t cin = cx == 0 ? carry : combine(carry, left);
        carry = combine(carry, __shfl_sync(0xffffffffu, v, hlast));
        if (act) {
            uint32_t o4[4];
#pragma unroll
            for (int i = 0; i < 4; i++) {
                const uint32_t cb = __byte_perm(cin, 0, 0x1111u * (uint32_t)i);   // row i's carry in every byte
                const uint32_t om = prmt(xf[i], cb, sel[i]);
                o4[i] = (xw[i] & ~maskb) | (om & maskb);
            }
            __stcs(reinterpret_cast<unsigned *>(op), o4[0]);
            __stcs(reinterpret_cast<unsigned *>(op + W), o4[1]);
            __stcs(reinterpret_cast<unsigned *>(op + 2 * W), o4[2]);
            __stcs(reinterpret_cast<unsigned *>(op + 3 * W), o4[3]);
            op += T;
            if constexpr (SSE) {                             // (I - I')^2 of the cell
#pragma unroll
                for (int i = 0; i < 4; i++) {
                    const uint32_t d = __vabsdiffu4(__ldcs(reinterpret_cast<const unsigned *>(ip + i * W)), o4[i]);
                    sq = __dp4a(d, d, sq);
                }
                ip += T;
            }
        }
        if (++s == kStages) { s = 0; ph ^= 1u; }
    }
    if constexpr (SSE) {                                 // the strip's sum: one atomic per warp
        unsigned long long v = sq;
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
        if (lane == 0 && v) atomicAdd(sse + img, v);
    }
}

// ======================================================================================
// The fused kernels (dynamic shared memory: max of the two roles' needs + the pyramid)
// ======================================================================================
template <int TP, int METHOD, bool SPLIT, bool XL>
__global__ void __launch_bounds__(256, 6) encode_kernel(Geo g, FusedSched sc, const uint8_t *__restrict__ images,
                                                     const uint8_t *__restrict__ keys, TileWS ws,
                                                     uint8_t *__restrict__ enc, uint8_t *__restrict__ ceta,
                                                     int32_t *__restrict__ b_out, int64_t *__restrict__ cap_out,
                                                     int32_t *__restrict__ status) {
    extern __shared__ __align__(128) uint8_t smem[];
    const Role ro = role_of(sc);
    if (ro.img >= g.B) return;
#ifdef MMSB_PROBE_ROLES   // performance probes only (tools/role_probe.py): 1 = keystream CTAs only, 2 = workers only
    if (!((MMSB_PROBE_ROLES >> (ro.key ? 0 : 1)) & 1)) return;
#endif
    if (ro.key) key_role<TP, true, METHOD>(g, ro.img, ro.idx, keys, images, ws, smem);
    else if constexpr (SPLIT)
        perm_role<TP, METHOD, true, XL>(g, ro.img, ro.idx >> sc.lgS, ro.idx & ((1 << sc.lgS) - 1), sc.lgS, 1 << sc.lgK, ws,
                                    enc, ceta, b_out, cap_out, status, smem);
    else
        perm_role<TP, METHOD, false, XL>(g, ro.img, ro.idx, 0, 0, 1 << sc.lgK, ws, enc, ceta, b_out, cap_out, status, smem);
}

template <int TP, int METHOD, bool SSE, bool XL>
__global__ void __launch_bounds__(256, 6) recover_kernel(Geo g, FusedSched sc, const uint8_t *__restrict__ marked,
                                                      const uint8_t *__restrict__ keys, TileWS ws,
                                                      const uint32_t *__restrict__ eta_bits,
                                                      const uint32_t *__restrict__ map_bits,
                                                      const int32_t *__restrict__ lmr_b, uint8_t *__restrict__ out,
                                                      int32_t *__restrict__ status, const uint8_t *__restrict__ orig,
                                                      unsigned long long *__restrict__ sse) {
    extern __shared__ __align__(128) uint8_t smem[];
    const Role ro = role_of(sc);
    if (ro.img >= g.B) return;
#ifdef MMSB_PROBE_ROLES
    if (!((MMSB_PROBE_ROLES >> (ro.key ? 0 : 1)) & 1)) return;
#endif
    if (ro.key) key_role<TP, false, METHOD>(g, ro.img, ro.idx, keys, marked, ws, smem);
    else rec_role<TP, METHOD, SSE, XL>(g, ro.img, ro.idx, 1 << sc.lgK, marked, ws, eta_bits, map_bits, lmr_b, out, status,
                                   orig, sse, smem);
}

// ---------------------------------------------------------------------------- launchers
FusedSched fused_sched(const Geo &g, bool split_strips) {
    FusedSched sc;
    const int TPC = 256 / g.T;
    const int nK = g.ntiles >= TPC ? g.ntiles / TPC : 1;       // powers of two
    sc.lgK = ilog2(nK);
    // one worker CTA per strip of tiles; encode cuts strips wider than 8 tiles into segments of
    // 8 (a 4096^2 image: 512 workers of 8 tiles instead of 64 of 64, so the batch's last image
    // does not leave a long tail of strip walks)
    sc.lgS = split_strips && g.tilesX > 8 ? ilog2(g.tilesX / 8) : 0;
    sc.lgW = ilog2(g.tilesY) + sc.lgS;
    int gi = 1;
    while ((long long)(gi * 2) * g.HW <= (2ll << 20) && gi < g.B) gi *= 2;   // ~2 Mpixel per group
    sc.GI = gi;
    sc.ngroups = (g.B + gi - 1) / gi;
    // keystream rows run L rows ahead of their workers: enough to hide the keystream latency,
    // few enough that the scratch (3 B/px) and the images of L groups stay in L2
    // (measured on config 2: 12 Mpixel of lag beat 4 / 6 Mpixel by 3-6 %, a cap of 8 or 10 rows changed nothing)
    constexpr long long budget = 12ll << 20;
    constexpr int lcap = 6;
    long long lag = budget / ((long long)gi * g.HW);
    sc.L = (int)(lag < 1 ? 1 : lag > lcap ? lcap : lag);
    return sc;
}

static dim3 fused_grid(const FusedSched &sc) {
    return dim3((unsigned)((sc.GI << sc.lgK) + (sc.GI << sc.lgW)), (unsigned)(sc.ngroups + sc.L));
}

// the XL instantiation: images whose upper pyramid is too large for shared memory (pyr_glob) or
// whose strips are longer than kMapInline tiles (H < 64 makes the tiles narrower than 64, e.g.
// 16 x 32768: 2048 tiles per strip)
static bool fused_xl(const Geo &g) { return pyr_glob(g) || g.tilesX > kMapInline; }

template <int TP, bool ENC>
static size_t fused_smem(const Geo &g) {
    // worker: the stage ring and the upper angle pyramid; XL: the ring and the strip's tile map
    const size_t k = sizeof(KSmem<TP>),
                 w = sizeof(WSmem<TP, ENC>) + (fused_xl(g) ? (size_t)g.tilesX * 4 : (size_t)g.npyr * 4);
    return k > w ? k : w;
}

template <int TP, bool SPLIT, bool XL>
static void launch_encode_x(const Geo &g, const FusedSched &sc, dim3 grid, size_t sm, const uint8_t *images,
                            const uint8_t *keys, const TileWS &ws, uint8_t *enc, uint8_t *ceta, int32_t *b_out,
                            int64_t *cap_out, int32_t *status, cudaStream_t st) {
    if (g.method == 0) {
        cudaFuncSetAttribute(encode_kernel<TP, 0, SPLIT, XL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        encode_kernel<TP, 0, SPLIT, XL><<<grid, 256, sm, st>>>(g, sc, images, keys, ws, enc, ceta, b_out, cap_out, status);
    } else {
        cudaFuncSetAttribute(encode_kernel<TP, 1, SPLIT, XL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        encode_kernel<TP, 1, SPLIT, XL><<<grid, 256, sm, st>>>(g, sc, images, keys, ws, enc, ceta, b_out, cap_out, status);
    }
}
template <int TP, bool SPLIT>
static void launch_encode_k(const Geo &g, const FusedSched &sc, dim3 grid, size_t sm, const uint8_t *images,
                            const uint8_t *keys, const TileWS &ws, uint8_t *enc, uint8_t *ceta, int32_t *b_out,
                            int64_t *cap_out, int32_t *status, cudaStream_t st) {
    if (fused_xl(g)) launch_encode_x<TP, SPLIT, true>(g, sc, grid, sm, images, keys, ws, enc, ceta, b_out, cap_out, status, st);
    else launch_encode_x<TP, SPLIT, false>(g, sc, grid, sm, images, keys, ws, enc, ceta, b_out, cap_out, status, st);
}

template <int TP>
static void launch_encode_tp(const Geo &g, const uint8_t *images, const uint8_t *keys, const TileWS &ws, uint8_t *enc,
                             uint8_t *ceta, int32_t *b_out, int64_t *cap_out, int32_t *status, cudaStream_t st) {
    const FusedSched sc = fused_sched(g, true);
    const dim3 grid = fused_grid(sc);
    const size_t sm = fused_smem<TP, true>(g);
    if (sc.lgS) launch_encode_k<TP, true>(g, sc, grid, sm, images, keys, ws, enc, ceta, b_out, cap_out, status, st);
    else launch_encode_k<TP, false>(g, sc, grid, sm, images, keys, ws, enc, ceta, b_out, cap_out, status, st);
}

void launch_encode(const Geo &g, const uint8_t *images, const uint8_t *keys, const TileWS &ws, uint8_t *enc,
                   uint8_t *ceta, int32_t *b_out, int64_t *cap_out, int32_t *status, cudaStream_t st) {
    switch (g.tp) {
        case 4: launch_encode_tp<4>(g, images, keys, ws, enc, ceta, b_out, cap_out, status, st); break;
        case 5: launch_encode_tp<5>(g, images, keys, ws, enc, ceta, b_out, cap_out, status, st); break;
        default: launch_encode_tp<6>(g, images, keys, ws, enc, ceta, b_out, cap_out, status, st); break;
    }
}

template <int TP, int METHOD, bool SSE>
static void launch_recover_k(const Geo &g, const FusedSched &sc, const uint8_t *marked, const uint8_t *keys,
                             const TileWS &ws, const uint32_t *eta, const uint32_t *map, const int32_t *lmr_b,
                             uint8_t *out, int32_t *status, const uint8_t *orig, unsigned long long *sse, cudaStream_t st) {
    const size_t sm = fused_smem<TP, false>(g);
    if (fused_xl(g)) {
        cudaFuncSetAttribute(recover_kernel<TP, METHOD, SSE, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        recover_kernel<TP, METHOD, SSE, true><<<fused_grid(sc), 256, sm, st>>>(g, sc, marked, keys, ws, eta, map, lmr_b,
                                                                                out, status, orig, sse);
    } else {
        cudaFuncSetAttribute(recover_kernel<TP, METHOD, SSE, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        recover_kernel<TP, METHOD, SSE, false><<<fused_grid(sc), 256, sm, st>>>(g, sc, marked, keys, ws, eta, map, lmr_b,
                                                                                 out, status, orig, sse);
    }
}

template <int TP>
static void launch_recover_tp(const Geo &g, const uint8_t *marked, const uint8_t *keys, const TileWS &ws,
                              const uint32_t *eta, const uint32_t *map, const int32_t *lmr_b, uint8_t *out,
                              int32_t *status, const uint8_t *orig, unsigned long long *sse, cudaStream_t st) {
    const FusedSched sc = fused_sched(g);
    if (g.method == 0) {
        if (sse) launch_recover_k<TP, 0, true>(g, sc, marked, keys, ws, eta, map, lmr_b, out, status, orig, sse, st);
        else launch_recover_k<TP, 0, false>(g, sc, marked, keys, ws, eta, map, lmr_b, out, status, orig, sse, st);
    } else {
        if (sse) launch_recover_k<TP, 1, true>(g, sc, marked, keys, ws, eta, map, lmr_b, out, status, orig, sse, st);
        else launch_recover_k<TP, 1, false>(g, sc, marked, keys, ws, eta, map, lmr_b, out, status, orig, sse, st);
    }
}

void launch_recover(const Geo &g, const uint8_t *marked, const uint8_t *keys, const TileWS &ws, const uint32_t *eta,
                    const uint32_t *map, const int32_t *lmr_b, uint8_t *out, int32_t *status, cudaStream_t st,
                    const uint8_t *original, unsigned long long *sse) {
    switch (g.tp) {
        case 4: launch_recover_tp<4>(g, marked, keys, ws, eta, map, lmr_b, out, status, original, sse, st); break;
        case 5: launch_recover_tp<5>(g, marked, keys, ws, eta, map, lmr_b, out, status, original, sse, st); break;
        default: launch_recover_tp<6>(g, marked, keys, ws, eta, map, lmr_b, out, status, original, sse, st); break;
    }
}

}  // namespace mmsb
