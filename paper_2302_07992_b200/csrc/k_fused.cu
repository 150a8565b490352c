// k_fused.cu -- the content owner's encode and the K1 receiver's recovery, each ONE launch
// over the whole batch (sm_100a).  Citations: P:<line> = /root/reference/PAPER.md; design
// and roofline: DESIGN.md §5.
//
// Each launch mixes two CTA roles, scheduled by blockIdx in image groups:
//   K (keystream) CTAs  -- a4: ChaCha20(K1) for TPC tiles (one 64-byte block per tile row,
//       P:656, Q12), the tile's in-tile angle record (levels 1..tp, eq. roration),
//       the tile total into the upper angle pyramid, and (encode) the per-image label
//       histogram (eq. gliding1/2 P:604-625 reduce to the left neighbour).  The
//       keystream goes to a tile-major scratch that only one consumer reads.
//   W (worker) CTAs -- one per tile, after the image's K CTAs have signalled:
//       encode (perm_role): a3 + a5, destination tile <- permuted source tile (+ left halo),
//       location map into the LSB (EMR) or label plane for the coder (LMR), XOR s.
//       recover (rec_role): a10, original tile <- de-permuted destination tile, decrypted,
//       rows copied forward with the carry from the tile to the left found by a per-row
//       decoupled look-back (the copy-forward of P:837 / P:1061 is a scan along each row).
// Grid order: K(0) | K(1) W(0) | K(2) W(1) | ... | W(n-1): the keystream of group g+1 runs
// while group g is permuted; a W CTA only ever waits for K CTAs dispatched before it.
// The consumed keystream tile and angle record are dropped from L2 (discard.global.L2),
// so the scratch never costs HBM bandwidth.
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

// destination tile -> source tile under the levels above the tile (walk e = emax .. tp+1)
__device__ __forceinline__ void upper_walk_inverse(const Geo &g, const uint32_t *pyr_img, int dty, int dtx,
                                                   int &sty, int &stx, int &q) {
    int y = dty, x = dtx;
    q = 0;
    for (int e = g.emax; e > g.tp; e--) {
        const int k = e - g.tp, m1 = (1 << k) - 1;
        const int by = y >> k, bx = x >> k;
        const int a = (int)(pyr_img[g.pyr_off[e] + by * (g.W >> e) + bx] & 3u);
        int oy = y & m1, ox = x & m1;
        inv_turn(a, m1, oy, ox);
        y = (by << k) | oy;
        x = (bx << k) | ox;
        q += a;
    }
    sty = y; stx = x; q &= 3;
}

// original tile -> destination tile (walk e = tp+1 .. emax)
__device__ __forceinline__ void upper_walk_forward(const Geo &g, const uint32_t *pyr_img, int oty, int otx,
                                                   int &dty, int &dtx, int &q) {
    int y = oty, x = otx;
    q = 0;
    for (int e = g.tp + 1; e <= g.emax; e++) {
        const int k = e - g.tp, m1 = (1 << k) - 1;
        const int by = y >> k, bx = x >> k;
        const int a = (int)(pyr_img[g.pyr_off[e] + by * (g.W >> e) + bx] & 3u);
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

__device__ __forceinline__ void wait_keys(const TileWS &ws, int img, int nK) {
#if defined(MMSB_PROBE_ROLES)
    if (!(MMSB_PROBE_ROLES & 1)) return;            // keystream CTAs disabled: nothing to wait for
#endif
    while (ld_acquire_u32(ws.kdone + img) < (unsigned)nK) __nanosleep(512);
}

// Warp 0 of a worker CTA: wait for the image's keystream CTAs, then make the upper angle
// pyramid walkable -- copied into shared memory in one parallel load when it is small
// (<= kPyrSmem counters: images up to 2048^2), else walked in L2.  Returns the pointer.
constexpr int kPyrSmem = 1536;
__device__ __forceinline__ const uint32_t *warp0_ready(const Geo &g, const TileWS &ws, int img, int nK,
                                                       uint32_t *spyr) {
    const int lane = threadIdx.x & 31;
    if (lane == 0) wait_keys(ws, img, nK);
    __syncwarp();
    const uint32_t *pyr_img = ws.pyr + (size_t)img * g.npyr;
    if (g.npyr > kPyrSmem) return pyr_img;
    for (int i = lane; i < g.npyr; i += 32) spyr[i] = __ldcg(pyr_img + i);
    __syncwarp();
    return spyr;
}

// ======================================================================================
// K role: one thread per tile row, TPC = 256 / T tiles per CTA.
// ======================================================================================
template <int TP, bool HIST, bool INV, bool LMR8 = true>
__device__ __forceinline__ void key_role(const Geo &g, int img, int kidx, const uint8_t *__restrict__ keys,
                                         const uint8_t *__restrict__ images, const TileWS &ws, uint8_t *smem) {
    constexpr int T = 1 << TP, NW = T / 4, TPC = 256 / T;
    uint64_t(*rec)[kRecSlots] = reinterpret_cast<uint64_t(*)[kRecSlots]>(smem);

    const int tid = threadIdx.x, lt = tid / T, row = tid % T;
    const int tile = kidx * TPC + lt;
    const bool valid = tile < g.ntiles;
    const int ty = valid ? (tile >> g.tlog) : 0, tx = valid ? (tile & (g.tilesX - 1)) : 0;
    const long long o = (long long)(ty * T + row) * g.W + (long long)tx * T;

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
    // keystream row -> tile-major scratch (a warp writes whole tiles rows: contiguous)
    if (valid) {
        uint8_t *sd = ws.s + ((size_t)img * g.ntiles + tile) * (T * T) + row * T;
#pragma unroll
        for (int i = 0; i < NW; i += 4)
            *reinterpret_cast<uint4 *>(sd + 4 * i) = make_uint4(w[i], w[i + 1], w[i + 2], w[i + 3]);
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
    if ((row & 1) == 0) rec[lt][g.lvl_off[1] + row / 2] = add2(h1, partner);

    if constexpr (HIST) {
        // label histogram of this tile row: for b = 2..8, pixels with c < b (non-redundant),
        // i.e. x = p ^ left >= 2^(8-b).  Bit-smear x into a thermometer code y, then count
        // bit (8-b) of y with byte-lane counters (<= 16 * 8 per lane: no overflow).
        const uint8_t *src = images + (size_t)img * g.HW + o;
        uint32_t iw[NW];
#pragma unroll
        for (int i = 0; i < NW; i += 4) {
            const uint4 u = valid ? __ldg(reinterpret_cast<const uint4 *>(src) + i / 4) : make_uint4(0, 0, 0, 0);
            iw[i] = u.x; iw[i + 1] = u.y; iw[i + 2] = u.z; iw[i + 3] = u.w;
        }
        uint32_t prev = (valid && tx > 0) ? ((uint32_t)__ldg(src - 1) << 24) : 0u;
        // The shifts (as multiply-high) and the counter adds (as multiply-add) go through the
        // opaque g.one so that they issue on the FMA pipe: the ALU pipe is busy with ChaCha.
        uint32_t acc[7] = {0, 0, 0, 0, 0, 0, 0};
        const uint32_t one = g.one, h1 = one << 31, h2 = one << 30, h4 = one << 28;
#pragma unroll
        for (int i = 0; i < NW; i++) {
            const uint32_t left = __byte_perm(prev, iw[i], 0x6543);   // [prev.b3, w.b0, w.b1, w.b2]
            uint32_t x = iw[i] ^ left;
            if (i == 0 && tx == 0) x |= 0xFFu;                     // column 0 is non-redundant
            prev = iw[i];
            uint32_t y = x | (__umulhi(x, h1) & 0x7F7F7F7Fu);
            y |= __umulhi(y, h2) & 0x3F3F3F3Fu;
            y |= __umulhi(y, h4) & 0x0F0F0F0Fu;                    // byte = 2^bitlen(x) - 1
            const uint32_t y4 = __umulhi(y, h4) & 0x0F0F0F0Fu;
            if (LMR8) acc[0] = (y & 0x01010101u) * one + acc[0];   // b = 8: LMR only
            acc[1] = (y & 0x02020202u) * one + acc[1];
            acc[2] = (y & 0x04040404u) * one + acc[2];
            acc[3] = (y & 0x08080808u) * one + acc[3];
            acc[4] = (y4 & 0x01010101u) * one + acc[4];
            acc[5] = (y4 & 0x02020202u) * one + acc[5];
            acc[6] = (y4 & 0x04040404u) * one + acc[6];
        }
        // threshold bit k <-> b = 8 - k; per-thread counts <= 64, warp sums <= 2048: two
        // counts per 32-bit word for the warp reduction
        uint32_t cnt[7];
#pragma unroll
        for (int k = 0; k < 7; k++) cnt[k] = valid ? (((acc[k] >> (k & 3)) * 0x01010101u) >> 24) : 0u;
        uint32_t pk[4] = {cnt[0] | (cnt[1] << 16), cnt[2] | (cnt[3] << 16), cnt[4] | (cnt[5] << 16), cnt[6]};
#pragma unroll
        for (int j = 0; j < 4; j++) {
#pragma unroll
            for (int s = 16; s > 0; s >>= 1) pk[j] += __shfl_xor_sync(0xffffffffu, pk[j], s);
        }
        // per-CTA sum, then one atomic per count: a 4096^2 image has 1024 keystream CTAs, and
        // per-warp atomics on the image's 7 counters serialised at L2
        uint32_t *hsum = reinterpret_cast<uint32_t *>(&rec[TPC][0]);       // [8 warps][4]
        if ((tid & 31) == 0) {
#pragma unroll
            for (int j = 0; j < 4; j++) hsum[(tid >> 5) * 4 + j] = pk[j];
        }
        __syncthreads();
        if (tid < 7) {
            uint32_t v = 0;
            for (int w = 0; w < 8; w++) v += (hsum[w * 4 + (tid >> 1)] >> (16 * (tid & 1))) & 0xFFFFu;
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
            const uint64_t v = add2(rec[l2][g.lvl_off[e - 1] + 2 * r], rec[l2][g.lvl_off[e - 1] + 2 * r + 1]);
            const uint64_t pe = v & 0x3333333333333333ull, po = (v >> 2) & 0x3333333333333333ull;
            uint64_t s = (pe + po) & 0x3333333333333333ull;
            s = (s | (s >> 2)) & 0x0F0F0F0F0F0F0F0Full;
            s = (s | (s >> 4)) & 0x00FF00FF00FF00FFull;
            s = (s | (s >> 8)) & 0x0000FFFF0000FFFFull;
            s = (s | (s >> 16)) & 0x00000000FFFFFFFFull;
            rec[l2][g.lvl_off[e] + r] = s;
        }
        __syncthreads();
    }

    // in-tile 8x8-group map: levels 4..tp move 2x2-cell groups rigidly.  Forward (recover):
    // entry[original group] = group after those levels << 2 | turns; inverse (encode):
    // entry[group after those levels] = original group << 2 | turns (3-bit coordinates).
    {
        constexpr int NG = T / 8, NGG = NG * NG;
        for (int t = tid; t < TPC * NGG; t += 256) {
            const int l2 = t / NGG, gi = t % NGG;
            int gy = gi / NG, gx = gi % NG, q = 0;
            for (int e = (g.emin > 4 ? g.emin : 4); e <= TP; e++) {
                const int k = e - 3, m1 = (1 << k) - 1;
                const int by = gy >> k, bx = gx >> k;
                const int a = rec_angle(rec[l2], g, e, by, bx);
                int oy = gy & m1, ox = gx & m1;
                fwd_turn(a, m1, oy, ox);
                gy = (by << k) | oy;
                gx = (bx << k) | ox;
                q += a;
            }
            uint8_t *tab = reinterpret_cast<uint8_t *>(&rec[l2][kRecGroupSlot]);
            if (INV) tab[gy * NG + gx] = (uint8_t)((((gi / NG) << 5) | ((gi % NG) << 2)) | (q & 3));
            else tab[gi] = (uint8_t)((gy << 5) | (gx << 2) | (q & 3));
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
                acc += (uint32_t)(rec[l2][g.lvl_off[TP]] & 3u);
            }
            if (acc) atomicAdd(&ws.pyr[(size_t)img * g.npyr + g.pyr_off[e] + cur], acc);
        }
    }
    // records out
    for (int t = tid; t < TPC * kRecSlots; t += 256) {
        const int l2 = t / kRecSlots, slot = t % kRecSlots;
        const int tl = kidx * TPC + l2;
        if (tl < g.ntiles) ws.rec[((size_t)img * g.ntiles + tl) * kRecSlots + slot] = rec[l2][slot];
    }
    // publish: the barrier orders the CTA's writes before thread 0's release arrival on the
    // image's counter (release is cumulative)
    __syncthreads();
    if (tid == 0) red_release_add_u32(ws.kdone + img, 1u);
}

// ======================================================================================
// Worker roles.  One worker CTA per strip of tiles (one tile row of the image), walking the
// strip left to right with a two-stage cp.async pipeline: the next tile's data is in flight
// while the current one is transformed.  The tile map of the strip (upper-level walks) is
// computed once, up front, by warp 0 from the angle pyramid.
// ======================================================================================
constexpr int kMaxTilesX = 512;                  // W <= 32768 with 64-pixel tiles

__device__ __forceinline__ uint32_t bits4_to_bytes(uint32_t m4) { return ((m4 & 0xFu) * 0x00204081u) & 0x01010101u; }
// byte LSBs (bits 0, 8, 16, 24) -> bits 0..3: one multiply puts them at bits 21..24 (no other term lands there)
__device__ __forceinline__ uint32_t bytes_to_bits4(uint32_t l) { return ((l * 0x00204081u) >> 21) & 0xFu; }

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async4(void *smem, const void *gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// ======================================================================================
// W role, encode (a3, a5): destination strip dty, tiles left to right.
//   EMR: carrier v = (I & 0xFE) | l with l = [c < b] (location map), permuted as a
//        whole byte; E = v_r XOR (s & 0xFE) (eq. image_encryption P:739 + LSB map P:744);
//        header b-2 in the LSBs of r = 0..2 (Q14).
//   LMR: E = I_r XOR s; second plane ceta = (I & 0x80) | c permuted alongside (for the coder).
// The carrier / label of a source pixel needs its left neighbour: computed per cell row from
// the staged source tile (and, at the tile's left edge, the staged halo word).
// ======================================================================================
template <int TP>
struct PermSmem {
    static constexpr int T = 1 << TP;
    struct Stage {
        uint32_t is[T * T / 4];              // source tile of I (row-major words)
        uint32_t halo[T];                    // per row: the aligned word left of the row (byte 3)
        uint32_t ss[T * T / 4];              // keystream of the destination tile (tile-major)
        uint64_t rec[kRecSlots];             // angle record of the source tile
    } st[2];
    uint32_t pyr[kPyrSmem];                  // upper angle pyramid of the image (small images)
    int smap[kMaxTilesX];                    // per destination tile of the strip: source << 2 | q
    int sh[4];
};

template <int TP, int METHOD>
__device__ __forceinline__ void perm_role(const Geo &g, int img, int dty, int nK, const uint8_t *__restrict__ images,
                                          const TileWS &ws, uint8_t *__restrict__ enc, uint8_t *__restrict__ ceta_out,
                                          int32_t *__restrict__ b_out, int64_t *__restrict__ cap_out,
                                          int32_t *__restrict__ status, uint8_t *smem) {
    constexpr int T = 1 << TP, NW = T / 4, NC = T / 4, NCELL = NC * NC, CPT = T * T / 16, NG = NC / 2;
    PermSmem<TP> &S = *reinterpret_cast<PermSmem<TP> *>(smem);
    const int tid = threadIdx.x;
    const uint8_t *I = images + (size_t)img * g.HW;

    if (tid < 32) {
        const uint32_t *pyr = warp0_ready(g, ws, img, nK, S.pyr);
        for (int j = tid; j < g.tilesX; j += 32) {
            int sty, stx, q;
            upper_walk_inverse(g, pyr, dty, j, sty, stx, q);
            S.smap[j] = (((sty << g.tlog) + stx) << 2) | q;
        }
        if (tid == 0) S.sh[0] = METHOD == 0 ? emr_select_b(ws.hist + img * kHistStride, g.HW) : 0;
    }
    __syncthreads();
    const int b = S.sh[0];
    const uint32_t MB = METHOD == 0 ? ((0xFFu << (8 - b)) & 0xFFu) * 0x01010101u : 0u;

    auto issue = [&](int j) {
        typename PermSmem<TP>::Stage &st = S.st[j & 1];
        const int stile = S.smap[j] >> 2, sty = stile >> g.tlog, stx = stile & (g.tilesX - 1);
        const size_t dslot = (size_t)img * g.ntiles + ((size_t)dty << g.tlog) + j;
        for (int c = tid; c < CPT; c += 256) {
            const int r = c / (T / 16), seg = c % (T / 16);
            cp_async16(&st.is[r * NW + seg * 4], I + (size_t)(sty * T + r) * g.W + (size_t)stx * T + seg * 16);
            cp_async16(&st.ss[4 * c], ws.s + dslot * (T * T) + 16 * c);
        }
        if (tid < T && stx > 0) cp_async4(&st.halo[tid], I + (size_t)(sty * T + tid) * g.W + (size_t)stx * T - 4);
        if (tid < kRecSlots / 2)
            cp_async16(&st.rec[2 * tid], ws.rec + ((size_t)img * g.ntiles + stile) * kRecSlots + 2 * tid);
        cp_async_commit();
    };

    issue(0);
    for (int j = 0; j < g.tilesX; j++) {
        if (j + 1 < g.tilesX) {
            issue(j + 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();                                           // stage j landed for everyone
        const typename PermSmem<TP>::Stage &st = S.st[j & 1];
        const int mp = S.smap[j], stile = mp >> 2, q_up = mp & 3;
        const int stx = stile & (g.tilesX - 1);
        const int dtile = (dty << g.tlog) + j;
        {   // the consumed scratch (destination keystream, source record) leaves L2 unwritten
            const size_t dslot = (size_t)img * g.ntiles + dtile;
            if (tid < (T * T) / 128) discard_l2(ws.s + dslot * (T * T) + 128 * tid);
            else if (tid >= 64 && tid < 64 + kRecSlots * 8 / 128)
                discard_l2(ws.rec + ((size_t)img * g.ntiles + stile) * kRecSlots + 16 * (tid - 64));
        }
        for (int c = tid; c < NCELL; c += 256) {
            // destination cell -> source cell: group walk (levels >= 4, q_up), level 3 inside the
            // group, then in-cell levels 1, 2
            const int gi = c >> 2, sub = c & 3;
            const int cy = 2 * (gi / NG) + (sub >> 1), cx = 2 * (gi % NG) + (sub & 1);
            int dgy = gi / NG, dgx = gi % NG;
            inv_turn(q_up, NG - 1, dgy, dgx);               // undo the tile's own turn, then the
            const uint32_t ge = reinterpret_cast<const uint8_t *>(st.rec + kRecGroupSlot)[dgy * NG + dgx];
            const int sgy = ge >> 5, sgx = (ge >> 2) & 7;    // in-tile levels >= 4 (group table)
            int q = q_up + (int)(ge & 3);
            if (g.emin <= 3) q += rec_angle(st.rec, g, 3, sgy, sgx);
            int sy = sub >> 1, sx = sub & 1;
            inv_turn(q & 3, 1, sy, sx);
            const int py = 2 * sgy + sy, px = 2 * sgx + sx;
            // source cell rows -> carrier (EMR) / image + label|eta (LMR)
            uint32_t vr[4], cr[4] = {0, 0, 0, 0};
#pragma unroll
            for (int i = 0; i < 4; i++) {
                const int row = 4 * py + i;
                const uint32_t w = st.is[row * NW + px];
                const uint32_t pw = px > 0 ? st.is[row * NW + px - 1] : (stx > 0 ? st.halo[row] : 0u);
                uint32_t x = w ^ __byte_perm(pw, w, 0x6543);      // p ^ left neighbour, per byte
                if (px == 0 && stx == 0) x |= 0xFFu;               // column 0: always non-redundant
                if constexpr (METHOD == 0) {
                    const uint32_t t = x & MB;
                    const uint32_t nz = (((t & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | t) & 0x80808080u;   // byte != 0
                    vr[i] = (w & 0xFEFEFEFEu) | (nz >> 7);
                } else {
                    uint32_t cv = 0;                               // c = # leading equal bits per byte
#pragma unroll
                    for (int k = 0; k < 4; k++) {
                        const uint32_t xb = (x >> (8 * k)) & 0xFFu;
                        cv |= (xb ? (uint32_t)(__clz(xb) - 24) : 8u) << (8 * k);
                    }
                    cr[i] = cv | (w & 0x80808080u);
                    vr[i] = w;
                }
            }
            Cell v = {vr[0], vr[1], vr[2], vr[3]};
            Cell cl = {cr[0], cr[1], cr[2], cr[3]};
            if (g.emin <= 1) {
                const uint32_t a01 = (uint32_t)(st.rec[g.lvl_off[1] + 2 * py] >> (4 * px)) & 0xFu;
                const uint32_t a23 = (uint32_t)(st.rec[g.lvl_off[1] + 2 * py + 1] >> (4 * px)) & 0xFu;
                pair_rot_cw(v.r0, v.r1, a01 & 3, a01 >> 2);
                pair_rot_cw(v.r2, v.r3, a23 & 3, a23 >> 2);
                if constexpr (METHOD == 1) {
                    pair_rot_cw(cl.r0, cl.r1, a01 & 3, a01 >> 2);
                    pair_rot_cw(cl.r2, cl.r3, a23 & 3, a23 >> 2);
                }
            }
            if (g.emin <= 2) q += rec_angle(st.rec, g, 2, py, px);
            v = cell_rot_cw(v, q & 3);
            if constexpr (METHOD == 1) cl = cell_rot_cw(cl, q & 3);

            const uint32_t *sw = st.ss + (4 * cy) * NW + cx;
            const uint32_t s0 = sw[0], s1 = sw[NW], s2 = sw[2 * NW], s3 = sw[3 * NW];
            const size_t base = (size_t)(dty * T + 4 * cy) * g.W + (size_t)j * T + 4 * cx;
            uint32_t e0, e1, e2, e3;
            if constexpr (METHOD == 0) {
                e0 = v.r0 ^ (s0 & 0xFEFEFEFEu); e1 = v.r1 ^ (s1 & 0xFEFEFEFEu);
                e2 = v.r2 ^ (s2 & 0xFEFEFEFEu); e3 = v.r3 ^ (s3 & 0xFEFEFEFEu);
                if (dtile == 0 && c == 0) {
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
                e0 = v.r0 ^ s0; e1 = v.r1 ^ s1; e2 = v.r2 ^ s2; e3 = v.r3 ^ s3;
                uint8_t *co = ceta_out + (size_t)img * g.HW + base;
                *reinterpret_cast<uint32_t *>(co) = cl.r0;
                *reinterpret_cast<uint32_t *>(co + g.W) = cl.r1;
                *reinterpret_cast<uint32_t *>(co + 2 * (size_t)g.W) = cl.r2;
                *reinterpret_cast<uint32_t *>(co + 3 * (size_t)g.W) = cl.r3;
            }
            uint8_t *eo = enc + (size_t)img * g.HW + base;
            *reinterpret_cast<uint32_t *>(eo) = e0;
            *reinterpret_cast<uint32_t *>(eo + g.W) = e1;
            *reinterpret_cast<uint32_t *>(eo + 2 * (size_t)g.W) = e2;
            *reinterpret_cast<uint32_t *>(eo + 3 * (size_t)g.W) = e3;
        }
        __syncthreads();                                           // stage j free for tile j + 2
    }
}

// ======================================================================================
// W role, recover (a10): original strip ty, tiles left to right.
//   X = I_e' XOR s (every bit, Q20); EMR: map bit = raw LSB of I_e' (r < 3 forced to 1);
//   LMR: MSB := eta_r and the map come from the decoded planes.  Inverse cell transform into
//   the original domain, then per row omega := masked bits of the last non-redundant pixel,
//   replaced into the redundant ones; the row's omega carries from tile to
//   tile inside the CTA.
// ======================================================================================
template <int TP>
struct RecSmem {
    static constexpr int T = 1 << TP, RS = T / 4 + 1;
    struct Stage {
        uint32_t es[T * T / 4];              // marked destination tile (row-major words)
        uint32_t ss[T * T / 4];              // keystream of the destination tile (tile-major)
        uint64_t rec[kRecSlots];             // angle record of the original tile
        uint32_t mbits[T][2], ebits[T][2];   // LMR: decoded map / eta bits of the destination rows
    } st[2];
    uint32_t xo[T * RS], lo[T * RS];         // original domain of the current tile
    uint32_t pyr[kPyrSmem];
    int dmap[kMaxTilesX];                    // per original tile of the strip: destination << 2 | q
    uint8_t carry[T];                        // per row: omega at the right edge of the previous tile
    uint32_t fsel[16];                       // copy-forward PRMT selectors by 4-bit map
    int sh[4];
};

template <int TP, int METHOD>
__device__ __forceinline__ void rec_role(const Geo &g, int img, int ty, int nK, const uint8_t *__restrict__ marked,
                                         const TileWS &ws, const uint32_t *__restrict__ eta_bits,
                                         const uint32_t *__restrict__ map_bits, const int32_t *__restrict__ lmr_b,
                                         uint8_t *__restrict__ out, int32_t *__restrict__ status, uint8_t *smem) {
    constexpr int T = 1 << TP, NW = T / 4, RS = T / 4 + 1, NC = T / 4, NCELL = NC * NC, CPT = T * T / 16;
    constexpr int SEGS = T / 16, NG = NC / 2;
    RecSmem<TP> &S = *reinterpret_cast<RecSmem<TP> *>(smem);
    const int tid = threadIdx.x;
    const uint8_t *Em = marked + (size_t)img * g.HW;
    uint8_t *O = out + (size_t)img * g.HW;

    if (tid >= 32 && tid < 48) {                        // fsel[m] nibble i: last set bit <= i, else 4
        const int m = tid - 32;
        uint32_t v = 0;
        int last = 4;
        for (int i = 0; i < 4; i++) {
            if ((m >> i) & 1) last = i;
            v |= (uint32_t)last << (4 * i);
        }
        S.fsel[m] = v;
    }
    if (tid < 32) {
        int b = 0;
        if (tid == 0) {
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
            const uint32_t *pyr = warp0_ready(g, ws, img, nK, S.pyr);
            for (int j = tid; j < g.tilesX; j += 32) {
                int dty, dtx, q;
                upper_walk_forward(g, pyr, ty, j, dty, dtx, q);
                S.dmap[j] = (((dty << g.tlog) + dtx) << 2) | q;
            }
        }
    }
    __syncthreads();
    const int b = S.sh[0];
    if (b <= 0) {                                       // FORMAT / BADCASE: zero-filled output
        for (int c = tid; c < T * g.W / 16; c += 256) {
            const int r = c / (g.W / 16), col = c % (g.W / 16);
            *reinterpret_cast<uint4 *>(O + (size_t)(ty * T + r) * g.W + col * 16) = make_uint4(0, 0, 0, 0);
        }
        return;
    }
    const uint32_t mask = METHOD == 0 ? ((0xFFu << (8 - b)) & 0xFFu) : (0x7Fu & ~(0xFFu >> b));
    const uint32_t maskb = mask * 0x01010101u;

    auto issue = [&](int j) {
        typename RecSmem<TP>::Stage &st = S.st[j & 1];
        const int dt = S.dmap[j] >> 2, dty = dt >> g.tlog, dtx = dt & (g.tilesX - 1);
        const size_t dslot = (size_t)img * g.ntiles + dt;
        for (int c = tid; c < CPT; c += 256) {
            const int r = c / (T / 16), seg = c % (T / 16);
            cp_async16(&st.es[r * NW + seg * 4], Em + (size_t)(dty * T + r) * g.W + (size_t)dtx * T + seg * 16);
            cp_async16(&st.ss[4 * c], ws.s + dslot * (T * T) + 16 * c);
        }
        if (tid < kRecSlots / 2)
            cp_async16(&st.rec[2 * tid],
                       ws.rec + ((size_t)img * g.ntiles + ((size_t)ty << g.tlog) + j) * kRecSlots + 2 * tid);
        if constexpr (METHOD == 1) {
            if (tid < T) {
                const size_t bit = (size_t)img * g.HW + (size_t)(dty * T + tid) * g.W + (size_t)dtx * T;
                if constexpr (T >= 32) {
                    for (int k = 0; k < T / 32; k++) {
                        cp_async4(&st.mbits[tid][k], map_bits + (bit >> 5) + k);
                        cp_async4(&st.ebits[tid][k], eta_bits + (bit >> 5) + k);
                    }
                } else {                                 // 16-pixel rows share words: plain loads
                    st.mbits[tid][0] = __ldg(map_bits + (bit >> 5)) >> (bit & 31);
                    st.ebits[tid][0] = __ldg(eta_bits + (bit >> 5)) >> (bit & 31);
                }
            }
        }
        cp_async_commit();
    };

    const bool rowthr = tid < T * SEGS;
    const int r = tid / SEGS, seg = tid % SEGS;
    issue(0);
    for (int j = 0; j < g.tilesX; j++) {
        if (j + 1 < g.tilesX) {
            issue(j + 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();                                           // stage j landed for everyone
        const typename RecSmem<TP>::Stage &st = S.st[j & 1];
        const int mp = S.dmap[j], dt = mp >> 2, q_up = mp & 3;
        // cells: original cell -> destination cell; X, L from the staged destination tile
        for (int c = tid; c < NCELL; c += 256) {
            const int gi = c >> 2, sub = c & 3;
            const int ogy = gi / NG, ogx = gi % NG;
            const int cy = 2 * ogy + (sub >> 1), cx = 2 * ogx + (sub & 1);
            const uint32_t ge = reinterpret_cast<const uint8_t *>(st.rec + kRecGroupSlot)[gi];
            int dgy = ge >> 5, dgx = (ge >> 2) & 7;          // in-tile levels >= 4 (group table),
            fwd_turn(q_up, NG - 1, dgy, dgx);                // then the tile's own turn
            int q = q_up + (int)(ge & 3);
            if (g.emin <= 3) q += rec_angle(st.rec, g, 3, ogy, ogx);   // level 3 = the group itself
            int sy = sub >> 1, sx = sub & 1;
            fwd_turn(q & 3, 1, sy, sx);
            const int py = 2 * dgy + sy, px = 2 * dgx + sx;
            if (g.emin <= 2) q += rec_angle(st.rec, g, 2, cy, cx);
            uint32_t xr[4], lr[4];
#pragma unroll
            for (int i = 0; i < 4; i++) {
                const int row = 4 * py + i;
                const uint32_t e = st.es[row * NW + px];
                uint32_t x = e ^ st.ss[row * NW + px];
                uint32_t l;
                if constexpr (METHOD == 0) {
                    l = e & 0x01010101u;
                    if (i == 0 && dt == 0 && py == 0 && px == 0) l |= 0x00010101u;   // header pixels, map 1
                } else {
                    const int bp = 4 * px;
                    l = bits4_to_bytes(st.mbits[row][bp >> 5] >> (bp & 31));
                    x = (x & 0x7F7F7F7Fu) | (bits4_to_bytes(st.ebits[row][bp >> 5] >> (bp & 31)) << 7);  // MSB <- eta
                }
                xr[i] = x;
                lr[i] = l;
            }
            Cell x = {xr[0], xr[1], xr[2], xr[3]};
            Cell l = {lr[0], lr[1], lr[2], lr[3]};
            const int rinv = (4 - (q & 3)) & 3;
            x = cell_rot_cw(x, rinv);
            l = cell_rot_cw(l, rinv);
            if (g.emin <= 1) {
                const uint32_t a01 = (uint32_t)(st.rec[g.lvl_off[1] + 2 * cy] >> (4 * cx)) & 0xFu;
                const uint32_t a23 = (uint32_t)(st.rec[g.lvl_off[1] + 2 * cy + 1] >> (4 * cx)) & 0xFu;
                const int aL0 = (4 - (a01 & 3)) & 3, aR0 = (4 - (a01 >> 2)) & 3;
                const int aL1 = (4 - (a23 & 3)) & 3, aR1 = (4 - (a23 >> 2)) & 3;
                pair_rot_cw(x.r0, x.r1, aL0, aR0);
                pair_rot_cw(x.r2, x.r3, aL1, aR1);
                pair_rot_cw(l.r0, l.r1, aL0, aR0);
                pair_rot_cw(l.r2, l.r3, aL1, aR1);
            }
            S.xo[(4 * cy) * RS + cx] = x.r0; S.xo[(4 * cy + 1) * RS + cx] = x.r1;
            S.xo[(4 * cy + 2) * RS + cx] = x.r2; S.xo[(4 * cy + 3) * RS + cx] = x.r3;
            S.lo[(4 * cy) * RS + cx] = l.r0; S.lo[(4 * cy + 1) * RS + cx] = l.r1;
            S.lo[(4 * cy + 2) * RS + cx] = l.r2; S.lo[(4 * cy + 3) * RS + cx] = l.r3;
        }
        __syncthreads();                                           // tile j in the original domain
        {   // the consumed scratch (destination keystream, original record) leaves L2 unwritten
            const size_t dslot = (size_t)img * g.ntiles + dt;
            if (tid < (T * T) / 128) discard_l2(ws.s + dslot * (T * T) + 128 * tid);
            else if (tid >= 64 && tid < 64 + kRecSlots * 8 / 128)
                discard_l2(ws.rec + ((size_t)img * g.ntiles + ((size_t)ty << g.tlog) + j) * kRecSlots + 16 * (tid - 64));
        }
        // ---- rows: SEGS threads per row, 16 pixels each.  Copy-forward 4 pixels at a time:
        // om = PRMT(x & mask, carry, fsel[m4]) gives every byte the masked value of the last
        // non-redundant pixel at or before it (or the carry); out = (x & ~mask) | om is exact for
        // both kinds of pixel (a non-redundant pixel takes its own bits).
        uint32_t xw[4] = {0, 0, 0, 0}, sel[4] = {0, 0, 0, 0};
        uint32_t m16 = 0;
        if (rowthr) {
#pragma unroll
            for (int i = 0; i < 4; i++) {
                xw[i] = S.xo[r * RS + seg * 4 + i];
                m16 |= bytes_to_bits4(S.lo[r * RS + seg * 4 + i]) << (4 * i);
            }
            if (j == 0 && seg == 0) m16 |= 1u;         // column 0: omega starts at its bits
        }
        uint32_t c4 = 0;                                // segment summary with a zero carry-in
#pragma unroll
        for (int i = 0; i < 4; i++) {
            sel[i] = S.fsel[(m16 >> (4 * i)) & 0xFu];
            c4 = __byte_perm(__byte_perm(xw[i] & maskb, c4, sel[i]), 0, 0x3333);
        }
        const int has = m16 != 0, val = (int)(c4 & 0xFFu);
        int ehas = 0, evl = 0;                          // last non-redundant before this segment
#pragma unroll
        for (int s2 = 0; s2 < SEGS - 1; s2++) {
            const int oh = __shfl_sync(0xffffffffu, has, s2, SEGS);
            const int ov = __shfl_sync(0xffffffffu, val, s2, SEGS);
            if (s2 < seg && oh) { ehas = 1; evl = ov; }
        }
        if (rowthr) {
            uint32_t cin = (ehas ? (uint32_t)evl : (uint32_t)S.carry[r]) * 0x01010101u;
#pragma unroll
            for (int i = 0; i < 4; i++) {
                const uint32_t om = __byte_perm(xw[i] & maskb, cin, sel[i]);
                xw[i] = (xw[i] & ~maskb) | om;
                cin = __byte_perm(om, 0, 0x3333);
            }
            *reinterpret_cast<uint4 *>(O + (size_t)(ty * T + r) * g.W + (size_t)j * T + seg * 16) =
                make_uint4(xw[0], xw[1], xw[2], xw[3]);
            if (seg == SEGS - 1) S.carry[r] = (uint8_t)cin;   // omega leaving the tile
        }
        __syncthreads();                                           // xo/lo, carry, stage j reusable
    }
}

// ======================================================================================
// The fused kernels
// ======================================================================================
template <int TP, int METHOD>
__global__ void __launch_bounds__(256, 6) encode_kernel(Geo g, FusedSched sc, const uint8_t *__restrict__ images,
                                                     const uint8_t *__restrict__ keys, TileWS ws,
                                                     uint8_t *__restrict__ enc, uint8_t *__restrict__ ceta,
                                                     int32_t *__restrict__ b_out, int64_t *__restrict__ cap_out,
                                                     int32_t *__restrict__ status) {
    constexpr int T = 1 << TP, TPC = 256 / T;
    constexpr size_t KB = (TPC + 1) * kRecSlots * 8, PB = sizeof(PermSmem<TP>);
    __shared__ __align__(128) uint8_t smem[KB > PB ? KB : PB];
    const Role ro = role_of(sc);
    if (ro.img >= g.B) return;
#ifdef MMSB_PROBE_ROLES   // performance probes only (tools/role_probe.py): 1 = keystream CTAs only, 2 = workers only
    if (!((MMSB_PROBE_ROLES >> (ro.key ? 0 : 1)) & 1)) return;
#endif
    if (ro.key) key_role<TP, true, true, METHOD == 1>(g, ro.img, ro.idx, keys, images, ws, smem);
    else perm_role<TP, METHOD>(g, ro.img, ro.idx, 1 << sc.lgK, images, ws, enc, ceta, b_out, cap_out, status, smem);
}

template <int TP, int METHOD>
__global__ void __launch_bounds__(256, 6) recover_kernel(Geo g, FusedSched sc, const uint8_t *__restrict__ marked,
                                                      const uint8_t *__restrict__ keys, TileWS ws,
                                                      const uint32_t *__restrict__ eta_bits,
                                                      const uint32_t *__restrict__ map_bits,
                                                      const int32_t *__restrict__ lmr_b, uint8_t *__restrict__ out,
                                                      int32_t *__restrict__ status) {
    constexpr int T = 1 << TP, TPC = 256 / T;
    constexpr size_t KB = (TPC + 1) * kRecSlots * 8, RB = sizeof(RecSmem<TP>);
    __shared__ __align__(128) uint8_t smem[KB > RB ? KB : RB];
    const Role ro = role_of(sc);
    if (ro.img >= g.B) return;
#ifdef MMSB_PROBE_ROLES
    if (!((MMSB_PROBE_ROLES >> (ro.key ? 0 : 1)) & 1)) return;
#endif
    if (ro.key) key_role<TP, false, false>(g, ro.img, ro.idx, keys, nullptr, ws, smem);
    else rec_role<TP, METHOD>(g, ro.img, ro.idx, 1 << sc.lgK, marked, ws, eta_bits, map_bits, lmr_b, out, status, smem);
}

// ---------------------------------------------------------------------------- launchers
FusedSched fused_sched(const Geo &g) {
    FusedSched sc;
    const int TPC = 256 / g.T;
    const int nK = g.ntiles >= TPC ? g.ntiles / TPC : 1;       // powers of two
    sc.lgK = ilog2(nK);
    sc.lgW = ilog2(g.tilesY);                           // one worker CTA per strip of tiles
    int gi = 1;
    while ((long long)(gi * 2) * g.HW <= (2ll << 20) && gi < g.B) gi *= 2;   // ~2 Mpixel per group
    sc.GI = gi;
    sc.ngroups = (g.B + gi - 1) / gi;
    // keystream rows run L rows ahead of their workers: enough to hide the keystream latency,
    // few enough that the scratch (1 B/px) and the re-read images of L groups stay in L2
    long long lag = (12ll << 20) / ((long long)gi * g.HW);
    sc.L = (int)(lag < 1 ? 1 : lag > 6 ? 6 : lag);
    return sc;
}

static dim3 fused_grid(const FusedSched &sc) {
    return dim3((unsigned)((sc.GI << sc.lgK) + (sc.GI << sc.lgW)), (unsigned)(sc.ngroups + sc.L));
}

template <int TP>
static void launch_encode_tp(const Geo &g, const uint8_t *images, const uint8_t *keys, const TileWS &ws, uint8_t *enc,
                             uint8_t *ceta, int32_t *b_out, int64_t *cap_out, int32_t *status, cudaStream_t st) {
    const FusedSched sc = fused_sched(g);
    const dim3 grid = fused_grid(sc);
    if (g.method == 0)
        encode_kernel<TP, 0><<<grid, 256, 0, st>>>(g, sc, images, keys, ws, enc, ceta, b_out, cap_out, status);
    else
        encode_kernel<TP, 1><<<grid, 256, 0, st>>>(g, sc, images, keys, ws, enc, ceta, b_out, cap_out, status);
}

void launch_encode(const Geo &g, const uint8_t *images, const uint8_t *keys, const TileWS &ws, uint8_t *enc,
                   uint8_t *ceta, int32_t *b_out, int64_t *cap_out, int32_t *status, cudaStream_t st) {
    switch (g.tp) {
        case 4: launch_encode_tp<4>(g, images, keys, ws, enc, ceta, b_out, cap_out, status, st); break;
        case 5: launch_encode_tp<5>(g, images, keys, ws, enc, ceta, b_out, cap_out, status, st); break;
        default: launch_encode_tp<6>(g, images, keys, ws, enc, ceta, b_out, cap_out, status, st); break;
    }
}

template <int TP>
static void launch_recover_tp(const Geo &g, const uint8_t *marked, const uint8_t *keys, const TileWS &ws,
                              const uint32_t *eta, const uint32_t *map, const int32_t *lmr_b, uint8_t *out,
                              int32_t *status, cudaStream_t st) {
    const FusedSched sc = fused_sched(g);
    const dim3 grid = fused_grid(sc);
    if (g.method == 0)
        recover_kernel<TP, 0><<<grid, 256, 0, st>>>(g, sc, marked, keys, ws, eta, map, lmr_b, out, status);
    else
        recover_kernel<TP, 1><<<grid, 256, 0, st>>>(g, sc, marked, keys, ws, eta, map, lmr_b, out, status);
}

void launch_recover(const Geo &g, const uint8_t *marked, const uint8_t *keys, const TileWS &ws, const uint32_t *eta,
                    const uint32_t *map, const int32_t *lmr_b, uint8_t *out, int32_t *status, cudaStream_t st) {
    switch (g.tp) {
        case 4: launch_recover_tp<4>(g, marked, keys, ws, eta, map, lmr_b, out, status, st); break;
        case 5: launch_recover_tp<5>(g, marked, keys, ws, eta, map, lmr_b, out, status, st); break;
        default: launch_recover_tp<6>(g, marked, keys, ws, eta, map, lmr_b, out, status, st); break;
    }
}

}  // namespace mmsb
