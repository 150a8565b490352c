// k_tile.cu -- tile kernels of the hot path (sm_100a):
//   ks_tile_kernel        K1 keystream (ChaCha20) -> L2 scratch, per-tile angle records
//                         (levels 1..tp), upper-pyramid block sums, and (encode) the
//                         per-image label histogram                                (a1, a4)
//   perm_encode_kernel    labels -> location map -> rotate -> encrypt -> LSB map embed (a3, a5)
//   recover_strip_kernel  decrypt -> de-rotate -> row copy-forward                  (a10)
// Citations: P:<line> = /root/reference/PAPER.md.  Design: DESIGN.md §5.
#include "mmsb_device.cuh"
#include "mmsb_kernels.h"

namespace mmsb {

// ======================================================================================
// ks_tile_kernel: one thread per tile row, 256 / T tiles per CTA.
//   s(i, j) = byte (i W + j) of ChaCha20(K1) (Q12), written to the group scratch;
//   angle(e, block) = (sum of s over the block) mod 4 (eq. roration) for e = 1..tp,
//   kept as 2-bit fields, one u64 per block row (record of kRecSlots u64 per tile);
//   block sums above the tile level are accumulated with atomics (counters mod 4 on read).
//   HIST: non-redundant counts per b = 2..8 of the label c = #leading equal bits of p and
//   its left neighbour (eq. gliding1/2 P:611-625 reduce to the left neighbour).
// ======================================================================================
// destination tile -> source tile under the levels above the tile (walk e = emax .. tp+1)
__device__ __forceinline__ void upper_walk_inverse(const Geo &g, const uint32_t *pyr_img, int dty, int dtx,
                                                   int &sty, int &stx, int &q) {
    int y = dty, x = dtx;
    q = 0;
    for (int e = g.emax; e > g.tp; e--) {
        const int k = e - g.tp, m1 = (1 << k) - 1;
        const int by = y >> k, bx = x >> k;
        const int a = (int)(__ldcg(pyr_img + g.pyr_off[e] + by * (g.W >> e) + bx) & 3u);
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
        const int a = (int)(__ldcg(pyr_img + g.pyr_off[e] + by * (g.W >> e) + bx) & 3u);
        int oy = y & m1, ox = x & m1;
        fwd_turn(a, m1, oy, ox);
        y = (by << k) | oy;
        x = (bx << k) | ox;
        q += a;
    }
    dty = y; dtx = x; q &= 3;
}

template <int TP, bool HIST>
__global__ void __launch_bounds__(256) ks_tile_kernel(Geo g, const uint8_t *__restrict__ keys,
                                                      const uint8_t *__restrict__ images,
                                                      uint8_t *__restrict__ s_out, uint64_t *__restrict__ rec_out,
                                                      uint32_t *__restrict__ pyr, uint32_t *__restrict__ hist,
                                                      uint32_t *__restrict__ done, int32_t *__restrict__ fwd_map,
                                                      int32_t *__restrict__ inv_map) {
    constexpr int T = 1 << TP, NW = T / 4, TPC = 256 / T;
    __shared__ __align__(16) uint32_t sbuf[TPC][T][NW];
    __shared__ uint64_t rec[TPC][kRecSlots];

    const int tid = threadIdx.x, lt = tid / T, row = tid % T;
    const int img = blockIdx.y;
    const int tile = blockIdx.x * TPC + lt;
    const bool valid = tile < g.ntiles;
    const int ty = valid ? tile / g.tilesX : 0, tx = valid ? tile % g.tilesX : 0;
    const long long o = (long long)(ty * T + row) * g.W + (long long)tx * T;

    uint32_t key[8];
    load_key(keys, img, key);
    uint32_t blk[16];
    chacha20_block(key, (uint32_t)(o >> 6), blk);
    uint32_t w[NW];
    if constexpr (NW == 16) {
#pragma unroll
        for (int i = 0; i < 16; i++) w[i] = blk[i];
    } else {
        const int boff = (int)((o & 63) >> 2);
#pragma unroll
        for (int i = 0; i < NW; i++) w[i] = blk[boff + i];
    }
#pragma unroll
    for (int i = 0; i < NW; i += 4)
        *reinterpret_cast<uint4 *>(&sbuf[lt][row][i]) = make_uint4(w[i], w[i + 1], w[i + 2], w[i + 3]);

    // level 1: 2x2 block sums mod 4 -- horizontal pair sums per row, then the partner row
    uint64_t h1 = 0;
#pragma unroll
    for (int i = 0; i < NW; i++) {
        uint32_t v = w[i] & 0x03030303u;
        uint32_t p = (v + (v >> 8)) & 0x00030003u;
        uint32_t q = (p & 3u) | ((p >> 14) & 0xCu);
        h1 |= (uint64_t)q << (4 * i);
    }
    uint64_t partner = __shfl_xor_sync(0xffffffffu, h1, 1);
    if (valid && (row & 1) == 0) rec[lt][g.lvl_off[1] + row / 2] = add2(h1, partner);

    if constexpr (HIST) {
        // label histogram over this tile row (non-redundant counts for b = 2..8)
        const uint8_t *src = images + (size_t)img * g.HW + o;
        uint32_t iw[NW];
#pragma unroll
        for (int i = 0; i < NW; i += 4) {
            uint4 u = valid ? __ldg(reinterpret_cast<const uint4 *>(src) + i / 4) : make_uint4(0, 0, 0, 0);
            iw[i] = u.x; iw[i + 1] = u.y; iw[i + 2] = u.z; iw[i + 3] = u.w;
        }
        uint32_t prev = (valid && tx > 0) ? ((uint32_t)__ldg(src - 1) << 24) : 0u;
        uint32_t nr[7] = {0, 0, 0, 0, 0, 0, 0};
#pragma unroll
        for (int i = 0; i < NW; i++) {
            uint32_t left = __byte_perm(prev, iw[i], 0x6543);   // [prev.b3, w.b0, w.b1, w.b2]
            uint32_t x = iw[i] ^ left;
            if (i == 0 && tx == 0) x |= 0xFFu;                   // column 0 is non-redundant
            prev = iw[i];
            uint32_t y = x | ((x >> 1) & 0x7F7F7F7Fu);
            y |= (y >> 2) & 0x3F3F3F3Fu;
            y |= (y >> 4) & 0x0F0F0F0Fu;                         // byte = 2^bitlen(x) - 1
#pragma unroll
            for (int b = 2; b <= 8; b++) nr[b - 2] += __popc(y & (0x01010101u << (8 - b)));
        }
        if (!valid) {
#pragma unroll
            for (int k = 0; k < 7; k++) nr[k] = 0;
        }
#pragma unroll
        for (int k = 0; k < 7; k++) {
            uint32_t v = nr[k];
#pragma unroll
            for (int s = 16; s > 0; s >>= 1) v += __shfl_xor_sync(0xffffffffu, v, s);
            if ((tid & 31) == 0 && v) atomicAdd(&hist[img * 8 + k + 2], v);
        }
    }
    __syncthreads();

    // levels 2..tp: quad-tree sums mod 4 of the level below
#pragma unroll
    for (int e = 2; e <= TP; e++) {
        const int R = T >> e;
        for (int t = tid; t < TPC * R; t += 256) {
            const int l2 = t / R, r = t % R;
            uint64_t v = add2(rec[l2][g.lvl_off[e - 1] + 2 * r], rec[l2][g.lvl_off[e - 1] + 2 * r + 1]);
            uint64_t pe = v & 0x3333333333333333ull, po = (v >> 2) & 0x3333333333333333ull;
            uint64_t s = (pe + po) & 0x3333333333333333ull;
            s = (s | (s >> 2)) & 0x0F0F0F0F0F0F0F0Full;
            s = (s | (s >> 4)) & 0x00FF00FF00FF00FFull;
            s = (s | (s >> 8)) & 0x0000FFFF0000FFFFull;
            s = (s | (s >> 16)) & 0x00000000FFFFFFFFull;
            rec[l2][g.lvl_off[e] + r] = s;
        }
        __syncthreads();
    }

    // upper pyramid: the tile total (= level-tp angle) into every enclosing block
    if (valid && row == 0) {
        const uint32_t tv = (uint32_t)(rec[lt][g.lvl_off[TP]] & 3u);
        if (tv)
            for (int e = TP + 1; e <= g.emax; e++) {
                const int k = e - TP;
                atomicAdd(&pyr[(size_t)img * g.npyr + g.pyr_off[e] + (ty >> k) * (g.W >> e) + (tx >> k)], tv);
            }
    }
    // records out (one u64 per thread per pass)
    for (int t = tid; t < TPC * kRecSlots; t += 256) {
        const int l2 = t / kRecSlots, slot = t % kRecSlots;
        const int tl = blockIdx.x * TPC + l2;
        if (tl < g.ntiles) rec_out[((size_t)img * g.ntiles + tl) * kRecSlots + slot] = rec[l2][slot];
    }
    // keystream out, coalesced 16-byte chunks
    constexpr int CPT = T * T / 16;                 // 16-byte chunks per tile
    for (int c = tid; c < TPC * CPT; c += 256) {
        const int l2 = c / CPT, cc = c % CPT, r = cc / (T / 16), seg = cc % (T / 16);
        const int tl = blockIdx.x * TPC + l2;
        if (tl >= g.ntiles) continue;
        const int tyy = tl / g.tilesX, txx = tl % g.tilesX;
        uint4 v = *reinterpret_cast<const uint4 *>(&sbuf[l2][r][seg * 4]);
        *reinterpret_cast<uint4 *>(s_out + (size_t)img * g.HW + (size_t)(tyy * T + r) * g.W + txx * T + seg * 16) = v;
    }
    // the image's last CTA turns the completed upper pyramid into tile maps (one walk per tile):
    //   inv_map[dest tile] = source tile << 2 | q,  fwd_map[original tile] = dest tile << 2 | q
    __shared__ int last;
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        last = atomicAdd(done + img, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    const uint32_t *pyr_img = pyr + (size_t)img * g.npyr;
    for (int t = tid; t < g.ntiles; t += 256) {
        const int ty2 = t / g.tilesX, tx2 = t % g.tilesX;
        int y, x, q;
        upper_walk_inverse(g, pyr_img, ty2, tx2, y, x, q);
        inv_map[(size_t)img * g.ntiles + t] = ((y * g.tilesX + x) << 2) | q;
        upper_walk_forward(g, pyr_img, ty2, tx2, y, x, q);
        fwd_map[(size_t)img * g.ntiles + t] = ((y * g.tilesX + x) << 2) | q;
    }
}

// EMR optimal b from the non-redundant counts (eq. optimial_b; ties -> smaller b)
__device__ __forceinline__ int emr_select_b(const uint32_t *hist_img, long long HW) {
    int best = 2;
    long long bestv = 2 * (HW - (long long)hist_img[2]);
    for (int b = 3; b <= 7; b++) {
        long long v = (long long)b * (HW - (long long)hist_img[b]);
        if (v > bestv) { best = b; bestv = v; }
    }
    return best;
}

// ======================================================================================
// perm_encode_kernel: one CTA per destination tile.
//   EMR: carrier v = (I & 0xFE) | l with l = [c < b] (location map), permuted as a
//        whole byte; E = v_r XOR (s & 0xFE) (eq. image_encryption P:739 + LSB map P:744);
//        header b-2 in the LSBs of r = 0..2 (Q14).
//   LMR: E = I_r XOR s; second plane ceta = (I & 0x80) | c permuted alongside (for the coder).
// ======================================================================================
template <int TP, int METHOD>
__global__ void __launch_bounds__(256) perm_encode_kernel(Geo g, const uint8_t *__restrict__ images,
                                                          const uint8_t *__restrict__ s_scr,
                                                          const uint64_t *__restrict__ recs,
                                                          const uint32_t *__restrict__ pyr,
                                                          const uint32_t *__restrict__ hist,
                                                          const int32_t *__restrict__ inv_map,
                                                          uint8_t *__restrict__ enc, uint8_t *__restrict__ ceta_out,
                                                          int32_t *__restrict__ b_out, int64_t *__restrict__ cap_out,
                                                          int32_t *__restrict__ status) {
    constexpr int T = 1 << TP, NW = T / 4, RS = NW + 1, NC = T / 4, NCELL = NC * NC, CPT = T * T / 16;
    __shared__ uint32_t src[T * RS];
    __shared__ uint32_t lab[METHOD == 1 ? T * RS : 1];
    __shared__ uint64_t rec[kRecSlots];
    __shared__ int sh[1];

    const int tid = threadIdx.x, img = blockIdx.y;
    const int dty = blockIdx.x / g.tilesX, dtx = blockIdx.x % g.tilesX;
    const uint8_t *I = images + (size_t)img * g.HW;

    const int mp = __ldg(inv_map + (size_t)img * g.ntiles + blockIdx.x);
    const int stile = mp >> 2, q_up = mp & 3;
    const int sty = stile / g.tilesX, stx = stile % g.tilesX;
    if (tid == 0) sh[0] = METHOD == 0 ? emr_select_b(hist + img * 8, g.HW) : 0;
    if (tid < kRecSlots) rec[tid] = recs[((size_t)img * g.ntiles + stile) * kRecSlots + tid];
    __syncthreads();
    const int b = sh[0];
    (void)pyr;

    // source tile + left halo -> labels -> carrier (EMR) or I and ceta (LMR)
    const uint32_t M = METHOD == 0 ? (0xFFu << (8 - b)) & 0xFFu : 0;
    const uint32_t MB = M * 0x01010101u;
    for (int c = tid; c < CPT; c += 256) {
        const int r = c / (T / 16), seg = c % (T / 16);
        const long long gx = (long long)stx * T + seg * 16;
        const uint8_t *p = I + (size_t)(sty * T + r) * g.W + gx;
        uint4 u = __ldg(reinterpret_cast<const uint4 *>(p));
        uint32_t iw[4] = {u.x, u.y, u.z, u.w};
        uint32_t prev = gx > 0 ? ((uint32_t)__ldg(p - 1) << 24) : 0u;
        uint32_t vw[4], cw[4];
#pragma unroll
        for (int i = 0; i < 4; i++) {
            uint32_t x = iw[i] ^ __byte_perm(prev, iw[i], 0x6543);
            if (i == 0 && gx == 0) x |= 0xFFu;                     // column 0: always non-redundant
            prev = iw[i];
            if constexpr (METHOD == 0) {
                uint32_t t = x & MB;
                uint32_t nz = (((t & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | t) & 0x80808080u;   // byte != 0
                vw[i] = (iw[i] & 0xFEFEFEFEu) | (nz >> 7);
            } else {
                // c = #leading equal bits (8 if equal), per byte; column 0 -> 0
                uint32_t cv = 0;
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    uint32_t xb = (x >> (8 * j)) & 0xFFu;
                    uint32_t cj = xb ? (uint32_t)(__clz(xb) - 24) : 8u;
                    cv |= cj << (8 * j);
                }
                cw[i] = cv | (iw[i] & 0x80808080u);
                vw[i] = iw[i];
            }
        }
#pragma unroll
        for (int i = 0; i < 4; i++) {
            src[r * RS + seg * 4 + i] = vw[i];
            if constexpr (METHOD == 1) lab[r * RS + seg * 4 + i] = cw[i];
        }
    }
    __syncthreads();

    // cells: destination cell -> source cell (levels 3..tp), then in-cell levels 1, 2
    const uint8_t *S = s_scr + (size_t)img * g.HW;
    for (int c = tid; c < NCELL; c += 256) {
        const int cy = c / NC, cx = c % NC;
        int py = cy, px = cx;
        inv_turn(q_up, NC - 1, py, px);
        int q = q_up;
        for (int e = TP; e >= 3 && e >= g.emin; e--) {
            const int k = e - 2, m1 = (1 << k) - 1;
            const int by = py >> k, bx = px >> k;
            const int a = rec_angle(rec, g, e, by, bx);
            int oy = py & m1, ox = px & m1;
            inv_turn(a, m1, oy, ox);
            py = (by << k) | oy;
            px = (bx << k) | ox;
            q += a;
        }
        Cell v = {src[(4 * py) * RS + px], src[(4 * py + 1) * RS + px], src[(4 * py + 2) * RS + px],
                  src[(4 * py + 3) * RS + px]};
        Cell cl;
        if constexpr (METHOD == 1)
            cl = {lab[(4 * py) * RS + px], lab[(4 * py + 1) * RS + px], lab[(4 * py + 2) * RS + px],
                  lab[(4 * py + 3) * RS + px]};
        if (g.emin <= 1) {
            const uint32_t a01 = (uint32_t)(rec[g.lvl_off[1] + 2 * py] >> (4 * px)) & 0xFu;
            const uint32_t a23 = (uint32_t)(rec[g.lvl_off[1] + 2 * py + 1] >> (4 * px)) & 0xFu;
            pair_rot_cw(v.r0, v.r1, a01 & 3, a01 >> 2);
            pair_rot_cw(v.r2, v.r3, a23 & 3, a23 >> 2);
            if constexpr (METHOD == 1) {
                pair_rot_cw(cl.r0, cl.r1, a01 & 3, a01 >> 2);
                pair_rot_cw(cl.r2, cl.r3, a23 & 3, a23 >> 2);
            }
        }
        if (g.emin <= 2) q += rec_angle(rec, g, 2, py, px);
        v = cell_rot_cw(v, q & 3);
        if constexpr (METHOD == 1) cl = cell_rot_cw(cl, q & 3);

        const size_t base = (size_t)(dty * T + 4 * cy) * g.W + (size_t)dtx * T + 4 * cx;
        const uint32_t s0 = __ldg(reinterpret_cast<const uint32_t *>(S + base));
        const uint32_t s1 = __ldg(reinterpret_cast<const uint32_t *>(S + base + g.W));
        const uint32_t s2 = __ldg(reinterpret_cast<const uint32_t *>(S + base + 2 * (size_t)g.W));
        const uint32_t s3 = __ldg(reinterpret_cast<const uint32_t *>(S + base + 3 * (size_t)g.W));
        uint32_t e0, e1, e2, e3;
        if constexpr (METHOD == 0) {
            e0 = v.r0 ^ (s0 & 0xFEFEFEFEu); e1 = v.r1 ^ (s1 & 0xFEFEFEFEu);
            e2 = v.r2 ^ (s2 & 0xFEFEFEFEu); e3 = v.r3 ^ (s3 & 0xFEFEFEFEu);
            if (blockIdx.x == 0 && c == 0) {
                // header: LSB(E[r]) = bit (2 - r) of b - 2 for r = 0..2; the map there is forced
                // to 1, so capacity counts zeros after forcing (Q14)
                const uint32_t m = v.r0 & 0x00010101u;
                const int forced = (int)(m & 1u) + (int)((m >> 8) & 1u) + (int)((m >> 16) & 1u);
                const uint32_t hb = (uint32_t)(b - 2);
                const uint32_t hdr = ((hb >> 2) & 1u) | (((hb >> 1) & 1u) << 8) | ((hb & 1u) << 16);
                e0 = (e0 & 0xFFFEFEFEu) | hdr;
                const long long zeros = g.HW - (long long)hist[img * 8 + b];
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
}

// expand 4 bits to 4 bytes of 0/1
__device__ __forceinline__ uint32_t bits4_to_bytes(uint32_t m4) { return ((m4 & 0xFu) * 0x00204081u) & 0x01010101u; }
// compress 4 bytes of 0/1 into 4 bits
__device__ __forceinline__ uint32_t bytes_to_bits4(uint32_t l) { return (l | (l >> 7) | (l >> 14) | (l >> 21)) & 0xFu; }

// ======================================================================================
// recover_strip_kernel: one CTA per strip of T original-domain rows; walks the strip's tiles
// left to right carrying omega per row (the copy-forward of P:837 / P:1061 is per row).
//   X = I_e' XOR s (every bit, Q20); EMR: map bit = raw LSB of I_e' (r < 3 forced to 1);
//   LMR: MSB := eta_r and the map come from the decoded planes.  Inverse cell transform,
//   then omega := masked bits of the last non-redundant pixel, replaced into redundant ones.
//   The next destination tile (I_e', s, angle record) is prefetched with cp.async while the
//   current one is processed (double buffer).
// ======================================================================================
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int TP, int METHOD>
__global__ void __launch_bounds__(256) recover_strip_kernel(Geo g, const uint8_t *__restrict__ marked,
                                                            const uint8_t *__restrict__ s_scr,
                                                            const uint64_t *__restrict__ recs,
                                                            const int32_t *__restrict__ fwd_map,
                                                            const uint32_t *__restrict__ eta_bits,
                                                            const uint32_t *__restrict__ map_bits,
                                                            const int32_t *__restrict__ lmr_b,
                                                            uint8_t *__restrict__ out, int32_t *__restrict__ status) {
    constexpr int T = 1 << TP, NW = T / 4, RS = NW + 1, NC = T / 4, NCELL = NC * NC, CPT = T * T / 16;
    constexpr int SEGS = T / 16;                      // 16-pixel segments per row
    __shared__ __align__(16) uint8_t eraw[2][T * T];
    __shared__ __align__(16) uint8_t sraw[2][T * T];
    __shared__ __align__(16) uint64_t rec[2][kRecSlots];
    __shared__ uint32_t xin[T * RS], lin[T * RS], xo[T * RS], lo[T * RS];
    __shared__ uint8_t carry[T];
    __shared__ int sh_b;

    const int tid = threadIdx.x, img = blockIdx.y, ty = blockIdx.x;
    const uint8_t *Em = marked + (size_t)img * g.HW;
    const uint8_t *S = s_scr + (size_t)img * g.HW;
    const int32_t *fm = fwd_map + (size_t)img * g.ntiles + (size_t)ty * g.tilesX;
    uint8_t *O = out + (size_t)img * g.HW;

    auto prefetch = [&](int tx, int buf) {
        const int mp = __ldg(fm + tx), dt = mp >> 2;
        const int dty = dt / g.tilesX, dtx = dt % g.tilesX;
        for (int c = tid; c < CPT; c += 256) {
            const int r = c / (T / 16), seg = c % (T / 16);
            const size_t off = (size_t)(dty * T + r) * g.W + (size_t)dtx * T + seg * 16;
            cp_async16(&eraw[buf][r * T + seg * 16], Em + off);
            cp_async16(&sraw[buf][r * T + seg * 16], S + off);
        }
        if (tid < kRecSlots / 2)
            cp_async16(&rec[buf][2 * tid], recs + ((size_t)img * g.ntiles + (size_t)ty * g.tilesX + tx) * kRecSlots + 2 * tid);
        cp_async_commit();
    };

    prefetch(0, 0);
    if (tid == 0) {
        int b;
        if constexpr (METHOD == 0) {
            const int field = ((Em[0] & 1) << 2) | ((Em[1] & 1) << 1) | (Em[2] & 1);
            b = field > 5 ? -1 : field + 2;
            if (ty == 0) status[img] = b < 0 ? 8 : 0;
        } else {
            b = lmr_b[img];                             // <= 0: status already set by the decoder
            if (ty == 0 && b > 0) status[img] = 0;
        }
        sh_b = b;
    }
    __syncthreads();
    const int b = sh_b;
    if (b <= 0) {
        cp_async_wait<0>();
        for (int c = tid; c < T * g.W / 16; c += 256) {
            const int r = c / (g.W / 16), col = c % (g.W / 16);
            *reinterpret_cast<uint4 *>(O + (size_t)(ty * T + r) * g.W + col * 16) = make_uint4(0, 0, 0, 0);
        }
        return;
    }
    const uint32_t mask = METHOD == 0 ? ((0xFFu << (8 - b)) & 0xFFu) : (0x7Fu & ~(0xFFu >> b));

    for (int tx = 0; tx < g.tilesX; tx++) {
        const int buf = tx & 1;
        if (tx + 1 < g.tilesX) {
            prefetch(tx + 1, buf ^ 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const int mp = __ldg(fm + tx), dt = mp >> 2, q_up = mp & 3;
        const int dty = dt / g.tilesX, dtx = dt % g.tilesX;
        // destination tile: X = E' ^ s, map bits
        for (int c = tid; c < CPT; c += 256) {
            const int r = c / (T / 16), seg = c % (T / 16);
            const uint4 e = *reinterpret_cast<const uint4 *>(&eraw[buf][r * T + seg * 16]);
            const uint4 sv = *reinterpret_cast<const uint4 *>(&sraw[buf][r * T + seg * 16]);
            uint32_t ew[4] = {e.x, e.y, e.z, e.w}, sw[4] = {sv.x, sv.y, sv.z, sv.w};
            uint32_t mb16 = 0, eb16 = 0;
            if constexpr (METHOD == 1) {
                const size_t bit = (size_t)img * g.HW + (size_t)(dty * T + r) * g.W + (size_t)dtx * T + seg * 16;
                mb16 = (__ldg(map_bits + (bit >> 5)) >> (bit & 31)) & 0xFFFFu;
                eb16 = (__ldg(eta_bits + (bit >> 5)) >> (bit & 31)) & 0xFFFFu;
            }
            const bool first = dt == 0 && r == 0 && seg == 0;
#pragma unroll
            for (int i = 0; i < 4; i++) {
                uint32_t x = ew[i] ^ sw[i], l;
                if constexpr (METHOD == 0) {
                    l = ew[i] & 0x01010101u;
                    if (i == 0 && first) l |= 0x00010101u;      // r = 0..2 carry the header, map = 1
                } else {
                    l = bits4_to_bytes(mb16 >> (4 * i));
                    x = (x & 0x7F7F7F7Fu) | (bits4_to_bytes(eb16 >> (4 * i)) << 7);   // MSB from eta
                }
                xin[r * RS + seg * 4 + i] = x;
                lin[r * RS + seg * 4 + i] = l;
            }
        }
        __syncthreads();
        const uint64_t *rc = rec[buf];
        // cells: original cell -> destination cell, inverse content transform
        for (int c = tid; c < NCELL; c += 256) {
            const int cy = c / NC, cx = c % NC;
            int py = cy, px = cx, q = 0;
            for (int e = (g.emin > 3 ? g.emin : 3); e <= TP; e++) {
                const int k = e - 2, m1 = (1 << k) - 1;
                const int by = py >> k, bx = px >> k;
                const int a = rec_angle(rc, g, e, by, bx);
                int oy = py & m1, ox = px & m1;
                fwd_turn(a, m1, oy, ox);
                py = (by << k) | oy;
                px = (bx << k) | ox;
                q += a;
            }
            fwd_turn(q_up, NC - 1, py, px);
            q += q_up;
            if (g.emin <= 2) q += rec_angle(rc, g, 2, cy, cx);
            Cell x = {xin[(4 * py) * RS + px], xin[(4 * py + 1) * RS + px], xin[(4 * py + 2) * RS + px],
                      xin[(4 * py + 3) * RS + px]};
            Cell l = {lin[(4 * py) * RS + px], lin[(4 * py + 1) * RS + px], lin[(4 * py + 2) * RS + px],
                      lin[(4 * py + 3) * RS + px]};
            const int rinv = (4 - (q & 3)) & 3;
            x = cell_rot_cw(x, rinv);
            l = cell_rot_cw(l, rinv);
            if (g.emin <= 1) {
                const uint32_t a01 = (uint32_t)(rc[g.lvl_off[1] + 2 * cy] >> (4 * cx)) & 0xFu;
                const uint32_t a23 = (uint32_t)(rc[g.lvl_off[1] + 2 * cy + 1] >> (4 * cx)) & 0xFu;
                const int aL0 = (4 - (a01 & 3)) & 3, aR0 = (4 - (a01 >> 2)) & 3;
                const int aL1 = (4 - (a23 & 3)) & 3, aR1 = (4 - (a23 >> 2)) & 3;
                pair_rot_cw(x.r0, x.r1, aL0, aR0);
                pair_rot_cw(x.r2, x.r3, aL1, aR1);
                pair_rot_cw(l.r0, l.r1, aL0, aR0);
                pair_rot_cw(l.r2, l.r3, aL1, aR1);
            }
            xo[(4 * cy) * RS + cx] = x.r0; xo[(4 * cy + 1) * RS + cx] = x.r1;
            xo[(4 * cy + 2) * RS + cx] = x.r2; xo[(4 * cy + 3) * RS + cx] = x.r3;
            lo[(4 * cy) * RS + cx] = l.r0; lo[(4 * cy + 1) * RS + cx] = l.r1;
            lo[(4 * cy + 2) * RS + cx] = l.r2; lo[(4 * cy + 3) * RS + cx] = l.r3;
        }
        __syncthreads();
        // row copy-forward: SEGS threads per row, 16 pixels each
        if (tid < T * SEGS) {
            const int r = tid / SEGS, seg = tid % SEGS;
            uint32_t xw[4], lw[4];
#pragma unroll
            for (int i = 0; i < 4; i++) { xw[i] = xo[r * RS + seg * 4 + i]; lw[i] = lo[r * RS + seg * 4 + i]; }
            if (tx == 0 && seg == 0) lw[0] |= 1u;           // column 0: omega starts at its bits
            uint32_t m16 = 0;
#pragma unroll
            for (int i = 0; i < 4; i++) m16 |= bytes_to_bits4(lw[i]) << (4 * i);
            int has = m16 != 0, val = 0;
            if (has) {
                const int li = 31 - __clz(m16);
                val = (int)((xw[li >> 2] >> (8 * (li & 3))) & mask);
            }
            // exclusive "last non-redundant" across the row's segments, seeded by the carry
            int inc = (tx == 0) ? 0 : carry[r];
            const unsigned gm = SEGS >= 32 ? 0xffffffffu : (((1u << SEGS) - 1u) << ((tid & 31) & ~(SEGS - 1)));
            for (int s2 = 0; s2 < SEGS - 1; s2++) {
                const int oh = __shfl_sync(gm, has, (tid & 31 & ~(SEGS - 1)) + s2, 32);
                const int ov = __shfl_sync(gm, val, (tid & 31 & ~(SEGS - 1)) + s2, 32);
                if (s2 < seg && oh) inc = ov;
            }
            uint32_t om = (uint32_t)inc;
#pragma unroll
            for (int i = 0; i < 16; i++) {
                const int wi = i >> 2, sh8 = 8 * (i & 3);
                const uint32_t px8 = (xw[wi] >> sh8) & 0xFFu;
                if ((lw[wi] >> sh8) & 1u) om = px8 & mask;
                else xw[wi] = (xw[wi] & ~(0xFFu << sh8)) | (((px8 & ~mask) | om) << sh8);
            }
            *reinterpret_cast<uint4 *>(O + (size_t)(ty * T + r) * g.W + (size_t)tx * T + seg * 16) =
                make_uint4(xw[0], xw[1], xw[2], xw[3]);
            // every lane of the row read carry[r] before the shuffles above synchronised it
            if (seg == SEGS - 1) carry[r] = (uint8_t)om;
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------- launchers
template <int TP>
static void launch_ks_tp(const Geo &g, int G, const uint8_t *keys, const uint8_t *images, uint8_t *s, uint64_t *rec,
                         uint32_t *pyr, uint32_t *hist, uint32_t *done, int32_t *fwd, int32_t *inv, cudaStream_t st) {
    constexpr int T = 1 << TP, TPC = 256 / T;
    dim3 grid((g.ntiles + TPC - 1) / TPC, G);
    if (images) ks_tile_kernel<TP, true><<<grid, 256, 0, st>>>(g, keys, images, s, rec, pyr, hist, done, fwd, inv);
    else ks_tile_kernel<TP, false><<<grid, 256, 0, st>>>(g, keys, images, s, rec, pyr, hist, done, fwd, inv);
}

void launch_ks_tile(const Geo &g, int G, const uint8_t *keys, const uint8_t *images, uint8_t *s, uint64_t *rec,
                    uint32_t *pyr, uint32_t *hist, uint32_t *done, int32_t *fwd, int32_t *inv, cudaStream_t st) {
    switch (g.tp) {
        case 4: launch_ks_tp<4>(g, G, keys, images, s, rec, pyr, hist, done, fwd, inv, st); break;
        case 5: launch_ks_tp<5>(g, G, keys, images, s, rec, pyr, hist, done, fwd, inv, st); break;
        default: launch_ks_tp<6>(g, G, keys, images, s, rec, pyr, hist, done, fwd, inv, st); break;
    }
}

template <int TP>
static void launch_perm_tp(const Geo &g, int G, const uint8_t *images, const uint8_t *s, const uint64_t *rec,
                           const uint32_t *pyr, const uint32_t *hist, const int32_t *inv, uint8_t *enc, uint8_t *ceta,
                           int32_t *b_out, int64_t *cap_out, int32_t *status, cudaStream_t st) {
    dim3 grid(g.ntiles, G);
    if (g.method == 0)
        perm_encode_kernel<TP, 0><<<grid, 256, 0, st>>>(g, images, s, rec, pyr, hist, inv, enc, ceta, b_out, cap_out, status);
    else
        perm_encode_kernel<TP, 1><<<grid, 256, 0, st>>>(g, images, s, rec, pyr, hist, inv, enc, ceta, b_out, cap_out, status);
}

void launch_perm_encode(const Geo &g, int G, const uint8_t *images, const uint8_t *s, const uint64_t *rec,
                        const uint32_t *pyr, const uint32_t *hist, const int32_t *inv, uint8_t *enc, uint8_t *ceta,
                        int32_t *b_out, int64_t *cap_out, int32_t *status, cudaStream_t st) {
    switch (g.tp) {
        case 4: launch_perm_tp<4>(g, G, images, s, rec, pyr, hist, inv, enc, ceta, b_out, cap_out, status, st); break;
        case 5: launch_perm_tp<5>(g, G, images, s, rec, pyr, hist, inv, enc, ceta, b_out, cap_out, status, st); break;
        default: launch_perm_tp<6>(g, G, images, s, rec, pyr, hist, inv, enc, ceta, b_out, cap_out, status, st); break;
    }
}

template <int TP>
static void launch_rec_tp(const Geo &g, int G, const uint8_t *marked, const uint8_t *s, const uint64_t *rec,
                          const int32_t *fwd, const uint32_t *eta, const uint32_t *map, const int32_t *lmr_b,
                          uint8_t *out, int32_t *status, cudaStream_t st) {
    dim3 grid(g.tilesY, G);
    if (g.method == 0)
        recover_strip_kernel<TP, 0><<<grid, 256, 0, st>>>(g, marked, s, rec, fwd, eta, map, lmr_b, out, status);
    else
        recover_strip_kernel<TP, 1><<<grid, 256, 0, st>>>(g, marked, s, rec, fwd, eta, map, lmr_b, out, status);
}

void launch_recover_strip(const Geo &g, int G, const uint8_t *marked, const uint8_t *s, const uint64_t *rec,
                          const int32_t *fwd, const uint32_t *eta, const uint32_t *map, const int32_t *lmr_b,
                          uint8_t *out, int32_t *status, cudaStream_t st) {
    switch (g.tp) {
        case 4: launch_rec_tp<4>(g, G, marked, s, rec, fwd, eta, map, lmr_b, out, status, st); break;
        case 5: launch_rec_tp<5>(g, G, marked, s, rec, fwd, eta, map, lmr_b, out, status, st); break;
        default: launch_rec_tp<6>(g, G, marked, s, rec, fwd, eta, map, lmr_b, out, status, st); break;
    }
}

}  // namespace mmsb
