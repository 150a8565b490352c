// mmsb_geo.h -- shape-derived geometry shared by the host orchestration and the kernels.
#pragma once
#include <cstdint>

namespace mmsb {

constexpr int kScanThreads = 256;   // threads per scan CTA
constexpr int kScanRounds = 4;      // 16-pixel groups per thread
constexpr int kChunk = kScanRounds * kScanThreads * 16;   // raster pixels per scan chunk (16384)
constexpr int kRecSlots = 80;       // u64 slots of a tile's in-CTA angle record: levels 1..6 (slots 0..62)
constexpr int kWRecBytes = 384;     // a tile's worker record: group table (64 B), level-1 rows (32 x u64),
constexpr int kWRecL1 = 64;         //   level-2 rows (16 x u32); byte offsets of the two row tables
constexpr int kWRecL2 = 320;
constexpr int kHistStride = 16;  // u32 per image of the label histogram (counts for b = 2..8 at index b)

struct Geo {
    int method;          // 0 EMR, 1 LMR
    int B;               // images in this launch group
    int H, W, hlog, wlog;
    long long HW;
    int emax;            // floor(log2 min(H, W))                  (reading Q6)
    int emin;            // 1 (EMR), min(4, emax) (LMR)            (Q10)
    int tp;              // tile side 2^tp = min(64, min(H, W))
    int T;
    int tilesY, tilesX, ntiles, tlog;   // tlog = log2(tilesX)
    int lvl_off[8];      // record slot of level e's first row (e = 1..tp)
    int pyr_off[16];     // upper pyramid: counter offset of level e (tp < e <= emax), per image
    int npyr;            // counters per image
    int nchunks;         // scan chunks per image
    int tile_log2;       // LMR coder tile side 2^t
    int ntiles_coder;    // LMR coder tiles per plane
    uint32_t one;        // = 1, opaque to the compiler: multiplies that keep adds / shifts on the FMA pipe
    int dr;              // keystream double rounds: 10 (ChaCha20), 6 (ChaCha12) or 4 (ChaCha8)
};

// the workers walk the upper angle pyramid in global memory when it is too large for shared
// memory (> 32 KB per image: images above 8192^2), else a copy in shared memory
__host__ __device__ inline bool pyr_glob(const Geo &g) { return g.npyr > 8192; }

inline int ilog2(long long v) {
    int e = 0;
    while ((2LL << e) <= v) e++;
    return e;
}

inline bool make_geo(int method, int B, int H, int W, int tile_log2, int lmr_emin, Geo *g, int cipher_rounds = 0) {
    if (B < 1 || H < 16 || W < 16 || H > 32768 || W > 32768) return false;
    if (cipher_rounds != 0 && cipher_rounds != 20 && cipher_rounds != 12 && cipher_rounds != 8) return false;
    g->dr = cipher_rounds ? cipher_rounds / 2 : 10;
    if ((H & (H - 1)) || (W & (W - 1))) return false;
    if (method != 0 && method != 1) return false;
    if (lmr_emin < 0 || lmr_emin > 4) return false;
    if (tile_log2 == 0) tile_log2 = 7;
    if (tile_log2 < 3 || tile_log2 > 7) return false;   // GPU coder rows hold <= 128 pixels
    g->method = method;
    g->B = B;
    g->H = H; g->W = W;
    g->hlog = ilog2(H); g->wlog = ilog2(W);
    g->HW = (long long)H * W;
    g->emax = g->hlog < g->wlog ? g->hlog : g->wlog;
    {
        const int e = lmr_emin ? lmr_emin : 4;                // Tab. LMR_block_size schedules
        g->emin = method == 0 ? 1 : (g->emax < e ? g->emax : e);
    }
    g->tp = g->emax < 6 ? g->emax : 6;
    g->T = 1 << g->tp;
    g->tilesY = H >> g->tp;
    g->tilesX = W >> g->tp;
    g->ntiles = g->tilesY * g->tilesX;
    g->tlog = ilog2(g->tilesX);
    int off = 0;
    for (int e = 0; e < 8; e++) g->lvl_off[e] = 0;
    for (int e = 1; e <= g->tp; e++) { g->lvl_off[e] = off; off += g->T >> e; }
    int p = 0;
    for (int e = 0; e < 16; e++) g->pyr_off[e] = 0;
    for (int e = g->tp + 1; e <= g->emax; e++) { g->pyr_off[e] = p; p += (H >> e) * (W >> e); }
    g->npyr = p;
    g->nchunks = (int)((g->HW + kChunk - 1) / kChunk);
    g->tile_log2 = tile_log2;
    g->one = 1;
    {
        const int th = (1 << tile_log2) < H ? (1 << tile_log2) : H, tw = (1 << tile_log2) < W ? (1 << tile_log2) : W;
        g->ntiles_coder = ((H + th - 1) / th) * ((W + tw - 1) / tw);
    }
    return true;
}

}  // namespace mmsb
