// mmsb_kernels.h -- launchers of the sm_100a kernels (host side of csrc/).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "mmsb_geo.h"

namespace mmsb {

struct ScanWS {
    unsigned long long *states;      // [B][nchunks] flag | value (decoupled look-back)
    unsigned long long *parts;       // [B][nchunks][2] boundary words of the extracted bit string
    uint32_t *hdr;                   // [B] frame length word (extract)
    uint32_t *ef;                    // [B][ef_words] encrypted frame E_F = F XOR KS2 (embed)
    long long ef_words;              // words per image: ceil(7 HW / 512) + 1 ChaCha blocks of 16
    uint32_t *counts;                // [B][nchunks] zero pixels per chunk (embed: scan_count_kernel)
    unsigned long long *ztot;        // [B] zero pixels per image (embed)                -- zeroed per call
    uint32_t *err;                   // [B] a look-back wait timed out (status E_CUDA)  -- zeroed per call
};
__host__ __device__ inline long long ef_words_of(long long HW) { return ((7 * HW + 511) / 512 + 1) * 16; }

// LMR encode state of one image: candidate order (P:985 walk), decision and header length K
struct LmrPlan {
    int8_t order[7];
    int8_t state;                    // 0 undecided, 1 fits (b), 2 bad case
    int32_t b;
    int32_t dslot;                   // stream slot of the decided map (1 + its candidate index)
    int32_t eta_bytes;               // coded eta bytes (after wave 0; -1: a tile over cap)
    long long K;                     // MSB-plane bits used: 7 + 32 T + 8 (bytes_eta + bytes_map)
};

// Candidate waves: wave w codes, for the count[w] images still undecided
// (list[w]), candidates nc[w] .. nc[w]+k_w-1 of their order at once, k_w as many as fill two
// rounds of resident tiles (wave 0: eta and candidate 0 for every image); the fit then takes the
// first candidate in order that fits, exactly the serial walk's choice.
constexpr int kLmrSlots = 8;         // stream slots per image: eta, candidates 0..6
constexpr int kMapStats = 32;        // ints per image of LmrEncWS::mapbytes
struct LmrWaveCtl {
    int count[8];                    // images entering wave w (count[0] = B)
    int nc[8];                       // candidates tried before wave w
};
struct LmrEncWS {
    LmrPlan *plan;                   // [B]
    LmrWaveCtl *ctl;
    int32_t *lists;                  // [8][B] image list of each wave
    uint8_t *streams;                // [B][kLmrSlots][Tc] slots of lmr_tile_stride bytes
    int32_t *sizes;                  // [B][kLmrSlots][Tc] stream bytes (-1: over cap)
    int32_t *dsizes;                 // [B][2][Tc] sizes of the decided eta + map streams
    int32_t *offsets;                // [B][2][Tc] their exclusive byte offsets
    uint8_t *cat;                    // [B][HW/8] the decided streams concatenated (the mbuf region)
    int32_t *mapbytes;               // [B][kMapStats]: [c] running coded bytes of candidate c's map (early
                                     // abort), [8 + c] its finished tiles, [16] the first candidate known to fit
};
#ifndef MMSB_LMR_WAVE_ROUNDS
#define MMSB_LMR_WAVE_ROUNDS 3
#endif
constexpr int kLmrWaveRounds = MMSB_LMR_WAVE_ROUNDS;
__host__ __device__ inline int lmr_wave_k(int wave, int A, int Tc, int B, int R, int nc) {
    if (wave == 0) {                                            // eta + k candidates per image
        const int k = R / (B * Tc) - 1;
        return k < 1 ? 1 : (k > 7 ? 7 : k);
    }
    // later waves: up to kLmrWaveRounds rounds of tiles (3 measured best: 2 / 5 rounds -1 %);
    // their items are candidate-major, so the CTAs of a
    // failing candidate abort together and the next candidate's CTAs take their SMs
    if (A <= 0) return 1;
    const int k = kLmrWaveRounds * R / (A * Tc), left = 7 - nc;
    return k < 1 ? 1 : (k > left ? left : k);
}

void launch_lmr_plan(const Geo &g, const uint32_t *hist, const LmrEncWS &e, cudaStream_t st);
void launch_coder_encode(const Geo &g, int wave, const uint8_t *ceta, const LmrEncWS &e,
                         unsigned long long *sym_count, cudaStream_t st);
void launch_lmr_fit(const Geo &g, int wave, const LmrEncWS &e, cudaStream_t st);
void launch_lmr_msb_write(const Geo &g, const LmrEncWS &e, const uint32_t *hist, uint8_t *enc, int32_t *b_out,
                          int64_t *cap_out, int32_t *status, cudaStream_t st);
void launch_lmr_decode(const Geo &g, bool want_eta, const uint8_t *marked, uint8_t *mbuf, int32_t *lmr_b,
                       int32_t *lmr_t, int32_t *offsets, int32_t *sizes, uint32_t *eta_bits, uint32_t *map_bits,
                       int32_t *status, int64_t *msg_bits_out,
                       unsigned long long *sym_count, cudaStream_t st);
int lmr_tile_cap_host(int t, int H, int W);
int lmr_tile_stride_host(int t, int H, int W);

// per-call device state of the fused encode / recover kernels (k_fused.cu).  Per tile a scratch
// block of three T x T planes (row-major, rows swapped in pairs for odd cell rows: TileBlock):
// written by the keystream CTAs, read once by one worker CTA of the same launch with bulk copies,
// then discarded from L2.
struct TileWS {
    uint8_t *s;          // [B][ntiles][3][T*T] per tile: K1 keystream (destination-domain tile), the
                         // call's input image tile (encode: I; recover: I_e'), encode's label plane
                         // (EMR: thermometer code of p ^ left; LMR: eta | its bits 0..6)
    uint64_t *rec;       // [B][ntiles][kRecSlots] worker record: group table + cell table
    uint32_t *pyr;       // [B][npyr] upper-level block sums (mod 4 on read)        -- zeroed per call
    uint32_t *hist;      // [B][kHistStride] non-redundant counts for b = 2..8 at index b -- zeroed per call
    uint32_t *kdone;     // [B] keystream CTAs finished                               -- zeroed per call
};
// blockIdx -> role schedule: groups of GI images (a power of two), 2^lgK keystream and 2^lgW
// worker CTAs per image, worker CTAs of group g dispatched L grid rows after its keystream CTAs
// worker CTAs per image = 2^lgW = strips x 2^lgS segments per strip (encode splits wide strips;
// recovery keeps whole strips: its row copy-forward carries from tile to tile)
struct FusedSched { int GI, ngroups, lgK, lgW, lgS, L; };
FusedSched fused_sched(const Geo &g, bool split_strips = false);

void launch_encode(const Geo &g, const uint8_t *images, const uint8_t *keys, const TileWS &ws, uint8_t *enc,
                   uint8_t *ceta, int32_t *b_out, int64_t *cap_out, int32_t *status, cudaStream_t st);
void launch_recover(const Geo &g, const uint8_t *marked, const uint8_t *keys, const TileWS &ws, const uint32_t *eta,
                    const uint32_t *map, const int32_t *lmr_b, uint8_t *out, int32_t *status, cudaStream_t st,
                    const uint8_t *original = nullptr, unsigned long long *sse = nullptr);
void launch_scan(const Geo &g, bool embed, const uint8_t *in, uint8_t *out, const uint8_t *keys, const uint8_t *msg,
                 const int64_t *msg_bits, long long stride, uint8_t *msg_out, int64_t *msg_bits_out, int32_t *status,
                 const ScanWS &ws, const uint32_t *map_bits, const int32_t *lmr_b, cudaStream_t st);
void launch_histogram(long long HW, int B, const uint8_t *img, int64_t *hist, cudaStream_t st);
void launch_diff_stats(long long HW, int B, const uint8_t *a, const uint8_t *b, int64_t *sse, int64_t *ndiff,
                       int64_t *absd, cudaStream_t st);
void launch_ssim(int B, int H, int W, const uint8_t *a, const uint8_t *b, double *ssim, cudaStream_t st);
void launch_status_merge(int B, const int32_t *second, int32_t *status, cudaStream_t st);
void launch_capacity(const Geo &g, const uint8_t *in, const uint32_t *map_bits, const int32_t *lmr_b,
                     int32_t *b_out, int64_t *cap_out, int32_t *status, cudaStream_t st);
void launch_stats(long long HW, int B, const uint8_t *a, const uint8_t *b, int64_t *sse, cudaStream_t st);

}  // namespace mmsb
