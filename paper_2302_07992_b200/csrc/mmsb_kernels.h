// mmsb_kernels.h -- launchers of the sm_100a kernels (host side of csrc/).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "mmsb_geo.h"

namespace mmsb {

struct ScanWS {
    unsigned int *ticket;            // CTA issue order (decoupled look-back needs it)
    unsigned long long *states;      // [B][nchunks] flag | value
    unsigned int *done;              // [B] finished chunks (last CTA does the per-image fixup)
    unsigned long long *parts;       // [B][nchunks][2] boundary words of the extracted bit string
    uint32_t *hdr;                   // [B] frame length word (extract)
};

struct LmrWS {
    uint8_t *ceta;                   // [G][H][W] rotated (I & 0x80) | label c
    uint32_t *eta_bits;              // [B][H*W/32] decoded rotated eta (MSB map)
    uint32_t *map_bits;              // [B][H*W/32] decoded rotated location map
    int32_t *b;                      // [B] decoded b (<= 0: bad / malformed)
    uint8_t *streams;                // coder output scratch
    int32_t *sizes;                  // per tile byte counts
    int32_t *cand;                   // per image candidate state
};

void launch_ks_tile(const Geo &g, int G, const uint8_t *keys, const uint8_t *images, uint8_t *s, uint64_t *rec,
                    uint32_t *pyr, uint32_t *hist, cudaStream_t st);
void launch_perm_encode(const Geo &g, int G, const uint8_t *images, const uint8_t *s, const uint64_t *rec,
                        const uint32_t *pyr, const uint32_t *hist, uint8_t *enc, uint8_t *ceta, int32_t *b_out,
                        int64_t *cap_out, int32_t *status, cudaStream_t st);
void launch_recover_strip(const Geo &g, int G, const uint8_t *marked, const uint8_t *s, const uint64_t *rec,
                          const uint32_t *pyr, const uint32_t *eta, const uint32_t *map, const int32_t *lmr_b,
                          uint8_t *out, int32_t *status, cudaStream_t st);
void launch_scan(const Geo &g, bool embed, const uint8_t *in, uint8_t *out, const uint8_t *keys, const uint8_t *msg,
                 const int64_t *msg_bits, long long stride, uint8_t *msg_out, int64_t *msg_bits_out, int32_t *status,
                 const ScanWS &ws, const uint32_t *map_bits, const int32_t *lmr_b, cudaStream_t st);
void launch_stats(long long HW, int B, const uint8_t *a, const uint8_t *b, int64_t *sse, cudaStream_t st);

}  // namespace mmsb
