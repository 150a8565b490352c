/*
 * mmsb.h -- C ABI of the B200-native multi-MSB replacement RDHEI hot path
 * (EMR-RDHEI and LMR-RDHEI, arXiv 2302.07992; /root/reference/PAPER.md cited as P:<line>).
 *
 * The four calls follow the three parties of the paper (Fig. fig:General_EMR P:467-565,
 * Fig. fig:General_LMR P:848-970): the content owner ENCODES with K1, the data hider
 * EMBEDS with K2, the receiver EXTRACTS with K2 only and/or RECOVERS with K1 only
 * (separability).  Formats, bit orders and readings: DESIGN.md §3.
 *
 * Conventions for every call
 *  - All data pointers (images, keys, messages, per-image outputs, workspace) are DEVICE
 *    pointers owned by the caller; the library allocates nothing and never synchronises.
 *    Every call is asynchronous on `stream` (a cudaStream_t passed as void*).
 *  - Images are [batch][height][width] uint8, row-major (raster index r = y*W + x).
 *    The GPU path accepts power-of-two height and width in [16, 32768].
 *  - Keys are [batch][32] bytes (ChaCha20 / RFC 8439 key, nonce 0, counter 0; reading Q12).
 *  - Message buffers are [batch][stride_bytes], stride_bytes % 16 == 0; message bit k is
 *    bit (7 - k%8) of byte k/8 (numpy.packbits(bitorder='big')); a stride of
 *    ceil(7*H*W/8) bytes covers any capacity.
 *  - Return value = synchronous validation (E_INVAL: null pointer, unsupported shape,
 *    workspace too small; E_CUDA: a launch failed).  Data-dependent outcomes are written,
 *    asynchronously, to the per-image device array img_status[batch] (OK, CAPACITY,
 *    INTEGRITY, BADCASE, FORMAT).  img_status = E_CUDA marks an image whose cross-CTA wait
 *    inside encode / recover (keystream CTAs -> worker CTAs) or extract (decoupled look-back)
 *    timed out (~2 s): those waits rely on in-order CTA dispatch, and a launch that cannot
 *    provide it (e.g. an SM partition holding back earlier CTAs) ends instead of hanging.
 *  - `ws` is caller-allocated device scratch of at least mmsb_workspace_bytes(shape) bytes,
 *    256-byte aligned; one workspace may serve every call made on the same stream.
 */
#ifndef MMSB_H
#define MMSB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    MMSB_OK = 0,
    MMSB_E_INVAL = 2,
    MMSB_E_CAPACITY = 3,     /* 32 + n > C: the frame does not fit (reading Q17)          */
    MMSB_E_INTEGRITY = 4,    /* decrypted length n > C - 32 (wrong K2 or tampering)               */
    MMSB_E_BADCASE = 5,      /* LMR: no candidate map fits the MSB plane          */
    MMSB_E_CUDA = 6,
    MMSB_E_UNIMPLEMENTED = 7,
    MMSB_E_FORMAT = 8        /* malformed header / stream                                         */
} mmsb_status;

typedef enum { MMSB_EMR = 0, MMSB_LMR = 1 } mmsb_method;

typedef struct {
    int32_t method;      /* mmsb_method                                                        */
    int32_t batch;       /* images in the batch (>= 1)                                         */
    int32_t height;      /* M (power of two, 16..32768)                                        */
    int32_t width;       /* N (power of two, 16..32768)                                        */
    int32_t tile_log2;   /* LMR map-coder tile side 2^t, t in [3, 7] (0 = default 7)           */
    int32_t lmr_emin;    /* LMR rotation blocks {2^e_min .. 2^e_max}: 0 = the paper's e_min = 4;
                            1..3 = the schedules of Tab. LMR_block_size.  Shared
                            protocol knowledge like the method (not stored in the image).  EMR: 1.  */
    int32_t cipher_rounds; /* keystream cipher: 0 or 20 = ChaCha20 (RFC 8439, reading Q12); 12 or 8 =
                            the reduced-round format option (P:656 asks only for
                            "a cryptographically secure stream cipher").  Shared knowledge of both
                            parties like the method; every K1 and K2 keystream uses it.            */
} mmsb_shape;

/* Bytes of device workspace the four calls need for this shape. 0 if the shape is invalid. */
size_t mmsb_workspace_bytes(const mmsb_shape *shape);

/*
 * Content owner, encoding phase (EMR: P:575-747; LMR: P:972-988).
 *   images     [B][H][W] original images I
 *   k1         [B][32]   image-encryption keys K1
 *   encrypted  [B][H][W] output I_e (EMR: LSB plane = header || rotated map, P:743-744;
 *                        LMR: MSB plane = header || tile tables || coded maps)
 *   b_out      [B] int32 chosen b (eq. optimial_b; LMR P:979); 0 on BADCASE
 *   capacity_out [B] int64 C = b*zeros (EMR) or (b-1)*zeros (LMR) bits; 0 on BADCASE
 *   img_status [B] int32 OK or BADCASE (LMR)
 */
mmsb_status mmsb_content_owner_encode(const mmsb_shape *shape, const uint8_t *images, const uint8_t *k1,
                                      uint8_t *encrypted, int32_t *b_out, int64_t *capacity_out,
                                      int32_t *img_status, void *ws, size_t ws_bytes, void *stream);

/*
 * Data hider (EMR: P:749-750; LMR: P:990-991).  Needs no K1.
 *   encrypted  [B][H][W] I_e
 *   k2         [B][32]   data-hiding keys K2
 *   msg_bytes  [B][stride_bytes] plain messages, msg_bits[B] (int64) bits each
 *   marked     [B][H][W] output I_e' (may alias encrypted: embedding in place)
 * The frame BE32(n) || message is XORed with the K2 keystream and written b (EMR, bit
 * positions 1..b) or b-1 (LMR, positions 2..b) bits per redundant pixel in raster order of
 * the rotated domain; all other bits are copied.  img_status: OK, CAPACITY (then marked ==
 * encrypted: nothing is embedded), FORMAT, BADCASE.
 */
mmsb_status mmsb_hider_embed(const mmsb_shape *shape, const uint8_t *encrypted, const uint8_t *k2,
                             const uint8_t *msg_bytes, const int64_t *msg_bits, int64_t stride_bytes,
                             uint8_t *marked, int32_t *img_status, void *ws, size_t ws_bytes, void *stream);

/*
 * Receiver with K2 only: data extraction, no de-rotation (EMR: P:839-840; LMR: P:1063-1064).
 *   msg_out     [B][stride_bytes]: the first ceil(max(C-32,0)/32) 32-bit words receive the message bits
 *               [0, n) followed by zeros; later bytes are untouched.
 *   msg_bits_out [B] int64: n, or -1 on INTEGRITY / FORMAT / BADCASE.
 */
mmsb_status mmsb_receiver_extract(const mmsb_shape *shape, const uint8_t *marked, const uint8_t *k2,
                                  uint8_t *msg_out, int64_t stride_bytes, int64_t *msg_bits_out,
                                  int32_t *img_status, void *ws, size_t ws_bytes, void *stream);

/*
 * Receiver with K1 only: image recovery (EMR: P:819-837; LMR: P:1060-1061).
 *   recovered [B][H][W]: EMR -> original except the LSB plane (= decrypted bits, reading Q20);
 *   LMR -> the original exactly.  Zero-filled on FORMAT / BADCASE.
 */
mmsb_status mmsb_receiver_recover(const mmsb_shape *shape, const uint8_t *marked, const uint8_t *k1,
                                  uint8_t *recovered, int32_t *img_status, void *ws, size_t ws_bytes,
                                  void *stream);

/*
 * The same recovery fused with the statistics call's SSE (evaluation harnesses only: the
 * receiver of the protocol does not hold the original).  sse_out[i] = sum over pixels of
 * (original - recovered)^2 as int64 (PSNR P:746 via mmsb_der_psnr_host), computed from the
 * recovered pixels while they are in registers: no second pass over I and I'.  original is
 * [B][H][W] device memory; sse_out [B] int64 device memory (written, not accumulated);
 * recovered and img_status exactly as mmsb_receiver_recover.
 */
mmsb_status mmsb_receiver_recover_sse(const mmsb_shape *shape, const uint8_t *marked, const uint8_t *k1,
                                      const uint8_t *original, uint8_t *recovered, int64_t *sse_out,
                                      int32_t *img_status, void *ws, size_t ws_bytes, void *stream);

/*
 * Capacity query (the SPEC's `capacity`): what an encrypted or marked image
 * offers, derived the way the hider and the K2 receiver derive it -- no key needed.  b from the
 * header (EMR: the LSBs of pixels 0..2, reading Q14; LMR: the MSB-plane header) and
 * C = b' * (redundant pixels of the location map), b' = b (EMR) or b - 1 (LMR).
 *   image        [B][H][W] device, an output of mmsb_content_owner_encode or mmsb_hider_embed.
 *   b_out        [B] int32; 0 on FORMAT / BADCASE.
 *   capacity_out [B] int64 bits (the frame, 32 + n, must fit); 0 on FORMAT / BADCASE.
 *   img_status   [B]: OK, FORMAT or BADCASE.  Uses ws (LMR: the map decode).
 */
mmsb_status mmsb_capacity(const mmsb_shape *shape, const uint8_t *image, int32_t *b_out, int64_t *capacity_out,
                          int32_t *img_status, void *ws, size_t ws_bytes, void *stream);

/*
 * Receiver holding both keys (EMR: P:842-843; LMR: P:1066-1067): extraction
 * with K2 and recovery with K1 in one call.  Outputs are those of mmsb_receiver_extract and
 * mmsb_receiver_recover on the same arguments; LMR decodes the coded maps (eta and the location
 * map) from the MSB plane once for both steps instead of once per call.  img_status: the
 * extraction's status if it is not OK (INTEGRITY, FORMAT, BADCASE, E_INVAL region), else the
 * recovery's.
 */
mmsb_status mmsb_receiver_both(const mmsb_shape *shape, const uint8_t *marked, const uint8_t *k1, const uint8_t *k2,
                               uint8_t *msg_out, int64_t stride_bytes, int64_t *msg_bits_out, uint8_t *recovered,
                               int32_t *img_status, void *ws, size_t ws_bytes, void *stream);

/* Per-image sum of squared differences (int64) of two image batches (P:746 PSNR numerator). */
mmsb_status mmsb_stats(const mmsb_shape *shape, const uint8_t *original, const uint8_t *recovered,
                       int64_t *sse_out, void *stream);

/* HOST function on HOST arrays: DER_i = C_i / (H W); PSNR_i = 10 log10(65025 H W / SSE_i),
 * +inf when SSE_i == 0. */
void mmsb_der_psnr_host(int32_t batch, int32_t height, int32_t width, const int64_t *capacity_bits,
                        const int64_t *sse, double *der_out, double *psnr_out);

/*
 * The paper's security / quality statistics.
 * Device arrays in, device arrays out, asynchronous on `stream`; integer counts are exact, SSIM is
 * computed in fp64.  The host functions turn the counts into the paper's quantities.
 *   mmsb_histogram   hist_out [B][256] int64: grey-level counts of each image (overwritten)
 *   mmsb_diff_stats  per image: sse = sum (a-b)^2, ndiff = #{a != b}, absdiff = sum |a-b|
 *   mmsb_ssim        ssim_out [B] double: mean local SSIM, 11x11 Gaussian window sigma 1.5,
 *                    K1 = 0.01, K2 = 0.03, L = 255, over the (H-10)(W-10) windows inside
 *                    the image (reading in DESIGN.md §3)
 */
mmsb_status mmsb_histogram(const mmsb_shape *shape, const uint8_t *images, int64_t *hist_out, void *stream);
mmsb_status mmsb_diff_stats(const mmsb_shape *shape, const uint8_t *a, const uint8_t *b, int64_t *sse_out,
                            int64_t *ndiff_out, int64_t *absdiff_out, void *stream);
mmsb_status mmsb_ssim(const mmsb_shape *shape, const uint8_t *a, const uint8_t *b, double *ssim_out, void *stream);
/* HOST: Shannon entropy H = -sum P log2 P and chi^2 = 256 (H W) sum (P - 1/256)^2
 * from the histograms; NPCR = 100 ndiff / (H W), UACI = 100 absdiff / (255 H W) (Q26) */
void mmsb_entropy_chi2_host(int32_t batch, int32_t height, int32_t width, const int64_t *hist, double *entropy_out,
                            double *chi2_out);
void mmsb_npcr_uaci_host(int32_t batch, int32_t height, int32_t width, const int64_t *ndiff, const int64_t *absdiff,
                         double *npcr_out, double *uaci_out);

const char *mmsb_status_string(mmsb_status status);

/* Number of kernels the library launched since load (for the bench's gpu_launches claim). */
uint64_t mmsb_kernel_launches(void);

/* Live per-kernel timing.  mmsb_profile_enable(1) clears the record and brackets every later
 * kernel launch with CUDA events on its launch stream; mmsb_profile_enable(0) stops.  After the
 * caller synchronises, mmsb_profile_read(k, ...) returns, for kernel class k in [0, K), its name,
 * the summed event time in ms, the number of launches and the pixels they processed (for the LMR
 * tile coder classes: the symbols coded / decoded, counted on the device); the return value is K
 * (the number of kernel classes), or < 0 for an invalid k / unfinished events. */
void mmsb_profile_enable(int on);
int mmsb_profile_read(int kernel, const char **name, double *total_ms, int64_t *launches, int64_t *units);

#ifdef __cplusplus
}
#endif

#endif /* MMSB_H */
