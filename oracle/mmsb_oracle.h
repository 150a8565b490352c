/*
 * mmsb_oracle.h -- plain, slow, single-threaded CPU ORACLE of the multi-MSB replacement
 * RDHEI methods EMR-RDHEI and LMR-RDHEI (arXiv 2302.07992, /root/reference/PAPER.md).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or constant generator with the CUDA product path (csrc/, include/);
 * neither side includes or links the other.
 *
 * Citations: "P:<line>" = PAPER.md line (+ section / equation label);
 *            "S:<line>" = SPEC.md line; "Qn" = a reading listed in DESIGN.md §3.
 *
 * Conventions (all fixed in DESIGN.md §3):
 *   - images are M x N uint8, row-major, raster index r = y*N + x;
 *   - bit position 1 = MSB (weight 128) ... 8 = LSB;
 *   - bit planes / maps are uint8 arrays holding 0 or 1;
 *   - message bits: bit k of a byte string is bit (7 - k%8) of byte k/8 (MSB first);
 *   - keys are 32 bytes (ChaCha20, RFC 8439, nonce 0, counter 0; Q12).
 *
 * Status values (returned per image; identical numbering to the product ABI by
 * specification, defined independently here):
 *   0 OK, 3 CAPACITY, 4 INTEGRITY, 5 BADCASE, 8 FORMAT.
 */
#ifndef MMSB_ORACLE_H
#define MMSB_ORACLE_H
#include <stdint.h>
#include <stddef.h>

#define ORC_OK 0
#define ORC_E_INVAL 2
#define ORC_E_CAPACITY 3
#define ORC_E_INTEGRITY 4
#define ORC_E_BADCASE 5
#define ORC_E_FORMAT 8

#define ORC_EMR 0
#define ORC_LMR 1

/* ---- keystream ("a cryptographically secure stream cipher"; Q12) ---- */
void orc_chacha20_block(const uint8_t key[32], uint32_t counter, const uint8_t nonce[12], uint8_t out[64]);
/* the same block with `rounds` rounds (20, or the reduced-round option 12 / 8) */
void orc_chacha_block(const uint8_t key[32], uint32_t counter, const uint8_t nonce[12], int rounds, uint8_t out[64]);
/* rounds of the keystream every call uses: 20 (reading Q12) unless set to 8 or 12 */
void orc_set_cipher_rounds(int rounds);
int orc_cipher_rounds(void);
/* bytes [offset, offset+n) of ChaCha(key, nonce=0, counter=0) with orc_cipher_rounds() rounds */
void orc_keystream(const uint8_t key[32], uint64_t offset, uint64_t n, uint8_t *out);

/* ---- location maps (eq. gliding1/gliding2; Q1-Q3) ---- */
void orc_location_map(const uint8_t *I, int M, int N, int b, uint8_t *L);
/* zeros[b] = #{L_b == 0} for b = 1..8 (zeros[0] = 0) (P:630 inner sum) */
void orc_zero_counts(const uint8_t *I, int M, int N, int64_t zeros[9]);
int orc_select_b_emr(const int64_t zeros[9]);               /* eq. optimial_b, Q4 */
void orc_lmr_candidates(const int64_t zeros[9], int order[7]); /* P:979, Q5, Q22 */

/* ---- block rotation (P:659-671 eq. roration; P:819-835 eq. roration2; Q6-Q11) ---- */
int orc_emax(int M, int N);
/* angle of every complete 2^e block (row-major over blocks): (sum of s over block) mod 4 */
void orc_block_angles(const uint8_t *s, int M, int N, int e, uint8_t *ang);
/* one pass at level e with given angles; inverse=0: clockwise by 90*ang, inverse=1: counter-clockwise */
void orc_rotate_pass(uint8_t *grid, int M, int N, int e, const uint8_t *ang, int inverse);
/* all passes e_min..e_max ascending (forward) or descending with inverse angles (inverse) */
void orc_rotate_all(uint8_t *grid, int M, int N, const uint8_t *s, int emin, int inverse);

/* ---- tile coder for bi-level planes ("JBIG-KIT"; builder-defined, Q16) ---- */
/* codes one tile of h x w bits (row-major, values 0/1); returns byte count or -1 if > cap */
int orc_tile_encode(const uint8_t *bits, int h, int w, uint8_t *out, int cap);
/* decodes nbytes into h x w bits; bytes past the end read as 0 */
void orc_tile_decode(const uint8_t *in, int nbytes, int h, int w, uint8_t *bits);
/* tile geometry of a plane: side = min(2^t, dim) */
int orc_tile_count(int M, int N, int t);

/* ---- the four calls (P:575, P:816-843 EMR; P:972-1067 LMR) ---- */
int orc_encode(int method, const uint8_t *I, int M, int N, const uint8_t k1[32], int tile_log2,
               uint8_t *E, int32_t *b_out, int64_t *capacity_out);
/* tile_log2: LMR coder tile side, shared protocol knowledge (must equal the header's t) */
int orc_hide(int method, const uint8_t *E, int M, int N, int tile_log2, const uint8_t k2[32],
             const uint8_t *msg, int64_t msg_bits, uint8_t *marked);
int orc_extract(int method, const uint8_t *marked, int M, int N, int tile_log2, const uint8_t k2[32],
                uint8_t *msg_out, int64_t stride_bytes, int64_t *msg_bits_out);
int orc_recover(int method, const uint8_t *marked, int M, int N, int tile_log2, const uint8_t k1[32], uint8_t *out);
/* LMR rotation-schedule variants of Tab. LMR_block_size: blocks {2^e_min .. 2^e_max} with
 * e_min = lmr_emin_req in 1..4 (0 = the paper's default 4), shared protocol knowledge like the method */
int orc_encode_s(int method, const uint8_t *I, int M, int N, const uint8_t k1[32], int tile_log2, int lmr_emin_req,
                 uint8_t *E, int32_t *b_out, int64_t *capacity_out);
int orc_recover_s(int method, const uint8_t *marked, int M, int N, int tile_log2, int lmr_emin_req, const uint8_t k1[32],
                  uint8_t *out);
/* capacity C that the hider/receiver derive from a marked image (header + map) */
int orc_capacity(int method, const uint8_t *marked, int M, int N, int tile_log2, int32_t *b_out, int64_t *capacity_out);

/* ---- statistics (P:630 DER, P:746 PSNR; Q23) ---- */
int64_t orc_sse(const uint8_t *a, const uint8_t *b, int64_t n);

/* ---- security / quality statistics ---- */
/* Shannon entropy H = -sum P(a_i) log2 P(a_i) over the 256 grey levels */
double orc_entropy(const uint8_t *img, int64_t n);
/* chi^2 = 256 (h w) sum (P(a_i) - 1/256)^2 */
double orc_chi2(const uint8_t *img, int64_t n);
/* NPCR = 100 * #{a != b} / n (reading Q26: sigma = 1 where the pixels DIFFER), UACI = 100 * mean(|a-b|) / 255 */
void orc_npcr_uaci(const uint8_t *a, const uint8_t *b, int64_t n, double *npcr, double *uaci);
/* mean local SSIM, 11x11 Gaussian window sigma 1.5 (normalised), K1 = 0.01, K2 = 0.03, L = 255,
 * over the windows lying fully inside the image ("valid" positions, reading in DESIGN.md) */
double orc_ssim(const uint8_t *a, const uint8_t *b, int M, int N);
void orc_der_psnr(int M, int N, int64_t capacity_bits, int64_t sse, double *der, double *psnr);

#endif
