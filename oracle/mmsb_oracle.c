/*
 * mmsb_oracle.c -- plain, slow, single-threaded CPU ORACLE of EMR-RDHEI / LMR-RDHEI
 * (arXiv 2302.07992).  TEST INFRASTRUCTURE ONLY -- see mmsb_oracle.h for who may use it.
 *
 * Every function follows the paper's algorithm step by step, in the paper's order and
 * notation, with no blocking, fusion or reordering.  Where the paper is silent or garbled
 * the reading taken is the one named (Qn) and listed in DESIGN.md §3.
 *
 * Pins (tests/test_oracle_*.py, run with -m "not gpu"):
 *   keystream     RFC 8439 vectors + the `cryptography` package's ChaCha20
 *   maps / b      an independent left-neighbour formula (numpy), SPEC worked examples,
 *                 exhaustive two-valued 4x4 images, brute force over b
 *   rotation      numpy.rot90 per block, worked example S:218, round trip, exhaustive
 *                 angle injection on 4x4 two-level schedules
 *   EMR           extract(hide(m)) = m, capacity boundary, bits 1..7 of I' = I,
 *                 PSNR closed form 10*log10(65025*MN/n_mis), constant-image DER
 *   LMR           I' = I exactly, MSB plane untouched by the hider, (b-1)/b identity
 *   coder         round trip (exhaustive 4x4, random planes), ideal-code-length bound
 *   statistics    one-pixel-255 closed form (54.1854 dB), +inf on equality
 * Nothing here is "parity unpinned".
 */
#include "mmsb_oracle.h"
#include <stdlib.h>
#include <string.h>
#include <math.h>

/* ===================================================================================
 * Keystream: ChaCha20 per RFC 8439 §2.3 (P:656 permits any cryptographically secure
 * stream cipher; Q12 fixes ChaCha20, nonce 0, counter 0, bytes in raster order).
 * =================================================================================== */
static uint32_t rd_le32(const uint8_t *p)
{
    return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}

static uint32_t rotl32(uint32_t v, int c) { return (v << c) | (v >> (32 - c)); }

static void quarter_round(uint32_t *x, int a, int b, int c, int d)
{
    x[a] += x[b]; x[d] ^= x[a]; x[d] = rotl32(x[d], 16);
    x[c] += x[d]; x[b] ^= x[c]; x[b] = rotl32(x[b], 12);
    x[a] += x[b]; x[d] ^= x[a]; x[d] = rotl32(x[d], 8);
    x[c] += x[d]; x[b] ^= x[c]; x[b] = rotl32(x[b], 7);
}

/* ChaCha block with an explicit round count (20 = RFC 8439; 12 and 8 = the reduced-round
 * format option of SURVEY §8(f) NEXT 4: the same double rounds, fewer of them). */
void orc_chacha_block(const uint8_t key[32], uint32_t counter, const uint8_t nonce[12], int rounds, uint8_t out[64])
{
    uint32_t st[16], x[16];
    st[0] = 0x61707865u; st[1] = 0x3320646eu; st[2] = 0x79622d32u; st[3] = 0x6b206574u;
    for (int i = 0; i < 8; i++) st[4 + i] = rd_le32(key + 4 * i);
    st[12] = counter;
    for (int i = 0; i < 3; i++) st[13 + i] = rd_le32(nonce + 4 * i);
    memcpy(x, st, sizeof x);
    for (int r = 0; r < rounds / 2; r++) {       /* column + diagonal round pairs (20 rounds = 10) */
        quarter_round(x, 0, 4, 8, 12); quarter_round(x, 1, 5, 9, 13);
        quarter_round(x, 2, 6, 10, 14); quarter_round(x, 3, 7, 11, 15);
        quarter_round(x, 0, 5, 10, 15); quarter_round(x, 1, 6, 11, 12);
        quarter_round(x, 2, 7, 8, 13); quarter_round(x, 3, 4, 9, 14);
    }
    for (int i = 0; i < 16; i++) {
        uint32_t v = x[i] + st[i];
        out[4 * i + 0] = (uint8_t)v; out[4 * i + 1] = (uint8_t)(v >> 8);
        out[4 * i + 2] = (uint8_t)(v >> 16); out[4 * i + 3] = (uint8_t)(v >> 24);
    }
}

/* rounds of the keystream cipher used by every call below: 20 (ChaCha20, reading Q12) unless a
 * test selects the reduced-round option (8 or 12) -- process-wide, like the image format */
static int g_cipher_rounds = 20;
void orc_set_cipher_rounds(int rounds) { g_cipher_rounds = (rounds == 8 || rounds == 12) ? rounds : 20; }
int orc_cipher_rounds(void) { return g_cipher_rounds; }

void orc_chacha20_block(const uint8_t key[32], uint32_t counter, const uint8_t nonce[12], uint8_t out[64])
{
    orc_chacha_block(key, counter, nonce, 20, out);
}

void orc_keystream(const uint8_t key[32], uint64_t offset, uint64_t n, uint8_t *out)
{
    static const uint8_t zero_nonce[12] = {0};
    uint8_t blk[64];
    for (uint64_t i = 0; i < n; i++) {
        uint64_t pos = offset + i;
        if (i == 0 || pos % 64 == 0) orc_chacha_block(key, (uint32_t)(pos / 64), zero_nonce, g_cipher_rounds, blk);
        out[i] = blk[pos % 64];
    }
}

/* ===================================================================================
 * Location map generation: the literal Omega glide of eq. gliding1 / gliding2
 * (P:604-625).  Omega(i) is initialised from the first column and L(i,0) = 1;
 * for j = 1..N-1, L = 0 (redundant) iff the b MSBs equal Omega's (text polarity, Q1;
 * all b MSBs compared, Q2), and Omega := Phi(i,j) whenever L = 1 (eq. gliding2).
 * =================================================================================== */
static int top_bits(int p, int b) { return p >> (8 - b); }

void orc_location_map(const uint8_t *I, int M, int N, int b, uint8_t *L)
{
    for (int i = 0; i < M; i++) {
        int omega = top_bits(I[(size_t)i * N], b);
        L[(size_t)i * N] = 1;
        for (int j = 1; j < N; j++) {
            int phi = top_bits(I[(size_t)i * N + j], b);
            if (phi == omega) {
                L[(size_t)i * N + j] = 0;
            } else {
                L[(size_t)i * N + j] = 1;
                omega = phi;
            }
        }
    }
}

void orc_zero_counts(const uint8_t *I, int M, int N, int64_t zeros[9])
{
    uint8_t *L = (uint8_t *)malloc((size_t)M * N);
    zeros[0] = 0;
    for (int b = 1; b <= 8; b++) {
        orc_location_map(I, M, N, b, L);
        int64_t z = 0;
        for (size_t r = 0; r < (size_t)M * N; r++) z += (L[r] == 0);   /* sum_{i,j} I(L=0), P:630 (Q3) */
        zeros[b] = z;
    }
    free(L);
}

/* eq. optimial_b: b = argmax_{b in [2,7]} b * zeros(b) / MN; ties -> smaller b (Q4) */
int orc_select_b_emr(const int64_t zeros[9])
{
    int best = 2;
    for (int b = 3; b <= 7; b++)
        if ((int64_t)b * zeros[b] > (int64_t)best * zeros[best]) best = b;
    return best;
}

/* LMR: b in [2,8] (footnote P:979), ordered by real capacity (b-1)*zeros(b) descending
 * (Q5), ties -> smaller b; the encoder walks this order (Q22). */
void orc_lmr_candidates(const int64_t zeros[9], int order[7])
{
    for (int k = 0; k < 7; k++) order[k] = k + 2;
    for (int k = 1; k < 7; k++) {                  /* stable insertion sort */
        int b = order[k], j = k - 1;
        while (j >= 0 && (int64_t)(order[j] - 1) * zeros[order[j]] < (int64_t)(b - 1) * zeros[b]) {
            order[j + 1] = order[j];
            j--;
        }
        order[j + 1] = b;
    }
}

/* ===================================================================================
 * Multi-scale block rotation (eq. roration; de-rotation P:819-835,
 * eq. roration2).  Block sides 2^e for e in [e_min, e_max], e_max = floor(log2 min(M,N))
 * (Q6); only complete blocks rotate (Q7, Q11); forward = clockwise 90*angle,
 * ascending e; inverse = counter-clockwise, descending e (Q8, Q9).
 * =================================================================================== */
int orc_emax(int M, int N)
{
    int m = M < N ? M : N, e = 0;
    while ((2 << e) <= m) e++;
    return e;
}

void orc_block_angles(const uint8_t *s, int M, int N, int e, uint8_t *ang)
{
    int n = 1 << e, BM = M / n, BN = N / n;
    for (int by = 0; by < BM; by++)
        for (int bx = 0; bx < BN; bx++) {
            uint64_t sum = 0;
            for (int i = by * n; i < (by + 1) * n; i++)
                for (int j = bx * n; j < (bx + 1) * n; j++) sum += s[(size_t)i * N + j];
            ang[by * BN + bx] = (uint8_t)(sum % 4);
        }
}

void orc_rotate_pass(uint8_t *grid, int M, int N, int e, const uint8_t *ang, int inverse)
{
    int n = 1 << e, BM = M / n, BN = N / n;
    uint8_t *in = (uint8_t *)malloc((size_t)n * n), *out = (uint8_t *)malloc((size_t)n * n);
    for (int by = 0; by < BM; by++)
        for (int bx = 0; bx < BN; bx++) {
            int a = ang[by * BN + bx];
            for (int i = 0; i < n; i++)
                memcpy(in + (size_t)i * n, grid + (size_t)(by * n + i) * N + bx * n, n);
            for (int t = 0; t < a; t++) {
                for (int i = 0; i < n; i++)
                    for (int j = 0; j < n; j++) {
                        if (!inverse) out[i * n + j] = in[(n - 1 - j) * n + i];   /* 90 deg clockwise */
                        else out[i * n + j] = in[j * n + (n - 1 - i)];            /* 90 deg counter-clockwise */
                    }
                memcpy(in, out, (size_t)n * n);
            }
            for (int i = 0; i < n; i++)
                memcpy(grid + (size_t)(by * n + i) * N + bx * n, in + (size_t)i * n, n);
        }
    free(in);
    free(out);
}

void orc_rotate_all(uint8_t *grid, int M, int N, const uint8_t *s, int emin, int inverse)
{
    int emax = orc_emax(M, N);
    uint8_t *ang = (uint8_t *)malloc((size_t)M * N / 4 + 1);
    if (!inverse) {
        for (int e = emin; e <= emax; e++) {
            orc_block_angles(s, M, N, e, ang);
            orc_rotate_pass(grid, M, N, e, ang, 0);
        }
    } else {
        for (int e = emax; e >= emin; e--) {
            orc_block_angles(s, M, N, e, ang);
            orc_rotate_pass(grid, M, N, e, ang, 1);
        }
    }
    free(ang);
}

static int emr_emin(int M, int N) { (void)M; (void)N; return 1; }          /* P:1073 {2^1..2^n} */
static int lmr_emin(int M, int N, int req)           /* P:985 {2^4..}, Q10; Tab. LMR_block_size variants */
{
    int emax = orc_emax(M, N), e = (req >= 1 && req <= 4) ? req : 4;
    return emax < e ? emax : e;
}

/* ===================================================================================
 * Bi-level tile coder: stands in for JBIG-KIT (builder-defined, Q16).
 * Context: 9 causal tile-local pixels (out-of-tile = 0), MSB->LSB:
 *   (0,-1) (-1,-2) (-1,-1) (-1,0) (-1,+1) (-1,+2) (-2,-1) (-2,0) (-2,+1)   (Q16).
 * Model: per context a 16-bit probability of a 0, p0, initially 32768; after a 0,
 *   p0 += (65536 - p0) >> 4; after a 1, p0 -= p0 >> 4.
 * Coder: carry-propagating binary range coder, 32-bit range, bound = (range >> 16) * p0;
 *   0 -> range = bound; 1 -> low += bound, range -= bound; renormalise while range < 2^24
 *   by shifting out one byte (pending 0xFF run + cache byte); flush = 5 byte shifts.
 * =================================================================================== */
#define ORC_RATE 4
#define ORC_NCTX 512

static int ctx_of(const uint8_t *bits, int h, int w, int y, int x)
{
    (void)h;
#define PX(dy, dx) ((y + (dy) >= 0 && x + (dx) >= 0 && x + (dx) < w) ? bits[(size_t)(y + (dy)) * w + (x + (dx))] : 0)
    int c = (PX(0, -1) << 8) | (PX(-1, -2) << 7) | (PX(-1, -1) << 6) | (PX(-1, 0) << 5) |
            (PX(-1, 1) << 4) | (PX(-1, 2) << 3) | (PX(-2, -1) << 2) | (PX(-2, 0) << 1) | PX(-2, 1);
#undef PX
    return c;
}

typedef struct {
    uint64_t low;
    uint32_t range;
    uint8_t cache;
    uint64_t cache_size;
    uint8_t *out;
    int n, cap, overflow;
} rc_enc;

static void rc_put(rc_enc *e, uint8_t v)
{
    if (e->n < e->cap) e->out[e->n] = v; else e->overflow = 1;
    e->n++;
}

static void rc_shift_low(rc_enc *e)
{
    if ((uint32_t)e->low < 0xFF000000u || (e->low >> 32) != 0) {
        uint8_t carry = (uint8_t)(e->low >> 32);
        uint8_t temp = e->cache;
        do {
            rc_put(e, (uint8_t)(temp + carry));
            temp = 0xFF;
        } while (--e->cache_size != 0);
        e->cache = (uint8_t)((uint32_t)e->low >> 24);
    }
    e->cache_size++;
    e->low = (uint64_t)((uint32_t)e->low << 8);
}

int orc_tile_encode(const uint8_t *bits, int h, int w, uint8_t *out, int cap)
{
    uint16_t p0[ORC_NCTX];
    for (int i = 0; i < ORC_NCTX; i++) p0[i] = 32768;
    rc_enc e = {0, 0xFFFFFFFFu, 0, 1, out, 0, cap, 0};
    for (int y = 0; y < h; y++)
        for (int x = 0; x < w; x++) {
            int c = ctx_of(bits, h, w, y, x);
            uint32_t bound = (e.range >> 16) * p0[c];
            if (bits[(size_t)y * w + x] == 0) {
                e.range = bound;
                p0[c] = (uint16_t)(p0[c] + ((65536u - p0[c]) >> ORC_RATE));
            } else {
                e.low += bound;
                e.range -= bound;
                p0[c] = (uint16_t)(p0[c] - (p0[c] >> ORC_RATE));
            }
            while (e.range < (1u << 24)) {
                e.range <<= 8;
                rc_shift_low(&e);
            }
        }
    for (int i = 0; i < 5; i++) rc_shift_low(&e);
    return e.overflow ? -1 : e.n;
}

void orc_tile_decode(const uint8_t *in, int nbytes, int h, int w, uint8_t *bits)
{
    uint16_t p0[ORC_NCTX];
    for (int i = 0; i < ORC_NCTX; i++) p0[i] = 32768;
    int pos = 0;
#define NEXT() ((uint32_t)(pos < nbytes ? in[pos++] : (pos++, 0)))
    uint32_t range = 0xFFFFFFFFu, code = 0;
    for (int i = 0; i < 5; i++) code = (code << 8) | NEXT();
    for (int y = 0; y < h; y++)
        for (int x = 0; x < w; x++) {
            int c = ctx_of(bits, h, w, y, x);
            uint32_t bound = (range >> 16) * p0[c];
            int bit;
            if (code < bound) {
                range = bound;
                bit = 0;
                p0[c] = (uint16_t)(p0[c] + ((65536u - p0[c]) >> ORC_RATE));
            } else {
                code -= bound;
                range -= bound;
                bit = 1;
                p0[c] = (uint16_t)(p0[c] - (p0[c] >> ORC_RATE));
            }
            bits[(size_t)y * w + x] = (uint8_t)bit;
            while (range < (1u << 24)) {
                range <<= 8;
                code = (code << 8) | NEXT();
            }
        }
#undef NEXT
}

static int tile_side(int t, int dim) { return (1 << t) < dim ? (1 << t) : dim; }

int orc_tile_count(int M, int N, int t)
{
    int th = tile_side(t, M), tw = tile_side(t, N);
    return ((M + th - 1) / th) * ((N + tw - 1) / tw);
}

/* copies tile k (raster order of tiles) of a plane out / in */
static void tile_rect(int M, int N, int t, int k, int *y0, int *x0, int *h, int *w)
{
    int th = tile_side(t, M), tw = tile_side(t, N), TN = (N + tw - 1) / tw;
    int ty = k / TN, tx = k % TN;
    *y0 = ty * th; *x0 = tx * tw;
    *h = (M - *y0) < th ? (M - *y0) : th;
    *w = (N - *x0) < tw ? (N - *x0) : tw;
}

/* ===================================================================================
 * Bit helpers for the payload frame and the MSB-plane stream (MSB-first everywhere).
 * =================================================================================== */
static int get_bit(const uint8_t *buf, int64_t k) { return (buf[k >> 3] >> (7 - (k & 7))) & 1; }
static void set_bit(uint8_t *buf, int64_t k, int v)
{
    if (v) buf[k >> 3] |= (uint8_t)(1u << (7 - (k & 7)));
    else buf[k >> 3] &= (uint8_t)~(1u << (7 - (k & 7)));
}

/* bits per redundant pixel and their positions: EMR uses positions 1..b,
 * LMR positions 2..b; returns the value-bit index of the k-th carried bit */
static int carried_bits(int method, int b) { return method == ORC_EMR ? b : b - 1; }
static int carried_bit_index(int method, int k) { return method == ORC_EMR ? 7 - k : 6 - k; }

/* ===================================================================================
 * EMR-RDHEI
 * =================================================================================== */
static int emr_encode(const uint8_t *I, int M, int N, const uint8_t k1[32], uint8_t *E, int32_t *b_out,
                      int64_t *cap_out)
{
    size_t MN = (size_t)M * N;
    /* step 1: optimal location map generation */
    int64_t zeros[9];
    orc_zero_counts(I, M, N, zeros);
    int b = orc_select_b_emr(zeros);
    uint8_t *l = (uint8_t *)malloc(MN);
    orc_location_map(I, M, N, b, l);
    /* secret key generation: keystream s the size of the image */
    uint8_t *s = (uint8_t *)malloc(MN);
    orc_keystream(k1, 0, MN, s);
    /* steps 2-3: location map rotation and original image rotation */
    uint8_t *Ir = (uint8_t *)malloc(MN);
    memcpy(Ir, I, MN);
    orc_rotate_all(l, M, N, s, emr_emin(M, N), 0);
    orc_rotate_all(Ir, M, N, s, emr_emin(M, N), 0);
    /* step 4: encryption I_e = s XOR I (eq. image_encryption) */
    for (size_t r = 0; r < MN; r++) E[r] = (uint8_t)(s[r] ^ Ir[r]);
    /* step 5: location map embedding into the LSBs of I_e; the receiver learns b
     * from 3 header bits stored where the map is forced to 1 (Q14, safe by monotone safety) */
    l[0] = l[1] = l[2] = 1;
    for (size_t r = 0; r < MN; r++) {
        int bit = r < 3 ? (((b - 2) >> (2 - (int)r)) & 1) : l[r];
        E[r] = (uint8_t)((E[r] & 0xFE) | bit);
    }
    int64_t z = 0;
    for (size_t r = 0; r < MN; r++) z += (l[r] == 0);
    *b_out = b;
    *cap_out = (int64_t)b * z;                         /* capacity counted after forcing (Q14) */
    free(l); free(s); free(Ir);
    return ORC_OK;
}

/* reads b and the rotated map from the LSB plane (Q14) */
static int emr_read_map(const uint8_t *Em, int M, int N, int *b, uint8_t *l)
{
    size_t MN = (size_t)M * N;
    int field = ((Em[0] & 1) << 2) | ((Em[1] & 1) << 1) | (Em[2] & 1);
    if (field > 5) return ORC_E_FORMAT;
    *b = field + 2;
    for (size_t r = 0; r < MN; r++) l[r] = r < 3 ? 1 : (Em[r] & 1);
    return ORC_OK;
}

/* ===================================================================================
 * LMR-RDHEI
 * =================================================================================== */
static int lmr_header_bits(int T, int64_t bytes_eta, int64_t bytes_map, int64_t *K)
{
    *K = 7 + 32 * (int64_t)T + 8 * (bytes_eta + bytes_map);
    return 0;
}

static void put_bits(uint8_t *plane, int64_t *pos, uint32_t v, int nbits)
{
    for (int i = nbits - 1; i >= 0; i--) plane[(*pos)++] = (uint8_t)((v >> i) & 1);
}

/* codes every tile of a plane; sizes[k] = byte length, data concatenated into buf */
static int code_plane(const uint8_t *plane, int M, int N, int t, int *sizes, uint8_t **buf, int64_t *total)
{
    int T = orc_tile_count(M, N, t);
    int tmax = tile_side(t, M) * tile_side(t, N);
    int cap = tmax / 8 + tmax / 64 + 64;              /* >= 1.1 * raw + 64 bytes */
    uint8_t *tilebits = (uint8_t *)malloc((size_t)tmax);
    uint8_t *tmp = (uint8_t *)malloc((size_t)cap);
    *buf = (uint8_t *)malloc((size_t)T * cap);
    *total = 0;
    for (int k = 0; k < T; k++) {
        int y0, x0, h, w;
        tile_rect(M, N, t, k, &y0, &x0, &h, &w);
        for (int y = 0; y < h; y++)
            for (int x = 0; x < w; x++) tilebits[y * w + x] = plane[(size_t)(y0 + y) * N + x0 + x];
        int nb = orc_tile_encode(tilebits, h, w, tmp, cap);
        if (nb < 0 || nb > 65535) { free(tilebits); free(tmp); return -1; }
        sizes[k] = nb;
        memcpy(*buf + *total, tmp, (size_t)nb);
        *total += nb;
    }
    free(tilebits);
    free(tmp);
    return 0;
}

static int lmr_encode(const uint8_t *I, int M, int N, const uint8_t k1[32], int t, int emin_req, uint8_t *E,
                      int32_t *b_out, int64_t *cap_out)
{
    size_t MN = (size_t)M * N;
    if (t < 3 || t > 9) return ORC_E_INVAL;
    int emin = lmr_emin(M, N, emin_req);
    /* (1) location map candidates and first MSB map eta = (I AND 128) mod 127 (eq. MSB_map, Q21) */
    int64_t zeros[9];
    int order[7];
    orc_zero_counts(I, M, N, zeros);
    orc_lmr_candidates(zeros, order);
    uint8_t *eta = (uint8_t *)malloc(MN);
    for (size_t r = 0; r < MN; r++) eta[r] = (uint8_t)((I[r] & 128) % 127);
    /* keystream from K1 and rotation of eta, image */
    uint8_t *s = (uint8_t *)malloc(MN);
    orc_keystream(k1, 0, MN, s);
    uint8_t *Ir = (uint8_t *)malloc(MN);
    memcpy(Ir, I, MN);
    orc_rotate_all(Ir, M, N, s, emin, 0);
    orc_rotate_all(eta, M, N, s, emin, 0);
    /* (2) compression of the rotated eta (fixed) and of the rotated map, walking candidates
     * "until both maps can be sufficiently compressed to fit in the first MSB bit-plane" */
    int T = orc_tile_count(M, N, t);
    int *sz_eta = (int *)malloc(sizeof(int) * T), *sz_map = (int *)malloc(sizeof(int) * T);
    uint8_t *buf_eta = NULL, *buf_map = NULL;
    int64_t tot_eta = 0, tot_map = 0, K = 0;
    int ok_eta = code_plane(eta, M, N, t, sz_eta, &buf_eta, &tot_eta) == 0;
    uint8_t *l = (uint8_t *)malloc(MN);
    int b = 0;
    for (int k = 0; k < 7 && ok_eta; k++) {
        int cb = order[k];
        orc_location_map(I, M, N, cb, l);
        orc_rotate_all(l, M, N, s, emin, 0);
        free(buf_map);
        buf_map = NULL;
        if (code_plane(l, M, N, t, sz_map, &buf_map, &tot_map) != 0) continue;
        lmr_header_bits(T, tot_eta, tot_map, &K);
        if (K <= (int64_t)MN) { b = cb; break; }
    }
    /* (4) encryption of the rotated image (eq. image_encryption) */
    for (size_t r = 0; r < MN; r++) E[r] = (uint8_t)(s[r] ^ Ir[r]);
    int status = ORC_OK;
    if (b == 0) {
        /* bad case: mark the image with the invalid b-field 7 */
        for (int r = 0; r < 3; r++) E[r] |= 0x80;
        *b_out = 0;
        *cap_out = 0;
        status = ORC_E_BADCASE;
    } else {
        /* (5) compressed maps embedding into the first MSB bit-plane (layout Q15) */
        uint8_t *hdr = (uint8_t *)malloc((size_t)K);
        int64_t pos = 0;
        put_bits(hdr, &pos, (uint32_t)(b - 2), 3);
        put_bits(hdr, &pos, (uint32_t)t, 4);
        for (int k = 0; k < T; k++) put_bits(hdr, &pos, (uint32_t)sz_eta[k], 16);
        for (int k = 0; k < T; k++) put_bits(hdr, &pos, (uint32_t)sz_map[k], 16);
        for (int64_t i = 0; i < tot_eta; i++) put_bits(hdr, &pos, buf_eta[i], 8);
        for (int64_t i = 0; i < tot_map; i++) put_bits(hdr, &pos, buf_map[i], 8);
        for (int64_t r = 0; r < K; r++) E[r] = (uint8_t)((E[r] & 0x7F) | (hdr[r] << 7));
        int64_t z = 0;
        for (size_t r = 0; r < MN; r++) z += (l[r] == 0);
        *b_out = b;
        *cap_out = (int64_t)(b - 1) * z;               /* (b-1) bits per redundant pixel */
        free(hdr);
    }
    free(eta); free(s); free(Ir); free(sz_eta); free(sz_map); free(buf_eta); free(buf_map); free(l);
    return status;
}

/* parses the MSB-plane header and decodes the rotated map (want_eta: also eta) */
static int lmr_read_maps(const uint8_t *Em, int M, int N, int t_expected, int *b, uint8_t *l, uint8_t *eta)
{
    int64_t MN = (int64_t)M * N, pos = 0;
#define RD(nb) ({ uint32_t v_ = 0; for (int i_ = 0; i_ < (nb); i_++) v_ = (v_ << 1) | (Em[pos++] >> 7); v_; })
    if (MN < 7) return ORC_E_FORMAT;
    int field = (int)RD(3);
    if (field == 7) return ORC_E_BADCASE;
    int t = (int)RD(4);
    /* t is shared protocol knowledge like the method (reading Q15); the header repeats it */
    if (t < 3 || t > 9 || t != t_expected) return ORC_E_FORMAT;
    int T = orc_tile_count(M, N, t);
    if (7 + 32 * (int64_t)T > MN) return ORC_E_FORMAT;
    int *sz = (int *)malloc(sizeof(int) * 2 * T);
    int64_t total = 0;
    for (int k = 0; k < 2 * T; k++) { sz[k] = (int)RD(16); total += sz[k]; }
    if (7 + 32 * (int64_t)T + 8 * total > MN) { free(sz); return ORC_E_FORMAT; }
    uint8_t *bytes = (uint8_t *)malloc((size_t)total + 1);
    for (int64_t i = 0; i < total; i++) bytes[i] = (uint8_t)RD(8);
#undef RD
    *b = field + 2;
    int tmax = tile_side(t, M) * tile_side(t, N);
    uint8_t *tilebits = (uint8_t *)malloc((size_t)tmax);
    int64_t off = 0;
    for (int plane = 0; plane < 2; plane++) {
        uint8_t *dst = plane == 0 ? eta : l;
        for (int k = 0; k < T; k++) {
            int nb = sz[plane * T + k];
            if (dst) {
                int y0, x0, h, w;
                tile_rect(M, N, t, k, &y0, &x0, &h, &w);
                orc_tile_decode(bytes + off, nb, h, w, tilebits);
                for (int y = 0; y < h; y++)
                    for (int x = 0; x < w; x++) dst[(size_t)(y0 + y) * N + x0 + x] = tilebits[y * w + x];
            }
            off += nb;
        }
    }
    free(tilebits);
    free(bytes);
    free(sz);
    return ORC_OK;
}

/* ===================================================================================
 * The four calls.
 * =================================================================================== */
int orc_encode_s(int method, const uint8_t *I, int M, int N, const uint8_t k1[32], int tile_log2, int lmr_emin_req,
                 uint8_t *E, int32_t *b_out, int64_t *capacity_out)
{
    if (M < 4 || N < 4) return ORC_E_INVAL;
    if (method == ORC_EMR) return emr_encode(I, M, N, k1, E, b_out, capacity_out);
    if (method == ORC_LMR) return lmr_encode(I, M, N, k1, tile_log2, lmr_emin_req, E, b_out, capacity_out);
    return ORC_E_INVAL;
}

int orc_encode(int method, const uint8_t *I, int M, int N, const uint8_t k1[32], int tile_log2, uint8_t *E,
               int32_t *b_out, int64_t *capacity_out)
{
    return orc_encode_s(method, I, M, N, k1, tile_log2, 0, E, b_out, capacity_out);
}

static int read_map(int method, const uint8_t *Em, int M, int N, int t, int *b, uint8_t *l, uint8_t *eta)
{
    if (method == ORC_EMR) return emr_read_map(Em, M, N, b, l);
    return lmr_read_maps(Em, M, N, t, b, l, eta);
}

int orc_capacity(int method, const uint8_t *marked, int M, int N, int tile_log2, int32_t *b_out, int64_t *capacity_out)
{
    size_t MN = (size_t)M * N;
    uint8_t *l = (uint8_t *)malloc(MN);
    int b = 0;
    int st = read_map(method, marked, M, N, tile_log2, &b, l, NULL);
    int64_t z = 0;
    if (st == ORC_OK)
        for (size_t r = 0; r < MN; r++) z += (l[r] == 0);
    *b_out = st == ORC_OK ? b : 0;
    *capacity_out = st == ORC_OK ? (int64_t)carried_bits(method, b) * z : 0;
    free(l);
    return st;
}

/* data hiding (EMR P:749-750; LMR P:990-991): frame F = BE32(n) || msg (Q17), encrypted with
 * the K2 keystream, written b (EMR) or b-1 (LMR) bits per redundant pixel in raster order of
 * the rotated domain, MSB first (Q18); unused capacity is left untouched (Q19). */
int orc_hide(int method, const uint8_t *E, int M, int N, int tile_log2, const uint8_t k2[32], const uint8_t *msg,
             int64_t msg_bits, uint8_t *marked)
{
    size_t MN = (size_t)M * N;
    memcpy(marked, E, MN);
    uint8_t *l = (uint8_t *)malloc(MN);
    int b = 0;
    int st = read_map(method, E, M, N, tile_log2, &b, l, NULL);
    if (st != ORC_OK) { free(l); return st; }
    int bp = carried_bits(method, b);
    int64_t z = 0;
    for (size_t r = 0; r < MN; r++) z += (l[r] == 0);
    int64_t C = (int64_t)bp * z;
    if (msg_bits < 0 || 32 + msg_bits > C) { free(l); return ORC_E_CAPACITY; }
    int64_t F = 32 + msg_bits;
    uint8_t *ks = (uint8_t *)malloc((size_t)((F + 7) / 8));
    orc_keystream(k2, 0, (uint64_t)((F + 7) / 8), ks);
    int64_t k = 0;                                   /* next frame bit */
    for (size_t r = 0; r < MN && k < F; r++) {
        if (l[r] != 0) continue;
        for (int i = 0; i < bp && k < F; i++, k++) {
            int fbit = k < 32 ? (int)((msg_bits >> (31 - k)) & 1) : get_bit(msg, k - 32);
            int ebit = fbit ^ get_bit(ks, k);
            int vb = carried_bit_index(method, i);
            marked[r] = (uint8_t)((marked[r] & ~(1u << vb)) | ((unsigned)ebit << vb));
        }
    }
    free(ks);
    free(l);
    return ORC_OK;
}

/* extraction with K2 only, no de-rotation (EMR P:839-840; LMR P:1063-1064).
 * Output: the first ceil(max(C-32,0)/32) 32-bit words (4-byte units) of msg_out hold the
 * message bits [0,n) followed by zeros; bytes after that region are untouched. */
int orc_extract(int method, const uint8_t *marked, int M, int N, int tile_log2, const uint8_t k2[32],
                uint8_t *msg_out, int64_t stride_bytes, int64_t *msg_bits_out)
{
    size_t MN = (size_t)M * N;
    uint8_t *l = (uint8_t *)malloc(MN);
    int b = 0;
    *msg_bits_out = -1;
    int st = read_map(method, marked, M, N, tile_log2, &b, l, NULL);
    if (st != ORC_OK) { free(l); return st; }
    int bp = carried_bits(method, b);
    int64_t z = 0;
    for (size_t r = 0; r < MN; r++) z += (l[r] == 0);
    int64_t C = (int64_t)bp * z;
    int64_t region = C > 32 ? 4 * ((C - 32 + 31) / 32) : 0;
    if (region > stride_bytes) { free(l); return ORC_E_INVAL; }
    memset(msg_out, 0, (size_t)region);
    /* G: concatenated carried bits of the redundant pixels, D = G XOR KS2 */
    uint8_t *G = (uint8_t *)calloc((size_t)(C + 7) / 8 + 1, 1);
    int64_t k = 0;
    for (size_t r = 0; r < MN; r++) {
        if (l[r] != 0) continue;
        for (int i = 0; i < bp; i++, k++) set_bit(G, k, (marked[r] >> carried_bit_index(method, i)) & 1);
    }
    uint8_t *ks = (uint8_t *)malloc((size_t)(C + 7) / 8 + 1);
    orc_keystream(k2, 0, (uint64_t)(C + 7) / 8, ks);
    for (int64_t i = 0; i < (C + 7) / 8; i++) G[i] ^= ks[i];
    int status = ORC_OK;
    if (C < 32) {
        status = ORC_E_INTEGRITY;
    } else {
        int64_t n = 0;
        for (int i = 0; i < 32; i++) n = (n << 1) | get_bit(G, i);
        if (n > C - 32) {
            status = ORC_E_INTEGRITY;
        } else {
            for (int64_t i = 0; i < n; i++) set_bit(msg_out, i, get_bit(G, 32 + i));
            *msg_bits_out = n;
        }
    }
    free(G);
    free(ks);
    free(l);
    return status;
}

/* image recovery with K1 only (EMR P:819-837; LMR P:1060-1061): decrypt all bits (Q20),
 * restore the MSB plane from eta (LMR), de-rotate image and map(s), then restore the b MSBs
 * (EMR) or bits 2..b (LMR) row by row from omega = the last non-redundant pixel. */
int orc_recover(int method, const uint8_t *marked, int M, int N, int tile_log2, const uint8_t k1[32], uint8_t *out)
{
    return orc_recover_s(method, marked, M, N, tile_log2, 0, k1, out);
}

int orc_recover_s(int method, const uint8_t *marked, int M, int N, int tile_log2, int lmr_emin_req, const uint8_t k1[32],
                  uint8_t *out)
{
    size_t MN = (size_t)M * N;
    uint8_t *l = (uint8_t *)malloc(MN), *eta = (uint8_t *)malloc(MN);
    int b = 0;
    int st = read_map(method, marked, M, N, tile_log2, &b, l, method == ORC_LMR ? eta : NULL);
    if (st != ORC_OK) {
        memset(out, 0, MN);
        free(l); free(eta);
        return st;
    }
    uint8_t *s = (uint8_t *)malloc(MN);
    orc_keystream(k1, 0, MN, s);
    for (size_t r = 0; r < MN; r++) out[r] = (uint8_t)(marked[r] ^ s[r]);
    int emin = method == ORC_EMR ? emr_emin(M, N) : lmr_emin(M, N, lmr_emin_req);
    orc_rotate_all(out, M, N, s, emin, 1);
    orc_rotate_all(l, M, N, s, emin, 1);
    if (method == ORC_LMR) {
        /* "the decompressed de-rotated eta is used to recover the original first MSB bit-plane" */
        orc_rotate_all(eta, M, N, s, emin, 1);
        for (size_t r = 0; r < MN; r++) out[r] = (uint8_t)((out[r] & 0x7F) | (eta[r] << 7));
    }
    int mask = method == ORC_EMR ? (0xFF & ~(0xFF >> b)) : (0x7F & ~(0xFF >> b));
    for (int i = 0; i < M; i++) {
        int omega = out[(size_t)i * N] & mask;
        for (int j = 1; j < N; j++) {
            size_t r = (size_t)i * N + j;
            if (l[r]) omega = out[r] & mask;
            else out[r] = (uint8_t)((out[r] & ~mask) | omega);
        }
    }
    free(s); free(l); free(eta);
    return ORC_OK;
}

/* ===================================================================================
 * Statistics: DER = C / MN, PSNR = 10 log10(255^2 / MSE), +inf if equal.
 * =================================================================================== */
int64_t orc_sse(const uint8_t *a, const uint8_t *b, int64_t n)
{
    int64_t s = 0;
    for (int64_t i = 0; i < n; i++) {
        int64_t d = (int64_t)a[i] - (int64_t)b[i];
        s += d * d;
    }
    return s;
}

void orc_der_psnr(int M, int N, int64_t capacity_bits, int64_t sse, double *der, double *psnr)
{
    double MN = (double)M * (double)N;
    *der = (double)capacity_bits / MN;
    *psnr = sse == 0 ? INFINITY : 10.0 * log10(255.0 * 255.0 * MN / (double)sse);
}

/* ===================================================================================
 * Security / quality statistics (P:1437-1467 Shannon entropy, chi^2, NPCR, UACI; SSIM
 * P:1071, P:1235 with the window of S:524).  Plain definitions, fp64.
 * =================================================================================== */
static void histogram(const uint8_t *img, int64_t n, int64_t h[256])
{
    for (int i = 0; i < 256; i++) h[i] = 0;
    for (int64_t k = 0; k < n; k++) h[img[k]]++;
}

double orc_entropy(const uint8_t *img, int64_t n)
{
    int64_t h[256];
    histogram(img, n, h);
    double H = 0.0;
    for (int i = 0; i < 256; i++) {
        if (h[i] == 0) continue;                       /* 0 log 0 = 0 */
        double P = (double)h[i] / (double)n;
        H -= P * log2(P);
    }
    return H;
}

double orc_chi2(const uint8_t *img, int64_t n)
{
    int64_t h[256];
    histogram(img, n, h);
    double s = 0.0;
    for (int i = 0; i < 256; i++) {
        double d = (double)h[i] / (double)n - 1.0 / 256.0;
        s += d * d;
    }
    return 256.0 * (double)n * s;
}

void orc_npcr_uaci(const uint8_t *a, const uint8_t *b, int64_t n, double *npcr, double *uaci)
{
    int64_t diff = 0, absum = 0;
    for (int64_t k = 0; k < n; k++) {
        if (a[k] != b[k]) diff++;
        absum += a[k] > b[k] ? a[k] - b[k] : b[k] - a[k];
    }
    *npcr = 100.0 * (double)diff / (double)n;
    *uaci = 100.0 * (double)absum / (255.0 * (double)n);
}

double orc_ssim(const uint8_t *a, const uint8_t *b, int M, int N)
{
    const double C1 = (0.01 * 255.0) * (0.01 * 255.0), C2 = (0.03 * 255.0) * (0.03 * 255.0);
    double w[11][11], tot = 0.0;
    for (int i = 0; i < 11; i++)
        for (int j = 0; j < 11; j++) {
            w[i][j] = exp(-((i - 5) * (i - 5) + (j - 5) * (j - 5)) / (2.0 * 1.5 * 1.5));
            tot += w[i][j];
        }
    for (int i = 0; i < 11; i++)
        for (int j = 0; j < 11; j++) w[i][j] /= tot;
    if (M < 11 || N < 11) return 0.0;
    double sum = 0.0;
    for (int y = 0; y + 11 <= M; y++)
        for (int x = 0; x + 11 <= N; x++) {
            double ma = 0, mb = 0, saa = 0, sbb = 0, sab = 0;
            for (int i = 0; i < 11; i++)
                for (int j = 0; j < 11; j++) {
                    double va = a[(size_t)(y + i) * N + x + j], vb = b[(size_t)(y + i) * N + x + j];
                    ma += w[i][j] * va;
                    mb += w[i][j] * vb;
                    saa += w[i][j] * va * va;
                    sbb += w[i][j] * vb * vb;
                    sab += w[i][j] * va * vb;
                }
            double va2 = saa - ma * ma, vb2 = sbb - mb * mb, cov = sab - ma * mb;
            sum += ((2 * ma * mb + C1) * (2 * cov + C2)) / ((ma * ma + mb * mb + C1) * (va2 + vb2 + C2));
        }
    return sum / ((double)(M - 10) * (double)(N - 10));
}
