// mmsb_api.cu -- host orchestration behind the C ABI of include/mmsb.h:
// validation, workspace carving, L2-sized image groups, launch sequencing.
// No allocation, no synchronisation: every call is stream-ordered on the caller's stream.
#include <atomic>
#include <cmath>
#include <cstring>

#include "mmsb.h"
#include "mmsb_geo.h"
#include "mmsb_kernels.h"

namespace mmsb {

static std::atomic<unsigned long long> g_launches{0};

// Images per tile-kernel group: the group's keystream scratch (1 B/px), its images and
// their outputs are meant to stay in the 126 MB L2 between the keystream kernel and the
// permutation kernel that consumes them.
constexpr long long kGroupBytes = 24ll << 20;

static size_t align256(size_t v) { return (v + 255) & ~(size_t)255; }

struct Layout {
    int G;
    size_t s, rec, pyr, hist, tile_zero_end;                 // per-group tile state
    size_t ticket, states, done, parts, hdr, scan_zero_end;  // per-call scan state
    size_t ceta, eta_bits, map_bits, lmr_b, total;
};

static Layout layout(const Geo &g) {
    Layout L{};
    long long G = kGroupBytes / g.HW;
    if (G < 1) G = 1;
    if (G > g.B) G = g.B;
    L.G = (int)G;
    size_t o = 0;
    L.s = o; o = align256(o + (size_t)G * g.HW);
    L.rec = o; o = align256(o + (size_t)G * g.ntiles * kRecSlots * 8);
    L.pyr = o; o = align256(o + (size_t)G * (g.npyr > 0 ? g.npyr : 1) * 4);
    L.hist = o; o = align256(o + (size_t)G * 8 * 4);
    L.tile_zero_end = o;
    L.ticket = o; o = align256(o + 16);
    L.states = o; o = align256(o + (size_t)g.B * g.nchunks * 8);
    L.done = o; o = align256(o + (size_t)g.B * 4);
    L.parts = o; o = align256(o + (size_t)g.B * g.nchunks * 16);
    L.hdr = o; o = align256(o + (size_t)g.B * 4);
    L.scan_zero_end = o;
    L.ceta = o; o = align256(o + (g.method == 1 ? (size_t)G * g.HW : 0));
    L.eta_bits = o; o = align256(o + (g.method == 1 ? (size_t)g.B * g.HW / 8 : 0));
    L.map_bits = o; o = align256(o + (g.method == 1 ? (size_t)g.B * g.HW / 8 : 0));
    L.lmr_b = o; o = align256(o + (size_t)g.B * 4);
    L.total = o;
    return L;
}

static bool geo_of(const mmsb_shape *s, Geo *g) {
    if (!s) return false;
    return make_geo(s->method, s->batch, s->height, s->width, s->tile_log2, g);
}

static mmsb_status check_launch() {
    return cudaGetLastError() == cudaSuccess ? MMSB_OK : MMSB_E_CUDA;
}

template <class T> static T *at(void *ws, size_t off) { return reinterpret_cast<T *>(static_cast<char *>(ws) + off); }

}  // namespace mmsb

using namespace mmsb;

extern "C" {

size_t mmsb_workspace_bytes(const mmsb_shape *shape) {
    Geo g;
    if (!geo_of(shape, &g)) return 0;
    return layout(g).total;
}

mmsb_status mmsb_content_owner_encode(const mmsb_shape *shape, const uint8_t *images, const uint8_t *k1,
                                      uint8_t *encrypted, int32_t *b_out, int64_t *capacity_out,
                                      int32_t *img_status, void *ws, size_t ws_bytes, void *stream) {
    Geo g;
    if (!geo_of(shape, &g) || !images || !k1 || !encrypted || !b_out || !capacity_out || !img_status || !ws)
        return MMSB_E_INVAL;
    const Layout L = layout(g);
    if (ws_bytes < L.total) return MMSB_E_INVAL;
    if (g.method != 0) return MMSB_E_UNIMPLEMENTED;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    for (int g0 = 0; g0 < g.B; g0 += L.G) {
        const int n = g.B - g0 < L.G ? g.B - g0 : L.G;
        if (cudaMemsetAsync(at<char>(ws, L.pyr), 0, L.tile_zero_end - L.pyr, st) != cudaSuccess) return MMSB_E_CUDA;
        launch_ks_tile(g, n, k1 + (size_t)g0 * 32, images + (size_t)g0 * g.HW, at<uint8_t>(ws, L.s),
                       at<uint64_t>(ws, L.rec), at<uint32_t>(ws, L.pyr), at<uint32_t>(ws, L.hist), st);
        launch_perm_encode(g, n, images + (size_t)g0 * g.HW, at<uint8_t>(ws, L.s), at<uint64_t>(ws, L.rec),
                           at<uint32_t>(ws, L.pyr), at<uint32_t>(ws, L.hist), encrypted + (size_t)g0 * g.HW,
                           at<uint8_t>(ws, L.ceta), b_out + g0, capacity_out + g0, img_status + g0, st);
        g_launches += 2;
    }
    return check_launch();
}

mmsb_status mmsb_hider_embed(const mmsb_shape *shape, const uint8_t *encrypted, const uint8_t *k2,
                             const uint8_t *msg_bytes, const int64_t *msg_bits, int64_t stride_bytes,
                             uint8_t *marked, int32_t *img_status, void *ws, size_t ws_bytes, void *stream) {
    Geo g;
    if (!geo_of(shape, &g) || !encrypted || !k2 || !msg_bytes || !msg_bits || !marked || !img_status || !ws)
        return MMSB_E_INVAL;
    if (stride_bytes <= 0 || stride_bytes % 16 || marked == encrypted) return MMSB_E_INVAL;
    const Layout L = layout(g);
    if (ws_bytes < L.total) return MMSB_E_INVAL;
    if (g.method != 0) return MMSB_E_UNIMPLEMENTED;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (cudaMemsetAsync(at<char>(ws, L.ticket), 0, L.scan_zero_end - L.ticket, st) != cudaSuccess) return MMSB_E_CUDA;
    ScanWS sw{at<unsigned int>(ws, L.ticket), at<unsigned long long>(ws, L.states), at<unsigned int>(ws, L.done),
              at<unsigned long long>(ws, L.parts), at<uint32_t>(ws, L.hdr)};
    launch_scan(g, true, encrypted, marked, k2, msg_bytes, msg_bits, stride_bytes, nullptr, nullptr, img_status, sw,
                at<uint32_t>(ws, L.map_bits), at<int32_t>(ws, L.lmr_b), st);
    g_launches += 1;
    return check_launch();
}

mmsb_status mmsb_receiver_extract(const mmsb_shape *shape, const uint8_t *marked, const uint8_t *k2,
                                  uint8_t *msg_out, int64_t stride_bytes, int64_t *msg_bits_out,
                                  int32_t *img_status, void *ws, size_t ws_bytes, void *stream) {
    Geo g;
    if (!geo_of(shape, &g) || !marked || !k2 || !msg_out || !msg_bits_out || !img_status || !ws)
        return MMSB_E_INVAL;
    // every capacity (<= 7 bits per pixel) must fit the caller's rows
    if (stride_bytes <= 0 || stride_bytes % 16 || stride_bytes < (7 * g.HW + 7) / 8) return MMSB_E_INVAL;
    const Layout L = layout(g);
    if (ws_bytes < L.total) return MMSB_E_INVAL;
    if (g.method != 0) return MMSB_E_UNIMPLEMENTED;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (cudaMemsetAsync(at<char>(ws, L.ticket), 0, L.scan_zero_end - L.ticket, st) != cudaSuccess) return MMSB_E_CUDA;
    ScanWS sw{at<unsigned int>(ws, L.ticket), at<unsigned long long>(ws, L.states), at<unsigned int>(ws, L.done),
              at<unsigned long long>(ws, L.parts), at<uint32_t>(ws, L.hdr)};
    launch_scan(g, false, marked, nullptr, k2, nullptr, nullptr, stride_bytes, msg_out, msg_bits_out, img_status, sw,
                at<uint32_t>(ws, L.map_bits), at<int32_t>(ws, L.lmr_b), st);
    g_launches += 1;
    return check_launch();
}

mmsb_status mmsb_receiver_recover(const mmsb_shape *shape, const uint8_t *marked, const uint8_t *k1,
                                  uint8_t *recovered, int32_t *img_status, void *ws, size_t ws_bytes,
                                  void *stream) {
    Geo g;
    if (!geo_of(shape, &g) || !marked || !k1 || !recovered || !img_status || !ws) return MMSB_E_INVAL;
    const Layout L = layout(g);
    if (ws_bytes < L.total) return MMSB_E_INVAL;
    if (g.method != 0) return MMSB_E_UNIMPLEMENTED;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    for (int g0 = 0; g0 < g.B; g0 += L.G) {
        const int n = g.B - g0 < L.G ? g.B - g0 : L.G;
        if (cudaMemsetAsync(at<char>(ws, L.pyr), 0, L.tile_zero_end - L.pyr, st) != cudaSuccess) return MMSB_E_CUDA;
        launch_ks_tile(g, n, k1 + (size_t)g0 * 32, nullptr, at<uint8_t>(ws, L.s), at<uint64_t>(ws, L.rec),
                       at<uint32_t>(ws, L.pyr), at<uint32_t>(ws, L.hist), st);
        launch_recover_strip(g, n, marked + (size_t)g0 * g.HW, at<uint8_t>(ws, L.s), at<uint64_t>(ws, L.rec),
                             at<uint32_t>(ws, L.pyr), at<uint32_t>(ws, L.eta_bits) + (size_t)g0 * g.HW / 32,
                             at<uint32_t>(ws, L.map_bits) + (size_t)g0 * g.HW / 32, at<int32_t>(ws, L.lmr_b) + g0,
                             recovered + (size_t)g0 * g.HW, img_status + g0, st);
        g_launches += 2;
    }
    return check_launch();
}

mmsb_status mmsb_stats(const mmsb_shape *shape, const uint8_t *original, const uint8_t *recovered,
                       int64_t *sse_out, void *stream) {
    Geo g;
    if (!geo_of(shape, &g) || !original || !recovered || !sse_out) return MMSB_E_INVAL;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (cudaMemsetAsync(sse_out, 0, (size_t)g.B * 8, st) != cudaSuccess) return MMSB_E_CUDA;
    launch_stats(g.HW, g.B, original, recovered, sse_out, st);
    g_launches += 1;
    return check_launch();
}

void mmsb_der_psnr_host(int32_t batch, int32_t height, int32_t width, const int64_t *capacity_bits,
                        const int64_t *sse, double *der_out, double *psnr_out) {
    const double MN = (double)height * (double)width;
    for (int i = 0; i < batch; i++) {
        if (der_out) der_out[i] = (double)capacity_bits[i] / MN;
        if (psnr_out) psnr_out[i] = sse[i] == 0 ? INFINITY : 10.0 * std::log10(65025.0 * MN / (double)sse[i]);
    }
}

const char *mmsb_status_string(mmsb_status s) {
    switch (s) {
        case MMSB_OK: return "ok";
        case MMSB_E_INVAL: return "invalid argument";
        case MMSB_E_CAPACITY: return "message exceeds capacity";
        case MMSB_E_INTEGRITY: return "integrity: decrypted length exceeds capacity";
        case MMSB_E_BADCASE: return "LMR bad case: maps do not fit the MSB plane";
        case MMSB_E_CUDA: return "CUDA launch error";
        case MMSB_E_UNIMPLEMENTED: return "unimplemented";
        case MMSB_E_FORMAT: return "malformed header or stream";
    }
    return "unknown";
}

uint64_t mmsb_kernel_launches(void) { return g_launches.load(); }

}  // extern "C"
