// mmsb_api.cu -- host orchestration behind the C ABI of include/mmsb.h:
// validation, workspace carving, L2-sized image groups, launch sequencing.
// No allocation, no synchronisation: every call is stream-ordered on the caller's stream.
#include <atomic>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <mutex>
#include <vector>

#include "mmsb.h"
#include "mmsb_geo.h"
#include "mmsb_kernels.h"

namespace mmsb {

static std::atomic<unsigned long long> g_launches{0};

// ---- live per-kernel timing (CUDA events recorded on the launch stream around each kernel)
enum KernelId { K_ENCODE = 0, K_RECOVER, K_EMBED, K_EXTRACT, K_STATS, K_LMR_PLAN, K_CODER_ENC, K_LMR_FIT,
                K_LMR_MSB, K_LMR_DECODE, K_RECOVER_SSE, K_COUNT };
static const char *kKernelNames[K_COUNT] = {"encode_kernel", "recover_kernel", "embed_prep+scan_kernel<embed>+finish",
                                            "scan_kernel<extract>+finish", "stats_kernel", "lmr_plan_kernel",
                                            "coder_encode_kernel", "lmr_fit_kernel", "lmr_concat+msb_write_kernels",
                                            "lmr_pack+header+coder_decode_kernels", "recover_kernel+sse"};
struct ProfRec { int id; cudaEvent_t a, b; long long units; };
static std::mutex g_prof_mu;
static bool g_prof_on = false;
static std::vector<ProfRec> g_prof;
static std::vector<cudaEvent_t> g_event_pool;
// profiling: symbols coded / decoded by the tile coder (device counters, read by mmsb_profile_read)
static unsigned long long *g_sym = nullptr;
static unsigned long long *sym_counter(int which) {   // (called inside run_kernel, which holds g_prof_mu)
    return g_prof_on && g_sym ? g_sym + which : nullptr;
}

static cudaEvent_t prof_event() {
    if (!g_event_pool.empty()) { cudaEvent_t e = g_event_pool.back(); g_event_pool.pop_back(); return e; }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

// runs `launch` (one kernel) and, when profiling, brackets it with events; `units` = pixels it processes
template <class F> static void run_kernel(int id, cudaStream_t st, long long units, F &&launch, int nkernels = 1) {
    std::unique_lock<std::mutex> lk(g_prof_mu);
    g_launches += nkernels;
    if (!g_prof_on) {
        lk.unlock();
        launch();
        return;
    }
    ProfRec r{id, prof_event(), prof_event(), units};
    cudaEventRecord(r.a, st);
    launch();
    cudaEventRecord(r.b, st);
    g_prof.push_back(r);
}

static size_t align256(size_t v) { return (v + 255) & ~(size_t)255; }

// Workspace carving.  The keystream scratch and angle records are sized for
// the whole batch but are transient: each tile is written by one keystream CTA, read by one
// worker CTA of the same launch shortly after, and then discarded from L2.
struct Layout {
    size_t s, rec, pyr, hist, kdone, tile_zero_end;                          // fused tile kernels
    size_t states, parts, hdr, ztot, err, scan_zero_end, ef, counts;           // scan kernels
    size_t ceta, eta_bits, map_bits, lmr_b, lmr_t, plan, wctl, lists, mapbytes, streams, sizes, dsizes, offsets, mbuf, rstat, total;
};

static Layout layout(const Geo &g) {
    Layout L{};
    const size_t B = (size_t)g.B, nt = (size_t)g.ntiles;
    size_t o = 0;
    L.s = o; o = align256(o + 3 * B * g.HW);                // per tile: keystream | image | label planes
    L.rec = o; o = align256(o + B * nt * kRecSlots * 8);
    L.pyr = o; o = align256(o + B * (g.npyr > 0 ? g.npyr : 1) * 4);
    L.hist = o; o = align256(o + B * kHistStride * 4);
    L.kdone = o; o = align256(o + B * 4);
    L.tile_zero_end = o;
    L.states = o; o = align256(o + B * g.nchunks * 8);
    L.parts = o; o = align256(o + B * g.nchunks * 16);
    L.hdr = o; o = align256(o + B * 4);
    L.ztot = o; o = align256(o + B * 8);
    L.err = o; o = align256(o + B * 4);
    L.scan_zero_end = o;
    L.ef = o; o = align256(o + B * (size_t)ef_words_of(g.HW) * 4);
    L.counts = o; o = align256(o + B * g.nchunks * 4);
    const bool lmr = g.method == 1;
    L.ceta = o; o = align256(o + (lmr ? B * g.HW : 0));
    L.eta_bits = o; o = align256(o + (lmr ? B * g.HW / 8 : 0));
    L.map_bits = o; o = align256(o + (lmr ? B * g.HW / 8 : 0));
    L.lmr_b = o; o = align256(o + B * 4);
    L.lmr_t = o; o = align256(o + B * 4);
    const size_t Tc = (size_t)g.ntiles_coder;
    L.plan = o; o = align256(o + (lmr ? B * sizeof(LmrPlan) : 0));
    L.wctl = o; o = align256(o + (lmr ? sizeof(LmrWaveCtl) : 0));
    L.lists = o; o = align256(o + (lmr ? 8 * B * 4 : 0));
    L.mapbytes = o; o = align256(o + (lmr ? (size_t)kMapStats * B * 4 : 0));
    L.streams = o; o = align256(o + (lmr ? B * kLmrSlots * Tc * lmr_tile_stride_host(g.tile_log2, g.H, g.W) : 0));
    L.sizes = o; o = align256(o + (lmr ? B * kLmrSlots * Tc * 4 : 0));
    L.dsizes = o; o = align256(o + (lmr ? B * 2 * Tc * 4 : 0));
    L.offsets = o; o = align256(o + (lmr ? B * 2 * Tc * 4 : 0));
    L.mbuf = o; o = align256(o + (lmr ? B * g.HW / 8 + 128 : 0));   // + decoder look-ahead past the last stream
    L.rstat = o; o = align256(o + B * 4);
    L.total = o;
    return L;
}

static ScanWS scan_ws(const Geo &g, const Layout &L, void *ws) {
    char *w = static_cast<char *>(ws);
    return ScanWS{reinterpret_cast<unsigned long long *>(w + L.states), reinterpret_cast<unsigned long long *>(w + L.parts),
                  reinterpret_cast<uint32_t *>(w + L.hdr), reinterpret_cast<uint32_t *>(w + L.ef), ef_words_of(g.HW),
                  reinterpret_cast<uint32_t *>(w + L.counts), reinterpret_cast<unsigned long long *>(w + L.ztot),
                  reinterpret_cast<uint32_t *>(w + L.err)};
}

static TileWS tile_ws(const Layout &L, void *ws) {
    char *w = static_cast<char *>(ws);
    TileWS t;
    t.s = reinterpret_cast<uint8_t *>(w + L.s);
    t.rec = reinterpret_cast<uint64_t *>(w + L.rec);
    t.pyr = reinterpret_cast<uint32_t *>(w + L.pyr);
    t.hist = reinterpret_cast<uint32_t *>(w + L.hist);
    t.kdone = reinterpret_cast<uint32_t *>(w + L.kdone);
    return t;
}

static bool geo_of(const mmsb_shape *s, Geo *g) {
    if (!s) return false;
    return make_geo(s->method, s->batch, s->height, s->width, s->tile_log2, s->lmr_emin, g, s->cipher_rounds);
}

static mmsb_status check_launch() {
    return cudaGetLastError() == cudaSuccess ? MMSB_OK : MMSB_E_CUDA;
}

template <class T> static T *at(void *ws, size_t off) { return reinterpret_cast<T *>(static_cast<char *>(ws) + off); }

// LMR receiving side: MSB plane -> header -> decoded rotated map (and eta) planes
static void lmr_decode_all(const Geo &g, const Layout &L, bool want_eta, const uint8_t *marked, void *ws,
                           int32_t *img_status, int64_t *msg_bits_out, cudaStream_t st) {
    const int tw = (1 << g.tile_log2) < g.W ? (1 << g.tile_log2) : g.W;
    if (tw % 32) {   // tiles narrower than a word share words: the decoder ORs into zeroed planes
        cudaMemsetAsync(at<char>(ws, L.map_bits), 0, (size_t)g.B * g.HW / 8, st);
        if (want_eta) cudaMemsetAsync(at<char>(ws, L.eta_bits), 0, (size_t)g.B * g.HW / 8, st);
    }
    run_kernel(K_LMR_DECODE, st, (long long)g.B * g.HW, [&] {
        launch_lmr_decode(g, want_eta, marked, at<uint8_t>(ws, L.mbuf), at<int32_t>(ws, L.lmr_b),
                          at<int32_t>(ws, L.lmr_t), at<int32_t>(ws, L.offsets), at<int32_t>(ws, L.sizes),
                          at<uint32_t>(ws, L.eta_bits), at<uint32_t>(ws, L.map_bits), img_status, msg_bits_out,
                          sym_counter(1), st);
    }, 3);
}

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
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (cudaMemsetAsync(at<char>(ws, L.pyr), 0, L.tile_zero_end - L.pyr, st) != cudaSuccess) return MMSB_E_CUDA;
    const long long px = (long long)g.B * g.HW;
    run_kernel(K_ENCODE, st, px, [&] {
        launch_encode(g, images, k1, tile_ws(L, ws), encrypted, at<uint8_t>(ws, L.ceta), b_out, capacity_out,
                      img_status, st);
    });
    if (g.method == 1) {
        // LMR: code eta and the candidate maps until both fit the MSB plane, then write it
        const LmrEncWS ew{at<LmrPlan>(ws, L.plan), at<LmrWaveCtl>(ws, L.wctl), at<int32_t>(ws, L.lists),
                          at<uint8_t>(ws, L.streams), at<int32_t>(ws, L.sizes), at<int32_t>(ws, L.dsizes),
                          at<int32_t>(ws, L.offsets), at<uint8_t>(ws, L.mbuf), at<int32_t>(ws, L.mapbytes)};
        run_kernel(K_LMR_PLAN, st, px, [&] { launch_lmr_plan(g, at<uint32_t>(ws, L.hist), ew, st); });
        for (int w = 0; w < 7; w++) {      // candidate waves; waves after the last undecided image exit at once
            run_kernel(K_CODER_ENC, st, px, [&] {
                launch_coder_encode(g, w, at<uint8_t>(ws, L.ceta), ew, sym_counter(0), st);
            });
            run_kernel(K_LMR_FIT, st, px, [&] { launch_lmr_fit(g, w, ew, st); });
        }
        run_kernel(K_LMR_MSB, st, px, [&] {
            launch_lmr_msb_write(g, ew, at<uint32_t>(ws, L.hist), encrypted, b_out, capacity_out, img_status, st);
        }, 2);
    }
    return check_launch();
}

mmsb_status mmsb_hider_embed(const mmsb_shape *shape, const uint8_t *encrypted, const uint8_t *k2,
                             const uint8_t *msg_bytes, const int64_t *msg_bits, int64_t stride_bytes,
                             uint8_t *marked, int32_t *img_status, void *ws, size_t ws_bytes, void *stream) {
    Geo g;
    if (!geo_of(shape, &g) || !encrypted || !k2 || !msg_bytes || !msg_bits || !marked || !img_status || !ws)
        return MMSB_E_INVAL;
    if (stride_bytes <= 0 || stride_bytes % 16) return MMSB_E_INVAL;      // (marked may alias encrypted)
    const Layout L = layout(g);
    if (ws_bytes < L.total) return MMSB_E_INVAL;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (cudaMemsetAsync(at<char>(ws, L.states), 0, L.scan_zero_end - L.states, st) != cudaSuccess) return MMSB_E_CUDA;
    if (g.method == 1) lmr_decode_all(g, L, false, encrypted, ws, img_status, nullptr, st);
    const ScanWS sw = scan_ws(g, L, ws);
    run_kernel(K_EMBED, st, (long long)g.B * g.HW, [&] {
        launch_scan(g, true, encrypted, marked, k2, msg_bytes, msg_bits, stride_bytes, nullptr, nullptr, img_status,
                    sw, at<uint32_t>(ws, L.map_bits), at<int32_t>(ws, L.lmr_b), st);
    }, 3);
    return check_launch();
}

mmsb_status mmsb_receiver_extract(const mmsb_shape *shape, const uint8_t *marked, const uint8_t *k2,
                                  uint8_t *msg_out, int64_t stride_bytes, int64_t *msg_bits_out,
                                  int32_t *img_status, void *ws, size_t ws_bytes, void *stream) {
    Geo g;
    if (!geo_of(shape, &g) || !marked || !k2 || !msg_out || !msg_bits_out || !img_status || !ws)
        return MMSB_E_INVAL;
    // a capacity region larger than the caller's rows is reported per image (E_INVAL status)
    if (stride_bytes <= 0 || stride_bytes % 16) return MMSB_E_INVAL;
    const Layout L = layout(g);
    if (ws_bytes < L.total) return MMSB_E_INVAL;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (cudaMemsetAsync(at<char>(ws, L.states), 0, L.scan_zero_end - L.states, st) != cudaSuccess) return MMSB_E_CUDA;
    if (g.method == 1) lmr_decode_all(g, L, false, marked, ws, img_status, msg_bits_out, st);
    const ScanWS sw = scan_ws(g, L, ws);
    run_kernel(K_EXTRACT, st, (long long)g.B * g.HW, [&] {
        launch_scan(g, false, marked, nullptr, k2, nullptr, nullptr, stride_bytes, msg_out, msg_bits_out,
                    img_status, sw, at<uint32_t>(ws, L.map_bits), at<int32_t>(ws, L.lmr_b), st);
    }, 2);
    return check_launch();
}

mmsb_status mmsb_receiver_recover(const mmsb_shape *shape, const uint8_t *marked, const uint8_t *k1,
                                  uint8_t *recovered, int32_t *img_status, void *ws, size_t ws_bytes,
                                  void *stream) {
    Geo g;
    if (!geo_of(shape, &g) || !marked || !k1 || !recovered || !img_status || !ws) return MMSB_E_INVAL;
    const Layout L = layout(g);
    if (ws_bytes < L.total) return MMSB_E_INVAL;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (g.method == 1) lmr_decode_all(g, L, true, marked, ws, img_status, nullptr, st);
    if (cudaMemsetAsync(at<char>(ws, L.pyr), 0, L.tile_zero_end - L.pyr, st) != cudaSuccess) return MMSB_E_CUDA;
    run_kernel(K_RECOVER, st, (long long)g.B * g.HW, [&] {
        launch_recover(g, marked, k1, tile_ws(L, ws), at<uint32_t>(ws, L.eta_bits), at<uint32_t>(ws, L.map_bits),
                       at<int32_t>(ws, L.lmr_b), recovered, img_status, st);
    });
    return check_launch();
}

mmsb_status mmsb_receiver_recover_sse(const mmsb_shape *shape, const uint8_t *marked, const uint8_t *k1,
                                      const uint8_t *original, uint8_t *recovered, int64_t *sse_out,
                                      int32_t *img_status, void *ws, size_t ws_bytes, void *stream) {
    Geo g;
    if (!geo_of(shape, &g) || !marked || !k1 || !original || !recovered || !sse_out || !img_status || !ws)
        return MMSB_E_INVAL;
    const Layout L = layout(g);
    if (ws_bytes < L.total) return MMSB_E_INVAL;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (g.method == 1) lmr_decode_all(g, L, true, marked, ws, img_status, nullptr, st);
    if (cudaMemsetAsync(at<char>(ws, L.pyr), 0, L.tile_zero_end - L.pyr, st) != cudaSuccess) return MMSB_E_CUDA;
    if (cudaMemsetAsync(sse_out, 0, (size_t)g.B * 8, st) != cudaSuccess) return MMSB_E_CUDA;
    run_kernel(K_RECOVER_SSE, st, (long long)g.B * g.HW, [&] {
        launch_recover(g, marked, k1, tile_ws(L, ws), at<uint32_t>(ws, L.eta_bits), at<uint32_t>(ws, L.map_bits),
                       at<int32_t>(ws, L.lmr_b), recovered, img_status, st, original,
                       reinterpret_cast<unsigned long long *>(sse_out));
    });
    return check_launch();
}

mmsb_status mmsb_receiver_both(const mmsb_shape *shape, const uint8_t *marked, const uint8_t *k1, const uint8_t *k2,
                               uint8_t *msg_out, int64_t stride_bytes, int64_t *msg_bits_out, uint8_t *recovered,
                               int32_t *img_status, void *ws, size_t ws_bytes, void *stream) {
    Geo g;
    if (!geo_of(shape, &g) || !marked || !k1 || !k2 || !msg_out || !msg_bits_out || !recovered || !img_status || !ws)
        return MMSB_E_INVAL;
    if (stride_bytes <= 0 || stride_bytes % 16) return MMSB_E_INVAL;
    const Layout L = layout(g);
    if (ws_bytes < L.total) return MMSB_E_INVAL;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    int32_t *rstat = at<int32_t>(ws, L.rstat);
    if (cudaMemsetAsync(at<char>(ws, L.states), 0, L.scan_zero_end - L.states, st) != cudaSuccess) return MMSB_E_CUDA;
    if (cudaMemsetAsync(rstat, 0, (size_t)g.B * 4, st) != cudaSuccess) return MMSB_E_CUDA;
    // LMR: the coded maps (eta and the location map) are decoded once for both parties' steps
    if (g.method == 1) lmr_decode_all(g, L, true, marked, ws, img_status, msg_bits_out, st);
    if (cudaMemsetAsync(at<char>(ws, L.pyr), 0, L.tile_zero_end - L.pyr, st) != cudaSuccess) return MMSB_E_CUDA;
    const ScanWS sw = scan_ws(g, L, ws);
    // the two receivers back to back (LMR: on the maps decoded once above).  Tried and not kept: one
    // launch with the extraction's chunk CTAs as a third CTA role beside the recovery's keystream
    // and worker CTAs (EMR config 2: 0.81 ms against 0.70 ms back to back; the three ALU-bound
    // roles' code overflows the instruction cache)
    run_kernel(K_EXTRACT, st, (long long)g.B * g.HW, [&] {
        launch_scan(g, false, marked, nullptr, k2, nullptr, nullptr, stride_bytes, msg_out, msg_bits_out,
                    img_status, sw, at<uint32_t>(ws, L.map_bits), at<int32_t>(ws, L.lmr_b), st);
    }, 2);
    run_kernel(K_RECOVER, st, (long long)g.B * g.HW, [&] {
        launch_recover(g, marked, k1, tile_ws(L, ws), at<uint32_t>(ws, L.eta_bits), at<uint32_t>(ws, L.map_bits),
                       at<int32_t>(ws, L.lmr_b), recovered, rstat, st);
    });
    g_launches += 1;
    launch_status_merge(g.B, rstat, img_status, st);
    return check_launch();
}

mmsb_status mmsb_capacity(const mmsb_shape *shape, const uint8_t *image, int32_t *b_out, int64_t *capacity_out,
                          int32_t *img_status, void *ws, size_t ws_bytes, void *stream) {
    Geo g;
    if (!geo_of(shape, &g) || !image || !b_out || !capacity_out || !img_status || !ws) return MMSB_E_INVAL;
    const Layout L = layout(g);
    if (ws_bytes < L.total) return MMSB_E_INVAL;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (cudaMemsetAsync(img_status, 0, (size_t)g.B * 4, st) != cudaSuccess) return MMSB_E_CUDA;
    if (g.method == 1) lmr_decode_all(g, L, false, image, ws, img_status, nullptr, st);
    launch_capacity(g, image, at<uint32_t>(ws, L.map_bits), at<int32_t>(ws, L.lmr_b), b_out, capacity_out,
                    img_status, st);
    g_launches += 1;
    return check_launch();
}

mmsb_status mmsb_stats(const mmsb_shape *shape, const uint8_t *original, const uint8_t *recovered,
                       int64_t *sse_out, void *stream) {
    Geo g;
    if (!geo_of(shape, &g) || !original || !recovered || !sse_out) return MMSB_E_INVAL;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (cudaMemsetAsync(sse_out, 0, (size_t)g.B * 8, st) != cudaSuccess) return MMSB_E_CUDA;
    run_kernel(K_STATS, st, (long long)g.B * g.HW, [&] { launch_stats(g.HW, g.B, original, recovered, sse_out, st); });
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

mmsb_status mmsb_histogram(const mmsb_shape *shape, const uint8_t *images, int64_t *hist_out, void *stream) {
    Geo g;
    if (!geo_of(shape, &g) || !images || !hist_out) return MMSB_E_INVAL;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (cudaMemsetAsync(hist_out, 0, (size_t)g.B * 256 * 8, st) != cudaSuccess) return MMSB_E_CUDA;
    g_launches += 1;
    launch_histogram(g.HW, g.B, images, hist_out, st);
    return check_launch();
}

mmsb_status mmsb_diff_stats(const mmsb_shape *shape, const uint8_t *a, const uint8_t *b, int64_t *sse_out,
                            int64_t *ndiff_out, int64_t *absdiff_out, void *stream) {
    Geo g;
    if (!geo_of(shape, &g) || !a || !b || !sse_out || !ndiff_out || !absdiff_out) return MMSB_E_INVAL;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    for (int64_t *p : {sse_out, ndiff_out, absdiff_out})
        if (cudaMemsetAsync(p, 0, (size_t)g.B * 8, st) != cudaSuccess) return MMSB_E_CUDA;
    g_launches += 1;
    launch_diff_stats(g.HW, g.B, a, b, sse_out, ndiff_out, absdiff_out, st);
    return check_launch();
}

mmsb_status mmsb_ssim(const mmsb_shape *shape, const uint8_t *a, const uint8_t *b, double *ssim_out, void *stream) {
    Geo g;
    if (!geo_of(shape, &g) || !a || !b || !ssim_out) return MMSB_E_INVAL;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (cudaMemsetAsync(ssim_out, 0, (size_t)g.B * 8, st) != cudaSuccess) return MMSB_E_CUDA;
    g_launches += 2;
    launch_ssim(g.B, g.H, g.W, a, b, ssim_out, st);
    return check_launch();
}

void mmsb_entropy_chi2_host(int32_t batch, int32_t height, int32_t width, const int64_t *hist, double *entropy_out,
                            double *chi2_out) {
    const double n = (double)height * (double)width;
    for (int i = 0; i < batch; i++) {
        double H = 0.0, s = 0.0;
        for (int v = 0; v < 256; v++) {
            const double P = (double)hist[(size_t)i * 256 + v] / n;
            if (P > 0) H -= P * std::log2(P);
            const double d = P - 1.0 / 256.0;
            s += d * d;
        }
        if (entropy_out) entropy_out[i] = H;
        if (chi2_out) chi2_out[i] = 256.0 * n * s;
    }
}

void mmsb_npcr_uaci_host(int32_t batch, int32_t height, int32_t width, const int64_t *ndiff, const int64_t *absdiff,
                         double *npcr_out, double *uaci_out) {
    const double n = (double)height * (double)width;
    for (int i = 0; i < batch; i++) {
        if (npcr_out) npcr_out[i] = 100.0 * (double)ndiff[i] / n;
        if (uaci_out) uaci_out[i] = 100.0 * (double)absdiff[i] / (255.0 * n);
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

void mmsb_profile_enable(int on) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    for (auto &r : g_prof) { g_event_pool.push_back(r.a); g_event_pool.push_back(r.b); }
    g_prof.clear();
    g_prof_on = on != 0;
    if (g_prof_on) {
        if (!g_sym && cudaMalloc(&g_sym, 2 * sizeof(unsigned long long)) != cudaSuccess) g_sym = nullptr;
        if (g_sym) cudaMemset(g_sym, 0, 2 * sizeof(unsigned long long));
    }
}

int mmsb_profile_read(int kernel, const char **name, double *total_ms, int64_t *launches, int64_t *units) {
    if (kernel < 0 || kernel >= K_COUNT) return -1;
    std::lock_guard<std::mutex> lk(g_prof_mu);
    double t = 0;
    int64_t n = 0, u = 0;
    for (auto &r : g_prof) {
        if (r.id != kernel) continue;
        float ms = 0;
        if (cudaEventElapsedTime(&ms, r.a, r.b) != cudaSuccess) return -2;
        t += ms;
        n++;
        u += r.units;
    }
    if ((kernel == K_CODER_ENC || kernel == K_LMR_DECODE) && g_sym && n) {   // coded symbols, not pixels
        unsigned long long c = 0;
        if (cudaMemcpy(&c, g_sym + (kernel == K_CODER_ENC ? 0 : 1), sizeof c, cudaMemcpyDeviceToHost) == cudaSuccess)
            u = (int64_t)c;
    }
    if (name) *name = kKernelNames[kernel];
    if (total_ms) *total_ms = t;
    if (launches) *launches = n;
    if (units) *units = u;
    return K_COUNT;
}

}  // extern "C"
