// k_stats.cu -- the paper's image statistics on the GPU: per-image grey-level
// histograms (Shannon entropy P:1441 and chi^2 P:1447 follow on the host from the counts),
// difference counts for NPCR / UACI (reading Q26) next to the SSE of PSNR,
// and the mean windowed SSIM (11x11 Gaussian sigma 1.5, K1 0.01, K2 0.03, L 255,
// S:524; windows inside the image).  Integer counts are exact; SSIM is computed in fp64.
#include "mmsb_device.cuh"
#include "mmsb_kernels.h"

namespace mmsb {

// ---- histograms: per-warp private bins in shared memory, merged into int64 per image
__global__ void __launch_bounds__(256) hist_kernel(long long HW, const uint8_t *__restrict__ img,
                                                   unsigned long long *__restrict__ hist) {
    __shared__ uint32_t bins[8][256];
    const int tid = threadIdx.x, wid = tid >> 5, b = blockIdx.y;
    for (int i = tid; i < 8 * 256; i += 256) (&bins[0][0])[i] = 0;
    __syncthreads();
    const uint4 *p = reinterpret_cast<const uint4 *>(img + (size_t)b * HW);
    for (long long i = (long long)blockIdx.x * 256 + tid; i < HW / 16; i += (long long)gridDim.x * 256) {
        const uint4 u = __ldg(p + i);
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int k = 0; k < 4; k++)
#pragma unroll
            for (int j = 0; j < 4; j++) atomicAdd(&bins[wid][(w[k] >> (8 * j)) & 0xFFu], 1u);
    }
    __syncthreads();
    uint32_t v = 0;
#pragma unroll
    for (int w = 0; w < 8; w++) v += bins[w][tid];
    if (v) atomicAdd(hist + (size_t)b * 256 + tid, (unsigned long long)v);
}

// ---- differences: sum (a-b)^2, #{a != b}, sum |a-b|
__global__ void __launch_bounds__(256) diff_kernel(long long HW, const uint8_t *__restrict__ a,
                                                   const uint8_t *__restrict__ b, unsigned long long *__restrict__ sse,
                                                   unsigned long long *__restrict__ ndiff,
                                                   unsigned long long *__restrict__ absd) {
    __shared__ unsigned long long red[3][8];
    const int img = blockIdx.y;
    const uint4 *pa = reinterpret_cast<const uint4 *>(a + (size_t)img * HW);
    const uint4 *pb = reinterpret_cast<const uint4 *>(b + (size_t)img * HW);
    unsigned long long s2 = 0, nd = 0, s1 = 0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < HW / 16; i += (long long)gridDim.x * blockDim.x) {
        const uint4 u = __ldg(pa + i), v = __ldg(pb + i);
        const uint32_t x[4] = {u.x, u.y, u.z, u.w}, y[4] = {v.x, v.y, v.z, v.w};
        uint32_t q2 = 0, q1 = 0, qn = 0;
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const uint32_t d = __vabsdiffu4(x[k], y[k]);
            q1 += __dp4a(d, 0x01010101u, 0u);                 // sum of the 4 byte differences
            q2 += __dp4a(d, d, 0u);                           // sum of their squares
            qn += __popc(__vcmpne4(x[k], y[k]) & 0x01010101u);
        }
        s2 += q2; s1 += q1; nd += qn;
    }
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
        s2 += __shfl_xor_sync(0xffffffffu, s2, s);
        s1 += __shfl_xor_sync(0xffffffffu, s1, s);
        nd += __shfl_xor_sync(0xffffffffu, nd, s);
    }
    if ((threadIdx.x & 31) == 0) { red[0][threadIdx.x >> 5] = s2; red[1][threadIdx.x >> 5] = nd; red[2][threadIdx.x >> 5] = s1; }
    __syncthreads();
    if (threadIdx.x < 3) {
        unsigned long long t = 0;
        for (int w = 0; w < 8; w++) t += red[threadIdx.x][w];
        unsigned long long *dst = threadIdx.x == 0 ? sse : threadIdx.x == 1 ? ndiff : absd;
        if (t) atomicAdd(dst + img, t);
    }
}

// ---- SSIM: one CTA per 32x32 block of window positions; the 42x42 source region of both
// images in smem, a horizontal 11-tap pass of mu_a, mu_b, E[a^2], E[b^2], E[ab] into smem (fp64),
// a vertical pass per position, the SSIM values summed per CTA and added into the image's sum
// (fixed point, so the mean is reproducible bit for bit).
constexpr int kSsimTile = 32, kSsimSrc = kSsimTile + 10;

struct SsimSmem {
    uint8_t a[kSsimSrc][kSsimSrc + 2], b[kSsimSrc][kSsimSrc + 2];
    double h[5][kSsimSrc][kSsimTile];
    double g[11];
    double red[8];
};

__global__ void __launch_bounds__(256) ssim_kernel(int H, int W, const uint8_t *__restrict__ A,
                                                   const uint8_t *__restrict__ Bi, double *__restrict__ sum) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    SsimSmem &S = *reinterpret_cast<SsimSmem *>(smem_raw);
    const int tid = threadIdx.x, img = blockIdx.z;
    const int x0 = blockIdx.x * kSsimTile, y0 = blockIdx.y * kSsimTile;
    const int VH = H - 10, VW = W - 10;                  // window positions
    const uint8_t *a = A + (size_t)img * H * W, *b = Bi + (size_t)img * H * W;
    if (tid < 11) {
        double t = 0;
        for (int i = 0; i < 11; i++) t += exp(-((i - 5) * (i - 5)) / (2.0 * 1.5 * 1.5));
        S.g[tid] = exp(-((tid - 5) * (tid - 5)) / (2.0 * 1.5 * 1.5)) / t;
    }
    for (int i = tid; i < kSsimSrc * kSsimSrc; i += 256) {
        const int r = i / kSsimSrc, c = i % kSsimSrc, y = y0 + r, x = x0 + c;
        const bool in = y < H && x < W;
        S.a[r][c] = in ? a[(size_t)y * W + x] : 0;
        S.b[r][c] = in ? b[(size_t)y * W + x] : 0;
    }
    __syncthreads();
    for (int i = tid; i < kSsimSrc * kSsimTile; i += 256) {
        const int r = i / kSsimTile, c = i % kSsimTile;
        double ma = 0, mb = 0, aa = 0, bb = 0, ab = 0;
#pragma unroll
        for (int j = 0; j < 11; j++) {
            const double va = S.a[r][c + j], vb = S.b[r][c + j], w = S.g[j];
            ma = fma(w, va, ma);
            mb = fma(w, vb, mb);
            aa = fma(w, va * va, aa);
            bb = fma(w, vb * vb, bb);
            ab = fma(w, va * vb, ab);
        }
        S.h[0][r][c] = ma; S.h[1][r][c] = mb; S.h[2][r][c] = aa; S.h[3][r][c] = bb; S.h[4][r][c] = ab;
    }
    __syncthreads();
    const double C1 = (0.01 * 255.0) * (0.01 * 255.0), C2 = (0.03 * 255.0) * (0.03 * 255.0);
    double acc = 0;
    for (int i = tid; i < kSsimTile * kSsimTile; i += 256) {
        const int r = i / kSsimTile, c = i % kSsimTile;
        if (y0 + r >= VH || x0 + c >= VW) continue;
        double q[5] = {0, 0, 0, 0, 0};
#pragma unroll
        for (int k = 0; k < 11; k++) {
            const double w = S.g[k];
#pragma unroll
            for (int m = 0; m < 5; m++) q[m] = fma(w, S.h[m][r + k][c], q[m]);
        }
        const double va = q[2] - q[0] * q[0], vb = q[3] - q[1] * q[1], cab = q[4] - q[0] * q[1];
        acc += ((2 * q[0] * q[1] + C1) * (2 * cab + C2)) / ((q[0] * q[0] + q[1] * q[1] + C1) * (va + vb + C2));
    }
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, s);
    if ((tid & 31) == 0) S.red[tid >> 5] = acc;
    __syncthreads();
    if (tid == 0) {
        double t = 0;
        for (int w = 0; w < 8; w++) t += S.red[w];
        // the image's sum accumulates in its output slot as 2^-32 fixed point (int64 adds are
        // associative: the result does not depend on the order the CTAs finish in)
        atomicAdd(reinterpret_cast<unsigned long long *>(sum + img), (unsigned long long)llrint(t * 4294967296.0));
    }
}

__global__ void ssim_finish_kernel(int B, double npos, double *__restrict__ ssim) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < B) {
        const long long fx = reinterpret_cast<const long long *>(ssim)[i];
        ssim[i] = npos > 0 ? ((double)fx / 4294967296.0) / npos : 0.0;
    }
}

// ---------------------------------------------------------------------------- launchers
void launch_histogram(long long HW, int B, const uint8_t *img, int64_t *hist, cudaStream_t st) {
    int bx = (int)((HW / 16 + 256 * 16 - 1) / (256 * 16));
    hist_kernel<<<dim3(bx < 1 ? 1 : bx, B), 256, 0, st>>>(HW, img, reinterpret_cast<unsigned long long *>(hist));
}

void launch_diff_stats(long long HW, int B, const uint8_t *a, const uint8_t *b, int64_t *sse, int64_t *ndiff,
                       int64_t *absd, cudaStream_t st) {
    int bx = (int)((HW / 16 + 256 * 8 - 1) / (256 * 8));
    diff_kernel<<<dim3(bx < 1 ? 1 : bx, B), 256, 0, st>>>(HW, a, b, reinterpret_cast<unsigned long long *>(sse),
                                                           reinterpret_cast<unsigned long long *>(ndiff),
                                                           reinterpret_cast<unsigned long long *>(absd));
}

void launch_ssim(int B, int H, int W, const uint8_t *a, const uint8_t *b, double *ssim, cudaStream_t st) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(ssim_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(SsimSmem));
        attr = true;
    }
    const int VH = H - 10, VW = W - 10;
    if (VH > 0 && VW > 0) {
        dim3 grid((VW + kSsimTile - 1) / kSsimTile, (VH + kSsimTile - 1) / kSsimTile, B);
        ssim_kernel<<<grid, 256, sizeof(SsimSmem), st>>>(H, W, a, b, ssim);
    }
    ssim_finish_kernel<<<(B + 255) / 256, 256, 0, st>>>(B, VH > 0 && VW > 0 ? (double)VH * VW : 0.0, ssim);
}

}  // namespace mmsb
