// ft_pyramid.cu -- device image-pyramid build, bit-exact with the reference
// (extraction.py:97-125 build_pyramid = kernels.py:230-245 binomial5_u8 +
// kernels.py:248-268 resample_bilinear_u8), so frames can ship their raw
// 752x480 images (0.36 MB each) instead of 1.1 MB pyramids.
//
// Level 0 is the caller's image, already in place in the flat pyramid
// buffer; levels 1..L-1 are written here.  One cooperative launch: G blocks
// per image, a group barrier between levels.  A block owns a band of output
// rows of the level: it horizontally blurs the previous-level rows the band
// needs into shared memory (int32, exact), blurs those vertically to the
// smoothed rows (round half up, >> 8), and resamples bilinearly in fp64 with
// the reference's evaluation order (compiled with -fmad=false).
#include <cmath>
#include <cstring>

#include "ft_common.cuh"
#include "ft_ws.cuh"

namespace ft {

constexpr int PY_THREADS = 512;
constexpr int PY_MAX_W = 4096;
constexpr int PY_SUB = 8;  // output rows per shared-memory pass

struct PyrArgs {
    uint8_t *data;
    int64_t frame_bytes;
    int32_t n_levels;
    int64_t offsets[FT_MAX_LEVELS];
    int32_t widths[FT_MAX_LEVELS];
    int32_t heights[FT_MAX_LEVELS];
    int32_t n_images, G, sub;  // G blocks per image, <= sub output rows per pass
    unsigned long long *bar;  // [n_images]
    const uint8_t *src0;      // optional separate level-0 images (else in place)
    int64_t src0_stride;
};

FT_DEV int reflect101(int i, int n) {  // kernels.py:196-201
    if (i < 0) return -i;
    if (i >= n) return 2 * n - 2 - i;
    return i;
}

// Source-row span [lo, hi] of the smoothed previous level that output rows
// [r0, r1) sample (kernels.py:255-259).
FT_DEV void needed_rows(int r0, int r1, double sy, int hs, int &lo, int &hi) {
    const double f0 = ((double)r0 + 0.5) * sy - 0.5;
    const double f1 = ((double)(r1 - 1) + 0.5) * sy - 0.5;
    int y0 = (int)floor(f0), y1 = (int)floor(f1) + 1;
    lo = y0 < 0 ? 0 : (y0 > hs - 1 ? hs - 1 : y0);
    hi = y1 < 0 ? 0 : (y1 > hs - 1 ? hs - 1 : y1);
}

__global__ void __launch_bounds__(PY_THREADS) pyramid_kernel(const PyrArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int img = blockIdx.x / a.G, rank = blockIdx.x - img * a.G;
    uint8_t *base = a.data + (int64_t)img * a.frame_bytes;
    // smem: tmp (horizontally blurred rows, int32) | smooth rows (u8)
    int *tmp = reinterpret_cast<int *>(smem);
    const uint8_t *img0 = a.src0 ? a.src0 + (int64_t)img * a.src0_stride : nullptr;
    if (img0) {  // level 0 <- the raw image (this block's band, 16-B chunks)
        const int64_t n0 = (int64_t)a.widths[0] * a.heights[0];
        const int64_t per = ((n0 + a.G - 1) / a.G + 15) & ~(int64_t)15;
        const int64_t b0 = rank * per, b1 = min(n0, b0 + per);
        uint8_t *l0 = base + a.offsets[0];
        const bool vec = ((((uintptr_t)img0) | ((uintptr_t)l0)) & 15) == 0;
        const int64_t nvec = vec ? (b1 - b0) / 16 : 0;
        for (int64_t q = threadIdx.x; q < nvec; q += PY_THREADS)
            *reinterpret_cast<uint4 *>(l0 + b0 + 16 * q) =
                __ldg(reinterpret_cast<const uint4 *>(img0 + b0 + 16 * q));
        for (int64_t t = b0 + 16 * nvec + threadIdx.x; t < b1; t += PY_THREADS) l0[t] = img0[t];
    }
    for (int l = 1; l < a.n_levels; ++l) {
        const int ws = a.widths[l - 1], hs = a.heights[l - 1];
        const int wd = a.widths[l], hd = a.heights[l];
        const uint8_t *src = (l == 1 && img0) ? img0 : base + a.offsets[l - 1];
        uint8_t *dst = base + a.offsets[l];
        const double sy = (double)hs / (double)hd, sx = (double)ws / (double)wd;
        const int band = (hd + a.G - 1) / a.G;
        const int b0 = rank * band, b1 = min(hd, b0 + band);
        for (int r0 = b0; r0 < b1; r0 += a.sub) {  // shared memory holds `sub` rows
            const int r1 = min(b1, r0 + a.sub);
            int slo, shi;  // smoothed rows needed
            needed_rows(r0, r1, sy, hs, slo, shi);
            const int tlo = slo - 2, thi = shi + 2;  // blurred rows (pre-reflection)
            const int nt = thi - tlo + 1, ns = shi - slo + 1;
            uint8_t *sm_s = reinterpret_cast<uint8_t *>(tmp + (size_t)nt * ws);
            // horizontal pass: tmp[t][x] = sum_k W5[k] * src[reflect(y)][reflect(x + k - 2)]
            for (int e = threadIdx.x; e < nt * ws; e += PY_THREADS) {
                const int t = e / ws, x = e - t * ws;
                const uint8_t *row = src + (int64_t)reflect101(tlo + t, hs) * ws;
                const int acc = (int)row[reflect101(x - 2, ws)] + 4 * (int)row[reflect101(x - 1, ws)] +
                                6 * (int)row[x] + 4 * (int)row[reflect101(x + 1, ws)] +
                                (int)row[reflect101(x + 2, ws)];
                tmp[e] = acc;
            }
            __syncthreads();
            // vertical pass -> smoothed u8 rows [slo, shi]: (acc + 128) >> 8
            for (int e = threadIdx.x; e < ns * ws; e += PY_THREADS) {
                const int s = e / ws, x = e - s * ws;
                const int y = slo + s;
                int acc = 0;
                const int w5[5] = {1, 4, 6, 4, 1};
#pragma unroll
                for (int k = 0; k < 5; ++k) acc += w5[k] * tmp[(reflect101(y + k - 2, hs) - tlo) * ws + x];
                sm_s[e] = (uint8_t)((acc + 128) >> 8);
            }
            __syncthreads();
            // bilinear resample (kernels.py:254-268), fp64 in reference order
            for (int e = threadIdx.x; e < (r1 - r0) * wd; e += PY_THREADS) {
                const int i = r0 + e / wd, j = e - (e / wd) * wd;
                const double fy = ((double)i + 0.5) * sy - 0.5;
                const int y0 = (int)floor(fy);
                const double ay = fy - (double)y0;
                const int y0c = min(max(y0, 0), hs - 1), y1c = min(max(y0 + 1, 0), hs - 1);
                const double fx = ((double)j + 0.5) * sx - 0.5;
                const int x0 = (int)floor(fx);
                const double ax = fx - (double)x0;
                const int x0c = min(max(x0, 0), ws - 1), x1c = min(max(x0 + 1, 0), ws - 1);
                const uint8_t *s0 = sm_s + (y0c - slo) * ws, *s1 = sm_s + (y1c - slo) * ws;
                const double top = (1.0 - ax) * (double)s0[x0c] + ax * (double)s0[x1c];
                const double bot = (1.0 - ax) * (double)s1[x0c] + ax * (double)s1[x1c];
                dst[(int64_t)i * wd + j] = (uint8_t)(int)((1.0 - ay) * top + ay * bot + 0.5);
            }
            __syncthreads();
        }
        if (l + 1 < a.n_levels) group_barrier(a.bar + img, a.G);
    }
}

}  // namespace ft

using namespace ft;

extern "C" int ft_build_pyramids(int32_t n_images, const ft_pyramid *pyr,
                                 const uint8_t *images, int64_t image_stride,
                                 const ft_workspace *ws, ft_stream_t stream) {
    if (!pyr || !ws || !pyr->data) return FT_E_NULL;
    if (n_images < 1 || pyr->n_levels < 1 || pyr->n_levels > FT_MAX_LEVELS) return FT_E_RANGE;
    if (pyr->n_levels == 1) return FT_OK;
    for (int l = 0; l < pyr->n_levels; ++l)
        if (pyr->widths[l] < 3 || pyr->heights[l] < 3 || pyr->widths[l] > PY_MAX_W) return FT_E_RANGE;
    const int st = ws_check(ws, (n_images + 1) / 2, 1, 1);  // 2 images per workspace frame
    if (st != FT_OK) return st;
    PyrArgs a;
    memset(&a, 0, sizeof(a));
    a.data = const_cast<uint8_t *>(pyr->data);
    a.frame_bytes = pyr->frame_bytes;
    a.n_levels = pyr->n_levels;
    for (int l = 0; l < pyr->n_levels; ++l) {
        a.offsets[l] = pyr->offsets[l];
        a.widths[l] = pyr->widths[l];
        a.heights[l] = pyr->heights[l];
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    a.bar = ws_ptr<unsigned long long>(ws, ws_layout(ws).pyr_bar);
    if (images && image_stride < (int64_t)a.widths[0] * a.heights[0]) return FT_E_RANGE;
    // shared memory for one pass of PY_SUB output rows (worst level)
    a.sub = PY_SUB;
    size_t smem = 0;
    for (int l = 1; l < pyr->n_levels; ++l) {
        const int hd = a.heights[l], hs = a.heights[l - 1], ws_ = a.widths[l - 1];
        const int src_rows = (int)ceil((double)PY_SUB * hs / hd) + 4;
        const size_t b = (size_t)(src_rows + 4) * ws_ * 4 + (size_t)src_rows * ws_ + 64;
        smem = b > smem ? b : smem;
    }
    if (smem > 227 * 1024) return FT_E_RANGE;
    cudaError_t e = cudaFuncSetAttribute(pyramid_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return (int)e;
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pyramid_kernel, PY_THREADS, smem);
    if (occ < 1) return FT_E_RANGE;
    const int resident = occ * sms;
    // images in chunks that fit one resident wave (cooperative launch);
    // G blocks per image: bands of ~PY_SUB rows at level 1 when they fit
    for (int i0 = 0; i0 < n_images;) {
        const int rem = n_images - i0;
        const int chunk = rem < resident ? rem : resident;
        int G = (a.heights[1] + PY_SUB - 1) / PY_SUB;
        if ((long long)G * chunk > resident) G = resident / chunk;
        if (G < 1) G = 1;
        a.G = G;
        a.n_images = chunk;
        a.data = const_cast<uint8_t *>(pyr->data) + (int64_t)i0 * pyr->frame_bytes;
        a.src0 = images ? images + (int64_t)i0 * image_stride : nullptr;
        a.src0_stride = image_stride;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(G * chunk);
        cfg.blockDim = dim3(PY_THREADS);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = (cudaStream_t)stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeCooperative;
        attr[0].val.cooperative = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        e = cudaLaunchKernelEx(&cfg, pyramid_kernel, a);
        if (e != cudaSuccess) return (int)e;
        i0 += chunk;
    }
    return (int)cudaGetLastError();
}
