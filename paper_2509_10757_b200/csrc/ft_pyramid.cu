// ft_pyramid.cu -- standalone ft_build_pyramids launch: extraction.py:97-125
// build_pyramid for many images in one cooperative launch (G blocks per
// image, the shared routine in ft_pyr.cuh), so frames can ship their raw
// 752x480 images (0.36 MB each) instead of 1.1 MB pyramids.  Optionally
// copies level 0 from separate raw images first.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "ft_common.cuh"
#include "ft_pyr.cuh"
#include "ft_ws.cuh"

namespace ft {

struct PyrArgs {
    PyrGeom g;
    PyrPlan p;
    uint8_t *data;
    int64_t frame_bytes;
    int32_t n_images, G;      // G blocks per image
    unsigned long long *bar;  // [n_images][2]
    const uint8_t *src0;      // optional separate level-0 images (else in place)
    int64_t src0_stride;
    unsigned long long *tl;  // debug timeline [grid][16] (FT_DEBUG_PYR_TIMELINE)
};

__global__ void __launch_bounds__(PY_THREADS, 2) pyramid_kernel(const PyrArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int img = blockIdx.x / a.G, rank = blockIdx.x - img * a.G;
    uint8_t *base = a.data + (int64_t)img * a.frame_bytes;
    const uint8_t *img0 = a.src0 ? a.src0 + (int64_t)img * a.src0_stride : nullptr;
    if (img0) {  // level 0 <- the raw image (this block's slice, 16-B chunks)
        const int64_t n0 = (int64_t)a.g.widths[0] * a.g.heights[0];
        const int64_t per = ((n0 + a.G - 1) / a.G + 15) & ~(int64_t)15;
        const int64_t b0 = rank * per, b1 = min(n0, b0 + per);
        uint8_t *l0 = base + a.g.offsets[0];
        const bool vec = ((((uintptr_t)img0) | ((uintptr_t)l0)) & 15) == 0;
        const int64_t nvec = vec && b1 > b0 ? (b1 - b0) / 16 : 0;
        for (int64_t q = threadIdx.x; q < nvec; q += PY_THREADS)
            *reinterpret_cast<uint4 *>(l0 + b0 + 16 * q) =
                __ldg(reinterpret_cast<const uint4 *>(img0 + b0 + 16 * q));
        for (int64_t t = b0 + 16 * nvec + threadIdx.x; t < b1; t += PY_THREADS) l0[t] = img0[t];
    }
    pyr_build_image(a.g, a.p, base, img0 ? img0 : base + a.g.offsets[0], rank, a.G, a.bar + 2 * img,
                    smem, a.tl ? a.tl + 64 * blockIdx.x : nullptr);
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
    a.g.n_levels = pyr->n_levels;
    for (int l = 0; l < pyr->n_levels; ++l) {
        a.g.offsets[l] = pyr->offsets[l];
        a.g.widths[l] = pyr->widths[l];
        a.g.heights[l] = pyr->heights[l];
    }
    a.frame_bytes = pyr->frame_bytes;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    a.bar = ws_ptr<unsigned long long>(ws, ws_layout(ws).pyr_bar);
    if (images && image_stride < (int64_t)a.g.widths[0] * a.g.heights[0]) return FT_E_RANGE;
    pyr_geom_scales(a.g);
    // plan for the first chunk's blocks-per-image (occupancy from a probe plan)
    if (!pyr_make_plan(a.g, a.p, 1 << 30, n_images)) return FT_E_RANGE;
    size_t smem = pyr_plan_capacities(a.g, a.p);
    if (smem > 227 * 1024) return FT_E_RANGE;
    cudaError_t e = cudaFuncSetAttribute(pyramid_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         227 * 1024);
    if (e != cudaSuccess) return (int)e;
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pyramid_kernel, PY_THREADS, smem);
    if (occ < 1) return FT_E_RANGE;
    {
        const int chunk0 = n_images < occ * sms ? n_images : occ * sms;
        PyrPlan q = a.p;
        if (pyr_make_plan(a.g, q, occ * sms / chunk0, n_images)) {
            const size_t sq = pyr_plan_capacities(a.g, q);
            int occ_q = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_q, pyramid_kernel, PY_THREADS, sq);
            if (sq <= 227 * 1024 && occ_q >= occ) {
                a.p = q;
                smem = sq;
            }
        }
    }
    const int resident = occ * sms;
    int max_tiles = 1;
    for (int s = 0; s < a.p.n_stages; ++s)
        max_tiles = a.p.ty[s] * a.p.tx[s] > max_tiles ? a.p.ty[s] * a.p.tx[s] : max_tiles;
    // images in chunks that fit one resident wave (cooperative launch); G
    // blocks per image, at most one per tile of the widest stage
    for (int i0 = 0; i0 < n_images;) {
        const int rem = n_images - i0;
        const int chunk = rem < resident ? rem : resident;
        int G = resident / chunk;
        if (G > max_tiles) G = max_tiles;
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
        static unsigned long long *tl_buf = nullptr;
        const char *tl_path = getenv("FT_DEBUG_PYR_TIMELINE");
        a.tl = nullptr;
        cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
        cudaStreamIsCapturing((cudaStream_t)stream, &cap);
        if (tl_path && cap == cudaStreamCaptureStatusNone) {
            if (!tl_buf) cudaMalloc(&tl_buf, 64 * 8 * 4096);
            cudaMemsetAsync(tl_buf, 0, 64 * 8 * 4096, (cudaStream_t)stream);
            a.tl = tl_buf;
        }
        e = cudaLaunchKernelEx(&cfg, pyramid_kernel, a);
        if (e != cudaSuccess) return (int)e;
        if (a.tl) {
            static unsigned long long host[64 * 4096];
            const int nb = G * chunk < 4096 ? G * chunk : 4096;
            cudaMemcpyAsync(host, a.tl, 64 * 8 * nb, cudaMemcpyDeviceToHost, (cudaStream_t)stream);
            cudaStreamSynchronize((cudaStream_t)stream);
            FILE *fp = fopen(tl_path, "a");
            if (fp) {
                fprintf(fp, "launch images=%d G=%d stages=%d\n", chunk, G, a.p.n_stages);
                for (int b = 0; b < nb; ++b) {
                    fprintf(fp, "%d", b);
                    for (int k = 0; k < 64; ++k) fprintf(fp, " %llu", host[64 * b + k]);
                    fprintf(fp, "\n");
                }
                fclose(fp);
            }
        }
        i0 += chunk;
    }
    return (int)cudaGetLastError();
}
