// ft_pyr.cuh -- device image-pyramid build, bit-exact with the reference
// (extraction.py:97-125 build_pyramid = kernels.py:230-245 binomial5_u8 +
// kernels.py:248-268 resample_bilinear_u8).  Shared by the standalone
// ft_build_pyramids launch (ft_pyramid.cu) and the pyramid role of the fused
// per-frame kernel (ft_track.cu).
//
// G blocks build one image.  Level 0 is the caller's image; for each level
// l = 1..L-1 a block owns a band of output rows and processes it in passes of
// `sub` rows, all staged in shared memory:
//   1. the previous level's source rows the pass needs (one contiguous byte
//      range: rows are stored back to back) -> `raw` with 16-B loads,
//   2. 5x5 binomial (separable; the integer sum is exact, so the vertical-
//      then-horizontal order here equals the reference's horizontal-then-
//      vertical one), round half up, >> 8 -> smoothed rows as fp64,
//   3. bilinear resample with per-column coefficients hoisted into shared
//      memory (the same fp64 values the reference recomputes per pixel, so
//      the per-pixel expression rounds identically; -fmad=false).
// A group barrier separates levels (the next level reads other blocks'
// rows).  The u8 outputs are written with coalesced byte stores.
#pragma once

#include "ft_common.cuh"

namespace ft {

constexpr int PY_THREADS = 512;
constexpr int PY_MAX_W = 4096;

struct PyrGeom {
    int32_t n_levels;
    int64_t offsets[FT_MAX_LEVELS];
    int32_t widths[FT_MAX_LEVELS];
    int32_t heights[FT_MAX_LEVELS];
};

FT_DEV int reflect101(int i, int n) {  // kernels.py:196-201
    if (i < 0) return -i;
    if (i >= n) return 2 * n - 2 - i;
    return i;
}

// Smoothed-row span [lo, hi] of the previous level that output rows [r0, r1)
// sample (kernels.py:255-259).
__host__ __device__ inline void pyr_needed_rows(int r0, int r1, double sy, int hs, int &lo,
                                                int &hi) {
    const double f0 = ((double)r0 + 0.5) * sy - 0.5;
    const double f1 = ((double)(r1 - 1) + 0.5) * sy - 0.5;
    const int y0 = (int)floor(f0), y1 = (int)floor(f1) + 1;
    lo = y0 < 0 ? 0 : (y0 > hs - 1 ? hs - 1 : y0);
    hi = y1 < 0 ? 0 : (y1 > hs - 1 ? hs - 1 : y1);
}

// Upper bound on the smoothed rows one pass of `sub` output rows needs at
// any level (host sizing; 2 extra rows cover the floor/+1 ends).
__host__ __device__ inline int pyr_max_smooth_rows(const PyrGeom &g, int sub) {
    int m = 0;
    for (int l = 1; l < g.n_levels; ++l) {
        const double sy = (double)g.heights[l - 1] / (double)g.heights[l];
        const int r = (int)ceil((double)(sub - 1) * sy) + 3;
        m = r > m ? r : m;
    }
    return m;
}

__host__ __device__ inline int pyr_max_width(const PyrGeom &g) {
    int m = 0;
    for (int l = 0; l < g.n_levels; ++l) m = g.widths[l] > m ? g.widths[l] : m;
    return m;
}

// Per-pass shared-memory layout (W = widest level, NQ = quads of 4 columns):
//   raw    u8   [(ns+4) rows x W] + 32 B slack (source rows, contiguous)
//   hsum   u32x2 [(ns+4) rows x NQ]  horizontal sums, packed u16 pairs
//          (word 0 = columns 4q, 4q+2; word 1 = 4q+1, 4q+3)
//   smooth f64  [ns rows x 4 NQ]     smoothed pixels
//   colw   f64x2 [W] (1 - ax, ax), colx u16x2 [W] (x0c, x1c)
//   rows   f64x2 [sub] (1 - ay, ay), int2 [sub] (y0c, y1c) - slo
struct PyrSmem {
    uint8_t *raw;
    uint2 *hsum;
    double *smooth;
    double2 *colw;
    uint32_t *colx;
    double2 *roww;
    int2 *rowy;
    int nq_max;
};

__host__ __device__ inline size_t pyr_al16(size_t x) { return (x + 15) & ~(size_t)15; }

__host__ __device__ inline size_t pyr_layout(const PyrGeom &g, int sub, unsigned char *base,
                                             PyrSmem *out) {
    const int ns = pyr_max_smooth_rows(g, sub), W = pyr_max_width(g);
    const int nq = (W + 3) / 4;
    size_t o = 0;
    const size_t raw = o;
    o += pyr_al16((size_t)(ns + 4) * W + 32);
    const size_t hs = o;
    o += pyr_al16((size_t)(ns + 4) * nq * 8);
    const size_t sm = o;
    o += pyr_al16((size_t)ns * nq * 32);
    const size_t cw = o;
    o += pyr_al16((size_t)W * 16);
    const size_t cx = o;
    o += pyr_al16((size_t)W * 4);
    const size_t rw = o;
    o += pyr_al16((size_t)sub * 16);
    const size_t ry = o;
    o += pyr_al16((size_t)sub * 8);
    if (out) {
        out->raw = base + raw;
        out->hsum = reinterpret_cast<uint2 *>(base + hs);
        out->smooth = reinterpret_cast<double *>(base + sm);
        out->colw = reinterpret_cast<double2 *>(base + cw);
        out->colx = reinterpret_cast<uint32_t *>(base + cx);
        out->roww = reinterpret_cast<double2 *>(base + rw);
        out->rowy = reinterpret_cast<int2 *>(base + ry);
        out->nq_max = nq;
    }
    return o;
}

inline size_t pyr_smem_bytes(const PyrGeom &g, int sub) { return pyr_layout(g, sub, nullptr, nullptr) + 16; }

// Copy n contiguous bytes global -> shared; `dst` is chosen by the caller to
// share src's alignment mod 16 so the body moves as uint4.
FT_DEV void pyr_copy_bytes(uint8_t *dst, const uint8_t *src, int n) {
    const int head = min(n, (int)((16 - ((uintptr_t)src & 15)) & 15));
    const int nv = (n - head) >> 4;
    const int tail0 = head + (nv << 4);
    for (int t = threadIdx.x; t < head; t += blockDim.x) dst[t] = src[t];
    const uint4 *s4 = reinterpret_cast<const uint4 *>(src + head);
    uint4 *d4 = reinterpret_cast<uint4 *>(dst + head);
    for (int q = threadIdx.x; q < nv; q += blockDim.x) d4[q] = __ldcg(s4 + q);
    for (int t = tail0 + threadIdx.x; t < n; t += blockDim.x) dst[t] = src[t];
}

constexpr uint32_t PY_LO = 0x00ff00ffu;

// Horizontal 5-tap binomial of columns 4q..4q+3 of one raw row (interior:
// 4q-2 >= 0 and 4q+5 < w).  b0..b7 = row[4q-2 .. 4q+5] via two funnel shifts
// of three aligned words; sums of u8 taps stay < 2^12, so two columns share a
// 32-bit word with no carry between them.  Returns (c0 | c2 << 16, c1 | c3 << 16).
FT_DEV uint2 pyr_hsum_quad(const uint8_t *p) {
    const uintptr_t ad = (uintptr_t)p;
    const uint32_t *wp = reinterpret_cast<const uint32_t *>(ad & ~(uintptr_t)3);
    const uint32_t sh = (uint32_t)(ad & 3) * 8;
    const uint32_t w0 = wp[0], w1 = wp[1], w2 = wp[2];
    const uint32_t x0 = __funnelshift_r(w0, w1, sh);  // b0 b1 b2 b3
    const uint32_t x1 = __funnelshift_r(w1, w2, sh);  // b4 b5 b6 b7
    const uint32_t y = __funnelshift_r(x0, x1, 16);   // b2 b3 b4 b5
    const uint32_t e0 = x0 & PY_LO;                   // (b0, b2)
    const uint32_t o0 = __byte_perm(x0, 0, 0x4341);   // (b1, b3)
    const uint32_t e1 = x1 & PY_LO;                   // (b4, b6)
    const uint32_t o1 = __byte_perm(x1, 0, 0x4341);   // (b5, b7)
    const uint32_t m = y & PY_LO;                     // (b2, b4)
    const uint32_t n = __byte_perm(y, 0, 0x4341);     // (b3, b5)
    // column c needs b[c-4q .. c-4q+4]: even (c0, c2), odd (c1, c3)
    const uint32_t ev = e0 + e1 + 4u * (o0 + n) + 6u * m;
    const uint32_t od = o0 + o1 + 4u * (m + e1) + 6u * n;
    return make_uint2(ev, od);
}

// Same for border quads (reflect-101 per column; columns >= w give 0).
FT_DEV uint2 pyr_hsum_quad_border(const uint8_t *row, int q, int w) {
    uint32_t c[4];
#pragma unroll
    for (int m = 0; m < 4; ++m) {
        const int x = 4 * q + m;
        uint32_t acc = 0;
        if (x < w)
            acc = (uint32_t)row[reflect101(x - 2, w)] + 4u * row[reflect101(x - 1, w)] +
                  6u * row[x] + 4u * row[reflect101(x + 1, w)] + (uint32_t)row[reflect101(x + 2, w)];
        c[m] = acc;
    }
    return make_uint2(c[0] | (c[2] << 16), c[1] | (c[3] << 16));
}

// Build levels 1..L-1 of one image (this block = `rank` of G).  `base` is the
// image's flat pyramid; `lvl0` the level-0 pixels (== base + offsets[0] or a
// separate raw image).  `bar` is the image's group-barrier counter.  Every
// thread of the block calls this.
FT_DEV void pyr_build_image(const PyrGeom &g, uint8_t *base, const uint8_t *lvl0, int rank,
                            int G, int sub, unsigned long long *bar, unsigned char *smem) {
    PyrSmem S;
    pyr_layout(g, sub, smem, &S);
    const int nt = blockDim.x, tid = threadIdx.x;

    for (int l = 1; l < g.n_levels; ++l) {
        const int ws = g.widths[l - 1], hs = g.heights[l - 1];
        const int wd = g.widths[l], hd = g.heights[l];
        const int nq = (ws + 3) >> 2, sstr = 4 * nq;  // quads per row, smooth row stride
        const uint8_t *src = l == 1 ? lvl0 : base + g.offsets[l - 1];
        uint8_t *dst = base + g.offsets[l];
        const double sy = (double)hs / (double)hd, sx = (double)ws / (double)wd;
        const int band = (hd + G - 1) / G;
        const int b0 = min(hd, rank * band), b1 = min(hd, b0 + band);
        if (b0 < b1) {
            // column coefficients (kernels.py:260-264), once per level
            for (int j = tid; j < wd; j += nt) {
                const double fx = ((double)j + 0.5) * sx - 0.5;
                const int x0 = (int)floor(fx);
                const double ax = fx - (double)x0;
                S.colw[j] = make_double2(1.0 - ax, ax);
                S.colx[j] = (uint32_t)min(max(x0, 0), ws - 1) |
                            ((uint32_t)min(max(x0 + 1, 0), ws - 1) << 16);
            }
        }
        for (int r0 = b0; r0 < b1; r0 += sub) {
            const int r1 = min(b1, r0 + sub);
            int slo, shi;
            pyr_needed_rows(r0, r1, sy, hs, slo, shi);
            const int t0 = max(slo - 2, 0), t1 = min(shi + 2, hs - 1);
            const int ns = shi - slo + 1, nr = t1 - t0 + 1;
            const uint8_t *s0 = src + (int64_t)t0 * ws;
            uint8_t *rawp = S.raw + ((uintptr_t)s0 & 15);
            __syncthreads();  // previous pass / level done with every buffer
            // 1. source rows [t0, t1] (reflection stays inside this span)
            pyr_copy_bytes(rawp, s0, nr * ws);
            if (tid < r1 - r0) {  // row coefficients (kernels.py:255-259)
                const double fy = ((double)(r0 + tid) + 0.5) * sy - 0.5;
                const int y0 = (int)floor(fy);
                const double ay = fy - (double)y0;
                S.roww[tid] = make_double2(1.0 - ay, ay);
                S.rowy[tid] = make_int2((min(max(y0, 0), hs - 1) - slo) * sstr,
                                        (min(max(y0 + 1, 0), hs - 1) - slo) * sstr);
            }
            __syncthreads();
            // 2a. horizontal 5-tap of every source row (kernels.py:235-239)
            {
                int r = tid / nq, q = tid - r * nq;
                const int dr = nt / nq, dq = nt - dr * nq;
                for (; r < nr; r += dr, q += dq) {
                    if (q >= nq) {
                        q -= nq;
                        if (++r >= nr) break;
                    }
                    const uint8_t *row = rawp + r * ws;
                    S.hsum[r * nq + q] = (4 * q >= 2 && 4 * q + 5 < ws)
                                             ? pyr_hsum_quad(row + 4 * q - 2)
                                             : pyr_hsum_quad_border(row, q, ws);
                }
            }
            __syncthreads();
            // 2b. vertical 5-tap + round half up (kernels.py:240-245) -> fp64.
            // Thread = (quad, row group); a 5-row register window slides down.
            {
                const int groups = max(1, min(nt / nq, ns));
                const int per = (ns + groups - 1) / groups;
                const int q = tid % nq, grp = tid / nq;
                if (grp < groups) {
                    const int sa = grp * per, sb = min(ns, sa + per);
                    uint2 w[5];
                    if (sa < sb) {
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            w[k + 1] = S.hsum[(reflect101(slo + sa + k - 2, hs) - t0) * nq + q];
                    }
                    for (int s = sa; s < sb; ++s) {
#pragma unroll
                        for (int k = 0; k < 4; ++k) w[k] = w[k + 1];
                        w[4] = S.hsum[(reflect101(slo + s + 2, hs) - t0) * nq + q];
                        const uint32_t ev = ((w[0].x + w[4].x + 4u * (w[1].x + w[3].x) +
                                              6u * w[2].x) + 0x00800080u) >> 8;
                        const uint32_t od = ((w[0].y + w[4].y + 4u * (w[1].y + w[3].y) +
                                              6u * w[2].y) + 0x00800080u) >> 8;
                        double2 *o = reinterpret_cast<double2 *>(S.smooth + s * sstr + 4 * q);
                        o[0] = make_double2((double)(ev & 0xffu), (double)(od & 0xffu));
                        o[1] = make_double2((double)((ev >> 16) & 0xffu), (double)((od >> 16) & 0xffu));
                    }
                }
            }
            __syncthreads();
            // 3. bilinear (kernels.py:260-268), the reference's fp64 order
            {
                const int nrow = r1 - r0;
                int ii = tid / wd, j = tid - ii * wd;
                const int di = nt / wd, dj = nt - di * wd;
                for (; ii < nrow; ii += di, j += dj) {
                    if (j >= wd) {
                        j -= wd;
                        if (++ii >= nrow) break;
                    }
                    const double2 rw = S.roww[ii], cw = S.colw[j];
                    const int2 ry = S.rowy[ii];
                    const uint32_t cx = S.colx[j];
                    const int xa = cx & 0xffff, xb = cx >> 16;
                    const double *q0 = S.smooth + ry.x, *q1 = S.smooth + ry.y;
                    const double top = cw.x * q0[xa] + cw.y * q0[xb];
                    const double bot = cw.x * q1[xa] + cw.y * q1[xb];
                    dst[(int64_t)(r0 + ii) * wd + j] = (uint8_t)(int)(rw.x * top + rw.y * bot + 0.5);
                }
            }
        }
        if (l + 1 < g.n_levels) group_barrier(bar, G);
    }
}

}  // namespace ft
