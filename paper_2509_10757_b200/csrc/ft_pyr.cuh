// ft_pyr.cuh -- device image-pyramid build, bit-exact with the reference
// (extraction.py:97-125 build_pyramid = kernels.py:230-245 binomial5_u8 +
// kernels.py:248-268 resample_bilinear_u8).  Shared by the standalone
// ft_build_pyramids launch (ft_pyramid.cu) and the pyramid role of the fused
// per-frame kernel (ft_track.cu).
//
// Latency design: the 7 levels are a dependent chain, and a grid-wide barrier
// per level costs more than the arithmetic of a level.  So levels are grouped
// into STAGES (e.g. 1-3 and 4-7) and each stage is computed tile by tile with
// its halo recomputed inside the block: a tile owns a rectangle of every level
// of the stage (a Ty x Tx grid partition of that level), and the block derives
// top-down the region of each level it must compute (its own rectangle plus
// what the next level's region samples: bilinear footprint + 2-px blur
// halo), loads the stage's input region of the previous level once, and runs
// the stage's levels entirely in shared memory.  Only stage boundaries need
// the image's G blocks to meet at a group barrier.
//
// Per level, on a region (all in shared memory):
//   1. horizontal 5-tap binomial of the source rows, 4 columns per thread as
//      packed u16 pairs (u8 taps sum below 2^12, so no carry crosses halves),
//   2. vertical 5-tap over a sliding 5-row register window, round half up,
//      >> 8 (kernels.py:244), stored as fp32 (exact) -- the integer sum is exact, so
//      vertical-after-horizontal equals the reference's order,
//   3. bilinear resample with row / column coefficients hoisted into tables
//      (the same fp64 values the reference recomputes per pixel), split into
//      the per-(source row, output column) top/bot terms and the per-pixel
//      vertical blend -- each the reference's expression in its order
//      (-fmad=false), so the result is bit-identical.
// Reflect-101 borders: a region clamped to the image contains every
// reflected tap, so border columns only need index reflection.
#pragma once

#include <math.h>
#include <stdlib.h>

#include "ft_common.cuh"

namespace ft {

constexpr int PY_THREADS = 512;
constexpr int PY_MAX_W = 4096;
constexpr int PY_MAX_STAGES = 4;
constexpr int PY_MAX_T = 32;  // tiles per axis

struct PyrGeom {
    int32_t n_levels;
    int64_t offsets[FT_MAX_LEVELS];
    int32_t widths[FT_MAX_LEVELS];
    int32_t heights[FT_MAX_LEVELS];
    double sy[FT_MAX_LEVELS], sx[FT_MAX_LEVELS];  // level l-1 -> l: hs / hd, ws / wd
};

// Stages: levels (stage_end[s-1], stage_end[s]] (stage_end[-1] = 0), each
// tiled by ty[s] x tx[s].  The region chain is separable per axis, so the
// host tabulates it per tile row / column: own_*[l][t..t+1] = tile t's own
// span of level l, reg_*[l][t] = the span it computes, in_*[s][t] = the
// stage's input span of level first-1.  Buffer capacities are maxima.
struct PyrPlan {
    int32_t n_stages;
    int32_t stage_end[PY_MAX_STAGES];
    int32_t ty[PY_MAX_STAGES], tx[PY_MAX_STAGES];
    int32_t cap_region;  // bytes of one u8 region buffer
    int32_t cap_hsum;    // uint2 entries
    int32_t cap_smooth;  // floats
    int32_t cap_h;       // doubles of the horizontally interpolated rows
    int32_t cap_rows;    // row-table entries
    int32_t cap_cols;    // column-table entries
    int16_t own_y[FT_MAX_LEVELS][PY_MAX_T + 1], own_x[FT_MAX_LEVELS][PY_MAX_T + 1];
    int16_t reg_y[FT_MAX_LEVELS][PY_MAX_T][2], reg_x[FT_MAX_LEVELS][PY_MAX_T][2];
    int16_t in_y[PY_MAX_STAGES][PY_MAX_T][2], in_x[PY_MAX_STAGES][PY_MAX_T][2];
    int16_t smp_y[FT_MAX_LEVELS][PY_MAX_T][2], smp_x[FT_MAX_LEVELS][PY_MAX_T][2];  // smoothed span
};

struct PyrRect {
    int y0, y1, x0, x1;  // [y0, y1) x [x0, x1)
};

__host__ __device__ inline int pyr_reflect(int i, int n) {  // kernels.py:196-201
    if (i < 0) return -i;
    if (i >= n) return 2 * n - 2 - i;
    return i;
}
FT_DEV int reflect101(int i, int n) { return pyr_reflect(i, n); }

// Source span [lo, hi] (clamped) that outputs [r0, r1) sample along one axis
// (kernels.py:255-264: floor((i + 0.5) * s - 0.5) and +1).
__host__ __device__ inline void pyr_needed_rows(int r0, int r1, double s, int n, int &lo,
                                                int &hi) {
    const double f0 = ((double)r0 + 0.5) * s - 0.5;
    const double f1 = ((double)(r1 - 1) + 0.5) * s - 0.5;
    const int y0 = (int)floor(f0), y1 = (int)floor(f1) + 1;
    lo = y0 < 0 ? 0 : (y0 > n - 1 ? n - 1 : y0);
    hi = y1 < 0 ? 0 : (y1 > n - 1 ? n - 1 : y1);
}

// Host: fill sy / sx (the reference's hs / hd in fp64, kernels.py:251-252).
inline void pyr_geom_scales(PyrGeom &g) {
    for (int l = 1; l < g.n_levels; ++l) {
        g.sy[l] = (double)g.heights[l - 1] / (double)g.heights[l];
        g.sx[l] = (double)g.widths[l - 1] / (double)g.widths[l];
    }
}

// 1-D span [a, b) of level l-1 (unsmoothed) needed for outputs [c0, c1) of
// level l along one axis of size n (source): bilinear footprint + 2-px blur.
inline void pyr_need_1d(int c0, int c1, double s, int n, int &a, int &b) {
    int lo, hi;
    pyr_needed_rows(c0, c1, s, n, lo, hi);
    a = lo - 2 < 0 ? 0 : lo - 2;
    b = (hi + 2 > n - 1 ? n - 1 : hi + 2) + 1;
}

__device__ inline PyrRect pyr_rect_reg(const PyrPlan &p, int l, int ty, int tx) {
    return PyrRect{p.reg_y[l][ty][0], p.reg_y[l][ty][1], p.reg_x[l][tx][0], p.reg_x[l][tx][1]};
}
__device__ inline PyrRect pyr_rect_own(const PyrPlan &p, int l, int ty, int tx) {
    return PyrRect{p.own_y[l][ty], p.own_y[l][ty + 1], p.own_x[l][tx], p.own_x[l][tx + 1]};
}
__device__ inline PyrRect pyr_rect_in(const PyrPlan &p, int s, int ty, int tx) {
    return PyrRect{p.in_y[s][ty][0], p.in_y[s][ty][1], p.in_x[s][tx][0], p.in_x[s][tx][1]};
}

// Host: tabulate one axis of stage s (dims[l] = level sizes along the axis,
// scale[l] = level l-1 -> l ratio).
inline void pyr_axis_tables(int first, int last, int T, const int32_t *dims, const double *scale,
                            int16_t own[][PY_MAX_T + 1], int16_t reg[][PY_MAX_T][2],
                            int16_t in[PY_MAX_T][2], int16_t smp[][PY_MAX_T][2]) {
    for (int l = first; l <= last; ++l)
        for (int t = 0; t <= T; ++t) own[l][t] = (int16_t)((long long)t * dims[l] / T);
    for (int t = 0; t < T; ++t) {
        int a = own[last][t], b = own[last][t + 1];
        reg[last][t][0] = (int16_t)a;
        reg[last][t][1] = (int16_t)b;
        for (int l = last; l >= first; --l) {
            int na, nb;
            pyr_need_1d(a, b, scale[l], dims[l - 1], na, nb);
            if (l - 1 >= first) {  // bbox with the tile's own span of level l-1
                na = na < own[l - 1][t] ? na : own[l - 1][t];
                nb = nb > own[l - 1][t + 1] ? nb : own[l - 1][t + 1];
                reg[l - 1][t][0] = (int16_t)na;
                reg[l - 1][t][1] = (int16_t)nb;
            } else {
                in[t][0] = (int16_t)na;
                in[t][1] = (int16_t)nb;
            }
            a = na;
            b = nb;
        }
        for (int l = first; l <= last; ++l) {  // smoothed span level l samples
            int lo, hi;
            pyr_needed_rows(reg[l][t][0], reg[l][t][1], scale[l], dims[l - 1], lo, hi);
            smp[l][t][0] = (int16_t)lo;
            smp[l][t][1] = (int16_t)hi;
        }
    }
}

__host__ __device__ inline size_t pyr_al16(size_t x) { return (x + 15) & ~(size_t)15; }

// Everything one level of one tile needs, copied out of the (large) kernel
// parameter tables into shared memory once per tile by parallel loads: the
// constant cache does not hold the tables, and dependent misses at every
// phase would serialise the block.
struct PyrLevelDesc {
    PyrRect reg, own, src;        // computed region, own rectangle, source region
    int slo, shi, clo, chi;       // smoothed span sampled (kernels.py:255-264)
    int hs, ws, wd, pad;          // source dims, destination width (stride)
    long long off_dst, off_src;   // level byte offsets in the image's pyramid
    double sy, sx;
};

// Shared-memory layout of one block (host sizing and device carving agree).
struct PyrSmem {
    PyrLevelDesc *desc;  // [FT_MAX_LEVELS]
    uint8_t *reg[2];    // ping-pong u8 regions
    uint2 *hsum;        // packed horizontal sums
    float *smooth;      // smoothed pixels (u8 values, exact in fp32)
    double *hint;       // smoothed rows interpolated at the output columns
    double2 *roww;      // (1 - ay, ay)
    int2 *rowy;         // smooth offsets of rows y0c, y1c
    double2 *colw;      // (1 - ax, ax)
    int2 *colx;         // x0c - clo, x1c - clo
};

__host__ __device__ inline size_t pyr_layout(const PyrPlan &p, unsigned char *base, PyrSmem *S) {
    size_t o = 0, off[10];
    off[0] = o; o += pyr_al16((size_t)p.cap_region + 32);
    off[1] = o; o += pyr_al16((size_t)p.cap_region + 32);
    off[2] = o; o += pyr_al16((size_t)p.cap_hsum * 8);
    off[3] = o; o += pyr_al16((size_t)p.cap_smooth * 4);
    off[8] = o; o += pyr_al16((size_t)p.cap_h * 8);
    off[9] = o; o += pyr_al16(sizeof(PyrLevelDesc) * FT_MAX_LEVELS);
    off[4] = o; o += pyr_al16((size_t)p.cap_rows * 16);
    off[5] = o; o += pyr_al16((size_t)p.cap_rows * 8);
    off[6] = o; o += pyr_al16((size_t)p.cap_cols * 16);
    off[7] = o; o += pyr_al16((size_t)p.cap_cols * 8);
    if (S) {
        S->reg[0] = base + off[0];
        S->reg[1] = base + off[1];
        S->hsum = reinterpret_cast<uint2 *>(base + off[2]);
        S->smooth = reinterpret_cast<float *>(base + off[3]);
        S->hint = reinterpret_cast<double *>(base + off[8]);
        S->desc = reinterpret_cast<PyrLevelDesc *>(base + off[9]);
        S->roww = reinterpret_cast<double2 *>(base + off[4]);
        S->rowy = reinterpret_cast<int2 *>(base + off[5]);
        S->colw = reinterpret_cast<double2 *>(base + off[6]);
        S->colx = reinterpret_cast<int2 *>(base + off[7]);
    }
    return o;
}

// Host: tabulate every stage's spans and fill the capacities; returns the
// shared-memory bytes.
inline size_t pyr_plan_capacities(const PyrGeom &g, PyrPlan &p) {
    int cap_region = 0, cap_hsum = 0, cap_smooth = 0, cap_rows = 0, cap_cols = 0, cap_h = 0;
    for (int s = 0; s < p.n_stages; ++s) {
        const int first = (s == 0 ? 0 : p.stage_end[s - 1]) + 1, last = p.stage_end[s];
        pyr_axis_tables(first, last, p.ty[s], g.heights, g.sy, p.own_y, p.reg_y, p.in_y[s], p.smp_y);
        pyr_axis_tables(first, last, p.tx[s], g.widths, g.sx, p.own_x, p.reg_x, p.in_x[s], p.smp_x);
        for (int ty = 0; ty < p.ty[s]; ++ty)
            for (int tx = 0; tx < p.tx[s]; ++tx) {
                const int ih = p.in_y[s][ty][1] - p.in_y[s][ty][0];
                const int iw = p.in_x[s][tx][1] - p.in_x[s][tx][0];
                cap_region = ih * iw > cap_region ? ih * iw : cap_region;
                for (int l = first; l <= last; ++l) {
                    const int rh = p.reg_y[l][ty][1] - p.reg_y[l][ty][0];
                    const int rw = p.reg_x[l][tx][1] - p.reg_x[l][tx][0];
                    cap_region = rh * rw > cap_region ? rh * rw : cap_region;
                    cap_rows = rh > cap_rows ? rh : cap_rows;
                    cap_cols = rw > cap_cols ? rw : cap_cols;
                    // smoothed span = needed span of level l-1 (<= need_1d's)
                    int ya, yb, xa, xb;
                    pyr_need_1d(p.reg_y[l][ty][0], p.reg_y[l][ty][1], g.sy[l], g.heights[l - 1], ya, yb);
                    pyr_need_1d(p.reg_x[l][tx][0], p.reg_x[l][tx][1], g.sx[l], g.widths[l - 1], xa, xb);
                    const int nr = yb - ya, nq = (xb - xa + 3) / 4 + 1;
                    cap_hsum = nr * nq > cap_hsum ? nr * nq : cap_hsum;
                    cap_smooth = nr * 4 * nq > cap_smooth ? nr * 4 * nq : cap_smooth;
                    cap_h = nr * rw > cap_h ? nr * rw : cap_h;
                }
            }
    }
    p.cap_region = cap_region;
    p.cap_hsum = cap_hsum;
    p.cap_smooth = cap_smooth;
    p.cap_h = cap_h;
    p.cap_rows = cap_rows;
    p.cap_cols = cap_cols;
    return pyr_layout(p, nullptr, nullptr) + 16;
}

// Host: stages and tile grids.  Default: levels 1-3 and 4..L-1 (one group
// barrier), tiles of about `tile_px` pixels of the stage's first level with the
// level's aspect ratio.  FT_PYR_STAGES="3,7" / FT_PYR_TILE_PX="1600,1600"
// override (profiling).  Default 900 px: measured best single-frame latency.
inline bool pyr_make_plan(const PyrGeom &g, PyrPlan &p, int g_blocks, int n_images = 1) {
    const int L = g.n_levels;
    if (L < 2) return false;
    int ends[PY_MAX_STAGES], n = 0;
    if (const char *e = getenv("FT_PYR_STAGES")) {
        int v = 0, have = 0;
        for (const char *c = e;; ++c) {
            if (*c >= '0' && *c <= '9') {
                v = v * 10 + (*c - '0');
                have = 1;
            } else {
                if (have && n < PY_MAX_STAGES) ends[n++] = v;
                v = 0;
                have = 0;
                if (!*c) break;
            }
        }
    }
    if (n == 0) {
        if (L - 1 <= 3) {
            ends[n++] = L - 1;
        } else {
            ends[n++] = 3;
            ends[n++] = L - 1;
        }
    }
    int px[PY_MAX_STAGES];
    // latency (few images): small tiles, more blocks; throughput (many
    // images): bigger tiles, less halo recompute (measured, r1)
    for (int s = 0; s < PY_MAX_STAGES; ++s) px[s] = n_images <= 8 ? 900 : 1600;
    if (const char *e = getenv("FT_PYR_TILE_PX")) {
        int v = 0, k = 0, have = 0;
        for (const char *c = e;; ++c) {
            if (*c >= '0' && *c <= '9') {
                v = v * 10 + (*c - '0');
                have = 1;
            } else {
                if (have && k < PY_MAX_STAGES) px[k++] = v;
                v = 0;
                have = 0;
                if (!*c) break;
            }
        }
        for (int s = k; s > 0 && s < PY_MAX_STAGES; ++s) px[s] = px[k - 1];
    }
    p.n_stages = n;
    int prev = 0;
    for (int s = 0; s < n; ++s) {
        if (ends[s] <= prev || ends[s] > L - 1) return false;
        if (s == n - 1 && ends[s] != L - 1) return false;
        p.stage_end[s] = ends[s];
        const int first = prev + 1;
        const double h = g.heights[first], w = g.widths[first];
        double tiles = h * w / (px[s] > 16 ? px[s] : 16);
        // one tile per block when the blocks nearly cover the tiles (no
        // second round for a few blocks); many tiles per block otherwise
        if (tiles > g_blocks && tiles < 2.0 * g_blocks) tiles = g_blocks;
        int ty = (int)floor(sqrt(tiles * h / w) + 0.5);
        ty = ty < 1 ? 1 : (ty > g.heights[ends[s]] ? g.heights[ends[s]] : ty);
        ty = ty > PY_MAX_T ? PY_MAX_T : ty;
        int tx = (int)floor(tiles / ty);
        tx = tx < 1 ? 1 : (tx > g.widths[ends[s]] ? g.widths[ends[s]] : tx);
        tx = tx > PY_MAX_T ? PY_MAX_T : tx;
        p.ty[s] = ty;
        p.tx[s] = tx;
        prev = ends[s];
    }
    return true;
}

constexpr uint32_t PY_LO = 0x00ff00ffu;


// Horizontal 5-tap binomial of 4 consecutive columns c..c+3 given p = &row[c-2]
// (interior: all taps inside the row).  b0..b7 = row[c-2 .. c+5] via two
// funnel shifts of three aligned words.  Returns (c0 | c2 << 16, c1 | c3 << 16).
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
    const uint32_t ev = e0 + e1 + 4u * (o0 + n) + 6u * m;  // columns c, c+2
    const uint32_t od = o0 + o1 + 4u * (m + e1) + 6u * n;  // columns c+1, c+3
    return make_uint2(ev, od);
}

// Border quad: reflect-101 per column; `row` points at image column `x0r`
// of the region row; columns > xmax give 0.
FT_DEV uint2 pyr_hsum_quad_border(const uint8_t *row, int x0r, int c, int w, int xmax) {
    uint32_t v[4];
#pragma unroll
    for (int m = 0; m < 4; ++m) {
        const int x = c + m;
        uint32_t acc = 0;
        if (x <= xmax)
            acc = (uint32_t)row[reflect101(x - 2, w) - x0r] + 4u * row[reflect101(x - 1, w) - x0r] +
                  6u * row[x - x0r] + 4u * row[reflect101(x + 1, w) - x0r] +
                  (uint32_t)row[reflect101(x + 2, w) - x0r];
        v[m] = acc;
    }
    return make_uint2(v[0] | (v[2] << 16), v[1] | (v[3] << 16));
}

// One level: region `c` of level l from region `sr` of level l-1 held in
// `src` (u8, row stride sr.x1 - sr.x0), into `dst` (stride c.x1 - c.x0).
// Starts by writing tables (caller synchronised the buffers), ends synced.
#ifdef PYR_TIMELINE
#define PYR_MARK()                                                  \
    do {                                                            \
        if (tl && threadIdx.x == 0 && *tk < 64) tl[*tk] = pyr_ns(); \
        if (tl) ++*tk;                                              \
    } while (0)
#else
#define PYR_MARK() \
    do {           \
    } while (0)
#endif

FT_DEV unsigned long long pyr_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// One level: region `c` of level l (tile row ty / column tx of the plan) from
// region `sr` of level l-1 held in `src` (u8, row stride sr.x1 - sr.x0), into
// `dst` (stride c.x1 - c.x0).  Thread mapping is warp-per-row, lanes over
// columns (no integer division): warp w of NW takes rows w, w + NW, ...
// Starts by writing tables (caller synchronised the buffers), ends synced.
FT_DEV void pyr_level_region(const PyrLevelDesc &d, const uint8_t *src, uint8_t *dst,
                             const PyrSmem &S, unsigned long long *tl = nullptr,
                             int *tk = nullptr) {
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, NW = blockDim.x >> 5;
    const PyrRect sr = d.src, c = d.reg;
    const int hs = d.hs, ws = d.ws;
    const int slo = d.slo, shi = d.shi, clo = d.clo, chi = d.chi;
    const int t0 = max(slo - 2, 0), t1 = min(shi + 2, hs - 1);
    const int nr = t1 - t0 + 1, ns = shi - slo + 1;
    const int ncol = chi - clo + 1, nq = (ncol + 3) >> 2, sstr = 4 * nq;
    const int sw = sr.x1 - sr.x0;
    const int crow = c.y1 - c.y0, ccol = c.x1 - c.x0;
    // coefficient tables (kernels.py:255-264)
    {
        const double sy = d.sy, sx = d.sx;
        for (int i = tid; i < crow; i += blockDim.x) {
            const double fy = ((double)(c.y0 + i) + 0.5) * sy - 0.5;
            const int y0 = (int)floor(fy);
            const double ay = fy - (double)y0;
            S.roww[i] = make_double2(1.0 - ay, ay);
            S.rowy[i] = make_int2((min(max(y0, 0), hs - 1) - slo) * ccol,
                                  (min(max(y0 + 1, 0), hs - 1) - slo) * ccol);
        }
        for (int j = tid; j < ccol; j += blockDim.x) {
            const double fx = ((double)(c.x0 + j) + 0.5) * sx - 0.5;
            const int x0 = (int)floor(fx);
            const double ax = fx - (double)x0;
            S.colw[j] = make_double2(1.0 - ax, ax);
            S.colx[j] = make_int2(min(max(x0, 0), ws - 1) - clo, min(max(x0 + 1, 0), ws - 1) - clo);
        }
    }
    // quads across lanes: lpr lanes per row (power of two >= nq, <= 32),
    // rpw = 32 / lpr rows per warp step
    const int qb = nq >= 32 ? 5 : (nq <= 1 ? 0 : 32 - __clz(nq - 1));
    const int lpr = 1 << qb, rpw = 32 >> qb;
    const int ql = lane & (lpr - 1), rl = lane >> qb;
    // 1. horizontal sums of source rows [t0, t1], columns [clo, chi]
    for (int r = w * rpw + rl; r < nr; r += NW * rpw) {
        const uint8_t *row = src + (t0 + r - sr.y0) * sw;
        for (int q = ql; q < nq; q += lpr) {
            const int cq = clo + 4 * q;
            S.hsum[r * nq + q] = (cq >= 2 && cq + 5 <= ws - 1)
                                     ? pyr_hsum_quad(row + (cq - 2 - sr.x0))
                                     : pyr_hsum_quad_border(row, sr.x0, cq, ws, chi);
        }
    }
    __syncthreads();
    PYR_MARK();
    // 2. vertical sums + round -> smoothed rows [slo, shi] (fp32, exact):
    // each thread slides a 5-row register window down a contiguous chunk
    {
        const int chunks = NW * rpw, per = (ns + chunks - 1) / chunks;
        const int k = w * rpw + rl, sa = k * per, sb = min(ns, sa + per);
        for (int q = ql; q < nq; q += lpr) {
            if (sa >= sb) break;
            uint2 win[5];
#pragma unroll
            for (int m = 0; m < 4; ++m)
                win[m + 1] = S.hsum[(reflect101(slo + sa + m - 2, hs) - t0) * nq + q];
            for (int s = sa; s < sb; ++s) {
#pragma unroll
                for (int m = 0; m < 4; ++m) win[m] = win[m + 1];
                win[4] = S.hsum[(reflect101(slo + s + 2, hs) - t0) * nq + q];
                const uint32_t ev = ((win[0].x + win[4].x + 4u * (win[1].x + win[3].x) +
                                      6u * win[2].x) + 0x00800080u) >> 8;
                const uint32_t od = ((win[0].y + win[4].y + 4u * (win[1].y + win[3].y) +
                                      6u * win[2].y) + 0x00800080u) >> 8;
                *reinterpret_cast<float4 *>(S.smooth + s * sstr + 4 * q) =
                    make_float4((float)(ev & 0xffu), (float)(od & 0xffu),
                                (float)((ev >> 16) & 0xffu), (float)((od >> 16) & 0xffu));
            }
        }
    }
    __syncthreads();
    PYR_MARK();
    // 3. bilinear (kernels.py:260-268), separated exactly: the reference's
    // top / bot terms depend only on (source row, output column), so they are
    // computed once per smoothed row (3a) and the vertical blend per output
    // pixel (3b) reads them -- the same fp64 operations in the same order.
    for (int j = lane; j < ccol; j += 32) {  // 3a
        const double2 cw = S.colw[j];
        const int2 cx = S.colx[j];
        for (int r = w; r < ns; r += NW) {
            const float *q = S.smooth + r * sstr;
            S.hint[r * ccol + j] = cw.x * (double)q[cx.x] + cw.y * (double)q[cx.y];
        }
    }
    __syncthreads();
    for (int i = w; i < crow; i += NW) {  // 3b (row terms: warp broadcast)
        const double2 rw = S.roww[i];
        const int2 ry = S.rowy[i];
        for (int j = lane; j < ccol; j += 32) {
            const double top = S.hint[ry.x + j], bot = S.hint[ry.y + j];
            dst[i * ccol + j] = (uint8_t)(int)(rw.x * top + rw.y * bot + 0.5);
        }
    }
    __syncthreads();
    PYR_MARK();
}

// Copy a rectangle of a global u8 image (row stride `stride`) into a packed
// shared-memory region (warp per row).
FT_DEV void pyr_load_region(const uint8_t *img, int stride, const PyrRect &r, uint8_t *dst) {
    const int w = r.x1 - r.x0, h = r.y1 - r.y0;
    const int lane = threadIdx.x & 31, NW = blockDim.x >> 5;
    for (int y = threadIdx.x >> 5; y < h; y += NW) {
        const uint8_t *s = img + (int64_t)(r.y0 + y) * stride + r.x0;
#pragma unroll 4
        for (int x = lane; x < w; x += 32) dst[y * w + x] = __ldcg(s + x);
    }
}

// Write the tile's own rectangle `o` (inside region c held packed in `src`)
// to the global level image (warp per row).
FT_DEV void pyr_store_own(const uint8_t *src, const PyrRect &c, const PyrRect &o, uint8_t *img,
                          int stride) {
    const int w = o.x1 - o.x0, h = o.y1 - o.y0, cw = c.x1 - c.x0;
    const int lane = threadIdx.x & 31, NW = blockDim.x >> 5;
    for (int y = threadIdx.x >> 5; y < h; y += NW) {
        uint8_t *d = img + (int64_t)(o.y0 + y) * stride + o.x0;
        const uint8_t *s = src + (o.y0 - c.y0 + y) * cw + (o.x0 - c.x0);
        for (int x = lane; x < w; x += 32) d[x] = s[x];
    }
}

// Build levels 1..L-1 of one image (this block = `rank` of G).  `base` is the
// image's flat pyramid; `lvl0` the level-0 pixels (== base + offsets[0] or a
// separate raw image).  `bar` is the image's group-barrier word pair.  Every
// thread of the block calls this; on return this block's tiles are written
// (other blocks' may not be).
FT_DEV void pyr_build_image(const PyrGeom &g, const PyrPlan &p, uint8_t *base,
                            const uint8_t *lvl0, int rank, int G, unsigned long long *bar,
                            unsigned char *smem, unsigned long long *tl = nullptr) {
    int tk_ = 0, *tk = &tk_;
    unsigned bpar = 0;
    PYR_MARK();
    PyrSmem S;
    pyr_layout(p, smem, &S);
    for (int s = 0; s < p.n_stages; ++s) {
        const int first = (s == 0 ? 0 : p.stage_end[s - 1]) + 1, last = p.stage_end[s];
        const int tiles = p.ty[s] * p.tx[s];
        for (int t = rank; t < tiles; t += G) {
            const int ty = t / p.tx[s], tx = t - ty * p.tx[s];
            __syncthreads();  // previous tile done with the buffers
            if (threadIdx.x <= last - first) {  // one thread per level: parallel loads
                const int l = first + threadIdx.x;
                PyrLevelDesc d;
                d.reg = pyr_rect_reg(p, l, ty, tx);
                d.own = pyr_rect_own(p, l, ty, tx);
                d.src = l == first ? pyr_rect_in(p, s, ty, tx) : pyr_rect_reg(p, l - 1, ty, tx);
                d.slo = p.smp_y[l][ty][0];
                d.shi = p.smp_y[l][ty][1];
                d.clo = p.smp_x[l][tx][0];
                d.chi = p.smp_x[l][tx][1];
                d.hs = g.heights[l - 1];
                d.ws = g.widths[l - 1];
                d.wd = g.widths[l];
                d.pad = 0;
                d.off_dst = g.offsets[l];
                d.off_src = g.offsets[l - 1];
                d.sy = g.sy[l];
                d.sx = g.sx[l];
                S.desc[l] = d;
            }
            __syncthreads();
            const PyrLevelDesc &d0 = S.desc[first];
            const uint8_t *srcimg = first == 1 ? lvl0 : base + d0.off_src;
            pyr_load_region(srcimg, d0.ws, d0.src, S.reg[0]);
            __syncthreads();
            PYR_MARK();
            int cur = 0;
            for (int l = first; l <= last; ++l) {
                const PyrLevelDesc &d = S.desc[l];
                pyr_level_region(d, S.reg[cur], S.reg[cur ^ 1], S, tl, tk);
                pyr_store_own(S.reg[cur ^ 1], d.reg, d.own, base + d.off_dst, d.wd);
                cur ^= 1;
                PYR_MARK();
            }
        }
        if (s + 1 < p.n_stages) group_barrier(bar, G, bpar);
        PYR_MARK();
    }
}

}  // namespace ft
