// ft_track.cu -- the per-frame tracking hot path as ONE cooperative sm_100a
// kernel: pinhole stereo matching and search-by-projection / SearchLocalPoints
// run side by side in block groups, with in-kernel group barriers replacing
// the reference's host round trips.
//
// Reference semantics (trackfront, pkg/src/trackfront):
//   stereo phase 1   kernels.py:300-345 stereo_phase1_kernel; stereo.py:67-103
//   stereo phase 2   kernels.py:351-428 stereo_phase2_kernel; stereo.py:106-140
//   no-image accept  stereo.py:143-168 matches_from_candidates
//   reject           stereo.py:171-188 reject_outliers (np.median semantics)
//   phase A          kernels.py:470-579 project_search_kernel; projection.py:118-158
//   grid             mapping.py:68-100 FrameGrid (truncate, clip)
//   phase B          projection.py:161-178 resolve_conflicts
//   phase C          projection.py:181-200 rotation_consistency_filter
//   local search     localmap.py:79-122 search_local_points
//
// Launch geometry (host picks it, see track_launch):
//   grid = W group slots x (Gs stereo blocks + Gm map blocks), 512 threads,
//   launched cooperatively so every block is resident.  Slot w processes
//   frames w, w+W, w+2W, ... ; within a frame the Gs stereo blocks split the
//   left keypoints and the Gm map blocks split the map points.
//
// Stereo block: stage the right keypoint table (u, v, octave, descriptor) in
//   shared memory with coalesced loads and build the row-bucket CSR there;
//   one warp per left keypoint: phase 1 over the contiguous CSR range of rows
//   [r0, r1] with a redux.sync min of (dist << 16 | j) (= the reference's
//   lexicographic (dist, j) order), then phase 2 with the 11x11 / 11x21
//   patches staged per warp in shared memory.  REJECT: each accepted SAD is
//   added to the group's coarse + fine histograms (L2 reds) as it is found;
//   after the group barrier every stereo block locates the same median with
//   two dependent histogram reads and resets its own rejected matches (no
//   serial tail; a median above the fine range gathers every SAD instead).
// Map block: stage the frame's keypoint table + cell-grid CSR (+ a hash set
//   of slotted point ids) in shared memory; thread-per-point fp64 projection
//   in the reference's evaluation order; warp per visible point over the
//   window's cell rows with a shuffle merge of (best key, second);
//   claims are 64-bit atomicMin keys (~epoch << 32 | dist << 23 | point) so
//   the minimum is the reference's (lowest dist, lowest point) winner and
//   stale claims from earlier launches always lose (no reset pass).  After a
//   group barrier each block resolves its own points; ordered outputs use
//   one more barrier for the cross-block prefix.
// Persistent mode (track_persist_kernel; ft_runner_create_persistent,
//   ft_track_frames_ring): one launch steps through a ring of frame slots;
//   its plans add a dedicated tail block to each role (stereo median /
//   rejection / count, map resolve / slot writes), so the keypoint and point
//   blocks publish their results with release reductions and move on to the
//   next frame instead of waiting at group barriers.
#include <cstdio>
#include <nvtx3/nvToolsExt.h>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "ft_common.cuh"
#include "ft_ws.cuh"

#ifndef FT_MAP_LANES_PER_POINT
#define FT_MAP_LANES_PER_POINT 16
#endif

namespace ft {

#ifndef FT_TK_THREADS
#define FT_TK_THREADS 512
#endif
constexpr int TK_THREADS = FT_TK_THREADS;  // threads per block (one block per SM)
constexpr int TK_WARPS = TK_THREADS / 32;
constexpr int TK_MAX_BINS = 256;
constexpr int TK_MAP_CHUNK_MAX = 2048;  // points per map block (shared per-point arrays)
constexpr long long NO_PID = -1;  // mapping.py:13 NO_POINT

struct TrackArgs {
    int32_t F, W, Gs, Gm;
    // stereo
    int32_t smode;
    ft_keypoints L, R;
    ft_pyramid PL, PR;
    ft_stereo_params sp;
    ft_stereo_out so;
    int32_t patch_ints;
    // map
    int32_t pmode;
    ft_map_points P;
    ft_keypoints K;
    ft_project_params pp;
    ft_project_io io;
    ft_project_out po;
    int32_t hash_bits;
    int32_t map_chunk_cap;  // max points per map block (smem sizing), even
    int32_t stage_rdesc;    // stereo: right descriptors staged in smem (else read from L2)
    int32_t stage_kdesc;    // map: keypoint descriptors staged in smem
    // workspace
    unsigned long long *bar_s;   // [W][2]
    unsigned long long *bar_m;   // [W][2]
    unsigned long long *ep_m;    // [F] claim epochs per claims row (group_ticket)
    unsigned long long *ep_s;    // [W] stereo-group instance tickets
    unsigned *med;               // [W][3][MED_WS] SAD-median histograms
    unsigned long long *tail_s;  // [W] stereo-group arrivals (tail mode)
    unsigned long long *tail_m;  // [W] map-group arrivals (tail mode)
    int4 *mcand;                 // [W][cap_points] map candidates (tail mode)
    int *mcnt;                   // [W][WS_MAX_GROUP][2] candidates, prefilled slots per block
    int32_t stereo_tail;         // one frame per group: a dedicated block runs the stereo tail
    int32_t map_tail;            // ... and the map resolve
    unsigned long long *claims;  // [F][cap_kp]
    int *blk_counts;             // [F][Gm]
    int *hist;                   // [F][TK_MAX_BINS]
    unsigned long long *tl;      // optional timeline [grid][TL_SLOTS] (FT_DEBUG_TIMELINE)
    // 1 when the inputs may be rewritten while the kernel is alive (the
    // persistent runner's H2D copies between steps): per-step inputs are then
    // read with coherent loads (ld.global.ca, ordered by the step's acquire)
    // instead of the read-only path (ld.global.nc), which PTX defines only
    // for data that stays constant for the kernel's lifetime.
    int32_t coherent;
    int32_t pad_;
};

constexpr int TL_SLOTS = 16;

FT_DEV unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// timeline mark (debug only): slot k of this block
#define TL_MARK(a, k)                                                               \
    do {                                                                            \
        if ((a).tl && threadIdx.x == 0) (a).tl[blockIdx.x * TL_SLOTS + (k)] = global_ns(); \
    } while (0)

// Per-step input load: read-only path unless the launch is coherent (above).
template <typename T>
FT_DEV T ld_in(const TrackArgs &a, const T *p) {
    return a.coherent ? __ldca(p) : __ldg(p);
}

// ---------------------------------------------------------------------------
// group barrier among the G blocks of one role in one slot: one 64-bit
// counter, low word = arrivals, high word = generation.  The last arrival
// resets the count and bumps the generation in one atomic, so the counter is
// back to (gen, 0) after every barrier and launches of any geometry may share
// a workspace.

// Warm the TLB / L2 for a page the block will touch later (no data use).
FT_DEV void prefetch_l2(const void *p) {
    if (p) asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// Instance number of a group's current frame: each of the G blocks takes
// one ticket ((instance << 32) | tickets); the G-th resets the tickets and
// bumps the instance in one atomic.  Every block of an instance reads the
// same instance number, for any G -- the next instance's tickets are taken
// after a group barrier that orders them behind this reset.  Monotonic
// across launches sharing the workspace.
FT_DEV unsigned group_ticket(unsigned long long *ctr, int G) {
    const unsigned long long old = atomicAdd(ctr, 1ull);
    if ((uint32_t)old == (uint32_t)(G - 1)) atomicAdd(ctr, (1ull << 32) - (unsigned long long)G);
    return (unsigned)(old >> 32);
}


// ---------------------------------------------------------------------------
// np.median of the accepted SADs (stereo.py:180): the values of ranks
// (n-1)/2 and n/2 found together by an 8-bit radix select from the top
// non-zero digit.  vals[k] holds the SAD of left keypoint k or 0xffffffff
// when unmatched (skipped).  Per digit: two shared histograms (one per
// rank), warp 0 / warp 1 locate the digits, 2 block barriers.

// Warp-level search of a 256-bin histogram for the bin holding rank k.
FT_DEV void warp_find_rank(const int *hist, int k, int *out_digit, int *out_k) {
    const int lane = threadIdx.x & 31;
    int c[8], loc = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        c[i] = hist[lane * 8 + i];
        loc += c[i];
    }
    int incl = loc;
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
        const int y = __shfl_up_sync(FULL, incl, s);
        if (lane >= s) incl += y;
    }
    int run = incl - loc;
    if (k >= run && k < incl) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (k < run + c[i]) {
                *out_digit = lane * 8 + i;
                *out_k = k - run;
                break;
            }
            run += c[i];
        }
    }
}

// Single-pass variant for small SADs (vmax < MED_SMALL_BINS, the common case:
// an accepted 11x11 SAD of normalised intensities is a few hundred): one
// value histogram in shared memory, one block scan, both ranks (n-1)/2 and
// n/2 located in the same pass.  Same result as block_median_pair.
constexpr int MED_SMALL_BINS = 4096;
constexpr int MED_PER_THREAD = (MED_SMALL_BINS + TK_THREADS - 1) / TK_THREADS;

__device__ void block_median_pair_small(const uint32_t *vals, int n, int nm, int *hist,
                                        int *scan_tmp, int *misc, uint32_t &v_lo,
                                        uint32_t &v_hi) {
    const int k_lo = (nm - 1) / 2, k_hi = nm / 2;
    for (int b = threadIdx.x; b < MED_SMALL_BINS; b += TK_THREADS) hist[b] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += TK_THREADS) {
        const uint32_t x = vals[i];
        if (x != 0xffffffffu) atomicAdd(&hist[x], 1);
    }
    __syncthreads();
    // thread t owns bins [t * PT, (t + 1) * PT)
    const int b0 = threadIdx.x * MED_PER_THREAD;
    int local[MED_PER_THREAD];
    int sum = 0;
#pragma unroll
    for (int j = 0; j < MED_PER_THREAD; ++j) {
        local[j] = b0 + j < MED_SMALL_BINS ? hist[b0 + j] : 0;
        sum += local[j];
    }
    int total;
    int before = block_exclusive_scan<TK_THREADS>(sum, scan_tmp, total);
#pragma unroll
    for (int j = 0; j < MED_PER_THREAD; ++j) {
        const int c = local[j];
        if (c > 0) {
            if (before <= k_lo && k_lo < before + c) misc[8] = b0 + j;
            if (before <= k_hi && k_hi < before + c) misc[10] = b0 + j;
        }
        before += c;
    }
    __syncthreads();
    v_lo = (uint32_t)misc[8];
    v_hi = (uint32_t)misc[10];
}

__device__ void block_median_pair(const uint32_t *vals, int n, int nm, uint32_t vmax, int *hist,
                                  int *misc, uint32_t &v_lo, uint32_t &v_hi) {
    int k_lo = (nm - 1) / 2, k_hi = nm / 2;
    int top = 24;
    while (top > 0 && (vmax >> top) == 0) top -= 8;
    uint32_t pre_lo = 0, pre_hi = 0, mask = 0;
    int *h_lo = hist, *h_hi = hist + 256;
    for (int sh = top; sh >= 0; sh -= 8) {
        if (threadIdx.x < 256) {
            h_lo[threadIdx.x] = 0;
            h_hi[threadIdx.x] = 0;
        }
        __syncthreads();
        for (int i = threadIdx.x; i < n; i += TK_THREADS) {
            const uint32_t x = vals[i];
            if (x == 0xffffffffu) continue;
            const int d = (x >> sh) & 0xffu;
            if ((x & mask) == pre_lo) atomicAdd(&h_lo[d], 1);
            if ((x & mask) == pre_hi) atomicAdd(&h_hi[d], 1);
        }
        __syncthreads();
        const int wid = threadIdx.x >> 5;
        if (wid == 0) warp_find_rank(h_lo, k_lo, &misc[8], &misc[9]);
        if (wid == 1) warp_find_rank(h_hi, k_hi, &misc[10], &misc[11]);
        __syncthreads();
        pre_lo |= (uint32_t)misc[8] << sh;
        pre_hi |= (uint32_t)misc[10] << sh;
        k_lo = misc[9];
        k_hi = misc[11];
        mask |= 0xffu << sh;
    }
    v_lo = pre_lo;
    v_hi = pre_hi;
}

// ---------------------------------------------------------------------------
// packed records (include/fasttrack_b200.h)

FT_DEV Desc rec_desc(const ft_kp_record &r) {
    const uint4 *p = reinterpret_cast<const uint4 *>(r.desc);
    Desc d;
    d.lo = p[0];
    d.hi = p[1];
    return d;
}

FT_DEV Desc rec_desc(const ft_point_record &r) {
    const uint4 *p = reinterpret_cast<const uint4 *>(r.desc);
    Desc d;
    d.lo = p[0];
    d.hi = p[1];
    return d;
}

// ---------------------------------------------------------------------------
// stereo role

struct StereoSmem {
    const ft_kp_record *rtab;  // right table: shared copy (staged) or global
    ft_kp_record *rtab_s;      // shared table region (also the median scratch)
    int *row_start;   // [H+1]
    int *row_cursor;  // [H]
    uint16_t *items;  // [cap]
    uint16_t *binbuf; // [cap]
    int *patch;       // [TK_WARPS][patch_ints]
    int *scan_tmp;    // [32]
    int *misc;        // [16]
    int *hist;        // [512] median digit histograms
};

// One warp's left keypoint, loaded once (every lane issues the same
// broadcast loads, so the values are warp-uniform).
struct LeftKp {
    double u, v;
    int o;
    Desc d;
};

FT_DEV LeftKp load_left(const TrackArgs &a, int64_t lk) {
    LeftKp k;
    // volatile: issued where written (the prefetch before the TMA wait must
    // not be sunk to the first use by the compiler)
    const ft_kp_record *r = a.L.rec + lk;
    if (a.coherent) {
        asm volatile("ld.global.ca.v2.f64 {%0, %1}, [%2];" : "=d"(k.u), "=d"(k.v) : "l"(r));
        asm volatile("ld.global.ca.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(k.d.lo.x), "=r"(k.d.lo.y), "=r"(k.d.lo.z), "=r"(k.d.lo.w)
                     : "l"(r->desc));
        asm volatile("ld.global.ca.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(k.d.hi.x), "=r"(k.d.hi.y), "=r"(k.d.hi.z), "=r"(k.d.hi.w)
                     : "l"(r->desc + 2));
        asm volatile("ld.global.ca.s32 %0, [%1];" : "=r"(k.o) : "l"(&r->octave));
        return k;
    }
    asm volatile("ld.global.nc.v2.f64 {%0, %1}, [%2];" : "=d"(k.u), "=d"(k.v) : "l"(r));
    asm volatile("ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(k.d.lo.x), "=r"(k.d.lo.y), "=r"(k.d.lo.z), "=r"(k.d.lo.w)
                 : "l"(r->desc));
    asm volatile("ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(k.d.hi.x), "=r"(k.d.hi.y), "=r"(k.d.hi.z), "=r"(k.d.hi.w)
                 : "l"(r->desc + 2));
    asm volatile("ld.global.nc.s32 %0, [%1];" : "=r"(k.o) : "l"(&r->octave));
    return k;
}

// Phase 1 (kernels.py:312-345) over the contiguous CSR range of rows
// [floor(v - band), ceil(v + band)] held in shared memory.
static_assert(offsetof(ft_kp_record, v) == 8 && offsetof(ft_kp_record, desc) == 16 &&
                  offsetof(ft_kp_record, octave) == 56 && sizeof(ft_kp_record) == 64,
              "ft_kp_record field offsets used by the shared-memory readers");
// SH: the right table is staged in shared memory (read with 32-bit LDS
// addressing; the generic path serves a table left in global memory).
// LPP: lanes per keypoint (32, or 16 for two keypoints per warp: `lane` is
// then the lane within the keypoint's half and the arg-min stays in it);
// live = false runs no candidates (the idle half of a warp's last pair).
template <bool SH = false, int LPP = 32>
FT_DEV int phase1(const TrackArgs &a, const StereoSmem &sm, const LeftKp &kp, int lane,
                  int &cdist, bool live = true) {
    const double band = a.sp.band_factor * a.sp.scale_pow[clampi(kp.o, 0, FT_MAX_LEVELS - 1)];
    long long r0 = (long long)floor(kp.v - band);
    long long r1 = (long long)ceil(kp.v + band);
    const int H = a.sp.height;
    if (r0 < 0) r0 = 0;
    if (r1 > H - 1) r1 = H - 1;
    uint32_t best = NO_KEY;
    if (!live) r1 = r0 - 1;
    if (SH && r0 <= r1) {
        const unsigned rs = smem_u32(sm.row_start), it = smem_u32(sm.items),
                       tb = smem_u32(sm.rtab_s);
        const int beg = lds_s32(rs + 4 * (unsigned)r0), end = lds_s32(rs + 4 * (unsigned)(r1 + 1));
        for (int ii = beg + lane; ii < end; ii += LPP) {
            const int j = lds_u16(it + 2 * ii);
            const unsigned rec = tb + 64u * (unsigned)j;  // ft_kp_record
            // every field in one round trip, then the predicates
            const int ro = lds_s32(rec + 56);
            const double rv = lds_f64(rec + 8), ru = lds_f64(rec);
            Desc rd;
            rd.lo = lds_v4(rec + 16);
            rd.hi = lds_v4(rec + 32);
            if (ro < kp.o - 1 || ro > kp.o + 1) continue;
            if (fabs(rv - kp.v) > band) continue;
            const double disp = kp.u - ru;
            if (disp < a.sp.min_disparity || disp > a.sp.max_disparity) continue;
            best = min(best, (hamming(kp.d, rd) << 16) | (uint32_t)j);
        }
    } else if (r0 <= r1) {
        const int beg = sm.row_start[r0], end = sm.row_start[r1 + 1];
        for (int ii = beg + lane; ii < end; ii += LPP) {
            const int j = sm.items[ii];
            const ft_kp_record &rr = sm.rtab[j];
            const int ro = rr.octave;
            if (ro < kp.o - 1 || ro > kp.o + 1) continue;
            if (fabs(rr.v - kp.v) > band) continue;
            const double disp = kp.u - rr.u;
            if (disp < a.sp.min_disparity || disp > a.sp.max_disparity) continue;
            best = min(best, (hamming(kp.d, rec_desc(rr)) << 16) | (uint32_t)j);
        }
    }
    if (LPP == 32) {
        best = __reduce_min_sync(FULL, best);
    } else {
#pragma unroll
        for (int sh = LPP / 2; sh > 0; sh >>= 1) best = min(best, __shfl_xor_sync(FULL, best, sh));
    }
    if (best != NO_KEY && (int)(best >> 16) <= a.sp.t_match) {
        cdist = (int)(best >> 16);
        return (int)(best & 0xffffu);
    }
    cdist = 10000;
    return -1;
}

// Phase-2 patch geometry on the keypoint's octave level (kernels.py:371-387).
struct P2Geom {
    int o;
    double s;
    long long xi, yi, wl, wr;
    bool left_ok;
    const uint8_t *lp, *rp;
};

FT_DEV P2Geom p2_geom(const TrackArgs &a, int f, const LeftKp &kp) {
    P2Geom g;
    g.o = clampi(kp.o, 0, a.PL.n_levels - 1);
    g.s = a.sp.scale_pow[g.o];
    const double ulev = kp.u / g.s, vlev = kp.v / g.s;
    g.xi = round_half_even(ulev);
    g.yi = round_half_even(vlev);
    const int hw = a.sp.half_window;
    g.wl = a.PL.widths[g.o];
    g.wr = a.PR.widths[g.o];
    const long long hl = a.PL.heights[g.o];
    g.left_ok = !(g.xi - hw < 0 || g.xi + hw >= g.wl || g.yi - hw < 0 || g.yi + hw >= hl);
    g.lp = a.PL.data + (int64_t)f * a.PL.frame_bytes + a.PL.offsets[g.o];
    g.rp = a.PR.data + (int64_t)f * a.PR.frame_bytes + a.PR.offsets[g.o];
    return g;
}

// SAD sweep + parabola (kernels.py:388-428) on patches staged in `patch`:
// pl [nw][nw] = L - cl, pr [nw][nr] = R.  Every lane returns the same verdict.
FT_DEV bool p2_sweep(const TrackArgs &a, int *patch, const LeftKp &kp, const P2Geom &g,
                     long long xr0, int lane, double &disp_out, double &ur_out, int &sad_out) {
    const int hw = a.sp.half_window, hs = a.sp.half_slide;
    const int nw = 2 * hw + 1, nr = 2 * hs + 2 * hw + 1, noff = 2 * hs + 1;
    const int *pl = patch, *pr = patch + nw * nw;
    int *sads = patch + nw * nw + nw * nr;
    for (int t = lane; t < noff; t += 32) sads[t] = 0;
    __syncwarp();
    for (int t = lane; t < noff * nw; t += 32) {  // job = (offset, row)
        const int oi = t / nw, dy = t - oi * nw;
        const int cr = pr[hw * nr + oi + hw];  // R[yi, xr0 + off]
        const int *lrow = pl + dy * nw;
        const int *rrow = pr + dy * nr + oi;
        int acc = 0;
        for (int dx = 0; dx < nw; ++dx) acc += abs(lrow[dx] + cr - rrow[dx]);
        atomicAdd(&sads[oi], acc);
    }
    __syncwarp();
    int best_sad = 0x7fffffff, best_oi = 0;
    for (int oi = 0; oi < noff; ++oi) {  // strict <: lowest offset wins ties
        const int sv = sads[oi];
        if (sv < best_sad) {
            best_sad = sv;
            best_oi = oi;
        }
    }
    const bool interior = best_oi > 0 && best_oi < noff - 1;
    const int s_m = interior ? sads[best_oi - 1] : 0;
    const int s_p = interior ? sads[best_oi + 1] : 0;
    __syncwarp();
    if (!interior) return false;
    const double d_m = (double)s_m, d_0 = (double)best_sad, d_p = (double)s_p;
    const double denom = d_m + d_p - 2.0 * d_0;
    if (denom <= 0.0) return false;
    const double delta = (d_m - d_p) / (2.0 * denom);
    if (delta < -1.0 || delta > 1.0) return false;
    const double ur_ref = ((double)(xr0 + (best_oi - hs)) + delta) * g.s;
    const double disp = kp.u - ur_ref;
    if (disp < a.sp.min_disparity || disp > a.sp.max_disparity) return false;
    disp_out = disp;
    ur_out = ur_ref;
    sad_out = best_sad;
    return true;
}

// Fixed-size SAD sweep for the default 11x11 window / +-5 slide: the 121
// (offset, row) jobs are spread over the warp with independent accumulators
// (no shared atomics), row partials are summed by the 11 offset lanes, and
// the arg-min over offsets is a redux.sync over (sad << 4 | offset), which
// keeps the reference's "lowest offset on ties" (kernels.py:407-409).
template <int HW, int HS>
FT_DEV bool p2_sweep_fixed(const TrackArgs &a, int *patch, const LeftKp &kp, const P2Geom &g,
                           long long xr0, int lane, double &disp_out, double &ur_out,
                           int &sad_out) {
    constexpr int NW = 2 * HW + 1, NR = 2 * HS + 2 * HW + 1, NOFF = 2 * HS + 1;
    constexpr int NJOB = NOFF * NW, QJ = (NJOB + 31) / 32;
    const int *pl = patch, *pr = patch + NW * NW;
    int *part = patch + NW * NW + NW * NR;  // [NJOB]
    int acc[QJ];
#pragma unroll
    for (int q = 0; q < QJ; ++q) acc[q] = 0;
#pragma unroll
    for (int q = 0; q < QJ; ++q) {
        const int t = lane + 32 * q;
        if (t < NJOB) {
            const int oi = t / NW, dy = t - oi * NW;
            const int cr = pr[HW * NR + oi + HW];  // R[yi, xr0 + off]
            const int *lrow = pl + dy * NW;
            const int *rrow = pr + dy * NR + oi;
#pragma unroll
            for (int dx = 0; dx < NW; ++dx) acc[q] += abs(lrow[dx] + cr - rrow[dx]);
        }
    }
#pragma unroll
    for (int q = 0; q < QJ; ++q) {
        const int t = lane + 32 * q;
        if (t < NJOB) part[t] = acc[q];
    }
    __syncwarp();
    int sad = 0x7fffffff;
    if (lane < NOFF) {
        sad = 0;
#pragma unroll
        for (int dy = 0; dy < NW; ++dy) sad += part[lane * NW + dy];
    }
    __syncwarp();  // patch buffers are reused by the next keypoint
    const unsigned key = lane < NOFF ? ((unsigned)sad << 5) | (unsigned)lane : 0xffffffffu;
    const unsigned best = __reduce_min_sync(FULL, key);
    const int best_oi = (int)(best & 31u), best_sad = (int)(best >> 5);
    const int s_m = __shfl_sync(FULL, sad, best_oi > 0 ? best_oi - 1 : 0);
    const int s_p = __shfl_sync(FULL, sad, best_oi < NOFF - 1 ? best_oi + 1 : 0);
    if (best_oi == 0 || best_oi == NOFF - 1) return false;
    const double d_m = (double)s_m, d_0 = (double)best_sad, d_p = (double)s_p;
    const double denom = d_m + d_p - 2.0 * d_0;
    if (denom <= 0.0) return false;
    const double delta = (d_m - d_p) / (2.0 * denom);
    if (delta < -1.0 || delta > 1.0) return false;
    const double ur_ref = ((double)(xr0 + (best_oi - HS)) + delta) * g.s;
    const double disp = kp.u - ur_ref;
    if (disp < a.sp.min_disparity || disp > a.sp.max_disparity) return false;
    disp_out = disp;
    ur_out = ur_ref;
    sad_out = best_sad;
    return true;
}

// Full per-keypoint stereo step for one warp.  The left patch loads are
// issued before phase 1 (they depend only on the keypoint), so their latency
// hides behind the candidate search; the right strip follows phase 1.
template <int HW, int HS>
FT_DEV void stereo_kp(const TrackArgs &a, const StereoSmem &sm, int *patch, int f, int64_t lk,
                      int64_t rbase, int n_right, const LeftKp &kp, int lane, unsigned *medh) {
    constexpr bool FIXED = HW > 0;
    const int hw = FIXED ? HW : a.sp.half_window;
    const int hs = FIXED ? HS : a.sp.half_slide;
    const int nw = 2 * hw + 1, nr = 2 * hs + 2 * hw + 1;
    constexpr int LPL = FIXED ? ((2 * HW + 1) * (2 * HW + 1) + 31) / 32 : 1;
    constexpr int RPL = FIXED ? ((2 * HW + 1) * (2 * HS + 2 * HW + 1) + 31) / 32 : 1;
    const bool do_p1 = a.smode & FT_STEREO_PHASE1;
    const bool do_ref = a.smode & FT_STEREO_REFINE;

    P2Geom g;
    int lreg[LPL];
    if (do_ref) {
        g = p2_geom(a, f, kp);
        if (FIXED && g.left_ok) {
#pragma unroll
            for (int q = 0; q < LPL; ++q) {
                const int t = lane + 32 * q;
                const int dy = t / nw, dx = t - dy * nw;
                lreg[q] = t < nw * nw ? ld_in(a, g.lp + (g.yi - hw + dy) * g.wl + (g.xi - hw + dx)) : 0;
            }
        }
    }
    int cand, cdist;
    const bool tlw = (a.tl != nullptr) && threadIdx.x < 32 && lk == (int64_t)f * a.L.cap +
                     blockIdx.x % (a.Gs + a.Gm) * ((min(a.L.count[f], a.L.cap) + a.Gs - 1) / a.Gs);
    if (tlw && lane == 0) a.tl[blockIdx.x * TL_SLOTS + 8] = global_ns();
    if (do_p1) {
        cand = phase1(a, sm, kp, lane, cdist);
        if (tlw && lane == 0) a.tl[blockIdx.x * TL_SLOTS + 9] = global_ns();
        if (lane == 0 && a.so.cand_idx) {
            a.so.cand_idx[lk] = cand;
            a.so.cand_dist[lk] = cdist;
        }
    } else {
        cand = (int)a.so.cand_idx[lk];
        cdist = (int)a.so.cand_dist[lk];
    }
    if (!(do_ref || (a.smode & FT_STEREO_FROM_CAND))) return;
    bool ok = false;
    double disp = 0.0, ur = 0.0;
    int sad = 0;
    if (cand >= 0 && cand < n_right) {
        const double urc = do_p1 ? sm.rtab[cand].u : ld_in(a, &a.R.rec[rbase + cand].u);
        if (do_ref) {
            if (g.left_ok) {
                const long long xr0 = round_half_even(urc / g.s);
                const long long hr = a.PR.heights[g.o];
                if (!(xr0 - hs - hw < 0 || xr0 + hs + hw >= g.wr || g.yi - hw < 0 ||
                      g.yi + hw >= hr)) {
                    int *pl = patch, *pr = patch + nw * nw;
                    if (FIXED) {
                        int rreg[RPL];
#pragma unroll
                        for (int q = 0; q < RPL; ++q) {
                            const int t = lane + 32 * q;
                            const int dy = t / nr, dx = t - dy * nr;
                            rreg[q] = t < nw * nr
                                          ? ld_in(a, g.rp + (g.yi - hw + dy) * g.wr + (xr0 - hs - hw + dx))
                                          : 0;
                        }
                        const int c_idx = hw * nw + hw;  // centre pixel of the left patch
                        const int cl = __shfl_sync(FULL, lreg[c_idx / 32], c_idx % 32);
#pragma unroll
                        for (int q = 0; q < LPL; ++q) {
                            const int t = lane + 32 * q;
                            if (t < nw * nw) pl[t] = lreg[q] - cl;
                        }
#pragma unroll
                        for (int q = 0; q < RPL; ++q) {
                            const int t = lane + 32 * q;
                            if (t < nw * nr) pr[t] = rreg[q];
                        }
                    } else {
                        const int cl = ld_in(a, g.lp + g.yi * g.wl + g.xi);
                        for (int t = lane; t < nw * nw; t += 32) {
                            const int dy = t / nw, dx = t - dy * nw;
                            pl[t] = (int)ld_in(a, g.lp + (g.yi - hw + dy) * g.wl + (g.xi - hw + dx)) - cl;
                        }
                        for (int t = lane; t < nw * nr; t += 32) {
                            const int dy = t / nr, dx = t - dy * nr;
                            pr[t] = ld_in(a, g.rp + (g.yi - hw + dy) * g.wr + (xr0 - hs - hw + dx));
                        }
                    }
                    // every lane's patch elements are stored before any lane
                    // reads its neighbours' (independent thread scheduling;
                    // found by compute-sanitizer racecheck)
                    __syncwarp();
                    if (tlw && lane == 0) a.tl[blockIdx.x * TL_SLOTS + 10] = global_ns();
                    if constexpr (FIXED)
                        ok = p2_sweep_fixed<HW, HS>(a, patch, kp, g, xr0, lane, disp, ur, sad);
                    else
                        ok = p2_sweep(a, patch, kp, g, xr0, lane, disp, ur, sad);
                    if (tlw && lane == 0) a.tl[blockIdx.x * TL_SLOTS + 11] = global_ns();
                }
            }
        } else {  // matches_from_candidates (stereo.py:154-160)
            disp = kp.u - urc;
            ok = !(disp < a.sp.min_disparity || disp > a.sp.max_disparity);
            ur = urc;
        }
    }
    if (lane == 0) {
        if (ok && medh) {  // SAD-median histogram of the frame (fire-and-forget reds)
            const uint32_t x = (uint32_t)sad;
            atomicAdd(medh + (x < MED_FINE ? x / MED_CW : MED_NC), 1u);
            if (x < MED_FINE) atomicAdd(medh + 128 + x, 1u);
        }
        a.so.right_idx[lk] = ok ? cand : -1;
        a.so.distance[lk] = ok ? cdist : 10000;
        a.so.disparity[lk] = ok ? disp : 0.0;
        a.so.refined_u[lk] = ok ? ur : 0.0;
        a.so.depth[lk] = ok ? a.sp.baseline_times_fx / disp : 0.0;
        a.so.sad[lk] = ok ? sad : 0;
        if (tlw) a.tl[blockIdx.x * TL_SLOTS + 12] = global_ns();
    }
}

// ---------------------------------------------------------------------------
// Block-batched stereo for the default 11x11 window / +-5 slide with phase 1
// and phase 2 in the launch.  The per-keypoint scalar work -- level
// geometry with its fp64 divisions, the parabola, depth and the six output
// stores -- runs one THREAD per keypoint instead of once per warp per
// keypoint, and the warps' SAD loop only streams patches.  Per batch of up
// to KB_N keypoints of the block's range:
//   records -> shared memory (one TMA bulk copy; the first batch's copy is
//     issued before the right table's CSR is built)
//   B  warp per keypoint: phase 1 over the shared row band -> cand, cdist
//   G  thread per keypoint: level geometry, the right strip's column and
//      bounds -> patch row addresses; the keypoints with a SAD sweep to run
//      are compacted into a list (block scan)
//   C  warp per listed keypoint, one item ahead: cp.async of item j+1's
//      left patch and right strip while item j's SAD sweep runs -> the best
//      offset and its neighbours' SADs
//   D  thread per keypoint: parabola, disparity range, depth, outputs
//      (coalesced), SAD-median histogram
// Results are those of stereo_kp<5, 5> (same predicates, same order).
// Patch rows are copied as whole 16-B chunks (2 per left row, 3 per right
// row; the bytes of a row start at (row address & 15) inside its chunks);
// a chunk reaching outside the level's bytes is copied byte by byte (only
// the in-level bytes).
constexpr int PIPE_LROW = 48, PIPE_RROW = 48;  // bytes per staged row (2-way banks)
constexpr int PIPE_SLOT = 11 * PIPE_LROW + 11 * PIPE_RROW;  // 1056 B per keypoint
#ifndef FT_PIPE_NS
#define FT_PIPE_NS 3
#endif
constexpr int PIPE_NS = FT_PIPE_NS;                         // patch slots per warp
constexpr int PIPE_PART = PIPE_NS * PIPE_SLOT;              // SAD partials [121] int
constexpr int PIPE_WARP = PIPE_PART + 496;                  // per-warp buffer
#ifndef FT_P1_PAIRS
#define FT_P1_PAIRS 1  // two keypoints per warp in phase 1 (+2-3 % ring, ab4)
#endif
#ifndef FT_KB_N
#define FT_KB_N 384  // one batch per stereo block at 20 step groups (320 keypoints); 256: +6 % slower there
#endif
constexpr int KB_N = FT_KB_N;  // keypoints per batch (<= TK_THREADS: G and D run a thread each)
static_assert(KB_N <= TK_THREADS, "one thread per batch keypoint");                                   // keypoints per batch
struct KbMeta {  // one keypoint between the passes (40 B)
    unsigned long long lrow0, rrow0;  // patch row 0 (left) / strip row 0 (right)
    int xr0, cand;
    short cdist;
    unsigned char o, state;        // state 1: SAD sweep to run
    unsigned char loff, lw, roff, rw;  // row 0 address & 15, row pitch & 15
    unsigned short wl, wr;         // row pitches (level widths)
    unsigned char inside, pad_[3];  // 1: every 16-B chunk of both patches is in its level
};
static_assert(sizeof(KbMeta) == 40, "KbMeta is 40 B");
// byte offsets inside the stereo patch region (16-B aligned)
constexpr int KB_REC = TK_WARPS * PIPE_WARP;  // ft_kp_record [KB_N]
constexpr int KB_META = KB_REC + KB_N * 64;   // KbMeta [KB_N]
constexpr int KB_SAD = KB_META + KB_N * 40;   // int4 (best offset, s-, s0, s+) [KB_N]
constexpr int KB_LIST = KB_SAD + KB_N * 16;   // uint16 [KB_N]
constexpr int KB_END = KB_LIST + KB_N * 2;
// per-warp share of the region (the host sizes patch_ints from it)
constexpr int PIPE_BYTES = ((KB_END + TK_WARPS - 1) / TK_WARPS + 15) & ~15;
static_assert(KB_REC % 16 == 0 && KB_META % 16 == 0 && KB_SAD % 16 == 0, "16-B aligned");

FT_DEV void cp_async16(void *smem_dst, const void *gsrc) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem_dst)),
                 "l"(gsrc)
                 : "memory");
}
FT_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
FT_DEV void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// One 16-B chunk of pyramid bytes at gsrc (16-B aligned) into shared memory;
// bytes outside [beg, end) are not read (and left as they are).
FT_DEV void pipe_chunk(unsigned char *dst, const unsigned char *gsrc, const unsigned char *beg,
                       const unsigned char *end, bool coherent) {
    if (gsrc >= beg && gsrc + 16 <= end) {
        cp_async16(dst, gsrc);
        return;
    }
    for (int b = 0; b < 16; ++b)
        if (gsrc + b >= beg && gsrc + b < end) dst[b] = coherent ? __ldca(gsrc + b) : __ldg(gsrc + b);
}

FT_DEV unsigned long long lds_u64(unsigned a) {
    unsigned long long v;
    asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(a));
    return v;
}

// Records of keypoints [kb, kb + nb) -> the batch area (thread 0).
FT_DEV void kb_issue_records(const TrackArgs &a, const StereoSmem &sm, int64_t lbase, int kb,
                             int nb, unsigned long long *mbar1) {
    fence_proxy_async_smem();
    mbar_arrive_expect_tx(mbar1, 64u * (unsigned)nb);
    bulk_g2s(reinterpret_cast<unsigned char *>(sm.patch) + KB_REC, a.L.rec + lbase + kb,
             64u * (unsigned)nb, mbar1);
}

__device__ void stereo_block_pipe55(const TrackArgs &a, const StereoSmem &sm, int f, int64_t lbase,
                                    int k0, int k1, int n_right, unsigned *medh,
                                    unsigned long long *mbar1, unsigned &mphase) {
    constexpr int HW = 5, HS = 5, NW = 11, NOFF = 11;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const bool coh = a.coherent;
    unsigned char *pb = reinterpret_cast<unsigned char *>(sm.patch);
    const unsigned base = smem_u32(pb);  // shared addresses for the warp loops
    const unsigned wbs = base + wid * PIPE_WARP, pt = wbs + PIPE_PART;
    const ft_kp_record *krec = reinterpret_cast<const ft_kp_record *>(pb + KB_REC);
    KbMeta *km = reinterpret_cast<KbMeta *>(pb + KB_META);
    int4 *ks = reinterpret_cast<int4 *>(pb + KB_SAD);
    uint16_t *list = reinterpret_cast<uint16_t *>(pb + KB_LIST);
    const uint8_t *lframe = a.PL.data + (int64_t)f * a.PL.frame_bytes;
    const uint8_t *rframe = a.PR.data + (int64_t)f * a.PR.frame_bytes;
    for (int kb = k0, bt = 0; kb < k1; kb += KB_N, ++bt) {
        const int nb = min(KB_N, k1 - kb);
        if (bt > 0 && threadIdx.x == 0) kb_issue_records(a, sm, lbase, kb, nb, mbar1);
        mbar_wait(mbar1, (mphase >> 1) & 1u);  // bit 1: phase of mbar[1]
        mphase ^= 2u;
        // ---- B: phase 1, warp per keypoint (kernels.py:312-345)
#if FT_P1_PAIRS  // FT_P1_PAIRS keypoints per warp (2 or 4), 32 / that lanes each
        constexpr int KPW = FT_P1_PAIRS >= 4 ? 4 : 2, LW = 32 / KPW;
        for (int i2 = KPW * wid; i2 < nb; i2 += KPW * TK_WARPS) {
            const int h = lane / LW, hl = lane % LW, i = i2 + h;
            const bool live = i < nb;
            const unsigned r = base + KB_REC + 64u * (unsigned)(live ? i : i2);
#else
        for (int i = wid; i < nb; i += TK_WARPS) {
            constexpr bool live = true;
            const int hl = lane;
            const unsigned r = base + KB_REC + 64u * (unsigned)i;
#endif
            LeftKp kp;
            kp.u = lds_f64(r);
            kp.v = lds_f64(r + 8);
            kp.d.lo = lds_v4(r + 16);
            kp.d.hi = lds_v4(r + 32);
            kp.o = lds_s32(r + 56);
            int cdist;
            constexpr int LPP = FT_P1_PAIRS ? (FT_P1_PAIRS >= 4 ? 8 : 16) : 32;
            const int cand = a.stage_rdesc ? phase1<true, LPP>(a, sm, kp, hl, cdist, live)
                                           : phase1<false, LPP>(a, sm, kp, hl, cdist, live);
            if (live && hl == 0) {
                km[i].cand = cand;
                km[i].cdist = (short)cdist;
            }
        }
        __syncthreads();
        if (bt == 0) TL_MARK(a, 8);
        // ---- G: geometry, thread per keypoint (kernels.py:371-397)
        const int i = threadIdx.x;
        int need = 0;
        if (i < nb) {
            LeftKp kp;
            kp.u = krec[i].u;
            kp.v = krec[i].v;
            kp.o = krec[i].octave;
            const P2Geom g = p2_geom(a, f, kp);
            KbMeta m = km[i];
            const int64_t lk = lbase + kb + i;
            if (a.so.cand_idx) {
                a.so.cand_idx[lk] = m.cand;
                a.so.cand_dist[lk] = m.cdist;
            }
            long long xr0 = 0;
            const uint8_t *rrow0 = nullptr;
            m.state = 0;
            if (m.cand >= 0 && m.cand < n_right && g.left_ok) {
                xr0 = round_half_even(sm.rtab[m.cand].u / g.s);
                const long long hr = a.PR.heights[g.o];
                if (!(xr0 - HS - HW < 0 || xr0 + HS + HW >= g.wr || g.yi - HW < 0 ||
                      g.yi + HW >= hr)) {
                    m.state = 1;
                    rrow0 = g.rp + (g.yi - HW) * g.wr + (xr0 - HS - HW);
                }
            }
            const uint8_t *lrow0 = g.lp + (g.yi - HW) * g.wl + (g.xi - HW);
            m.lrow0 = (unsigned long long)lrow0;
            m.rrow0 = (unsigned long long)rrow0;
            m.xr0 = (int)xr0;
            m.o = (unsigned char)g.o;
            m.loff = (unsigned char)((uintptr_t)lrow0 & 15);
            m.lw = (unsigned char)(g.wl & 15);
            m.roff = (unsigned char)((uintptr_t)rrow0 & 15);
            m.rw = (unsigned char)(g.wr & 15);
            m.wl = (unsigned short)g.wl;
            m.wr = (unsigned short)g.wr;
            m.inside = 0;
            if (m.state) {  // all chunks of both patches inside their levels: no per-chunk checks
                const uintptr_t l0 = (uintptr_t)lrow0 & ~(uintptr_t)15,
                                l1 = (((uintptr_t)lrow0 + 10 * g.wl) & ~(uintptr_t)15) + 32,
                                r0 = (uintptr_t)rrow0 & ~(uintptr_t)15,
                                r1 = (((uintptr_t)rrow0 + 10 * g.wr) & ~(uintptr_t)15) + 48;
                const uintptr_t lb0 = (uintptr_t)g.lp, lb1 = lb0 + g.wl * a.PL.heights[g.o];
                const uintptr_t rb0 = (uintptr_t)g.rp, rb1 = rb0 + g.wr * a.PR.heights[g.o];
                m.inside = l0 >= lb0 && l1 <= lb1 && r0 >= rb0 && r1 <= rb1;
            }
            km[i] = m;
            need = m.state;
        }
        int nl;
        const int pos = block_exclusive_scan<TK_THREADS>(need, sm.scan_tmp, nl);
        if (need) list[pos] = (uint16_t)i;
        __syncthreads();
        if (bt == 0) TL_MARK(a, 9);
        // ---- C: SAD sweeps (kernels.py:388-409), warp per listed keypoint
        // per-lane chunk of the copies: left (row lane / 2, chunk lane & 1)
        // for lanes < 22, right (row lane / 3, chunk lane % 3) and, lane 0,
        // the right strip's 33rd chunk (row 10, chunk 2)
        const int lcr = lane >> 1, lcq = lane & 1, rcr = lane / 3, rcq = lane - 3 * (lane / 3);
        auto issue = [&](int j, int sl) {  // item j's patches -> slot sl
            const unsigned mr = base + KB_META + 40u * (unsigned)lds_u16(base + KB_LIST + 2u * j);
            const uint8_t *lrow0 = reinterpret_cast<const uint8_t *>(lds_u64(mr));
            const uint8_t *rrow0 = reinterpret_cast<const uint8_t *>(lds_u64(mr + 8));
            const int wlr = lds_s32(mr + 32);
            unsigned char *lb = pb + wid * PIPE_WARP + sl * PIPE_SLOT;
            unsigned char *rb = lb + 11 * PIPE_LROW;
            if (lds_u8(mr + 36)) {  // interior: plain 16-B copies
                const int wl = wlr & 0xffff, wr = (wlr >> 16) & 0xffff;
                if (lane < 2 * NW) {
                    const uintptr_t c0 = ((uintptr_t)lrow0 + lcr * wl) & ~(uintptr_t)15;
                    cp_async16(lb + lcr * PIPE_LROW + 16 * lcq,
                               reinterpret_cast<const void *>(c0 + 16 * lcq));
                }
                {
                    const uintptr_t c0 = ((uintptr_t)rrow0 + rcr * wr) & ~(uintptr_t)15;
                    cp_async16(rb + rcr * PIPE_RROW + 16 * rcq,
                               reinterpret_cast<const void *>(c0 + 16 * rcq));
                }
                if (lane == 0) {
                    const uintptr_t c0 = ((uintptr_t)rrow0 + 10 * wr) & ~(uintptr_t)15;
                    cp_async16(rb + 10 * PIPE_RROW + 32, reinterpret_cast<const void *>(c0 + 32));
                }
                return;
            }
            const int o = lds_u8(mr + 26);
            const long long wl = a.PL.widths[o], wr = a.PR.widths[o];
            const uint8_t *lp = lframe + a.PL.offsets[o], *rp = rframe + a.PR.offsets[o];
            if (lane < 2 * NW) {  // chunks bounded by the level's own bytes
                const uint8_t *row = lrow0 + (lane >> 1) * wl;
                const uint8_t *c0 = reinterpret_cast<const uint8_t *>((uintptr_t)row & ~(uintptr_t)15);
                pipe_chunk(lb + (lane >> 1) * PIPE_LROW + 16 * (lane & 1), c0 + 16 * (lane & 1), lp,
                           lp + wl * a.PL.heights[o], coh);
            }
            for (int c = lane; c < 3 * NW; c += 32) {
                const int r = c / 3, q = c - 3 * r;
                const uint8_t *row = rrow0 + r * wr;
                const uint8_t *c0 = reinterpret_cast<const uint8_t *>((uintptr_t)row & ~(uintptr_t)15);
                pipe_chunk(rb + r * PIPE_RROW + 16 * q, c0 + 16 * q, rp, rp + wr * a.PR.heights[o], coh);
            }
        };
        // PIPE_NS slots per warp: items PIPE_NS - 1 ahead are in flight
        int j = wid;
#pragma unroll
        for (int q = 0; q < PIPE_NS - 1; ++q) {
            if (j + q * TK_WARPS < nl) issue(j + q * TK_WARPS, q);
            cp_async_commit();
        }
        for (int t = 0; j < nl; j += TK_WARPS, ++t) {
            const int sl = t % PIPE_NS;
            const int ja = j + (PIPE_NS - 1) * TK_WARPS;
            if (ja < nl) issue(ja, (t + PIPE_NS - 1) % PIPE_NS);
            cp_async_commit();
            cp_async_wait<PIPE_NS - 1>();  // item j's patches
            __syncwarp();
            const int idx = lds_u16(base + KB_LIST + 2u * j);
            const unsigned mr = base + KB_META + 40u * (unsigned)idx;
            const int pk = lds_s32(mr + 28);  // loff, lw, roff, rw
            const int loff = pk & 255, lw = (pk >> 8) & 255, roff = (pk >> 16) & 255,
                      rw = (pk >> 24) & 255;
            const unsigned lb = wbs + sl * PIPE_SLOT, rb = lb + 11 * PIPE_LROW;
            // centre pixels: cl = L[yi, xi], cr(oi) = R[yi, xr0 + oi - HS]
            const int lo5 = (loff + HW * lw) & 15, ro5 = (roff + HW * rw) & 15;
            const int cl = lds_u8(lb + HW * PIPE_LROW + lo5 + HW);
            // lane (g, dy), 22 lanes: row dy, offsets 6g .. 6g + 5 (g = 1: .. 10).
            // A lane reads its left row once (11 B) and the 16 right bytes its
            // offsets cover, then runs 6 independent VABSDIFF chains (|x - y| +
            // acc): 33 LDS per lane instead of 22 per (offset, row) job.
            const int g = lane < 11 ? 0 : (lane < 22 ? 1 : 2), dy = lane - 11 * g;
            if (g < 2) {
                const int o0 = 6 * g;
                const int lo = (loff + dy * lw) & 15, ro = (roff + dy * rw) & 15;
                const unsigned lr = lb + dy * PIPE_LROW + lo;
                const unsigned rr = rb + dy * PIPE_RROW + ro + o0;  // + 15 stays in the row
                const unsigned rc = rb + HW * PIPE_RROW + ro5 + HW + o0;
                int L[NW], Rv[16], cc[6], acc[6];
#pragma unroll
                for (int dx = 0; dx < NW; ++dx) L[dx] = lds_u8(lr + dx);
#pragma unroll
                for (int x = 0; x < 16; ++x) Rv[x] = lds_u8(rr + x);
#pragma unroll
                for (int k = 0; k < 6; ++k) cc[k] = lds_u8(rc + k) - cl;  // cr - cl
#pragma unroll
                for (int k = 0; k < 6; ++k) acc[k] = 0;
#pragma unroll
                for (int dx = 0; dx < NW; ++dx)
#pragma unroll
                    for (int k = 0; k < 6; ++k)
                        acc[k] = (int)__sad(L[dx] + cc[k], Rv[k + dx], (unsigned)acc[k]);
#pragma unroll
                for (int k = 0; k < 6; ++k)
                    if (o0 + k < NOFF) sts_s32(pt + 4 * ((o0 + k) * NW + dy), acc[k]);
            }
            __syncwarp();
            int sv = 0x7fffffff;
            if (lane < NOFF) {
                sv = 0;
#pragma unroll
                for (int d = 0; d < NW; ++d) sv += lds_s32(pt + 4 * (lane * NW + d));
            }
            const unsigned key = lane < NOFF ? ((unsigned)sv << 5) | (unsigned)lane : 0xffffffffu;
            const unsigned best = __reduce_min_sync(FULL, key);
            const int best_oi = (int)(best & 31u), best_sad = (int)(best >> 5);
            const int s_m = __shfl_sync(FULL, sv, best_oi > 0 ? best_oi - 1 : 0);
            const int s_p = __shfl_sync(FULL, sv, best_oi < NOFF - 1 ? best_oi + 1 : 0);
            if (lane == 0) ks[idx] = make_int4(best_oi, s_m, best_sad, s_p);
            __syncwarp();  // slot sl and the partials are refilled next iteration
        }
        cp_async_wait<0>();
        __syncthreads();
        if (bt == 0) TL_MARK(a, 10);
        // ---- D: parabola + outputs, thread per keypoint (kernels.py:410-428)
        if (i < nb) {
            const KbMeta m = km[i];
            const int64_t lk = lbase + kb + i;
            bool ok = false;
            double disp = 0.0, ur = 0.0;
            int sad = 0;
            if (m.state) {
                const int4 r = ks[i];
                const int best_oi = r.x, best_sad = r.z;
                if (best_oi > 0 && best_oi < NOFF - 1) {
                    const double d_m = (double)r.y, d_0 = (double)best_sad, d_p = (double)r.w;
                    const double denom = d_m + d_p - 2.0 * d_0;
                    if (denom > 0.0) {
                        const double delta = (d_m - d_p) / (2.0 * denom);
                        if (!(delta < -1.0 || delta > 1.0)) {
                            const double s = a.sp.scale_pow[m.o];
                            const double ur_ref = ((double)((long long)m.xr0 + (best_oi - HS)) + delta) * s;
                            const double dsp = krec[i].u - ur_ref;
                            if (!(dsp < a.sp.min_disparity || dsp > a.sp.max_disparity)) {
                                ok = true;
                                disp = dsp;
                                ur = ur_ref;
                                sad = best_sad;
                            }
                        }
                    }
                }
            }
            if (ok && medh) {  // SAD-median histogram of the frame (fire-and-forget reds)
                const uint32_t x = (uint32_t)sad;
                atomicAdd(medh + (x < MED_FINE ? x / MED_CW : MED_NC), 1u);
                if (x < MED_FINE) atomicAdd(medh + 128 + x, 1u);
            }
            a.so.right_idx[lk] = ok ? m.cand : -1;
            a.so.distance[lk] = ok ? (int)m.cdist : 10000;
            a.so.disparity[lk] = ok ? disp : 0.0;
            a.so.refined_u[lk] = ok ? ur : 0.0;
            a.so.depth[lk] = ok ? a.sp.baseline_times_fx / disp : 0.0;
            a.so.sad[lk] = ok ? sad : 0;
        }
        __syncthreads();  // the batch area is refilled by the next batch
    }
}

// np.median (stereo.py:180) of a group's accepted SADs from its histograms
// (warp 0): coarse bins locate the bins of ranks (n-1)/2 and n/2, one fine
// read resolves them.  misc[4] = n, misc[7] = resolved (0: the median lies
// at or above MED_FINE -- decide from the values), misc[8] / misc[10] = the
// two order statistics.
FT_DEV void warp_hist_median(const unsigned *hb, int lane, int *misc) {
    const unsigned c0 = __ldcg(hb + 2 * lane), c1 = __ldcg(hb + 2 * lane + 1);
    const unsigned ov = __ldcg(hb + MED_NC);
    const int sl = (int)(c0 + c1);
    int incl = sl;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int y = __shfl_up_sync(FULL, incl, d);
        if (lane >= d) incl += y;
    }
    const int below = __shfl_sync(FULL, incl, 31);
    const int nm = below + (int)ov;
    const int k_lo = (nm - 1) / 2, k_hi = nm / 2;
    const bool fast = nm == 0 || k_hi < below;
    int v[2] = {0, 0};
    if (nm > 0 && fast) {
        const int excl = incl - sl;
        int bin[2], rk[2];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const int kk = q ? k_hi : k_lo;
            const unsigned bl = __ballot_sync(FULL, excl <= kk && kk < incl);
            const int src = __ffs(bl) - 1;
            const int e = __shfl_sync(FULL, excl, src);
            const int cz = __shfl_sync(FULL, (int)c0, src);
            bin[q] = kk < e + cz ? 2 * src : 2 * src + 1;
            rk[q] = kk < e + cz ? kk - e : kk - e - cz;
        }
        const unsigned *fb = hb + 128;
        const unsigned f0 = __ldcg(fb + bin[0] * MED_CW + 2 * lane);
        const unsigned f1 = __ldcg(fb + bin[0] * MED_CW + 2 * lane + 1);
        const unsigned g0 = __ldcg(fb + bin[1] * MED_CW + 2 * lane);
        const unsigned g1 = __ldcg(fb + bin[1] * MED_CW + 2 * lane + 1);
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const int a0 = (int)(q ? g0 : f0), a1 = (int)(q ? g1 : f1);
            int in2 = a0 + a1;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int y = __shfl_up_sync(FULL, in2, d);
                if (lane >= d) in2 += y;
            }
            const int ex2 = in2 - a0 - a1;
            const unsigned bl = __ballot_sync(FULL, ex2 <= rk[q] && rk[q] < in2);
            const int src = __ffs(bl) - 1;
            const int e = __shfl_sync(FULL, ex2, src);
            const int cz = __shfl_sync(FULL, a0, src);
            v[q] = bin[q] * MED_CW + 2 * src + (rk[q] < e + cz ? 0 : 1);
        }
    }
    if (lane == 0) {
        misc[4] = nm;
        misc[7] = fast;
        misc[8] = v[0];
        misc[10] = v[1];
    }
}

// shared table region of a stereo block: the staged right table, or at least
// the median scratch (4 B per left keypoint)
__host__ __device__ inline size_t stereo_table_bytes(const TrackArgs &a) {
    const size_t t = a.stage_rdesc ? (size_t)64 * a.R.cap : 0;
    const size_t m = (size_t)4 * a.L.cap;
    return ((t > m ? t : m) + 15) & ~(size_t)15;
}

// The frame's stereo tail in one block (tail mode): every keypoint's
// (right_idx, sad) into shared memory, the median of the accepted SADs (the
// group histograms when this launch produced them, else radix select over
// the values), rejection (stereo.py:171-188) and the match count.
__device__ void stereo_tail(const TrackArgs &a, const StereoSmem &sm, int f, int slot,
                            int n_left, int64_t lbase, bool med_h) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const bool do_rej = a.smode & FT_STEREO_REJECT;
    uint32_t *vals = reinterpret_cast<uint32_t *>(sm.rtab_s);  // table no longer needed
    const unsigned ep = med_h ? (unsigned)sm.misc[6] : 0u;
    const unsigned *hb = med_h ? a.med + ((size_t)slot * 3 + ep % 3u) * MED_WS : nullptr;
    if (threadIdx.x == 0) {
        sm.misc[4] = 0;
        sm.misc[5] = 0;
        sm.misc[12] = 0;
    }
    __syncthreads();
    if (med_h && do_rej && wid == 0) warp_hist_median(hb, lane, sm.misc);
    int cnt = 0;
    uint32_t vmax = 0;
    for (int k = threadIdx.x; k < n_left; k += TK_THREADS) {
        const bool m = __ldcg(a.so.right_idx + lbase + k) >= 0;
        const uint32_t x = m ? (uint32_t)__ldcg(a.so.sad + lbase + k) : 0xffffffffu;
        vals[k] = x;
        cnt += m;
        if (m) vmax = max(vmax, x);
    }
    cnt = __reduce_add_sync(FULL, cnt);
    vmax = __reduce_max_sync(FULL, vmax);
    __syncthreads();  // warp 0's histogram result in misc[4, 7, 8, 10]
    const bool resolved = med_h && do_rej && sm.misc[7];
    if (lane == 0) {
        atomicAdd(&sm.misc[12], cnt);
        atomicMax(reinterpret_cast<unsigned *>(&sm.misc[5]), vmax);
    }
    __syncthreads();
    const int nm = sm.misc[12];
    int kept = 0;
    if (do_rej && nm > 0) {
        uint32_t v_lo, v_hi;
        if (resolved) {
            v_lo = (uint32_t)sm.misc[8];
            v_hi = (uint32_t)sm.misc[10];
        } else {
            const size_t vbytes = ((size_t)4 * a.L.cap + 15) & ~(size_t)15;
            if ((uint32_t)sm.misc[5] < (uint32_t)MED_SMALL_BINS &&
                stereo_table_bytes(a) >= vbytes + 4 * (size_t)MED_SMALL_BINS)
                block_median_pair_small(vals, n_left, nm,
                                        reinterpret_cast<int *>(
                                            reinterpret_cast<unsigned char *>(sm.rtab_s) + vbytes),
                                        sm.scan_tmp, sm.misc, v_lo, v_hi);
            else
                block_median_pair(vals, n_left, nm, (uint32_t)sm.misc[5], sm.hist, sm.misc, v_lo,
                                  v_hi);
        }
        const double med = (nm & 1) ? (double)v_lo : ((double)v_lo + (double)v_hi) / 2.0;
        const double thr = a.sp.outlier_multiplier * med;
        TL_MARK(a, 14);
        for (int k = threadIdx.x; k < n_left; k += TK_THREADS) {
            const uint32_t x = vals[k];
            if (x == 0xffffffffu) continue;
            if ((double)x > thr) {
                const int64_t i = lbase + k;
                a.so.right_idx[i] = -1;
                a.so.distance[i] = 10000;
                a.so.disparity[i] = 0.0;
                a.so.refined_u[i] = 0.0;
                a.so.depth[i] = 0.0;
                a.so.sad[i] = 0;
            } else {
                ++kept;
            }
        }
    } else {
        for (int k = threadIdx.x; k < n_left; k += TK_THREADS) kept += vals[k] != 0xffffffffu;
    }
    if (a.so.n_matched) {
        kept = __reduce_add_sync(FULL, kept);
        if (lane == 0 && kept) atomicAdd(a.so.n_matched + f, kept);
    }
    if (med_h) {  // next instance's histogram buffer: zero (nobody else is on it)
        unsigned *nb = a.med + ((size_t)slot * 3 + (ep + 1u) % 3u) * MED_WS;
        for (int i = threadIdx.x; i < MED_WS; i += TK_THREADS) nb[i] = 0u;
    }
    __syncthreads();  // smem reuse by the next frame of this block
}

__device__ void stereo_frame(const TrackArgs &a, int f, int rank, int slot,
                             unsigned char *smem, unsigned long long *mbar, unsigned &mphase,
                             unsigned &bpar) {
    unsigned long long *bar = a.bar_s + 2 * slot;
    const int G = a.Gs;
    const int n_left = min(a.L.count[f], a.L.cap);
    const int n_right = min(a.R.count[f], a.R.cap);
    const int64_t lbase = (int64_t)f * a.L.cap, rbase = (int64_t)f * a.R.cap;
    // tail mode: rank G-1 is the group's tail block (no keypoints)
    const int Gw = a.stereo_tail ? G - 1 : G;
    const int chunk = (n_left + Gw - 1) / Gw;
    const int k0 = rank < Gw ? rank * chunk : n_left, k1 = min(n_left, k0 + chunk);
    const int H = a.sp.height;
    const bool do_p1 = a.smode & FT_STEREO_PHASE1;
    const bool do_ref = a.smode & FT_STEREO_REFINE;
    const bool do_fc = a.smode & FT_STEREO_FROM_CAND;
    const bool do_rej = a.smode & FT_STEREO_REJECT;
    const bool finalize = do_ref || do_fc;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;

    StereoSmem sm;
    unsigned char *p = smem;
    sm.rtab_s = reinterpret_cast<ft_kp_record *>(p);
    p += stereo_table_bytes(a);
    sm.rtab = a.stage_rdesc ? sm.rtab_s : a.R.rec + rbase;
    sm.scan_tmp = reinterpret_cast<int *>(p);
    p += 32 * 4;
    sm.misc = reinterpret_cast<int *>(p);
    p += 16 * 4;
    sm.hist = reinterpret_cast<int *>(p);
    p += 512 * 4;
    sm.row_start = reinterpret_cast<int *>(p);
    p += (size_t)4 * (H + 1);
    sm.row_cursor = reinterpret_cast<int *>(p);
    p += (size_t)4 * H;
    p = reinterpret_cast<unsigned char *>(((uintptr_t)p + 15) & ~(uintptr_t)15);  // cp.async dst
    sm.patch = reinterpret_cast<int *>(p);
    p += (size_t)4 * TK_WARPS * a.patch_ints;
    sm.items = reinterpret_cast<uint16_t *>(p);
    p += (size_t)2 * a.R.cap;
    sm.binbuf = reinterpret_cast<uint16_t *>(p);

    if (rank == 0 && threadIdx.x == 0 && a.so.n_matched) a.so.n_matched[f] = 0;
    // SAD median through the group's histograms (hot path), see below
    const bool med_h = do_rej && finalize && a.med;  // SADs produced by this launch
    if (med_h && threadIdx.x == 32) sm.misc[6] = (int)group_ticket(a.ep_s + slot, G);
    TL_MARK(a, 0);
    if (threadIdx.x < 32) {  // translate every page the block touches later, now
        const int l = threadIdx.x;
        if (l == 0) prefetch_l2(bar);
        if (l == 1) prefetch_l2(a.so.right_idx ? a.so.right_idx + lbase : nullptr);
        if (l == 2) prefetch_l2(a.so.sad ? a.so.sad + lbase : nullptr);
        if (l == 3) prefetch_l2(a.so.depth ? a.so.depth + lbase : nullptr);
        if (l == 4) prefetch_l2(a.L.rec + lbase + k0);
        if (do_ref && l >= 8 && l < 8 + a.PL.n_levels)
            prefetch_l2(a.PL.data + (int64_t)f * a.PL.frame_bytes + a.PL.offsets[l - 8]);
        if (do_ref && l >= 16 && l < 16 + a.PR.n_levels)
            prefetch_l2(a.PR.data + (int64_t)f * a.PR.frame_bytes + a.PR.offsets[l - 16]);
    }

    // default window with both phases here: the block-batched passes
    // (stereo_block_pipe55; the per-warp timeline debug marks live in
    // stereo_kp only)
    const bool fixed55 = a.sp.half_window == 5 && a.sp.half_slide == 5;
    const bool pipe = fixed55 && do_p1 && do_ref && a.patch_ints * 4 >= PIPE_BYTES;
    if (k0 < k1 && (do_p1 || finalize)) {
        const int kf = k0 + wid;
        LeftKp kp_first;  // issued now: lands while the right table streams in
        if (!pipe && kf < k1) kp_first = load_left(a, lbase + kf);
        if (do_p1) {
            // right keypoint table -> shared memory with TMA bulk copies
            // (pipe: the first batch of left records too, on mbar[1])
            if (threadIdx.x == 0) {
                fence_proxy_async_smem();
                if (pipe) kb_issue_records(a, sm, lbase, k0, min(KB_N, k1 - k0), mbar + 1);
                const unsigned bytes = a.stage_rdesc ? 64u * n_right : 0u;
                mbar_arrive_expect_tx(mbar, bytes);
                if (bytes) bulk_g2s(sm.rtab_s, a.R.rec + rbase, bytes, mbar);
            }
            for (int b = threadIdx.x; b < H; b += TK_THREADS) sm.row_cursor[b] = 0;
            mbar_wait(mbar, mphase & 1u);  // bit 0: phase of mbar[0]
            mphase ^= 1u;
            __syncthreads();  // cursor zeroed, ticket in misc[6]
            TL_MARK(a, 6);
            block_csr<TK_THREADS>(
                n_right, H,
                [&](int j) {
                    long long r = round_half_even(sm.rtab[j].v);  // np.round: half-even
                    return (int)(r < 0 ? 0 : (r > H - 1 ? H - 1 : r));
                },
                sm.row_start, sm.row_cursor, sm.items, sm.binbuf,
                sm.scan_tmp);
        }
        TL_MARK(a, 1);
        if (!do_p1) __syncthreads();  // ticket in misc[6]
        unsigned *medh = med_h ? a.med + ((size_t)slot * 3 + (unsigned)sm.misc[6] % 3u) * MED_WS
                               : nullptr;
        int *patch = sm.patch + wid * a.patch_ints;
        if (pipe) {
            stereo_block_pipe55(a, sm, f, lbase, k0, k1, n_right, medh, mbar + 1, mphase);
        } else
        for (int k = kf; k < k1; k += TK_WARPS) {
            const LeftKp kp = k == kf ? kp_first : load_left(a, lbase + k);
            if (fixed55)
                stereo_kp<5, 5>(a, sm, patch, f, lbase + k, rbase, n_right, kp, lane, medh);
            else
                stereo_kp<0, 0>(a, sm, patch, f, lbase + k, rbase, n_right, kp, lane, medh);
        }
    }
    __syncthreads();
    TL_MARK(a, 2);
    if (!do_rej && !a.so.n_matched) return;
    if (a.stereo_tail) {
        // Tail mode (one frame per group in this launch): no group barrier.
        // The G-1 keypoint blocks publish their results with one release
        // reduction each and are done (persistent mode: on to the next
        // step); the dedicated tail block waits for them and runs the frame's
        // tail -- median, rejection, match count over every keypoint.
        if (rank < Gw) {
            if (threadIdx.x == 0) {
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
                atomicAdd(a.tail_s + slot, 1ull);
            }
            return;
        }
        if (threadIdx.x == 0) {
            while ((uint32_t)ld_acquire_u64(a.tail_s + slot) != (uint32_t)Gw) __nanosleep(20);
            // arrivals back to 0 for the group's next frame (after this one)
            atomicAdd(a.tail_s + slot, (1ull << 32) - (unsigned long long)Gw);
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
        }
        __syncthreads();
        TL_MARK(a, 3);
        stereo_tail(a, sm, f, slot, n_left, lbase, med_h);
        TL_MARK(a, 4);
        return;
    }
    if (med_h) {  // zero this block's share of the next instance's buffer
        const unsigned ep = (unsigned)sm.misc[6];
        unsigned *nb = a.med + ((size_t)slot * 3 + (ep + 1u) % 3u) * MED_WS;
        const int per = (MED_WS + G - 1) / G, z0 = rank * per, z1 = min(MED_WS, z0 + per);
        for (int i = z0 + threadIdx.x; i < z1; i += TK_THREADS) nb[i] = 0u;
    }
    group_barrier(bar, G, bpar);
    TL_MARK(a, 3);
    int kept = 0;
    bool med_done = false;
    if (med_h) {
        // np.median (stereo.py:180) from the group's histograms: coarse bins
        // locate the bins of ranks (n-1)/2 and n/2, one fine read resolves
        // them -- two dependent L2 reads by warp 0 instead of gathering every
        // SAD into every block.  A median among values >= MED_FINE (not seen
        // in practice) takes the gather path below.
        const unsigned ep = (unsigned)sm.misc[6];
        const unsigned *hb = a.med + ((size_t)slot * 3 + ep % 3u) * MED_WS;
        int64_t ri0 = -1;
        uint32_t x0 = 0;
        if (k0 + (int)threadIdx.x < k1) {  // own values, loaded beside the histogram reads
            ri0 = __ldcg(a.so.right_idx + lbase + k0 + threadIdx.x);
            x0 = (uint32_t)__ldcg(a.so.sad + lbase + k0 + threadIdx.x);
        }
        if (wid == 0) warp_hist_median(hb, lane, sm.misc);
        __syncthreads();
        if (sm.misc[7]) {
            med_done = true;
            const int nm = sm.misc[4];
            const uint32_t v_lo = (uint32_t)sm.misc[8], v_hi = (uint32_t)sm.misc[10];
            const double med = (nm & 1) ? (double)v_lo : ((double)v_lo + (double)v_hi) / 2.0;
            const double thr = a.sp.outlier_multiplier * med;
            TL_MARK(a, 14);
            for (int k = k0 + threadIdx.x; k < k1; k += TK_THREADS) {
                int64_t ri = ri0;
                uint32_t x = x0;
                if (k != k0 + (int)threadIdx.x) {
                    ri = __ldcg(a.so.right_idx + lbase + k);
                    x = (uint32_t)__ldcg(a.so.sad + lbase + k);
                }
                if (ri < 0) continue;
                if ((double)x > thr) {
                    const int64_t i = lbase + k;
                    a.so.right_idx[i] = -1;
                    a.so.distance[i] = 10000;
                    a.so.disparity[i] = 0.0;
                    a.so.refined_u[i] = 0.0;
                    a.so.depth[i] = 0.0;
                    a.so.sad[i] = 0;
                } else {
                    ++kept;
                }
            }
        }
    }
    if (do_rej && !med_done) {
        // every block computes the same median over the frame's accepted SADs
        uint32_t *vals = reinterpret_cast<uint32_t *>(sm.rtab_s);  // table no longer needed
        int *hist = sm.hist;
        if (threadIdx.x == 0) {
            sm.misc[4] = 0;
            sm.misc[5] = 0;
        }
        __syncthreads();
        int cnt = 0;
        uint32_t vmax = 0;
        for (int k = threadIdx.x; k < n_left; k += TK_THREADS) {
            const bool m = __ldcg(a.so.right_idx + lbase + k) >= 0;
            const uint32_t x = m ? (uint32_t)__ldcg(a.so.sad + lbase + k) : 0xffffffffu;
            vals[k] = x;
            cnt += m;
            if (m) vmax = max(vmax, x);
        }
        cnt = __reduce_add_sync(FULL, cnt);
        vmax = __reduce_max_sync(FULL, vmax);
        if (lane == 0) {
            atomicAdd(&sm.misc[4], cnt);
            atomicMax(reinterpret_cast<unsigned *>(&sm.misc[5]), vmax);
        }
        // Every block must have gathered the frame's values before any block
        // writes its rejections below (a lagging block would otherwise read
        // right_idx = -1 / sad = 0 of another block's slice and compute a
        // different median).  Uniform across the group: med_done is decided
        // from the same histogram in every block.
        group_barrier(bar, G, bpar);  // includes the block barriers
        TL_MARK(a, 13);
        const int nm = sm.misc[4];
        if (nm > 0) {
            uint32_t v_lo, v_hi;
            // histogram after the values in the (no longer needed) table area
            const size_t vbytes = ((size_t)4 * a.L.cap + 15) & ~(size_t)15;
            if ((uint32_t)sm.misc[5] < (uint32_t)MED_SMALL_BINS &&
                stereo_table_bytes(a) >= vbytes + 4 * (size_t)MED_SMALL_BINS)
                block_median_pair_small(vals, n_left, nm,
                                        reinterpret_cast<int *>(
                                            reinterpret_cast<unsigned char *>(sm.rtab_s) + vbytes),
                                        sm.scan_tmp,
                                        sm.misc, v_lo, v_hi);
            else
                block_median_pair(vals, n_left, nm, (uint32_t)sm.misc[5], hist, sm.misc, v_lo,
                                  v_hi);
            const double med = (nm & 1) ? (double)v_lo : ((double)v_lo + (double)v_hi) / 2.0;
            const double thr = a.sp.outlier_multiplier * med;
            TL_MARK(a, 14);
            for (int k = k0 + threadIdx.x; k < k1; k += TK_THREADS) {
                const uint32_t x = vals[k];
                if (x == 0xffffffffu) continue;
                if ((double)x > thr) {
                    const int64_t i = lbase + k;
                    a.so.right_idx[i] = -1;
                    a.so.distance[i] = 10000;
                    a.so.disparity[i] = 0.0;
                    a.so.refined_u[i] = 0.0;
                    a.so.depth[i] = 0.0;
                    a.so.sad[i] = 0;
                } else {
                    ++kept;
                }
            }
        }
    } else if (!do_rej) {
        for (int k = k0 + threadIdx.x; k < k1; k += TK_THREADS)
            kept += __ldcg(a.so.right_idx + lbase + k) >= 0;
    }
    if (a.so.n_matched) {
        kept = __reduce_add_sync(FULL, kept);
        if (lane == 0 && kept) atomicAdd(a.so.n_matched + f, kept);
    }
    __syncthreads();  // smem reuse by the next frame of this slot
    TL_MARK(a, 4);
}

// ---------------------------------------------------------------------------
// map role

struct QItem {
    double ucen, v, r;
    int li;   // point index within the staged round
    int lvl;
    short cx0, cx1, cy0, cy1;
};

struct MapSmem {
    const ft_kp_record *ktab;  // keypoint table: shared copy (staged) or global
    ft_kp_record *ktab_s;
    long long *kslots;  // [cap_kp] slots_in (hash source)
    int *htab;          // [1 << hash_bits] indices into kslots, -1 = empty
    ft_point_record *prnd;  // staged round of map points
    int *cell_start, *cell_cursor;
    uint16_t *items;
    uint16_t *binbuf;   // [cap_kp]
    QItem *queue;       // [round_cap]
    int *res;           // [chunk] packed claim (kp | dist << 16 | lvl << 25) or -1
    long long *res_pid; // [chunk] id of the claiming point
    int *res_empty;     // [chunk] slots_in[kp] == NO_POINT
    int *scan_tmp, *misc;
    int *hist;  // [TK_MAX_BINS / 32] kept-bin mask
    double *pose;  // [12] R (row-major) | t of the frame, loaded at block start
};

FT_DEV unsigned hash_slot(long long id, int bits) {
    return (unsigned)(((unsigned long long)id * 0x9E3779B97F4A7C15ull) >> (64 - bits));
}

// Open-addressing set of slotted point ids: the table stores indices k into
// kslots (4 B per entry); duplicates of an id are inserted once.
FT_DEV void hash_insert(int *tab, int bits, const long long *kslots, int k) {
    const unsigned mask = (1u << bits) - 1u;
    const long long id = kslots[k];
    unsigned h = hash_slot(id, bits);
    while (true) {
        const int prev = atomicCAS(tab + h, -1, k);
        if (prev == -1 || kslots[prev] == id) return;
        h = (h + 1) & mask;
    }
}

FT_DEV bool hash_contains(const int *tab, int bits, const long long *kslots, long long id) {
    const unsigned mask = (1u << bits) - 1u;
    unsigned h = hash_slot(id, bits);
    while (true) {
        const int x = tab[h];
        if (x == -1) return false;
        if (kslots[x] == id) return true;
        h = (h + 1) & mask;
    }
}

// One map point's inputs, loaded once.
struct PointIn {
    double px, py, pz, nx, ny, nz, mind, maxd;
};

FT_DEV PointIn staged_point(const MapSmem &sm, int li) {
    const ft_point_record &r = sm.prnd[li];
    PointIn q;
    q.px = r.pos[0];
    q.py = r.pos[1];
    q.pz = r.pos[2];
    q.nx = r.nrm[0];
    q.ny = r.nrm[1];
    q.nz = r.nrm[2];
    q.mind = r.min_dist;
    q.maxd = r.max_dist;
    return q;
}

// kernels.py:496-551: visibility gate of one point in the reference's fp64
// evaluation order; fills the window of the candidate scan.
FT_DEV bool project_point(const TrackArgs &a, const PointIn &pt, double ccx, double ccy,
                          double ccz, const double *R, const double *T, QItem &q) {
    const ft_project_params &p = a.pp;
    const double px = pt.px, py = pt.py, pz = pt.pz;
    const double pcx = R[0] * px + R[1] * py + R[2] * pz + T[0];
    const double pcy = R[3] * px + R[4] * py + R[5] * pz + T[1];
    const double pcz = R[6] * px + R[7] * py + R[8] * pz + T[2];
    if (pcz <= 1e-6) return false;
    double u, v;
    if (p.cam_kind == 0) {
        u = p.fx * pcx / pcz + p.cx;
        v = p.fy * pcy / pcz + p.cy;
    } else {
        const double r = hypot(pcx, pcy);
        if (r < 1e-12) {
            u = p.cx;
            v = p.cy;
        } else {
            const double theta = atan2(r, pcz);
            const double t2 = theta * theta;
            const double dth = theta * (1.0 + t2 * (p.k1 + t2 * (p.k2 + t2 * (p.k3 + t2 * p.k4))));
            u = p.fx * dth * pcx / r + p.cx;
            v = p.fy * dth * pcy / r + p.cy;
        }
    }
    if (u < 0.0 || u >= p.width || v < 0.0 || v >= p.height) return false;
    const double dist = sqrt(pcx * pcx + pcy * pcy + pcz * pcz);
    if (dist < pt.mind || dist > pt.maxd) return false;
    const double vx = px - ccx, vy = py - ccy, vz = pz - ccz;
    const double cosang = (vx * pt.nx + vy * pt.ny + vz * pt.nz) / dist;
    if (cosang < p.view_cos_min) return false;
    long long lvl = (long long)ceil(log(pt.maxd / dist) * p.inv_log_scale - 1e-9);
    if (lvl < 0) lvl = 0;
    if (lvl > p.n_levels - 1) lvl = p.n_levels - 1;
    const double r_win = p.window_px * p.scale_pow[lvl];
    const double ucen = u + p.u_offset;
    const double cell = (double)p.cell_px;
    long long cx0 = (long long)((ucen - r_win) / cell);
    long long cx1 = (long long)((ucen + r_win) / cell);
    long long cy0 = (long long)((v - r_win) / cell);
    long long cy1 = (long long)((v + r_win) / cell);
    if (cx1 < 0 || cy1 < 0 || cx0 > p.grid_nx - 1 || cy0 > p.grid_ny - 1) return false;
    if (cx0 < 0) cx0 = 0;
    if (cy0 < 0) cy0 = 0;
    if (cx1 > p.grid_nx - 1) cx1 = p.grid_nx - 1;
    if (cy1 > p.grid_ny - 1) cy1 = p.grid_ny - 1;
    q.ucen = ucen;
    q.v = v;
    q.r = r_win;
    q.lvl = (int)lvl;
    q.cx0 = (short)cx0;
    q.cx1 = (short)cx1;
    q.cy0 = (short)cy0;
    q.cy1 = (short)cy1;
    return true;
}

FT_DEV double py_mod(double a, double b) {  // numpy float remainder
    double r = fmod(a, b);
    if (r != 0.0 && ((b < 0.0) != (r < 0.0))) r += b;
    return r;
}

FT_DEV int rotation_bin(const TrackArgs &a, int64_t kbase, int64_t pbase, int kp, int pi) {
    const double two_pi = 2.0 * 3.141592653589793;
    const int nb = a.pp.histogram_bins;
    const double diff = py_mod(a.K.rec[kbase + kp].angle - a.io.ref_angles[pbase + pi], two_pi);
    long long b = (long long)floor(diff / two_pi * (double)nb);
    return (int)(b < 0 ? 0 : (b > nb - 1 ? nb - 1 : b));
}

// Stage points [q0, q1) of the frame into the shared round buffer (one TMA copy).
FT_DEV void stage_points(const TrackArgs &a, const MapSmem &sm, int64_t pbase, int q0, int q1,
                         unsigned long long *mbar) {
    const unsigned bytes = 112u * (unsigned)(q1 - q0);
    mbar_arrive_expect_tx(mbar, bytes);
    if (bytes) bulk_g2s(sm.prnd, a.P.rec + pbase + q0, bytes, mbar);
}

// Resident-table variant: points [q0, q1) gathered through the slot index
// into the round buffer by all threads (visible after the caller's next
// __syncthreads).  Two round trips however many points: the round's indices
// into shared memory (the search queue's space, free until the projection
// refills it), then every 16-B piece of every record as a cp.async copy, all
// in flight at once.  (One dependent index + record load per piece in a
// loop cost ~12 serial round trips per round at 854 points per block: the
// map role's bottleneck at 8 step groups, r2h.)
FT_DEV void gather_points(const TrackArgs &a, const MapSmem &sm, const int32_t *pidx, int q0,
                          int q1) {
    uint4 *dst = reinterpret_cast<uint4 *>(sm.prnd);
    int *ix = reinterpret_cast<int *>(sm.queue);
    const int n = q1 - q0;
    for (int i = threadIdx.x; i < n; i += TK_THREADS) ix[i] = ld_in(a, pidx + q0 + i);
    __syncthreads();
    for (int t = threadIdx.x; t < 7 * n; t += TK_THREADS) {
        const int r = t / 7;
        cp_async16(dst + t, reinterpret_cast<const uint4 *>(a.P.rec + ix[r]) + (t - 7 * r));
    }
    cp_async_commit();
    cp_async_wait<0>();
}

// Tail mode of the map group (one frame per group, resolve without ordered
// outputs / rotation filter): no group barrier.  The Gw point blocks publish
// their accepted candidates -- (point id, point index | slot-was-empty << 31,
// keypoint | dist << 16 | level << 25) -- compactly at [p0, p0 + n) of the
// frame slot's candidate list plus (n, prefilled slots), arrive with one
// release reduction and are done.  The dedicated resolve block (rank Gw)
// waits for them, then runs phase B (projection.py:161-178: a candidate wins
// iff its claim is the keypoint's minimum) and the slot writes
// (localmap.py:113-121) over every candidate, and stores the counts.
__device__ void map_tail(const TrackArgs &a, const MapSmem &sm, int f, int rank, int slot, int Gw,
                         int chunk, int p0, int p1, int n_pts, int64_t pbase, int64_t kbase,
                         unsigned epoch_hi, bool write_slots, int prefilled) {
    const int lane = threadIdx.x & 31;
    int4 *list = a.mcand + (size_t)slot * a.P.cap;
    int *cnt = a.mcnt + (size_t)slot * WS_MAX_GROUP * 2;
    if (threadIdx.x == 0) sm.misc[9] = 0;
    __syncthreads();
    {
        const int pf = __reduce_add_sync(FULL, prefilled);
        if (lane == 0 && pf) atomicAdd(&sm.misc[9], pf);
    }
    if (rank < Gw) {
        int base = p0;
        for (int r0 = p0; r0 < p1; r0 += TK_THREADS) {
            const int i = r0 + threadIdx.x;
            const int r = i < p1 ? sm.res[i - p0] : -1;
            int total;
            const int pos = base + block_exclusive_scan<TK_THREADS>(r >= 0, sm.scan_tmp, total);
            if (r >= 0) {
                const long long pid = sm.res_pid[i - p0];
                const int em = write_slots && sm.res_empty[i - p0];
                list[pos] = make_int4((int)(unsigned long long)pid, (int)((unsigned long long)pid >> 32),
                                      i | (em << 31), r);
            }
            base += total;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            cnt[2 * rank] = base - p0;
            cnt[2 * rank + 1] = sm.misc[9];
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
            atomicAdd(a.tail_m + slot, 1ull);
        }
        return;
    }
    if (threadIdx.x == 0) {
        while ((uint32_t)ld_acquire_u64(a.tail_m + slot) != (uint32_t)Gw) __nanosleep(20);
        atomicAdd(a.tail_m + slot, (1ull << 32) - (unsigned long long)Gw);
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    __syncthreads();
    TL_MARK(a, 4);
    // per-block counts -> prefix in sm.res (host guarantees map_chunk_cap > Gw)
    int c = 0, pf = 0;
    if (threadIdx.x < Gw) {
        c = __ldcg(cnt + 2 * threadIdx.x);
        pf = __ldcg(cnt + 2 * threadIdx.x + 1);
    }
    int total;
    const int before = block_exclusive_scan<TK_THREADS>(c, sm.scan_tmp, total);
    int *pre = sm.res;
    if (threadIdx.x < Gw) pre[threadIdx.x] = before;
    if (threadIdx.x == 0) pre[Gw] = total;
    pf = __reduce_add_sync(FULL, pf);
    if (lane == 0 && pf) atomicAdd(&sm.misc[9], pf);
    __syncthreads();
    int added = 0, n_win = 0;
    for (int q = threadIdx.x; q < total; q += TK_THREADS) {
        int lo = 0, hi = Gw - 1;  // block b: pre[b] <= q < pre[b + 1]
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (pre[mid] <= q) lo = mid;
            else hi = mid - 1;
        }
        const int4 e = __ldcg(list + lo * chunk + (q - pre[lo]));
        const int i = e.z & 0x7fffffff, r = e.w;
        const int kp = r & 0xffff, d = (r >> 16) & 0x1ff;
        const unsigned long long key = ((unsigned long long)epoch_hi << 32) |
                                       ((unsigned long long)d << 23) | (unsigned)i;
        if (__ldcg(a.claims + kbase + kp) != key) continue;
        ++n_win;
        if (e.z < 0) {  // slot empty before the search
            a.io.slots_out[kbase + kp] =
                (long long)(((unsigned long long)(unsigned)e.y << 32) | (unsigned)e.x);
            ++added;
        }
    }
    added = __reduce_add_sync(FULL, added);
    n_win = __reduce_add_sync(FULL, n_win);
    if (threadIdx.x == 0) {
        sm.misc[10] = 0;
        sm.misc[11] = 0;
    }
    __syncthreads();
    if (lane == 0) {
        if (added) atomicAdd(&sm.misc[10], added);
        if (n_win) atomicAdd(&sm.misc[11], n_win);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (write_slots && a.po.slot_count) a.po.slot_count[f] = sm.misc[9] + sm.misc[10];
        if (a.po.corr_count) a.po.corr_count[f] = sm.misc[11];
    }
    (void)n_pts;
    (void)pbase;
    __syncthreads();
    TL_MARK(a, 5);
}

__device__ void map_frame(const TrackArgs &a, int f, int rank, int slot, unsigned char *smem,
                          unsigned long long *mbar, unsigned &mphase, unsigned &bpar) {
    const int G = a.Gm;
    const int n_pts = min(a.P.count[f], a.P.cap);
    const int n_kp = min(a.K.count[f], a.K.cap);
    const int64_t pbase = (int64_t)f * a.P.cap, kbase = (int64_t)f * a.K.cap;
    // tail mode: rank G-1 is the group's resolve block (no points)
    const int Gw = a.map_tail ? G - 1 : G;
    const int chunk = (((n_pts + Gw - 1) / Gw) + 1) & ~1;  // even: 16-B aligned TMA sources
    const int p0 = rank < Gw ? min(n_pts, rank * chunk) : n_pts, p1 = min(n_pts, p0 + chunk);
    const ft_project_params &pp = a.pp;
    const int nx = pp.grid_nx, ny = pp.grid_ny, ncell = nx * ny;
    const int cap_kp = a.K.cap;
    const bool resolve = a.pmode & FT_PROJ_RESOLVE;
    const bool rotation = (a.pmode & FT_PROJ_ROTATION) && a.io.ref_angles;
    const bool use_hash = (a.pmode & FT_PROJ_SKIP_SLOTS) && a.hash_bits;
    const bool write_slots = a.pmode & FT_PROJ_WRITE_SLOTS;
    const bool ordered = resolve && a.po.corr_point;
    const int round_cap = min(TK_THREADS, a.map_chunk_cap);
    unsigned long long *bar = a.bar_m + 2 * slot;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;

    MapSmem sm;
    unsigned char *p = smem;
    sm.ktab_s = reinterpret_cast<ft_kp_record *>(p);
    p += a.stage_kdesc ? (size_t)64 * cap_kp : 0;
    sm.ktab = a.stage_kdesc ? sm.ktab_s : a.K.rec + kbase;
    sm.prnd = reinterpret_cast<ft_point_record *>(p);
    p += (size_t)112 * round_cap;
    sm.kslots = reinterpret_cast<long long *>(p);
    p += use_hash ? (size_t)8 * cap_kp : 0;
    sm.res_pid = reinterpret_cast<long long *>(p);
    p += (size_t)8 * a.map_chunk_cap;
    sm.queue = reinterpret_cast<QItem *>(p);
    p += sizeof(QItem) * (size_t)round_cap;
    sm.htab = reinterpret_cast<int *>(p);
    p += a.hash_bits ? ((size_t)4 << a.hash_bits) : 0;
    sm.scan_tmp = reinterpret_cast<int *>(p);
    p += 32 * 4;
    sm.misc = reinterpret_cast<int *>(p);
    p += 16 * 4;
    sm.hist = reinterpret_cast<int *>(p);
    p += (TK_MAX_BINS / 32) * 4;
    sm.res = reinterpret_cast<int *>(p);
    p += (size_t)4 * a.map_chunk_cap;
    sm.res_empty = reinterpret_cast<int *>(p);
    p += (size_t)4 * a.map_chunk_cap;
    sm.cell_start = reinterpret_cast<int *>(p);
    p += (size_t)4 * (ncell + 1);
    sm.cell_cursor = reinterpret_cast<int *>(p);
    p += (size_t)4 * ncell;
    sm.items = reinterpret_cast<uint16_t *>(p);
    p += (size_t)2 * cap_kp;
    sm.binbuf = reinterpret_cast<uint16_t *>(p);
    p += (size_t)2 * cap_kp;
    sm.pose = reinterpret_cast<double *>(((uintptr_t)p + 7) & ~(uintptr_t)7);
    // the frame's pose is read by every projection: fetch it now, off the
    // critical path (cold HBM), with the other first-touch loads
    if (threadIdx.x >= TK_THREADS - 12) {
        const int t = threadIdx.x - (TK_THREADS - 12);
        sm.pose[t] = t < 9 ? ld_in(a, a.io.rot + 9 * (int64_t)f + t) : ld_in(a, a.io.trans + 3 * (int64_t)f + t - 9);
    }

    TL_MARK(a, 0);
    const bool have_pts = p0 < p1;
    // The first round of this block's points is unique per block (cold in
    // HBM): every thread loads its share with 16-B loads right away -- many
    // requests in flight -- instead of one TMA stream.  Later rounds (batched
    // mode) use TMA.
    const int n0 = have_pts ? min(p1, p0 + round_cap) - p0 : 0;
    const bool pre_regs = have_pts && 7 * n0 <= 2 * TK_THREADS;
    // resident map table: point i of the frame is P.rec[pidx[i]] (gathered
    // by the threads; no TMA stream, no per-frame copy)
    const int32_t *pidx = a.P.index ? a.P.index + pbase : nullptr;
    uint4 pre[2] = {make_uint4(0, 0, 0, 0), make_uint4(0, 0, 0, 0)};
    if (pre_regs) {
        const uint4 *src = reinterpret_cast<const uint4 *>(a.P.rec + pbase + p0);
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const int t = threadIdx.x + q * TK_THREADS;
            if (t < 7 * n0) {
                const uint4 *s = src + t;
                if (pidx) {
                    const int r = t / 7;
                    s = reinterpret_cast<const uint4 *>(a.P.rec + ld_in(a, pidx + p0 + r)) + (t - 7 * r);
                }
                if (a.coherent)
                    pre[q] = __ldca(s);
                else
                    asm volatile("ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];"
                                 : "=r"(pre[q].x), "=r"(pre[q].y), "=r"(pre[q].z), "=r"(pre[q].w)
                                 : "l"(s));
            }
        }
    } else if (pidx && have_pts) {
        gather_points(a, sm, pidx, p0, min(p1, p0 + round_cap));
    }
    if (threadIdx.x < 32) {  // translate every page the block touches later, now
        const int l = threadIdx.x;
        if (l == 0) prefetch_l2(bar);
        if (l == 1) prefetch_l2(a.claims + kbase);
        if (l == 2) prefetch_l2(a.io.slots_out ? a.io.slots_out + kbase : nullptr);
        if (l == 3) prefetch_l2(a.po.out_kp ? a.po.out_kp + pbase + p0 : nullptr);
        if (l == 4) prefetch_l2(a.po.corr_point ? a.po.corr_point + pbase : nullptr);
        if (l == 5) prefetch_l2(a.po.slot_count ? a.po.slot_count + f : nullptr);
        if (l == 6) prefetch_l2(a.blk_counts + (int64_t)f * G);
    }
    // ---- every first-touch global read of the setup is one TMA batch -------
    if (threadIdx.x == 0 && have_pts) {
        fence_proxy_async_smem();
        const unsigned bt = a.stage_kdesc ? 64u * n_kp : 0u;
        const unsigned bsl = use_hash ? round16(8u * n_kp) : 0u;
        mbar_arrive_expect_tx(mbar, bt + bsl);
        if (bt) bulk_g2s(sm.ktab_s, a.K.rec + kbase, bt, mbar);
        if (bsl) bulk_g2s(sm.kslots, a.io.slots_in + kbase, bsl, mbar);
        if (!pre_regs && !pidx) stage_points(a, sm, pbase, p0, min(p1, p0 + round_cap), mbar + 1);
    }
    // claim epoch of this frame instance, the same for every block of the
    // group.  Keyed by the claims row (frame f), not by the group slot: the
    // row's epochs then grow monotonically whatever geometry (W) earlier
    // launches on this workspace used, so stale claims always lose.
    unsigned ticket = 0;
    if (threadIdx.x == 0 && resolve) ticket = group_ticket(a.ep_m + f, G);
    if (rank == 0 && threadIdx.x == 0) {
        if (a.po.slot_count) a.po.slot_count[f] = 0;
        if (a.po.corr_count) a.po.corr_count[f] = 0;
    }
    if (rank == 0 && rotation)
        for (int b = threadIdx.x; b < TK_MAX_BINS; b += TK_THREADS)
            a.hist[(int64_t)f * TK_MAX_BINS + b] = 0;
    int prefilled = 0;
    if (write_slots) {  // slots_out <- slots_in (this block's share)
        const int sc = (n_kp + G - 1) / G, s0 = rank * sc, s1 = min(n_kp, s0 + sc);
        for (int k = s0 + threadIdx.x; k < s1; k += TK_THREADS) {
            const long long v = ld_in(a, a.io.slots_in + kbase + k);
            if (a.io.slots_out != a.io.slots_in) a.io.slots_out[kbase + k] = v;
            prefilled += v != NO_PID;
        }
    }
    if (have_pts && use_hash)
        for (int h = threadIdx.x; h < (1 << a.hash_bits); h += TK_THREADS) sm.htab[h] = -1;
    if (have_pts)
        for (int b = threadIdx.x; b < ncell; b += TK_THREADS) sm.cell_cursor[b] = 0;
    if (threadIdx.x == 0) sm.misc[0] = (int)ticket;
    __syncthreads();
    const unsigned epoch_hi = 0xffffffffu - (unsigned)sm.misc[0];

    if (have_pts) {
        mbar_wait(mbar, mphase & 1u);  // keypoint table (+ slots) landed
        mphase ^= 1u;
        TL_MARK(a, 6);
        if (pre_regs) {
            uint4 *dst = reinterpret_cast<uint4 *>(sm.prnd);
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const int t = threadIdx.x + q * TK_THREADS;
                if (t < 7 * n0) dst[t] = pre[q];
            }
        }
        if (use_hash)
            for (int k = threadIdx.x; k < n_kp; k += TK_THREADS)
                if (sm.kslots[k] != NO_PID) hash_insert(sm.htab, a.hash_bits, sm.kslots, k);
        const double cellf = (double)pp.cell_px;
        block_csr<TK_THREADS>(
            n_kp, ncell,
            [&](int j) {  // FrameGrid cell: truncation, then clip (mapping.py:81-83)
                long long cx = (long long)(sm.ktab[j].u / cellf),
                          cy = (long long)(sm.ktab[j].v / cellf);  // once per keypoint
                cx = cx < 0 ? 0 : (cx > nx - 1 ? nx - 1 : cx);
                cy = cy < 0 ? 0 : (cy > ny - 1 ? ny - 1 : cy);
                return (int)(cy * nx + cx);
            },
            sm.cell_start, sm.cell_cursor, sm.items, sm.binbuf,
            sm.scan_tmp);
        TL_MARK(a, 1);
        const double *R = sm.pose, *T = sm.pose + 9;
        const double ccx = -(R[0] * T[0] + R[3] * T[1] + R[6] * T[2]);
        const double ccy = -(R[1] * T[0] + R[4] * T[1] + R[7] * T[2]);
        const double ccz = -(R[2] * T[0] + R[5] * T[1] + R[8] * T[2]);
        for (int r0 = p0; r0 < p1; r0 += round_cap) {
            const int r1 = min(p1, r0 + round_cap);
            if (r0 != p0) {  // later rounds (batched mode): stage this round's points
                __syncthreads();
                if (pidx) {
                    gather_points(a, sm, pidx, r0, r1);
                } else if (threadIdx.x == 0) {
                    fence_proxy_async_smem();
                    stage_points(a, sm, pbase, r0, r1, mbar + 1);
                }
            }
            if (threadIdx.x == 0) sm.misc[1] = 0;
            if (!pidx && (r0 != p0 || !pre_regs)) {
                mbar_wait(mbar + 1, (mphase >> 1) & 1u);  // bit 1: phase of mbar[1]
                mphase ^= 2u;
            }
            if (r0 == p0) TL_MARK(a, 7);
            __syncthreads();
            const int rr = (r0 - p0) / round_cap;  // round (debug marks 8..15: rounds 0-3)
            if (rr < 4) TL_MARK(a, 8 + 2 * rr);
            const int li = threadIdx.x;
            const int i = r0 + li;
            if (i < r1) {
                const int64_t gi = pbase + i;
                sm.res[i - p0] = -1;
                if (a.po.out_kp) {
                    a.po.out_kp[gi] = -1;
                    a.po.out_dist[gi] = 10000;
                    a.po.out_oct[gi] = -1;
                }
                const bool skip = a.io.skip && a.io.skip[gi] != 0;
                QItem q;
                if (!skip && project_point(a, staged_point(sm, li), ccx, ccy, ccz, R, T, q)) {
                    q.li = li;
                    sm.queue[atomicAdd(&sm.misc[1], 1)] = q;
                }
            }
            __syncthreads();
            TL_MARK(a, 2);
            const int nq = sm.misc[1];
            // two visible points per warp (half-warps: lanes 0-15 and 16-31): a
            // point's window holds ~10-20 candidates, so 16 lanes cover it in
            // one pass and the Best2 reduction (4 xor-shuffle levels) serves
            // two points
            constexpr int LPP = FT_MAP_LANES_PER_POINT;  // lanes per visible point
            const int hl = lane & (LPP - 1), hh = lane / LPP;
            for (int qb = (32 / LPP) * wid; qb < nq; qb += (32 / LPP) * TK_WARPS) {
                const int qi = qb + hh;
                bool live = qi < nq;
                const QItem &q = sm.queue[live ? qi : 0];
                const long long qpid = live ? sm.prnd[q.li].id : 0;
                if (live && use_hash && hash_contains(sm.htab, a.hash_bits, sm.kslots, qpid))
                    live = false;
                Best2 b;
                best2_init(b);
                if (live) {
                    const Desc pd = rec_desc(sm.prnd[q.li]);
                    for (int gy = q.cy0; gy <= q.cy1; ++gy) {
                        const int beg = sm.cell_start[gy * nx + q.cx0];
                        const int end = sm.cell_start[gy * nx + q.cx1 + 1];
                        for (int ii = beg + hl; ii < end; ii += LPP) {
                            const int j = sm.items[ii];
                            const ft_kp_record &kr = sm.ktab[j];
                            if (fabs(kr.u - q.ucen) > q.r || fabs(kr.v - q.v) > q.r) continue;
                            const int ko = kr.octave;
                            if (ko < q.lvl - 1 || ko > q.lvl + 1) continue;
                            best2_push(b, hamming(pd, rec_desc(kr)), (uint32_t)j);
                        }
                    }
                }
#pragma unroll
                for (int sh = LPP / 2; sh > 0; sh >>= 1) {  // within the point's lanes
                    const uint32_t ok = __shfl_xor_sync(FULL, b.key, sh);
                    const uint32_t os = __shfl_xor_sync(FULL, b.second, sh);
                    best2_merge(b, ok, os);
                }
                if (live && hl == 0 && ratio_accept(b, pp.t_proj, pp.ratio)) {
                    const int kp = (int)(b.key & 0xffffu), d = (int)(b.key >> 16);
                    const int i = r0 + q.li;
                    const int64_t gi = pbase + i;
                    if (a.po.out_kp) {
                        a.po.out_kp[gi] = kp;
                        a.po.out_dist[gi] = d;
                        a.po.out_oct[gi] = q.lvl;
                    }
                    sm.res[i - p0] = kp | (d << 16) | (q.lvl << 25);
                    sm.res_pid[i - p0] = qpid;
                    if (write_slots)  // staged copy of slots_in when the hash set uses it
                        sm.res_empty[i - p0] =
                            (use_hash ? sm.kslots[kp] : ld_in(a, a.io.slots_in + kbase + kp)) == NO_PID;
                    if (resolve)
                        atomicMin(a.claims + kbase + kp, ((unsigned long long)epoch_hi << 32) |
                                                             ((unsigned long long)d << 23) |
                                                             (unsigned)i);
                }
            }
            __syncthreads();
            if (rr < 4) TL_MARK(a, 9 + 2 * rr);
        }
    }
    TL_MARK(a, 3);
    if (!resolve) return;
    if (a.map_tail) {
        map_tail(a, sm, f, rank, slot, Gw, chunk, p0, p1, n_pts, pbase, kbase, epoch_hi,
                 write_slots, prefilled);
        return;
    }
    group_barrier(bar, G, bpar);
    TL_MARK(a, 4);

    // phase B on this block's points: winner iff its claim is the minimum.
    // The block's claim words are loaded in one round trip (a chunk is at
    // most TK_MAP_CHUNK_MAX points), then compared.
    int n_win = 0;
    {
        constexpr int MAXI = (TK_MAP_CHUNK_MAX + TK_THREADS - 1) / TK_THREADS;
        int rr[MAXI];
        unsigned long long cl[MAXI];
#pragma unroll
        for (int u = 0; u < MAXI; ++u) {
            const int i = p0 + (int)threadIdx.x + u * TK_THREADS;
            rr[u] = i < p1 ? sm.res[i - p0] : -1;
            cl[u] = rr[u] >= 0 ? __ldcg(a.claims + kbase + (rr[u] & 0xffff)) : 0ull;
        }
#pragma unroll
        for (int u = 0; u < MAXI; ++u) {
            const int i = p0 + (int)threadIdx.x + u * TK_THREADS;
            const int r = rr[u];
            if (r < 0) continue;
            const int kp = r & 0xffff, d = (r >> 16) & 0x1ff;
            const unsigned long long key = ((unsigned long long)epoch_hi << 32) |
                                           ((unsigned long long)d << 23) | (unsigned)i;
            if (cl[u] != key) {
                sm.res[i - p0] = -1;
                continue;
            }
            ++n_win;
            if (rotation)
                atomicAdd(a.hist + (int64_t)f * TK_MAX_BINS + rotation_bin(a, kbase, pbase, kp, i), 1);
        }
    }
    if (rotation) {
        group_barrier(bar, G, bpar);
        if (threadIdx.x == 0) {  // top-K bins by (-count, bin)
            const int nb = pp.histogram_bins;
            const int *h = a.hist + (int64_t)f * TK_MAX_BINS;
            unsigned keep[TK_MAX_BINS / 32] = {0};
            for (int t = 0; t < pp.histogram_keep && t < nb; ++t) {
                int sel = -1, best = -1;
                for (int b = 0; b < nb; ++b) {
                    if (keep[b >> 5] & (1u << (b & 31))) continue;
                    const int c = __ldcg(h + b);
                    if (sel < 0 || c > best) {
                        sel = b;
                        best = c;
                    }
                }
                if (sel >= 0) keep[sel >> 5] |= 1u << (sel & 31);
            }
            for (int w = 0; w < TK_MAX_BINS / 32; ++w) sm.hist[w] = (int)keep[w];
        }
        __syncthreads();
        n_win = 0;
        for (int i = p0 + threadIdx.x; i < p1; i += TK_THREADS) {
            const int r = sm.res[i - p0];
            if (r < 0) continue;
            const int b = rotation_bin(a, kbase, pbase, r & 0xffff, i);
            if ((sm.hist[b >> 5] >> (b & 31)) & 1) ++n_win;
            else sm.res[i - p0] = -1;
        }
    }
    __syncthreads();
    // search_local_points slot write (localmap.py:113-121): only slots empty
    // before the search; winners hold distinct keypoints, so no races.
    if (write_slots) {
        int added = 0;
        for (int i = p0 + threadIdx.x; i < p1; i += TK_THREADS) {
            const int r = sm.res[i - p0];
            if (r < 0 || !sm.res_empty[i - p0]) continue;
            a.io.slots_out[kbase + (r & 0xffff)] = sm.res_pid[i - p0];
            ++added;
        }
        const int tot = __reduce_add_sync(FULL, added + prefilled);
        if (lane == 0 && tot && a.po.slot_count) atomicAdd(a.po.slot_count + f, tot);
    }
    if (!ordered) {
        if (a.po.corr_count) {
            const int tot = __reduce_add_sync(FULL, n_win);
            if (lane == 0 && tot) atomicAdd(a.po.corr_count + f, tot);
        }
        __syncthreads();
        TL_MARK(a, 5);
        return;
    }
    // ordered correspondences: block counts -> prefix over ranks -> write
    {
        const int tot = __reduce_add_sync(FULL, n_win);
        if (threadIdx.x == 0) sm.misc[2] = 0;
        __syncthreads();
        if (lane == 0 && tot) atomicAdd(&sm.misc[2], tot);
        __syncthreads();
        if (threadIdx.x == 0) a.blk_counts[(int64_t)f * G + rank] = sm.misc[2];
    }
    group_barrier(bar, G, bpar);
    int before = 0, all = 0;
    for (int b = threadIdx.x; b < G; b += TK_THREADS) {
        const int c = __ldcg(a.blk_counts + (int64_t)f * G + b);
        all += c;
        if (b < rank) before += c;
    }
    before = __reduce_add_sync(FULL, before);
    all = __reduce_add_sync(FULL, all);
    if (threadIdx.x == 0) {
        sm.misc[3] = 0;
        sm.misc[4] = 0;
    }
    __syncthreads();
    if (lane == 0) {
        atomicAdd(&sm.misc[3], before);
        atomicAdd(&sm.misc[4], all);
    }
    __syncthreads();
    int base = sm.misc[3];
    if (rank == 0 && threadIdx.x == 0 && a.po.corr_count) a.po.corr_count[f] = sm.misc[4];
    for (int r0 = p0; r0 < p1; r0 += TK_THREADS) {
        const int i = r0 + threadIdx.x;
        const int r = i < p1 ? sm.res[i - p0] : -1;
        const int win = r >= 0;
        int total;
        const int pos = base + block_exclusive_scan<TK_THREADS>(win, sm.scan_tmp, total);
        if (win) {
            a.po.corr_point[pbase + pos] = i;
            a.po.corr_kp[pbase + pos] = r & 0xffff;
            a.po.corr_dist[pbase + pos] = (r >> 16) & 0x1ff;
            a.po.corr_oct[pbase + pos] = r >> 25;
        }
        base += total;
    }
    __syncthreads();
    TL_MARK(a, 5);
}

__global__ void __launch_bounds__(TK_THREADS) track_kernel(const TrackArgs a) {
    extern __shared__ __align__(16) unsigned char smem_all[];
    // two mbarriers (table / point rounds) ahead of the role's buffers
    unsigned long long *mbar = reinterpret_cast<unsigned long long *>(smem_all);
    unsigned char *smem = smem_all + 16;
    if (threadIdx.x == 0) {
        mbar_init(mbar, 1);
        mbar_init(mbar + 1, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    unsigned mphase = 0, bpar = 0;
    const int per = a.Gs + a.Gm;
    const int slot = blockIdx.x / per, r = blockIdx.x - slot * per;
    for (int f = slot; f < a.F; f += a.W) {
        if (r < a.Gs) stereo_frame(a, f, r, slot, smem, mbar, mphase, bpar);
        else map_frame(a, f, r - a.Gs, slot, smem, mbar, mphase, bpar);
    }
}

// ---------------------------------------------------------------------------
// Persistent mode (ft_runner_create_persistent): ONE long-lived cooperative
// launch steps through a ring of n input/output slots, removing the per-frame
// launch (graph launch, block scheduling, drain).  Step k uses slot k % n:
// the runner's host thread sets ready[slot] = k + 1 (pinned, mapped host
// memory) once the slot's inputs have landed; block 0 watches that word and
// forwards it to a device word every other block polls (one PCIe poller,
// not 120); each block runs its role on the slot's arguments and arrives on
// arrive[slot]; the step's last arrival publishes done[slot] = k + 1 into
// mapped host memory, where the runner picks it up and issues the D2H copy.
// Blocks run ahead independently -- a block that finished step k starts
// step k + 1 while others finish k (each slot has its own workspace, so the
// groups' barrier words and tickets never mix).  ready[] == FT_PERSIST_STOP
// ends the launch.
constexpr int PERSIST_MAX_SLOTS = 16;
constexpr unsigned FT_PERSIST_STOP = 0xffffffffu;

struct PersistArgs {
    const TrackArgs *args;  // [n] in device memory, identical geometry in every slot
    int n, W, Gs, Gm;
    int Q;                  // step groups: group g = blocks [g B, (g+1) B) runs steps k = g mod Q
    unsigned max_steps;     // the launch ends after this many steps (or at a stop)
    int gate;               // step k waits for the slot's step k - n to be done (ring)
    int red_arrive;         // arrivals by reduction; the last block publishes done
    unsigned poll_ns;       // PCIe watcher: sleep between polls of the host-mapped ready word
    const unsigned *ready;  // [n] host-mapped: step + 1 whose inputs are in the slot
    unsigned *dready;       // [n] device copy of ready (forwarded by block 0)
    unsigned *done;         // [n] host-mapped: step + 1 whose outputs are complete
    unsigned *arrive;       // [n] block arrivals (monotonic)
    unsigned long long *ts;  // debug (FT_DEBUG_PERSIST): [4096][2] step start / done (ns)
    // push mode (runner): the step's last block writes the slot's outputs
    // into its pinned host range itself (no D2H copy / event per step)
    unsigned long long out_bytes;
    unsigned long long out_dev[PERSIST_MAX_SLOTS];   // slot output ranges (device)
    unsigned long long out_host[PERSIST_MAX_SLOTS];  // ... their pinned host ranges
};

// Push mode, step end (the step's last block, after every arrival): the
// slot's outputs -> its pinned host range with 16-B stores over PCIe (posted
// writes), ordered before done for the host: the block's stores are
// performed relative to thread 0 at the barrier, and thread 0's release
// store of done at system scope is cumulative over them.  (A fence.sc.sys
// per thread serialises, ~0.5 us each.)
__device__ void push_outputs(const PersistArgs &p, int i) {
    constexpr int U = 8;  // 16-B loads in flight per thread
    const uint4 *s4 = reinterpret_cast<const uint4 *>(p.out_dev[i]);
    uint4 *d4 = reinterpret_cast<uint4 *>(p.out_host[i]);
    const unsigned long long nv = p.out_bytes >> 4;
    for (unsigned long long t = threadIdx.x; t < nv; t += U * TK_THREADS) {
        uint4 x[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (t + u * TK_THREADS < nv) x[u] = __ldcg(s4 + t + u * TK_THREADS);
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (t + u * TK_THREADS < nv) d4[t + u * TK_THREADS] = x[u];
    }
    const char *sb = reinterpret_cast<const char *>(p.out_dev[i]);
    char *db = reinterpret_cast<char *>(p.out_host[i]);
    for (unsigned long long x = (nv << 4) + threadIdx.x; x < p.out_bytes; x += TK_THREADS)
        db[x] = __ldcg(sb + x);
    __syncthreads();
}

FT_DEV unsigned ld_acquire_u32(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

FT_DEV unsigned ld_acquire_sys_u32(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// (The roles are inlined here as in track_kernel.  Out of line -- so the
// step loop's own state no longer shares the roles' peak register pressure --
// ptxas's spill drops from 140 / 136 B to 16 / 12 B in the kernel body (plus
// 48-108 B inside the callees) but the resident ring measured 3 % slower
// (r2o: 12.48 vs 12.07 us per frame at G = 1, 6.95 vs 6.75 at G = 4); the
// spill slots stay in L1.)
// PUSH: the push-mode instantiation (the default one carries none of its
// code, so its register allocation is unchanged)
template <bool PUSH>
__global__ void __launch_bounds__(TK_THREADS) track_persist_kernel(const __grid_constant__ PersistArgs p) {
    extern __shared__ __align__(16) unsigned char smem_all[];
    __shared__ int s_go, s_last;
    __shared__ __align__(16) TrackArgs s_args;  // the current slot's arguments
    unsigned long long *mbar = reinterpret_cast<unsigned long long *>(smem_all);
    unsigned char *smem = smem_all + 16;
    if (threadIdx.x == 0) {
        mbar_init(mbar, 1);
        mbar_init(mbar + 1, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    unsigned mphase = 0, bpar = 0;
    const int per = p.Gs + p.Gm;
    const unsigned B = (unsigned)(p.W * per);  // blocks per step group
    const int grp = (int)(blockIdx.x / B), gb = (int)(blockIdx.x - grp * B);
    const int wslot = gb / per, r = gb - wslot * per;
    constexpr int ARG_WORDS = (int)(sizeof(TrackArgs) / 8);
    static_assert(sizeof(TrackArgs) % 8 == 0, "TrackArgs copied as 8-byte words");
    // Step groups: the Q groups take steps round robin, so Q frames are in
    // flight at once on disjoint blocks.  Slot i = k mod n is only ever run
    // by group i mod Q (the host requires Q | n), so its arrival counter and
    // workspace see one group's blocks.
    for (unsigned k = (unsigned)grp; k < p.max_steps; k += (unsigned)p.Q) {
        const int i = (int)(k % (unsigned)p.n);
        if (threadIdx.x == 0) {
            unsigned v;
            if (p.gate) {
                // ring (ft_track_frames_ring): every step's inputs are resident
                // before the launch (the loop ends at max_steps), so only the
                // slot's previous step (k - n, same workspace) must be
                // complete -- its tail blocks may still be counting arrivals.
                // Every block checks the device-memory done word itself.
                v = k + 1;
                if (k >= (unsigned)p.n)
                    while (ld_acquire_u32(p.done + i) < k + 1 - (unsigned)p.n) __nanosleep(64);
            } else if (gb == 0) {  // the group's PCIe watcher
                // (the runner's host ordering already implies that the slot's
                // previous step k - n is complete)
                while ((v = ld_acquire_sys_u32(p.ready + i)) != FT_PERSIST_STOP && v < k + 1)
                    __nanosleep(p.poll_ns);
                // forward exactly this step (the host word may already allow later ones)
                const unsigned fwd = v == FT_PERSIST_STOP ? v : k + 1;
                asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p.dready + i), "r"(fwd)
                             : "memory");
            } else {
                while ((v = ld_acquire_u32(p.dready + i)) != FT_PERSIST_STOP && v < k + 1)
                    __nanosleep(64);
            }
            s_go = v != FT_PERSIST_STOP;
            if (p.ts && gb == 0 && s_go) p.ts[2 * (k & 4095u)] = global_ns();
        }
        if (threadIdx.x < ARG_WORDS)  // slot i's arguments -> shared memory
            reinterpret_cast<unsigned long long *>(&s_args)[threadIdx.x] =
                __ldg(reinterpret_cast<const unsigned long long *>(p.args + i) + threadIdx.x);
        __syncthreads();
        if (!s_go) break;
        const TrackArgs &a = s_args;
        for (int f = wslot; f < a.F; f += a.W) {
            if (r < a.Gs) stereo_frame(a, f, r, wslot, smem, mbar, mphase, bpar);
            else map_frame(a, f, r - a.Gs, wslot, smem, mbar, mphase, bpar);
        }
        __syncthreads();
        if (p.red_arrive) {
            // every block but the last one arrives with a release reduction (no
            // round trip); the last block collects them and publishes the step
            if (threadIdx.x == 0) {
                if (gb != (int)B - 1) {
                    asm volatile("fence.acq_rel.gpu;" ::: "memory");
                    atomicAdd(p.arrive + i, 1u);
                    s_last = 0;
                } else {
                    const unsigned want = (k / (unsigned)p.n + 1u) * (B - 1u);
                    while ((int)(ld_acquire_u32(p.arrive + i) - want) < 0) __nanosleep(32);
                    asm volatile("fence.acq_rel.gpu;" ::: "memory");
                    s_last = 1;
                }
            }
        } else if (threadIdx.x == 0) {
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
            const unsigned old = atomicAdd(p.arrive + i, 1u);
            const bool last = old + 1u == (k / (unsigned)p.n + 1u) * B;  // the step's last block
            if (last) asm volatile("fence.acq_rel.gpu;" ::: "memory");
            s_last = last;
        }
        __syncthreads();
        if (s_last) {
            if (PUSH) push_outputs(p, i);
            if (threadIdx.x == 0) {
                asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p.done + i), "r"(k + 1u)
                             : "memory");
                if (p.ts) p.ts[2 * (k & 4095u) + 1] = global_ns();
            }
        }
    }
}

// ---------------------------------------------------------------------------
// host side

size_t stereo_smem(const TrackArgs &a) {
    const int cap = a.R.cap, H = a.sp.height;
    return 16 + stereo_table_bytes(a) + 4 * (32 + 16 + 512) + 4 * (size_t)(2 * H + 1) + 16 +
           4 * (size_t)TK_WARPS * a.patch_ints + 4 * (size_t)cap + 64;
}

size_t map_smem(const TrackArgs &a) {
    const int cap = a.K.cap, ncell = a.pp.grid_nx * a.pp.grid_ny;
    const int round_cap = a.map_chunk_cap < TK_THREADS ? a.map_chunk_cap : TK_THREADS;
    const bool hash = a.hash_bits > 0;
    return 16 + (a.stage_kdesc ? (size_t)64 * cap : 0) + (size_t)112 * round_cap +
           (hash ? (size_t)8 * cap : 0) + sizeof(QItem) * (size_t)round_cap +
           (hash ? ((size_t)4 << a.hash_bits) : 0) + 4 * (32 + 16 + TK_MAX_BINS / 32) +
           16 * (size_t)a.map_chunk_cap + 4 * (size_t)(2 * ncell + 1) + 4 * (size_t)cap + 64 +
           12 * 8 + 8;  // pose
}

}  // namespace ft

using namespace ft;

namespace {
// Launch geometry depends only on shapes; cache it so graph capture and
// steady-state launches make no attribute / occupancy queries.
struct GeomKey {
    int dev, F, lcap, rcap, pcap, kcap, H, patch_ints, ncell, hash_bits, ws, wm, reserve, rej_only,
        groups;
    bool operator==(const GeomKey &o) const { return memcmp(this, &o, sizeof(*this)) == 0; }
};
struct Geom {
    int Gs, Gm, W, chunk, stage_rdesc, stage_kdesc;
    size_t smem;
};
constexpr int GEOM_CACHE = 8;
thread_local GeomKey g_keys[GEOM_CACHE];
thread_local Geom g_vals[GEOM_CACHE];
thread_local int g_n = 0, g_next = 0;
size_t g_attr_smem[64] = {0};  // process-wide, guarded by g_attr_mu
std::mutex g_attr_mu;
}  // namespace

static int track_geometry(TrackArgs &a, bool want_stereo, bool want_map, Geom &out,
                          int reserve, bool rej_only, int groups);

// The kernel's max-dynamic-smem attribute only ever grows (one attribute per
// function: lowering it for a small launch would break a cached large one).
static int raise_smem_attr(int dev, size_t smem) {
    if (dev < 0 || dev >= 64) return FT_E_RANGE;
    std::lock_guard<std::mutex> lock(g_attr_mu);
    if (smem <= g_attr_smem[dev]) return FT_OK;
    const cudaError_t e =
        cudaFuncSetAttribute(track_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return (int)e;
    g_attr_smem[dev] = smem;
    return FT_OK;
}

// Geometry, kernel attribute and workspace pointers of a launch (shared by
// the per-launch path and the persistent plans).
static int track_prepare(TrackArgs &a, bool want_stereo, bool want_map, const ft_workspace *ws,
                         Geom &g_out, bool tails, int groups = 1) {
    int dev = 0;
    cudaGetDevice(&dev);
    GeomKey key;
    memset(&key, 0, sizeof(key));
    key.dev = dev;
    key.F = a.F;
    key.lcap = want_stereo ? a.L.cap : 0;
    key.rcap = want_stereo ? a.R.cap : 0;
    key.pcap = want_map ? a.P.cap : 0;
    key.kcap = want_map ? a.K.cap : 0;
    key.H = want_stereo ? a.sp.height : 0;
    key.patch_ints = a.patch_ints;
    key.ncell = want_map ? a.pp.grid_nx * a.pp.grid_ny : 0;
    key.hash_bits = a.hash_bits;
    key.ws = want_stereo;
    key.wm = want_map;
    // persistent plans (tails) leave SMs for the tail blocks and the copies'
    // helper kernels: the whole grid must stay <= SMs - 4 with 2 tail blocks
    key.reserve = tails ? 6 : 0;
    // stereo without any per-keypoint work (reject_outliers alone): one
    // block per frame gathers, selects the median and rejects
    key.rej_only = want_stereo && !want_map &&
                   !(a.smode & (FT_STEREO_PHASE1 | FT_STEREO_REFINE | FT_STEREO_FROM_CAND));
    // persistent step groups: each group gets 1 / groups of the SMs
    key.groups = groups < 1 ? 1 : groups;
    Geom g;
    int hit = -1;
    for (int i = 0; i < g_n; ++i)
        if (g_keys[i] == key) hit = i;
    if (hit >= 0) {
        g = g_vals[hit];
    } else {
        const int st = track_geometry(a, want_stereo, want_map, g, key.reserve, key.rej_only,
                                      key.groups);
        if (st != FT_OK) return st;
        g_keys[g_next] = key;
        g_vals[g_next] = g;
        g_next = (g_next + 1) % GEOM_CACHE;
        if (g_n < GEOM_CACHE) ++g_n;
    }
    a.Gs = g.Gs;
    a.Gm = g.Gm;
    a.W = g.W;
    a.map_chunk_cap = g.chunk;
    a.stage_rdesc = g.stage_rdesc;
    a.stage_kdesc = g.stage_kdesc;
    {
        const int st = raise_smem_attr(dev, g.smem);
        if (st != FT_OK) return st;
    }
    if (getenv("FT_DEBUG_GEOMETRY")) {
        int occ = -1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, track_kernel, TK_THREADS, g.smem);
        cudaFuncAttributes fa;
        cudaFuncGetAttributes(&fa, track_kernel);
        fprintf(stderr,
                "[ft_track] F=%d W=%d Gs=%d Gm=%d smem=%zu grid=%d cached=%d occ=%d "
                "maxDyn=%d regs=%d\n",
                a.F, a.W, a.Gs, a.Gm, g.smem, a.W * (a.Gs + a.Gm), hit >= 0, occ,
                fa.maxDynamicSharedSizeBytes, fa.numRegs);
    }
    if (a.W > ws->n_frames || a.Gm > WS_MAX_GROUP) return FT_E_WORKSPACE;
    const WsLayout wl = ws_layout(ws);
    a.bar_s = ws_ptr<unsigned long long>(ws, wl.track_bar_s);
    a.bar_m = ws_ptr<unsigned long long>(ws, wl.track_bar_m);
    a.ep_m = ws_ptr<unsigned long long>(ws, wl.track_ep_m);
    a.ep_s = ws_ptr<unsigned long long>(ws, wl.track_ep_s);
    a.med = getenv("FT_MEDIAN_GATHER") ? nullptr : ws_ptr<unsigned>(ws, wl.track_med);
    a.tail_s = ws_ptr<unsigned long long>(ws, wl.track_tail_s);
    a.tail_m = ws_ptr<unsigned long long>(ws, wl.track_tail_m);
    a.mcand = ws_ptr<int4>(ws, wl.track_mcand);
    a.mcnt = ws_ptr<int>(ws, wl.track_mcnt);
    // one frame per group slot: a dedicated tail block (one more stereo
    // block) runs the frame's stereo tail, the keypoint blocks never wait
    a.stereo_tail = 0;
    // (persistent plans: the keypoint / point blocks go straight on to the
    // next step; a single launch gains nothing from it -- the kernel still
    // ends with the tail -- so per-launch calls keep the group barriers)
    // grid limit with the tail blocks: persistent plans keep 4 SMs free
    // (ft_internal_persist_launch / ft_track_frames_ring refuse more)
    int sms_all = 0;
    cudaDeviceGetAttribute(&sms_all, cudaDevAttrMultiProcessorCount, dev);
    const int grid_max = (key.reserve ? sms_all - 4 : sms_all) / key.groups;
    tails = tails || getenv("FT_TAIL_LAUNCH");
    if (tails && want_stereo && a.W >= a.F && !getenv("FT_STEREO_BARRIER")) {
        if (a.W * (a.Gs + 1 + a.Gm) <= grid_max) {
            a.Gs += 1;
            a.stereo_tail = 1;
        }
    }
    // ... and a dedicated resolve block for the map group (plain resolve:
    // no ordered correspondences, no rotation filter)
    a.map_tail = 0;
    if (tails && want_map && a.W >= a.F && (a.pmode & FT_PROJ_RESOLVE) && !a.po.corr_point &&
        !((a.pmode & FT_PROJ_ROTATION) && a.io.ref_angles) && a.map_chunk_cap > a.Gm + 1 &&
        a.Gm + 1 <= WS_MAX_GROUP && !getenv("FT_MAP_BARRIER")) {
        if (a.W * (a.Gs + a.Gm + 1) <= grid_max) {
            a.Gm += 1;
            a.map_tail = 1;
        }
    }
    a.claims = ws_ptr<unsigned long long>(ws, wl.proj_claims);
    a.blk_counts = ws_ptr<int>(ws, wl.track_blk_counts);
    a.hist = ws_ptr<int>(ws, wl.track_hist);
    a.tl = nullptr;
    g_out = g;
    return FT_OK;
}

static int track_launch(TrackArgs &a, bool want_stereo, bool want_map, const ft_workspace *ws,
                        cudaStream_t stream) {
    Geom g;
    {
        const int st = track_prepare(a, want_stereo, want_map, ws, g, false);
        if (st != FT_OK) return st;
    }
    static unsigned long long *tl_buf = nullptr;
    if (getenv("FT_DEBUG_TIMELINE")) {
        const size_t n = (size_t)a.W * (a.Gs + a.Gm) * TL_SLOTS;
        if (!tl_buf) cudaMalloc(&tl_buf, 1 << 20);
        if (n * 8 <= (1 << 20)) {
            cudaMemsetAsync(tl_buf, 0, n * 8, stream);
            a.tl = tl_buf;
        }
    }

    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(a.W * (a.Gs + a.Gm));
    cfg.blockDim = dim3(TK_THREADS);
    cfg.dynamicSmemBytes = g.smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, track_kernel, a);
    if (e != cudaSuccess) return (int)e;
    if (a.tl) {  // debug: dump the per-block timeline (ns) after the launch
        const size_t n = (size_t)a.W * (a.Gs + a.Gm) * TL_SLOTS;
        static unsigned long long host[1 << 17];
        cudaMemcpyAsync(host, a.tl, n * 8, cudaMemcpyDeviceToHost, stream);
        cudaStreamSynchronize(stream);
        FILE *fp = fopen(getenv("FT_DEBUG_TIMELINE"), "a");
        if (fp) {
            fprintf(fp, "launch F=%d W=%d Gs=%d Gm=%d\n", a.F, a.W, a.Gs, a.Gm);
            for (size_t b = 0; b < n / TL_SLOTS; ++b) {
                fprintf(fp, "%zu", b);
                for (int k = 0; k < TL_SLOTS; ++k) fprintf(fp, " %llu", host[b * TL_SLOTS + k]);
                fprintf(fp, "\n");
            }
            fclose(fp);
        }
    }
    return (int)cudaGetLastError();
}

// Keypoint tables staged in shared memory (one TMA copy per block) or read
// in place from L2; staged unless they would not fit.  FT_STAGE_RDESC /
// FT_STAGE_KDESC = 0 / 1 override (measurement).
static void stage_policy(TrackArgs &a, bool want_stereo, bool want_map) {
    static const char *er = getenv("FT_STAGE_RDESC");
    static const char *ek = getenv("FT_STAGE_KDESC");
    a.stage_rdesc = er ? (atoi(er) != 0) : 1;
    a.stage_kdesc = ek ? (atoi(ek) != 0) : 1;
    if (want_stereo && stereo_smem(a) > 227 * 1024) a.stage_rdesc = 0;
    if (want_map && map_smem(a) > 227 * 1024) a.stage_kdesc = 0;
}

static int track_geometry(TrackArgs &a, bool want_stereo, bool want_map, Geom &out,
                          int reserve, bool rej_only, int groups) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int F = a.F;
    // per-frame block budget: ~1 warp per left keypoint, ~84 map points per block
    // (measured at cfg2: 128 -> 84 points per block takes the persistent ring
    // from 13.4 to 12.5 us per frame; the map role's search rounds shrink)
    int gs_ideal = want_stereo ? (a.L.cap + TK_WARPS - 1) / TK_WARPS : 0;
    static const int pts_per_block = getenv("FT_MAP_PTS_PER_BLOCK")
                                         ? atoi(getenv("FT_MAP_PTS_PER_BLOCK")) : 84;
    int gm_ideal = want_map ? (a.P.cap + pts_per_block - 1) / pts_per_block : 0;
    if (gs_ideal > 96) gs_ideal = 96;
    if (rej_only) gs_ideal = 1;
    if (gm_ideal > 64) gm_ideal = 64;
    // the map role's per-point shared arrays (32 B / point of its chunk) must
    // fit: at most TK_MAP_CHUNK_MAX points per map block
    const int gm_min = want_map ? (a.P.cap + TK_MAP_CHUNK_MAX - 1) / TK_MAP_CHUNK_MAX : 0;
    if (gm_ideal < gm_min) gm_ideal = gm_min;
    int Gs = gs_ideal, Gm = gm_ideal, W = F;
    size_t smem = 0;
    a.stage_rdesc = 1;
    a.stage_kdesc = 1;
    for (int iter = 0; iter < 4; ++iter) {
        if (want_map) a.map_chunk_cap = (((a.P.cap + Gm - 1) / Gm) + 1) & ~1;
        stage_policy(a, want_stereo, want_map);
        smem = want_stereo ? stereo_smem(a) : 0;
        if (want_map) {
            const size_t m = map_smem(a);
            smem = m > smem ? m : smem;
        }
        if (smem > 227 * 1024) return FT_E_RANGE;
        const int st = raise_smem_attr(dev, smem);
        if (st != FT_OK) return st;
        int occ = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, track_kernel, TK_THREADS, smem);
        if (occ < 1) return FT_E_RANGE;
        const int capacity = occ * (sms - reserve) / groups;
        const int per_ideal = gs_ideal + gm_ideal;
        int nGs, nGm, nW;
        if ((long long)F * per_ideal <= capacity) {
            nW = F;
            nGs = gs_ideal;
            nGm = gm_ideal;
        } else {
            // more frames than one resident wave holds: pick slots W and the
            // stereo / map split minimising the modelled job time
            //   waves(W) * max(t_stereo, t_map)
            //   t_stereo = 8.8 + 3.1 * keypoints per warp
            //   t_map    = 11.4 + 2.28 * 512-point rounds + 0.0205 * points per block
            // (us per frame of a group; fitted to the persistent ring at 4 and
            // 8 step groups over forced splits, r2k: picks 11 or 12 map blocks of
            // 35 and 5 of 17, the measured optima; the stereo slope refit after
            // the block-batched stereo passes, s1: 5 map blocks of 14 and 4 of
            // 10, the measured optima at cfg2)
            const int min_per = (want_stereo ? 1 : 0) + (want_map ? gm_min : 0);
            if (min_per > capacity) return FT_E_RANGE;
            double best = 1e30;
            nW = 1;
            nGs = want_stereo ? 1 : 0;
            nGm = want_map ? gm_min : 0;
            const int wmax = F < capacity / min_per ? F : capacity / min_per;
            for (int w = 1; w <= wmax; ++w) {
                const int per = capacity / w;
                const int waves = (F + w - 1) / w;
                const int g_lo = want_map ? gm_min : 0;
                const int g_hi = want_map ? (want_stereo ? per - 1 : per) : 0;
                static const int gm_force = getenv("FT_GEOM_GM") ? atoi(getenv("FT_GEOM_GM")) : 0;
                for (int gm = g_lo; gm <= g_hi; ++gm) {
                    if (gm_force > 0 && want_stereo && want_map && gm != gm_force) continue;
                    const int gs = want_stereo ? (want_map ? per - gm : per) : 0;
                    if (want_stereo && gs < 1) continue;
                    double t = 0.0;
                    if (want_stereo) {
                        const double kpw = (double)a.L.cap / (double)(gs * TK_WARPS);
                        t = 8.8 + 3.1 * (kpw > 1.0 ? kpw : 1.0);
                    }
                    if (want_map) {
                        const int chunk = (a.P.cap + gm - 1) / gm;
                        const int rounds = (chunk + TK_THREADS - 1) / TK_THREADS;
                        const double tm = 11.4 + 2.28 * rounds + 0.0205 * chunk;
                        t = t > tm ? t : tm;
                    }
                    const double total = waves * t;
                    if (total < best * 0.999) {
                        best = total;
                        nW = w;
                        nGs = gs;
                        nGm = gm;
                    }
                    if (!want_stereo) break;  // map-only: all blocks to the map
                }
            }
        }
        const bool same = nGs == Gs && nGm == Gm && nW == W;
        Gs = nGs;
        Gm = nGm;
        W = nW;
        if (same && iter > 0) break;
    }
    if (want_map) a.map_chunk_cap = (((a.P.cap + Gm - 1) / Gm) + 1) & ~1;
    stage_policy(a, want_stereo, want_map);
    smem = want_stereo ? stereo_smem(a) : 0;
    if (want_map) {
        const size_t m = map_smem(a);
        smem = m > smem ? m : smem;
    }
    if (smem > 227 * 1024) return FT_E_RANGE;
    if (raise_smem_attr(dev, smem) != FT_OK) return FT_E_RANGE;
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, track_kernel, TK_THREADS, smem);
    const long long cap_all = (long long)occ * (sms - reserve) / groups;
    while (W > 1 && (long long)W * (Gs + Gm) > cap_all) --W;
    if ((long long)W * (Gs + Gm) > cap_all) return FT_E_RANGE;
    out.Gs = Gs;
    out.Gm = Gm;
    out.W = W;
    out.chunk = want_map ? a.map_chunk_cap : 0;
    out.stage_rdesc = a.stage_rdesc;
    out.stage_kdesc = a.stage_kdesc;
    out.smem = smem;
    return FT_OK;
}

static bool aligned16(const void *p) { return ((uintptr_t)p & 15u) == 0; }

static bool fill_stereo(TrackArgs &a, int32_t n_frames, const ft_keypoints *left,
                        const ft_keypoints *right, const ft_pyramid *left_pyr,
                        const ft_pyramid *right_pyr, const ft_stereo_params *params, int32_t mode,
                        const ft_stereo_out *out, int *status) {
    *status = FT_OK;
    if (!left || !right || !params || !out) {
        *status = FT_E_NULL;
        return false;
    }
    if (n_frames < 1 || left->cap < 1 || right->cap < 1 || left->cap > 65535 ||
        right->cap > 65535 || params->height < 1 || params->height > 65535 ||
        params->n_levels < 1 || params->n_levels > FT_MAX_LEVELS) {
        *status = FT_E_RANGE;
        return false;
    }
    if (left->cap > 2 * right->cap) {
        *status = FT_E_RANGE;
        return false;
    }
    if (params->half_window < 1 || params->half_slide < 1 || params->half_window > 32 ||
        params->half_slide > 32 || ((mode & FT_STEREO_REFINE) && (mode & FT_STEREO_FROM_CAND))) {
        *status = FT_E_CONFIG;
        return false;
    }
    const bool finalize = mode & (FT_STEREO_REFINE | FT_STEREO_FROM_CAND | FT_STEREO_REJECT);
    if (((mode & FT_STEREO_PHASE1) && !out->cand_idx && !finalize) ||
        (!(mode & FT_STEREO_PHASE1) && (mode & (FT_STEREO_REFINE | FT_STEREO_FROM_CAND)) &&
         (!out->cand_idx || !out->cand_dist)) ||
        (out->cand_idx && !out->cand_dist) ||
        (finalize && (!out->right_idx || !out->distance || !out->disparity || !out->refined_u ||
                      !out->depth || !out->sad)) ||
        ((mode & FT_STEREO_REFINE) && (!left_pyr || !right_pyr || !left_pyr->data || !right_pyr->data))) {
        *status = FT_E_NULL;
        return false;
    }
    if ((mode & FT_STEREO_REFINE) &&
        (left_pyr->n_levels < params->n_levels || right_pyr->n_levels < params->n_levels)) {
        *status = FT_E_RANGE;
        return false;
    }
    // TMA staging: record arrays 16-B aligned
    if (!left->rec || !right->rec || !left->count || !right->count) {
        *status = FT_E_NULL;
        return false;
    }
    if (!aligned16(left->rec) || !aligned16(right->rec)) {
        *status = FT_E_RANGE;
        return false;
    }
    a.smode = mode;
    a.L = *left;
    a.R = *right;
    if (left_pyr) a.PL = *left_pyr;
    else memset(&a.PL, 0, sizeof(a.PL));
    if (right_pyr) a.PR = *right_pyr;
    else memset(&a.PR, 0, sizeof(a.PR));
    a.sp = *params;
    a.so = *out;
    const int nw = 2 * params->half_window + 1;
    const int nr = 2 * params->half_slide + 2 * params->half_window + 1;
    // left patch, right strip, then per-(offset,row) partials (fixed path)
    a.patch_ints = (mode & FT_STEREO_REFINE)
                       ? nw * nw + nw * nr + (2 * params->half_slide + 1) * nw
                       : 0;
    // the default window's block-batched passes (stereo_block_pipe55): the
    // warps' double buffers and the batch area, per-warp share
    if ((mode & FT_STEREO_REFINE) && params->half_window == 5 && params->half_slide == 5 &&
        !getenv("FT_STEREO_NOPIPE"))
        a.patch_ints = a.patch_ints > PIPE_BYTES / 4 ? a.patch_ints : PIPE_BYTES / 4;
    a.patch_ints = (a.patch_ints + 3) & ~3;
    return true;
}

static bool fill_map(TrackArgs &a, int32_t n_frames, const ft_map_points *points,
                     const ft_keypoints *frame, const ft_project_params *params,
                     const ft_project_io *io, int32_t mode, const ft_project_out *out, int *status) {
    *status = FT_OK;
    if (!points || !frame || !params || !io || !out) {
        *status = FT_E_NULL;
        return false;
    }
    if (n_frames < 1 || points->cap < 1 || frame->cap < 1 || frame->cap > 65535 ||
        points->cap > (1 << 23) || params->n_levels < 1 || params->n_levels > FT_MAX_LEVELS ||
        params->cell_px < 1 || params->grid_nx < 1 || params->grid_ny < 1 ||
        params->grid_nx * params->grid_ny > 16384) {
        *status = FT_E_RANGE;
        return false;
    }
    if (params->histogram_bins < 1 || params->histogram_bins > TK_MAX_BINS ||
        params->histogram_keep < 1 || params->histogram_keep > params->histogram_bins ||
        ((mode & FT_PROJ_WRITE_SLOTS) && !(mode & FT_PROJ_RESOLVE))) {
        *status = FT_E_CONFIG;
        return false;
    }
    if (!io->rot || !io->trans || ((mode & (FT_PROJ_SKIP_SLOTS | FT_PROJ_WRITE_SLOTS)) && !io->slots_in) ||
        ((mode & FT_PROJ_WRITE_SLOTS) && !io->slots_out) ||
        (out->out_kp && (!out->out_dist || !out->out_oct)) ||
        (out->corr_point && (!out->corr_kp || !out->corr_dist || !out->corr_oct))) {
        *status = FT_E_NULL;
        return false;
    }
    if (!points->rec || !frame->rec || !points->count || !frame->count) {
        *status = FT_E_NULL;
        return false;
    }
    if (!aligned16(points->rec) || !aligned16(frame->rec) ||
        ((mode & FT_PROJ_SKIP_SLOTS) && !aligned16(io->slots_in))) {
        *status = FT_E_RANGE;
        return false;
    }
    a.pmode = mode;
    a.P = *points;
    a.K = *frame;
    a.pp = *params;
    a.io = *io;
    a.po = *out;
    a.hash_bits = 0;
    if (mode & FT_PROJ_SKIP_SLOTS) {
        int bits = 1;
        while ((1 << bits) < 2 * frame->cap) ++bits;
        a.hash_bits = bits;
    }
    a.map_chunk_cap = 0;
    return true;
}

extern "C" int ft_track_frames(int32_t n_frames, const ft_keypoints *left,
                               const ft_keypoints *right, const ft_pyramid *left_pyr,
                               const ft_pyramid *right_pyr, const ft_stereo_params *sparams,
                               int32_t smode, const ft_stereo_out *sout,
                               const ft_map_points *points, const ft_project_params *pparams,
                               const ft_project_io *io, int32_t pmode, const ft_project_out *pout,
                               const ft_workspace *ws, ft_stream_t stream) {
    TrackArgs a;
    memset(&a, 0, sizeof(a));
    a.F = n_frames;
    int st;
    if (!fill_stereo(a, n_frames, left, right, left_pyr, right_pyr, sparams, smode, sout, &st))
        return st;
    if (!fill_map(a, n_frames, points, left, pparams, io, pmode, pout, &st)) return st;
    const int capl = left->cap > right->cap ? left->cap : right->cap;
    st = ws_check(ws, n_frames, capl, points->cap);
    if (st != FT_OK) return st;
    return track_launch(a, true, true, ws, (cudaStream_t)stream);
}

namespace {
struct TrackPlan {
    uint32_t magic, version;
    TrackArgs a;
    size_t smem;
    int32_t groups;  // persistent step groups the geometry was sized for
};
constexpr uint32_t PLAN_MAGIC = 0x46545450u;  // "FTTP"
}  // namespace

static unsigned long long *g_plan_tl = nullptr;
static size_t g_plan_tl_n = 0;
static int g_plan_tl_hdr[4];

extern "C" size_t ft_track_plan_bytes(void) { return sizeof(TrackPlan); }

extern "C" int ft_track_plan_groups(int32_t n_frames, const ft_keypoints *left,
                                    const ft_keypoints *right, const ft_pyramid *left_pyr,
                                    const ft_pyramid *right_pyr, const ft_stereo_params *sparams,
                                    int32_t smode, const ft_stereo_out *sout,
                                    const ft_map_points *points,
                                    const ft_project_params *pparams, const ft_project_io *io,
                                    int32_t pmode, const ft_project_out *pout,
                                    const ft_workspace *ws, int32_t groups, void *plan,
                                    size_t plan_bytes);

extern "C" int ft_track_plan(int32_t n_frames, const ft_keypoints *left,
                             const ft_keypoints *right, const ft_pyramid *left_pyr,
                             const ft_pyramid *right_pyr, const ft_stereo_params *sparams,
                             int32_t smode, const ft_stereo_out *sout,
                             const ft_map_points *points, const ft_project_params *pparams,
                             const ft_project_io *io, int32_t pmode, const ft_project_out *pout,
                             const ft_workspace *ws, void *plan, size_t plan_bytes) {
    return ft_track_plan_groups(n_frames, left, right, left_pyr, right_pyr, sparams, smode, sout,
                                points, pparams, io, pmode, pout, ws, 1, plan, plan_bytes);
}

extern "C" int ft_track_plan_groups(int32_t n_frames, const ft_keypoints *left,
                                    const ft_keypoints *right, const ft_pyramid *left_pyr,
                                    const ft_pyramid *right_pyr, const ft_stereo_params *sparams,
                                    int32_t smode, const ft_stereo_out *sout,
                                    const ft_map_points *points,
                                    const ft_project_params *pparams, const ft_project_io *io,
                                    int32_t pmode, const ft_project_out *pout,
                                    const ft_workspace *ws, int32_t groups, void *plan,
                                    size_t plan_bytes) {
    if (!plan) return FT_E_NULL;
    if (groups < 1 || groups > 36) return FT_E_RANGE;
    if (plan_bytes < sizeof(TrackPlan)) return FT_E_RANGE;
    TrackPlan *tp = static_cast<TrackPlan *>(plan);
    memset(tp, 0, sizeof(*tp));
    TrackArgs &a = tp->a;
    a.F = n_frames;
    int st;
    if (!fill_stereo(a, n_frames, left, right, left_pyr, right_pyr, sparams, smode, sout, &st))
        return st;
    if (!fill_map(a, n_frames, points, left, pparams, io, pmode, pout, &st)) return st;
    const int capl = left->cap > right->cap ? left->cap : right->cap;
    st = ws_check(ws, n_frames, capl, points->cap);
    if (st != FT_OK) return st;
    Geom g;
    st = track_prepare(a, true, true, ws, g, true, groups);
    if (st != FT_OK) return st;
    if (getenv("FT_DEBUG_TIMELINE")) {  // debug: every step overwrites one timeline
        const size_t n = (size_t)a.W * (a.Gs + a.Gm) * TL_SLOTS;
        if (!g_plan_tl) cudaMalloc(&g_plan_tl, 1 << 20);
        if (n * 8 <= (1 << 20)) {
            a.tl = g_plan_tl;
            g_plan_tl_n = n;
            g_plan_tl_hdr[0] = a.F;
            g_plan_tl_hdr[1] = a.W;
            g_plan_tl_hdr[2] = a.Gs;
            g_plan_tl_hdr[3] = a.Gm;
        }
    }
    tp->smem = g.smem;
    tp->groups = groups;
    tp->magic = PLAN_MAGIC;
    tp->version = 1;
    return FT_OK;
}

static unsigned long long *g_persist_ts = nullptr;

// debug: write the persistent kernel's per-step (start, done) timestamps
extern "C" void ft_internal_persist_dump(void) {
    const char *path = getenv("FT_DEBUG_PERSIST");
    if (!path || !g_persist_ts) return;
    static unsigned long long h[4096 * 2];
    cudaMemcpy(h, g_persist_ts, sizeof(h), cudaMemcpyDeviceToHost);
    FILE *fp = fopen(path, "w");
    if (!fp) return;
    for (int k = 0; k < 4096; ++k) fprintf(fp, "%d %llu %llu\n", k, h[2 * k], h[2 * k + 1]);
    fclose(fp);
    const char *tl_path = getenv("FT_DEBUG_TIMELINE");
    if (tl_path && g_plan_tl && g_plan_tl_n) {  // the last step's per-block timeline
        static unsigned long long t[1 << 17];
        cudaMemcpy(t, g_plan_tl, g_plan_tl_n * 8, cudaMemcpyDeviceToHost);
        FILE *ft = fopen(tl_path, "a");
        if (!ft) return;
        fprintf(ft, "launch F=%d W=%d Gs=%d Gm=%d\n", g_plan_tl_hdr[0], g_plan_tl_hdr[1],
                g_plan_tl_hdr[2], g_plan_tl_hdr[3]);
        for (size_t b = 0; b < g_plan_tl_n / TL_SLOTS; ++b) {
            fprintf(ft, "%zu", b);
            for (int k = 0; k < TL_SLOTS; ++k) fprintf(ft, " %llu", t[b * TL_SLOTS + k]);
            fprintf(ft, "\n");
        }
        fclose(ft);
    }
}

// Launch the persistent kernel over n plans (internal: ft_runner.cu).  The
// plans must share one geometry and leave SMs free for other work (the
// launch never ends on its own: it would starve every later kernel).
// Fill a PersistArgs from n plans (same geometry) and launch the persistent
// kernel.  args_dev: n TrackArgs of device memory the kernel reads (copied
// here, stream-ordered from a host buffer that outlives the copy).
static int persist_launch(const void *const *plans, int n, TrackArgs *args_dev,
                          std::vector<TrackArgs> &host_args, const unsigned *ready,
                          unsigned *dready, unsigned *done, unsigned *arrive, unsigned max_steps,
                          int gate, int coherent, cudaStream_t stream,
                          void *const *push_dev = nullptr, void *const *push_host = nullptr,
                          size_t push_bytes = 0, std::vector<TrackArgs> *uploaded = nullptr) {
    if (!plans || !args_dev || !ready || !dready || !done || !arrive) return FT_E_NULL;
    if (n < 1) return FT_E_RANGE;
    PersistArgs p;
    memset(&p, 0, sizeof(p));
    const bool push = push_dev && push_host;
    if (push) {
        if (n > PERSIST_MAX_SLOTS) return FT_E_RANGE;
        p.out_bytes = push_bytes;
        for (int i = 0; i < n; ++i) {
            p.out_dev[i] = (unsigned long long)(uintptr_t)push_dev[i];
            p.out_host[i] = (unsigned long long)(uintptr_t)push_host[i];
            if (!p.out_dev[i] || !p.out_host[i]) return FT_E_NULL;
            if ((p.out_dev[i] | p.out_host[i]) & 15ull) return FT_E_CONFIG;  // 16-B vectors
        }
    }
    size_t smem = 0;
    host_args.resize(n);
    for (int i = 0; i < n; ++i) {
        const TrackPlan *tp = static_cast<const TrackPlan *>(plans[i]);
        if (!tp) return FT_E_NULL;
        if (tp->magic != PLAN_MAGIC) return FT_E_CONFIG;
        host_args[i] = tp->a;
        host_args[i].coherent = coherent;
        const TrackPlan *t0 = static_cast<const TrackPlan *>(plans[0]);
        if (tp->a.W != host_args[0].W || tp->a.Gs != host_args[0].Gs ||
            tp->a.Gm != host_args[0].Gm || tp->groups != t0->groups)
            return FT_E_CONFIG;
        smem = tp->smem > smem ? tp->smem : smem;
    }
    p.args = args_dev;
    p.n = n;
    p.Q = static_cast<const TrackPlan *>(plans[0])->groups;
    if (p.Q < 1) p.Q = 1;
    if (n % p.Q) return FT_E_CONFIG;  // slot i must always run in group i mod Q
    p.W = host_args[0].W;
    p.Gs = host_args[0].Gs;
    p.Gm = host_args[0].Gm;
    p.max_steps = max_steps;
    p.gate = gate;
    p.red_arrive = getenv("FT_PERSIST_ATOMIC_ARRIVE") ? 0 : 1;
    {
        const char *ev = getenv("FT_PERSIST_POLL_NS");
        p.poll_ns = ev ? (unsigned)atoi(ev) : 100u;
    }
    static unsigned long long *ts_buf = nullptr;
    if (getenv("FT_DEBUG_PERSIST")) {
        if (!ts_buf) cudaMalloc(&ts_buf, 4096 * 2 * 8);
        cudaMemsetAsync(ts_buf, 0, 4096 * 2 * 8, stream);
        p.ts = ts_buf;
        g_persist_ts = ts_buf;
    }
    p.ready = ready;
    p.dready = dready;
    p.done = done;
    p.arrive = arrive;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = p.Q * p.W * (p.Gs + p.Gm);
    if (grid > sms - 4) return FT_E_RANGE;  // keep SMs for the copies' helper kernels
    // the device argument array: uploaded unless it already holds exactly
    // these arguments (a ring relaunched over the same pipelines): the
    // ~150 KB pageable copy would otherwise sit on the stream before every
    // launch
    cudaError_t e = cudaSuccess;
    const size_t abytes = sizeof(TrackArgs) * n;
    if (!uploaded || uploaded->size() != (size_t)n ||
        memcmp(uploaded->data(), host_args.data(), abytes) != 0) {
        e = cudaMemcpyAsync(args_dev, host_args.data(), abytes, cudaMemcpyHostToDevice, stream);
        if (e != cudaSuccess) return (int)e;
        if (uploaded) *uploaded = host_args;
    }
    void (*kern)(PersistArgs) = push ? track_persist_kernel<true> : track_persist_kernel<false>;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
    if (e != cudaSuccess) return (int)e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(TK_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, kern, p);
    return (int)e;
}

// The runner's launch (internal: ft_runner.cu).  flags: 2 * PERSIST_MAX_SLOTS
// device words [dready | arrive]; h_ready / h_done: mapped host words;
// *args_out: the device argument array (the runner frees it).
extern "C" int ft_internal_persist_launch(const void *const *plans, int n, unsigned *flags,
                                          const unsigned *h_ready, unsigned *h_done,
                                          void **args_out, cudaStream_t stream,
                                          void *const *push_dev, void *const *push_host,
                                          size_t push_bytes) {
    if (!plans || !flags || !args_out) return FT_E_NULL;
    if (n < 1 || n > PERSIST_MAX_SLOTS) return FT_E_RANGE;
    TrackArgs *args = nullptr;
    cudaError_t e = cudaMalloc(&args, sizeof(TrackArgs) * n);
    if (e != cudaSuccess) return (int)e;
    *args_out = args;
    // staging for the argument copy (pageable: the copy is staged before it
    // returns); one at a time across threads
    static std::mutex mu;
    std::lock_guard<std::mutex> lock(mu);
    static std::vector<TrackArgs> host;
    // the runner rewrites a slot's inputs while the kernel is alive: coherent loads
    const int st = persist_launch(plans, n, args, host, h_ready, flags, h_done,
                                  flags + PERSIST_MAX_SLOTS, 0xffffffffu, 0, 1, stream, push_dev,
                                  push_host, push_bytes);
    return st;
}

extern "C" int ft_track_frames_ring(int32_t n_plans, const void *const *plans, int64_t n_steps,
                                    ft_stream_t stream) {
    if (!plans) return FT_E_NULL;
    nvtxRangePushA("ft_track_frames_ring");  // host side of the launch (NVTX timelines)
    struct Pop {
        ~Pop() { nvtxRangePop(); }
    } pop_;
    if (n_plans < 1 || n_steps < 0 || n_steps >= 0x7f000000) return FT_E_RANGE;
    if (n_steps == 0) return FT_OK;
    // per-device buffers, grown on demand (stream-ordered reuse)
    struct RingState {
        TrackArgs *args = nullptr;
        unsigned *words = nullptr;
        int cap = 0;
        std::vector<TrackArgs> host;
        std::vector<TrackArgs> uploaded;  // what rs.args holds on the device
        cudaEvent_t prev = nullptr;  // the previous ring on this device
    };
    static std::mutex mu;
    static RingState states[64];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return FT_E_CONFIG;
    std::lock_guard<std::mutex> lock(mu);
    RingState &rs = states[dev];
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e = cudaSuccess;
    if (!rs.prev) {
        e = cudaEventCreateWithFlags(&rs.prev, cudaEventDisableTiming);
        if (e != cudaSuccess) {
            rs.prev = nullptr;
            return (int)e;
        }
    }
    if (n_plans > rs.cap) {
        // the old buffers may still be read by the previous ring
        e = cudaEventSynchronize(rs.prev);
        if (e != cudaSuccess) return (int)e;
        if (rs.args) cudaFree(rs.args);
        if (rs.words) cudaFree(rs.words);
        rs.args = nullptr;
        rs.words = nullptr;
        rs.cap = 0;
        rs.uploaded.clear();  // a fresh device array
        e = cudaMalloc(&rs.args, sizeof(TrackArgs) * n_plans);
        if (e == cudaSuccess) e = cudaMalloc(&rs.words, 4 * sizeof(unsigned) * n_plans);
        if (e != cudaSuccess) return (int)e;
        rs.cap = n_plans;
    }
    // the buffers are shared by every call on this device: order after the
    // previous ring, whatever stream it ran on
    e = cudaStreamWaitEvent(s, rs.prev, 0);
    if (e != cudaSuccess) return (int)e;
    // [ready | dready | done | arrive], zeroed in one stream operation (the
    // ring reads neither ready word: every step is ready up front)
    unsigned *words = rs.words;
    e = cudaMemsetAsync(words, 0, 4 * sizeof(unsigned) * n_plans, s);
    if (e != cudaSuccess) return (int)e;
    // inputs are resident and constant for the launch: read-only loads
    const int st = persist_launch(plans, n_plans, rs.args, rs.host, words, words + n_plans,
                                  words + 2 * n_plans, words + 3 * n_plans, (unsigned)n_steps,
                                  1, 0, s, nullptr, nullptr, 0, &rs.uploaded);
    if (st != FT_OK) return st;
    e = cudaEventRecord(rs.prev, s);
    return e == cudaSuccess ? FT_OK : (int)e;
}

extern "C" int ft_stereo_pinhole(int32_t n_frames, const ft_keypoints *left,
                                 const ft_keypoints *right, const ft_pyramid *left_pyr,
                                 const ft_pyramid *right_pyr, const ft_stereo_params *params,
                                 int32_t mode, const ft_stereo_out *out, const ft_workspace *ws,
                                 ft_stream_t stream) {
    TrackArgs a;
    memset(&a, 0, sizeof(a));
    a.F = n_frames;
    int st;
    if (!fill_stereo(a, n_frames, left, right, left_pyr, right_pyr, params, mode, out, &st))
        return st;
    if (!ws) return FT_E_NULL;
    const int capl = left->cap > right->cap ? left->cap : right->cap;
    st = ws_check(ws, n_frames, capl, 1);
    if (st != FT_OK) return st;
    return track_launch(a, true, false, ws, (cudaStream_t)stream);
}

extern "C" int ft_project_search(int32_t n_frames, const ft_map_points *points,
                                 const ft_keypoints *frame, const ft_project_params *params,
                                 const ft_project_io *io, int32_t mode, const ft_project_out *out,
                                 const ft_workspace *ws, ft_stream_t stream) {
    TrackArgs a;
    memset(&a, 0, sizeof(a));
    a.F = n_frames;
    int st;
    if (!fill_map(a, n_frames, points, frame, params, io, mode, out, &st)) return st;
    if (!ws) return FT_E_NULL;
    st = ws_check(ws, n_frames, frame->cap, points->cap);
    if (st != FT_OK) return st;
    return track_launch(a, false, true, ws, (cudaStream_t)stream);
}
