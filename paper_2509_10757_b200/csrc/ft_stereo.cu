// ft_stereo.cu -- pinhole stereo matching on sm_100a: phase 1 (row-band
// Hamming search), phase 2 (SAD sub-pixel refinement) or the no-image
// candidate acceptance, and the median-SAD outlier rejection, fused into ONE
// kernel per batch of frames.
//
// Reference semantics (trackfront):
//   phase 1   kernels.py:300-345 stereo_phase1_kernel, stereo.py:77-103
//   buckets   stereo.py:67-74 build_row_buckets
//   phase 2   kernels.py:351-428 stereo_phase2_kernel, stereo.py:106-140
//   no image  stereo.py:143-168 matches_from_candidates
//   reject    stereo.py:171-188 reject_outliers (np.median semantics)
//
// Mapping:
//   grid = (ceil(cap_left / KPB), n_frames), block = 256 threads (8 warps).
//   Each block rebuilds the right image's row-bucket CSR in shared memory
//   (rows of rint(v), clipped).  Each warp owns one left keypoint at a time:
//   lanes stride the contiguous CSR range of rows [r0, r1] and the packed
//   (distance << 16 | j) key is reduced with redux.sync -- the lexicographic
//   minimum is the reference's "lower right index on ties", so bucket order
//   does not matter.  Phase 2 stages the (2w+1)^2 left patch and the
//   (2w+1) x (2s+2w+1) right strip in shared memory and spreads the
//   offsets x rows jobs over all 32 lanes.  With REJECT, the last block of
//   each frame (atomic ticket) radix-selects the median accepted SAD and
//   resets the rejected matches.
#include <cstring>

#include "ft_common.cuh"
#include "ft_ws.cuh"

namespace ft {

constexpr int ST_THREADS = 256;
constexpr int ST_WARPS = ST_THREADS / 32;
constexpr int ST_KP_PER_WARP = 2;
constexpr int ST_KPB = ST_WARPS * ST_KP_PER_WARP;  // left keypoints per block
constexpr int MED_BITS = 11;
constexpr int MED_BINS = 1 << MED_BITS;

struct StereoArgs {
    ft_keypoints L, R;
    ft_pyramid PL, PR;
    ft_stereo_params p;
    int32_t mode;
    ft_stereo_out o;
    unsigned *counters;  // [F] last-block tickets
    int32_t patch_ints;  // per-warp staging ints (phase 2)
};

struct StereoSmem {
    int *row_start;   // [H+1]
    int *row_cursor;  // [H]
    uint16_t *items;  // [cap_right]
    int *patch;       // [ST_WARPS][patch_ints]
    int *scan_tmp;    // [32]
    int *flag;
};

__device__ __forceinline__ int phase1_candidate(const StereoArgs &a, const StereoSmem &sm,
                                                int64_t lk, int64_t rbase, int lane,
                                                int &cand_dist) {
    const double v = a.L.v[lk], u = a.L.u[lk];
    const int o = a.L.octave[lk];
    const double band = a.p.band_factor * a.p.scale_pow[clampi(o, 0, FT_MAX_LEVELS - 1)];
    long long r0 = (long long)floor(v - band);
    long long r1 = (long long)ceil(v + band);
    const int H = a.p.height;
    if (r0 < 0) r0 = 0;
    if (r1 > H - 1) r1 = H - 1;
    uint32_t best = NO_KEY;
    if (r0 <= r1) {
        const int beg = sm.row_start[r0], end = sm.row_start[r1 + 1];
        if (beg < end) {
            const Desc ld = load_desc(a.L.desc, lk);
            for (int ii = beg + lane; ii < end; ii += 32) {
                const int j = sm.items[ii];
                const int64_t rj = rbase + j;
                const int ro = a.R.octave[rj];
                if (ro < o - 1 || ro > o + 1) continue;
                if (fabs(a.R.v[rj] - v) > band) continue;
                const double disp = u - a.R.u[rj];
                if (disp < a.p.min_disparity || disp > a.p.max_disparity) continue;
                const uint32_t d = hamming(ld, load_desc(a.R.desc, rj));
                best = min(best, (d << 16) | (uint32_t)j);
            }
        }
    }
    best = __reduce_min_sync(FULL, best);
    if (best != NO_KEY && (int)(best >> 16) <= a.p.t_match) {
        cand_dist = (int)(best >> 16);
        return (int)(best & 0xffffu);
    }
    cand_dist = 10000;
    return -1;
}

// Phase 2 for one candidate; all lanes return the same verdict.
__device__ __forceinline__ bool phase2_refine(const StereoArgs &a, int *patch, int f, int64_t lk,
                                              int64_t rj, int lane, double &disp_out,
                                              double &ur_out, long long &sad_out) {
    const int o = clampi(a.L.octave[lk], 0, a.PL.n_levels - 1);
    const double s = a.p.scale_pow[o];
    const double ulev = a.L.u[lk] / s, vlev = a.L.v[lk] / s, urlev = a.R.u[rj] / s;
    const long long xi = round_half_even(ulev), yi = round_half_even(vlev),
                    xr0 = round_half_even(urlev);
    const int hw = a.p.half_window, hs = a.p.half_slide;
    const long long wl = a.PL.widths[o], hl = a.PL.heights[o];
    const long long wr = a.PR.widths[o], hr = a.PR.heights[o];
    if (xi - hw < 0 || xi + hw >= wl || yi - hw < 0 || yi + hw >= hl) return false;
    if (xr0 - hs - hw < 0 || xr0 + hs + hw >= wr || yi - hw < 0 || yi + hw >= hr) return false;
    const uint8_t *lp = a.PL.data + (int64_t)f * a.PL.frame_bytes + a.PL.offsets[o];
    const uint8_t *rp = a.PR.data + (int64_t)f * a.PR.frame_bytes + a.PR.offsets[o];
    const int nw = 2 * hw + 1, nr = 2 * hs + 2 * hw + 1, noff = 2 * hs + 1;
    int *pl = patch;            // [nw][nw]  L - cl
    int *pr = pl + nw * nw;     // [nw][nr]  R
    int *sads = pr + nw * nr;   // [noff]
    const int cl = lp[yi * wl + xi];
    for (int t = lane; t < nw * nw; t += 32) {
        const int dy = t / nw, dx = t - dy * nw;
        pl[t] = (int)lp[(yi - hw + dy) * wl + (xi - hw + dx)] - cl;
    }
    for (int t = lane; t < nw * nr; t += 32) {
        const int dy = t / nr, dx = t - dy * nr;
        pr[t] = rp[(yi - hw + dy) * wr + (xr0 - hs - hw + dx)];
    }
    for (int t = lane; t < noff; t += 32) sads[t] = 0;
    __syncwarp();
    // job = (offset, row): |(L - cl) - (R - cr)| summed over the row
    for (int t = lane; t < noff * nw; t += 32) {
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
    __syncwarp();  // patch buffer is reused by the next keypoint
    if (!interior) return false;
    const double d_m = (double)s_m;
    const double d_0 = (double)best_sad;
    const double d_p = (double)s_p;
    const double denom = d_m + d_p - 2.0 * d_0;
    if (denom <= 0.0) return false;
    const double delta = (d_m - d_p) / (2.0 * denom);
    if (delta < -1.0 || delta > 1.0) return false;
    const long long best_off = best_oi - hs;
    const double ur_ref = ((double)(xr0 + best_off) + delta) * s;
    const double disp = a.L.u[lk] - ur_ref;
    if (disp < a.p.min_disparity || disp > a.p.max_disparity) return false;
    disp_out = disp;
    ur_out = ur_ref;
    sad_out = best_sad;
    return true;
}

// k-th smallest (0-based) of vals[0..n) by 3-pass radix select (11+11+10 bits).
__device__ uint32_t block_select(const uint32_t *vals, int n, int k, int *hist, int *scan_tmp,
                                 int *bcast) {
    uint32_t prefix = 0, mask = 0;
    const int shifts[3] = {21, 10, 0};
    const int widths[3] = {11, 11, 10};
    for (int pass = 0; pass < 3; ++pass) {
        const int sh = shifts[pass];
        const uint32_t bm = (1u << widths[pass]) - 1u;
        for (int b = threadIdx.x; b < MED_BINS; b += ST_THREADS) hist[b] = 0;
        __syncthreads();
        for (int i = threadIdx.x; i < n; i += ST_THREADS) {
            const uint32_t x = vals[i];
            if ((x & mask) == prefix) atomicAdd(&hist[(x >> sh) & bm], 1);
        }
        __syncthreads();
        constexpr int per = MED_BINS / ST_THREADS;
        const int b0 = threadIdx.x * per;
        int local = 0;
#pragma unroll
        for (int i = 0; i < per; ++i) local += hist[b0 + i];
        int total;
        int run = block_exclusive_scan<ST_THREADS>(local, scan_tmp, total);
        if (k >= run && k < run + local) {
            for (int i = 0; i < per; ++i) {
                const int c = hist[b0 + i];
                if (k < run + c) {
                    bcast[0] = b0 + i;
                    bcast[1] = k - run;
                    break;
                }
                run += c;
            }
        }
        __syncthreads();
        prefix |= (uint32_t)bcast[0] << sh;
        mask |= bm << sh;
        k = bcast[1];
        __syncthreads();
    }
    return prefix;
}

__device__ void reject_outliers_frame(const StereoArgs &a, int f, int n, StereoSmem &sm) {
    const int64_t base = (int64_t)f * a.L.cap;
    // gather accepted SADs (order irrelevant for the median)
    uint32_t *vals = reinterpret_cast<uint32_t *>(sm.row_cursor);  // reuse: >= cap ints
    int *hist = sm.row_start;
    int *misc = sm.flag + 1;  // misc[0] = count, misc[1..2] bcast, misc[3] min
    if (threadIdx.x == 0) misc[0] = 0;
    __syncthreads();
    for (int k = threadIdx.x; k < n; k += ST_THREADS) {
        if (__ldcg(a.o.right_idx + base + k) >= 0) {
            const int pos = atomicAdd(&misc[0], 1);
            vals[pos] = (uint32_t)__ldcg(a.o.sad + base + k);
        }
    }
    __syncthreads();
    const int nm = misc[0];
    if (nm == 0) {
        if (threadIdx.x == 0 && a.o.n_matched) a.o.n_matched[f] = 0;
        return;
    }
    const int k_lo = (nm - 1) / 2, k_hi = nm / 2;
    const uint32_t v_lo = block_select(vals, nm, k_lo, hist, sm.scan_tmp, misc + 1);
    uint32_t v_hi = v_lo;
    if (k_hi != k_lo) {
        // count of values <= v_lo, and the smallest value above it
        if (threadIdx.x == 0) {
            misc[1] = 0;
            misc[3] = 0x7fffffff;
        }
        __syncthreads();
        int cle = 0;
        int mabove = 0x7fffffff;
        for (int i = threadIdx.x; i < nm; i += ST_THREADS) {
            const uint32_t x = vals[i];
            if (x <= v_lo) ++cle;
            else mabove = min(mabove, (int)x);
        }
        atomicAdd(&misc[1], cle);
        atomicMin(&misc[3], mabove);
        __syncthreads();
        v_hi = misc[1] > k_hi ? v_lo : (uint32_t)misc[3];
    }
    // np.median: middle element, or mean of the two middles (float64)
    const double med = (k_hi == k_lo) ? (double)v_lo : ((double)v_lo + (double)v_hi) / 2.0;
    const double thr = a.p.outlier_multiplier * med;
    if (threadIdx.x == 0) misc[0] = 0;
    __syncthreads();
    int kept = 0;
    for (int k = threadIdx.x; k < n; k += ST_THREADS) {
        const int64_t i = base + k;
        if (__ldcg(a.o.right_idx + i) < 0) continue;
        if ((double)__ldcg(a.o.sad + i) > thr) {
            a.o.right_idx[i] = -1;
            a.o.distance[i] = 10000;
            a.o.disparity[i] = 0.0;
            a.o.refined_u[i] = 0.0;
            a.o.depth[i] = 0.0;
            a.o.sad[i] = 0;
        } else {
            ++kept;
        }
    }
    atomicAdd(&misc[0], kept);
    __syncthreads();
    if (threadIdx.x == 0 && a.o.n_matched) a.o.n_matched[f] = misc[0];
}

__global__ void __launch_bounds__(ST_THREADS) stereo_pinhole_kernel(const StereoArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int f = blockIdx.y;
    const int H = a.p.height;
    const int n_left = min(a.L.count[f], a.L.cap);
    const int n_right = min(a.R.count[f], a.R.cap);
    const int64_t lbase = (int64_t)f * a.L.cap;
    const int64_t rbase = (int64_t)f * a.R.cap;
    const int k0 = blockIdx.x * ST_KPB;

    StereoSmem sm;
    int *ip = reinterpret_cast<int *>(smem_raw);
    sm.scan_tmp = ip;
    ip += 32;
    sm.flag = ip;
    ip += 8;
    const int csr_ints = max(H + 1, MED_BINS);
    sm.row_start = ip;
    ip += csr_ints;
    sm.row_cursor = ip;
    ip += max(H, a.L.cap);
    sm.patch = ip;
    ip += ST_WARPS * a.patch_ints;
    sm.items = reinterpret_cast<uint16_t *>(ip);

    const bool do_p1 = a.mode & FT_STEREO_PHASE1;
    const bool do_ref = a.mode & FT_STEREO_REFINE;
    const bool do_fc = a.mode & FT_STEREO_FROM_CAND;
    const bool do_rej = a.mode & FT_STEREO_REJECT;
    const bool finalize = do_ref || do_fc;

    if (k0 < n_left && (do_p1 || finalize)) {
        if (do_p1) {
            const double *rv = a.R.v + rbase;
            block_csr<ST_THREADS>(
                n_right, H,
                [&](int j) {
                    long long r = round_half_even(rv[j]);
                    return (int)(r < 0 ? 0 : (r > H - 1 ? H - 1 : r));
                },
                sm.row_start, sm.row_cursor, sm.items, sm.scan_tmp);
        }
        const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
        int *patch = sm.patch + wid * a.patch_ints;
        for (int t = 0; t < ST_KP_PER_WARP; ++t) {
            const int k = k0 + t * ST_WARPS + wid;
            if (k >= n_left) break;
            const int64_t lk = lbase + k;
            int cand, cdist;
            if (do_p1) {
                cand = phase1_candidate(a, sm, lk, rbase, lane, cdist);
                if (lane == 0) {
                    a.o.cand_idx[lk] = cand;
                    a.o.cand_dist[lk] = cdist;
                }
            } else {
                cand = (int)a.o.cand_idx[lk];
                cdist = (int)a.o.cand_dist[lk];
            }
            if (!finalize) continue;
            bool ok = false;
            double disp = 0.0, ur = 0.0;
            long long sad = 0;
            if (cand >= 0 && cand < n_right) {
                const int64_t rj = rbase + cand;
                if (do_ref) {
                    ok = phase2_refine(a, patch, f, lk, rj, lane, disp, ur, sad);
                } else {  // matches_from_candidates (stereo.py:154-160)
                    disp = a.L.u[lk] - a.R.u[rj];
                    ok = !(disp < a.p.min_disparity || disp > a.p.max_disparity);
                    ur = a.R.u[rj];
                    sad = 0;
                }
            }
            if (lane == 0) {
                a.o.right_idx[lk] = ok ? cand : -1;
                a.o.distance[lk] = ok ? cdist : 10000;
                a.o.disparity[lk] = ok ? disp : 0.0;
                a.o.refined_u[lk] = ok ? ur : 0.0;
                a.o.depth[lk] = ok ? a.p.baseline_times_fx / disp : 0.0;
                a.o.sad[lk] = ok ? sad : 0;
            }
        }
    }
    if (!finalize && !do_rej) return;
    if (do_rej) {
        if (last_block_ticket(a.counters + f, gridDim.x, sm.flag))
            reject_outliers_frame(a, f, n_left, sm);
        return;
    }
    if (a.o.n_matched && last_block_ticket(a.counters + f, gridDim.x, sm.flag)) {
        if (threadIdx.x == 0) sm.flag[1] = 0;
        __syncthreads();
        int c = 0;
        for (int k = threadIdx.x; k < n_left; k += ST_THREADS)
            c += __ldcg(a.o.right_idx + lbase + k) >= 0;
        atomicAdd(&sm.flag[1], c);
        __syncthreads();
        if (threadIdx.x == 0) a.o.n_matched[f] = sm.flag[1];
    }
}

__global__ void hamming_pairs_kernel(const uint64_t *a, const uint64_t *b, int64_t n,
                                     int64_t *out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = hamming(load_desc(a, i), load_desc(b, i));
}

size_t stereo_smem_bytes(int H, int cap_left, int cap_right, int patch_ints) {
    size_t ints = 32 + 8 + (size_t)max(H + 1, MED_BINS) + (size_t)max(H, cap_left) +
                  (size_t)ST_WARPS * patch_ints;
    return ints * 4 + (size_t)cap_right * 2 + 16;
}

}  // namespace ft

using namespace ft;

extern "C" int ft_hamming_pairs(const uint64_t *a, const uint64_t *b, int64_t n, int64_t *out,
                                ft_stream_t stream) {
    if (n < 0) return FT_E_RANGE;
    if (n == 0) return FT_OK;
    if (!a || !b || !out) return FT_E_NULL;
    const int threads = 256;
    int64_t blocks = (n + threads - 1) / threads;
    if (blocks > 148 * 16) blocks = 148 * 16;
    hamming_pairs_kernel<<<(unsigned)blocks, threads, 0, (cudaStream_t)stream>>>(a, b, n, out);
    return (int)cudaGetLastError();
}

extern "C" int ft_stereo_pinhole(int32_t n_frames, const ft_keypoints *left,
                                 const ft_keypoints *right, const ft_pyramid *left_pyr,
                                 const ft_pyramid *right_pyr, const ft_stereo_params *params,
                                 int32_t mode, const ft_stereo_out *out, const ft_workspace *ws,
                                 ft_stream_t stream) {
    if (!left || !right || !params || !out || !ws) return FT_E_NULL;
    if (n_frames < 1 || left->cap < 1 || right->cap < 1 || left->cap > 65535 ||
        right->cap > 65535)
        return FT_E_RANGE;
    if (params->height < 1 || params->height > 65535 || params->n_levels < 1 ||
        params->n_levels > FT_MAX_LEVELS)
        return FT_E_RANGE;
    if (params->half_window < 1 || params->half_slide < 1 || params->half_window > 32 ||
        params->half_slide > 32)
        return FT_E_CONFIG;
    const bool finalize = mode & (FT_STEREO_REFINE | FT_STEREO_FROM_CAND | FT_STEREO_REJECT);
    if ((mode & FT_STEREO_REFINE) && (mode & FT_STEREO_FROM_CAND)) return FT_E_CONFIG;
    if (!out->cand_idx || !out->cand_dist) return FT_E_NULL;
    if (finalize && (!out->right_idx || !out->distance || !out->disparity || !out->refined_u ||
                     !out->depth || !out->sad))
        return FT_E_NULL;
    if ((mode & FT_STEREO_REFINE) && (!left_pyr || !right_pyr || !left_pyr->data ||
                                      !right_pyr->data))
        return FT_E_NULL;
    if ((mode & FT_STEREO_REFINE) &&
        (left_pyr->n_levels < params->n_levels || right_pyr->n_levels < params->n_levels))
        return FT_E_RANGE;
    const int wst = ws_check(ws, n_frames, left->cap > right->cap ? left->cap : right->cap, 1);
    if (wst != FT_OK) return wst;

    StereoArgs a;
    a.L = *left;
    a.R = *right;
    if (left_pyr) a.PL = *left_pyr;
    else memset(&a.PL, 0, sizeof(a.PL));
    if (right_pyr) a.PR = *right_pyr;
    else memset(&a.PR, 0, sizeof(a.PR));
    a.p = *params;
    a.mode = mode;
    a.o = *out;
    a.counters = ws_ptr<unsigned>(ws, ws_layout(ws).stereo_counters);
    const int nw = 2 * params->half_window + 1;
    const int nr = 2 * params->half_slide + 2 * params->half_window + 1;
    a.patch_ints = (mode & FT_STEREO_REFINE) ? nw * nw + nw * nr + 2 * params->half_slide + 1 : 0;
    const size_t smem = stereo_smem_bytes(params->height, left->cap, right->cap, a.patch_ints);
    if (smem > 227 * 1024) return FT_E_RANGE;
    static thread_local size_t configured = 0;
    if (smem > 48 * 1024 && smem > configured) {
        cudaFuncSetAttribute(stereo_pinhole_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        configured = smem;
    }
    dim3 grid((left->cap + ST_KPB - 1) / ST_KPB, n_frames);
    stereo_pinhole_kernel<<<grid, ST_THREADS, smem, (cudaStream_t)stream>>>(a);
    return (int)cudaGetLastError();
}
