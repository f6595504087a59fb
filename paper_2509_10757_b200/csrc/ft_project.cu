// ft_project.cu -- search by projection / SearchLocalPoints on sm_100a.
//
// Reference semantics (trackfront):
//   phase A   kernels.py:470-579 project_search_kernel, projection.py:118-158
//   grid      mapping.py:68-100 FrameGrid (48-px cells, truncation + clip)
//   phase B   projection.py:161-178 resolve_conflicts (lowest dist, then
//             lowest point index; output sorted by point index)
//   phase C   projection.py:181-200 rotation_consistency_filter
//   local     localmap.py:79-122 search_local_points (skip already-slotted
//             ids, write a slot only if empty, return the filled count)
//
// Mapping:
//   grid = (ceil(cap_points / PPB), n_frames), block = 256 threads.
//   Every block rebuilds the frame's keypoint grid (CSR over cells) in shared
//   memory and, for SKIP_SLOTS, a hash set of the frame's slotted point ids.
//   Thread-per-point projection/visibility (fp64, reference evaluation order)
//   pushes visible points into a shared queue; warps then take queued points
//   and stride the candidate keypoints of the window's cell rows (each cell
//   row is one contiguous CSR range), merging (best key, second) with
//   shuffles.  Accepted points claim their keypoint with a 64-bit atomicMin
//   of (dist << 32 | point) -- exactly the reference's (dist, point index)
//   winner order -- and each block writes its claimed points in point order.
//   The last block of the frame (atomic ticket) keeps the winners in point
//   order, applies the rotation histogram, writes slots, counts, and resets
//   the claims it used.
#include "ft_common.cuh"
#include "ft_ws.cuh"

namespace ft {

constexpr int PS_THREADS = 256;
constexpr int PS_WARPS = PS_THREADS / 32;
constexpr int PPB = PS_THREADS;  // map points per block
constexpr int MAX_BINS = 256;    // rotation histogram bins supported
constexpr unsigned long long NO_CLAIM = ~0ull;
constexpr long long HASH_EMPTY = (long long)0x8000000000000000ull;
constexpr long long NO_POINT_ID = -1;  // mapping.py:13 NO_POINT
constexpr int MAX_PROJ_BLOCKS = 1024;  // cap_points <= 262144

struct ProjArgs {
    ft_map_points P;
    ft_keypoints K;
    ft_project_params p;
    ft_project_io io;
    int32_t mode;
    ft_project_out o;
    unsigned long long *claims;  // [F][cap_kp]
    unsigned *counters;          // [F]
    uint2 *blk_list;             // [F][cap_points]
    int *blk_count;              // [F][n_blocks]
    int hash_bits;               // 0 = no hash
};

struct QItem {
    double ucen, v, r;
    int i;      // point index within frame
    int lvl;
    int cx0, cx1, cy0, cy1;
};

FT_DEV unsigned hash_slot(long long id, int bits) {
    return (unsigned)(((unsigned long long)id * 0x9E3779B97F4A7C15ull) >> (64 - bits));
}

FT_DEV void hash_insert(long long *tab, int bits, long long id) {
    const unsigned mask = (1u << bits) - 1u;
    unsigned h = hash_slot(id, bits);
    while (true) {
        const long long prev = (long long)atomicCAS(reinterpret_cast<unsigned long long *>(tab + h),
                                                    (unsigned long long)HASH_EMPTY,
                                                    (unsigned long long)id);
        if (prev == HASH_EMPTY || prev == id) return;
        h = (h + 1) & mask;
    }
}

FT_DEV bool hash_contains(const long long *tab, int bits, long long id) {
    const unsigned mask = (1u << bits) - 1u;
    unsigned h = hash_slot(id, bits);
    while (true) {
        const long long x = tab[h];
        if (x == id) return true;
        if (x == HASH_EMPTY) return false;
        h = (h + 1) & mask;
    }
}

// Phase-A visibility gate for one point (kernels.py:496-551).  Returns false
// when the point is not searched; else fills the window item.
FT_DEV bool project_point(const ProjArgs &a, int64_t gi, double ccx, double ccy, double ccz,
                          const double *R, const double *T, QItem &q) {
    const ft_project_params &p = a.p;
    const double px = a.P.positions[3 * gi], py = a.P.positions[3 * gi + 1],
                 pz = a.P.positions[3 * gi + 2];
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
    const double mind = a.P.min_dist[gi], maxd = a.P.max_dist[gi];
    if (dist < mind || dist > maxd) return false;
    const double vx = px - ccx, vy = py - ccy, vz = pz - ccz;
    const double cosang = (vx * a.P.normals[3 * gi] + vy * a.P.normals[3 * gi + 1] +
                           vz * a.P.normals[3 * gi + 2]) / dist;
    if (cosang < p.view_cos_min) return false;
    long long lvl = (long long)ceil(log(maxd / dist) * p.inv_log_scale - 1e-9);
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
    q.cx0 = (int)cx0;
    q.cx1 = (int)cx1;
    q.cy0 = (int)cy0;
    q.cy1 = (int)cy1;
    return true;
}

FT_DEV double py_mod(double a, double b) {  // numpy float remainder
    double r = fmod(a, b);
    if (r != 0.0 && ((b < 0.0) != (r < 0.0))) r += b;
    return r;
}

__device__ void resolve_frame(const ProjArgs &a, int f, int n_pts, int n_kp, int *scan_tmp,
                              int *misc, int *blk_prefix, int *hist) {
    const int nb = gridDim.x;
    const int64_t pbase = (int64_t)f * a.P.cap;
    const int64_t kbase = (int64_t)f * a.K.cap;
    // prefix over blocks' claimed counts
    {
        const int per = (nb + PS_THREADS - 1) / PS_THREADS;
        const int b0 = threadIdx.x * per;
        int local = 0;
        for (int i = 0; i < per; ++i)
            if (b0 + i < nb) local += __ldcg(a.blk_count + (int64_t)f * nb + b0 + i);
        int total;
        int run = block_exclusive_scan<PS_THREADS>(local, scan_tmp, total);
        for (int i = 0; i < per; ++i)
            if (b0 + i < nb) {
                blk_prefix[b0 + i] = run;
                run += __ldcg(a.blk_count + (int64_t)f * nb + b0 + i);
            }
        if (threadIdx.x == 0) {
            blk_prefix[nb] = total;
            misc[0] = total;
        }
        __syncthreads();
    }
    const int n_claimed = misc[0];
    // winners in point order
    int n_win = 0;
    for (int r0 = 0; r0 < n_claimed; r0 += PS_THREADS) {
        const int e = r0 + threadIdx.x;
        int win = 0;
        int pi = 0, kp = 0, dist = 0, oct = 0;
        if (e < n_claimed) {
            int lo = 0, hi = nb - 1;  // block b with blk_prefix[b] <= e < blk_prefix[b+1]
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (blk_prefix[mid] <= e) lo = mid;
                else hi = mid - 1;
            }
            const uint2 ent = __ldcg(a.blk_list + pbase + (int64_t)lo * PPB + (e - blk_prefix[lo]));
            pi = (int)ent.x;
            kp = (int)(ent.y & 0xffffu);
            dist = (int)((ent.y >> 16) & 0x1ffu);
            oct = (int)(ent.y >> 25);
            const unsigned long long c = __ldcg(a.claims + kbase + kp);
            win = c == (((unsigned long long)dist << 32) | (unsigned)pi);
        }
        int total;
        const int pos = n_win + block_exclusive_scan<PS_THREADS>(win, scan_tmp, total);
        if (win) {
            a.o.corr_point[pbase + pos] = pi;
            a.o.corr_kp[pbase + pos] = kp;
            a.o.corr_dist[pbase + pos] = dist;
            a.o.corr_oct[pbase + pos] = oct;
        }
        n_win += total;
    }
    __syncthreads();
    // reset every claim used in this launch (after all winner checks)
    for (int e = threadIdx.x; e < n_claimed; e += PS_THREADS) {
        int lo = 0, hi = nb - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (blk_prefix[mid] <= e) lo = mid;
            else hi = mid - 1;
        }
        const uint2 ent = __ldcg(a.blk_list + pbase + (int64_t)lo * PPB + (e - blk_prefix[lo]));
        a.claims[kbase + (ent.y & 0xffffu)] = NO_CLAIM;
    }
    int n_final = n_win;
    if ((a.mode & FT_PROJ_ROTATION) && a.io.ref_angles && a.K.angle && n_win > 0) {
        const int nbins = a.p.histogram_bins;
        const double two_pi = 2.0 * 3.141592653589793;
        for (int b = threadIdx.x; b < nbins; b += PS_THREADS) hist[b] = 0;
        __syncthreads();
        for (int c = threadIdx.x; c < n_win; c += PS_THREADS) {
            const int kp = (int)__ldcg(a.o.corr_kp + pbase + c);
            const int pi = (int)__ldcg(a.o.corr_point + pbase + c);
            const double diff = py_mod(a.K.angle[kbase + kp] - a.io.ref_angles[pbase + pi], two_pi);
            long long bin = (long long)floor(diff / two_pi * (double)nbins);
            bin = bin < 0 ? 0 : (bin > nbins - 1 ? nbins - 1 : bin);
            atomicAdd(&hist[bin], 1);
        }
        __syncthreads();
        if (threadIdx.x == 0) {  // top-K bins by (-count, bin)
            int keep_mask_words[MAX_BINS / 32] = {0};
            for (int t = 0; t < a.p.histogram_keep && t < nbins; ++t) {
                int sel = -1;
                for (int b = 0; b < nbins; ++b) {
                    if (keep_mask_words[b >> 5] & (1 << (b & 31))) continue;
                    if (sel < 0 || hist[b] > hist[sel]) sel = b;
                }
                if (sel >= 0) keep_mask_words[sel >> 5] |= 1 << (sel & 31);
            }
            for (int w = 0; w < MAX_BINS / 32; ++w) misc[4 + w] = keep_mask_words[w];
        }
        __syncthreads();
        n_final = 0;
        for (int r0 = 0; r0 < n_win; r0 += PS_THREADS) {
            const int c = r0 + threadIdx.x;
            int keep = 0;
            long long pi = 0, kp = 0, dist = 0, oct = 0;
            if (c < n_win) {
                pi = __ldcg(a.o.corr_point + pbase + c);
                kp = __ldcg(a.o.corr_kp + pbase + c);
                dist = __ldcg(a.o.corr_dist + pbase + c);
                oct = __ldcg(a.o.corr_oct + pbase + c);
                const double diff = py_mod(a.K.angle[kbase + kp] - a.io.ref_angles[pbase + pi], two_pi);
                long long bin = (long long)floor(diff / two_pi * (double)nbins);
                bin = bin < 0 ? 0 : (bin > nbins - 1 ? nbins - 1 : bin);
                keep = (misc[4 + (bin >> 5)] >> (bin & 31)) & 1;
            }
            int total;
            const int pos = n_final + block_exclusive_scan<PS_THREADS>(keep, scan_tmp, total);
            if (keep) {
                a.o.corr_point[pbase + pos] = pi;
                a.o.corr_kp[pbase + pos] = kp;
                a.o.corr_dist[pbase + pos] = dist;
                a.o.corr_oct[pbase + pos] = oct;
            }
            n_final += total;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0 && a.o.corr_count) a.o.corr_count[f] = n_final;
    if (a.mode & FT_PROJ_WRITE_SLOTS) {
        // localmap.py:113-121: write only slots that were empty before the
        // search; each keypoint appears at most once among the winners, so
        // the writes never race.
        if (a.io.slots_out != a.io.slots_in) {
            for (int k = threadIdx.x; k < n_kp; k += PS_THREADS)
                a.io.slots_out[kbase + k] = a.io.slots_in[kbase + k];
            __syncthreads();
        }
        for (int c = threadIdx.x; c < n_final; c += PS_THREADS) {
            const long long kp = __ldcg(a.o.corr_kp + pbase + c);
            const long long pi = __ldcg(a.o.corr_point + pbase + c);
            if (a.io.slots_in[kbase + kp] == NO_POINT_ID)
                a.io.slots_out[kbase + kp] = a.P.point_ids[pbase + pi];
        }
        __syncthreads();
        if (threadIdx.x == 0) misc[1] = 0;
        __syncthreads();
        int filled = 0;
        for (int k = threadIdx.x; k < n_kp; k += PS_THREADS)
            filled += __ldcg(a.io.slots_out + kbase + k) != NO_POINT_ID;
        atomicAdd(&misc[1], filled);
        __syncthreads();
        if (threadIdx.x == 0 && a.o.slot_count) a.o.slot_count[f] = misc[1];
    }
}

__global__ void __launch_bounds__(PS_THREADS) project_search_kernel(const ProjArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int f = blockIdx.y;
    const int n_pts = min(a.P.count[f], a.P.cap);
    const int n_kp = min(a.K.count[f], a.K.cap);
    const int p0 = blockIdx.x * PPB;
    const int64_t pbase = (int64_t)f * a.P.cap;
    const int64_t kbase = (int64_t)f * a.K.cap;
    const ft_project_params &p = a.p;
    const int ncell = p.grid_nx * p.grid_ny;

    // shared memory carve-up
    unsigned char *sp = smem_raw;
    QItem *queue = reinterpret_cast<QItem *>(sp);
    sp += sizeof(QItem) * PPB;
    long long *htab = reinterpret_cast<long long *>(sp);
    sp += a.hash_bits ? (sizeof(long long) << a.hash_bits) : 0;
    int *ip = reinterpret_cast<int *>(sp);
    int *scan_tmp = ip;
    ip += 32;
    int *misc = ip;  // [0] queue size, [1..3] scratch, [4..11] bin mask, [12] ticket
    ip += 16;
    int *res_kp = ip;
    ip += PPB;
    int *res_pack = ip;
    ip += PPB;
    int *cell_start = ip;  // [ncell + 1]
    ip += ncell + 1;
    int *cell_cursor = ip;  // [ncell]
    ip += ncell;
    int *blk_prefix = ip;  // [MAX_PROJ_BLOCKS + 1] (last block)
    ip += MAX_PROJ_BLOCKS + 1;
    int *hist = ip;  // [MAX_BINS] (last block)
    ip += MAX_BINS;
    uint16_t *items = reinterpret_cast<uint16_t *>(ip);

    const bool resolve = a.mode & FT_PROJ_RESOLVE;
    if (p0 < n_pts) {
        const double *ku = a.K.u + kbase, *kv = a.K.v + kbase;
        const double cellf = (double)p.cell_px;
        const int nx = p.grid_nx, ny = p.grid_ny;
        block_csr<PS_THREADS>(
            n_kp, ncell,
            [&](int j) {  // FrameGrid cell: truncation, then clip (mapping.py:81-83)
                long long cx = (long long)(ku[j] / cellf), cy = (long long)(kv[j] / cellf);
                cx = cx < 0 ? 0 : (cx > nx - 1 ? nx - 1 : cx);
                cy = cy < 0 ? 0 : (cy > ny - 1 ? ny - 1 : cy);
                return (int)(cy * nx + cx);
            },
            cell_start, cell_cursor, items, scan_tmp);
        const bool use_hash = (a.mode & FT_PROJ_SKIP_SLOTS) && a.hash_bits;
        if (use_hash) {
            for (int h = threadIdx.x; h < (1 << a.hash_bits); h += PS_THREADS) htab[h] = HASH_EMPTY;
            __syncthreads();
            for (int k = threadIdx.x; k < n_kp; k += PS_THREADS) {
                const long long id = a.io.slots_in[kbase + k];
                if (id != NO_POINT_ID) hash_insert(htab, a.hash_bits, id);
            }
        }
        if (threadIdx.x == 0) misc[0] = 0;
        __syncthreads();

        // thread-per-point projection + visibility
        const double *R = a.io.rot + 9 * f, *T = a.io.trans + 3 * f;
        const double ccx = -(R[0] * T[0] + R[3] * T[1] + R[6] * T[2]);
        const double ccy = -(R[1] * T[0] + R[4] * T[1] + R[7] * T[2]);
        const double ccz = -(R[2] * T[0] + R[5] * T[1] + R[8] * T[2]);
        const int i = p0 + threadIdx.x;
        res_kp[threadIdx.x] = -1;
        if (i < n_pts) {
            const int64_t gi = pbase + i;
            if (a.o.out_kp) {
                a.o.out_kp[gi] = -1;
                a.o.out_dist[gi] = 10000;
                a.o.out_oct[gi] = -1;
            }
            bool skip = a.io.skip && a.io.skip[gi] != 0;
            if (!skip && use_hash) skip = hash_contains(htab, a.hash_bits, a.P.point_ids[gi]);
            QItem q;
            if (!skip && project_point(a, gi, ccx, ccy, ccz, R, T, q)) {
                q.i = i;
                queue[atomicAdd(&misc[0], 1)] = q;
            }
        }
        __syncthreads();

        // warp per queued point: windowed candidate scan (kernels.py:552-579)
        const int nq = misc[0];
        const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
        for (int qi = wid; qi < nq; qi += PS_WARPS) {
            const QItem q = queue[qi];
            const int64_t gi = pbase + q.i;
            const Desc pd = load_desc(a.P.desc, gi);
            Best2 b;
            best2_init(b);
            for (int gy = q.cy0; gy <= q.cy1; ++gy) {
                const int beg = cell_start[gy * nx + q.cx0];
                const int end = cell_start[gy * nx + q.cx1 + 1];
                for (int ii = beg + lane; ii < end; ii += 32) {
                    const int j = items[ii];
                    const int64_t kj = kbase + j;
                    if (fabs(ku[j] - q.ucen) > q.r || fabs(kv[j] - q.v) > q.r) continue;
                    const int ko = a.K.octave[kj];
                    if (ko < q.lvl - 1 || ko > q.lvl + 1) continue;
                    best2_push(b, hamming(pd, load_desc(a.K.desc, kj)), (uint32_t)j);
                }
            }
            best2_warp_reduce(b);
            if (lane == 0 && ratio_accept(b, p.t_proj, p.ratio)) {
                const int kp = (int)(b.key & 0xffffu), d = (int)(b.key >> 16);
                if (a.o.out_kp) {
                    a.o.out_kp[gi] = kp;
                    a.o.out_dist[gi] = d;
                    a.o.out_oct[gi] = q.lvl;
                }
                res_kp[q.i - p0] = kp;
                res_pack[q.i - p0] = kp | (d << 16) | (q.lvl << 25);
                if (resolve)
                    atomicMin(a.claims + kbase + kp, ((unsigned long long)d << 32) | (unsigned)q.i);
            }
        }
        __syncthreads();
        if (resolve) {  // this block's claimed points, in point order
            const int claimed = res_kp[threadIdx.x] >= 0;
            int total;
            const int pos = block_exclusive_scan<PS_THREADS>(claimed, scan_tmp, total);
            if (claimed)
                a.blk_list[pbase + p0 + pos] =
                    make_uint2((unsigned)(p0 + threadIdx.x), (unsigned)res_pack[threadIdx.x]);
            if (threadIdx.x == 0) a.blk_count[(int64_t)f * gridDim.x + blockIdx.x] = total;
        }
    } else if (resolve && threadIdx.x == 0) {
        a.blk_count[(int64_t)f * gridDim.x + blockIdx.x] = 0;
    }
    if (!resolve) return;
    if (!last_block_ticket(a.counters + f, gridDim.x, misc + 12)) return;
    resolve_frame(a, f, n_pts, n_kp, scan_tmp, misc, blk_prefix, hist);
}

size_t project_smem_bytes(int ncell, int cap_kp, int hash_bits) {
    size_t b = sizeof(QItem) * PPB;
    b += hash_bits ? (sizeof(long long) << hash_bits) : 0;
    b += 4 * (32 + 16 + 2 * PPB);
    b += 4 * (size_t)(2 * ncell + 1 + MAX_PROJ_BLOCKS + 1 + MAX_BINS);
    b += 2 * (size_t)cap_kp + 16;
    return b;
}

}  // namespace ft

using namespace ft;

extern "C" int ft_project_search(int32_t n_frames, const ft_map_points *points,
                                 const ft_keypoints *frame, const ft_project_params *params,
                                 const ft_project_io *io, int32_t mode, const ft_project_out *out,
                                 const ft_workspace *ws, ft_stream_t stream) {
    if (!points || !frame || !params || !io || !out || !ws) return FT_E_NULL;
    if (n_frames < 1 || points->cap < 1 || frame->cap < 1 || frame->cap > 65535 ||
        points->cap > MAX_PROJ_BLOCKS * PPB)
        return FT_E_RANGE;
    if (params->n_levels < 1 || params->n_levels > FT_MAX_LEVELS || params->cell_px < 1 ||
        params->grid_nx < 1 || params->grid_ny < 1 || params->grid_nx * params->grid_ny > 65536)
        return FT_E_RANGE;
    if (params->histogram_bins < 1 || params->histogram_bins > MAX_BINS) return FT_E_CONFIG;
    if (!io->rot || !io->trans) return FT_E_NULL;
    if ((mode & (FT_PROJ_SKIP_SLOTS | FT_PROJ_WRITE_SLOTS)) && !io->slots_in) return FT_E_NULL;
    if ((mode & FT_PROJ_WRITE_SLOTS) && !io->slots_out) return FT_E_NULL;
    if ((mode & FT_PROJ_WRITE_SLOTS) && !(mode & FT_PROJ_RESOLVE)) return FT_E_CONFIG;
    if ((mode & FT_PROJ_RESOLVE) &&
        (!out->corr_point || !out->corr_kp || !out->corr_dist || !out->corr_oct))
        return FT_E_NULL;
    if (out->out_kp && (!out->out_dist || !out->out_oct)) return FT_E_NULL;
    const int wst = ws_check(ws, n_frames, frame->cap, points->cap);
    if (wst != FT_OK) return wst;

    ProjArgs a;
    a.P = *points;
    a.K = *frame;
    a.p = *params;
    a.io = *io;
    a.mode = mode;
    a.o = *out;
    const int nb = (points->cap + PPB - 1) / PPB;
    const WsLayout wl = ws_layout(ws);
    a.counters = ws_ptr<unsigned>(ws, wl.proj_counters);
    a.blk_count = ws_ptr<int>(ws, wl.proj_blk_count);
    a.claims = ws_ptr<unsigned long long>(ws, wl.proj_claims);
    a.blk_list = ws_ptr<uint2>(ws, wl.proj_blk_list);
    a.hash_bits = 0;
    if (mode & FT_PROJ_SKIP_SLOTS) {
        int bits = 1;
        while ((1 << bits) < 2 * frame->cap) ++bits;
        a.hash_bits = bits;
    }
    const int ncell = params->grid_nx * params->grid_ny;
    const size_t smem = project_smem_bytes(ncell, frame->cap, a.hash_bits);
    if (smem > 227 * 1024) return FT_E_RANGE;
    static thread_local size_t configured = 0;
    if (smem > 48 * 1024 && smem > configured) {
        cudaFuncSetAttribute(project_search_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        configured = smem;
    }
    dim3 grid(nb, n_frames);
    project_search_kernel<<<grid, PS_THREADS, smem, (cudaStream_t)stream>>>(a);
    return (int)cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Standalone phase B / phase C for callers that hold phase-A arrays
// (reference projection.py:161-178 resolve_conflicts and :181-200
// rotation_consistency_filter called on their own).  One frame.

namespace ft {

constexpr int RS_THREADS = 1024;

__global__ void claim_kernel(const int64_t *out_kp, const int64_t *out_dist, int n, int n_kp,
                             unsigned long long *claims) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const long long kp = out_kp[i];
        if (kp < 0 || kp >= n_kp) continue;
        atomicMin(claims + kp, ((unsigned long long)out_dist[i] << 32) | (unsigned)i);
    }
}

__global__ void __launch_bounds__(RS_THREADS)
compact_winners_kernel(const int64_t *out_kp, const int64_t *out_dist, const int64_t *out_oct,
                       int n, int n_kp, unsigned long long *claims, int64_t *cp, int64_t *ck,
                       int64_t *cd, int64_t *co, int32_t *count) {
    __shared__ int scan_tmp[32];
    int n_win = 0;
    for (int r0 = 0; r0 < n; r0 += RS_THREADS) {
        const int i = r0 + threadIdx.x;
        int win = 0;
        long long kp = -1;
        if (i < n) {
            kp = out_kp[i];
            if (kp >= 0 && kp < n_kp)
                win = claims[kp] == (((unsigned long long)out_dist[i] << 32) | (unsigned)i);
        }
        int total;
        const int pos = n_win + block_exclusive_scan<RS_THREADS>(win, scan_tmp, total);
        if (win) {
            cp[pos] = i;
            ck[pos] = kp;
            cd[pos] = out_dist[i];
            co[pos] = out_oct[i];
        }
        n_win += total;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += RS_THREADS) {
        const long long kp = out_kp[i];
        if (kp >= 0 && kp < n_kp) claims[kp] = NO_CLAIM;
    }
    if (threadIdx.x == 0) *count = n_win;
}

__global__ void __launch_bounds__(RS_THREADS)
rotation_filter_kernel(int64_t *cp, int64_t *ck, int64_t *cd, int64_t *co, int m,
                       const double *ref_angles, const double *kp_angles, int nbins, int keep_k,
                       int32_t *count) {
    __shared__ int scan_tmp[32];
    __shared__ int hist[MAX_BINS];
    __shared__ int keepw[MAX_BINS / 32];
    const double two_pi = 2.0 * 3.141592653589793;
    for (int b = threadIdx.x; b < nbins; b += RS_THREADS) hist[b] = 0;
    __syncthreads();
    auto bin_of = [&](int c) {
        const double diff = py_mod(kp_angles[ck[c]] - ref_angles[cp[c]], two_pi);
        long long b = (long long)floor(diff / two_pi * (double)nbins);
        return (int)(b < 0 ? 0 : (b > nbins - 1 ? nbins - 1 : b));
    };
    for (int c = threadIdx.x; c < m; c += RS_THREADS) atomicAdd(&hist[bin_of(c)], 1);
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 0; w < MAX_BINS / 32; ++w) keepw[w] = 0;
        for (int t = 0; t < keep_k && t < nbins; ++t) {
            int sel = -1;
            for (int b = 0; b < nbins; ++b) {
                if (keepw[b >> 5] & (1 << (b & 31))) continue;
                if (sel < 0 || hist[b] > hist[sel]) sel = b;
            }
            if (sel >= 0) keepw[sel >> 5] |= 1 << (sel & 31);
        }
    }
    __syncthreads();
    int n_keep = 0;
    for (int r0 = 0; r0 < m; r0 += RS_THREADS) {
        const int c = r0 + threadIdx.x;
        int keep = 0;
        long long p = 0, k = 0, d = 0, o = 0;
        if (c < m) {
            const int b = bin_of(c);
            keep = (keepw[b >> 5] >> (b & 31)) & 1;
            p = cp[c];
            k = ck[c];
            d = cd[c];
            o = co[c];
        }
        int total;
        const int pos = n_keep + block_exclusive_scan<RS_THREADS>(keep, scan_tmp, total);
        if (keep) {
            cp[pos] = p;
            ck[pos] = k;
            cd[pos] = d;
            co[pos] = o;
        }
        n_keep += total;
    }
    if (threadIdx.x == 0) *count = n_keep;
}

}  // namespace ft

extern "C" int ft_resolve_conflicts(int32_t n_points, const int64_t *out_kp,
                                    const int64_t *out_dist, const int64_t *out_oct, int32_t n_kp,
                                    const ft_project_out *out, const ft_workspace *ws,
                                    ft_stream_t stream) {
    if (!out || !ws || !out->corr_count) return FT_E_NULL;
    if (n_points < 0 || n_kp < 0 || n_kp > 65535) return FT_E_RANGE;
    if (n_points > 0 && (!out_kp || !out_dist || !out_oct || !out->corr_point || !out->corr_kp ||
                         !out->corr_dist || !out->corr_oct))
        return FT_E_NULL;
    const int wst = ws_check(ws, 1, n_kp > 0 ? n_kp : 1, 1);
    if (wst != FT_OK) return wst;
    unsigned long long *claims = ws_ptr<unsigned long long>(ws, ws_layout(ws).proj_claims);
    cudaStream_t s = (cudaStream_t)stream;
    if (n_points > 0) {
        const int blocks = (n_points + 255) / 256 < 1184 ? (n_points + 255) / 256 : 1184;
        claim_kernel<<<blocks, 256, 0, s>>>(out_kp, out_dist, n_points, n_kp, claims);
    }
    compact_winners_kernel<<<1, RS_THREADS, 0, s>>>(out_kp, out_dist, out_oct, n_points, n_kp,
                                                    claims, out->corr_point, out->corr_kp,
                                                    out->corr_dist, out->corr_oct,
                                                    out->corr_count);
    return (int)cudaGetLastError();
}

extern "C" int ft_rotation_filter(int32_t m, int64_t *corr_point, int64_t *corr_kp,
                                  int64_t *corr_dist, int64_t *corr_oct, const double *ref_angles,
                                  const double *kp_angles, int32_t histogram_bins,
                                  int32_t histogram_keep, int32_t *count, ft_stream_t stream) {
    if (!count) return FT_E_NULL;
    if (m < 0) return FT_E_RANGE;
    if (histogram_bins < 1 || histogram_bins > MAX_BINS || histogram_keep < 1 ||
        histogram_keep > histogram_bins)
        return FT_E_CONFIG;
    if (m > 0 && (!corr_point || !corr_kp || !corr_dist || !corr_oct || !ref_angles || !kp_angles))
        return FT_E_NULL;
    rotation_filter_kernel<<<1, RS_THREADS, 0, (cudaStream_t)stream>>>(
        corr_point, corr_kp, corr_dist, corr_oct, m, ref_angles, kp_angles, histogram_bins,
        histogram_keep, count);
    return (int)cudaGetLastError();
}
