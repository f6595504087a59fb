// ft_misc.cu -- small C-ABI entries: the Hamming self-test kernel and the
// standalone phase B / phase C kernels for callers that hold phase-A arrays.
#include "ft_common.cuh"
#include "ft_ws.cuh"

namespace ft {

constexpr unsigned long long NO_CLAIM = ~0ull;
constexpr int MAX_BINS = 256;

FT_DEV double py_mod_m(double a, double b) {  // numpy float remainder
    double r = fmod(a, b);
    if (r != 0.0 && ((b < 0.0) != (r < 0.0))) r += b;
    return r;
}

// reference kernels.py:48-51
__global__ void hamming_pairs_kernel(const uint64_t *a, const uint64_t *b, int64_t n,
                                     int64_t *out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = hamming(load_desc(a, i), load_desc(b, i));
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
        const double diff = py_mod_m(kp_angles[ck[c]] - ref_angles[cp[c]], two_pi);
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

// ---------------------------------------------------------------------------
// SoA (reference FeatureSet / MapPointSoA layout) -> packed records.

namespace ft {

__global__ void pack_kp_kernel(int F, const double *u, const double *v, const int32_t *octave,
                               const double *angle, const uint64_t *desc, const int32_t *count,
                               int cap, ft_kp_record *out) {
    const int64_t total = (int64_t)F * cap;
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total;
         g += (int64_t)gridDim.x * blockDim.x) {
        const int f = (int)(g / cap), i = (int)(g - (int64_t)f * cap);
        if (i >= count[f]) continue;
        ft_kp_record r;
        r.u = u[g];
        r.v = v[g];
        for (int w = 0; w < 4; ++w) r.desc[w] = desc[4 * g + w];
        r.angle = angle ? angle[g] : 0.0;
        r.octave = octave[g];
        r.pad = 0;
        out[g] = r;
    }
}

__global__ void pack_pt_kernel(int F, const double *pos, const double *nrm, const double *mind,
                               const double *maxd, const uint64_t *desc, const int64_t *ids,
                               const int32_t *count, int cap, ft_point_record *out) {
    const int64_t total = (int64_t)F * cap;
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total;
         g += (int64_t)gridDim.x * blockDim.x) {
        const int f = (int)(g / cap), i = (int)(g - (int64_t)f * cap);
        if (i >= count[f]) continue;
        ft_point_record r;
        for (int w = 0; w < 4; ++w) r.desc[w] = desc[4 * g + w];
        for (int c = 0; c < 3; ++c) {
            r.pos[c] = pos[3 * g + c];
            r.nrm[c] = nrm[3 * g + c];
        }
        r.min_dist = mind[g];
        r.max_dist = maxd[g];
        r.id = ids[g];
        r.pad = 0;
        out[g] = r;
    }
}

}  // namespace ft

extern "C" int ft_pack_keypoints(int32_t n_frames, const double *u, const double *v,
                                 const int32_t *octave, const double *angle,
                                 const uint64_t *desc, const int32_t *count, int32_t cap,
                                 ft_kp_record *out, ft_stream_t stream) {
    if (!u || !v || !octave || !desc || !count || !out) return FT_E_NULL;
    if (n_frames < 1 || cap < 1) return FT_E_RANGE;
    const int64_t total = (int64_t)n_frames * cap;
    const int blocks = (int)((total + 255) / 256 < 4096 ? (total + 255) / 256 : 4096);
    pack_kp_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(n_frames, u, v, octave, angle, desc,
                                                             count, cap, out);
    return (int)cudaGetLastError();
}

extern "C" int ft_pack_points(int32_t n_frames, const double *positions, const double *normals,
                              const double *min_dist, const double *max_dist,
                              const uint64_t *desc, const int64_t *point_ids,
                              const int32_t *count, int32_t cap, ft_point_record *out,
                              ft_stream_t stream) {
    if (!positions || !normals || !min_dist || !max_dist || !desc || !point_ids || !count || !out)
        return FT_E_NULL;
    if (n_frames < 1 || cap < 1) return FT_E_RANGE;
    const int64_t total = (int64_t)n_frames * cap;
    const int blocks = (int)((total + 255) / 256 < 4096 ? (total + 255) / 256 : 4096);
    pack_pt_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(n_frames, positions, normals,
                                                             min_dist, max_dist, desc, point_ids,
                                                             count, cap, out);
    return (int)cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Device-resident map-point table (north star (1): the map stays in HBM and
// only pose + map-point deltas cross PCIe).  The reference rebuilds each
// frame's LocalMap SoA on the host (mapping.py:204-235 decompose_map_points,
// localmap.py:22-39); here the table holds every point record once, frames
// name their local map as a list of table slots (in LocalMap order), and
// ft_gather_points builds the per-frame contiguous record table the track
// kernel stages with one bulk copy.  One 16-B vector per lane: a warp moves
// 4.5 records per instruction.

namespace {
constexpr int PT_VEC = sizeof(ft_point_record) / 16;  // 7 x uint4
static_assert(sizeof(ft_point_record) % 16 == 0, "record must be uint4-sized");

__global__ void gather_pt_kernel(int32_t n_frames, const uint4 *table, int64_t table_size,
                                 const int32_t *index, const int32_t *count, int32_t cap,
                                 uint4 *out, int32_t *status) {
    const int64_t total = (int64_t)n_frames * cap * PT_VEC;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t rec = e / PT_VEC;
        const int w = (int)(e - rec * PT_VEC);
        const int f = (int)(rec / cap), i = (int)(rec - (int64_t)f * cap);
        if (i >= min(count[f], cap)) continue;
        const int32_t slot = __ldg(index + rec);
        if (slot < 0 || slot >= table_size) {  // caller error: flag it, write a dead record
            if (status) atomicExch(status, FT_E_RANGE);
            continue;
        }
        out[e] = __ldg(table + (int64_t)slot * PT_VEC + w);
    }
}

__global__ void scatter_pt_kernel(int32_t n, const uint4 *recs, const int32_t *slots,
                                  uint4 *table, int64_t table_size) {
    const int64_t total = (int64_t)n * PT_VEC;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = e / PT_VEC;
        const int32_t slot = slots[r];
        if (slot < 0 || slot >= table_size) continue;
        table[(int64_t)slot * PT_VEC + (e - r * PT_VEC)] = recs[e];
    }
}
}  // namespace

extern "C" int ft_gather_points(int32_t n_frames, const ft_point_record *table,
                                int64_t table_size, const int32_t *index, const int32_t *count,
                                int32_t cap, ft_point_record *out, int32_t *status,
                                ft_stream_t stream) {
    if (!table || !index || !count || !out) return FT_E_NULL;
    if (n_frames < 1 || cap < 1 || table_size < 1) return FT_E_RANGE;
    if ((((uintptr_t)table) | ((uintptr_t)out)) & 15) return FT_E_RANGE;
    const int64_t total = (int64_t)n_frames * cap * PT_VEC;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t want = (total + 255) / 256;
    const int blocks = (int)(want < 4 * sms ? want : 4 * sms);
    gather_pt_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(
        n_frames, reinterpret_cast<const uint4 *>(table), table_size, index, count, cap,
        reinterpret_cast<uint4 *>(out), status);
    return (int)cudaGetLastError();
}

extern "C" int ft_scatter_points(int32_t n, const ft_point_record *recs, const int32_t *slots,
                                 ft_point_record *table, int64_t table_size, ft_stream_t stream) {
    if (n == 0) return FT_OK;
    if (!recs || !slots || !table) return FT_E_NULL;
    if (n < 0 || table_size < 1) return FT_E_RANGE;
    if ((((uintptr_t)table) | ((uintptr_t)recs)) & 15) return FT_E_RANGE;
    const int64_t total = (int64_t)n * PT_VEC;
    const int blocks = (int)((total + 255) / 256 < 1024 ? (total + 255) / 256 : 1024);
    scatter_pt_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(
        n, reinterpret_cast<const uint4 *>(recs), slots, reinterpret_cast<uint4 *>(table),
        table_size);
    return (int)cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Packed-upload scatter: one contiguous H2D of a step's needed bytes (the
// small inputs plus every stream's needed pyramid levels, packed by the host
// at staging time), then this kernel places each segment at its arena offset.
// desc[3i..3i+2] = (src offset, dst offset, length) relative to `base`; the
// host packs segments with src = dst (mod 16), so the body moves as uint4.
namespace {
__global__ void copy_ranges_kernel(unsigned char *base, const int64_t *desc, int32_t n,
                                   int32_t blocks_per) {
    const int seg = blockIdx.x / blocks_per, part = blockIdx.x - seg * blocks_per;
    if (seg >= n) return;
    const int64_t so = desc[3 * seg], dof = desc[3 * seg + 1], len = desc[3 * seg + 2];
    if (len <= 0) return;
    const unsigned char *src = base + so;
    unsigned char *dst = base + dof;
    const int64_t head = min(len, (int64_t)((16 - ((uintptr_t)dst & 15)) & 15));
    const bool vec = (((uintptr_t)src ^ (uintptr_t)dst) & 15) == 0;
    const int64_t nv = vec ? (len - head) >> 4 : 0;
    const int64_t tail0 = vec ? head + (nv << 4) : 0;
    const int64_t stride = (int64_t)blocks_per * blockDim.x;
    const int64_t t0 = (int64_t)part * blockDim.x + threadIdx.x;
    if (vec) {
        for (int64_t t = t0; t < head; t += stride) dst[t] = src[t];
        const uint4 *s4 = reinterpret_cast<const uint4 *>(src + head);
        uint4 *d4 = reinterpret_cast<uint4 *>(dst + head);
        for (int64_t q = t0; q < nv; q += stride) d4[q] = __ldcs(s4 + q);
        for (int64_t t = tail0 + t0; t < len; t += stride) dst[t] = src[t];
    } else {
        for (int64_t t = t0; t < len; t += stride) dst[t] = src[t];
    }
}
}  // namespace

extern "C" int ft_copy_ranges(void *base, const int64_t *desc, int32_t n, ft_stream_t stream) {
    if (!base || (!desc && n > 0)) return FT_E_NULL;
    if (n < 0) return FT_E_RANGE;
    if (n == 0) return FT_OK;
    const int blocks_per = 4;
    copy_ranges_kernel<<<n * blocks_per, 512, 0, (cudaStream_t)stream>>>(
        static_cast<unsigned char *>(base), desc, n, blocks_per);
    return (int)cudaGetLastError();
}
