// ft_fisheye.cu -- fisheye stereo brute-force matching on sm_100a: all-pairs
// 256-bit Hamming with best / second-best-with-multiplicity and the ratio
// test (reference kernels.py:434-464 bruteforce_match_kernel, launched by
// stereo.py:238-244 match_fisheye).
//
// Mapping (POPC-pipe bound: 8 POPC + 8 LOP3 per pair):
//   grid = (left tiles of BF_TL, right splits S, frames), block = BF_TL threads,
//   one left descriptor per thread in registers.  The block streams its right
//   split through shared memory in chunks of BF_CHUNK descriptors; every lane
//   of a warp reads the same descriptor (broadcast LDS.128).  Each (tile,
//   split) block writes its partial (key, second) state; the last block of a
//   tile (atomic ticket) merges the S partials in split order -- the merge is
//   associative and commutative, so the result is the reference's
//   ascending-j scan -- and applies the ratio test.  On rejection dist = best
//   (kernels.py:462-464).
#include <cooperative_groups.h>

#include <cstdlib>
#include <cstring>

#include "ft_common.cuh"
#include "ft_ws.cuh"

namespace cg = cooperative_groups;

namespace ft {

constexpr int BF_TL = 128;
constexpr int BF_CHUNK = 256;

struct BfArgs {
    ft_keypoints L, R;
    int32_t t_match;
    double ratio;
    int64_t *out_idx;
    int64_t *out_dist;
    uint2 *partials;     // [F][S][cap_left]
    unsigned *counters;  // [F][tiles]
    int32_t splits;
    int32_t split_len;   // right descriptors per split (of cap)
    int32_t tri_on;      // ft_stereo_fisheye: triangulate accepted pairs
    ft_fisheye_tri tri;
    int32_t *out_ok;
    double *out_points;
};

// cameras.py:139-157 FisheyeCamera.unproject: unit ray through (u, v),
// Newton inversion of the Kannala-Brandt radial polynomial (<= 20 steps,
// stop when |step| < 1e-14), in the reference's evaluation order.
FT_DEV void kb_unproject(const ft_fisheye_tri &c, double u, double v, double r[3]) {
    const double mx = (u - c.cx) / c.fx, my = (v - c.cy) / c.fy;
    const double rd = hypot(mx, my);
    if (rd < 1e-12) {
        r[0] = 0.0;
        r[1] = 0.0;
        r[2] = 1.0;
        return;
    }
    const double half_pi = 1.5707963267948966;
    double theta = rd < half_pi ? rd : half_pi;
    for (int it = 0; it < 20; ++it) {
        const double t2 = theta * theta;
        const double f = theta * (1.0 + t2 * (c.k1 + t2 * (c.k2 + t2 * (c.k3 + t2 * c.k4)))) - rd;
        const double df =
            1.0 + t2 * (3 * c.k1 + t2 * (5 * c.k2 + t2 * (7 * c.k3 + t2 * 9 * c.k4)));
        const double step = f / df;
        theta -= step;
        if (fabs(step) < 1e-14) break;
    }
    const double s = sin(theta) / rd;
    const double x = s * mx, y = s * my, z = cos(theta);
    const double n = sqrt(x * x + y * y + z * z);
    r[0] = x / n;
    r[1] = y / n;
    r[2] = z / n;
}

FT_DEV double dot3(const double a[3], const double b[3]) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }

// stereo.py:245-268 for one accepted pair: returns true and the left-frame
// point when the pair survives the parallel / gap / depth checks.
FT_DEV bool fisheye_triangulate(const ft_fisheye_tri &c, double ul, double vl, double ur,
                                double vr, double pt[3]) {
    double da[3], rr[3], db[3];
    kb_unproject(c, ul, vl, da);
    kb_unproject(c, ur, vr, rr);
    for (int k = 0; k < 3; ++k)  // dir_r = T_lr.rotation @ ray_r
        db[k] = c.rot_lr[3 * k] * rr[0] + c.rot_lr[3 * k + 1] * rr[1] + c.rot_lr[3 * k + 2] * rr[2];
    // _closest_ray_points(0, da, trans_lr, db) (stereo.py:200-220)
    const double cx = da[1] * db[2] - da[2] * db[1], cy = da[2] * db[0] - da[0] * db[2],
                 cz = da[0] * db[1] - da[1] * db[0];
    if (sqrt(cx * cx + cy * cy + cz * cz) < 1e-9) return false;
    const double *ob = c.trans_lr;
    const double a11 = dot3(da, da), a12 = dot3(da, db), a22 = dot3(db, db);
    const double b1 = dot3(da, ob), b2 = dot3(db, ob);  // r = ob - oa = ob
    const double den = a11 * a22 - a12 * a12;
    const double s = (b1 * a22 - a12 * b2) / den;
    const double t = (c.corrected ? (a12 * b1 - a11 * b2) : (a11 * b2 - a12 * b1)) / den;
    double pa[3], pb[3];
    for (int k = 0; k < 3; ++k) {
        pa[k] = 0.0 + s * da[k];
        pb[k] = ob[k] + t * db[k];
    }
    const double gx = pa[0] - pb[0], gy = pa[1] - pb[1], gz = pa[2] - pb[2];
    const double gap = sqrt(gx * gx + gy * gy + gz * gz);
    if (gap > c.ray_gap_ceiling) return false;
    for (int k = 0; k < 3; ++k) pt[k] = (pa[k] + pb[k]) / 2.0;
    if (pt[2] <= 0) return false;
    const double zr = c.rot_rl[6] * pt[0] + c.rot_rl[7] * pt[1] + c.rot_rl[8] * pt[2] + c.trans_rl[2];
    return zr > 0;
}

__device__ void bf_finish(const BfArgs &a, const Best2 &m, int f, int k, int64_t lbase,
                          int64_t rbase);

// One (left tile, right split) block's scan: best / second over right
// descriptors [j0, j1) for its BF_TL left keypoints, right descriptors
// streamed through shared memory (broadcast LDS.128).
__device__ __forceinline__ void bf_scan(const BfArgs &a, uint4 (*rdesc)[2], int k, int n_left,
                                        int64_t lbase, int64_t rbase, int j0, int j1, Best2 &b) {
    Desc ld;
    if (k < n_left) ld = load_desc(a.L.rec[lbase + k].desc, 0);
    else ld = Desc{make_uint4(0, 0, 0, 0), make_uint4(0, 0, 0, 0)};
    for (int c0 = j0; c0 < j1; c0 += BF_CHUNK) {
        const int cn = min(BF_CHUNK, j1 - c0);
        __syncthreads();
        // descriptor = 2nd and 3rd uint4 of each 64-B record
        const uint4 *src = reinterpret_cast<const uint4 *>(a.R.rec + rbase + c0);
        for (int t = threadIdx.x; t < 2 * cn; t += BF_TL)
            (&rdesc[0][0])[t] = __ldg(src + 4 * (t >> 1) + 1 + (t & 1));
        __syncthreads();
#pragma unroll 4
        for (int jj = 0; jj < cn; ++jj) {
            Desc rd;
            rd.lo = rdesc[jj][0];
            rd.hi = rdesc[jj][1];
            best2_push(b, hamming(ld, rd), (uint32_t)(c0 + jj));
        }
    }
}

// Latency path (few frames): the right splits of a left tile form ONE thread
// block cluster; each block leaves its partial (key, second) states in its
// own shared memory and the cluster's rank-0 block merges them through
// distributed shared memory -- no global partials, no atomic ticket, no
// second L2 round trip.  gridDim.y == cluster size == splits.
__global__ void __launch_bounds__(BF_TL) fisheye_bf_cluster_kernel(const BfArgs a) {
    __shared__ uint4 rdesc[BF_CHUNK][2];
    __shared__ uint2 part[BF_TL];
    cg::cluster_group cluster = cg::this_cluster();
    const int f = blockIdx.z;
    const int tile = blockIdx.x, split = blockIdx.y;
    const int n_left = min(a.L.count[f], a.L.cap);
    const int n_right = min(a.R.count[f], a.R.cap);
    if (tile * BF_TL >= n_left) return;  // uniform across the cluster (same tile)
    const int k = tile * BF_TL + threadIdx.x;
    const int64_t lbase = (int64_t)f * a.L.cap, rbase = (int64_t)f * a.R.cap;
    const int j0 = split * a.split_len;
    const int j1 = min(n_right, j0 + a.split_len);
    Best2 b;
    best2_init(b);
    if (j0 < j1) bf_scan(a, rdesc, k, n_left, lbase, rbase, j0, j1, b);
    part[threadIdx.x] = make_uint2(b.key, b.second);
    cluster.sync();  // every block's partials visible cluster-wide
    if (cluster.block_rank() == 0 && k < n_left) {
        Best2 m;
        best2_init(m);
        const int cs = (int)cluster.num_blocks();
        for (int r = 0; r < cs; ++r) {
            const uint2 p = cluster.map_shared_rank(part, r)[threadIdx.x];
            best2_merge(m, p.x, p.y);
        }
        bf_finish(a, m, f, k, lbase, rbase);
    }
    cluster.sync();  // keep every block's shared memory alive until rank 0 is done
}

__global__ void __launch_bounds__(BF_TL) fisheye_bf_kernel(const BfArgs a) {
    __shared__ uint4 rdesc[BF_CHUNK][2];
    __shared__ int flag;
    const int f = blockIdx.z;
    const int tile = blockIdx.x, split = blockIdx.y;
    const int n_left = min(a.L.count[f], a.L.cap);
    const int n_right = min(a.R.count[f], a.R.cap);
    const int k = tile * BF_TL + threadIdx.x;
    const int64_t lbase = (int64_t)f * a.L.cap, rbase = (int64_t)f * a.R.cap;
    const int j0 = split * a.split_len;
    const int j1 = min(n_right, j0 + a.split_len);
    const bool tile_live = tile * BF_TL < n_left;

    Best2 b;
    best2_init(b);
    if (tile_live && j0 < j1) bf_scan(a, rdesc, k, n_left, lbase, rbase, j0, j1, b);
    if (!tile_live) return;  // whole tile beyond the frame's keypoints
    if (k < n_left)
        a.partials[((int64_t)f * a.splits + split) * a.L.cap + k] = make_uint2(b.key, b.second);
    const int tiles = gridDim.x;
    if (!last_block_ticket(a.counters + (int64_t)f * tiles + tile, a.splits, &flag)) return;
    if (k >= n_left) return;
    Best2 m;
    best2_init(m);
    // issue the partial loads in groups of 8 before merging (independent L2
    // round trips overlap instead of serialising on the merge chain)
    const uint2 *pp = a.partials + (int64_t)f * a.splits * a.L.cap + k;
    for (int s0 = 0; s0 < a.splits; s0 += 8) {
        uint2 p[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
            p[u] = s0 + u < a.splits ? __ldcg(pp + (int64_t)(s0 + u) * a.L.cap)
                                     : make_uint2(NO_KEY, NO_SECOND);
#pragma unroll
        for (int u = 0; u < 8; ++u) best2_merge(m, p[u].x, p[u].y);
    }
    bf_finish(a, m, f, k, lbase, rbase);
}

// Ratio test + outputs (+ triangulation) of left keypoint k from its merged
// (key, second) state (kernels.py:459-464; stereo.py:245-268).
__device__ void bf_finish(const BfArgs &a, const Best2 &m, int f, int k, int64_t lbase,
                          int64_t rbase) {
    (void)f;
    const int64_t lk = lbase + k;
    const bool acc = ratio_accept(m, a.t_match, a.ratio);
    if (acc) {
        a.out_idx[lk] = m.key & 0xffffu;
        a.out_dist[lk] = m.key >> 16;
    } else {
        a.out_idx[lk] = -1;
        a.out_dist[lk] = key_dist(m.key);
    }
    if (a.tri_on) {  // stereo.py:245-268 for the accepted pair
        double pt[3] = {0.0, 0.0, 0.0};
        bool ok = false;
        if (acc) {
            const ft_kp_record &kl = a.L.rec[lk];
            const ft_kp_record &kr = a.R.rec[rbase + (m.key & 0xffffu)];
            ok = fisheye_triangulate(a.tri, kl.u, kl.v, kr.u, kr.v, pt);
        }
        a.out_ok[lk] = ok ? 1 : 0;
        a.out_points[3 * lk] = ok ? pt[0] : 0.0;
        a.out_points[3 * lk + 1] = ok ? pt[1] : 0.0;
        a.out_points[3 * lk + 2] = ok ? pt[2] : 0.0;
    }
}

}  // namespace ft

using namespace ft;

// Cluster size of the latency path, or 0 for the split-K path: used while the
// clusters alone fill the GPU with few frames (tiles x CS x F blocks within
// ~1.5 waves), CS = 16 (non-portable) or 8, at least 32 right keypoints per
// split.
static int cluster_splits(int n_frames, int tiles, int cap_right, int only) {
    for (int cs : {16, 8}) {
        if (only && cs != only) continue;
        if (cap_right < 32 * cs) continue;
        const long long blocks = (long long)tiles * cs * n_frames;
        if (blocks <= 2 * 148) return cs;
    }
    return 0;
}

static int fisheye_launch(int32_t n_frames, const ft_keypoints *left, const ft_keypoints *right,
                          int32_t t_match, double ratio, const ft_fisheye_tri *tri,
                          int64_t *out_idx, int64_t *out_dist, int32_t *out_ok,
                          double *out_points, const ft_workspace *ws, ft_stream_t stream) {
    if (!left || !right || !out_idx || !out_dist || !ws || !left->rec || !right->rec)
        return FT_E_NULL;
    if (tri && (!out_ok || !out_points)) return FT_E_NULL;
    if (n_frames < 1 || left->cap < 1 || right->cap < 1 || left->cap > 65535 ||
        right->cap > 65535)
        return FT_E_RANGE;
    const int wst = ws_check(ws, n_frames, left->cap > right->cap ? left->cap : right->cap, 1);
    if (wst != FT_OK) return wst;
    BfArgs a;
    memset(&a, 0, sizeof(a));
    a.L = *left;
    a.R = *right;
    a.t_match = t_match;
    a.ratio = ratio;
    a.out_idx = out_idx;
    a.out_dist = out_dist;
    a.tri_on = tri != nullptr;
    if (tri) a.tri = *tri;
    a.out_ok = out_ok;
    a.out_points = out_points;
    const int tiles = (left->cap + BF_TL - 1) / BF_TL;
    const WsLayout wl = ws_layout(ws);
    int splits = fisheye_splits(n_frames, left->cap, right->cap);
    const size_t fit = wl.fisheye_partial_entries / ((size_t)n_frames * left->cap);
    if ((size_t)splits > fit) splits = (int)fit;
    if (splits < 1) return FT_E_WORKSPACE;
    a.splits = splits;
    a.split_len = (right->cap + a.splits - 1) / a.splits;
    a.counters = ws_ptr<unsigned>(ws, wl.fisheye_counters);
    a.partials = ws_ptr<uint2>(ws, wl.fisheye_partials);
    // Opt-in (FT_FISHEYE_CLUSTER=8 or 16): one cluster of CS right splits per
    // left tile, merged through DSMEM.  Measured slower than the split-K path
    // at 1-2 frames (r2u: 15.8 vs 14.4 us at 1 frame, 22.7 vs 19.4 at 2, equal
    // at 4), so the split-K path is the default.
    static const char *ce = getenv("FT_FISHEYE_CLUSTER");
    const int cs = ce ? cluster_splits(n_frames, tiles, right->cap, atoi(ce)) : 0;
    if (cs > 0) {
        static bool attr_done = false;
        if (!attr_done) {
            const cudaError_t e = cudaFuncSetAttribute(
                fisheye_bf_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
            if (e != cudaSuccess) return (int)e;
            attr_done = true;
        }
        a.splits = cs;
        a.split_len = (right->cap + cs - 1) / cs;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(tiles, cs, n_frames);
        cfg.blockDim = dim3(BF_TL);
        cfg.stream = (cudaStream_t)stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 1;
        attr[0].val.clusterDim.y = cs;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        return (int)cudaLaunchKernelEx(&cfg, fisheye_bf_cluster_kernel, a);
    }
    dim3 grid(tiles, a.splits, n_frames);
    fisheye_bf_kernel<<<grid, BF_TL, 0, (cudaStream_t)stream>>>(a);
    return (int)cudaGetLastError();
}

extern "C" int ft_stereo_fisheye_bf(int32_t n_frames, const ft_keypoints *left,
                                    const ft_keypoints *right, int32_t t_match, double ratio,
                                    int64_t *out_idx, int64_t *out_dist, const ft_workspace *ws,
                                    ft_stream_t stream) {
    return fisheye_launch(n_frames, left, right, t_match, ratio, nullptr, out_idx, out_dist,
                          nullptr, nullptr, ws, stream);
}

extern "C" int ft_stereo_fisheye(int32_t n_frames, const ft_keypoints *left,
                                 const ft_keypoints *right, int32_t t_match, double ratio,
                                 const ft_fisheye_tri *tri, int64_t *out_idx, int64_t *out_dist,
                                 int32_t *out_ok, double *out_points, const ft_workspace *ws,
                                 ft_stream_t stream) {
    if (!tri) return FT_E_NULL;
    if (!(tri->fx != 0.0 && tri->fy != 0.0)) return FT_E_CONFIG;
    return fisheye_launch(n_frames, left, right, t_match, ratio, tri, out_idx, out_dist, out_ok,
                          out_points, ws, stream);
}
