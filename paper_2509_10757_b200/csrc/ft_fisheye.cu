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
#include "ft_common.cuh"
#include "ft_ws.cuh"

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
};

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
    if (tile_live && j0 < j1) {
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
    if (!tile_live) return;  // whole tile beyond the frame's keypoints
    if (k < n_left)
        a.partials[((int64_t)f * a.splits + split) * a.L.cap + k] = make_uint2(b.key, b.second);
    const int tiles = gridDim.x;
    if (!last_block_ticket(a.counters + (int64_t)f * tiles + tile, a.splits, &flag)) return;
    if (k >= n_left) return;
    Best2 m;
    best2_init(m);
    for (int s = 0; s < a.splits; ++s) {
        const uint2 p = __ldcg(a.partials + ((int64_t)f * a.splits + s) * a.L.cap + k);
        best2_merge(m, p.x, p.y);
    }
    const int64_t lk = lbase + k;
    if (ratio_accept(m, a.t_match, a.ratio)) {
        a.out_idx[lk] = m.key & 0xffffu;
        a.out_dist[lk] = m.key >> 16;
    } else {
        a.out_idx[lk] = -1;
        a.out_dist[lk] = key_dist(m.key);
    }
}

}  // namespace ft

using namespace ft;

extern "C" int ft_stereo_fisheye_bf(int32_t n_frames, const ft_keypoints *left,
                                    const ft_keypoints *right, int32_t t_match, double ratio,
                                    int64_t *out_idx, int64_t *out_dist, const ft_workspace *ws,
                                    ft_stream_t stream) {
    if (!left || !right || !out_idx || !out_dist || !ws || !left->rec || !right->rec)
        return FT_E_NULL;
    if (n_frames < 1 || left->cap < 1 || right->cap < 1 || left->cap > 65535 ||
        right->cap > 65535)
        return FT_E_RANGE;
    const int wst = ws_check(ws, n_frames, left->cap > right->cap ? left->cap : right->cap, 1);
    if (wst != FT_OK) return wst;
    BfArgs a;
    a.L = *left;
    a.R = *right;
    a.t_match = t_match;
    a.ratio = ratio;
    a.out_idx = out_idx;
    a.out_dist = out_dist;
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
    dim3 grid(tiles, a.splits, n_frames);
    fisheye_bf_kernel<<<grid, BF_TL, 0, (cudaStream_t)stream>>>(a);
    return (int)cudaGetLastError();
}
