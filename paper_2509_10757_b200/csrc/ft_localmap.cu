// ft_localmap.cu -- update_local_map on a device-resident world (SURVEY
// 8(f)-4; reference localmap.py:42-76).
//
// The reference gathers a frame's local map on the host with Python sets:
// seeds = the frame's slotted point ids; keyframes = every keyframe that
// observes a seed (through each point's (keyframe, slot) observations); then
// every point those keyframes observe, sorted ascending.  On the cfg4
// sequences that host stage costs 6-19 ms per frame -- more than all the GPU
// stages together -- so it moves to the device.  A point's observations are
// exactly the keyframes whose observed-id list holds it (mapping.py:262-266
// builds them from KeyFrame.point_ids), so the keyframe set is "every
// keyframe with a seed in its list" and no reverse index is needed.
//
// One block (1024 threads), bitmaps in shared memory:
//   seed bits  <- the frame's slots                       (atomicOr)
//   kf flags   <- warp per keyframe: any seed bit in its list (vote)
//   local bits <- warp per flagged keyframe: OR in its list
//   compaction: ascending point ids (word popcounts, block scan) + their
//               table slots; ascending keyframe indices.
// Bit sets make the result order-independent (the reference's set
// semantics), and the compaction emits ids in ascending order (its
// sorted()).
#include <cuda_runtime.h>

#include "ft_common.cuh"

namespace ft {

constexpr int LM_THREADS = 1024;
constexpr int LM_WARPS = LM_THREADS / 32;

struct LmArgs {
    const int64_t *slots;
    int32_t n_slots;
    const int32_t *kf_obs;
    const int64_t *kf_off;
    int32_t n_kf;
    const int32_t *id_slot;
    int64_t id_cap;  // point ids in [0, id_cap)
    int32_t *kf_out;
    int64_t *point_out;
    int32_t *slot_out;
    int32_t *counts;  // [0] keyframes, [1] points, [2] status (0 / bad id seen)
};

// exclusive scan of one value per thread over the block
__device__ int lm_block_scan(int x, int *tmp, int &total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int incl = x;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int y = __shfl_up_sync(FULL, incl, d);
        if (lane >= d) incl += y;
    }
    if (lane == 31) tmp[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        int w = lane < LM_WARPS ? tmp[lane] : 0;
        int wi = w;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int y = __shfl_up_sync(FULL, wi, d);
            if (lane >= d) wi += y;
        }
        if (lane < LM_WARPS) tmp[32 + lane] = wi - w;
        if (lane == 31) tmp[64] = wi;
    }
    __syncthreads();
    total = tmp[64];
    const int r = tmp[32 + wid] + incl - x;
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(LM_THREADS) update_local_map_kernel(const LmArgs a) {
    extern __shared__ __align__(16) uint32_t lm_smem[];
    const int words = (int)((a.id_cap + 31) >> 5);
    uint32_t *seed = lm_smem;                     // [words]
    uint32_t *local = seed + words;               // [words]
    uint32_t *kfl = local + words;                // [(n_kf + 31) / 32] keyframe flags
    const int kwords = (a.n_kf + 31) >> 5;
    int *tmp = reinterpret_cast<int *>(kfl + kwords);  // [65] scan scratch
    __shared__ int s_bad;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int w = threadIdx.x; w < 2 * words + kwords; w += LM_THREADS) seed[w] = 0u;
    if (threadIdx.x == 0) s_bad = 0;
    __syncthreads();
    // seeds: the frame's slotted ids (Frame.slotted_point_ids, mapping.py:120-123)
    for (int i = threadIdx.x; i < a.n_slots; i += LM_THREADS) {
        const int64_t v = a.slots[i];
        if (v == -1) continue;
        if (v < 0 || v >= a.id_cap) {  // not a point of this world (reference: KeyError)
            s_bad = 1;
            continue;
        }
        atomicOr(seed + (v >> 5), 1u << (v & 31));
    }
    __syncthreads();
    // keyframes observing any seed (localmap.py:57-60)
    for (int k = wid; k < a.n_kf; k += LM_WARPS) {
        const int64_t b = a.kf_off[k], e = a.kf_off[k + 1];
        bool hit = false;
        for (int64_t j = b + lane; j < e && !hit; j += 32) {
            const int p = a.kf_obs[j];
            hit = (seed[p >> 5] >> (p & 31)) & 1u;
        }
        if (__any_sync(FULL, hit) && lane == 0) atomicOr(kfl + (k >> 5), 1u << (k & 31));
    }
    __syncthreads();
    // every point those keyframes observe (localmap.py:61-65)
    for (int k = wid; k < a.n_kf; k += LM_WARPS) {
        if (!((kfl[k >> 5] >> (k & 31)) & 1u)) continue;
        const int64_t b = a.kf_off[k], e = a.kf_off[k + 1];
        for (int64_t j = b + lane; j < e; j += 32) {
            const int p = a.kf_obs[j];
            atomicOr(local + (p >> 5), 1u << (p & 31));
        }
    }
    __syncthreads();
    // ascending point ids (sorted(point_ids), localmap.py:66) + table slots:
    // thread t owns a contiguous run of bitmap words
    const int per = (words + LM_THREADS - 1) / LM_THREADS;
    const int w0 = threadIdx.x * per, w1 = min(words, w0 + per);
    int cnt = 0;
    for (int w = w0; w < w1; ++w) cnt += __popc(local[w]);
    int total;
    int pos = lm_block_scan(cnt, tmp, total);
    for (int w = w0; w < w1; ++w) {
        uint32_t bits = local[w];
        while (bits) {
            const int b = __ffs(bits) - 1;
            bits &= bits - 1;
            const int64_t id = ((int64_t)w << 5) + b;
            a.point_out[pos] = id;
            if (a.slot_out) a.slot_out[pos] = a.id_slot[id];
            ++pos;
        }
    }
    // ascending keyframe indices (tuple(sorted(kf_ids)), localmap.py:76)
    const int kper = (kwords + LM_THREADS - 1) / LM_THREADS;
    const int k0 = threadIdx.x * kper, k1 = min(kwords, k0 + kper);
    int kc = 0;
    for (int w = k0; w < k1; ++w) kc += __popc(kfl[w]);
    int ktotal;
    int kpos = lm_block_scan(kc, tmp, ktotal);
    for (int w = k0; w < k1; ++w) {
        uint32_t bits = kfl[w];
        while (bits) {
            const int b = __ffs(bits) - 1;
            bits &= bits - 1;
            a.kf_out[kpos++] = (w << 5) + b;
        }
    }
    if (threadIdx.x == 0) {
        a.counts[0] = ktotal;
        a.counts[1] = total;
        a.counts[2] = s_bad;
    }
}

}  // namespace ft

using namespace ft;

extern "C" int ft_update_local_map(const int64_t *slots, int32_t n_slots, const int32_t *kf_obs,
                                   const int64_t *kf_off, int32_t n_kf, const int32_t *id_slot,
                                   int64_t id_cap, int32_t *kf_out, int64_t *point_out,
                                   int32_t *slot_out, int32_t *counts, ft_stream_t stream) {
    if (!counts || !kf_out || !point_out || (n_slots > 0 && !slots) ||
        (n_kf > 0 && (!kf_obs || !kf_off)) || (slot_out && !id_slot))
        return FT_E_NULL;
    if (n_slots < 0 || n_kf < 0 || id_cap < 0) return FT_E_RANGE;
    const size_t words = (size_t)((id_cap + 31) >> 5), kwords = (size_t)((n_kf + 31) >> 5);
    const size_t smem = 4 * (2 * words + kwords + 65);
    if (smem > 227 * 1024) return FT_E_RANGE;  // > ~0.9M point ids: not supported
    LmArgs a;
    a.slots = slots;
    a.n_slots = n_slots;
    a.kf_obs = kf_obs;
    a.kf_off = kf_off;
    a.n_kf = n_kf;
    a.id_slot = id_slot;
    a.id_cap = id_cap;
    a.kf_out = kf_out;
    a.point_out = point_out;
    a.slot_out = slot_out;
    a.counts = counts;
    if (smem > 48 * 1024) {
        const cudaError_t e = cudaFuncSetAttribute(update_local_map_kernel,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   (int)smem);
        if (e != cudaSuccess) return (int)e;
    }
    update_local_map_kernel<<<1, LM_THREADS, smem, (cudaStream_t)stream>>>(a);
    return (int)cudaGetLastError();
}
