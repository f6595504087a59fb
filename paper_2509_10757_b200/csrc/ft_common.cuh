// ft_common.cuh -- shared device helpers for the sm_100a tracking kernels.
//
// Numerics: these translation units are compiled with -fmad=false so every
// double expression rounds exactly like the numba reference (no FMA
// contraction; numba leaves fastmath off, reference kernels.py:1-7).  Keep the
// reference's left-to-right evaluation order when editing fp64 expressions.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/fasttrack_b200.h"

#define FT_DEV __device__ __forceinline__

namespace ft {

constexpr unsigned FULL = 0xffffffffu;

// 256-bit descriptor held in registers as 8 x u32 (two 16-B loads).
struct Desc {
    uint4 lo, hi;
};

FT_DEV Desc load_desc(const uint64_t *base, int64_t row) {
    const uint4 *p = reinterpret_cast<const uint4 *>(base + 4 * row);
    Desc d;
    d.lo = __ldg(p);
    d.hi = __ldg(p + 1);
    return d;
}

// reference kernels.py:31-45 (_popcount64 x 4): XOR + POPC over 8 words.
FT_DEV uint32_t hamming(const Desc &a, const Desc &b) {
    return __popc(a.lo.x ^ b.lo.x) + __popc(a.lo.y ^ b.lo.y) + __popc(a.lo.z ^ b.lo.z) +
           __popc(a.lo.w ^ b.lo.w) + __popc(a.hi.x ^ b.hi.x) + __popc(a.hi.y ^ b.hi.y) +
           __popc(a.hi.z ^ b.hi.z) + __popc(a.hi.w ^ b.hi.w);
}

FT_DEV unsigned long long ld_acquire_u64(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Barrier among the G co-resident blocks sharing `ctr2` (cooperative
// launches only).  Two counter words used alternately (`parity`, a per-block
// count of barriers passed, identical in every block of the group); each is
// (generation << 32) | arrivals.  A block arrives with one atomic add and
// leaves as soon as it reads arrivals == G -- one L2 round trip after the
// last arrival, with no release write on the critical path.  The last
// arrival then resets its word (arrivals 0, generation + 1; a late poller
// accepts the new generation too).  The word is reused two barriers later,
// which no block reaches before the last arrival of the barrier in between --
// ordered after this reset by its release fence -- so arrivals never see a
// stale count.  Every word returns to arrivals == 0 after each barrier:
// launches of any G may reuse the pair, starting at parity 0, and nothing
// has to be reset between launches or graph replays.  Writes before the
// barrier are visible after it (release fence + acquire polls).
__device__ inline void group_barrier(unsigned long long *ctr2, int G, unsigned &parity) {
    unsigned long long *ctr = ctr2 + (parity & 1u);
    ++parity;
    __syncthreads();
    if (threadIdx.x == 0) {
        // acq_rel fences (not the sequentially consistent __threadfence): the
        // bar.sync above makes the block's writes visible to thread 0, the
        // release side publishes them with the arrival, the acquire side
        // orders the block's later reads after every other block's arrival
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        const unsigned long long old = atomicAdd(ctr, 1ull);
        if ((uint32_t)old == (uint32_t)(G - 1)) {
            atomicAdd(ctr, (1ull << 32) - (unsigned long long)G);
        } else {
            const uint32_t gen = (uint32_t)(old >> 32);
            for (;;) {
                const unsigned long long cur = ld_acquire_u64(ctr);
                if ((uint32_t)cur == (uint32_t)G || (uint32_t)(cur >> 32) != gen) break;
                __nanosleep(20);
            }
        }
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    __syncthreads();
}

// numba int(round(x)) and np.round are round-half-to-even.
FT_DEV long long round_half_even(double x) { return __double2ll_rn(x); }

FT_DEV int clampi(int x, int lo, int hi) { return x < lo ? lo : (x > hi ? hi : x); }

// Best / second-best-with-multiplicity state of the ratio-tested scans
// (kernels.py:444-464 and 552-579).  key = (dist << 16) | index, so the
// unsigned minimum is the lexicographic (dist, index) minimum -- the lowest
// index among the best distances, which both reference scans produce.
// `second` is the second order statistic of the distance multiset.
constexpr uint32_t NO_KEY = 0xffffffffu;
constexpr uint32_t NO_SECOND = 100000u;  // kernels.py:446,553

struct Best2 {
    uint32_t key;
    uint32_t second;
};

FT_DEV uint32_t key_dist(uint32_t key) { return key == NO_KEY ? NO_SECOND : (key >> 16); }

FT_DEV void best2_init(Best2 &b) {
    b.key = NO_KEY;
    b.second = NO_SECOND;
}

FT_DEV void best2_push(Best2 &b, uint32_t d, uint32_t j) {
    const uint32_t k = (d << 16) | j;
    if (k < b.key) {
        b.second = min(b.second, key_dist(b.key));
        b.key = k;
    } else {
        b.second = min(b.second, d);
    }
}

// Merge two disjoint candidate multisets.
FT_DEV void best2_merge(Best2 &b, uint32_t okey, uint32_t osec) {
    const uint32_t lo = min(b.key, okey), hi = max(b.key, okey);
    b.second = min(min(b.second, osec), key_dist(hi));
    b.key = lo;
}

FT_DEV void best2_warp_reduce(Best2 &b) {
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
        const uint32_t ok = __shfl_xor_sync(FULL, b.key, s);
        const uint32_t os = __shfl_xor_sync(FULL, b.second, s);
        best2_merge(b, ok, os);
    }
}

// Reference ratio test: bj >= 0 and best <= t and float(best) <= ratio * float(second).
FT_DEV bool ratio_accept(const Best2 &b, int t_max, double ratio) {
    if (b.key == NO_KEY) return false;
    const uint32_t best = b.key >> 16;
    return (int)best <= t_max && (double)best <= ratio * (double)b.second;
}

// Block-wide exclusive scan of one int per thread.  `tmp` holds >= NT/32
// ints.  Contains __syncthreads(); call from every thread of the block.
template <int NT>
__device__ int block_exclusive_scan(int v, int *tmp, int &total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
        const int y = __shfl_up_sync(FULL, x, s);
        if (lane >= s) x += y;
    }
    if (lane == 31) tmp[wid] = x;
    __syncthreads();
    if (wid == 0) {
        int w = lane < NT / 32 ? tmp[lane] : 0;
#pragma unroll
        for (int s = 1; s < 32; s <<= 1) {
            const int y = __shfl_up_sync(FULL, w, s);
            if (lane >= s) w += y;
        }
        if (lane < NT / 32) tmp[lane] = w;
    }
    __syncthreads();
    const int base = wid > 0 ? tmp[wid - 1] : 0;
    total = tmp[NT / 32 - 1];
    __syncthreads();
    return base + x - v;
}

// Counting-sort CSR of n items over nbins bins, built by one block in shared
// memory: start[nbins + 1], cursor[nbins], items[n], binbuf[n] (bin cache).
// `cursor` must be zeroed and a __syncthreads() passed before the call
// (callers fold that into an earlier barrier).  Three block barriers: after
// counting, after the single-warp scan, after the scatter.  Order inside a
// bin is arbitrary (atomics); every consumer reduces order-independently.
// With scan_tmp (32 ints) and nbins <= NT the bin counts are scanned by the
// whole block (one bin per thread) instead of one warp walking nbins/32 bins
// per lane.
template <int NT, typename BinFn>
__device__ void block_csr(int n, int nbins, BinFn bin_of, int *start, int *cursor,
                          uint16_t *items, uint16_t *binbuf, int *scan_tmp = nullptr) {
    for (int j = threadIdx.x; j < n; j += NT) {
        const int b = bin_of(j);
        binbuf[j] = (uint16_t)b;
        atomicAdd(&cursor[b], 1);
    }
    __syncthreads();
    if (scan_tmp && nbins <= NT) {
        const int c = threadIdx.x < nbins ? cursor[threadIdx.x] : 0;
        int total;
        const int ex = block_exclusive_scan<NT>(c, scan_tmp, total);
        if (threadIdx.x < nbins) {
            start[threadIdx.x] = ex;
            cursor[threadIdx.x] = ex;
        }
        if (threadIdx.x == 0) start[nbins] = total;
    } else if (threadIdx.x < 32) {  // one warp scans the bin counts
        const int lane = threadIdx.x;
        const int per = (nbins + 31) / 32, b0 = lane * per;
        int local = 0;
        for (int i = 0; i < per; ++i)
            if (b0 + i < nbins) local += cursor[b0 + i];
        int incl = local;
#pragma unroll
        for (int s = 1; s < 32; s <<= 1) {
            const int y = __shfl_up_sync(FULL, incl, s);
            if (lane >= s) incl += y;
        }
        int run = incl - local;
        for (int i = 0; i < per; ++i)
            if (b0 + i < nbins) {
                const int c = cursor[b0 + i];
                start[b0 + i] = run;
                cursor[b0 + i] = run;
                run += c;
            }
        if (lane == 31) start[nbins] = incl;
    }
    __syncthreads();
    for (int j = threadIdx.x; j < n; j += NT) {
        const int pos = atomicAdd(&cursor[binbuf[j]], 1);
        items[pos] = (uint16_t)j;
    }
    __syncthreads();
}

// "Last block done": true in exactly one block of the group, after every
// block has passed here with its global writes fenced.  The winner resets the
// counter for the next launch.
__device__ inline bool last_block_ticket(unsigned *counter, unsigned n_blocks, int *smem_flag) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned t = atomicAdd(counter, 1u);
        *smem_flag = (t == n_blocks - 1);
        if (t == n_blocks - 1) *counter = 0;
    }
    __syncthreads();
    const bool last = *smem_flag != 0;
    if (last) __threadfence();
    return last;
}

}  // namespace ft

// ---------------------------------------------------------------------------
// TMA bulk copies (cp.async.bulk, global -> shared) completed on an mbarrier.
// Sizes and addresses must be multiples of 16 bytes.

namespace ft {

FT_DEV unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

// Explicit shared-space accesses at 32-bit addresses, for buffers whose
// pointers reach a loop through a struct (the compiler then emits generic
// 64-bit LD / ST, which are slower and carry 64-bit address arithmetic).
// volatile: kept in order with the cp.async waits and warp barriers.
FT_DEV int lds_u8(unsigned a) {
    unsigned v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
    return (int)v;
}
FT_DEV int lds_s32(unsigned a) {
    int v;
    asm volatile("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
FT_DEV int lds_u16(unsigned a) {
    unsigned short v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
    return (int)v;
}
FT_DEV double lds_f64(unsigned a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
FT_DEV uint4 lds_v4(unsigned a) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(a));
    return v;
}
FT_DEV void sts_s32(unsigned a, int v) {
    asm volatile("st.shared.s32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

FT_DEV void mbar_init(unsigned long long *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}

FT_DEV void mbar_arrive_expect_tx(unsigned long long *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

FT_DEV void mbar_wait(unsigned long long *bar, unsigned phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

// Order earlier generic-proxy shared-memory accesses before later async
// (TMA) writes into the same buffers.
FT_DEV void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

FT_DEV void bulk_g2s(void *dst, const void *src, unsigned bytes, unsigned long long *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

FT_DEV unsigned round16(unsigned b) { return (b + 15u) & ~15u; }

}  // namespace ft
