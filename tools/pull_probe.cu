// Pull-mode probe: GPU-initiated copies of a 448 KB step from pinned host
// memory into device memory, 142 blocks x 512 threads, by load flavour
// (plain / .cv / .volatile / .nc / relaxed.sys) and host allocation flags;
// back-to-back launches timed with events.  Debug tool.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

template <int MODE>
__device__ __forceinline__ uint4 ldh(const uint4 *p) {
    uint4 v;
    if (MODE == 0) v = *p;
    if (MODE == 1) asm volatile("ld.global.cv.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    if (MODE == 2) asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    if (MODE == 3) asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    if (MODE == 4) asm volatile("ld.relaxed.sys.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    if (MODE == 5) asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}

template <int MODE>
__global__ void pull(const uint4 *src, uint4 *dst, unsigned long long nv) {
    const unsigned long long per = (nv + gridDim.x - 1) / gridDim.x;
    const unsigned long long v0 = per * blockIdx.x, v1 = min(nv, v0 + per);
    for (unsigned long long t = v0 + threadIdx.x; t < v1; t += 4 * blockDim.x) {
        uint4 x[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (t + u * blockDim.x < v1) x[u] = ldh<MODE>(src + t + u * blockDim.x);
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (t + u * blockDim.x < v1) dst[t + u * blockDim.x] = x[u];
    }
}

template <int MODE>
float run(const void *h, void *d, size_t bytes, int grid, cudaStream_t s) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int w = 0; w < 5; ++w) pull<MODE><<<grid, 512, 0, s>>>((const uint4 *)h, (uint4 *)d, bytes / 16);
    const int N = 200;
    cudaEventRecord(a, s);
    for (int it = 0; it < N; ++it)
        pull<MODE><<<grid, 512, 0, s>>>((const uint4 *)((const char *)h + (it % 4) * bytes), (uint4 *)d, bytes / 16);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms * 1000 / N;
}

int main() {
    const size_t bytes = 458752;
    void *d;
    cudaMalloc(&d, bytes);
    cudaStream_t s;
    cudaStreamCreate(&s);
    // empty-launch cost
    float t0 = run<0>(nullptr, d, 0, 142, s);
    printf("empty launch: %.2f us\n", t0);
    for (int flags : {(int)cudaHostAllocDefault, (int)cudaHostAllocMapped,
                      (int)(cudaHostAllocMapped | cudaHostAllocWriteCombined)}) {
        void *h;
        cudaHostAlloc(&h, 4 * bytes, flags);
        memset(h, 1, 4 * bytes);
        for (int grid : {2, 4, 6, 8, 12, 18, 36, 142}) {
            printf("flags %d grid %3d: plain %.2f  cv %.2f  volatile %.2f  nc %.2f  relaxed.sys %.2f  cg %.2f us/step\n",
                   flags, grid, run<0>(h, d, bytes, grid, s), run<1>(h, d, bytes, grid, s),
                   run<2>(h, d, bytes, grid, s), run<3>(h, d, bytes, grid, s),
                   run<4>(h, d, bytes, grid, s), run<5>(h, d, bytes, grid, s));
        }
        cudaFreeHost(h);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
