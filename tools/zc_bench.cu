// Microbenchmark: GPU-initiated reads of pinned host memory (zero-copy) vs
// DMA memcpy, for the e2e input-staging design decision.  Debug tool.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>

__global__ void zc_copy(const uint4 *__restrict__ src, uint4 *__restrict__ dst, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

__global__ void zc_write(uint4 *__restrict__ host_dst, const uint4 *__restrict__ src, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        host_dst[i] = src[i];
}

__global__ void tma_from_host(const void *src, unsigned bytes, int *ok) {
    __shared__ __align__(16) unsigned char buf[16384];
    __shared__ __align__(8) unsigned long long bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(&bar)), "r"(bytes));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"((unsigned)__cvta_generic_to_shared(buf)), "l"(src), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(&bar)) : "memory");
        asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" ::"r"((unsigned)__cvta_generic_to_shared(&bar)) : "memory");
        *ok = buf[0] + buf[bytes - 1];
    }
}

int main() {
    cudaFree(0);
    cudaStream_t s; cudaStreamCreate(&s);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (double mb : {0.07, 0.25, 0.75, 1.5, 3.0}) {
        size_t n = (size_t)(mb * (1 << 20)) / 16 * 16;
        void *h; cudaHostAlloc(&h, n, cudaHostAllocMapped);
        memset(h, 1, n);
        void *d; cudaMalloc(&d, n);
        auto timeit = [&](auto fn) {
            std::vector<float> t;
            for (int it = 0; it < 25; ++it) {
                cudaEventRecord(a, s); fn(); cudaEventRecord(b, s); cudaEventSynchronize(b);
                float ms; cudaEventElapsedTime(&ms, a, b); t.push_back(ms * 1000);
            }
            std::sort(t.begin(), t.end()); return t[t.size() / 2];
        };
        float t_dma = timeit([&] { cudaMemcpyAsync(d, h, n, cudaMemcpyHostToDevice, s); });
        float t_d2h = timeit([&] { cudaMemcpyAsync(h, d, n, cudaMemcpyDeviceToHost, s); });
        float t_zc = timeit([&] { zc_copy<<<592, 256, 0, s>>>((const uint4 *)h, (uint4 *)d, n / 16); });
        float t_zw = timeit([&] { zc_write<<<592, 256, 0, s>>>((uint4 *)h, (const uint4 *)d, n / 16); });
        float t_k = timeit([&] { zc_copy<<<592, 256, 0, s>>>((const uint4 *)d, (uint4 *)d, 0); });
        printf("%5.2f MB: H2D dma %7.1f us | D2H dma %7.1f us | zero-copy read kernel %7.1f us | zero-copy write kernel %7.1f us | empty kernel %5.1f us\n",
               mb, t_dma, t_d2h, t_zc, t_zw, t_k);
        cudaFreeHost(h); cudaFree(d);
    }
    void *h; cudaHostAlloc(&h, 16384, cudaHostAllocMapped); memset(h, 3, 16384);
    int *ok; cudaMallocManaged(&ok, 4);
    tma_from_host<<<1, 32, 0, s>>>(h, 16384, ok);
    cudaError_t e = cudaStreamSynchronize(s);
    printf("TMA bulk copy from pinned host memory: %s (value %d, expect 6)\n", cudaGetErrorString(e), e == cudaSuccess ? *ok : -1);
    return 0;
}
