// Probe: does one strided 2D copy of m step ranges (cudaMemcpy2DAsync, host
// and device pitches = slot strides) amortise the fixed per-copy cost of the
// H2D copy engine?  Times back-to-back 448 KB ranges as m-row 2D copies,
// m = 1 (plain 1D copy), 2, 4, 8, from pinned host memory into 8 device slots.
// Build: nvcc -O2 -gencode arch=compute_100a,code=sm_100a tools/h2d2d_probe.cu -o tools/h2d2d_probe
#include <cstdio>
#include <cuda_runtime.h>

int main() {
    const size_t slot = 2600 * 1024, width = 448 * 1024, lo = 1200 * 1024;
    const int nslots = 8, steps = 4000;
    char *h, *d;
    cudaHostAlloc(&h, slot * nslots, cudaHostAllocDefault);
    cudaMalloc(&d, slot * nslots);
    for (size_t i = 0; i < slot * nslots; i += 4096) h[i] = (char)i;
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int m : {1, 2, 4, 8}) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a, s);
            for (int k = 0; k < steps; k += m) {
                const int i = k % nslots;  // m consecutive slots (nslots % m == 0)
                if (m == 1)
                    cudaMemcpyAsync(d + i * slot + lo, h + i * slot + lo, width, cudaMemcpyHostToDevice, s);
                else
                    cudaMemcpy2DAsync(d + i * slot + lo, slot, h + i * slot + lo, slot, width, m,
                                      cudaMemcpyHostToDevice, s);
            }
            cudaEventRecord(b, s);
            cudaEventSynchronize(b);
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            if (rep)
                printf("rows/copy %d: %.2f us per 448 KB range, %.1f GB/s, %.0f ranges/s\n", m,
                       1e3 * ms / steps, width * steps / (ms * 1e6), steps / (ms * 1e-3));
        }
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
