// Probe: does one strided 2D copy of m step ranges (cudaMemcpy2DAsync, host
// and device pitches = slot strides) amortise the fixed per-copy cost of the
// H2D copy engine?  Times back-to-back 448 KB ranges as m-row 2D copies,
// m = 1 (plain 1D copy), 2, 4, 8, from pinned host memory into 8 device slots.
// Build: nvcc -O2 -gencode arch=compute_100a,code=sm_100a tools/h2d2d_probe.cu -o tools/h2d2d_probe
#include <cstdio>
#include <cuda_runtime.h>

// stand-in for the persistent runner's PCIe traffic beside the uploads: per
// "step" a block pushes 72 KB of results into mapped host memory (16-B
// stores) and polls a mapped host word (as the kernel polls ready flags)
__device__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// write: 72 KB of results pushed every period_ns; poll: thread 0 polls a
// mapped host word (the runner kernel's PCIe watcher: ld + nanosleep(100))
__global__ void push_kernel(uint4 *hout, volatile unsigned *hflag, unsigned long long dur_ns,
                            int write, int poll, unsigned period_ns, unsigned *sink) {
    unsigned acc = 0;
    const unsigned long long t0 = gtime();
    unsigned long long next = t0;
    __shared__ int stop;
    for (int it = 0;; ++it) {
        if (threadIdx.x == 0) stop = gtime() - t0 > dur_ns;
        __syncthreads();
        if (stop) break;
        if (write && gtime() >= next) {
            for (int t = threadIdx.x; t < 72 * 1024 / 16; t += blockDim.x)
                hout[t] = make_uint4(it, t, 0, 0);
            __threadfence_system();
            next += period_ns;
        }
        if (threadIdx.x == 0) {
            if (poll) {
                for (int q = 0; q < 16; ++q) {
                    acc += hflag[0];
                    __nanosleep(100);
                }
            } else {
                __nanosleep(1000);
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) *sink = acc;
}

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
    uint4 *hout;
    unsigned *hflag, *sink;
    cudaHostAlloc(&hout, 72 * 1024, cudaHostAllocMapped);
    cudaHostAlloc(&hflag, 64, cudaHostAllocMapped);
    cudaMalloc(&sink, 4);
    cudaStream_t s2;
    cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
    // 1D copies with an event after each (the runner's per-step record), alone
    // and beside the push kernel
    cudaEvent_t per;
    cudaEventCreateWithFlags(&per, cudaEventDisableTiming);
    const char *names[6] = {"", ", polls beside", ", 72 KB push / 14 us beside",
                            ", polls + 72 KB push / 14 us beside", ", 72 KB push / 28 us beside",
                            ", 72 KB push / 7 us beside"};
    for (int mode = 0; mode < 6; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            const unsigned period = mode == 4 ? 28000 : (mode == 5 ? 7000 : 14000);
            if (mode)
                push_kernel<<<1, 512, 0, s2>>>(hout, hflag, 80000000ull, mode >= 4 || (mode & 2),
                                               mode < 4 && (mode & 1), period, sink);
            cudaEventRecord(a, s);
            for (int k = 0; k < steps; ++k) {
                const int i = k % nslots;
                cudaMemcpyAsync(d + i * slot + lo, h + i * slot + lo, width, cudaMemcpyHostToDevice, s);
                cudaEventRecord(per, s);
            }
            cudaEventRecord(b, s);
            cudaEventSynchronize(b);
            cudaStreamSynchronize(s2);
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            if (rep)
                printf("1D + event per copy%s: %.2f us per 448 KB range, %.0f ranges/s\n",
                       names[mode], 1e3 * ms / steps, steps / (ms * 1e-3));
        }
    }
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
