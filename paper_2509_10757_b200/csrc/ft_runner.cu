// ft_runner.cu -- native multi-buffered step executor (host side of the
// C ABI).  It is the real-time shape of the tracker (reference tracker.py
// track_frame called once per incoming frame): while step k computes, the
// inputs of the next steps upload and the results of the previous ones
// download.
//
// n "slots" (buffer sets, 2..FT_RUNNER_MAX_SLOTS) take steps round robin;
// each slot owns a pre-instantiated CUDA graph of the per-step compute
// (pyramids / ft_track_frames, captured by the caller), a device input range,
// a device output range and a pinned host output range.  Per step k (slot
// i = k % n):
//   H2D stream : wait comp[i] (step k-n done reading the slot's inputs)
//                memcpy host_in ranges -> dev_in[i]; record h2d[i]
//   comp stream: wait h2d[i], wait d2h[i] (step k-n's outputs are out)
//                graph launch exec[i]; record comp[i]
//   D2H stream : wait comp[i]; memcpy dev_out[i] -> host_out[i]; record d2h[i]
// Compute is one stream, so cooperative kernels never overlap each other.
// Everything is issued from C: one host call per step.  With n = 3 the host
// may submit step k once step k-3 is out, so uploads run a full step ahead.
//
// Persistent mode (ft_runner_create_persistent): no per-step launch.  One
// long-lived track kernel (ft_track.cu track_persist_kernel) serves the n
// slots:
//   H2D stream   : wait d2h[i] (step k-n fully out); memcpy ranges;
//                  write ready[i] = k + 1 (stream memory op)
//   kernel       : polls ready[i], computes; the step's last block publishes
//                  done[i] = k + 1
//   D2H stream i : wait done[i] >= k + 1 (stream memory op); memcpy outputs;
//                  record d2h[i]
// One D2H stream per slot: a stream wait resolves by polling at coarse
// intervals, and on a single stream those latencies queued up step after
// step (capping the rate at ~19 us per step); per slot they overlap.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdlib>
#include <new>

#include "../../include/fasttrack_b200.h"

extern "C" int ft_internal_persist_launch(const void *const *plans, int n, unsigned *flags,
                                          cudaStream_t stream);
extern "C" void ft_internal_persist_dump(void);

namespace {
constexpr int PERSIST_MAX_SLOTS = 8;  // == ft_track.cu
constexpr unsigned PERSIST_STOP = 0xffffffffu;
typedef CUresult (*WaitValue32Fn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*WriteValue32Fn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

// cuStreamWaitValue32 / cuStreamWriteValue32 through the runtime's driver
// entry-point query (no link-time libcuda dependency)
bool stream_memops(WaitValue32Fn *wait, WriteValue32Fn *write) {
    static WaitValue32Fn w = nullptr;
    static WriteValue32Fn v = nullptr;
    if (!w || !v) {
        void *a = nullptr, *b = nullptr;
        cudaDriverEntryPointQueryResult qa, qb;
        if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &a, cudaEnableDefault, &qa) !=
                cudaSuccess ||
            qa != cudaDriverEntryPointSuccess)
            return false;
        if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &b, cudaEnableDefault, &qb) !=
                cudaSuccess ||
            qb != cudaDriverEntryPointSuccess)
            return false;
        w = (WaitValue32Fn)a;
        v = (WriteValue32Fn)b;
    }
    *wait = w;
    *write = v;
    return true;
}
}  // namespace

struct ft_runner {
    int n;
    bool persistent;
    unsigned *flags;  // persistent: [ready x 8 | done x 8 | arrive x 8] device words
    int64_t last_k;
    cudaStream_t d2hs[FT_RUNNER_MAX_SLOTS];  // persistent: one D2H stream per slot
    WaitValue32Fn wait32;
    WriteValue32Fn write32;
    cudaStream_t h2d, comp, d2h;
    cudaEvent_t ev_h2d[FT_RUNNER_MAX_SLOTS], ev_comp[FT_RUNNER_MAX_SLOTS],
        ev_d2h[FT_RUNNER_MAX_SLOTS];
    cudaGraphExec_t exec[FT_RUNNER_MAX_SLOTS];
    void *dev_in[FT_RUNNER_MAX_SLOTS];
    void *dev_out[FT_RUNNER_MAX_SLOTS];
    void *host_out[FT_RUNNER_MAX_SLOTS];
    size_t in_bytes, out_bytes;
};

extern "C" int ft_runner_create_n(int32_t n_slots, const void *const *graph_exec,
                                  void *const *dev_in, size_t in_bytes, void *const *dev_out,
                                  void *const *host_out, size_t out_bytes, ft_runner **out) {
    if (!graph_exec || !dev_in || !dev_out || !host_out || !out) return FT_E_NULL;
    if (n_slots < 2 || n_slots > FT_RUNNER_MAX_SLOTS) return FT_E_RANGE;
    for (int i = 0; i < n_slots; ++i)
        if (!graph_exec[i] || !dev_in[i] || !dev_out[i] || !host_out[i]) return FT_E_NULL;
    ft_runner *r = new (std::nothrow) ft_runner();
    if (!r) return FT_E_RANGE;
    r->n = n_slots;
    cudaError_t e = cudaSuccess;
    const unsigned fl = cudaStreamNonBlocking;
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&r->h2d, fl);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&r->comp, fl);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&r->d2h, fl);
    for (int i = 0; i < n_slots && e == cudaSuccess; ++i) {
        e = cudaEventCreateWithFlags(&r->ev_h2d[i], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&r->ev_comp[i], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&r->ev_d2h[i], cudaEventDisableTiming);
        // recorded once so the first waits are satisfied
        if (e == cudaSuccess) e = cudaEventRecord(r->ev_comp[i], r->comp);
        if (e == cudaSuccess) e = cudaEventRecord(r->ev_d2h[i], r->d2h);
        r->exec[i] = (cudaGraphExec_t)graph_exec[i];
        r->dev_in[i] = dev_in[i];
        r->dev_out[i] = dev_out[i];
        r->host_out[i] = host_out[i];
    }
    r->in_bytes = in_bytes;
    r->out_bytes = out_bytes;
    if (e != cudaSuccess) {
        delete r;
        return (int)e;
    }
    *out = r;
    return FT_OK;
}

extern "C" int ft_runner_create_persistent(int32_t n_slots, const void *const *plans,
                                           void *const *dev_in, size_t in_bytes,
                                           void *const *dev_out, void *const *host_out,
                                           size_t out_bytes, ft_runner **out) {
    if (!plans || !dev_in || !dev_out || !host_out || !out) return FT_E_NULL;
    if (n_slots < 2 || n_slots > FT_RUNNER_MAX_SLOTS || n_slots > PERSIST_MAX_SLOTS)
        return FT_E_RANGE;
    WaitValue32Fn w;
    WriteValue32Fn v;
    if (!stream_memops(&w, &v)) return FT_E_CONFIG;
    // graph_exec slots are unused in persistent mode: reuse the plan pointers
    // as non-null placeholders for the shared constructor
    int st = ft_runner_create_n(n_slots, plans, dev_in, in_bytes, dev_out, host_out, out_bytes,
                                out);
    if (st != FT_OK) return st;
    ft_runner *r = *out;
    r->persistent = true;
    r->wait32 = w;
    r->write32 = v;
    r->last_k = -1;
    cudaError_t e = cudaMalloc(&r->flags, 3 * PERSIST_MAX_SLOTS * sizeof(unsigned));
    if (e == cudaSuccess)
        e = cudaMemsetAsync(r->flags, 0, 3 * PERSIST_MAX_SLOTS * sizeof(unsigned), r->comp);
    for (int i = 0; i < n_slots && e == cudaSuccess; ++i)
        e = cudaStreamCreateWithFlags(&r->d2hs[i], cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamSynchronize(r->comp);
    if (e == cudaSuccess) {
        st = ft_internal_persist_launch(plans, n_slots, r->flags, r->comp);
        if (st != FT_OK) {
            cudaStreamSynchronize(r->comp);
            cudaFree(r->flags);
            r->flags = nullptr;
            r->persistent = false;
            ft_runner_destroy(r);
            *out = nullptr;
            return st;
        }
    }
    if (e != cudaSuccess) {
        ft_runner_destroy(r);
        *out = nullptr;
        return (int)e;
    }
    return FT_OK;
}

extern "C" int ft_runner_create(const void *const graph_exec[2], void *const dev_in[2],
                                size_t in_bytes, void *const dev_out[2],
                                void *const host_out[2], size_t out_bytes, ft_runner **out) {
    return ft_runner_create_n(2, graph_exec, dev_in, in_bytes, dev_out, host_out, out_bytes, out);
}

extern "C" int ft_runner_submit_ranges(ft_runner *r, int64_t k, const void *host_in,
                                       const uint64_t *ranges, int32_t n_ranges) {
    if (!r || !host_in || (!ranges && n_ranges > 0)) return FT_E_NULL;
    if (k < 0 || n_ranges < 0) return FT_E_RANGE;
    for (int q = 0; q < n_ranges; ++q)
        if (ranges[2 * q] > ranges[2 * q + 1] || ranges[2 * q + 1] > r->in_bytes) return FT_E_RANGE;
    const int i = (int)(k % r->n);
    if (r->persistent) {
        // slot i's step k-n is out (its outputs copied, so its inputs are
        // consumed too); then inputs -> ready -> (kernel) -> done -> outputs
        cudaError_t e = cudaStreamWaitEvent(r->h2d, r->ev_d2h[i], 0);
        for (int q = 0; q < n_ranges && e == cudaSuccess; ++q) {
            const size_t lo = ranges[2 * q], n = ranges[2 * q + 1] - lo;
            if (n)
                e = cudaMemcpyAsync(static_cast<char *>(r->dev_in[i]) + lo,
                                    static_cast<const char *>(host_in) + lo, n,
                                    cudaMemcpyHostToDevice, r->h2d);
        }
        const cuuint32_t step = (cuuint32_t)(k + 1);
        if (e == cudaSuccess &&
            r->write32((CUstream)r->h2d, (CUdeviceptr)(r->flags + i), step,
                       CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS)
            return FT_E_CONFIG;
        cudaStream_t ds = r->d2hs[i];
        if (e == cudaSuccess &&
            r->wait32((CUstream)ds, (CUdeviceptr)(r->flags + PERSIST_MAX_SLOTS + i), step,
                      CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
            return FT_E_CONFIG;
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(r->host_out[i], r->dev_out[i], r->out_bytes,
                                cudaMemcpyDeviceToHost, ds);
        if (e == cudaSuccess) e = cudaEventRecord(r->ev_d2h[i], ds);
        if (e == cudaSuccess && k > r->last_k) r->last_k = k;
        return (int)e;
    }
    cudaError_t e = cudaStreamWaitEvent(r->h2d, r->ev_comp[i], 0);
    for (int q = 0; q < n_ranges && e == cudaSuccess; ++q) {
        const size_t lo = ranges[2 * q], n = ranges[2 * q + 1] - lo;
        if (n)
            e = cudaMemcpyAsync(static_cast<char *>(r->dev_in[i]) + lo,
                                static_cast<const char *>(host_in) + lo, n,
                                cudaMemcpyHostToDevice, r->h2d);
    }
    if (e == cudaSuccess) e = cudaEventRecord(r->ev_h2d[i], r->h2d);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(r->comp, r->ev_h2d[i], 0);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(r->comp, r->ev_d2h[i], 0);
    if (e == cudaSuccess) e = cudaGraphLaunch(r->exec[i], r->comp);
    if (e == cudaSuccess) e = cudaEventRecord(r->ev_comp[i], r->comp);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(r->d2h, r->ev_comp[i], 0);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(r->host_out[i], r->dev_out[i], r->out_bytes, cudaMemcpyDeviceToHost,
                            r->d2h);
    if (e == cudaSuccess) e = cudaEventRecord(r->ev_d2h[i], r->d2h);
    return (int)e;
}

extern "C" int ft_runner_submit_range(ft_runner *r, int64_t k, const void *host_in,
                                      size_t offset, size_t bytes) {
    if (!r || !host_in) return FT_E_NULL;
    if (offset > r->in_bytes || bytes > r->in_bytes - offset) return FT_E_RANGE;
    const uint64_t rg[2] = {offset, offset + bytes};
    return ft_runner_submit_ranges(r, k, host_in, rg, 1);
}

extern "C" int ft_runner_submit(ft_runner *r, int64_t k, const void *host_in) {
    if (!r) return FT_E_NULL;
    return ft_runner_submit_range(r, k, host_in, 0, r->in_bytes);
}

extern "C" int ft_runner_wait(ft_runner *r, int64_t k) {
    if (!r) return FT_E_NULL;
    if (k < 0) return FT_E_RANGE;

    return (int)cudaEventSynchronize(r->ev_d2h[k % r->n]);
}

extern "C" int ft_runner_destroy(ft_runner *r) {
    if (!r) return FT_OK;
    if (r->persistent && r->flags) {
        // every submitted step completes first, so all blocks are polling the
        // next ready word -- then stop the persistent kernel (a stop seen
        // mid-step by a late block would leave its group at a barrier)
        cudaStreamSynchronize(r->h2d);
        for (int i = 0; i < r->n; ++i) cudaStreamSynchronize(r->d2hs[i]);
        for (int i = 0; i < PERSIST_MAX_SLOTS; ++i)
            r->write32((CUstream)r->h2d, (CUdeviceptr)(r->flags + i), PERSIST_STOP,
                       CU_STREAM_WRITE_VALUE_DEFAULT);
        cudaStreamSynchronize(r->h2d);
        cudaStreamSynchronize(r->comp);
        ft_internal_persist_dump();
        cudaFree(r->flags);
        r->flags = nullptr;
    }
    for (int i = 0; i < r->n; ++i)
        if (r->d2hs[i]) cudaStreamDestroy(r->d2hs[i]);
    cudaStreamSynchronize(r->h2d);
    cudaStreamSynchronize(r->comp);
    cudaStreamSynchronize(r->d2h);
    for (int i = 0; i < r->n; ++i) {
        cudaEventDestroy(r->ev_h2d[i]);
        cudaEventDestroy(r->ev_comp[i]);
        cudaEventDestroy(r->ev_d2h[i]);
    }
    cudaStreamDestroy(r->h2d);
    cudaStreamDestroy(r->comp);
    cudaStreamDestroy(r->d2h);
    delete r;
    return FT_OK;
}
