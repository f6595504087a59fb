// ft_runner.cu -- native double-buffered step executor (host side of the
// C ABI).  It is the real-time shape of the tracker (reference tracker.py
// track_frame called once per incoming frame): while step k computes, the
// inputs of step k+1 upload and the results of step k-1 download.
//
// Two "slots" (buffer sets) alternate; each slot owns a pre-instantiated
// CUDA graph of the per-step compute (gather / pyramids / ft_track_frames,
// captured by the caller), a device input range, a device output range and a
// pinned host output range.  Per step k (slot i = k % 2):
//   H2D stream : wait comp[i] (step k-2 done reading inputs)
//                memcpy host_in -> dev_in[i]; record h2d[i]
//   comp stream: wait h2d[i], wait d2h[i] (step k-2's outputs are out)
//                graph launch exec[i]; record comp[i]
//   D2H stream : wait comp[i]; memcpy dev_out[i] -> host_out[i]; record d2h[i]
// Compute is one stream, so cooperative kernels never overlap each other.
// Everything is issued from C: one host call per step.
#include <cuda_runtime.h>

#include <cstdlib>
#include <new>

#include "../../include/fasttrack_b200.h"

struct ft_runner {
    cudaStream_t h2d, comp, d2h;
    cudaEvent_t ev_h2d[2], ev_comp[2], ev_d2h[2];
    cudaGraphExec_t exec[2];
    void *dev_in[2];
    void *dev_out[2];
    void *host_out[2];
    size_t in_bytes, out_bytes;
};

extern "C" int ft_runner_create(const void *const graph_exec[2], void *const dev_in[2],
                                size_t in_bytes, void *const dev_out[2],
                                void *const host_out[2], size_t out_bytes, ft_runner **out) {
    if (!graph_exec || !dev_in || !dev_out || !host_out || !out) return FT_E_NULL;
    for (int i = 0; i < 2; ++i)
        if (!graph_exec[i] || !dev_in[i] || !dev_out[i] || !host_out[i]) return FT_E_NULL;
    ft_runner *r = new (std::nothrow) ft_runner();
    if (!r) return FT_E_RANGE;
    cudaError_t e = cudaSuccess;
    const unsigned fl = cudaStreamNonBlocking;
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&r->h2d, fl);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&r->comp, fl);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&r->d2h, fl);
    for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
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

extern "C" int ft_runner_submit_range(ft_runner *r, int64_t k, const void *host_in,
                                      size_t offset, size_t bytes) {
    if (!r || !host_in) return FT_E_NULL;
    if (k < 0 || offset > r->in_bytes || bytes > r->in_bytes - offset) return FT_E_RANGE;
    const int i = (int)(k & 1);
    cudaError_t e = cudaStreamWaitEvent(r->h2d, r->ev_comp[i], 0);
    if (e == cudaSuccess && bytes)
        e = cudaMemcpyAsync(static_cast<char *>(r->dev_in[i]) + offset,
                            static_cast<const char *>(host_in) + offset, bytes,
                            cudaMemcpyHostToDevice, r->h2d);
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

extern "C" int ft_runner_submit_ranges(ft_runner *r, int64_t k, const void *host_in,
                                       const uint64_t *ranges, int32_t n_ranges) {
    if (!r || !host_in || (!ranges && n_ranges > 0)) return FT_E_NULL;
    if (k < 0 || n_ranges < 0) return FT_E_RANGE;
    for (int q = 0; q < n_ranges; ++q)
        if (ranges[2 * q] > ranges[2 * q + 1] || ranges[2 * q + 1] > r->in_bytes) return FT_E_RANGE;
    const int i = (int)(k & 1);
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

extern "C" int ft_runner_submit(ft_runner *r, int64_t k, const void *host_in) {
    if (!r) return FT_E_NULL;
    return ft_runner_submit_range(r, k, host_in, 0, r->in_bytes);
}

extern "C" int ft_runner_wait(ft_runner *r, int64_t k) {
    if (!r) return FT_E_NULL;
    if (k < 0) return FT_E_RANGE;
    return (int)cudaEventSynchronize(r->ev_d2h[k & 1]);
}

extern "C" int ft_runner_destroy(ft_runner *r) {
    if (!r) return FT_OK;
    cudaStreamSynchronize(r->h2d);
    cudaStreamSynchronize(r->comp);
    cudaStreamSynchronize(r->d2h);
    for (int i = 0; i < 2; ++i) {
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
