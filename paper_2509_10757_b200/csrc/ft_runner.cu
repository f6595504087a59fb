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
// slots, and a native pump thread schedules the copies around it:
//   submit(k)  : (caller) H2D of slot i's ranges + event h2d[i]
//   pump       : h2d[i] complete -> ready[i] = k + 1 (pinned, mapped word the
//                kernel watches); done[i] >= k + 1 (mapped word the kernel
//                publishes) -> D2H of the outputs on slot i's stream + d2h[i];
//                d2h[i] complete -> step k is out (atomic counter)
//   wait(k)    : (caller) spins on that counter -- no CUDA call
// The pump's API calls run beside the caller's, so a step costs the caller
// one copy + one event record.  Push mode (default when host_out is pinned
// and device-mapped): the kernel's last block writes the outputs into
// host_out itself before publishing done, so the pump only watches done --
// no D2H copy, stream or event per step.
// No stream memory operations: each costs several microseconds of stream
// time, and one per step on the H2D stream capped the step rate.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <cstdio>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <mutex>
#include <cstdlib>
#include <new>
#include <thread>

#include "../../include/fasttrack_b200.h"

extern "C" int ft_internal_persist_launch(const void *const *plans, int n, unsigned *flags,
                                          const unsigned *h_ready, unsigned *h_done,
                                          void **args_out, cudaStream_t stream,
                                          void *const *push_dev, void *const *push_host,
                                          size_t push_bytes);
extern "C" void ft_internal_persist_dump(void);

namespace {
constexpr int PERSIST_MAX_SLOTS = 16;  // == ft_track.cu
constexpr unsigned PERSIST_STOP = 0xffffffffu;
}  // namespace

struct ft_runner {
    int n;
    bool persistent;
    unsigned *flags;  // persistent: [device ready x 8 | arrive x 8] device words
    void *args_dev;   // persistent: the kernel's argument array
    volatile unsigned *hflags;  // persistent: pinned mapped [ready x 8 | done x 8]
    unsigned *hflags_dev;
    std::atomic<int64_t> last_k;    // last submitted step (caller -> pump)
    std::atomic<int64_t> out_k;     // last step whose outputs are on the host (pump -> caller)
    std::atomic<int> pump_err;      // first error the pump met (FT_OK while healthy)
    std::atomic<bool> pump_stop;
    std::mutex pump_mu;               // idle pump: sleeps until a submit (or stop)
    std::condition_variable pump_cv;
    std::thread *pump;
    int device;
    int64_t next_ready;  // pump: oldest step whose ready word is not yet published
    int64_t next_d2h;    // pump: oldest step whose D2H is not yet issued
    int64_t next_out;    // pump: oldest step whose D2H has not yet completed
    cudaStream_t d2hs[FT_RUNNER_MAX_SLOTS];  // persistent: one D2H stream per slot
    cudaStream_t h2dx[3];  // persistent: extra H2D streams (steps round robin)
    int n_h2d;
    cudaStream_t h2d, comp, d2h;
    cudaEvent_t ev_h2d[FT_RUNNER_MAX_SLOTS], ev_comp[FT_RUNNER_MAX_SLOTS],
        ev_d2h[FT_RUNNER_MAX_SLOTS];
    cudaGraphExec_t exec[FT_RUNNER_MAX_SLOTS];
    void *dev_in[FT_RUNNER_MAX_SLOTS];
    void *dev_out[FT_RUNNER_MAX_SLOTS];
    void *host_out[FT_RUNNER_MAX_SLOTS];
    size_t in_bytes, out_bytes;
    bool push;  // persistent: the kernel writes the outputs to host_out itself
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

static void persist_pump_loop(ft_runner *r);

extern "C" int ft_runner_create_persistent(int32_t n_slots, const void *const *plans,
                                           void *const *dev_in, size_t in_bytes,
                                           void *const *dev_out, void *const *host_out,
                                           size_t out_bytes, ft_runner **out) {
    if (!plans || !dev_in || !dev_out || !host_out || !out) return FT_E_NULL;
    if (n_slots < 2 || n_slots > FT_RUNNER_MAX_SLOTS || n_slots > PERSIST_MAX_SLOTS)
        return FT_E_RANGE;
    // graph_exec slots are unused in persistent mode: reuse the plan pointers
    // as non-null placeholders for the shared constructor
    int st = ft_runner_create_n(n_slots, plans, dev_in, in_bytes, dev_out, host_out, out_bytes,
                                out);
    if (st != FT_OK) return st;
    ft_runner *r = *out;
    r->last_k.store(-1);
    r->out_k.store(-1);
    r->pump_err.store(FT_OK);
    r->pump_stop.store(false);
    r->next_ready = r->next_d2h = r->next_out = 0;
    cudaGetDevice(&r->device);
    cudaError_t e = cudaMalloc(&r->flags, 2 * PERSIST_MAX_SLOTS * sizeof(unsigned));
    if (e == cudaSuccess)
        e = cudaMemsetAsync(r->flags, 0, 2 * PERSIST_MAX_SLOTS * sizeof(unsigned), r->comp);
    void *hf = nullptr;
    if (e == cudaSuccess)
        e = cudaHostAlloc(&hf, 2 * PERSIST_MAX_SLOTS * sizeof(unsigned), cudaHostAllocMapped);
    if (e == cudaSuccess) {
        r->hflags = static_cast<volatile unsigned *>(hf);
        for (int i = 0; i < 2 * PERSIST_MAX_SLOTS; ++i) r->hflags[i] = 0;
        e = cudaHostGetDevicePointer(reinterpret_cast<void **>(&r->hflags_dev), hf, 0);
    }
    for (int i = 0; i < n_slots && e == cudaSuccess; ++i)
        e = cudaStreamCreateWithFlags(&r->d2hs[i], cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamSynchronize(r->comp);
    // push mode: the kernel's last block of a step writes the outputs into
    // host_out (pinned, device-mapped) with its own stores -- no D2H copy,
    // event or pump call per step (FT_RUNNER_PUSH=0 turns it off)
    void *hout_dev[PERSIST_MAX_SLOTS] = {nullptr};
    {
        const char *ev = getenv("FT_RUNNER_PUSH");
        r->push = !(ev && atoi(ev) == 0);
        for (int i = 0; i < n_slots && r->push; ++i) {
            cudaPointerAttributes at;
            if (cudaPointerGetAttributes(&at, host_out[i]) != cudaSuccess ||
                at.type != cudaMemoryTypeHost || !at.devicePointer ||
                (((uintptr_t)at.devicePointer | (uintptr_t)dev_out[i]) & 15u)) {
                cudaGetLastError();
                r->push = false;  // not device-mapped / aligned: the copy engine moves them
            } else {
                hout_dev[i] = at.devicePointer;
            }
        }
    }
    {
        // H2D streams used round robin: one in push mode (no D2H copies share
        // the link: 13.8 vs 14.3 us per step with two, r2ak), else two
        const char *ev = getenv("FT_RUNNER_H2D_STREAMS");
        const int want = ev ? atoi(ev) : (r->push ? 1 : 2);
        r->n_h2d = want < 1 ? 1 : (want > 4 ? 4 : want);
    }
    for (int q = 0; q + 1 < r->n_h2d && e == cudaSuccess; ++q)
        e = cudaStreamCreateWithFlags(&r->h2dx[q], cudaStreamNonBlocking);
    if (e == cudaSuccess) {
        st = ft_internal_persist_launch(plans, n_slots, r->flags, r->hflags_dev,
                                        r->hflags_dev + PERSIST_MAX_SLOTS, &r->args_dev,
                                        r->comp, r->push ? dev_out : nullptr,
                                        r->push ? hout_dev : nullptr, out_bytes);
        if (st != FT_OK) {  // no kernel to stop
            ft_runner_destroy(r);
            *out = nullptr;
            return st;
        }
        r->persistent = true;
        r->pump = new (std::nothrow) std::thread(persist_pump_loop, r);
        if (!r->pump) {
            ft_runner_destroy(r);
            *out = nullptr;
            return FT_E_RANGE;
        }
    }
    if (e != cudaSuccess) {
        ft_runner_destroy(r);
        *out = nullptr;
        return (int)e;
    }
    return FT_OK;
}

// Persistent mode: one pass of the pump -- publish the ready words of landed
// inputs, issue the D2H copies of finished steps, retire completed copies,
// oldest first (the H2D stream, the kernel and each slot complete steps in
// order), so a pass checks at most one event / flag per stage.  Returns
// whether anything moved, or a negative status.
static int persist_pump(ft_runner *r) {
    int moved = 0;
    const int64_t last = r->last_k.load(std::memory_order_acquire);
    if (r->next_ready <= last) {
        const int i = (int)(r->next_ready % r->n);
        const cudaError_t q = cudaEventQuery(r->ev_h2d[i]);
        if (q == cudaSuccess) {
            r->hflags[i] = (unsigned)(r->next_ready + 1);
            ++r->next_ready;
            moved = 1;
        } else if (q != cudaErrorNotReady) {
            return -(int)q;
        }
    }
    if (r->push && r->next_d2h < r->next_ready) {  // outputs written by the kernel
        const int i = (int)(r->next_d2h % r->n);
        const uint32_t want = (uint32_t)(r->next_d2h + 1);
        if ((int32_t)(r->hflags[PERSIST_MAX_SLOTS + i] - want) >= 0) {
            std::atomic_thread_fence(std::memory_order_acquire);
            r->out_k.store(r->next_d2h, std::memory_order_release);
            ++r->next_d2h;
            r->next_out = r->next_d2h;
            moved = 1;
        }
        return moved;
    }
    if (r->next_d2h < r->next_ready) {
        const int i = (int)(r->next_d2h % r->n);
        const uint32_t want = (uint32_t)(r->next_d2h + 1);
        if ((int32_t)(r->hflags[PERSIST_MAX_SLOTS + i] - want) >= 0) {
            cudaError_t e = cudaMemcpyAsync(r->host_out[i], r->dev_out[i], r->out_bytes,
                                            cudaMemcpyDeviceToHost, r->d2hs[i]);
            if (e == cudaSuccess) e = cudaEventRecord(r->ev_d2h[i], r->d2hs[i]);
            if (e != cudaSuccess) return -(int)e;
            ++r->next_d2h;
            moved = 1;
        }
    }
    if (r->next_out < r->next_d2h) {
        const cudaError_t q = cudaEventQuery(r->ev_d2h[r->next_out % r->n]);
        if (q == cudaSuccess) {
            r->out_k.store(r->next_out, std::memory_order_release);
            ++r->next_out;
            moved = 1;
        } else if (q != cudaErrorNotReady) {
            return -(int)q;
        }
    }
    return moved;
}

static void persist_pump_loop(ft_runner *r) {
    cudaSetDevice(r->device);
    auto idle_since = std::chrono::steady_clock::now();
    bool idle = false;
    while (!r->pump_stop.load(std::memory_order_acquire)) {
        const int m = persist_pump(r);
        if (m < 0) {
            r->pump_err.store(-m);  // the CUDA error
            return;
        }
        if (!m) {
            // nothing in flight (every submitted step is out) for 200 us: sleep
            // until the next submit instead of spinning a host core between
            // frames (a real-time tracker submits every ~50 ms).  While steps
            // are in flight, and briefly after, the pump spins -- its latency
            // is on every step's path.
            const bool none = r->next_out > r->last_k.load(std::memory_order_acquire);
            if (none && !idle) {
                idle = true;
                idle_since = std::chrono::steady_clock::now();
            } else if (!none) {
                idle = false;
            }
            if (idle && std::chrono::steady_clock::now() - idle_since >
                            std::chrono::microseconds(200)) {
                std::unique_lock<std::mutex> lk(r->pump_mu);
                r->pump_cv.wait_for(lk, std::chrono::milliseconds(5), [r] {
                    return r->pump_stop.load(std::memory_order_acquire) ||
                           r->next_out <= r->last_k.load(std::memory_order_acquire);
                });
                idle = false;
                continue;
            }
#if defined(__x86_64__) || defined(__i386__)
            __builtin_ia32_pause();
#endif
        }
    }
}

// Persistent mode: wait until step k's outputs are on the host (the pump
// thread's counter; no CUDA call on the caller's thread).
static int persist_wait(ft_runner *r, int64_t k) {
    if (k > r->last_k.load()) return FT_E_RANGE;  // never submitted
    const auto t0 = std::chrono::steady_clock::now();
    for (unsigned it = 1;; ++it) {
        if (r->out_k.load(std::memory_order_acquire) >= k) return FT_OK;
        const int err = r->pump_err.load();
        if (err != FT_OK) return err;
        if ((it & 4095u) == 0 &&
            std::chrono::steady_clock::now() - t0 > std::chrono::seconds(20))
            return FT_E_TIMEOUT;
#if defined(__x86_64__) || defined(__i386__)
        __builtin_ia32_pause();
#endif
    }
}

extern "C" int ft_runner_create(const void *const graph_exec[2], void *const dev_in[2],
                                size_t in_bytes, void *const dev_out[2],
                                void *const host_out[2], size_t out_bytes, ft_runner **out) {
    return ft_runner_create_n(2, graph_exec, dev_in, in_bytes, dev_out, host_out, out_bytes, out);
}

namespace {
struct NvtxRange {  // NVTX range for nsys / ncu timelines (a few ns without a tool)
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

extern "C" int ft_runner_submit_ranges(ft_runner *r, int64_t k, const void *host_in,
                                       const uint64_t *ranges, int32_t n_ranges) {
    if (!r || !host_in || (!ranges && n_ranges > 0)) return FT_E_NULL;
    NvtxRange nv("ft_runner_submit");
    if (k < 0 || n_ranges < 0) return FT_E_RANGE;
    for (int q = 0; q < n_ranges; ++q)
        if (ranges[2 * q] > ranges[2 * q + 1] || ranges[2 * q + 1] > r->in_bytes) return FT_E_RANGE;
    const int i = (int)(k % r->n);
    if (r->persistent) {
        if (k != r->last_k.load() + 1) return FT_E_RANGE;  // steps are submitted in order
        // slot i's step k-n must be fully out (outputs on the host, inputs consumed)
        if (k >= r->n) {
            const int st = persist_wait(r, k - r->n);
            if (st != FT_OK) return st;
        }
        // H2D streams round robin (several copy engines): one step's copy
        // overhead overlaps the other's transfer
        const int hq = (int)(k % r->n_h2d);
        cudaStream_t hs = hq == 0 ? r->h2d : r->h2dx[hq - 1];
        cudaError_t e = cudaSuccess;
        for (int q = 0; q < n_ranges && e == cudaSuccess; ++q) {
            const size_t lo = ranges[2 * q], n = ranges[2 * q + 1] - lo;
            if (n)
                e = cudaMemcpyAsync(static_cast<char *>(r->dev_in[i]) + lo,
                                    static_cast<const char *>(host_in) + lo, n,
                                    cudaMemcpyHostToDevice, hs);
        }
        if (e == cudaSuccess) e = cudaEventRecord(r->ev_h2d[i], hs);
        if (e != cudaSuccess) return (int)e;
        {
            std::lock_guard<std::mutex> lk(r->pump_mu);  // (pairs with the idle pump's wait)
            r->last_k.store(k, std::memory_order_release);  // the pump takes it from here
        }
        r->pump_cv.notify_one();
        return FT_OK;
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

extern "C" int ft_runner_submit_batch(ft_runner *r, int64_t k, int32_t m, const void *host_in,
                                      size_t host_pitch, const uint64_t *ranges,
                                      int32_t n_ranges) {
    if (!r || !host_in || (!ranges && n_ranges > 0)) return FT_E_NULL;
    if (k < 0 || n_ranges < 0 || m < 1 || m > r->n) return FT_E_RANGE;
    if (m > 1 && host_pitch < r->in_bytes) return FT_E_RANGE;
    for (int q = 0; q < n_ranges; ++q)
        if (ranges[2 * q] > ranges[2 * q + 1] || ranges[2 * q + 1] > r->in_bytes) return FT_E_RANGE;
    const int i0 = (int)(k % r->n);
    // one strided copy per range needs the m slots' device inputs at one pitch
    size_t dpitch = 0;
    bool strided = r->persistent && m > 1 && i0 + m <= r->n;
    if (strided) {
        const char *b0 = static_cast<const char *>(r->dev_in[i0]);
        const char *b1 = static_cast<const char *>(r->dev_in[i0 + 1]);
        strided = b1 > b0 && (size_t)(b1 - b0) >= r->in_bytes;
        dpitch = strided ? (size_t)(b1 - b0) : 0;
        for (int j = 2; j < m && strided; ++j)
            strided = static_cast<const char *>(r->dev_in[i0 + j]) == b0 + j * dpitch;
    }
    if (!strided) {  // step by step (graph mode, wrapped slots, scattered buffers)
        for (int j = 0; j < m; ++j) {
            const int st = ft_runner_submit_ranges(
                r, k + j, static_cast<const char *>(host_in) + j * host_pitch, ranges, n_ranges);
            if (st != FT_OK) return st;
        }
        return FT_OK;
    }
    NvtxRange nv("ft_runner_submit_batch");
    if (k != r->last_k.load() + 1) return FT_E_RANGE;  // steps are submitted in order
    // slots i0 .. i0+m-1: their steps k-n .. k+m-1-n must be fully out
    if (k + m - 1 >= r->n) {
        const int st = persist_wait(r, k + m - 1 - r->n);
        if (st != FT_OK) return st;
    }
    cudaStream_t hs = r->h2d;
    cudaError_t e = cudaSuccess;
    for (int q = 0; q < n_ranges && e == cudaSuccess; ++q) {
        const size_t lo = ranges[2 * q], w = ranges[2 * q + 1] - lo;
        if (w)
            e = cudaMemcpy2DAsync(static_cast<char *>(r->dev_in[i0]) + lo, dpitch,
                                  static_cast<const char *>(host_in) + lo, host_pitch, w, m,
                                  cudaMemcpyHostToDevice, hs);
    }
    for (int j = 0; j < m && e == cudaSuccess; ++j) e = cudaEventRecord(r->ev_h2d[i0 + j], hs);
    if (e != cudaSuccess) return (int)e;
    {
        std::lock_guard<std::mutex> lk(r->pump_mu);
        r->last_k.store(k + m - 1, std::memory_order_release);
    }
    r->pump_cv.notify_one();
    return FT_OK;
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
    NvtxRange nv("ft_runner_wait");
    if (k < 0) return FT_E_RANGE;
    if (r->persistent) return persist_wait(r, k);
    return (int)cudaEventSynchronize(r->ev_d2h[k % r->n]);
}

extern "C" int ft_runner_destroy(ft_runner *r) {
    if (!r) return FT_OK;
    if (r->persistent) {
        // every submitted step completes first, so all blocks are polling the
        // next ready word -- then stop the persistent kernel (a stop seen
        // mid-step by a late block would leave its group at a barrier)
        const int64_t last = r->last_k.load();
        if (last >= 0) persist_wait(r, last);
        {
            std::lock_guard<std::mutex> lk(r->pump_mu);
            r->pump_stop.store(true);
        }
        r->pump_cv.notify_one();
        if (r->pump) {
            r->pump->join();
            delete r->pump;
            r->pump = nullptr;
        }
        for (int i = 0; i < PERSIST_MAX_SLOTS; ++i) r->hflags[i] = PERSIST_STOP;
        cudaStreamSynchronize(r->comp);
        ft_internal_persist_dump();
    }
    if (r->flags) cudaFree(r->flags);
    r->flags = nullptr;
    if (r->args_dev) cudaFree(r->args_dev);
    r->args_dev = nullptr;
    if (r->hflags) cudaFreeHost(const_cast<unsigned *>(r->hflags));
    r->hflags = nullptr;
    for (int i = 0; i < r->n; ++i)
        if (r->d2hs[i]) cudaStreamDestroy(r->d2hs[i]);
    for (int q = 0; q < 3; ++q)
        if (r->h2dx[q]) {
            cudaStreamSynchronize(r->h2dx[q]);
            cudaStreamDestroy(r->h2dx[q]);
        }
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
