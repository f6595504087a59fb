// ft_session.cu -- host-side drop-in calls: the reference's stage functions
// (trackfront stereo.py / projection.py / localmap.py) called with HOST
// arrays -- the reference's numpy SoA fields -- in ONE C call each:
//
//   pack the SoA fields into records in pinned staging (C loops, no Python
//   per element) -> one H2D per contiguous input range -> the device entry
//   (ft_stereo_pinhole / ft_project_search / ft_stereo_fisheye[_bf]) -> one
//   D2H of exactly the requested outputs -> synchronise -> copy into the
//   caller's arrays.
//
// The per-call Python work is then a handful of pointer fields (the
// reference objects' arrays are passed in place).  A session owns one
// stream, pinned staging, a device arena and a workspace, all grown on
// demand and reused (the reference's BufferPool contract, buffers.py:13-55).
// A session serves one tracking thread (the reference's single-writer rule,
// tracker.py:1-7); calls are synchronous like the reference's.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>

#include "../../include/fasttrack_b200.h"

struct ft_session {
    int device = 0;
    cudaStream_t stream = nullptr;
    char *h = nullptr;  // pinned staging
    size_t h_cap = 0;
    char *d = nullptr;  // device arena
    size_t d_cap = 0;
    void *ws_mem = nullptr;
    ft_workspace ws{};
    int cap_kp = 1024, cap_pts = 1024;  // high-water capacities (workspace geometry)
    // host-side phase timers (us) accumulated over calls: pack, issue (copies +
    // launch enqueue), device (kernel, cudaEvents, FT_SESSION_TIMING=1 only),
    // sync (wait for the stream), unpack; [5] = calls
    double stats[6] = {0, 0, 0, 0, 0, 0};
    bool timing = getenv("FT_SESSION_TIMING") != nullptr;
    cudaEvent_t ev[2] = {nullptr, nullptr};
};

namespace {

constexpr size_t SALIGN = 256;
size_t salign(size_t x) { return (x + SALIGN - 1) & ~(SALIGN - 1); }

struct Lay {
    size_t total = 0;
    size_t add(size_t n) {
        const size_t o = total;
        total += salign(n ? n : 1);
        return o;
    }
};

int reserve(ft_session *s, size_t bytes) {
    cudaError_t e;
    if (bytes > s->h_cap) {
        const size_t cap = salign(std::max(bytes, std::max(2 * s->h_cap, (size_t)1 << 20)));
        if (s->h) cudaFreeHost(s->h);
        s->h = nullptr;
        s->h_cap = 0;
        e = cudaHostAlloc((void **)&s->h, cap, cudaHostAllocDefault);
        if (e != cudaSuccess) return (int)e;
        memset(s->h, 0, cap);  // capacity-strided layouts ship bytes past the counts
        s->h_cap = cap;
    }
    if (bytes > s->d_cap) {
        const size_t cap = salign(std::max(bytes, std::max(2 * s->d_cap, (size_t)1 << 20)));
        if (s->d) cudaFree(s->d);
        s->d = nullptr;
        s->d_cap = 0;
        e = cudaMalloc((void **)&s->d, cap);
        if (e == cudaSuccess) e = cudaMemsetAsync(s->d, 0, cap, s->stream);
        if (e != cudaSuccess) return (int)e;
        s->d_cap = cap;
    }
    return FT_OK;
}

// high-water capacities (multiples of 256 keypoints / 1024 points) and the
// workspace for them, re-initialised only when they grow
int caps(ft_session *s, int64_t n_kp, int64_t n_pts) {
    if (n_kp > 65535) return FT_E_RANGE;  // 16-bit keypoint index in the kernels' keys
    bool grow = s->ws_mem == nullptr;
    if (n_kp > s->cap_kp) {
        s->cap_kp = (int)((n_kp + 255) / 256 * 256);
        grow = true;
    }
    if (n_pts > s->cap_pts) {
        s->cap_pts = (int)((n_pts + 1023) / 1024 * 1024);
        grow = true;
    }
    if (!grow) return FT_OK;
    if (s->ws_mem) cudaFree(s->ws_mem);
    s->ws_mem = nullptr;
    const size_t b = ft_workspace_bytes(1, s->cap_kp, s->cap_pts);
    cudaError_t e = cudaMalloc(&s->ws_mem, b);
    if (e != cudaSuccess) return (int)e;
    s->ws.base = s->ws_mem;
    s->ws.bytes = b;
    s->ws.n_frames = 1;
    s->ws.cap_left = s->cap_kp;
    s->ws.cap_points = s->cap_pts;
    return ft_workspace_init(&s->ws, s->stream);
}

void pack_kp(const ft_host_features *f, ft_kp_record *out) {
    const int64_t n = f->n;
    for (int64_t i = 0; i < n; ++i) {
        ft_kp_record &r = out[i];
        r.u = f->u ? f->u[i] : 0.0;
        r.v = f->v ? f->v[i] : 0.0;
        if (f->desc)
            memcpy(r.desc, f->desc + 4 * i, 32);
        else
            memset(r.desc, 0, 32);
        r.angle = f->angle ? f->angle[i] : 0.0;
        r.octave = f->octave ? f->octave[i] : 0;
        r.pad = 0;
    }
}

void pack_points(const ft_host_points *p, ft_point_record *out) {
    for (int64_t i = 0; i < p->m; ++i) {
        ft_point_record &r = out[i];
        memcpy(r.desc, p->desc + 4 * i, 32);
        memcpy(r.pos, p->positions + 3 * i, 24);
        memcpy(r.nrm, p->normals + 3 * i, 24);
        r.min_dist = p->min_dist[i];
        r.max_dist = p->max_dist[i];
        r.id = p->ids ? p->ids[i] : 0;
        r.pad = 0;
    }
}

int h2d(ft_session *s, size_t off, size_t bytes) {
    if (!bytes) return FT_OK;
    return (int)cudaMemcpyAsync(s->d + off, s->h + off, bytes, cudaMemcpyHostToDevice, s->stream);
}

int d2h(ft_session *s, size_t off, size_t bytes) {
    if (!bytes) return FT_OK;
    return (int)cudaMemcpyAsync(s->h + off, s->d + off, bytes, cudaMemcpyDeviceToHost, s->stream);
}

ft_pyramid dev_pyramid(const ft_host_pyramid *p, const uint8_t *dev) {
    ft_pyramid q;
    memset(&q, 0, sizeof(q));
    q.data = dev;
    q.frame_bytes = 0;
    q.n_levels = p->n_levels;
    for (int l = 0; l < p->n_levels; ++l) {
        q.offsets[l] = p->offsets[l];
        q.widths[l] = p->widths[l];
        q.heights[l] = p->heights[l];
    }
    return q;
}

using Clock = std::chrono::steady_clock;
double us_since(Clock::time_point t) {
    return std::chrono::duration<double, std::micro>(Clock::now() - t).count();
}

// Phase timer of one session call (host clock; kernel time by events when
// the session was created with FT_SESSION_TIMING set).
// NVTX: one range per session call ("ft_session_<stage>"), with nested
// phase ranges (pack, issue, sync, unpack) -- visible in nsys / ncu
// timelines; a few ns per call without a tool attached (tracing).
const char *const PHASE_NAMES[5] = {"pack", "issue", "kernel", "sync", "unpack"};

struct Phases {
    ft_session *s;
    Clock::time_point t;
    explicit Phases(ft_session *s_, const char *name = "ft_session") : s(s_), t(Clock::now()) {
        nvtxRangePushA(name);
        nvtxRangePushA(PHASE_NAMES[0]);
    }
    ~Phases() {
        nvtxRangePop();  // phase
        nvtxRangePop();  // call
    }
    void mark(int k) {
        s->stats[k] += us_since(t);
        t = Clock::now();
        nvtxRangePop();
        nvtxRangePushA(k == 0 ? PHASE_NAMES[1] : k == 1 ? PHASE_NAMES[3] : PHASE_NAMES[4]);
    }
    void kernel_begin() {
        if (s->timing) cudaEventRecord(s->ev[0], s->stream);
    }
    void kernel_end() {
        if (s->timing) cudaEventRecord(s->ev[1], s->stream);
    }
    void done() {
        if (s->timing) {
            float ms = 0.f;
            if (cudaEventElapsedTime(&ms, s->ev[0], s->ev[1]) == cudaSuccess) s->stats[2] += 1e3 * ms;
        }
        s->stats[5] += 1;
    }
};

#define FT_TRY(x)                     \
    do {                              \
        const int st_ = (x);          \
        if (st_ != FT_OK) return st_; \
    } while (0)

}  // namespace

extern "C" int ft_host_pack_keypoints(const ft_host_features *f, ft_kp_record *out) {
    if (!f || (f->n && !out)) return FT_E_NULL;
    if (f->n < 0) return FT_E_RANGE;
    pack_kp(f, out);
    return FT_OK;
}

extern "C" int ft_host_pack_points(const ft_host_points *p, ft_point_record *out) {
    if (!p || (p->m && (!out || !p->positions || !p->normals || !p->min_dist || !p->max_dist ||
                        !p->desc)))
        return FT_E_NULL;
    if (p->m < 0) return FT_E_RANGE;
    pack_points(p, out);
    return FT_OK;
}

extern "C" int ft_session_create(int32_t device, ft_session **out) {
    if (!out) return FT_E_NULL;
    *out = nullptr;
    ft_session *s = new ft_session();
    s->device = device;
    cudaError_t e = cudaSetDevice(device);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking);
    if (e == cudaSuccess && s->timing) e = cudaEventCreate(&s->ev[0]);
    if (e == cudaSuccess && s->timing) e = cudaEventCreate(&s->ev[1]);
    if (e != cudaSuccess) {
        delete s;
        return (int)e;
    }
    *out = s;
    return FT_OK;
}

extern "C" int ft_session_destroy(ft_session *s) {
    if (!s) return FT_OK;
    cudaSetDevice(s->device);
    if (s->stream) cudaStreamSynchronize(s->stream);
    if (s->h) cudaFreeHost(s->h);
    if (s->d) cudaFree(s->d);
    if (s->ws_mem) cudaFree(s->ws_mem);
    if (s->ev[0]) cudaEventDestroy(s->ev[0]);
    if (s->ev[1]) cudaEventDestroy(s->ev[1]);
    if (s->stream) cudaStreamDestroy(s->stream);
    delete s;
    return FT_OK;
}

extern "C" int ft_session_stats(ft_session *s, double *out, int32_t reset) {
    if (!s || !out) return FT_E_NULL;
    for (int k = 0; k < 6; ++k) {
        out[k] = s->stats[k];
        if (reset) s->stats[k] = 0;
    }
    return FT_OK;
}

extern "C" int ft_session_stereo(ft_session *s, const ft_host_features *left,
                                 const ft_host_features *right, const ft_host_pyramid *left_pyr,
                                 const ft_host_pyramid *right_pyr, const ft_stereo_params *params,
                                 int32_t mode, int64_t *cand_idx, int64_t *cand_dist,
                                 const ft_host_matches *matches) {
    if (!s || !left || !right || !params) return FT_E_NULL;
    const int64_t n = left->n, nr = right->n;
    if (n < 0 || nr < 0) return FT_E_RANGE;
    if (n == 0) return FT_OK;
    const bool p1 = mode & FT_STEREO_PHASE1, ref = mode & FT_STEREO_REFINE;
    const bool fin = ref || (mode & FT_STEREO_FROM_CAND);
    const bool rej_only = (mode & FT_STEREO_REJECT) && !fin && !p1;
    if (!p1 && !fin && !rej_only) return FT_E_CONFIG;
    if (ref && (!left_pyr || !right_pyr || !left_pyr->data || !right_pyr->data)) return FT_E_NULL;
    if (p1 && !fin && (!cand_idx || !cand_dist)) return FT_E_NULL;  // phase-1 outputs
    if (!p1 && fin && (!cand_idx || !cand_dist)) return FT_E_NULL;  // candidate inputs
    if ((fin || rej_only) && !matches) return FT_E_NULL;
    if ((p1 || ref) && (!left->u || !left->v || !left->octave || !left->desc))
        return FT_E_NULL;
    if ((p1 || ref) && nr && (!right->u || !right->v || !right->octave || !right->desc))
        return FT_E_NULL;
    if (ref && (left_pyr->n_levels < 1 || left_pyr->n_levels > FT_MAX_LEVELS ||
                right_pyr->n_levels != left_pyr->n_levels))
        return FT_E_RANGE;
    cudaSetDevice(s->device);
    FT_TRY(caps(s, std::max(n, nr), 0));
    const int cap = s->cap_kp;
    // Layout [right pyramid | small inputs | left pyramid, levels L-1..0]:
    // phase 2 reads levels >= the lowest left octave m of both images, so
    // the bytes a call needs -- the right pyramid's tail, the small inputs,
    // the left pyramid's first levels (reversed) -- are ONE contiguous H2D
    // (each copy costs ~3.6 us of fixed DMA setup; r2d_pcie_copies).
    Lay L;
    size_t o_pl = 0, o_pr = 0, pl_bytes = 0, pr_bytes = 0;
    if (ref) {
        pl_bytes = (size_t)left_pyr->offsets[left_pyr->n_levels];
        pr_bytes = (size_t)right_pyr->offsets[right_pyr->n_levels];
        // the right region ends exactly where the small inputs start
        const size_t pad = (SALIGN - pr_bytes % SALIGN) % SALIGN;
        o_pr = L.add(pr_bytes + pad) + pad;
    }
    const size_t o_ln = L.add(4), o_lr = L.add(64 * (size_t)cap);
    const size_t o_rn = L.add(4), o_rr = L.add(64 * (size_t)cap);
    const size_t o_cand = L.add(16 * (size_t)cap);  // cand_idx | cand_dist
    const size_t small_end = L.total;
    if (ref) o_pl = L.add(pl_bytes);
    const size_t o_out = L.add(48 * (size_t)cap);  // right_idx distance disparity refined_u depth sad
    const size_t o_nm = L.add(4);
    FT_TRY(reserve(s, L.total));
    Phases ph(s, "ft_session_stereo");
    char *h = s->h;
    *reinterpret_cast<int32_t *>(h + o_ln) = (int32_t)n;
    *reinterpret_cast<int32_t *>(h + o_rn) = (int32_t)nr;
    if (!rej_only) {
        pack_kp(left, reinterpret_cast<ft_kp_record *>(h + o_lr));
        pack_kp(right, reinterpret_cast<ft_kp_record *>(h + o_rr));
    }
    int64_t *hc = reinterpret_cast<int64_t *>(h + o_cand);
    if (!p1 && fin) {
        memcpy(hc, cand_idx, 8 * n);
        memcpy(hc + cap, cand_dist, 8 * n);
    }
    size_t out_in = 0;  // bytes of the output area uploaded (REJECT-only input)
    if (rej_only) {
        char *o = h + o_out;
        memcpy(o + 0 * 8 * (size_t)cap, matches->right_idx, 8 * n);
        memcpy(o + 1 * 8 * (size_t)cap, matches->distance, 8 * n);
        memcpy(o + 2 * 8 * (size_t)cap, matches->disparity, 8 * n);
        memcpy(o + 3 * 8 * (size_t)cap, matches->refined_u, 8 * n);
        memcpy(o + 4 * 8 * (size_t)cap, matches->depth, 8 * n);
        memcpy(o + 5 * 8 * (size_t)cap, matches->sad, 8 * n);
        out_in = 48 * (size_t)cap;
    }
    int64_t b0r = 0;
    size_t left_tail = 0;
    int64_t lrev[FT_MAX_LEVELS + 1] = {0};  // left level l at o_pl + lrev[l]
    if (ref) {  // only the levels phase 2 reads (>= m)
        const int nl = left_pyr->n_levels;
        int m = nl - 1;
        for (int64_t i = 0; i < n && m > 0; ++i)
            m = std::min(m, std::max(0, std::min(left->octave[i], nl - 1)));
        int64_t acc = 0;
        for (int l = nl - 1; l >= 0; --l) {
            lrev[l] = acc;
            acc += left_pyr->offsets[l + 1] - left_pyr->offsets[l];
        }
        for (int l = m; l < nl; ++l)
            memcpy(h + o_pl + lrev[l], left_pyr->data + left_pyr->offsets[l],
                   left_pyr->offsets[l + 1] - left_pyr->offsets[l]);
        left_tail = (size_t)(lrev[m] + left_pyr->offsets[m + 1] - left_pyr->offsets[m]);
        b0r = right_pyr->offsets[std::min(m, right_pyr->n_levels - 1)];
        memcpy(h + o_pr + b0r, right_pyr->data + b0r, pr_bytes - b0r);
    }
    ph.mark(0);
    if (ref)  // right tail | small | left head: one copy
        FT_TRY(h2d(s, o_pr + b0r, o_pl + left_tail - (o_pr + b0r)));
    else
        FT_TRY(h2d(s, o_ln, (rej_only ? o_rn + 4 : small_end) - o_ln));
    if (out_in) FT_TRY(h2d(s, o_out, out_in));
    ft_keypoints kl{reinterpret_cast<const ft_kp_record *>(s->d + o_lr),
                    reinterpret_cast<const int32_t *>(s->d + o_ln), cap};
    ft_keypoints kr{reinterpret_cast<const ft_kp_record *>(s->d + o_rr),
                    reinterpret_cast<const int32_t *>(s->d + o_rn), cap};
    ft_pyramid pl, pr;
    if (ref) {
        pl = dev_pyramid(left_pyr, reinterpret_cast<const uint8_t *>(s->d + o_pl));
        for (int l = 0; l < left_pyr->n_levels; ++l) pl.offsets[l] = lrev[l];  // reversed levels
        pr = dev_pyramid(right_pyr, reinterpret_cast<const uint8_t *>(s->d + o_pr));
    }
    int64_t *dc = reinterpret_cast<int64_t *>(s->d + o_cand);
    char *dout = s->d + o_out;
    ft_stereo_out so;
    so.cand_idx = dc;
    so.cand_dist = dc + cap;
    so.right_idx = reinterpret_cast<int64_t *>(dout);
    so.distance = reinterpret_cast<int64_t *>(dout + 8 * (size_t)cap);
    so.disparity = reinterpret_cast<double *>(dout + 16 * (size_t)cap);
    so.refined_u = reinterpret_cast<double *>(dout + 24 * (size_t)cap);
    so.depth = reinterpret_cast<double *>(dout + 32 * (size_t)cap);
    so.sad = reinterpret_cast<int64_t *>(dout + 40 * (size_t)cap);
    so.n_matched = reinterpret_cast<int32_t *>(s->d + o_nm);
    ph.kernel_begin();
    FT_TRY(ft_stereo_pinhole(1, &kl, &kr, ref ? &pl : nullptr, ref ? &pr : nullptr, params, mode,
                             &so, &s->ws, s->stream));
    ph.kernel_end();
    const bool want_cand = p1 && cand_idx && cand_dist;
    const bool want_m = fin || rej_only;
    if (want_cand) FT_TRY(d2h(s, o_cand, 16 * (size_t)cap));
    if (want_m) FT_TRY(d2h(s, o_out, 48 * (size_t)cap));
    ph.mark(1);
    const cudaError_t e = cudaStreamSynchronize(s->stream);
    if (e != cudaSuccess) return (int)e;
    ph.mark(3);
    if (want_cand) {
        memcpy(cand_idx, hc, 8 * n);
        memcpy(cand_dist, hc + cap, 8 * n);
    }
    if (want_m) {
        const char *o = h + o_out;
        memcpy(matches->right_idx, o + 0 * 8 * (size_t)cap, 8 * n);
        memcpy(matches->distance, o + 1 * 8 * (size_t)cap, 8 * n);
        memcpy(matches->disparity, o + 2 * 8 * (size_t)cap, 8 * n);
        memcpy(matches->refined_u, o + 3 * 8 * (size_t)cap, 8 * n);
        memcpy(matches->depth, o + 4 * 8 * (size_t)cap, 8 * n);
        memcpy(matches->sad, o + 5 * 8 * (size_t)cap, 8 * n);
    }
    ph.mark(4);
    ph.done();
    return FT_OK;
}

extern "C" int ft_session_project(ft_session *s, const ft_host_points *points,
                                  const ft_point_record *table, int64_t table_size,
                                  const int32_t *table_index, const ft_host_features *frame,
                                  const ft_project_params *params, const double *rot,
                                  const double *trans, const uint8_t *skip,
                                  const double *ref_angles, const int64_t *slots_in,
                                  int32_t mode, const ft_host_project_out *out) {
    if (!s || !points || !frame || !params || !rot || !trans || !out) return FT_E_NULL;
    const int64_t m = points->m, n_kp = frame->n;
    if (m < 0 || n_kp < 0) return FT_E_RANGE;
    if (table && m && !table_index) return FT_E_NULL;
    if (!table && m && (!points->positions || !points->normals || !points->min_dist ||
                        !points->max_dist || !points->desc))
        return FT_E_NULL;
    if ((mode & (FT_PROJ_SKIP_SLOTS | FT_PROJ_WRITE_SLOTS)) && n_kp && !slots_in) return FT_E_NULL;
    cudaSetDevice(s->device);
    FT_TRY(caps(s, n_kp, m));
    const int ck = s->cap_kp, cp = s->cap_pts;
    Lay L;
    const size_t o_kn = L.add(4), o_kr = L.add(64 * (size_t)ck);
    const size_t o_pn = L.add(4);
    const size_t o_pr = table ? L.add(4 * (size_t)cp) : L.add(112 * (size_t)cp);
    const size_t o_rot = L.add(96);  // rot[9] | trans[3]
    const size_t o_skip = skip ? L.add((size_t)cp) : 0;
    const size_t o_ref = ref_angles ? L.add(8 * (size_t)cp) : 0;
    // the counts sit right before the slots, so the slot read-back and the
    // counts are ONE D2H (the kernel zeroes the counts itself)
    const size_t o_cnt = L.add(8);                                 // corr_count, slot_count
    const size_t o_sl = slots_in ? L.add(8 * (size_t)ck) : 0;
    const size_t in_end = L.total;
    const bool pa = out->out_kp || out->out_dist || out->out_oct;
    const size_t o_pa = pa ? L.add(24 * (size_t)cp) : 0;           // out_kp | dist | oct
    const size_t o_c = L.add(32 * (size_t)cp);                     // corr point | kp | dist | oct
    FT_TRY(reserve(s, L.total));
    Phases ph(s, "ft_session_project");
    char *h = s->h;
    *reinterpret_cast<int32_t *>(h + o_kn) = (int32_t)n_kp;
    pack_kp(frame, reinterpret_cast<ft_kp_record *>(h + o_kr));
    *reinterpret_cast<int32_t *>(h + o_pn) = (int32_t)m;
    if (table) {
        memcpy(h + o_pr, table_index, 4 * m);
    } else {
        pack_points(points, reinterpret_cast<ft_point_record *>(h + o_pr));
    }
    memcpy(h + o_rot, rot, 72);
    memcpy(h + o_rot + 72, trans, 24);
    if (skip) memcpy(h + o_skip, skip, m);
    if (ref_angles) memcpy(h + o_ref, ref_angles, 8 * m);
    if (slots_in) memcpy(h + o_sl, slots_in, 8 * n_kp);
    ph.mark(0);
    FT_TRY(h2d(s, 0, in_end));
    char *d = s->d;
    ft_keypoints K{reinterpret_cast<const ft_kp_record *>(d + o_kr),
                   reinterpret_cast<const int32_t *>(d + o_kn), ck};
    ft_map_points P;
    P.count = reinterpret_cast<const int32_t *>(d + o_pn);
    P.cap = cp;
    if (table) {
        P.rec = table;
        P.index = reinterpret_cast<const int32_t *>(d + o_pr);
    } else {
        P.rec = reinterpret_cast<const ft_point_record *>(d + o_pr);
        P.index = nullptr;
    }
    ft_project_io io;
    io.rot = reinterpret_cast<const double *>(d + o_rot);
    io.trans = reinterpret_cast<const double *>(d + o_rot + 72);
    io.skip = skip ? reinterpret_cast<const uint8_t *>(d + o_skip) : nullptr;
    io.ref_angles = ref_angles ? reinterpret_cast<const double *>(d + o_ref) : nullptr;
    io.slots_in = slots_in ? reinterpret_cast<const int64_t *>(d + o_sl) : nullptr;
    io.slots_out = slots_in ? reinterpret_cast<int64_t *>(d + o_sl) : nullptr;
    ft_project_out po;
    memset(&po, 0, sizeof(po));
    if (pa) {
        po.out_kp = reinterpret_cast<int64_t *>(d + o_pa);
        po.out_dist = po.out_kp + cp;
        po.out_oct = po.out_kp + 2 * (size_t)cp;
    }
    // ordered correspondences only when the caller wants them (search_local_points
    // needs the slots and the count: the kernel then skips the ordered-output pass)
    const bool want_c = (mode & FT_PROJ_RESOLVE) && out->corr_point;
    int64_t *dc = reinterpret_cast<int64_t *>(d + o_c);
    if (want_c) {
        po.corr_point = dc;
        po.corr_kp = dc + cp;
        po.corr_dist = dc + 2 * (size_t)cp;
        po.corr_oct = dc + 3 * (size_t)cp;
    }
    po.corr_count = reinterpret_cast<int32_t *>(d + o_cnt);
    po.slot_count = reinterpret_cast<int32_t *>(d + o_cnt + 4);
    if (table) {  // slot range check is the gather's; here the kernel reads in place
        for (int64_t i = 0; i < m; ++i)
            if (table_index[i] < 0 || table_index[i] >= table_size) return FT_E_RANGE;
    }
    ph.kernel_begin();
    FT_TRY(ft_project_search(1, &P, &K, params, &io, mode, &po, &s->ws, s->stream));
    ph.kernel_end();
    if (pa) FT_TRY(d2h(s, o_pa, 24 * (size_t)cp));
    if (want_c) FT_TRY(d2h(s, o_c, 32 * (size_t)cp));
    if (slots_in && out->slots_out)  // counts + slots
        FT_TRY(d2h(s, o_cnt, o_sl + 8 * (size_t)n_kp - o_cnt));
    else
        FT_TRY(d2h(s, o_cnt, 8));
    ph.mark(1);
    const cudaError_t e = cudaStreamSynchronize(s->stream);
    if (e != cudaSuccess) return (int)e;
    ph.mark(3);
    if (pa) {
        const int64_t *a = reinterpret_cast<const int64_t *>(h + o_pa);
        if (out->out_kp) memcpy(out->out_kp, a, 8 * m);
        if (out->out_dist) memcpy(out->out_dist, a + cp, 8 * m);
        if (out->out_oct) memcpy(out->out_oct, a + 2 * (size_t)cp, 8 * m);
    }
    const int32_t cc = *reinterpret_cast<const int32_t *>(h + o_cnt);
    const int32_t sc = *reinterpret_cast<const int32_t *>(h + o_cnt + 4);
    if (out->corr_count) *out->corr_count = (mode & FT_PROJ_RESOLVE) ? cc : 0;
    if (out->slot_count) *out->slot_count = sc;
    if (want_c) {
        const int64_t *c = reinterpret_cast<const int64_t *>(h + o_c);
        memcpy(out->corr_point, c, 8 * (size_t)cc);
        memcpy(out->corr_kp, c + cp, 8 * (size_t)cc);
        memcpy(out->corr_dist, c + 2 * (size_t)cp, 8 * (size_t)cc);
        memcpy(out->corr_oct, c + 3 * (size_t)cp, 8 * (size_t)cc);
    }
    if (slots_in && out->slots_out) memcpy(out->slots_out, h + o_sl, 8 * n_kp);
    ph.mark(4);
    ph.done();
    return FT_OK;
}

extern "C" int ft_session_fisheye(ft_session *s, const ft_host_features *left,
                                  const ft_host_features *right, int32_t t_match, double ratio,
                                  const ft_fisheye_tri *tri, int64_t *out_idx, int64_t *out_dist,
                                  int32_t *out_ok, double *out_points) {
    if (!s || !left || !right || !out_idx || !out_dist) return FT_E_NULL;
    if (tri && (!out_ok || !out_points)) return FT_E_NULL;
    const int64_t n = left->n, nr = right->n;
    if (n < 0 || nr < 0) return FT_E_RANGE;
    if (n == 0) return FT_OK;
    cudaSetDevice(s->device);
    FT_TRY(caps(s, std::max(n, nr), 0));
    const int cap = s->cap_kp;
    Lay L;
    const size_t o_ln = L.add(4), o_lr = L.add(64 * (size_t)cap);
    const size_t o_rn = L.add(4), o_rr = L.add(64 * (size_t)cap);
    const size_t in_end = L.total;
    const size_t o_idx = L.add(16 * (size_t)cap);  // idx | dist
    const size_t o_ok = L.add(4 * (size_t)cap);
    const size_t o_pts = L.add(24 * (size_t)cap);
    FT_TRY(reserve(s, L.total));
    char *h = s->h;
    *reinterpret_cast<int32_t *>(h + o_ln) = (int32_t)n;
    *reinterpret_cast<int32_t *>(h + o_rn) = (int32_t)nr;
    pack_kp(left, reinterpret_cast<ft_kp_record *>(h + o_lr));
    pack_kp(right, reinterpret_cast<ft_kp_record *>(h + o_rr));
    FT_TRY(h2d(s, 0, in_end));
    char *d = s->d;
    ft_keypoints kl{reinterpret_cast<const ft_kp_record *>(d + o_lr),
                    reinterpret_cast<const int32_t *>(d + o_ln), cap};
    ft_keypoints kr{reinterpret_cast<const ft_kp_record *>(d + o_rr),
                    reinterpret_cast<const int32_t *>(d + o_rn), cap};
    int64_t *di = reinterpret_cast<int64_t *>(d + o_idx);
    if (tri)
        FT_TRY(ft_stereo_fisheye(1, &kl, &kr, t_match, ratio, tri, di, di + cap,
                                 reinterpret_cast<int32_t *>(d + o_ok),
                                 reinterpret_cast<double *>(d + o_pts), &s->ws, s->stream));
    else
        FT_TRY(ft_stereo_fisheye_bf(1, &kl, &kr, t_match, ratio, di, di + cap, &s->ws, s->stream));
    FT_TRY(d2h(s, o_idx, 16 * (size_t)cap));
    if (tri) FT_TRY(d2h(s, o_ok, o_pts - o_ok + 24 * (size_t)n));
    const cudaError_t e = cudaStreamSynchronize(s->stream);
    if (e != cudaSuccess) return (int)e;
    const int64_t *hi = reinterpret_cast<const int64_t *>(h + o_idx);
    memcpy(out_idx, hi, 8 * n);
    memcpy(out_dist, hi + cap, 8 * n);
    if (tri) {
        memcpy(out_ok, h + o_ok, 4 * n);
        memcpy(out_points, h + o_pts, 24 * n);
    }
    return FT_OK;
}

extern "C" int ft_session_update_local_map(ft_session *s, const int64_t *slots, int64_t n_slots,
                                           const ft_world_dev *world, int64_t out_cap,
                                           int32_t *kf_out, int64_t *point_out,
                                           int32_t *slot_out, int32_t *counts) {
    if (!s || !world || !counts || !kf_out || !point_out || (n_slots > 0 && !slots))
        return FT_E_NULL;
    if (n_slots < 0 || out_cap < 0 || world->n_kf < 0) return FT_E_RANGE;
    cudaSetDevice(s->device);
    Lay L;
    const size_t o_sl = L.add(8 * (size_t)n_slots);
    const size_t o_cnt = L.add(16);
    const size_t o_kf = L.add(4 * (size_t)std::max<int64_t>(world->n_kf, 1));
    const size_t o_pt = L.add(8 * (size_t)std::max<int64_t>(world->id_cap, 1));
    const size_t o_ps = L.add(4 * (size_t)std::max<int64_t>(world->id_cap, 1));
    FT_TRY(reserve(s, L.total));
    Phases ph(s, "ft_session_update_local_map");
    if (n_slots) memcpy(s->h + o_sl, slots, 8 * n_slots);
    ph.mark(0);
    FT_TRY(h2d(s, o_sl, 8 * (size_t)n_slots));
    char *d = s->d;
    ph.kernel_begin();
    FT_TRY(ft_update_local_map(reinterpret_cast<const int64_t *>(d + o_sl), (int32_t)n_slots,
                               world->kf_obs, world->kf_off, world->n_kf, world->id_slot,
                               world->id_cap, reinterpret_cast<int32_t *>(d + o_kf),
                               reinterpret_cast<int64_t *>(d + o_pt),
                               slot_out ? reinterpret_cast<int32_t *>(d + o_ps) : nullptr,
                               reinterpret_cast<int32_t *>(d + o_cnt), s->stream));
    ph.kernel_end();
    // outputs up to out_cap entries in the same round trip; more -> FT_E_RANGE
    // with the counts set (the caller retries with bigger buffers)
    const size_t np = (size_t)std::min<int64_t>(out_cap, world->id_cap);
    const size_t nk = (size_t)std::min<int64_t>(out_cap, world->n_kf);
    FT_TRY(d2h(s, o_cnt, 16));
    FT_TRY(d2h(s, o_kf, 4 * nk));
    FT_TRY(d2h(s, o_pt, 8 * np));
    if (slot_out) FT_TRY(d2h(s, o_ps, 4 * np));
    ph.mark(1);
    const cudaError_t e = cudaStreamSynchronize(s->stream);
    if (e != cudaSuccess) return (int)e;
    ph.mark(3);
    const int32_t *c = reinterpret_cast<const int32_t *>(s->h + o_cnt);
    counts[0] = c[0];
    counts[1] = c[1];
    counts[2] = c[2];
    if (c[2]) return FT_E_RANGE;  // a slotted id outside the world
    if ((size_t)c[0] > nk || (size_t)c[1] > np) return FT_E_RANGE;
    memcpy(kf_out, s->h + o_kf, 4 * (size_t)c[0]);
    memcpy(point_out, s->h + o_pt, 8 * (size_t)c[1]);
    if (slot_out) memcpy(slot_out, s->h + o_ps, 4 * (size_t)c[1]);
    ph.mark(4);
    ph.done();
    return FT_OK;
}
