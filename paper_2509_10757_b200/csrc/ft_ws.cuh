// ft_ws.cuh -- workspace layout shared by the C-ABI entries (host side).
//
// Sections (disjoint; offsets depend only on the workspace's own F / caps,
// so any launch with F <= ws.n_frames and capacities <= the workspace's may
// use it, and the stereo and projection entries may run concurrently):
//   stereo   counters u32[F]
//   fisheye  counters u32[F * tiles(cap_left)] | partials uint2[fisheye_entries]
//   project  claims u64[F * cap_left]
//   track    barrier counters u64[F] (stereo) | u64[F] (map) | epoch counters
//            u64[F] | per-block counts i32[F * WS_MAX_GROUP] | hist i32[F * 256]
//   pyramid  barrier counters u64[2F]
// Counters start at 0 and claims at ~0 (ft_workspace_init).  Barrier and
// epoch counters only grow; claims carry the launch epoch in their high word,
// so no kernel has to reset anything.
#pragma once

#include <stddef.h>
#include <stdint.h>

#include "../../include/fasttrack_b200.h"

namespace ft {

constexpr size_t WS_ALIGN = 256;
constexpr int WS_BF_TL = 128;   // fisheye left tile (ft_fisheye.cu)
constexpr int WS_MAX_GROUP = 1024;  // max map blocks per frame (ft_track.cu)
constexpr int WS_SM_HINT = 148;

inline size_t ws_align(size_t x) { return (x + WS_ALIGN - 1) & ~(WS_ALIGN - 1); }
inline int ws_tiles(int cap_left) { return (cap_left + WS_BF_TL - 1) / WS_BF_TL; }

// Right-set splits of the fisheye all-pairs kernel: about 4 blocks per SM.
inline int fisheye_splits(int F, int cap_left, int cap_right) {
    const int tiles = ws_tiles(cap_left);
    int s = (4 * WS_SM_HINT + tiles * F - 1) / (tiles * F);
    const int max_s = (cap_right + 63) / 64;
    if (s > max_s) s = max_s;
    return s < 1 ? 1 : s;
}

inline size_t fisheye_entries(int F, int cap_left) {
    size_t e = (size_t)F * cap_left * fisheye_splits(F, cap_left, 65535);
    const size_t floor_e = (size_t)F * cap_left * 8;
    return e > floor_e ? e : floor_e;
}

// SAD-median histogram buffer of one stereo group (ft_track.cu): coarse bins
// of MED_CW values over [0, MED_FINE) + one overflow bin, padded to 128
// words, then the fine (one bin per value) histogram.
constexpr int MED_FINE = 4096, MED_CW = 64, MED_NC = MED_FINE / MED_CW;
constexpr int MED_WS = 128 + MED_FINE;

struct WsLayout {
    size_t stereo_counters, fisheye_counters, fisheye_partials, proj_claims, track_bar_s,
        track_bar_m, track_ep_m, track_ep_s, track_tail_s, track_tail_m, track_mcand,
        track_mcnt, track_med, track_blk_counts, track_hist, pyr_bar, total;
    size_t fisheye_partial_entries;
};

inline WsLayout ws_layout(int F, int cap_left, int cap_points) {
    WsLayout L;
    size_t o = 0;
    L.stereo_counters = o;
    o += ws_align((size_t)F * 4);
    L.fisheye_counters = o;
    o += ws_align((size_t)F * ws_tiles(cap_left) * 4);
    L.fisheye_partials = o;
    L.fisheye_partial_entries = fisheye_entries(F, cap_left);
    o += ws_align(L.fisheye_partial_entries * 8);
    L.proj_claims = o;
    o += ws_align((size_t)F * cap_left * 8);
    L.track_bar_s = o;  // two barrier words per group (group_barrier)
    o += ws_align((size_t)F * 16);
    L.track_bar_m = o;
    o += ws_align((size_t)F * 16);
    L.track_ep_m = o;
    o += ws_align((size_t)F * 8);
    L.track_ep_s = o;
    o += ws_align((size_t)F * 8);
    L.track_tail_s = o;
    o += ws_align((size_t)F * 8);
    L.track_tail_m = o;
    o += ws_align((size_t)F * 8);
    L.track_mcand = o;  // map resolve candidates (tail mode), 16 B per point
    o += ws_align((size_t)F * cap_points * 16);
    L.track_mcnt = o;
    o += ws_align((size_t)F * WS_MAX_GROUP * 8);
    L.track_med = o;  // SAD-median histograms: 3 rotating buffers per stereo group
    o += ws_align((size_t)F * 3 * MED_WS * 4);
    L.track_blk_counts = o;
    o += ws_align((size_t)F * WS_MAX_GROUP * 4);
    L.track_hist = o;
    o += ws_align((size_t)F * 256 * 4);
    L.pyr_bar = o;  // two images (left, right) per frame, two words each
    o += ws_align((size_t)F * 2 * 16);
    L.total = o;
    return L;
}

// Validates a workspace against a launch; returns FT_OK or an FT_E code.
inline int ws_check(const ft_workspace *ws, int F, int cap_left, int cap_points) {
    if (!ws || !ws->base) return FT_E_NULL;
    if (ws->n_frames < 1 || ws->cap_left < 1 || ws->cap_points < 1) return FT_E_RANGE;
    if (F > ws->n_frames || cap_left > ws->cap_left || cap_points > ws->cap_points)
        return FT_E_WORKSPACE;
    if (ws->bytes < ws_layout(ws->n_frames, ws->cap_left, ws->cap_points).total)
        return FT_E_WORKSPACE;
    return FT_OK;
}

template <typename T>
inline T *ws_ptr(const ft_workspace *ws, size_t off) {
    return reinterpret_cast<T *>(static_cast<char *>(ws->base) + off);
}

inline WsLayout ws_layout(const ft_workspace *ws) {
    return ws_layout(ws->n_frames, ws->cap_left, ws->cap_points);
}

}  // namespace ft
