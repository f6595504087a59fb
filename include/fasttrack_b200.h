/*
 * fasttrack_b200.h -- C ABI of the B200 tracking hot path.
 *
 * One entry point per reference stage function (reference = trackfront,
 * pkg/src/trackfront).  Every entry:
 *   - takes DEVICE pointers, plain sizes and a POD parameter struct,
 *   - enqueues kernels on `stream` (a cudaStream_t) and returns without
 *     synchronising,
 *   - allocates nothing: scratch lives in a caller-provided ft_workspace
 *     (size from ft_workspace_bytes(), initialised once by ft_workspace_init();
 *     launches may use any F / capacities up to the workspace's),
 *   - returns 0 on success, a negative FT_E* code for argument errors, or a
 *     positive cudaError_t from the launch.
 *
 * Batched layout: every entry processes F independent frames ("frame
 * streams") in one launch.  Frame f's items live at [f * cap, f * cap + n_f)
 * of each array; the per-frame counts n_f are read from DEVICE memory, so a
 * CUDA graph captured once replays every frame with new counts.
 *
 * Inputs are packed records (ft_kp_record, ft_point_record): a frame's table
 * is staged into shared memory with ONE TMA bulk copy.  ft_pack_keypoints /
 * ft_pack_points build them from the reference's SoA arrays (FeatureSet /
 * MapPointSoA) on the device.  Descriptors are 256-bit ORB strings, bit b in
 * 64-bit word b >> 6 at bit b & 63 (reference descriptors.py:7-9,23-30).
 *
 * Alignment: record arrays must be 16-byte aligned and capacities even
 * (FT_E_RANGE otherwise).
 *
 * Reference interface each entry replaces:
 *   ft_hamming_pairs        kernels.py:48-51        hamming_pairs_kernel
 *   ft_stereo_pinhole       stereo.py:77-188        match_pinhole_phase1 ->
 *                                                   refine_match_phase2 |
 *                                                   matches_from_candidates ->
 *                                                   reject_outliers
 *                           (also tracker.py:415-427 _run_stereo, pinhole branch)
 *   ft_stereo_fisheye_bf    stereo.py:238-244       bruteforce_match_kernel as
 *                                                   launched by match_fisheye
 *   ft_stereo_fisheye       stereo.py:223-273       match_fisheye: brute force +
 *                                                   ray triangulation (cameras.py
 *                                                   :139-157 unproject, stereo.py
 *                                                   :200-220 closest points)
 *   ft_track_frames         tracker.py:279 + :354   stereo + SearchLocalPoints fused
 *   ft_build_pyramids       extraction.py:97-125    build_pyramid
 *   ft_gather_points /      mapping.py:204-235      decompose_map_points (per-frame
 *   ft_scatter_points                               local map from a resident table)
 *   ft_project_search       projection.py:118-221   run_phase_a ->
 *                                                   resolve_conflicts ->
 *                                                   rotation_consistency_filter
 *                           localmap.py:79-122      search_local_points (skip mask,
 *                                                   slot write, filled count)
 */
#ifndef FASTTRACK_B200_H
#define FASTTRACK_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FT_ABI_VERSION 1
#define FT_MAX_LEVELS 16

enum {
    FT_OK = 0,
    FT_E_NULL = -1,       /* required pointer is NULL */
    FT_E_RANGE = -2,      /* size / capacity / level count out of range */
    FT_E_WORKSPACE = -3,  /* workspace too small */
    FT_E_CONFIG = -4,     /* invalid parameter value */
    FT_E_TIMEOUT = -5     /* persistent runner: a step did not complete within 20 s */
};

typedef void *ft_stream_t; /* cudaStream_t */

/* Device scratch shared by all entries.  Sections are disjoint, so the
 * stereo and projection entries may run concurrently on two streams. */
typedef struct {
    void *base;
    size_t bytes;
    int32_t n_frames;    /* max frames per launch */
    int32_t cap_left;    /* max keypoints per frame (left or right) */
    int32_t cap_points;  /* max map points per frame */
} ft_workspace;

/* One keypoint, packed (64 B) so a frame's table is one contiguous TMA copy.
 * Fields are the reference FeatureSet's (mapping.py:18-65). */
typedef struct {
    double u;            /* level-0 column */
    double v;            /* level-0 row */
    uint64_t desc[4];    /* 256-bit descriptor (descriptors.py:23-30 bit order) */
    double angle;        /* orientation (rad), rotation check only */
    int32_t octave;      /* pyramid level */
    int32_t pad;
} ft_kp_record;

/* Keypoints of one image side, F frames at stride `cap` records. */
typedef struct {
    const ft_kp_record *rec;  /* [F*cap] */
    const int32_t *count;     /* DEVICE [F] keypoints per frame */
    int32_t cap;              /* per-frame stride (>= every count) */
} ft_keypoints;

/* Flat u8 image pyramid, F frames at stride `frame_bytes`
 * (reference extraction.py:67-94 ImagePyramid).  Level geometry is shared by
 * all frames and passed by value. */
typedef struct {
    const uint8_t *data;
    int64_t frame_bytes;
    int32_t n_levels;
    int64_t offsets[FT_MAX_LEVELS];
    int32_t widths[FT_MAX_LEVELS];
    int32_t heights[FT_MAX_LEVELS];
} ft_pyramid;

/* reference stereo.py:22-42 StereoMatchConfig + camera terms used. */
typedef struct {
    int32_t t_match;
    double band_factor;
    double min_disparity;
    double max_disparity;
    int32_t half_window;
    int32_t half_slide;
    double outlier_multiplier;
    double ratio;               /* fisheye ratio test */
    double baseline_times_fx;   /* depth = bf / disparity (stereo.py:131-132) */
    int32_t height;             /* image rows: row-bucket count (stereo.py:88) */
    int32_t n_levels;
    double scale_pow[FT_MAX_LEVELS]; /* scale ** arange(levels), host-computed */
} ft_stereo_params;

/* ft_stereo_pinhole mode bits */
#define FT_STEREO_PHASE1 0x1      /* run phase 1 (else read cand_idx/cand_dist) */
#define FT_STEREO_REFINE 0x2      /* phase 2 SAD refinement (needs pyramids) */
#define FT_STEREO_FROM_CAND 0x4   /* matches_from_candidates (no images) */
#define FT_STEREO_REJECT 0x8      /* reject_outliers (median SAD) */

/* Per-left-keypoint outputs at stride cap_left
 * (reference stereo.py:45-64 StereoMatches). */
typedef struct {
    int64_t *cand_idx;   /* phase-1 output / input when !PHASE1 */
    int64_t *cand_dist;
    int64_t *right_idx;  /* may be NULL in phase-1-only mode */
    int64_t *distance;
    double *disparity;
    double *refined_u;
    double *depth;
    int64_t *sad;
    int32_t *n_matched;  /* DEVICE [F] matches after rejection; may be NULL */
} ft_stereo_out;

/* One map point, packed (112 B) (reference mapping.py:163-201 MapPointSoA). */
typedef struct {
    uint64_t desc[4];    /* representative descriptor */
    double pos[3];       /* world position */
    double nrm[3];       /* mean viewing direction */
    double min_dist;
    double max_dist;
    int64_t id;          /* point id; ascending per frame (LocalMap contract) */
    int64_t pad;
} ft_point_record;

/* Map points of F local maps at stride `cap` records.  With `index` NULL,
 * point i of frame f is rec[f*cap + i]; otherwise rec is a resident map
 * table (ft_gather_points) and point i of frame f is rec[index[f*cap + i]]
 * -- read in place, no per-frame copy. */
typedef struct {
    const ft_point_record *rec;  /* [F*cap], or the table */
    const int32_t *count;        /* DEVICE [F] */
    int32_t cap;
    const int32_t *index;        /* DEVICE [F*cap] table slots, or NULL */
} ft_map_points;

/* reference projection.py:26-45 ProjectionSearchConfig + camera + grid. */
typedef struct {
    int32_t cam_kind;      /* 0 pinhole, 1 Kannala-Brandt fisheye */
    double fx, fy, cx, cy, k1, k2, k3, k4;
    double width, height;
    int32_t cell_px;       /* FrameGrid cell (mapping.py:15) */
    int32_t grid_nx, grid_ny;
    int32_t n_levels;
    double scale_pow[FT_MAX_LEVELS];
    double inv_log_scale;  /* 1.0 / log(scale), host-computed (projection.py:155) */
    double window_px;
    int32_t t_proj;
    double ratio;
    double view_cos_min;
    double u_offset;
    int32_t histogram_bins;
    int32_t histogram_keep;
} ft_project_params;

/* ft_project_search mode bits */
#define FT_PROJ_RESOLVE 0x1      /* resolve_conflicts -> correspondences */
#define FT_PROJ_ROTATION 0x2     /* rotation_consistency_filter (needs angles) */
#define FT_PROJ_SKIP_SLOTS 0x4   /* skip points whose id is already slotted */
#define FT_PROJ_WRITE_SLOTS 0x8  /* search_local_points slot write + count */

typedef struct {
    const double *rot;          /* DEVICE [F][9] row-major world->camera R */
    const double *trans;        /* DEVICE [F][3] */
    const uint8_t *skip;        /* [F*cap_points] explicit skip mask; may be NULL */
    const double *ref_angles;   /* [F*cap_points] for the rotation check; may be NULL */
    const int64_t *slots_in;    /* [F*cap_kp] frame slots before the search (read by
                                   SKIP_SLOTS and by the "only if empty" rule) */
    int64_t *slots_out;         /* [F*cap_kp] slots after WRITE_SLOTS; may equal
                                   slots_in (in place) */
} ft_project_io;

typedef struct {
    int64_t *out_kp;     /* [F*cap_points] phase A (run_phase_a) */
    int64_t *out_dist;
    int64_t *out_oct;
    int64_t *corr_point; /* [F*cap_points] resolved correspondences, point order */
    int64_t *corr_kp;
    int64_t *corr_dist;
    int64_t *corr_oct;
    int32_t *corr_count; /* DEVICE [F] */
    int32_t *slot_count; /* DEVICE [F] filled slots after WRITE_SLOTS */
} ft_project_out;

/* --- entry points ------------------------------------------------------- */

int ft_abi_version(void);
const char *ft_status_string(int status);

/* Bytes of device workspace for F frames of the given capacities. */
size_t ft_workspace_bytes(int32_t n_frames, int32_t cap_left, int32_t cap_points);

/* Initialise a workspace once after allocation (counters to 0, claims to
 * ~0); every kernel restores that state on exit. */
int ft_workspace_init(const ft_workspace *ws, ft_stream_t stream);

/* extraction.py:97-125 build_pyramid for n_images flat pyramids (image i at
 * pyr->data + i * frame_bytes).  Level 0 comes from `images` (image i at
 * images + i * image_stride; copied into the pyramid) or, when `images` is
 * NULL, is already in place.  Levels 1..L-1 (5x5 binomial, reflect-101,
 * round half up; then fp64 bilinear to floor(dims / scale^l)) are written
 * bit-exact with the reference.  n_images <= 2 * ws->n_frames. */
int ft_build_pyramids(int32_t n_images, const ft_pyramid *pyr, const uint8_t *images,
                      int64_t image_stride, const ft_workspace *ws, ft_stream_t stream);

/* SoA -> packed records for F frames (any pointer but u/v/octave/desc/ids may
 * be NULL: angle -> 0).  Caller-held reference-layout device arrays at
 * stride cap per frame. */
int ft_pack_keypoints(int32_t n_frames, const double *u, const double *v, const int32_t *octave,
                      const double *angle, const uint64_t *desc, const int32_t *count,
                      int32_t cap, ft_kp_record *out, ft_stream_t stream);
int ft_pack_points(int32_t n_frames, const double *positions, const double *normals,
                   const double *min_dist, const double *max_dist, const uint64_t *desc,
                   const int64_t *point_ids, const int32_t *count, int32_t cap,
                   ft_point_record *out, ft_stream_t stream);

/* Device-resident map-point table (north star (1)): the reference rebuilds a
 * frame's LocalMap SoA on the host every frame (mapping.py:204-235,
 * localmap.py:22-39); here every point record lives once in `table` and a
 * frame names its local map as table slots in LocalMap order.
 * ft_gather_points: out[f*cap + i] = table[index[f*cap + i]] for i < count[f]
 *   (the ft_map_points input of ft_track_frames / ft_project_search); an
 *   out-of-range slot sets *status (DEVICE, may be NULL) to FT_E_RANGE.
 * ft_scatter_points: table[slots[i]] = recs[i] -- upload new / changed points
 *   (the per-frame map delta). */
int ft_gather_points(int32_t n_frames, const ft_point_record *table, int64_t table_size,
                     const int32_t *index, const int32_t *count, int32_t cap,
                     ft_point_record *out, int32_t *status, ft_stream_t stream);
int ft_scatter_points(int32_t n, const ft_point_record *recs, const int32_t *slots,
                      ft_point_record *table, int64_t table_size, ft_stream_t stream);

/* Native multi-buffered step executor (csrc/ft_runner.cu): per step k, on
 * three streams, H2D of host_in into slot k % n's device inputs, a launch of
 * that slot's instantiated compute graph (cudaGraphExec_t, captured by the
 * caller), and D2H of its outputs into the slot's pinned host range.
 * Neighbouring steps' copies overlap the compute; computes are serialised.
 * ft_runner_wait(k) blocks until step k's outputs are on the host.  Slot
 * buffers are reused n steps later (the runner orders that itself). */
typedef struct ft_runner ft_runner;
#define FT_RUNNER_MAX_SLOTS 16
int ft_runner_create(const void *const graph_exec[2], void *const dev_in[2], size_t in_bytes,
                     void *const dev_out[2], void *const host_out[2], size_t out_bytes,
                     ft_runner **out);
/* n_slots (2..FT_RUNNER_MAX_SLOTS) buffer sets used round robin (slot k % n). */
int ft_runner_create_n(int32_t n_slots, const void *const *graph_exec, void *const *dev_in,
                       size_t in_bytes, void *const *dev_out, void *const *host_out,
                       size_t out_bytes, ft_runner **out);
int ft_runner_submit(ft_runner *r, int64_t k, const void *host_in);
/* As ft_runner_submit, copying only bytes [offset, offset + bytes) of the
 * step's inputs (the rest of the slot's device inputs is left as is). */
int ft_runner_submit_range(ft_runner *r, int64_t k, const void *host_in, size_t offset,
                           size_t bytes);
/* As ft_runner_submit, copying the n_ranges byte ranges [ranges[2q],
 * ranges[2q+1]) (e.g. the small inputs plus each stream's needed pyramid
 * levels). */
int ft_runner_submit_ranges(ft_runner *r, int64_t k, const void *host_in,
                            const uint64_t *ranges, int32_t n_ranges);
/* Steps k .. k+m-1 (1 <= m <= n_slots) at once: step k+j's inputs are at
 * host_in + j * host_pitch (host_pitch >= the slot input size when m > 1),
 * the same byte ranges for every step.  When the m slots do not wrap and
 * their device inputs sit at one pitch (one arena), each range goes up as ONE
 * strided 2D copy of m rows: the copy engine's fixed cost per copy (~3.6 us,
 * profiles/r3_h2d2d_probe.txt) is paid once per m steps instead of per step
 * (448 KB ranges: 84k -> 99k / 109k per s at m = 2 / 4).  Otherwise it issues
 * the m steps' copies one by one -- same results either way. */
int ft_runner_submit_batch(ft_runner *r, int64_t k, int32_t m, const void *host_in,
                           size_t host_pitch, const uint64_t *ranges, int32_t n_ranges);
int ft_runner_wait(ft_runner *r, int64_t k);
int ft_runner_destroy(ft_runner *r);

/* Persistent runner: instead of a graph launch per step, ONE long-lived
 * ft_track_frames kernel serves the n slots (2..16).  plans[i] holds slot i's
 * launch (ft_track_plan over that slot's device buffers; all slots the same
 * shapes).  The runner's host thread hands a step to the kernel through a
 * pinned, mapped flag once the step's inputs have landed, and issues the
 * step's D2H when the kernel's done flag (also mapped) shows up -- no launch,
 * block scheduling or drain sits between frames.  Submit / wait as above
 * (both drive that hand-off; wait returns FT_E_TIMEOUT after 20 s);
 * ft_runner_destroy finishes every submitted step, then ends the kernel.
 * The plan's grid must leave SMs free (FT_E_RANGE otherwise); other kernels
 * may run beside it on those SMs.  When host_out[i] are page-locked,
 * device-mapped and 16-B aligned (pinned tensors / cudaHostAlloc), the
 * kernel's last block of a step writes the outputs there itself (16-B stores
 * over PCIe, released with done) -- no D2H copy or event per step
 * (e2e 68k -> 71.6k frames/s, one-in-flight latency 55 -> 47 us, r2m);
 * FT_RUNNER_PUSH=0 keeps the copy engine. */
int ft_runner_create_persistent(int32_t n_slots, const void *const *plans, void *const *dev_in,
                                size_t in_bytes, void *const *dev_out, void *const *host_out,
                                size_t out_bytes, ft_runner **out);

/* Packed upload: after one contiguous H2D of a step's needed bytes, place
 * segment i (desc[3i] = source offset, desc[3i+1] = destination offset,
 * desc[3i+2] = length, bytes relative to `base`; desc in DEVICE memory, e.g.
 * uploaded with the segments) at its destination.  Segments must not overlap
 * each other's destinations. */
int ft_copy_ranges(void *base, const int64_t *desc, int32_t n, ft_stream_t stream);

/* kernels.py:48-51: out[i] = popcount(a[i] ^ b[i]) over 256 bits. */
int ft_hamming_pairs(const uint64_t *a, const uint64_t *b, int64_t n, int64_t *out,
                     ft_stream_t stream);

/* stereo.py:77-188 (pinhole). */
int ft_stereo_pinhole(int32_t n_frames, const ft_keypoints *left, const ft_keypoints *right,
                      const ft_pyramid *left_pyr, const ft_pyramid *right_pyr,
                      const ft_stereo_params *params, int32_t mode, const ft_stereo_out *out,
                      const ft_workspace *ws, ft_stream_t stream);

/* stereo.py:238-244 -> kernels.py:434-464 (fisheye brute force + ratio test). */
int ft_stereo_fisheye_bf(int32_t n_frames, const ft_keypoints *left, const ft_keypoints *right,
                         int32_t t_match, double ratio, int64_t *out_idx, int64_t *out_dist,
                         const ft_workspace *ws, ft_stream_t stream);

/* Fisheye triangulation terms (reference FisheyeCamera, cameras.py:100-157,
 * and StereoMatchConfig.ray_gap_ceiling, stereo.py:32).  rot_lr / trans_lr
 * = right_extrinsic.inverse() computed on the host (geometry.py:84-86). */
typedef struct {
    double fx, fy, cx, cy, k1, k2, k3, k4;
    double rot_rl[9], trans_rl[3];   /* left -> right camera (right_extrinsic) */
    double rot_lr[9], trans_lr[3];   /* right -> left camera */
    double ray_gap_ceiling;
    int32_t corrected;  /* 0: the reference's t at stereo.py:216 (its tracker's
                           behaviour); 1: least-squares closest points */
} ft_fisheye_tri;

/* stereo.py:223-273 match_fisheye for F frames: brute force + ratio test as
 * ft_stereo_fisheye_bf, then for every accepted pair the unproject / closest-
 * point triangulation and its gap / positive-depth checks, in the same
 * launch.  Per left keypoint: out_idx / out_dist (brute-force result),
 * out_ok = 1 if the pair survived triangulation (a member of the reference's
 * returned lists), out_points[3k..3k+2] = the left-frame point when ok. */
int ft_stereo_fisheye(int32_t n_frames, const ft_keypoints *left, const ft_keypoints *right,
                      int32_t t_match, double ratio, const ft_fisheye_tri *tri,
                      int64_t *out_idx, int64_t *out_dist, int32_t *out_ok, double *out_points,
                      const ft_workspace *ws, ft_stream_t stream);

/* projection.py:118-221 + localmap.py:79-122. */
int ft_project_search(int32_t n_frames, const ft_map_points *points, const ft_keypoints *frame,
                      const ft_project_params *params, const ft_project_io *io, int32_t mode,
                      const ft_project_out *out, const ft_workspace *ws, ft_stream_t stream);

/* The whole per-frame hot path in ONE cooperative launch: pinhole stereo
 * (ft_stereo_pinhole semantics, `smode`) on left/right and search by
 * projection / SearchLocalPoints (ft_project_search semantics, `pmode`) of
 * `points` into the LEFT keypoints, side by side in block groups.  Mirrors
 * the reference tracker's per-frame calls tracker.py:279 (_run_stereo) and
 * tracker.py:354 (search_local_points). */
int ft_track_frames(int32_t n_frames, const ft_keypoints *left, const ft_keypoints *right,
                    const ft_pyramid *left_pyr, const ft_pyramid *right_pyr,
                    const ft_stereo_params *sparams, int32_t smode, const ft_stereo_out *sout,
                    const ft_map_points *points, const ft_project_params *pparams,
                    const ft_project_io *io, int32_t pmode, const ft_project_out *pout,
                    const ft_workspace *ws, ft_stream_t stream);

/* The launch ft_track_frames would make with these arguments, recorded into
 * caller memory (ft_track_plan_bytes() bytes) instead of launched: the input
 * of ft_runner_create_persistent.  The pointed-to buffers must outlive it. */
size_t ft_track_plan_bytes(void);
int ft_track_plan(int32_t n_frames, const ft_keypoints *left, const ft_keypoints *right,
                  const ft_pyramid *left_pyr, const ft_pyramid *right_pyr,
                  const ft_stereo_params *sparams, int32_t smode, const ft_stereo_out *sout,
                  const ft_map_points *points, const ft_project_params *pparams,
                  const ft_project_io *io, int32_t pmode, const ft_project_out *pout,
                  const ft_workspace *ws, void *plan, size_t plan_bytes);

/* As ft_track_plan, for a persistent launch of `groups` step groups (1..36):
 * the geometry gets 1 / groups of the SMs and the launch runs `groups`
 * disjoint block groups, group g taking steps k = g mod groups -- that many
 * frames in flight at once.  All plans of one launch share `groups`, and the
 * slot count must be a multiple of it (FT_E_CONFIG). */
int ft_track_plan_groups(int32_t n_frames, const ft_keypoints *left, const ft_keypoints *right,
                         const ft_pyramid *left_pyr, const ft_pyramid *right_pyr,
                         const ft_stereo_params *sparams, int32_t smode,
                         const ft_stereo_out *sout, const ft_map_points *points,
                         const ft_project_params *pparams, const ft_project_io *io,
                         int32_t pmode, const ft_project_out *pout, const ft_workspace *ws,
                         int32_t groups, void *plan, size_t plan_bytes);

/* n_steps frames through ONE persistent launch: step k runs plans[k % n_plans]
 * (ft_track_plan records; same shapes), inputs already resident in the
 * plans' buffers, no launch or hand-off between steps (the device-resident
 * form of the persistent runner: a ring of resident frames processed back
 * to back).  Stream-ordered; n_steps < 2^31.  Successive calls share the
 * library's flag / argument buffers and are ordered after one another even
 * across streams.  Each plan's grid must leave 4 SMs free (FT_E_RANGE). */
int ft_track_frames_ring(int32_t n_plans, const void *const *plans, int64_t n_steps,
                         ft_stream_t stream);

/* projection.py:161-178 resolve_conflicts on caller-held phase-A arrays
 * (one frame): correspondences in point order into out->corr_* and
 * out->corr_count[0].  n_kp <= ws->cap_left. */
int ft_resolve_conflicts(int32_t n_points, const int64_t *out_kp, const int64_t *out_dist,
                         const int64_t *out_oct, int32_t n_kp, const ft_project_out *out,
                         const ft_workspace *ws, ft_stream_t stream);

/* projection.py:181-200 rotation_consistency_filter, in place on m
 * correspondences (one frame); kept count into *count. */
int ft_rotation_filter(int32_t m, int64_t *corr_point, int64_t *corr_kp, int64_t *corr_dist,
                       int64_t *corr_oct, const double *ref_angles, const double *kp_angles,
                       int32_t histogram_bins, int32_t histogram_keep, int32_t *count,
                       ft_stream_t stream);

/* Integer-pipe microbenchmark used for the roofline denominator: each thread
 * runs `iters` iterations of 8 independent XOR+POPC chains.  Writes a
 * checksum to *sink so nothing is dead code. */
int ft_bench_popc(int32_t blocks, int32_t threads, int32_t iters, uint32_t *sink,
                  ft_stream_t stream);

/* --- host-array drop-in session (csrc/ft_session.cu) ----------------------
 * The reference stage functions called with HOST arrays -- the fields of the
 * reference's numpy objects, passed in place -- one C call each: pack into
 * pinned staging, H2D, the device entry above, D2H of the requested outputs,
 * synchronise, copy into the caller's arrays.  This is what a ctypes / cffi
 * binding of the reference binds.  A session owns a stream,
 * pinned staging, a device arena and a workspace (grown on demand, reused);
 * one session per tracking thread; calls are synchronous.  n = 0 returns
 * FT_OK without touching the outputs (the caller returns empty results, as
 * the reference does). */
typedef struct ft_session ft_session;

/* reference FeatureSet (mapping.py:18-65) fields; angle may be NULL */
typedef struct {
    int64_t n;
    const double *u, *v;
    const int32_t *octave;
    const double *angle;
    const uint64_t *desc;   /* [n][4] */
} ft_host_features;

/* reference ImagePyramid (extraction.py:67-94): flat u8 + level table */
typedef struct {
    const uint8_t *data;
    int32_t n_levels;
    int64_t offsets[FT_MAX_LEVELS + 1];
    int32_t widths[FT_MAX_LEVELS];
    int32_t heights[FT_MAX_LEVELS];
} ft_host_pyramid;

/* reference StereoMatches (stereo.py:45-64), n entries each */
typedef struct {
    int64_t *right_idx, *distance;
    double *disparity, *refined_u, *depth;
    int64_t *sad;
} ft_host_matches;

/* reference MapPointSoA (mapping.py:163-201); ids may be NULL */
typedef struct {
    int64_t m;
    const double *positions, *normals;  /* [m][3] */
    const double *min_dist, *max_dist;
    const uint64_t *desc;               /* [m][4] */
    const int64_t *ids;
} ft_host_points;

/* outputs of ft_session_project; any pointer may be NULL (not copied) */
typedef struct {
    int64_t *out_kp, *out_dist, *out_oct;                /* [m] run_phase_a */
    int64_t *corr_point, *corr_kp, *corr_dist, *corr_oct; /* [m] resolved, point order */
    int32_t *corr_count;
    int64_t *slots_out;                                  /* [n_kp] after the slot write */
    int32_t *slot_count;
} ft_host_project_out;

/* Host packing of the reference SoA fields into records (the loops the
 * session runs; exported for callers that stage their own pinned buffers,
 * e.g. the per-frame pipelines).  Plain C, no CUDA calls. */
int ft_host_pack_keypoints(const ft_host_features *f, ft_kp_record *out);
int ft_host_pack_points(const ft_host_points *p, ft_point_record *out);

int ft_session_create(int32_t device, ft_session **out);
int ft_session_destroy(ft_session *s);
/* Accumulated host phase times of the session's stereo / project calls (us):
 * out[0] pack, [1] issue (copies + launch enqueue), [2] kernel (cudaEvents,
 * only when FT_SESSION_TIMING was set at creation), [3] synchronise, [4]
 * unpack, [5] calls.  reset != 0 zeroes them. */
int ft_session_stats(ft_session *s, double *out, int32_t reset);

/* stereo.py:77-188 with host arrays; mode bits as ft_stereo_pinhole.
 *   PHASE1 alone (match_pinhole_phase1): cand_idx / cand_dist [n_left] out.
 *   REFINE | FROM_CAND without PHASE1 (refine_match_phase2 /
 *     matches_from_candidates): cand_idx / cand_dist in, matches out.
 *   PHASE1 | REFINE | FROM_CAND [| REJECT] (fused ComputeStereoMatches):
 *     matches out (cand_* out too when non-NULL).
 *   REJECT alone (reject_outliers): matches in and out (in place).
 * Pyramids (REFINE only): only levels >= the lowest left octave are copied
 * (phase 2 reads no others, kernels.py:351-428). */
int ft_session_stereo(ft_session *s, const ft_host_features *left, const ft_host_features *right,
                      const ft_host_pyramid *left_pyr, const ft_host_pyramid *right_pyr,
                      const ft_stereo_params *params, int32_t mode, int64_t *cand_idx,
                      int64_t *cand_dist, const ft_host_matches *matches);

/* projection.py:118-221 / localmap.py:79-122 with host arrays.  Map points
 * from `points` (packed here), or -- with `table` non-NULL -- read in place
 * from a resident device table through the host slot list table_index[m]
 * (points->m gives m).  rot[9] / trans[3] host; skip [m], ref_angles [m],
 * slots_in [n_kp] host or NULL; mode bits as ft_project_search. */
int ft_session_project(ft_session *s, const ft_host_points *points, const ft_point_record *table,
                       int64_t table_size, const int32_t *table_index,
                       const ft_host_features *frame, const ft_project_params *params,
                       const double *rot, const double *trans, const uint8_t *skip,
                       const double *ref_angles, const int64_t *slots_in, int32_t mode,
                       const ft_host_project_out *out);

/* Device-resident world for update_local_map (localmap.py:42-76, SURVEY
 * 8(f)-4): keyframe k's observed point ids (KeyFrame.observed_point_ids,
 * mapping.py:142-145) at kf_obs[kf_off[k] .. kf_off[k+1]), point id p's slot
 * in the map table at id_slot[p] (-1 absent), ids in [0, id_cap).  All
 * DEVICE pointers. */
typedef struct {
    const int32_t *kf_obs;
    const int64_t *kf_off;   /* [n_kf + 1] */
    int32_t n_kf;
    const int32_t *id_slot;  /* [id_cap] */
    int64_t id_cap;
} ft_world_dev;

/* localmap.py:42-76 on the device: seeds = the frame's slotted ids (DEVICE
 * slots[n_slots], -1 empty); keyframes = those observing any seed; points =
 * every id they observe.  Outputs (DEVICE): kf_out ascending keyframe
 * indices, point_out ascending point ids, slot_out (may be NULL) their table
 * slots, counts[3] = (keyframes, points, 1 if a slot held an id outside
 * [0, id_cap)).  One block, bitmaps in shared memory: id_cap <= ~0.9M. */
int ft_update_local_map(const int64_t *slots, int32_t n_slots, const int32_t *kf_obs,
                        const int64_t *kf_off, int32_t n_kf, const int32_t *id_slot,
                        int64_t id_cap, int32_t *kf_out, int64_t *point_out, int32_t *slot_out,
                        int32_t *counts, ft_stream_t stream);

/* ft_update_local_map with the frame's HOST slots and host outputs (up to
 * out_cap entries each; FT_E_RANGE with counts set when more -- retry with
 * bigger buffers, or when a slot held an id outside the world). */
int ft_session_update_local_map(ft_session *s, const int64_t *slots, int64_t n_slots,
                                const ft_world_dev *world, int64_t out_cap, int32_t *kf_out,
                                int64_t *point_out, int32_t *slot_out, int32_t *counts);

/* stereo.py:223-273 with host arrays: brute force + ratio test (tri NULL,
 * bruteforce_match_kernel) or + triangulation (ft_stereo_fisheye). */
int ft_session_fisheye(ft_session *s, const ft_host_features *left,
                       const ft_host_features *right, int32_t t_match, double ratio,
                       const ft_fisheye_tri *tri, int64_t *out_idx, int64_t *out_dist,
                       int32_t *out_ok, double *out_points);

#ifdef __cplusplus
}
#endif

#endif /* FASTTRACK_B200_H */
