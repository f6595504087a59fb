"""Resident, graph-captured per-frame hot path for S independent frame
streams on one B200 (BASELINE cfg 2/4/5).

One step processes one frame of every stream:

    pinned staging --(1 H2D)--> device inputs
        ft_track_frames (ONE cooperative launch):
            stereo blocks: phase 1 -> phase 2 | from-candidates -> reject
            map blocks:    skip slotted -> phase A -> resolve -> slot write
    device results --(1 D2H)--> pinned results

Stereo and the local-map search are independent within a frame (the
reference runs them in sequence only because it is single-threaded,
tracker.py:268-358), so they run side by side in one launch.  The whole step
is captured ONCE as a CUDA graph; per-frame counts live in device memory, so
replays need no re-capture.  Layout: every per-frame array is at a fixed
stride (capacity) per stream, inputs packed first (one contiguous H2D range),
outputs last (one contiguous D2H range).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .runtime import (Layout, fill_kp_records, fill_point_records, make_workspace,
                      project_params, pyramid_struct, stereo_params)
from .types import ProjectionSearchConfig, StereoMatchConfig, StereoMatches


@dataclass
class StreamResult:
    matches: StereoMatches
    slots: np.ndarray
    n_slots: int
    n_matched: int


class DeviceArena:
    """One device allocation holding n pipelines' buffers at ONE pitch (a
    2 MB multiple, 2 MB aligned).  AsyncRunner(persistent=True) over such
    pipelines can then ship m consecutive steps' inputs as one strided copy
    per range (submit_batch; ft_runner_submit_batch)."""

    def __init__(self, n: int):
        self.n, self.used, self.pitch, self.buf = int(n), 0, None, None

    def take(self, nbytes: int, device) -> torch.Tensor:
        pitch = (int(nbytes) + (2 << 20) - 1) // (2 << 20) * (2 << 20)
        if self.buf is None:
            self._raw = torch.zeros(self.n * pitch + (2 << 20), dtype=torch.uint8, device=device)
            off = (-self._raw.data_ptr()) % (2 << 20)
            self.buf, self.pitch = self._raw[off:off + self.n * pitch], pitch
        if pitch != self.pitch or self.used >= self.n:
            raise ValueError(f"DeviceArena: {self.used}/{self.n} rows of {self.pitch} B taken; "
                             f"cannot place {nbytes} B")
        row = self.buf[self.used * pitch:self.used * pitch + int(nbytes)]
        self.used += 1
        return row


class FramePipeline:
    def __init__(self, cam, n_streams: int = 1, cap_kp: int = 2048, cap_points: int = 8192,
                 pyramid_geometry=None, stereo_cfg: StereoMatchConfig | None = None,
                 proj_cfg: ProjectionSearchConfig | None = None, scale: float = 1.2,
                 levels: int = 8, grid_cell_px: int = 48, device: int | None = None,
                 raw_images: bool = False, map_table=None, build_levels: int | None = None,
                 packed_upload: bool | None = None, arena: "DeviceArena | None" = None):
        if not torch.cuda.is_available():
            raise _lib.FtError("FramePipeline needs a CUDA device (no CPU fallback)")
        self.lib = _lib.load()
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.cam = cam
        self.S = int(n_streams)
        self.cap_kp = int(cap_kp)
        self.cap_pts = int(cap_points)
        self.scfg = stereo_cfg or StereoMatchConfig()
        self.pcfg = proj_cfg or ProjectionSearchConfig()
        self.scale, self.levels = float(scale), int(levels)
        self.scale_pow = self.scale ** np.arange(self.levels, dtype=np.float64)
        self.pyr = pyramid_geometry  # object with widths / heights / offsets, or None
        # raw_images: frames ship level 0 and ft_build_pyramids builds levels
        # 1..build_levels on the device (default: all); the levels above
        # build_levels are shipped (one contiguous range per image) -- a
        # copy / compute balance: the big levels are cheaper to build, the
        # small ones to ship
        self.raw = bool(raw_images) and pyramid_geometry is not None
        n_lv = len(pyramid_geometry.widths) if pyramid_geometry is not None else 0
        self.build_levels = (n_lv - 1 if build_levels is None else
                             max(1, min(int(build_levels), n_lv - 1))) if self.raw else 0
        # map_table (maptable.MapTable): frames ship table slots (4 B / point)
        # instead of point records; the map role reads the table in place
        self.table = map_table
        self.delta_bytes = 0
        self.cell = int(grid_cell_px)
        self.nx = max(1, (int(cam.width) + self.cell - 1) // self.cell)
        self.ny = max(1, (int(cam.height) + self.cell - 1) // self.cell)

        S, ck, cp = self.S, self.cap_kp, self.cap_pts
        lay = Layout()
        # per-image pyramid stride padded to 256 B: 16-B vector copies of level 0
        self.pyr_total = int(self.pyr.offsets[-1]) if self.pyr is not None else 0
        self.pyr_bytes = (self.pyr_total + 255) // 256 * 256
        # single stream, pyramids shipped: [right pyramid, levels 0..L-1 | small
        # inputs | left pyramid, levels L-1..0].  Phase 2 reads only levels >=
        # the lowest left-keypoint octave m (kernels.py:351-428 reads level o of
        # both images for a left keypoint of octave o), and those bytes form ONE
        # contiguous range around the small inputs: input_range() ships just
        # that (the whole pyramid when an octave-0 keypoint exists).
        # S > 1: [small inputs | R_0 L_0 | R_1 L_1 | ...] (each stream's right
        # pyramid normal, left reversed): one range for the small inputs and one
        # per stream (input_ranges()).
        self.level_ranges = (self.pyr is not None and not self.raw)
        if self.level_ranges and S == 1:
            lay.add("pyrR", self.pyr_bytes)
        # small per-frame inputs first (one 2 MB page holds them for a frame),
        # then the pyramids, then the outputs: the map blocks' reads all land
        # in the first page, so a cold TLB costs them one page walk
        for side in ("L", "R"):
            lay.add(f"{side}_n", 4 * S)
            lay.add(f"{side}_rec", _lib.KP_RECORD.itemsize * S * ck)
        lay.add("P_n", 4 * S)
        if self.table is None:
            lay.add("P_rec", _lib.POINT_RECORD.itemsize * S * cp)
        else:
            lay.add("P_idx", 4 * S * cp)
        lay.add("rot", 72 * S)
        lay.add("trans", 24 * S)
        lay.add("slots_in", 8 * S * ck)
        self.img_bytes = int(self.pyr.widths[0]) * int(self.pyr.heights[0]) if self.pyr is not None else 0
        self.upper_off = int(self.pyr.offsets[self.build_levels + 1]) if self.raw else 0
        self.upper_bytes = self.pyr_total - self.upper_off if self.raw else 0
        if self.raw:
            lay.add("imgs", 2 * S * self.img_bytes)  # [left x S | right x S]
            if self.upper_bytes:
                lay.add("upper", 2 * S * self.upper_bytes)
        elif self.level_ranges:
            self.small_end = lay.total
            if S == 1:
                lay.add("pyrL", self.pyr_bytes)
            else:
                lay.add("pairs", 2 * S * self.pyr_bytes)
            sizes = np.diff(np.asarray(self.pyr.offsets, dtype=np.int64))
            self.lvl_size = sizes
            # reversed-order offsets of the left pyramid: level l after levels > l
            self.rev_off = np.array([int(sizes[l + 1:].sum()) for l in range(len(sizes))],
                                    dtype=np.int64)
        elif self.pyr is not None:
            lay.add("pyrs", 2 * S * self.pyr_bytes)
        # packed upload (S > 1, level ranges): the step's S + 1 needed ranges
        # are packed on the host into ONE contiguous region -- a descriptor
        # header (src, dst, len per segment) then the segments, each placed so
        # src = dst (mod 16) -- shipped as one H2D and placed by ft_copy_ranges
        # ahead of the track kernel (one large DMA instead of S + 1 small ones)
        self.packed = bool(self.level_ranges and S > 1 and
                           (packed_upload is None or packed_upload))
        if self.packed:
            self.pack_hdr = (24 * (S + 1) + 255) // 256 * 256
            lay.add("pack", self.pack_hdr + self.small_end + 16 +
                    S * (2 * self.pyr_bytes + 16))
            self.pack_used = self.pack_hdr
            self._pack_dirty = True
        self.in_end = lay.total
        self.cur_range = (0, self.in_end)
        self.stream_m = np.zeros(S, dtype=np.int64)  # lowest left octave per stream
        self.out_begin = lay.total
        lay.add("slots", 8 * S * ck)   # updated slots (output)
        for name in ("right_idx", "distance", "disparity", "refined_u", "depth", "sad"):
            lay.add(name, 8 * S * ck)
        lay.add("n_matched", 4 * S)
        lay.add("slot_n", 4 * S)
        lay.add("c_n", 4 * S)
        self.out_end = lay.total
        if self.raw:  # device-built pyramids: not copied
            lay.add("pyrs", 2 * S * self.pyr_bytes)

        # device-only scratch (not copied)
        lay.add("cand_idx", 8 * S * ck)
        lay.add("cand_dist", 8 * S * ck)
        for name in ("c_point", "c_kp", "c_dist", "c_oct"):
            lay.add(name, 8 * S * cp)
        self.lay = lay
        # 2 MB-aligned arena (GPU large pages): fewest pages per frame; or a
        # row of a shared DeviceArena (slots at one pitch: batched submits)
        if arena is not None:
            self._dev_raw = arena
            self.dev = arena.take(lay.total, self.device)
        else:
            self._dev_raw = torch.zeros(lay.total + (2 << 20), dtype=torch.uint8,
                                        device=self.device)
            off = (-self._dev_raw.data_ptr()) % (2 << 20)
            self.dev = self._dev_raw[off:off + lay.total]
        self.host = torch.zeros(lay.total, dtype=torch.uint8).pin_memory()
        self.hnp = self.host.numpy()
        self.stream = torch.cuda.Stream(self.device)
        self.ws = make_workspace(self.lib, self.device, self.stream, S, ck, cp)
        self._build_structs()
        self.graph = None
        self.graph_compute = None
        self.graph_runner = None

    # -- host views ------------------------------------------------------------

    def _h(self, name: str, dtype, shape) -> np.ndarray:
        off = self.lay.offsets[name]
        n = int(np.prod(shape)) * np.dtype(dtype).itemsize
        return self.hnp[off:off + n].view(dtype).reshape(shape)

    def _d(self, name: str) -> int:
        return self.dev.data_ptr() + self.lay.offsets[name]

    def load_frame(self, s: int, left, right, local, pose, pyr_left=None, pyr_right=None,
                   slots=None) -> None:
        """Copy stream s's frame inputs into the pinned staging area."""
        S, ck, cp = self.S, self.cap_kp, self.cap_pts
        for side, fs in (("L", left), ("R", right)):
            n = len(fs.u)
            if n > ck:
                raise ValueError(f"{n} keypoints exceed capacity {ck}")
            self._h(f"{side}_n", np.int32, (S,))[s] = n
            fill_kp_records(self._h(f"{side}_rec", _lib.KP_RECORD, (S, ck))[s], fs)
        if self.pyr is not None:
            if pyr_left is None or pyr_right is None:
                raise ValueError("pipeline was built with pyramids: pass pyr_left / pyr_right "
                                 "(raw_images: level 0 is used)")
            if self.raw:
                ib = self.img_bytes
                imgs = self._h("imgs", np.uint8, (2, S, ib))
                imgs[0, s] = np.asarray(pyr_left.data)[:ib]
                imgs[1, s] = np.asarray(pyr_right.data)[:ib]
                if self.upper_bytes:
                    up = self._h("upper", np.uint8, (2, S, self.upper_bytes))
                    up[0, s] = np.asarray(pyr_left.data)[self.upper_off:self.pyr_total]
                    up[1, s] = np.asarray(pyr_right.data)[self.upper_off:self.pyr_total]
            elif self.level_ranges:
                if S == 1:
                    dr = self._h("pyrR", np.uint8, (self.pyr_total,))
                    dl = self._h("pyrL", np.uint8, (self.pyr_total,))
                else:
                    pairs = self._h("pairs", np.uint8, (S, 2, self.pyr_bytes))
                    dr = pairs[s, 0, :self.pyr_total]
                    dl = pairs[s, 1, :self.pyr_total]
                dr[:] = pyr_right.data
                src = np.asarray(pyr_left.data)
                offs = np.asarray(self.pyr.offsets, dtype=np.int64)
                for lv in range(len(self.lvl_size)):
                    dl[self.rev_off[lv]:self.rev_off[lv] + self.lvl_size[lv]] = \
                        src[offs[lv]:offs[lv + 1]]
                oct_ = np.asarray(left.octave)
                m = int(oct_.min()) if len(oct_) else len(self.lvl_size) - 1
                m = min(max(m, 0), len(self.lvl_size) - 1)
                self.stream_m[s] = m
                if S == 1:
                    lo = self.lay.offsets["pyrR"] + int(offs[m])
                    hi = self.lay.offsets["pyrL"] + int(self.rev_off[m] + self.lvl_size[m])
                    self.cur_range = (lo, hi)
            else:
                pb = self.pyr_bytes
                pyrs = self._h("pyrs", np.uint8, (2, S, pb))
                pyrs[0, s, :self.pyr_total] = pyr_left.data
                pyrs[1, s, :self.pyr_total] = pyr_right.data
        m = len(local.point_ids)
        soa = local.soa if (self.table is None or getattr(local, "table", None) is not self.table
                            ) else None
        if m > cp:
            raise ValueError(f"{m} map points exceed capacity {cp}")
        self._h("P_n", np.int32, (S,))[s] = m
        if self.table is not None and getattr(local, "table", None) is self.table and \
                getattr(local, "table_slots", None) is not None:
            # a ResidentLocalMap of this table (worldmap.update_local_map): slots known
            self._h("P_idx", np.int32, (S, cp))[s, :m] = local.table_slots
        elif self.table is None:
            fill_point_records(self._h("P_rec", _lib.POINT_RECORD, (S, cp))[s], soa)
        else:
            # points new to the table are the frame's map delta (uploaded now)
            self.delta_bytes += self.table.upsert(local.point_ids, soa, only_missing=True)
            self._h("P_idx", np.int32, (S, cp))[s, :m] = self.table.slots(local.point_ids)
        self._h("rot", np.float64, (S, 9))[s] = np.asarray(pose.rotation).reshape(9)
        self._h("trans", np.float64, (S, 3))[s] = np.asarray(pose.translation).reshape(3)
        sl = self._h("slots_in", np.int64, (S, ck))
        sl[s] = -1
        if slots is not None:
            sl[s, :len(left.u)] = slots
        if self.packed:
            self._pack_dirty = True

    def _segments(self) -> list[tuple[int, int]]:
        """The [lo, hi) ranges of the regular input layout the current step
        needs (level ranges, S > 1)."""
        pb, base = self.pyr_bytes, self.lay.offsets["pairs"]
        offs = np.asarray(self.pyr.offsets, dtype=np.int64)
        out = [(0, self.small_end)]
        for st in range(self.S):
            m = int(self.stream_m[st])
            lo = base + 2 * st * pb + int(offs[m])
            hi = base + (2 * st + 1) * pb + int(self.rev_off[m] + self.lvl_size[m])
            out.append((lo, hi))
        return out

    def pack(self) -> tuple[int, int]:
        """Pack the current step's needed ranges into the pack region of the
        staging (no-op when unchanged); returns the [lo, hi) to ship."""
        base = self.lay.offsets["pack"]
        if self._pack_dirty:
            segs = self._segments()
            desc = self.hnp[base:base + 24 * len(segs)].view(np.int64).reshape(-1, 3)
            cur = base + self.pack_hdr
            for q, (lo, hi) in enumerate(segs):
                cur += (lo - cur) % 16
                n = hi - lo
                self.hnp[cur:cur + n] = self.hnp[lo:hi]
                desc[q] = (cur, lo, n)
                cur += n
            self.pack_used = cur - base
            self._pack_dirty = False
        return (base, base + self.pack_used)

    def h2d_bytes(self) -> int:
        if self.packed:
            return self.in_end - self.lay.offsets["pack"]
        return self.in_end

    def input_range(self) -> tuple[int, int]:
        """[lo, hi) of the input staging the current frame needs on the device:
        the whole input area, or with level ranges the pyramid levels at or
        above the frame's lowest left-keypoint octave plus the small inputs
        (S > 1: the packed region)."""
        if self.packed:
            return self.pack()
        return self.cur_range

    def input_ranges(self) -> list[tuple[int, int]]:
        """The [lo, hi) byte ranges of the input staging the current step
        needs: one for S == 1 (input_range()); for S > 1 with level ranges the
        small inputs plus, per stream, its pyramid pair's levels >= that
        stream's lowest left octave; else the whole input area."""
        if not self.level_ranges:
            return [(0, self.in_end)]
        if self.S == 1:
            return [self.cur_range]
        if self.packed:
            return [self.pack()]
        return self._segments()

    def d2h_bytes(self) -> int:
        return self.out_end - self.out_begin

    # -- launch ----------------------------------------------------------------

    def _build_structs(self) -> None:
        S, ck, cp = self.S, self.cap_kp, self.cap_pts
        kps = {}
        for side in ("L", "R"):
            k = _lib.FtKeypoints()
            k.rec, k.count, k.cap = self._d(f"{side}_rec"), self._d(f"{side}_n"), ck
            kps[side] = k
        self.kl, self.kr = kps["L"], kps["R"]
        if self.level_ranges:
            if S == 1:
                self.pr = pyramid_struct(self.pyr, self._d("pyrR"), self.pyr_bytes)
                self.pl = pyramid_struct(self.pyr, self._d("pyrL"), self.pyr_bytes)
            else:  # stream s: right at pairs + 2 s pb, left at pairs + (2 s + 1) pb
                self.pr = pyramid_struct(self.pyr, self._d("pairs"), 2 * self.pyr_bytes)
                self.pl = pyramid_struct(self.pyr, self._d("pairs") + self.pyr_bytes,
                                         2 * self.pyr_bytes)
            for lv in range(len(self.lvl_size)):
                self.pl.offsets[lv] = int(self.rev_off[lv])
        elif self.pyr is not None:
            pyrs = self._d("pyrs")
            self.pl = pyramid_struct(self.pyr, pyrs, self.pyr_bytes)
            self.pr = pyramid_struct(self.pyr, pyrs + S * self.pyr_bytes, self.pyr_bytes)
            if self.raw:  # levels 0..build_levels built on the device, all 2S images
                self.pl_build = pyramid_struct(self.pyr, pyrs, self.pyr_bytes)
                self.pl_build.n_levels = self.build_levels + 1
        else:
            self.pl = self.pr = None
        self.sparams = stereo_params(self.scfg, int(self.cam.height), self.scale_pow,
                                     float(self.cam.baseline_times_fx))
        self.smode = _lib.FT_STEREO_PHASE1 | _lib.FT_STEREO_REJECT | (
            _lib.FT_STEREO_REFINE if self.pyr is not None else _lib.FT_STEREO_FROM_CAND)
        o = _lib.FtStereoOut()
        for name in ("cand_idx", "cand_dist", "right_idx", "distance", "disparity", "refined_u",
                     "depth", "sad", "n_matched"):
            setattr(o, name, self._d(name))
        self.sout = o
        P = _lib.FtMapPoints()
        if self.table is None:
            P.rec, P.count, P.cap, P.index = self._d("P_rec"), self._d("P_n"), cp, None
        else:  # read in place from the resident table through the slot list
            P.rec, P.count, P.cap, P.index = self.table.ptr, self._d("P_n"), cp, self._d("P_idx")
        self.points = P
        self.pparams = project_params(self.cam, self.pcfg, self.scale, self.levels, self.cell,
                                      self.nx, self.ny, None, 0.0)
        io = _lib.FtProjectIO()
        io.rot, io.trans, io.skip, io.ref_angles = self._d("rot"), self._d("trans"), None, None
        io.slots_in, io.slots_out = self._d("slots_in"), self._d("slots")
        self.pio = io
        po = _lib.FtProjectOut()
        # SearchLocalPoints needs the slots and counts, not the ordered
        # correspondence list: leave corr_* unset (saves a group barrier)
        po.corr_point = po.corr_kp = po.corr_dist = po.corr_oct = None
        po.corr_count, po.slot_count = self._d("c_n"), self._d("slot_n")
        self.pout = po
        self.pmode = (_lib.FT_PROJ_RESOLVE | _lib.FT_PROJ_SKIP_SLOTS | _lib.FT_PROJ_WRITE_SLOTS)

    def launch_stereo(self, stream) -> None:
        _lib.check(self.lib.ft_stereo_pinhole(self.S, self.kl, self.kr, self.pl, self.pr,
                                              self.sparams, self.smode, self.sout, self.ws,
                                              stream.cuda_stream), "ft_stereo_pinhole")

    def launch_project(self, stream) -> None:
        _lib.check(self.lib.ft_project_search(self.S, self.points, self.kl, self.pparams,
                                              self.pio, self.pmode, self.pout, self.ws,
                                              stream.cuda_stream), "ft_project_search")

    def launch_track(self, stream) -> None:
        _lib.check(self.lib.ft_track_frames(self.S, self.kl, self.kr, self.pl, self.pr,
                                            self.sparams, self.smode, self.sout, self.points,
                                            self.pparams, self.pio, self.pmode, self.pout,
                                            self.ws, stream.cuda_stream), "ft_track_frames")

    def plan(self, groups: int = 1):
        """The track launch of this pipeline's step recorded as an
        ft_track_plan (input of the persistent runner); None when the step is
        more than that one launch (device pyramid build / packed upload).
        groups > 1: sized for a persistent launch of that many step groups
        (ft_track_plan_groups: that many frames in flight)."""
        import ctypes
        if self.raw or self.packed:
            return None
        buf = (ctypes.c_ubyte * int(self.lib.ft_track_plan_bytes()))()
        _lib.check(self.lib.ft_track_plan_groups(self.S, self.kl, self.kr, self.pl, self.pr,
                                                 self.sparams, self.smode, self.sout,
                                                 self.points, self.pparams, self.pio,
                                                 self.pmode, self.pout, self.ws, int(groups),
                                                 buf, len(buf)), "ft_track_plan_groups")
        return buf

    def launch_pyramids(self, stream) -> None:
        if self.raw:
            S2 = 2 * self.S
            if self.upper_bytes:  # shipped upper levels into place (strided D2D)
                with torch.cuda.stream(stream):
                    base = self.lay.offsets["pyrs"]
                    dst = self.dev[base:base + S2 * self.pyr_bytes].view(S2, self.pyr_bytes)
                    ub = self.lay.offsets["upper"]
                    src = self.dev[ub:ub + S2 * self.upper_bytes].view(S2, self.upper_bytes)
                    dst[:, self.upper_off:self.pyr_total].copy_(src, non_blocking=True)
            _lib.check(self.lib.ft_build_pyramids(S2, self.pl_build, self._d("imgs"),
                                                  self.img_bytes, self.ws, stream.cuda_stream),
                       "ft_build_pyramids")

    def launch_unpack(self, stream) -> None:
        """Place the packed upload's segments (packed pipelines only)."""
        if self.packed:
            _lib.check(self.lib.ft_copy_ranges(self.dev.data_ptr(), self._d("pack"), self.S + 1,
                                               stream.cuda_stream), "ft_copy_ranges")

    def _step(self, copies: bool, unpack: bool | None = None) -> None:
        a = self.stream
        if copies:
            lo = self.lay.offsets["pack"] if self.packed else 0
            with torch.cuda.stream(a):
                self.dev[lo:self.in_end].copy_(self.host[lo:self.in_end], non_blocking=True)
        if copies if unpack is None else unpack:
            self.launch_unpack(a)
        self.launch_pyramids(a)
        self.launch_track(a)
        if copies:
            with torch.cuda.stream(a):
                self.host[self.out_begin:self.out_end].copy_(
                    self.dev[self.out_begin:self.out_end], non_blocking=True)

    def run_eager(self, copies: bool = True) -> None:
        from . import _guard
        _guard.check(self.device.index if self.device.index is not None else 0,
                     "FramePipeline.run_eager")
        if copies and self.packed:
            self.pack()
        self._step(copies)

    def capture(self) -> None:
        """Capture the full step (with copies), the compute-only step (inputs
        resident in place) and, for packed pipelines, the step AsyncRunner
        launches after its H2D (unpack + compute)."""
        self.run_eager(True)  # warm: sets kernel attributes, loads modules
        self.stream.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=self.stream):
            self._step(True)
        self.graph_compute = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph_compute, stream=self.stream):
            self._step(False)
        self.graph_runner = self.graph_compute
        if self.packed:
            self.graph_runner = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.graph_runner, stream=self.stream):
                self._step(False, unpack=True)
        self.stream.synchronize()

    def replay(self, copies: bool = True) -> None:
        from . import _guard
        _guard.check(self.device.index if self.device.index is not None else 0,
                     "FramePipeline.replay")
        if self.graph is None:
            self.capture()
        if copies and self.packed:
            self.pack()
        # CUDAGraph.replay() launches on torch's current stream
        with torch.cuda.stream(self.stream):
            (self.graph if copies else self.graph_compute).replay()

    def synchronize(self) -> None:
        self.stream.synchronize()

    # -- results ---------------------------------------------------------------

    def result(self, s: int, n_left: int) -> StreamResult:
        S, ck = self.S, self.cap_kp
        g = lambda name, dt: self._h(name, dt, (S, ck))[s, :n_left].copy()  # noqa: E731
        m = StereoMatches(right_idx=g("right_idx", np.int64), distance=g("distance", np.int64),
                          disparity=g("disparity", np.float64),
                          refined_u=g("refined_u", np.float64), depth=g("depth", np.float64),
                          sad=g("sad", np.int64))
        return StreamResult(matches=m, slots=g("slots", np.int64),
                            n_slots=int(self._h("slot_n", np.int32, (S,))[s]),
                            n_matched=int(self._h("n_matched", np.int32, (S,))[s]))

    def copy_outputs(self) -> None:
        """Device outputs -> the pinned host area result() reads (synchronous)."""
        with torch.cuda.stream(self.stream):
            self.host[self.out_begin:self.out_end].copy_(self.dev[self.out_begin:self.out_end],
                                                         non_blocking=True)
        self.stream.synchronize()

    def staged_inputs(self) -> torch.Tensor:
        """A pinned copy of the current input staging (what load_frame wrote):
        one step's inputs, ready for AsyncRunner.submit."""
        if self.packed:
            self.pack()
        return self.host[:self.in_end].clone().pin_memory()

    def staging_ring(self, n: int) -> torch.Tensor:
        """One pinned allocation of n input slots ([n, in_end], rows 256-B
        aligned): a ring a frame source fills and AsyncRunner.submit reads.
        One allocation keeps the DMA mappings few (IOMMU / TLB friendly)."""
        stride = (self.in_end + 255) // 256 * 256
        ring = torch.zeros((n, stride), dtype=torch.uint8).pin_memory()
        return ring[:, :self.in_end]

    def stage_into(self, dst: torch.Tensor) -> None:
        """Copy the current input staging into a ring slot."""
        if self.packed:
            self.pack()
        dst.copy_(self.host[:self.in_end])


def run_ring(pipes, n_steps: int, stream=None, groups: int = 1) -> None:
    """n_steps steps over pipelines whose inputs are already on the device, in
    ONE persistent launch (ft_track_frames_ring): step k runs pipes[k % n]'s
    track step.  groups > 1: that many disjoint block groups take the steps
    round robin (that many frames in flight; len(pipes) must be a multiple).
    Stream-ordered on `stream` (default pipes[0].stream); the outputs stay on
    the device (read them with copy_outputs())."""
    import ctypes
    from . import _guard
    _guard.check(pipes[0].device.index if pipes[0].device.index is not None else 0, "run_ring")
    if len(pipes) % groups:
        raise ValueError("run_ring: the pipeline count must be a multiple of groups")
    plans = []
    for p in pipes:
        cache = p.__dict__.setdefault("_plans", {})
        if groups not in cache:
            cache[groups] = p.plan(groups)
            if cache[groups] is None:
                raise ValueError("run_ring: each step must be the one track launch")
        plans.append(cache[groups])
    arr = (ctypes.c_void_p * len(plans))(*[ctypes.addressof(pl) for pl in plans])
    st = stream if stream is not None else pipes[0].stream
    _lib.check(pipes[0].lib.ft_track_frames_ring(len(plans), arr, int(n_steps), st.cuda_stream),
               "ft_track_frames_ring")


def _graph_exec_ptr(graph) -> int:
    """cudaGraphExec_t of an instantiated torch.cuda.CUDAGraph."""
    h = graph.raw_cuda_graph_exec()
    if isinstance(h, int):
        return h
    import ctypes
    get = ctypes.pythonapi.PyCapsule_GetPointer
    get.restype, get.argtypes = ctypes.c_void_p, [ctypes.py_object, ctypes.c_char_p]
    return get(h, None)


class _Ranges:
    """Byte ranges of a step's inputs as the C ABI's flat uint64 pairs."""

    def __init__(self, rng):
        import ctypes
        pairs = [rng] if len(rng) == 2 and not isinstance(rng[0], (tuple, list)) else list(rng)
        self.n = len(pairs)
        self.flat = (ctypes.c_uint64 * max(1, 2 * self.n))(*[int(x) for r in pairs for x in r])
        self.bytes = sum(int(hi) - int(lo) for lo, hi in pairs)


class AsyncRunner:
    """Copy / compute overlapped driver for a stream of steps (the real-time
    shape of the tracker: the next frame's images and keypoints upload while
    the current one tracks).  Two FramePipelines of identical shape take
    alternate steps; per step k, issued natively by ft_runner_submit
    (csrc/ft_runner.cu, one host call):

        H2D stream:     inputs(k)          -> pipe[k % 2] device inputs
        compute stream: pipe[k % 2]'s compute graph (gather / pyramids / track)
        D2H stream:     pipe[k % 2] outputs -> its pinned result area

    Compute is serialised on one stream (one cooperative launch at a time);
    H2D of step k+1 and D2H of step k-1 run on the two copy engines while
    step k computes.  ``wait(k)`` blocks until step k's results are in
    ``pipes[k % 2]`` host memory.

    persistent=True (pipelines whose step is the one track launch): no launch
    per step -- one long-lived track kernel serves the slots, handed each
    step by device flags the copy streams write / wait on
    (ft_runner_create_persistent).  close() ends it after the submitted
    steps; until then the kernel holds its SMs."""

    def __init__(self, pipes, persistent=False, groups: int = 1):
        """persistent: False (graph launch per step), True (one persistent
        kernel; raises where the step is not eligible) or "auto" (persistent
        where eligible, else graph launches; ``self.persistent`` says which).
        groups (persistent only): step groups of the persistent kernel --
        that many steps computed at once on disjoint SMs (len(pipes) must be a
        multiple)."""
        if persistent == "auto":
            try:
                self.__init__(pipes, persistent=True, groups=groups)
                return
            except (ValueError, _lib.FtError):
                persistent = False
        import ctypes
        if not 2 <= len(pipes) <= 16:
            raise ValueError("AsyncRunner takes 2..16 identically shaped pipelines")
        a = pipes[0]
        for b in pipes[1:]:
            if (a.S, a.cap_kp, a.cap_pts, a.in_end, a.out_begin, a.out_end) != \
                    (b.S, b.cap_kp, b.cap_pts, b.in_end, b.out_begin, b.out_end):
                raise ValueError("AsyncRunner pipelines differ in shape")
        self.pipes = pipes
        self.n = len(pipes)
        self.lib = a.lib
        self.persistent = bool(persistent)
        vpn = ctypes.c_void_p * self.n
        self._guard_dev = None
        self._r = ctypes.c_void_p()
        # before anything waits on the device: while a persistent kernel lives,
        # a device-wide synchronise (below) would never return
        from . import _guard
        dev = a.device.index if a.device.index is not None else torch.cuda.current_device()
        if self.persistent:
            _guard.acquire(dev)  # one persistent kernel per GPU
            self._guard_dev = dev
        else:
            _guard.check(dev, "AsyncRunner")
        try:
            self._setup(pipes, groups, vpn)
        except Exception:
            self.close()
            raise

    def _setup(self, pipes, groups, vpn) -> None:
        import ctypes
        a = pipes[0]
        if self.persistent:
            if len(pipes) % groups:
                raise ValueError("persistent runner: slots must be a multiple of groups")
            plans = [p.plan(groups) for p in pipes]
            if any(pl is None for pl in plans):
                raise ValueError("persistent runner: each step must be the one track launch "
                                 "(no raw images / packed upload)")
            execs = vpn(*[ctypes.addressof(pl) for pl in plans])
        else:
            plans = None
            for p in pipes:
                if p.graph_runner is None:
                    p.capture()
            execs = vpn(*[_graph_exec_ptr(p.graph_runner) for p in pipes])
        dev_in = vpn(*[p.dev.data_ptr() for p in pipes])
        dev_out = vpn(*[p.dev.data_ptr() + p.out_begin for p in pipes])
        host_out = vpn(*[p.host.data_ptr() + p.out_begin for p in pipes])
        torch.cuda.synchronize(a.device)
        create = (self.lib.ft_runner_create_persistent if self.persistent
                  else self.lib.ft_runner_create_n)
        _lib.check(create(self.n, execs, dev_in, a.in_end, dev_out, host_out,
                          a.out_end - a.out_begin, ctypes.byref(self._r)), "ft_runner_create")
        self._keep = (execs, dev_in, dev_out, host_out, plans)
        self._submit_ranges = self.lib.ft_runner_submit_ranges
        self._wait = self.lib.ft_runner_wait

    def submit(self, k: int, inputs: torch.Tensor | None = None,
               rng: tuple[int, int] | None = None) -> None:
        """Enqueue step k; inputs = a pinned tensor in the pipelines' input
        layout (staged_inputs() / a staging_ring() row) or its data pointer,
        or None to send pipes[k % n]'s own staging; rng = the [lo, hi) byte
        range(s) to ship (input_range() / input_ranges() of the staged frame,
        or ranges_arg() of them), default all."""
        if type(inputs) is int:
            src = inputs
        else:
            src = (self.pipes[k % self.n].host.data_ptr() if inputs is None
                   else inputs.data_ptr())
        if type(rng) is _Ranges:  # hot path: nothing to marshal
            st = self._submit_ranges(self._r, k, src, rng.flat, rng.n)
            if st:
                _lib.check(st, "ft_runner_submit")
            return
        if rng is None:
            st = self.lib.ft_runner_submit(self._r, k, src)
        elif isinstance(rng, _Ranges):  # pre-converted (ranges_arg)
            st = self.lib.ft_runner_submit_ranges(self._r, k, src, rng.flat, rng.n)
        elif len(rng) == 0 or isinstance(rng[0], (tuple, list)):  # several (input_ranges())
            import ctypes
            flat = (ctypes.c_uint64 * (2 * len(rng)))(*[int(x) for r in rng for x in r])
            st = self.lib.ft_runner_submit_ranges(self._r, k, src, flat, len(rng))
        else:
            lo, hi = int(rng[0]), int(rng[1])
            st = self.lib.ft_runner_submit_range(self._r, k, src, lo, hi - lo)
        _lib.check(st, "ft_runner_submit")

    def submit_batch(self, k: int, rows: torch.Tensor, rng) -> None:
        """Enqueue steps k .. k+m-1 whose inputs are the m rows of one pinned
        [m, >= in_end] tensor view (e.g. staging_ring(n)[j:j+m]), the same
        ranges (ranges_arg()) for each.  On persistent pipelines that share a
        DeviceArena each range goes up as one strided copy for all m steps
        (ft_runner_submit_batch); otherwise step by step."""
        m = int(rows.shape[0])
        pitch = int(rows.stride(0)) if m > 1 else 0
        if not isinstance(rng, _Ranges):
            rng = _Ranges(rng)
        st = self.lib.ft_runner_submit_batch(self._r, k, m, rows.data_ptr(), pitch,
                                             rng.flat, rng.n)
        if st:
            _lib.check(st, "ft_runner_submit_batch")

    @staticmethod
    def ranges_arg(rng) -> "_Ranges":
        """rng (input_range() / input_ranges()) converted once for submit():
        saves the per-step argument marshalling on the host's critical path."""
        return _Ranges(rng)

    def wait(self, k: int) -> FramePipeline:
        """Block until step k's results are on the host; returns its pipeline
        (read them with .result(s, n_left))."""
        st = self._wait(self._r, k)
        if st:
            _lib.check(st, "ft_runner_wait")
        return self.pipes[k % self.n]

    def synchronize(self) -> None:
        torch.cuda.synchronize(self.pipes[0].device)

    def close(self) -> None:
        if getattr(self, "_r", None):
            self.lib.ft_runner_destroy(self._r)
            self._r = None
        if getattr(self, "_guard_dev", None) is not None:
            from . import _guard
            _guard.release(self._guard_dev)
            self._guard_dev = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class FisheyePipeline:
    """Resident, graph-captured per-frame step of the reference tracker's
    fisheye branch (BASELINE cfg 3, TUM-VI shape): ComputeStereoFishEyeMatches
    (tracker.py:399-414 -> match_fisheye, stereo.py:223-273: all-pairs
    Hamming + ratio test + KB triangulation, ft_stereo_fisheye) then
    SearchLocalPoints with the Kannala-Brandt projection (localmap.py:79-122,
    ft_project_search).  S independent frame streams per launch; the local
    map is shipped as records or read in place from a resident MapTable.

    Per left keypoint outputs: right_idx / distance (brute force), ok (pair
    survived triangulation), point (left-camera frame), and the frame slots
    after the local-map search."""

    def __init__(self, cam, n_streams: int = 1, cap_kp: int = 2048, cap_points: int = 8192,
                 stereo_cfg: StereoMatchConfig | None = None,
                 proj_cfg: ProjectionSearchConfig | None = None, scale: float = 1.2,
                 levels: int = 8, grid_cell_px: int = 48, corrected: bool = False,
                 map_table=None, device: int | None = None):
        from .stereo import fisheye_tri_params
        if not torch.cuda.is_available():
            raise _lib.FtError("FisheyePipeline needs a CUDA device (no CPU fallback)")
        self.lib = _lib.load()
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None
                                   else device)
        self.cam = cam
        self.S, self.cap_kp, self.cap_pts = int(n_streams), int(cap_kp), int(cap_points)
        self.scfg = stereo_cfg or StereoMatchConfig()
        self.pcfg = proj_cfg or ProjectionSearchConfig()
        self.scale, self.levels = float(scale), int(levels)
        self.cell = int(grid_cell_px)
        self.nx = max(1, (int(cam.width) + self.cell - 1) // self.cell)
        self.ny = max(1, (int(cam.height) + self.cell - 1) // self.cell)
        self.table = map_table
        self.delta_bytes = 0
        self.tri = fisheye_tri_params(cam, self.scfg, corrected)
        S, ck, cp = self.S, self.cap_kp, self.cap_pts
        lay = Layout()
        for side in ("L", "R"):
            lay.add(f"{side}_n", 4 * S)
            lay.add(f"{side}_rec", _lib.KP_RECORD.itemsize * S * ck)
        lay.add("P_n", 4 * S)
        if self.table is None:
            lay.add("P_rec", _lib.POINT_RECORD.itemsize * S * cp)
        else:
            lay.add("P_idx", 4 * S * cp)
        lay.add("rot", 72 * S)
        lay.add("trans", 24 * S)
        lay.add("slots_in", 8 * S * ck)
        self.in_end = lay.total
        self.out_begin = lay.total
        lay.add("slots", 8 * S * ck)
        lay.add("idx", 8 * S * ck)
        lay.add("dist", 8 * S * ck)
        lay.add("ok", 4 * S * ck)
        lay.add("pts", 24 * S * ck)
        lay.add("slot_n", 4 * S)
        lay.add("c_n", 4 * S)
        self.out_end = lay.total
        self.lay = lay
        self._dev_raw = torch.zeros(lay.total + (2 << 20), dtype=torch.uint8, device=self.device)
        off = (-self._dev_raw.data_ptr()) % (2 << 20)
        self.dev = self._dev_raw[off:off + lay.total]
        self.host = torch.zeros(lay.total, dtype=torch.uint8).pin_memory()
        self.hnp = self.host.numpy()
        self.stream = torch.cuda.Stream(self.device)
        self.ws = make_workspace(self.lib, self.device, self.stream, S, ck, cp)
        k = {}
        for side in ("L", "R"):
            s_ = _lib.FtKeypoints()
            s_.rec, s_.count, s_.cap = self._d(f"{side}_rec"), self._d(f"{side}_n"), ck
            k[side] = s_
        self.kl, self.kr = k["L"], k["R"]
        P = _lib.FtMapPoints()
        if self.table is None:
            P.rec, P.count, P.cap, P.index = self._d("P_rec"), self._d("P_n"), cp, None
        else:
            P.rec, P.count, P.cap, P.index = self.table.ptr, self._d("P_n"), cp, self._d("P_idx")
        self.points = P
        self.pparams = project_params(cam, self.pcfg, self.scale, self.levels, self.cell,
                                      self.nx, self.ny, None, 0.0)
        io = _lib.FtProjectIO()
        io.rot, io.trans, io.skip, io.ref_angles = self._d("rot"), self._d("trans"), None, None
        io.slots_in, io.slots_out = self._d("slots_in"), self._d("slots")
        self.pio = io
        po = _lib.FtProjectOut()
        po.corr_point = po.corr_kp = po.corr_dist = po.corr_oct = None
        po.corr_count, po.slot_count = self._d("c_n"), self._d("slot_n")
        self.pout = po
        self.pmode = (_lib.FT_PROJ_RESOLVE | _lib.FT_PROJ_SKIP_SLOTS | _lib.FT_PROJ_WRITE_SLOTS)
        self.packed = False
        self.graph = None
        self.graph_compute = None
        self.graph_runner = None

    _h = FramePipeline._h
    _d = FramePipeline._d
    h2d_bytes = FramePipeline.h2d_bytes
    d2h_bytes = FramePipeline.d2h_bytes
    synchronize = FramePipeline.synchronize
    capture = FramePipeline.capture
    replay = FramePipeline.replay
    staged_inputs = FramePipeline.staged_inputs
    staging_ring = FramePipeline.staging_ring
    stage_into = FramePipeline.stage_into
    run_eager = FramePipeline.run_eager

    def load_frame(self, s: int, left, right, local, pose, slots=None) -> None:
        S, ck, cp = self.S, self.cap_kp, self.cap_pts
        for side, fs in (("L", left), ("R", right)):
            n = len(fs.u)
            if n > ck:
                raise ValueError(f"{n} keypoints exceed capacity {ck}")
            self._h(f"{side}_n", np.int32, (S,))[s] = n
            fill_kp_records(self._h(f"{side}_rec", _lib.KP_RECORD, (S, ck))[s], fs)
        m = len(local.point_ids)
        if m > cp:
            raise ValueError(f"{m} map points exceed capacity {cp}")
        self._h("P_n", np.int32, (S,))[s] = m
        if self.table is None:
            fill_point_records(self._h("P_rec", _lib.POINT_RECORD, (S, cp))[s], local.soa)
        else:
            self.delta_bytes += self.table.upsert(local.point_ids, local.soa, only_missing=True)
            self._h("P_idx", np.int32, (S, cp))[s, :m] = self.table.slots(local.point_ids)
        self._h("rot", np.float64, (S, 9))[s] = np.asarray(pose.rotation).reshape(9)
        self._h("trans", np.float64, (S, 3))[s] = np.asarray(pose.translation).reshape(3)
        sl = self._h("slots_in", np.int64, (S, ck))
        sl[s] = -1
        if slots is not None:
            sl[s, :len(left.u)] = slots

    def _step(self, copies: bool) -> None:
        # the fisheye stereo and the local-map search only share the left
        # keypoints (read-only): they run on two branches of the graph
        a = self.stream
        if not hasattr(self, "side"):
            self.side = torch.cuda.Stream(self.device)
            self.ev_fork, self.ev_join = torch.cuda.Event(), torch.cuda.Event()
        if copies:
            with torch.cuda.stream(a):
                self.dev[:self.in_end].copy_(self.host[:self.in_end], non_blocking=True)
        # the map search is launched first: its blocks need a whole SM's
        # register file each, so it must claim its SMs before the brute-force
        # blocks spread over all of them
        self.ev_fork.record(a)
        _lib.check(self.lib.ft_project_search(self.S, self.points, self.kl, self.pparams,
                                              self.pio, self.pmode, self.pout, self.ws,
                                              a.cuda_stream), "ft_project_search")
        self.side.wait_event(self.ev_fork)
        _lib.check(self.lib.ft_stereo_fisheye(self.S, self.kl, self.kr, int(self.scfg.t_match),
                                              float(self.scfg.ratio), self.tri, self._d("idx"),
                                              self._d("dist"), self._d("ok"), self._d("pts"),
                                              self.ws, self.side.cuda_stream), "ft_stereo_fisheye")
        self.ev_join.record(self.side)
        a.wait_event(self.ev_join)
        if copies:
            with torch.cuda.stream(a):
                self.host[self.out_begin:self.out_end].copy_(
                    self.dev[self.out_begin:self.out_end], non_blocking=True)

    def result(self, s: int, n_left: int) -> dict:
        S, ck = self.S, self.cap_kp
        g = lambda name, dt: self._h(name, dt, (S, ck))[s, :n_left].copy()  # noqa: E731
        return {"right_idx": g("idx", np.int64), "distance": g("dist", np.int64),
                "ok": g("ok", np.int32).astype(bool),
                "points": self._h("pts", np.float64, (S, ck, 3))[s, :n_left].copy(),
                "slots": g("slots", np.int64),
                "n_slots": int(self._h("slot_n", np.int32, (S,))[s])}
