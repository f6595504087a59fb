"""Device runtime for the drop-in calls: one CUDA device, one stream, packed
pinned staging, a growable device arena (the BufferPool analogue, reference
buffers.py:13-55) and the C-ABI parameter builders.

Every drop-in call packs its numpy inputs into ONE pinned host buffer and
issues ONE host->device copy, launches the fused kernel(s) through the C ABI
on the runtime's stream, and reads its outputs back with ONE device->host
copy.  Buffers only grow, so steady-state calls allocate nothing.

PyTorch provides device memory, pinned memory and streams (plumbing); all
compute runs in libfasttrack_b200.so.
"""

from __future__ import annotations

import math
import threading

import numpy as np
import torch

from . import _lib
from .types import is_fisheye

ALIGN = 256


def _align(n: int) -> int:
    return (int(n) + ALIGN - 1) // ALIGN * ALIGN


class Layout:
    """Named byte ranges packed at 256-B alignment."""

    def __init__(self) -> None:
        self.offsets: dict[str, int] = {}
        self.sizes: dict[str, int] = {}
        self.total = 0

    def add(self, name: str, nbytes: int) -> int:
        off = self.total
        self.offsets[name] = off
        self.sizes[name] = int(nbytes)
        self.total = off + _align(max(int(nbytes), 1))
        return off


class Runtime:
    """Per-device state shared by the drop-in functions (single tracking
    thread, like the reference engine; guarded by a lock for safety)."""

    def __init__(self, device: int | None = None):
        if not torch.cuda.is_available():
            raise _lib.FtError("no CUDA device: the B200 path has no CPU fallback")
        self.lib = _lib.load()
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        with torch.cuda.device(self.device):
            self.stream = torch.cuda.Stream(self.device)
        self.lock = threading.RLock()
        self._dev = torch.empty(0, dtype=torch.uint8, device=self.device)
        self._host = torch.empty(0, dtype=torch.uint8).pin_memory()
        self._hnp = self._host.numpy()
        self._ws = torch.empty(0, dtype=torch.uint8, device=self.device)
        self._ws_key = None
        self.cap_kp = 1024
        self.cap_pts = 1024

    # -- memory ---------------------------------------------------------------

    def reserve(self, nbytes: int) -> None:
        if nbytes > self._dev.numel():
            cap = _align(max(nbytes, 2 * self._dev.numel(), 1 << 20))
            self._dev = torch.zeros(cap, dtype=torch.uint8, device=self.device)
        if nbytes > self._host.numel():
            cap = _align(max(nbytes, 2 * self._host.numel(), 1 << 20))
            self._host = torch.zeros(cap, dtype=torch.uint8).pin_memory()
            self._hnp = self._host.numpy()

    @property
    def dev_base(self) -> int:
        return self._dev.data_ptr()

    def host_view(self, lay: Layout, name: str, dtype, shape) -> np.ndarray:
        off = lay.offsets[name]
        n = int(np.prod(shape)) * np.dtype(dtype).itemsize
        return self._hnp[off:off + n].view(dtype).reshape(shape)

    def put(self, lay: Layout, name: str, arr, dtype) -> None:
        arr = np.asarray(arr)
        view = self.host_view(lay, name, dtype, arr.shape)
        np.copyto(view, arr, casting="unsafe" if arr.dtype != np.dtype(dtype) else "no")

    def ptr(self, lay: Layout, name: str) -> int:
        return self.dev_base + lay.offsets[name]

    def h2d(self, begin: int, end: int) -> None:
        if end > begin:
            with torch.cuda.stream(self.stream):
                self._dev[begin:end].copy_(self._host[begin:end], non_blocking=True)

    def d2h(self, begin: int, end: int) -> None:
        if end > begin:
            with torch.cuda.stream(self.stream):
                self._host[begin:end].copy_(self._dev[begin:end], non_blocking=True)

    def sync(self) -> None:
        self.stream.synchronize()

    def caps(self, n_kp: int, n_pts: int = 0) -> tuple[int, int]:
        """High-water capacities (multiples of 256 keypoints / 1024 points,
        >= 1024) for single-frame calls; every launch of this runtime uses
        them so the workspace layout only changes when they grow."""
        if n_kp > self.cap_kp:
            self.cap_kp = (n_kp + 255) // 256 * 256
        if n_pts > self.cap_pts:
            self.cap_pts = (n_pts + 1023) // 1024 * 1024
        return self.cap_kp, self.cap_pts

    def workspace(self) -> _lib.FtWorkspace:
        """The C-ABI workspace for single-frame launches at the high-water
        caps, (re)initialised when the caps grow."""
        key = (1, self.cap_kp, self.cap_pts)
        if self._ws_key != key:
            self._ws_struct = make_workspace(self.lib, self.device, self.stream, *key)
            self._ws = self._ws_struct._tensor
            self._ws_key = key
        return self._ws_struct


def make_workspace(lib, device, stream, n_frames: int, cap_left: int,
                   cap_points: int) -> _lib.FtWorkspace:
    """Allocate + initialise an ft_workspace; the struct keeps its tensor alive."""
    nbytes = int(lib.ft_workspace_bytes(n_frames, cap_left, cap_points))
    t = torch.empty(_align(nbytes), dtype=torch.uint8, device=device)
    ws = _lib.FtWorkspace(t.data_ptr(), t.numel(), n_frames, cap_left, cap_points)
    ws._tensor = t
    _lib.check(lib.ft_workspace_init(ws, stream.cuda_stream), "ft_workspace_init")
    return ws


_RUNTIMES: dict[int, Runtime] = {}


def runtime() -> Runtime:
    dev = torch.cuda.current_device() if torch.cuda.is_available() else -1
    rt = _RUNTIMES.get(dev)
    if rt is None:
        rt = Runtime()
        _RUNTIMES[dev] = rt
    return rt


# ---------------------------------------------------------------------------
# parameter builders (C structs from the reference dataclasses)

def stereo_params(cfg, height: int, scale_pow, baseline_times_fx: float) -> _lib.FtStereoParams:
    sp = np.asarray(scale_pow, dtype=np.float64)
    if len(sp) > _lib.FT_MAX_LEVELS or len(sp) < 1:
        raise ValueError(f"need 1..{_lib.FT_MAX_LEVELS} pyramid levels, got {len(sp)}")
    p = _lib.FtStereoParams()
    p.t_match = int(cfg.t_match)
    p.band_factor = float(cfg.band_factor)
    p.min_disparity = float(cfg.min_disparity)
    p.max_disparity = float(cfg.max_disparity)
    p.half_window = int(cfg.half_window)
    p.half_slide = int(cfg.half_slide)
    p.outlier_multiplier = float(cfg.outlier_multiplier)
    p.ratio = float(cfg.ratio)
    p.baseline_times_fx = float(baseline_times_fx)
    p.height = int(height)
    p.n_levels = len(sp)
    for i, x in enumerate(sp):
        p.scale_pow[i] = float(x)
    return p


def project_params(cam, cfg, scale: float, levels: int, grid_cell: int, grid_nx: int,
                   grid_ny: int, window_px: float | None, u_offset: float) -> _lib.FtProjectParams:
    """projection.py:136-157 argument list of project_search_kernel."""
    if levels < 1 or levels > _lib.FT_MAX_LEVELS:
        raise ValueError(f"need 1..{_lib.FT_MAX_LEVELS} levels, got {levels}")
    p = _lib.FtProjectParams()
    if is_fisheye(cam):
        p.cam_kind = 1
        p.k1, p.k2, p.k3, p.k4 = (float(cam.k1), float(cam.k2), float(cam.k3), float(cam.k4))
    else:
        p.cam_kind = 0
        p.k1 = p.k2 = p.k3 = p.k4 = 0.0
    p.fx, p.fy, p.cx, p.cy = float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy)
    p.width, p.height = float(cam.width), float(cam.height)
    p.cell_px, p.grid_nx, p.grid_ny = int(grid_cell), int(grid_nx), int(grid_ny)
    p.n_levels = int(levels)
    sp = scale ** np.arange(levels, dtype=np.float64)
    for i, x in enumerate(sp):
        p.scale_pow[i] = float(x)
    p.inv_log_scale = 1.0 / math.log(scale)
    p.window_px = float(cfg.window_px if window_px is None else window_px)
    p.t_proj = int(cfg.t_proj)
    p.ratio = float(cfg.ratio)
    p.view_cos_min = float(cfg.view_cos_min)
    p.u_offset = float(u_offset)
    p.histogram_bins = int(cfg.histogram_bins)
    p.histogram_keep = int(cfg.histogram_keep)
    return p


def pyramid_struct(pyr, data_ptr: int, frame_bytes: int) -> _lib.FtPyramid:
    s = _lib.FtPyramid()
    n = len(pyr.widths)
    if n > _lib.FT_MAX_LEVELS:
        raise ValueError(f"at most {_lib.FT_MAX_LEVELS} pyramid levels")
    s.data = data_ptr
    s.frame_bytes = int(frame_bytes)
    s.n_levels = n
    for i in range(n):
        s.offsets[i] = int(pyr.offsets[i])
        s.widths[i] = int(pyr.widths[i])
        s.heights[i] = int(pyr.heights[i])
    return s


def keypoints_struct(rt: Runtime, lay: Layout, prefix: str, cap: int) -> _lib.FtKeypoints:
    k = _lib.FtKeypoints()
    k.rec = rt.ptr(lay, f"{prefix}_rec")
    k.count = rt.ptr(lay, f"{prefix}_n")
    k.cap = int(cap)
    return k


def add_keypoints(lay: Layout, prefix: str, cap: int, with_angle: bool = False) -> None:
    lay.add(f"{prefix}_n", 4)
    lay.add(f"{prefix}_rec", _lib.KP_RECORD.itemsize * cap)


def fill_kp_records(rec: np.ndarray, feats, with_angle: bool = False) -> int:
    """Pack a FeatureSet (reference SoA layout) into ft_kp_record rows
    (ft_host_pack_keypoints: a C loop over the arrays, passed in place)."""
    from . import session as S
    n = len(feats.u)
    if n:
        if len(rec) < n or not rec.flags.c_contiguous or rec.dtype != _lib.KP_RECORD:
            raise ValueError("record buffer: contiguous ft_kp_record rows, >= n")
        keep: list = []
        _lib.check(S.lib().ft_host_pack_keypoints(S.features(feats, with_angle, keep),
                                                  rec.ctypes.data), "ft_host_pack_keypoints")
    return n


def fill_point_records(rec: np.ndarray, pts) -> int:
    """Pack a MapPointSoA into ft_point_record rows (ft_host_pack_points)."""
    from . import session as S
    m = len(pts.point_ids)
    if m:
        if len(rec) < m or not rec.flags.c_contiguous or rec.dtype != _lib.POINT_RECORD:
            raise ValueError("record buffer: contiguous ft_point_record rows, >= m")
        keep: list = []
        _lib.check(S.lib().ft_host_pack_points(S.points(pts, keep), rec.ctypes.data),
                   "ft_host_pack_points")
    return m


def put_keypoints(rt: Runtime, lay: Layout, prefix: str, feats, with_angle: bool = False) -> int:
    n = len(feats.u)
    rt.put(lay, f"{prefix}_n", np.array([n], dtype=np.int32), np.int32)
    if n:
        rec = rt.host_view(lay, f"{prefix}_rec", _lib.KP_RECORD, (n,))
        fill_kp_records(rec, feats, with_angle)
    return n


def bind_host_to_gpu_numa(device: int = 0) -> list[int] | None:
    """Restrict this process's CPUs to the NUMA node of the GPU's PCIe root
    (sysfs local_cpulist), so pinned staging memory is allocated node-local
    and host <-> device copies do not cross the socket interconnect.  Call
    before allocating pinned memory.  Returns the CPU list, or None when the
    topology is unavailable (no-op)."""
    import os
    try:
        p = torch.cuda.get_device_properties(device)
        bdf = f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
        with open(f"/sys/bus/pci/devices/{bdf}/local_cpulist") as fp:
            spec = fp.read().strip()
        cpus = []
        for part in spec.split(","):
            if "-" in part:
                a, b = part.split("-")
                cpus.extend(range(int(a), int(b) + 1))
            elif part:
                cpus.append(int(part))
        avail = os.sched_getaffinity(0)
        cpus = [c for c in cpus if c in avail]
        if not cpus or len(cpus) == len(avail):
            return None
        os.sched_setaffinity(0, cpus)
        return cpus
    except (OSError, AttributeError, ValueError, RuntimeError):
        return None
