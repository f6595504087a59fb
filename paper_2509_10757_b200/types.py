"""Host-side data model of the hot path, mirroring the reference's types.

The drop-in functions only read attributes by name, so the reference's own
objects (``trackfront.mapping.FeatureSet`` etc.) work unchanged; these classes
exist so the package is usable where the reference is not installed (the GPU
box).  Field names, dtypes, defaults and validation follow the reference:

* ``StereoMatchConfig``        reference stereo.py:22-42
* ``StereoMatches``            reference stereo.py:45-64
* ``ProjectionSearchConfig``   reference projection.py:26-45
* ``Correspondences``          reference projection.py:48-67
* ``FeatureSet``               reference mapping.py:18-65
* ``FrameGrid``                reference mapping.py:68-100
* ``Frame``                    reference mapping.py:103-128
* ``MapPointSoA``              reference mapping.py:163-201
* ``LocalMap``                 reference localmap.py:22-39
* ``ImagePyramid``             reference extraction.py:67-94
* ``Pose``                     reference geometry.py:61-111 (x_cam = R x_w + t)
* ``PinholeCamera`` / ``FisheyeCamera``  reference cameras.py:18-157
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

NO_DEPTH = -1.0
NO_POINT = -1
DEFAULT_GRID_CELL_PX = 48
UNMATCHED_DISTANCE = 10000


# ---------------------------------------------------------------------------
# configs

@dataclass(frozen=True)
class StereoMatchConfig:
    t_match: int = 100
    band_factor: float = 2.0
    min_disparity: float = 0.1
    max_disparity: float = 376.0
    half_window: int = 5
    half_slide: int = 5
    outlier_multiplier: float = 2.0
    ratio: float = 0.8
    ray_gap_ceiling: float = 0.05

    def __post_init__(self) -> None:
        if not 0 < self.t_match <= 256:
            raise ValueError("t_match must be in (0, 256]")
        if self.min_disparity < 0 or self.max_disparity <= self.min_disparity:
            raise ValueError("need 0 <= min_disparity < max_disparity")
        if self.half_window < 1 or self.half_slide < 1:
            raise ValueError("window and slide half-sizes must be >= 1")
        if not 0 < self.ratio <= 1:
            raise ValueError("ratio must be in (0, 1]")


@dataclass(frozen=True)
class ProjectionSearchConfig:
    window_px: float = 5.7
    window_prev_px: float = 15.0
    t_proj: int = 100
    ratio: float = 0.9
    view_cos_min: float = 0.5
    histogram_bins: int = 30
    histogram_keep: int = 3
    rotation_check_prev: bool = True
    rotation_check_local: bool = False
    prev_u_offset_px: float = 1.0

    def __post_init__(self) -> None:
        if self.window_px <= 0 or not 0 < self.ratio <= 1:
            raise ValueError("need window_px > 0 and ratio in (0, 1]")
        if not -1 <= self.view_cos_min <= 1:
            raise ValueError("view_cos_min must be in [-1, 1]")
        if self.histogram_bins < 1 or not 1 <= self.histogram_keep <= self.histogram_bins:
            raise ValueError("need 1 <= histogram_keep <= histogram_bins")


# ---------------------------------------------------------------------------
# results

@dataclass
class StereoMatches:
    right_idx: np.ndarray   # int64 [n], -1 when unmatched
    distance: np.ndarray    # int64 [n], 10000 when unmatched
    disparity: np.ndarray   # float64 [n]
    refined_u: np.ndarray   # float64 [n]
    depth: np.ndarray       # float64 [n]
    sad: np.ndarray         # int64 [n]

    def matched_mask(self) -> np.ndarray:
        return self.right_idx >= 0

    def n_matched(self) -> int:
        return int(np.count_nonzero(self.right_idx >= 0))


@dataclass
class Correspondences:
    point_idx: np.ndarray
    keypoint_idx: np.ndarray
    distance: np.ndarray
    octave: np.ndarray

    def __len__(self) -> int:
        return len(self.point_idx)

    @staticmethod
    def empty() -> "Correspondences":
        return Correspondences(*(np.empty(0, dtype=np.int64) for _ in range(4)))


# ---------------------------------------------------------------------------
# geometry / cameras

@dataclass(frozen=True)
class Pose:
    """World-to-camera transform ``x_cam = rotation @ x_world + translation``."""

    rotation: np.ndarray
    translation: np.ndarray

    def __post_init__(self) -> None:
        object.__setattr__(self, "rotation",
                           np.asarray(self.rotation, dtype=np.float64).reshape(3, 3))
        object.__setattr__(self, "translation",
                           np.asarray(self.translation, dtype=np.float64).reshape(3))

    @staticmethod
    def identity() -> "Pose":
        return Pose(np.eye(3), np.zeros(3))

    def inverse(self) -> "Pose":
        rt = self.rotation.T
        return Pose(rt, -rt @ self.translation)

    def matrix(self) -> np.ndarray:
        m = np.eye(4)
        m[:3, :3] = self.rotation
        m[:3, 3] = self.translation
        return m

    def transform(self, pts: np.ndarray) -> np.ndarray:
        pts = np.asarray(pts, dtype=np.float64)
        if pts.ndim == 1:
            return self.rotation @ pts + self.translation
        return pts @ self.rotation.T + self.translation


@dataclass(frozen=True)
class PinholeCamera:
    fx: float
    fy: float
    cx: float
    cy: float
    baseline_times_fx: float
    width: int
    height: int

    def __post_init__(self) -> None:
        if self.fx <= 0 or self.fy <= 0 or self.baseline_times_fx <= 0:
            raise ValueError("focal lengths and baseline_times_fx must be positive")
        if not (0 <= self.cx < self.width and 0 <= self.cy < self.height):
            raise ValueError("principal point outside image")

    @property
    def baseline(self) -> float:
        return self.baseline_times_fx / self.fx


@dataclass(frozen=True)
class FisheyeCamera:
    """Kannala-Brandt: r(theta) = theta (1 + k1 t^2 + k2 t^4 + k3 t^6 + k4 t^8)."""

    fx: float
    fy: float
    cx: float
    cy: float
    k1: float
    k2: float
    k3: float
    k4: float
    width: int
    height: int
    right_extrinsic: Pose = field(default_factory=Pose.identity)

    def unproject(self, u: float, v: float) -> np.ndarray:
        """Unit ray through a pixel: Newton inversion of the radial polynomial
        (reference cameras.py:139-157; used by the host-side triangulation)."""
        mx = (u - self.cx) / self.fx
        my = (v - self.cy) / self.fy
        rd = float(np.hypot(mx, my))
        if rd < 1e-12:
            return np.array([0.0, 0.0, 1.0])
        theta = min(rd, np.pi / 2)
        for _ in range(20):
            t2 = theta * theta
            f = theta * (1.0 + t2 * (self.k1 + t2 * (self.k2 + t2 * (self.k3 + t2 * self.k4)))) - rd
            df = 1.0 + t2 * (3 * self.k1 + t2 * (5 * self.k2 + t2 * (7 * self.k3 + t2 * 9 * self.k4)))
            step = f / df
            theta -= step
            if abs(step) < 1e-14:
                break
        s = np.sin(theta) / rd
        ray = np.array([s * mx, s * my, np.cos(theta)])
        return ray / np.linalg.norm(ray)


def is_fisheye(cam) -> bool:
    """Duck-typed camera kind (the reference dispatches on isinstance,
    projection.py:110-115; a KB fisheye is the one with distortion terms)."""
    return hasattr(cam, "k1")


# ---------------------------------------------------------------------------
# features, grids, frames, map points

@dataclass
class FeatureSet:
    u: np.ndarray
    v: np.ndarray
    octave: np.ndarray
    angle: np.ndarray
    response: np.ndarray
    descriptors: np.ndarray   # uint64 [n, 4]: bit b -> word b >> 6, bit b & 63

    def __len__(self) -> int:
        return len(self.u)

    @staticmethod
    def empty() -> "FeatureSet":
        return FeatureSet(np.empty(0), np.empty(0), np.empty(0, dtype=np.int32), np.empty(0),
                          np.empty(0, dtype=np.float32), np.zeros((0, 4), dtype=np.uint64))


class FrameGrid:
    """CSR of keypoint indices over square cells (level-0 pixels)."""

    def __init__(self, u: np.ndarray, v: np.ndarray, width: int, height: int,
                 cell_px: int = DEFAULT_GRID_CELL_PX):
        self.cell_px = int(cell_px)
        self.nx = max(1, (int(width) + self.cell_px - 1) // self.cell_px)
        self.ny = max(1, (int(height) + self.cell_px - 1) // self.cell_px)
        cx = np.clip((np.asarray(u) / self.cell_px).astype(np.int64), 0, self.nx - 1)
        cy = np.clip((np.asarray(v) / self.cell_px).astype(np.int64), 0, self.ny - 1)
        cell = cy * self.nx + cx
        self.indices = np.argsort(cell, kind="stable").astype(np.int64)
        self.start = np.zeros(self.nx * self.ny + 1, dtype=np.int64)
        np.cumsum(np.bincount(cell, minlength=self.nx * self.ny), out=self.start[1:])
        self._n = len(u)

    def __len__(self) -> int:
        return self._n


@dataclass
class Frame:
    frame_id: int
    timestamp: float
    left: FeatureSet
    right: FeatureSet
    depth: np.ndarray
    slots: np.ndarray
    pose: Pose
    grid: FrameGrid

    @property
    def n_keypoints(self) -> int:
        return len(self.left)

    def slotted_point_ids(self) -> np.ndarray:
        return np.unique(self.slots[self.slots != NO_POINT])


@dataclass
class MapPointSoA:
    positions: np.ndarray      # (m, 3) float64
    descriptors: np.ndarray    # (m, 4) uint64
    normals: np.ndarray        # (m, 3) float64
    min_distances: np.ndarray  # (m,) float64
    max_distances: np.ndarray  # (m,) float64
    point_ids: np.ndarray      # (m,) int64

    def __len__(self) -> int:
        return len(self.point_ids)

    @staticmethod
    def empty() -> "MapPointSoA":
        return MapPointSoA(np.empty((0, 3)), np.zeros((0, 4), dtype=np.uint64), np.empty((0, 3)),
                           np.empty(0), np.empty(0), np.empty(0, dtype=np.int64))


@dataclass
class LocalMap:
    keyframe_ids: tuple
    point_ids: np.ndarray      # ascending ids
    soa: MapPointSoA

    def __len__(self) -> int:
        return len(self.point_ids)

    @staticmethod
    def empty() -> "LocalMap":
        return LocalMap((), np.empty(0, dtype=np.int64), MapPointSoA.empty())


class ImagePyramid:
    """Flat u8 multi-level image: level l at data[offsets[l]:offsets[l+1]],
    shaped (heights[l], widths[l])."""

    def __init__(self, data, offsets, widths, heights, scale: float):
        self.data = data
        self.offsets = offsets
        self.widths = widths
        self.heights = heights
        self.scale = scale

    @property
    def n_levels(self) -> int:
        return len(self.widths)

    @property
    def nbytes(self) -> int:
        return int(self.offsets[-1])

    def level(self, i: int) -> np.ndarray:
        flat = self.data[self.offsets[i]:self.offsets[i + 1]]
        return flat.reshape(self.heights[i], self.widths[i])
