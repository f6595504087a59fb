"""Load the committed golden fixtures (tests/golden/*.npz) into the
package's reference-shaped types.  Test infrastructure only."""

from __future__ import annotations

from pathlib import Path

import numpy as np

from paper_2509_10757_b200.types import (FeatureSet, FisheyeCamera, FrameGrid, ImagePyramid,
                                         LocalMap, MapPointSoA, PinholeCamera, Pose)

GOLDEN = Path(__file__).resolve().parent / "golden"


def load(name: str) -> dict:
    with np.load(GOLDEN / name) as z:
        return {k: z[k] for k in z.files}


def feats(d: dict, prefix: str) -> FeatureSet:
    return FeatureSet(u=d[f"{prefix}_u"], v=d[f"{prefix}_v"], octave=d[f"{prefix}_octave"],
                      angle=d[f"{prefix}_angle"], response=d[f"{prefix}_response"],
                      descriptors=d[f"{prefix}_desc"])


def soa(d: dict, prefix: str = "map") -> MapPointSoA:
    return MapPointSoA(positions=d[f"{prefix}_positions"], descriptors=d[f"{prefix}_descriptors"],
                       normals=d[f"{prefix}_normals"], min_distances=d[f"{prefix}_min_d"],
                       max_distances=d[f"{prefix}_max_d"], point_ids=d[f"{prefix}_ids"])


def local_map(d: dict) -> LocalMap:
    s = soa(d)
    return LocalMap((0,), s.point_ids.copy(), s)


def pose(d: dict, prefix: str = "pose") -> Pose:
    return Pose(d[f"{prefix}_rot"], d[f"{prefix}_trans"])


def pyramid(d: dict, side: str, scale: float = 1.2) -> ImagePyramid:
    p = f"pyr_{side}"
    return ImagePyramid(d[f"{p}_data"], d[f"{p}_offsets"], d[f"{p}_widths"],
                        d[f"{p}_heights"], scale)


def pinhole() -> PinholeCamera:
    """synthetic.py:53-55 default_pinhole (EuRoC shape)."""
    return PinholeCamera(fx=458.0, fy=458.0, cx=376.0, cy=240.0,
                         baseline_times_fx=458.0 * 0.11, width=752, height=480)


def fisheye() -> FisheyeCamera:
    """SURVEY.md §8(d) cfg3 camera (TUM-VI shape)."""
    return FisheyeCamera(fx=190.0, fy=190.0, cx=256.0, cy=256.0, k1=0.003, k2=-0.002,
                         k3=0.001, k4=-0.0005, width=512, height=512,
                         right_extrinsic=Pose(np.eye(3), np.array([-0.1, 0.0, 0.0])))


def grid_tuple(u, v, cam, cell_px: int = 48):
    g = FrameGrid(u, v, cam.width, cam.height, cell_px)
    return g.start, g.indices, g.nx, g.ny, g.cell_px


# ---------------------------------------------------------------------------
# cfg4: the reference StereoTracker's per-frame stage calls (make_golden.gen_cfg4)

def digest(*arrays) -> np.ndarray:
    """Same sha256 as make_golden.digest (dtype, shape, raw bytes)."""
    import hashlib
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype.str).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return np.frombuffer(h.digest(), dtype=np.uint8).copy()


class Cfg4:
    """One captured 100-frame sequence (trajectory "line" or "circle")."""

    def __init__(self, trajectory: str):
        self.d = load(f"cfg4_{trajectory}.npz")
        self.n_frames = int(self.d["n_frames"])
        self.n_points = len(self.d["world_min_d"])
        self.cam = pinhole()
        self._feats = {}

    def has(self, i: int, key: str) -> bool:
        return f"f{i}_{key}" in self.d

    def get(self, i: int, key: str):
        return self.d[f"f{i}_{key}"]

    def feats(self, i: int, side: str) -> FeatureSet:
        """Frame i's left ("l") or right ("r") feature bundle, rebuilt exactly:
        descriptors / angles are the landmarks' (synthetic.py:160-174)."""
        key = (i, side)
        if key not in self._feats:
            ids = self.get(i, f"{side}_ids").astype(np.int64)
            uv = self.get(i, f"{side}_uv")
            n = len(ids)
            self._feats[key] = FeatureSet(
                u=uv[0].copy(), v=uv[1].copy(), octave=self.get(i, f"{side}_octave").astype(np.int32),
                angle=self.d["landmark_angle"][ids].copy(),
                response=np.full(n, 100.0, dtype=np.float32),
                descriptors=self.d["landmark_desc"][ids].copy())
        return self._feats[key]

    def pose(self, i: int, key: str) -> Pose:
        p = self.get(i, key)
        return Pose(p[:9].reshape(3, 3).copy(), p[9:].copy())

    def world_soa(self, ids) -> MapPointSoA:
        ids = np.asarray(ids, dtype=np.int64)
        d = self.d
        return MapPointSoA(positions=d["world_positions"][ids], descriptors=d["world_descriptors"][ids],
                           normals=d["world_normals"][ids], min_distances=d["world_min_d"][ids],
                           max_distances=d["world_max_d"][ids], point_ids=ids.copy())

    def local_ids(self, i: int) -> np.ndarray:
        m = np.unpackbits(self.get(i, "local_mask"))[:self.n_points].astype(bool)
        return np.nonzero(m)[0].astype(np.int64)

    def local_map(self, i: int) -> LocalMap:
        ids = self.local_ids(i)
        return LocalMap((), ids, self.world_soa(ids))

    def world(self):
        """Minimal host WorldMap: the MapPoint fields decompose_map_points reads."""
        from types import SimpleNamespace
        d = self.d

        class _Pts(dict):
            def __missing__(s, pid):
                v = SimpleNamespace(point_id=int(pid), position=d["world_positions"][pid],
                                    descriptor=d["world_descriptors"][pid],
                                    normal=d["world_normals"][pid],
                                    min_distance=float(d["world_min_d"][pid]),
                                    max_distance=float(d["world_max_d"][pid]))
                s[pid] = v
                return v

        pts = _Pts()
        return SimpleNamespace(points=pts, points_by_ids=lambda ids: [pts[int(i)] for i in ids])

    def frame(self, i: int, pose: Pose, slots=None):
        """The tracker's Frame for frame i (tracker.py:285-290)."""
        from paper_2509_10757_b200.types import Frame
        left, right = self.feats(i, "l"), self.feats(i, "r")
        g = FrameGrid(left.u, left.v, self.cam.width, self.cam.height, 48)
        n = len(left.u)
        s = np.full(n, -1, np.int64) if slots is None else np.asarray(slots, np.int64).copy()
        return Frame(i, 0.0, left, right, np.full(n, -1.0), s, pose, g)

    def growing_world(self):
        """The reference WorldMap as the tracker grew it (advance(n_kf, n_pts)
        before frame i with its update_n_keyframes / update_n_points)."""
        return _GrowingWorld(self)


class _KF:
    """KeyFrame.observed_point_ids (mapping.py:142-145) of a captured keyframe."""

    def __init__(self, ids):
        self._ids = ids

    def observed_point_ids(self):
        return self._ids


class _GrowingWorld:
    """Keyframes and map points appear in creation order (ids sequential);
    both are immutable once created (the reference tracker only appends)."""

    def __init__(self, seq):
        self.seq, self.points, self.keyframes = seq, {}, {}

    def advance(self, n_kf, n_pts):
        from types import SimpleNamespace
        d = self.seq.d
        for k in range(len(self.keyframes), n_kf):
            self.keyframes[k] = _KF(d["kf_obs"][d["kf_off"][k]:d["kf_off"][k + 1]].astype(np.int64))
        for p in range(len(self.points), n_pts):
            self.points[p] = SimpleNamespace(point_id=p, position=d["world_positions"][p],
                                             descriptor=d["world_descriptors"][p],
                                             normal=d["world_normals"][p],
                                             min_distance=float(d["world_min_d"][p]),
                                             max_distance=float(d["world_max_d"][p]))
