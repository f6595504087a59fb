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
