"""Seeded synthetic workloads for the benchmarks and parity tests.

EuRoC-shaped pinhole stereo (752x480, fx=fy=458, baseline 0.11 m) and
TUM-VI-shaped Kannala-Brandt fisheye (512x512) frames built the way the
reference's SURVEY.md §8(d) recipes describe: landmarks on a cylindrical
shell around the camera, ground-truth feature bundles with pixel noise,
octave from distance, per-landmark 256-bit descriptors, a local map of the
visible landmarks plus random others (normals, [min, max] distances, 8 bit
flips), a slightly perturbed query pose, and optionally rendered textured
images with an 8-level, scale-1.2 pyramid so stereo phase 2 has pixels.

This is fixture generation (the reference keeps the equivalent in
synthetic.py); the hot path never calls it.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from paper_2509_10757_b200.types import (FeatureSet, FisheyeCamera, Frame, FrameGrid, ImagePyramid, LocalMap,
                    MapPointSoA, PinholeCamera, Pose, NO_POINT)

EXTENT = 8.0
LEVELS = 8
SCALE = 1.2


def euroc_camera() -> PinholeCamera:
    return PinholeCamera(fx=458.0, fy=458.0, cx=376.0, cy=240.0,
                         baseline_times_fx=458.0 * 0.11, width=752, height=480)


def tumvi_camera() -> FisheyeCamera:
    return FisheyeCamera(fx=190.0, fy=190.0, cx=256.0, cy=256.0, k1=0.003, k2=-0.002,
                         k3=0.001, k4=-0.0005, width=512, height=512,
                         right_extrinsic=Pose(np.eye(3), np.array([-0.1, 0.0, 0.0])))


def _rot_axis(axis: np.ndarray, ang: float) -> np.ndarray:
    axis = axis / np.linalg.norm(axis)
    k = np.array([[0, -axis[2], axis[1]], [axis[2], 0, -axis[0]], [-axis[1], axis[0], 0]])
    return np.eye(3) + math.sin(ang) * k + (1 - math.cos(ang)) * (k @ k)


def _project(cam, pc: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    x, y, z = pc[:, 0], pc[:, 1], pc[:, 2]
    if hasattr(cam, "k1"):
        r = np.hypot(x, y)
        th = np.arctan2(r, z)
        t2 = th * th
        d = th * (1 + t2 * (cam.k1 + t2 * (cam.k2 + t2 * (cam.k3 + t2 * cam.k4))))
        rs = np.where(r < 1e-12, 1.0, r)
        u = np.where(r < 1e-12, cam.cx, cam.fx * d * x / rs + cam.cx)
        v = np.where(r < 1e-12, cam.cy, cam.fy * d * y / rs + cam.cy)
        ok = (z > 0.05) & (th < 1.45)
    else:
        zs = np.where(z > 1e-6, z, 1.0)
        u = cam.fx * x / zs + cam.cx
        v = cam.fy * y / zs + cam.cy
        ok = z > 1e-6
    ok &= (u >= 0) & (u < cam.width) & (v >= 0) & (v < cam.height)
    return np.stack([u, v], axis=1), ok


def _octave(dist: np.ndarray) -> np.ndarray:
    o = np.floor(np.log(np.maximum(EXTENT / np.maximum(dist, 1e-6), 1.0)) / math.log(SCALE))
    return np.clip(o, 0, LEVELS - 1).astype(np.int32)


def _flip(desc: np.ndarray, rng, nflip: int) -> np.ndarray:
    out = desc.copy()
    if nflip <= 0:
        return out
    bits = np.argsort(rng.random((len(out), 256)), axis=1)[:, :nflip]
    for c in range(nflip):
        b = bits[:, c]
        out[np.arange(len(out)), b >> 6] ^= (np.uint64(1) << (b & 63).astype(np.uint64))
    return out


def _view(cam, pose: Pose, lm, desc, ang, rng, noise_px: float, nflip: int):
    pc = pose.transform(lm)
    uv, ok = _project(cam, pc)
    ids = np.nonzero(ok)[0]
    uv = uv[ids] + rng.normal(0.0, noise_px, size=(len(ids), 2))
    inb = (uv[:, 0] >= 0) & (uv[:, 0] < cam.width) & (uv[:, 1] >= 0) & (uv[:, 1] < cam.height)
    ids, uv = ids[inb], uv[inb]
    dist = np.linalg.norm(pc[ids], axis=1)
    fs = FeatureSet(u=uv[:, 0].copy(), v=uv[:, 1].copy(), octave=_octave(dist),
                    angle=ang[ids].copy(), response=np.full(len(ids), 100.0, np.float32),
                    descriptors=_flip(desc[ids], rng, nflip))
    return fs, ids


def _binomial5(img: np.ndarray) -> np.ndarray:
    w = np.array([1, 4, 6, 4, 1], dtype=np.int64)
    a = img.astype(np.int64)
    p = np.pad(a, ((0, 0), (2, 2)), mode="reflect")
    t = sum(w[k] * p[:, k:k + a.shape[1]] for k in range(5))
    p = np.pad(t, ((2, 2), (0, 0)), mode="reflect")
    t = sum(w[k] * p[k:k + a.shape[0], :] for k in range(5))
    return ((t + 128) >> 8).astype(np.uint8)


def _resample(src: np.ndarray, hd: int, wd: int) -> np.ndarray:
    hs, ws = src.shape
    fy = (np.arange(hd) + 0.5) * (hs / hd) - 0.5
    fx = (np.arange(wd) + 0.5) * (ws / wd) - 0.5
    y0, x0 = np.floor(fy).astype(np.int64), np.floor(fx).astype(np.int64)
    ay, ax = (fy - y0)[:, None], (fx - x0)[None, :]
    y0c, y1c = np.clip(y0, 0, hs - 1), np.clip(y0 + 1, 0, hs - 1)
    x0c, x1c = np.clip(x0, 0, ws - 1), np.clip(x0 + 1, 0, ws - 1)
    s = src.astype(np.float64)
    top = (1 - ax) * s[y0c][:, x0c] + ax * s[y0c][:, x1c]
    bot = (1 - ax) * s[y1c][:, x0c] + ax * s[y1c][:, x1c]
    return np.clip((1 - ay) * top + ay * bot + 0.5, 0, 255).astype(np.uint8)


def build_pyramid(img: np.ndarray, levels: int = LEVELS, scale: float = SCALE) -> ImagePyramid:
    """Flat u8 pyramid: level l = bilinear(binomial5(level l-1)) at
    floor(dims / scale^l) (layout of reference extraction.py:67-125)."""
    h, w = img.shape
    pw = scale ** np.arange(levels, dtype=np.float64)
    ws = np.floor(w / pw).astype(np.int64)
    hs = np.floor(h / pw).astype(np.int64)
    offs = np.zeros(levels + 1, dtype=np.int64)
    np.cumsum(ws * hs, out=offs[1:])
    data = np.empty(int(offs[-1]), dtype=np.uint8)
    cur = img
    data[:h * w] = img.ravel()
    for lvl in range(1, levels):
        cur = _resample(_binomial5(cur), int(hs[lvl]), int(ws[lvl]))
        data[offs[lvl]:offs[lvl + 1]] = cur.ravel()
    return ImagePyramid(data, offs, ws, hs, scale)


def _render(cam, pose: Pose, lm: np.ndarray, tex: np.ndarray) -> np.ndarray:
    """Textured dot per visible landmark, bilinearly splatted, max-combined."""
    h, w = int(cam.height), int(cam.width)
    img = np.full(h * w, 15.0)
    uv, ok = _project(cam, pose.transform(lm))
    ids = np.nonzero(ok)[0]
    half = tex.shape[1] // 2
    size = tex.shape[1]
    for i in ids:
        u, v = uv[i]
        x0, y0 = int(math.floor(u)), int(math.floor(v))
        fx, fy = u - x0, v - y0
        t = tex[i]
        c = np.zeros((size + 1, size + 1))
        c[:size, :size] += t * (1 - fx) * (1 - fy)
        c[:size, 1:] += t * fx * (1 - fy)
        c[1:, :size] += t * (1 - fx) * fy
        c[1:, 1:] += t * fx * fy
        ys, xs = y0 - half, x0 - half
        yy, xx = np.mgrid[ys:ys + size + 1, xs:xs + size + 1]
        m = (yy >= 0) & (yy < h) & (xx >= 0) & (xx < w)
        np.maximum.at(img, (yy[m] * w + xx[m]), c[m])
    return np.clip(np.round(img), 0, 255).astype(np.uint8).reshape(h, w)


@dataclass
class Workload:
    cam: object
    left: FeatureSet
    right: FeatureSet
    pose: Pose                  # query pose (perturbed ground truth)
    local: LocalMap
    scale_pow: np.ndarray
    pyr_left: ImagePyramid | None = None
    pyr_right: ImagePyramid | None = None

    def frame(self) -> Frame:
        g = FrameGrid(self.left.u, self.left.v, self.cam.width, self.cam.height, 48)
        n = len(self.left.u)
        return Frame(0, 0.0, self.left, self.right, np.full(n, -1.0),
                     np.full(n, NO_POINT, dtype=np.int64), self.pose, g)


def make_workload(seed: int = 0, n_landmarks: int = 12000, map_points: int = 5000,
                  images: bool = False, fisheye: bool = False, noise_px: float = 0.5,
                  offset: float = 0.0, id_base: int = 0) -> Workload:
    """One frame + local map.  ``offset`` slides the camera along the shell
    axis so consecutive frames of a stream differ; ``id_base`` is added to the
    map point ids (distinct worlds sharing one resident map table)."""
    rng = np.random.default_rng(seed)
    cam = tumvi_camera() if fisheye else euroc_camera()
    a = rng.uniform(0, 2 * math.pi, n_landmarks)
    r = rng.uniform(0.42 * EXTENT, 0.50 * EXTENT, n_landmarks)
    z = rng.uniform(-0.18 * EXTENT, 0.18 * EXTENT, n_landmarks)
    lm = np.stack([r * np.cos(a), r * np.sin(a), z], axis=1)
    desc = rng.integers(0, 2 ** 63, size=(n_landmarks, 4), dtype=np.int64).astype(np.uint64)
    desc ^= rng.integers(0, 2, size=(n_landmarks, 4), dtype=np.int64).astype(np.uint64) << np.uint64(63)
    ang = rng.uniform(0, 2 * math.pi, n_landmarks)
    # camera on the axis side looking along +x (x_cam = -y_w, y_cam = -z_w)
    r_wc = np.array([[0.0, 0.0, 1.0], [-1.0, 0.0, 0.0], [0.0, -1.0, 0.0]])
    center = np.array([1.5, offset, 0.0])
    pose_left = Pose(r_wc.T, -r_wc.T @ center)
    if fisheye:
        t_rl = cam.right_extrinsic
    else:
        t_rl = Pose(np.eye(3), np.array([-cam.baseline, 0.0, 0.0]))
    pose_right = Pose(t_rl.rotation @ pose_left.rotation,
                      t_rl.rotation @ pose_left.translation + t_rl.translation)
    left, lids = _view(cam, pose_left, lm, desc, ang, rng, noise_px, 0)
    right, _ = _view(cam, pose_right, lm, desc, ang, rng, noise_px, 4)
    # local map: visible landmarks + random others (ascending ids)
    others = np.setdiff1d(np.arange(n_landmarks), lids)
    extra = max(0, map_points - len(lids))
    pick = rng.choice(others, size=min(extra, len(others)), replace=False)
    ids = np.sort(np.concatenate([lids, pick]))[:max(map_points, len(lids))]
    pos = lm[ids]
    d = np.linalg.norm(pos - center, axis=1)
    octs = _octave(d).astype(np.float64)
    max_d = d * SCALE ** octs
    soa = MapPointSoA(positions=pos.copy(), descriptors=_flip(desc[ids], rng, 8),
                      normals=(pos - center) / d[:, None], min_distances=max_d / SCALE ** (LEVELS - 1),
                      max_distances=max_d, point_ids=ids.astype(np.int64) + int(id_base))
    local = LocalMap((0,), soa.point_ids.copy(), soa)
    pert = _rot_axis(np.array([0.3, -0.5, 0.2]), 0.002)
    query = Pose(pert @ pose_left.rotation, pose_left.translation + np.array([0.01, 0.0, -0.01]))
    w = Workload(cam, left, right, query, local, SCALE ** np.arange(LEVELS, dtype=np.float64))
    if images and not fisheye:
        tex_rng = np.random.default_rng(seed * 7919 + 1)
        size = 15
        yy, xx = np.mgrid[-7:8, -7:8]
        win = np.exp(-(xx * xx + yy * yy) / (2.0 * (7 / 1.8) ** 2))
        tex = tex_rng.integers(40, 255, size=(n_landmarks, size, size)).astype(np.float64) * win
        w.pyr_left = build_pyramid(_render(cam, pose_left, lm, tex))
        w.pyr_right = build_pyramid(_render(cam, pose_right, lm, tex))
    return w
