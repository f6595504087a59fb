"""Image pyramid on the device: drop-in for the reference's
``trackfront.extraction.build_pyramid`` (extraction.py:97-125), bit-exact
(``ft_build_pyramids``, csrc/ft_pyramid.cu).  Frames can ship raw images and
build the pyramid that stereo phase 2 reads on the B200."""

from __future__ import annotations

import numpy as np

from . import _lib
from .runtime import Layout, pyramid_struct, runtime
from .types import ImagePyramid


def pyramid_level_dims(width: int, height: int, scale: float, levels: int):
    """floor(level-0 dims / scale^level) (reference extraction.py:58-64)."""
    powers = scale ** np.arange(levels, dtype=np.float64)
    return (np.floor(width / powers).astype(np.int64), np.floor(height / powers).astype(np.int64))


def pyramid_geometry(width: int, height: int, scale: float = 1.2, levels: int = 8) -> ImagePyramid:
    """An ImagePyramid shell (offsets / dims, no data) for the given image size."""
    ws, hs = pyramid_level_dims(width, height, scale, levels)
    offsets = np.zeros(levels + 1, dtype=np.int64)
    np.cumsum(ws * hs, out=offsets[1:])
    return ImagePyramid(None, offsets, ws, hs, scale)


def build_pyramid(image: np.ndarray, cfg, pool=None, name: str = "pyr") -> ImagePyramid:
    """Build the scale pyramid of a 2-D uint8 image on the device; returns a
    host ImagePyramid (reference semantics and errors, extraction.py:97-109)."""
    image = np.asarray(image)
    if image.ndim != 2 or image.dtype != np.uint8 or image.size == 0:
        raise ValueError("expected a non-empty 2-d uint8 image")
    h, w = image.shape
    geo = pyramid_geometry(w, h, float(cfg.scale), int(cfg.levels))
    if geo.widths[-1] < cfg.patch_size or geo.heights[-1] < cfg.patch_size:
        raise ValueError(f"image {w}x{h} too small for {cfg.levels} levels at scale {cfg.scale}")
    total = int(geo.offsets[-1])
    rt = runtime()
    lay = Layout()
    lay.add("pyr", total)
    with rt.lock:
        rt.reserve(lay.total)
        rt.host_view(lay, "pyr", np.uint8, (h * w,))[:] = image.ravel()
        rt.h2d(0, h * w)
        st = rt.lib.ft_build_pyramids(1, pyramid_struct(geo, rt.ptr(lay, "pyr"), total), None, 0,
                                      rt.workspace(), rt.stream.cuda_stream)
        _lib.check(st, "ft_build_pyramids")
        rt.d2h(0, total)
        rt.sync()
        data = rt.host_view(lay, "pyr", np.uint8, (total,)).copy()
    return ImagePyramid(data, geo.offsets, geo.widths, geo.heights, float(cfg.scale))
