"""Drop the B200 path into a running reference (trackfront) process.

The reference binds its stage functions with ``from .x import y`` (reference
tracker.py:24,28-32; localmap.py:19), so replacing ``trackfront.stereo.f``
alone would not reach the tracker.  ``install()`` rebinds the names in every
module that imported them; ``uninstall()`` restores the originals.

    import trackfront, paper_2509_10757_b200 as ft
    ft.install()                      # StereoTracker now runs on the B200

With ``fuse_stereo=True`` (default) the tracker's pinhole ``_run_stereo``
(tracker.py:415-427: phase 1 -> phase 2 | from candidates -> reject, three
calls with host round trips in between) is also replaced, by ONE fused call
with the same outputs and the same side effects (phase-1 candidates written
into the pool's stereo_idx / stereo_dist buffers); the fisheye branch keeps
the reference's method, whose match_fisheye is rebound above.
"""

from __future__ import annotations

import importlib

from . import localmap as _localmap
from . import projection as _projection
from . import stereo as _stereo

# name -> replacement, per reference module that defines or imports it
_TARGETS = {
    "trackfront.stereo": {
        "match_pinhole_phase1": _stereo.match_pinhole_phase1,
        "refine_match_phase2": _stereo.refine_match_phase2,
        "matches_from_candidates": _stereo.matches_from_candidates,
        "reject_outliers": _stereo.reject_outliers,
        "match_fisheye": _stereo.match_fisheye,
    },
    "trackfront.projection": {
        "run_phase_a": _projection.run_phase_a,
        "resolve_conflicts": _projection.resolve_conflicts,
        "rotation_consistency_filter": _projection.rotation_consistency_filter,
        "search_by_projection": _projection.search_by_projection,
        "search_prev_frame": _projection.search_prev_frame,
    },
    "trackfront.localmap": {
        "search_by_projection": _projection.search_by_projection,
        "search_local_points": _localmap.search_local_points,
        "update_local_map": _localmap.update_local_map,
    },
    "trackfront.tracker": {
        "match_pinhole_phase1": _stereo.match_pinhole_phase1,
        "refine_match_phase2": _stereo.refine_match_phase2,
        "matches_from_candidates": _stereo.matches_from_candidates,
        "reject_outliers": _stereo.reject_outliers,
        "match_fisheye": _stereo.match_fisheye,
        "search_prev_frame": _projection.search_prev_frame,
        "search_local_points": _localmap.search_local_points,
        "update_local_map": _localmap.update_local_map,
    },
}

_saved: dict[tuple[str, str], object] = {}
_saved_method: dict[str, object] = {}


def _fused_run_stereo(self, left, right, pyr_l, pyr_r):
    """StereoTracker._run_stereo (tracker.py:397-427) with the pinhole branch
    as ONE fused ft_stereo_pinhole call; fisheye -> the reference method."""
    import numpy as np
    from . import _lib
    if hasattr(self.cam, "k1"):  # FisheyeCamera (cameras.py:79-157)
        return _saved_method["_run_stereo"](self, left, right, pyr_l, pyr_r)
    scale_pow = self.extraction.scale_powers()
    n = len(left.u)
    idx = self.pool.acquire("stereo_idx", (n,), np.int64)
    dist = self.pool.acquire("stereo_dist", (n,), np.int64)
    if n == 0:
        return _stereo.matches_from_candidates(idx, dist, left, right, self.cam, self.stereo)
    direct = idx.flags.c_contiguous and dist.flags.c_contiguous
    ci, cd = (idx, dist) if direct else (np.empty(n, np.int64), np.empty(n, np.int64))
    mode = _lib.FT_STEREO_PHASE1 | _lib.FT_STEREO_REJECT
    mode |= _lib.FT_STEREO_REFINE if pyr_l is not None else _lib.FT_STEREO_FROM_CAND
    res, _, _ = _stereo._run_stereo(mode, left, right, self.cam, self.stereo, scale_pow,
                                    int(self.cam.height), pyr_l, pyr_r, out_cand=(ci, cd))
    if not direct:
        idx[...] = ci
        dist[...] = cd
    return res


def install(fuse_stereo: bool = True, resident_world: bool = False) -> list[str]:
    """Rebind the reference's hot-path names; returns the rebound names.

    resident_world=True: search_prev_frame reads the previous frame's map
    points in place from the world mirror that update_local_map keeps in HBM
    (only new points are uploaded) instead of decomposing them on the host;
    the tracker's pooled ``soa_out`` is then not filled (the tracker never
    reads it, tracker.py:304-316)."""
    done = []
    _projection._RESIDENT_WORLD = bool(resident_world)
    for modname, names in _TARGETS.items():
        mod = importlib.import_module(modname)
        for name, fn in names.items():
            if not hasattr(mod, name):
                continue
            _saved.setdefault((modname, name), getattr(mod, name))
            setattr(mod, name, fn)
            done.append(f"{modname}.{name}")
    if fuse_stereo:
        tr = importlib.import_module("trackfront.tracker")
        cls = tr.StereoTracker
        if hasattr(cls, "_run_stereo"):
            _saved_method.setdefault("_run_stereo", cls._run_stereo)
            cls._run_stereo = _fused_run_stereo
            done.append("trackfront.tracker.StereoTracker._run_stereo")
    return done


def uninstall() -> None:
    _projection._RESIDENT_WORLD = False
    for (modname, name), orig in _saved.items():
        setattr(importlib.import_module(modname), name, orig)
    _saved.clear()
    if "_run_stereo" in _saved_method:
        tr = importlib.import_module("trackfront.tracker")
        tr.StereoTracker._run_stereo = _saved_method.pop("_run_stereo")
