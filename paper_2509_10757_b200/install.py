"""Drop the B200 path into a running reference (trackfront) process.

The reference binds its stage functions with ``from .x import y`` (reference
tracker.py:24,28-32; localmap.py:19), so replacing ``trackfront.stereo.f``
alone would not reach the tracker.  ``install()`` rebinds the names in every
module that imported them; ``uninstall()`` restores the originals.

    import trackfront, paper_2509_10757_b200 as ft
    ft.install()                      # StereoTracker now runs on the B200
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
    },
    "trackfront.tracker": {
        "match_pinhole_phase1": _stereo.match_pinhole_phase1,
        "refine_match_phase2": _stereo.refine_match_phase2,
        "matches_from_candidates": _stereo.matches_from_candidates,
        "reject_outliers": _stereo.reject_outliers,
        "match_fisheye": _stereo.match_fisheye,
        "search_prev_frame": _projection.search_prev_frame,
        "search_local_points": _localmap.search_local_points,
    },
}

_saved: dict[tuple[str, str], object] = {}


def install() -> list[str]:
    """Rebind the reference's hot-path names; returns the rebound names."""
    done = []
    for modname, names in _TARGETS.items():
        mod = importlib.import_module(modname)
        for name, fn in names.items():
            if not hasattr(mod, name):
                continue
            _saved.setdefault((modname, name), getattr(mod, name))
            setattr(mod, name, fn)
            done.append(f"{modname}.{name}")
    return done


def uninstall() -> None:
    for (modname, name), orig in _saved.items():
        setattr(importlib.import_module(modname), name, orig)
    _saved.clear()
