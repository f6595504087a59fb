"""install() rebinds the reference's hot-path names (CPU-only check; runs only
where the reference package is importable, i.e. the build container)."""

import os
import sys

import pytest

REF = "/root/reference/pkg/src"


@pytest.mark.reference
def test_install_rebinds_reference_names():
    if not os.path.isdir(REF):
        pytest.skip("reference not present")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.path.insert(0, REF)
    try:
        import trackfront.localmap as lm
        import trackfront.tracker as tr
    except Exception as e:  # pragma: no cover - numba/pillow missing
        pytest.skip(f"reference not importable: {e}")
    import paper_2509_10757_b200 as ft
    orig = tr.search_local_points
    orig_run = tr.StereoTracker._run_stereo
    done = ft.install()
    try:
        assert "trackfront.tracker.search_local_points" in done
        assert tr.search_local_points is ft.search_local_points
        assert lm.search_by_projection is ft.search_by_projection
        assert tr.match_pinhole_phase1 is ft.match_pinhole_phase1
        assert tr.update_local_map is ft.update_local_map  # SURVEY 8(f)-4, on the device
        assert lm.update_local_map is ft.update_local_map
        # the pinhole _run_stereo as one fused call (install(fuse_stereo=True))
        assert "trackfront.tracker.StereoTracker._run_stereo" in done
        assert tr.StereoTracker._run_stereo is not orig_run
    finally:
        ft.uninstall()
    assert tr.search_local_points is orig
    assert tr.StereoTracker._run_stereo is orig_run
    done = ft.install(fuse_stereo=False)
    try:
        assert tr.StereoTracker._run_stereo is orig_run
    finally:
        ft.uninstall()
