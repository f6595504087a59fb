"""B200-native tracking hot path of FastTrack (arXiv 2509.10757).

Drop-in for the reference package ``trackfront``'s hot-path stage functions
(stereo matching and search by projection / SearchLocalPoints), running as
hand-written sm_100a CUDA behind a C ABI (include/fasttrack_b200.h).  There is
no CPU fallback: calls raise if libfasttrack_b200.so or a CUDA device is
missing.
"""

from .types import (Correspondences, FeatureSet, FisheyeCamera, Frame, FrameGrid, ImagePyramid,
                    LocalMap, MapPointSoA, NO_DEPTH, NO_POINT, PinholeCamera, Pose,
                    ProjectionSearchConfig, StereoMatchConfig, StereoMatches)
from .stereo import (build_row_buckets, compute_stereo_fisheye_matches, compute_stereo_matches,
                     match_fisheye, match_pinhole_phase1, matches_from_candidates,
                     matches_to_csv_rows, refine_match_phase2, reject_outliers, triangulate_rays)
from .projection import (frustum_and_cone_check, predict_scale, resolve_conflicts,
                         rotation_consistency_filter, run_phase_a, search_by_projection,
                         search_prev_frame)
from .localmap import search_local_points, update_local_map
from .install import install, uninstall

# ORB-SLAM-style names (BASELINE.json north star)
SearchByProjection = search_by_projection
SearchLocalPoints = search_local_points
ComputeStereoMatches = compute_stereo_matches
ComputeStereoFishEyeMatches = compute_stereo_fisheye_matches

__all__ = [
    "Correspondences", "FeatureSet", "FisheyeCamera", "Frame", "FrameGrid", "ImagePyramid",
    "LocalMap", "MapPointSoA", "NO_DEPTH", "NO_POINT", "PinholeCamera", "Pose",
    "ProjectionSearchConfig", "StereoMatchConfig", "StereoMatches", "build_row_buckets",
    "compute_stereo_fisheye_matches", "compute_stereo_matches", "match_fisheye",
    "match_pinhole_phase1", "matches_from_candidates", "matches_to_csv_rows",
    "refine_match_phase2", "reject_outliers", "triangulate_rays", "frustum_and_cone_check",
    "predict_scale", "resolve_conflicts", "rotation_consistency_filter", "run_phase_a",
    "search_by_projection", "search_prev_frame", "search_local_points", "update_local_map",
    "SearchByProjection",
    "SearchLocalPoints", "ComputeStereoMatches", "ComputeStereoFishEyeMatches", "install",
    "uninstall",
]
