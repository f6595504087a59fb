"""Track-local-map point association (SearchLocalPoints) on B200.

Mirrors ``trackfront.localmap.search_local_points`` (reference
pkg/src/trackfront/localmap.py:79-122): skip points already slotted in the
frame, search the rest by projection, write each winner's point id into its
keypoint slot only if that slot is empty, return the filled-slot count.  The
skip mask (hash set of slotted ids), phases A-C, the slot write and the count
run in ONE ``ft_project_search`` launch; only the world-map bookkeeping
(MapPoint flags, a host object graph) stays on the host, as in the reference.
"""

from __future__ import annotations

import numpy as np

from .projection import project_search
from .types import LocalMap, NO_POINT

from .worldmap import update_local_map  # noqa: E402,F401  (device update_local_map)

__all__ = ["LocalMap", "search_local_points", "update_local_map"]


def search_local_points(local, frame, cam, cfg, scale: float, levels: int, engine=None,
                        world=None, pool=None, table=None) -> int:
    """Associate unmatched local points with frame keypoints; mutates
    ``frame.slots`` (and world point flags when ``world`` is given)."""
    if len(local.point_ids) == 0:
        return int(np.count_nonzero(frame.slots != NO_POINT))
    ref_angles = None
    rotation_check = bool(cfg.rotation_check_local)
    if rotation_check and world is not None:
        # source angle = keypoint angle of each point's earliest observation
        # (localmap.py:99-106)
        ref_angles = np.zeros(len(local.point_ids))
        for i, pid in enumerate(local.point_ids):
            obs = world.points[int(pid)].observations
            if obs:
                kf_id, slot = min(obs)
                ref_angles[i] = world.keyframes[kf_id].left.angle[slot]
    elif rotation_check:
        rotation_check = False
    before = np.asarray(frame.slots).copy()
    tslots = getattr(local, "table_slots", None)
    if tslots is not None:  # a ResidentLocalMap (worldmap.update_local_map): read in place
        from .projection import _IdsOnly
        r = project_search(_IdsOnly(local.point_ids), frame, frame.pose, cam, cfg, scale,
                           levels, ref_angles=ref_angles, rotation=rotation_check, slots=before,
                           skip_slotted=True, write_slots=True, table=local.table,
                           table_slots=tslots, want_corr=False)
    else:
        r = project_search(local.soa, frame, frame.pose, cam, cfg, scale, levels,
                           ref_angles=ref_angles, rotation=rotation_check, slots=before,
                           skip_slotted=True, write_slots=True, table=table, want_corr=False)
    after = r["slots"]
    frame.slots[...] = after
    if world is not None:
        for ki in np.nonzero(after != before)[0]:
            mp = world.points[int(after[ki])]
            mp.last_seen_frame = frame.frame_id
            mp.tracked_in_view = True
    return int(r["count"])
