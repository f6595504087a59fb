"""Device-resident world for update_local_map (reference
localmap.py:42-76, mapping.py:238-270).

The reference rebuilds a frame's local map on the host every frame: the
keyframes observing the frame's slotted points, every point those keyframes
observe (Python set unions), sorted, then decomposed into a fresh SoA.  On
the cfg4 sequences that costs 6-19 ms per frame (tests/golden/summary.json,
reference seq engine) -- more than every GPU stage together -- so it runs on
the device here:

* ``WorldTable`` mirrors a reference ``WorldMap`` in HBM: map-point records
  in a MapTable (read in place by the search), an id -> table-slot array, and
  every keyframe's observed point ids (KeyFrame.observed_point_ids,
  mapping.py:142-145) as one CSR.  Keyframes and map points are immutable once
  added (the tracker only appends), so ``sync`` uploads only the keyframes and
  points added since the last call -- the map delta.
* ``update_local_map(frame, world, pool)`` -- the reference's signature --
  syncs, then ONE kernel (csrc/ft_localmap.cu) computes the keyframe set and
  the ascending point ids with their table slots.  It returns a
  ``ResidentLocalMap``: keyframe ids and point ids like the reference's
  LocalMap, plus the table slots, so ``search_local_points`` reads the points
  in place (nothing re-shipped); its ``soa`` is materialised from the table
  only if someone reads it (into the caller's pool buffers, as the reference
  fills them).
"""

from __future__ import annotations

import weakref

import numpy as np
import torch

from . import _lib
from .maptable import MapTable, decompose_points
from .types import LocalMap, MapPointSoA

NO_POINT = -1


class WorldTable:
    def __init__(self, device: int | None = None, point_capacity: int = 1 << 16):
        if not torch.cuda.is_available():
            raise _lib.FtError("WorldTable needs a CUDA device (no CPU fallback)")
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None
                                   else device)
        self.table = MapTable(point_capacity, device=self.device.index)
        self.kf_keys: list[int] = []          # reference keyframe ids, upload order
        self._kf_index: dict[int, int] = {}
        self._obs = torch.empty(1 << 16, dtype=torch.int32, device=self.device)
        self._off = torch.zeros(1025, dtype=torch.int64, device=self.device)
        self._n_obs = 0
        self._id_slot = torch.full((1024,), -1, dtype=torch.int32, device=self.device)
        self._h_id_slot = np.full(1024, -1, dtype=np.int32)
        self.id_cap = 0
        self._n_pts = 0
        self.out_cap = 4096
        self.bytes_uploaded = 0

    # -- sync -----------------------------------------------------------------

    def _grow(self, t: torch.Tensor, need: int, fill=None) -> torch.Tensor:
        if need <= t.numel():
            return t
        cap = max(need, 2 * t.numel())
        n = (torch.full((cap,), fill, dtype=t.dtype, device=t.device) if fill is not None
             else torch.empty(cap, dtype=t.dtype, device=t.device))
        n[:t.numel()].copy_(t)
        return n

    def sync(self, world) -> int:
        """Upload the keyframes and map points added to ``world`` since the
        last call; returns the bytes shipped."""
        shipped = 0
        if len(world.points) != self._n_pts:
            ids = np.fromiter(world.points.keys(), dtype=np.int64, count=len(world.points))
            if len(ids) and int(ids.min()) < 0:
                raise KeyError("negative map point id")
            known = np.zeros(len(ids), bool)
            inside = ids < len(self._h_id_slot)
            known[inside] = self._h_id_slot[ids[inside]] >= 0
            missing = np.sort(ids[~known])  # not yet in the id -> slot map
            if len(missing):
                # records the table does not hold yet (another caller -- e.g.
                # search_prev_frame(table=) -- may have uploaded some already)
                absent = missing[self.table._lookup(missing) < 0]
                if len(absent):
                    shipped += self.table.upsert(absent, decompose_points(
                        [world.points[int(p)] for p in absent]), only_missing=True)
                hi = int(missing.max()) + 1
                if hi > len(self._h_id_slot):
                    grow = np.full(max(hi, 2 * len(self._h_id_slot)), -1, np.int32)
                    grow[:len(self._h_id_slot)] = self._h_id_slot
                    self._h_id_slot = grow
                    self._id_slot = self._grow(self._id_slot, len(grow), fill=-1)
                self._h_id_slot[missing] = self.table.slots(missing)
                lo = int(missing.min())
                self._id_slot[lo:hi].copy_(torch.from_numpy(self._h_id_slot[lo:hi]))
                shipped += 4 * (hi - lo)
                self.id_cap = max(self.id_cap, hi)
            self._n_pts = len(world.points)
        if len(world.keyframes) != len(self.kf_keys):
            new = sorted(k for k in world.keyframes if k not in self._kf_index)
            lists = []
            for k in new:
                kf = world.keyframes[k]
                obs = (kf.observed_point_ids() if hasattr(kf, "observed_point_ids")
                       else np.unique(kf.point_ids[kf.point_ids != NO_POINT]))
                lists.append(np.asarray(obs, dtype=np.int32))
                self._kf_index[k] = len(self.kf_keys)
                self.kf_keys.append(k)
            flat = np.concatenate(lists) if lists else np.zeros(0, np.int32)
            if len(flat) and int(flat.max()) >= self.id_cap:
                raise KeyError("a keyframe observes a point that is not in the world")
            n0, n1 = self._n_obs, self._n_obs + len(flat)
            self._obs = self._grow(self._obs, n1)
            k0 = len(self.kf_keys) - len(new)
            self._off = self._grow(self._off, len(self.kf_keys) + 1)
            offs = n0 + np.cumsum([len(x) for x in lists], dtype=np.int64)
            if len(flat):
                self._obs[n0:n1].copy_(torch.from_numpy(flat))
            self._off[k0 + 1:len(self.kf_keys) + 1].copy_(torch.from_numpy(offs))
            self._n_obs = n1
            shipped += 4 * len(flat) + 8 * len(offs)
        self.bytes_uploaded += shipped
        return shipped

    def world_dev(self):
        from . import session as S
        w = S.FtWorldDev()
        w.kf_obs, w.kf_off = self._obs.data_ptr(), self._off.data_ptr()
        w.n_kf = len(self.kf_keys)
        w.id_slot, w.id_cap = self._id_slot.data_ptr(), int(self.id_cap)
        return w


_TABLES: dict[int, tuple] = {}


def world_table(world) -> WorldTable:
    """The WorldTable mirroring ``world`` on the current device (one per
    world object, released with it)."""
    dev = torch.cuda.current_device()
    key = (id(world), dev)
    hit = _TABLES.get(key)
    if hit is not None and hit[0]() is world:
        return hit[1]
    wt = WorldTable(dev)
    try:
        ref = weakref.ref(world, lambda _r, k=key: _TABLES.pop(k, None))
    except TypeError:  # not weak-referenceable: keep it for the process
        ref = (lambda w=world: w)
    _TABLES[key] = (ref, wt)
    return wt


class ResidentLocalMap:
    """The reference's LocalMap (keyframe_ids, point_ids ascending, soa) whose
    points live in a device MapTable: ``table_slots[i]`` holds point_ids[i]'s
    record.  ``soa`` is gathered from the table on first access (into the
    caller's pool buffers when given, as localmap.py:67-75 fills them)."""

    def __init__(self, keyframe_ids, point_ids, table: MapTable, table_slots, pool=None):
        self.keyframe_ids = tuple(keyframe_ids)
        self.point_ids = point_ids
        self.table = table
        self.table_slots = table_slots
        self._pool = pool
        self._soa = None

    def __len__(self) -> int:
        return len(self.point_ids)

    @property
    def soa(self) -> MapPointSoA:
        if self._soa is None:
            self._soa = self.table.gather_soa(self.table_slots, self._pool)
        return self._soa


def update_local_map(frame, world, pool=None):
    """localmap.py:42-76: the keyframes observing the frame's slotted points
    and every point they observe (ascending), on the device.  Same keyframe
    ids and point ids as the reference; the SoA stays in the table until read."""
    from . import session as S
    slots = np.ascontiguousarray(frame.slots, dtype=np.int64)
    if not (slots != NO_POINT).any():
        return LocalMap.empty()
    wt = world_table(world)
    wt.sync(world)
    ses = S.session()
    counts = np.zeros(4, np.int32)
    while True:
        cap = wt.out_cap
        kf = np.empty(cap, np.int32)
        ids = np.empty(cap, np.int64)
        sl = np.empty(cap, np.int32)
        with ses.lock:
            st = ses.lib.ft_session_update_local_map(ses.handle, slots.ctypes.data, len(slots),
                                                     wt.world_dev(), cap, kf.ctypes.data,
                                                     ids.ctypes.data, sl.ctypes.data,
                                                     counts.ctypes.data)
        if st == -2 and counts[2] == 0 and max(counts[0], counts[1]) > cap:
            wt.out_cap = int(2 * max(counts[0], counts[1]))
            continue
        if st == -2 and counts[2]:
            raise KeyError("frame slot holds a point id that is not in the world")
        _lib.check(st, "ft_session_update_local_map")
        break
    nk, npnt = int(counts[0]), int(counts[1])
    if npnt == 0:
        return LocalMap((), np.empty(0, np.int64), MapPointSoA.empty())
    return ResidentLocalMap((wt.kf_keys[k] for k in kf[:nk]), ids[:npnt].copy(), wt.table,
                            sl[:npnt].copy(), pool)
