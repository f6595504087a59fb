"""Device-resident map-point table (north star subsystem (1)).

The reference rebuilds every frame's local map on the host: update_local_map
collects point ids (localmap.py:42-76) and decompose_map_points copies each
point's position / descriptor / normal / distance range into a fresh SoA
(mapping.py:204-235) that search_local_points consumes.  Shipping that SoA
every frame costs 104-112 B per point per frame over PCIe.

Here every map point's packed record (``ft_point_record``) lives once in HBM.
A frame names its local map as a list of table slots in LocalMap order (4 B
per point), ``ft_gather_points`` builds the contiguous per-frame table the
track kernel stages, and only new or changed points cross PCIe
(``upsert`` -> ``ft_scatter_points``).  Point order -- and with it the
reference's lowest-point-index tie rule -- is the caller's LocalMap order.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .runtime import fill_point_records


class MapTable:
    def __init__(self, capacity: int, device: int | None = None):
        if not torch.cuda.is_available():
            raise _lib.FtError("MapTable needs a CUDA device (no CPU fallback)")
        self.lib = _lib.load()
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None
                                   else device)
        self.capacity = int(capacity)
        rec = _lib.POINT_RECORD.itemsize
        # fixed allocation: graphs captured against the table keep its address
        self.table = torch.zeros(self.capacity * rec, dtype=torch.uint8, device=self.device)
        self.stream = torch.cuda.Stream(self.device)
        self._ids = np.empty(0, dtype=np.int64)    # sorted point ids
        self._slot = np.empty(0, dtype=np.int32)   # slot of _ids[k]
        self.size = 0
        self.bytes_uploaded = 0
        self._retired: list[int] = []   # slots of rewritten records (in-flight readers)
        self._free: list[int] = []      # reusable slots (after reclaim())

    @property
    def ptr(self) -> int:
        return self.table.data_ptr()

    def _lookup(self, ids: np.ndarray) -> np.ndarray:
        """Slots of ids (-1 where absent)."""
        if len(self._ids) == 0:
            return np.full(len(ids), -1, dtype=np.int32)
        pos = np.searchsorted(self._ids, ids)
        pos_c = np.minimum(pos, len(self._ids) - 1)
        hit = self._ids[pos_c] == ids
        return np.where(hit, self._slot[pos_c], -1).astype(np.int32)

    def slots(self, point_ids) -> np.ndarray:
        """Table slots of point_ids (all must be present)."""
        ids = np.asarray(point_ids, dtype=np.int64)
        s = self._lookup(ids)
        if (s < 0).any():
            raise KeyError(f"{int((s < 0).sum())} point ids are not in the map table")
        return s

    def upsert(self, point_ids, soa, only_missing: bool = False) -> int:
        """Upload the records of the given points.  Returns the bytes copied
        host -> device.  Synchronous on the table's stream.

        New ids get fresh slots.  Present ids (unless only_missing) are
        rewritten copy-on-write: the new record goes to a fresh slot and the
        id's old slot is retired, never overwritten in place -- a step that
        was submitted earlier (its slot list taken before this call) may
        still be reading the old record on another stream.  Retired slots
        are reused only after ``reclaim()``, which the caller issues once
        every step submitted before the upsert has completed (the reference
        likewise finishes a frame's search before the map changes)."""
        ids = np.asarray(point_ids, dtype=np.int64)
        n = len(ids)
        if n == 0:
            return 0
        slots = self._lookup(ids)
        new = slots < 0
        keep = np.nonzero(new)[0] if only_missing else np.arange(n)
        if len(keep) == 0:
            return 0
        # one record per distinct id (the last occurrence wins, as a serial
        # overwrite would)
        kids = ids[keep]
        _, last_rev = np.unique(kids[::-1], return_index=True)
        keep = keep[np.sort(len(kids) - 1 - last_rev)]
        kids = ids[keep]
        old = self._lookup(kids)
        fresh = self._alloc(len(kids))
        if (old >= 0).any():
            self._retired.extend(int(x) for x in old[old >= 0])
        # id -> slot map: drop the rewritten ids, add every uploaded id
        present = old >= 0
        if present.any():
            drop = np.isin(self._ids, kids[present])
            self._ids, self._slot = self._ids[~drop], self._slot[~drop]
        allids = np.concatenate([self._ids, kids])
        allslots = np.concatenate([self._slot, fresh])
        order = np.argsort(allids, kind="stable")
        self._ids, self._slot = allids[order], allslots[order]
        k = len(keep)
        rec = np.zeros(k, dtype=_lib.POINT_RECORD)
        sub = _SubSoA(soa, keep)
        fill_point_records(rec, sub)
        rec["id"][:] = kids
        host_rec = torch.from_numpy(rec.view(np.uint8)).pin_memory()
        host_slot = torch.from_numpy(fresh.astype(np.int32)).pin_memory()
        with torch.cuda.stream(self.stream):
            d_rec = host_rec.to(self.device, non_blocking=True)
            d_slot = host_slot.to(self.device, non_blocking=True)
            _lib.check(self.lib.ft_scatter_points(k, d_rec.data_ptr(), d_slot.data_ptr(),
                                                  self.ptr, self.capacity,
                                                  self.stream.cuda_stream), "ft_scatter_points")
        self.stream.synchronize()
        nbytes = host_rec.numel() + host_slot.numel() * 4
        self.bytes_uploaded += nbytes
        return nbytes

    def _alloc(self, k: int) -> np.ndarray:
        """k slots: recycled ones first, then never-used ones."""
        take = min(k, len(self._free))
        out = [self._free.pop() for _ in range(take)]
        rest = k - take
        if self.size + rest > self.capacity:
            self._free.extend(reversed(out))
            raise _lib.FtError(f"map table full ({self.capacity} points)")
        out.extend(range(self.size, self.size + rest))
        self.size += rest
        return np.asarray(out, dtype=np.int32)

    def reclaim(self) -> int:
        """Make the slots retired by earlier upserts reusable.  Call only once
        every step that may read them (submitted before those upserts) has
        completed.  Returns the number of slots recycled."""
        n = len(self._retired)
        self._free.extend(self._retired)
        self._retired = []
        return n


    def gather_soa(self, slots, pool=None) -> "MapPointSoA":
        """Decompose the records at table ``slots`` into a MapPointSoA (the
        reference's decompose_map_points, mapping.py:204-235), gathered on the
        device (ft_gather_points) and copied back once; into the pool's
        soa_* buffers when a pool is given (localmap.py:67-75)."""
        from .types import MapPointSoA
        slots = np.ascontiguousarray(slots, dtype=np.int32)
        m = len(slots)
        if m == 0:
            return MapPointSoA.empty()
        with torch.cuda.stream(self.stream):
            idx = torch.from_numpy(slots).pin_memory().to(self.device, non_blocking=True)
            cnt = torch.tensor([m], dtype=torch.int32).pin_memory().to(self.device,
                                                                        non_blocking=True)
            out = torch.empty(m * _lib.POINT_RECORD.itemsize, dtype=torch.uint8,
                              device=self.device)
            st = torch.zeros(1, dtype=torch.int32, device=self.device)
            _lib.check(self.lib.ft_gather_points(1, self.ptr, self.capacity, idx.data_ptr(),
                                                 cnt.data_ptr(), m, out.data_ptr(),
                                                 st.data_ptr(), self.stream.cuda_stream),
                       "ft_gather_points")
            host = out.to("cpu", non_blocking=True)
            hst = st.to("cpu", non_blocking=True)
        self.stream.synchronize()
        if int(hst.item()) != 0:
            raise _lib.FtError("map table gather: slot out of range")
        rec = host.numpy().view(_lib.POINT_RECORD)
        fields = (("positions", "pos", (m, 3), np.float64), ("descriptors", "desc", (m, 4), np.uint64),
                  ("normals", "nrm", (m, 3), np.float64), ("min_distances", "min_dist", (m,),
                                                            np.float64),
                  ("max_distances", "max_dist", (m,), np.float64), ("point_ids", "id", (m,),
                                                                  np.int64))
        pool_names = {"positions": "soa_positions", "descriptors": "soa_descriptors",
                      "normals": "soa_normals", "min_distances": "soa_min_d",
                      "max_distances": "soa_max_d", "point_ids": "soa_ids"}
        arrs = {}
        for name, f, shape, dt in fields:
            dst = pool.acquire(pool_names[name], shape, dt) if pool is not None else \
                np.empty(shape, dt)
            dst[...] = rec[f]
            arrs[name] = dst
        return MapPointSoA(**arrs)


def decompose_points(mps) -> "MapPointSoA":
    """decompose_map_points (reference mapping.py:204-235) of MapPoint-like
    objects (point_id, position, descriptor, normal, min_distance,
    max_distance), host side."""
    from .types import MapPointSoA
    return MapPointSoA(
        positions=np.array([p.position for p in mps], dtype=np.float64).reshape(-1, 3),
        descriptors=np.array([p.descriptor for p in mps], dtype=np.uint64).reshape(-1, 4),
        normals=np.array([p.normal for p in mps], dtype=np.float64).reshape(-1, 3),
        min_distances=np.array([p.min_distance for p in mps], dtype=np.float64),
        max_distances=np.array([p.max_distance for p in mps], dtype=np.float64),
        point_ids=np.array([p.point_id for p in mps], dtype=np.int64))


class _SubSoA:
    """Row subset of a MapPointSoA-like object (reference field names)."""

    def __init__(self, soa, rows):
        self.positions = np.asarray(soa.positions)[rows]
        self.normals = np.asarray(soa.normals)[rows]
        self.descriptors = np.asarray(soa.descriptors)[rows]
        self.min_distances = np.asarray(soa.min_distances)[rows]
        self.max_distances = np.asarray(soa.max_distances)[rows]
        pid = getattr(soa, "point_ids", None)
        self.point_ids = np.asarray(pid)[rows] if pid is not None else np.zeros(len(rows), np.int64)

    def __len__(self):
        return len(self.positions)
