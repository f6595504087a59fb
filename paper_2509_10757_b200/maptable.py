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
        self._h_rec = None
        self._h_slot = None

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
        """Upload the records of the given points (new ids get fresh slots,
        present ids are overwritten unless only_missing).  Returns the bytes
        copied host -> device.  Synchronous on the table's stream."""
        ids = np.asarray(point_ids, dtype=np.int64)
        n = len(ids)
        if n == 0:
            return 0
        slots = self._lookup(ids)
        new = slots < 0
        if only_missing:
            keep = np.nonzero(new)[0]
        else:
            keep = np.arange(n)
        if len(keep) == 0:
            return 0
        n_new = int(new.sum())
        if n_new:
            if self.size + n_new > self.capacity:
                raise _lib.FtError(f"map table full ({self.capacity} points)")
            new_ids, first = np.unique(ids[new], return_index=True)
            fresh = np.arange(self.size, self.size + len(new_ids), dtype=np.int32)
            self.size += len(new_ids)
            allids = np.concatenate([self._ids, new_ids])
            allslots = np.concatenate([self._slot, fresh])
            order = np.argsort(allids, kind="stable")
            self._ids, self._slot = allids[order], allslots[order]
            slots = self._lookup(ids)
        k = len(keep)
        rec = np.zeros(k, dtype=_lib.POINT_RECORD)
        sub = _SubSoA(soa, keep)
        fill_point_records(rec, sub)
        rec["id"][:] = ids[keep]
        host_rec = torch.from_numpy(rec.view(np.uint8)).pin_memory()
        host_slot = torch.from_numpy(slots[keep].astype(np.int32)).pin_memory()
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
