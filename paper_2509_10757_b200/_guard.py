"""Process-wide record of live persistent kernels, per CUDA device.

A persistent runner (AsyncRunner(persistent=True)) or ring keeps its blocks
resident on all but 4 SMs until it is closed.  A cooperative launch that needs
more SMs than are left (every track launch: its block groups synchronise
through group barriers) would wait forever, so calls that launch one check
here first and raise instead of hanging."""

from __future__ import annotations

import threading

from . import _lib

_lock = threading.Lock()
_active: dict[int, int] = {}


def acquire(device: int) -> None:
    with _lock:
        if _active.get(device, 0):
            raise _lib.FtError(f"a persistent runner already holds GPU {device}'s SMs: close() "
                               "it first (one persistent kernel per GPU)")
        _active[device] = 1


def release(device: int) -> None:
    with _lock:
        _active.pop(device, None)


def check(device: int, what: str) -> None:
    if _active.get(device, 0):  # lock-free fast path: a dict lookup
        raise _lib.FtError(f"{what}: a persistent runner holds GPU {device}'s SMs; close() it "
                           "before other track launches on this GPU (they could not become "
                           "resident and would never finish)")
