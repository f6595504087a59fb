"""Host-side logic of the step runners (no GPU): the submit argument
marshalling (pipeline._Ranges) and the runner's C-ABI argument checks."""

import ctypes

import pytest

from paper_2509_10757_b200 import _lib
from paper_2509_10757_b200.pipeline import AsyncRunner, _Ranges


@pytest.mark.parametrize("rng, pairs", [
    ((16, 4096), [(16, 4096)]),                       # input_range(): one pair
    ([(0, 100), (256, 1024)], [(0, 100), (256, 1024)]),  # input_ranges(): several
    ([(512, 512)], [(512, 512)]),                     # empty range
])
def test_ranges_marshalling(rng, pairs):
    r = AsyncRunner.ranges_arg(rng)
    assert isinstance(r, _Ranges)
    assert r.n == len(pairs)
    flat = [r.flat[q] for q in range(2 * r.n)]
    assert flat == [x for p in pairs for x in p]
    assert r.bytes == sum(hi - lo for lo, hi in pairs)


def test_ranges_empty_list():
    r = AsyncRunner.ranges_arg([])
    assert r.n == 0 and r.bytes == 0 and len(r.flat) >= 1  # valid pointer for the C call


def test_runner_submit_checks_without_gpu():
    L = _lib.load()
    # ranges beyond the slot / reversed ranges are refused before any copy
    flat = (ctypes.c_uint64 * 2)(8, 4)
    assert L.ft_runner_submit_ranges(None, 0, ctypes.c_void_p(16), flat, 1) == -1
    assert L.ft_runner_wait(None, -1) == -1


def test_device_arena_rows_at_one_pitch():
    """DeviceArena (batched submits' slot layout): rows 2 MB aligned at one
    2 MB-multiple pitch; a different size or one row too many is refused.
    Host tensors stand in for device memory (the layout logic is the same)."""
    from paper_2509_10757_b200.pipeline import DeviceArena
    a = DeviceArena(3)
    rows = [a.take(3_000_000, "cpu") for _ in range(3)]
    assert a.pitch == 4 << 20
    base = rows[0].data_ptr()
    assert base % (2 << 20) == 0
    assert [r.data_ptr() - base for r in rows] == [0, a.pitch, 2 * a.pitch]
    assert all(r.numel() == 3_000_000 for r in rows)
    with pytest.raises(ValueError):
        a.take(3_000_000, "cpu")  # all rows taken
    b = DeviceArena(2)
    b.take(100, "cpu")
    with pytest.raises(ValueError):
        b.take(5 << 20, "cpu")  # another pitch


def test_runner_submit_batch_checks_without_gpu():
    L = _lib.load()
    flat = (ctypes.c_uint64 * 2)(0, 16)
    assert L.ft_runner_submit_batch(None, 0, 2, ctypes.c_void_p(16), 64, flat, 1) == -1
    assert L.ft_runner_submit_batch(None, 0, 2, None, 64, flat, 1) == -1
