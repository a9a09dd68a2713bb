"""CPU checks of the boundary: the library builds for sm_100a, loads, and
exports every symbol include/orloj.h declares (no compute calls without a GPU);
O(1) argument errors are returned synchronously without touching the device."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_2209_00159_b200 import _abi


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(_abi.LIB_PATH):
        _abi.build()
    return _abi.lib()


def _declared():
    src = open(_abi.HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(orloj_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported(lib):
    names = _declared()
    assert len(names) >= 11
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_abi.SIGNATURES), "binding signatures out of sync with orloj.h"


def test_abi_version(lib):
    assert lib.orloj_abi_version() == 5 == _abi.ABI_VERSION


def test_sync_argument_errors(lib):
    st = _abi.Store(1, 6, 1, 16)          # B not a multiple of 4
    a = np.zeros(1, np.int64)
    w = np.ones(1, np.int64)
    prof = _abi.LatencyProfile(1, a.ctypes.data, w.ctypes.data)
    q = _abi.QueuesC(0, None, None, None, None, None)
    bk = ctypes.c_void_p(16)
    assert lib.orloj_pick_batch(ctypes.byref(st), ctypes.byref(prof), ctypes.byref(q), bk, bk, None) == 1
    assert b"multiple of 4" in lib.orloj_last_error()
    st = _abi.Store(1, 512, 1, 16)
    assert lib.orloj_pick_batch(ctypes.byref(st), ctypes.byref(prof), ctypes.byref(q), bk, bk, None) == 4
    st = _abi.Store(1, 8, 1, 16)
    w2 = np.array([1 << 30], np.int64)
    prof2 = _abi.LatencyProfile(1, a.ctypes.data, w2.ctypes.data)
    assert lib.orloj_pick_batch(ctypes.byref(st), ctypes.byref(prof2), ctypes.byref(q), bk, bk, None) == 4
    q1 = _abi.QueuesC(1, 16, None, 16, 16, 16)
    assert lib.orloj_score_batches(ctypes.byref(st), ctypes.byref(prof), ctypes.byref(q1), None, None, None,
                                   None) == 1
    assert lib.orloj_pick_batch_host_workspace(10, 100) > 0


def test_cubin_is_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _abi.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_replay_seg_workspace(lib):
    """Workspace of the segmented replay: none for 1 segment; 256 B of stats +
    the per-segment states, + 4 (2N + 34 S G) bytes of scratch log with a log."""
    f = lib.orloj_replay_seg_workspace
    assert f(8, 1000, 1, 0) == 0 and f(0, 0, 4, 0) == 0
    base = f(8, 1000, 4, 0)
    assert base > 256 and base % 256 == 0
    assert f(8, 1000, 8, 0) > base
    with_log = f(8, 1000, 4, 1)
    assert with_log - base >= 4 * (2 * 1000 + 34 * 8 * 4)
    st = _abi.Store(1, 8, 1, 16)
    a = np.zeros(1, np.int64)
    w = np.ones(1, np.int64)
    prof = _abi.LatencyProfile(1, a.ctypes.data, w.ctypes.data)
    tr = _abi.TraceC(2, 16, 16, 16, 16, 16, 16, 1)
    pol = _abi.ReplayPolicyC(0, None, None, None, None, 0.0)
    p = ctypes.c_void_p(16)
    assert lib.orloj_replay_trace_seg(ctypes.byref(st), ctypes.byref(prof), ctypes.byref(tr), ctypes.byref(pol), 0,
                                      10, p, 0, p, None, None) == 1
    assert b"segments" in lib.orloj_last_error()
    assert lib.orloj_replay_trace_seg(ctypes.byref(st), ctypes.byref(prof), ctypes.byref(tr), ctypes.byref(pol), 4,
                                      10, None, 0, p, None, None) == 1
    assert b"workspace" in lib.orloj_last_error()
