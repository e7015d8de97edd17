"""The C ABI's host packer (rcpsp_blob_words / rcpsp_pack_instance /
rcpsp_blob_shape, csrc/pack.cpp) against an independent restatement of the
blob layout written here from the reference's instance model
(instance.py:53-80 KernelArrays, 374-388 critical path, 396-415 levels).
No GPU needed: the packer is host code in the same library."""

from __future__ import annotations

import math

import numpy as np
import pytest

from conftest import chain_instance
from paper_1711_04556_b200 import compute_levels, critical_path_length, make_instance, synth
from paper_1711_04556_b200 import device, _native

pytestmark = pytest.mark.skipif(not _native.LIB_PATH.exists(), reason="library not built")


def reference_blob(inst) -> np.ndarray:
    """Blob layout restated in numpy (header[32] | dur | dem | cap | pred CSR |
    succ CSR | req | capw | levels CSR)."""
    ka = inst.kernel_arrays
    n, m = inst.n_activities, inst.n_resources
    dur = np.asarray(ka.durations, np.int32)
    dem = np.asarray(ka.demands, np.int32).reshape(n, m)
    cap = np.asarray(ka.capacities, np.int32)
    top = int(cap.max()) if m else 0
    if not m:
        lb, W = 8, 1
    elif top > 32767:
        lb, W = 0, 0
    else:
        lb = 8 if top <= 127 else 16
        W = math.ceil(m / (32 // lb))
        if W > 2:
            lb, W = 0, 0
    req = np.zeros((n, W), np.uint32)
    capw = np.zeros(W, np.uint32)
    if W:
        lanes = 32 // lb
        for k in range(m):
            w, sh = divmod(k, lanes)
            req[:, w] |= dem[:, k].astype(np.uint32) << np.uint32(sh * lb)
            capw[w] |= np.uint32(int(cap[k]) << (sh * lb))
    levels = compute_levels(inst)
    lptr = np.concatenate([[0], np.cumsum([len(lv) for lv in levels])]).astype(np.int32)
    ldat = np.array([a for lv in levels for a in lv], np.int32)
    parts = [dur, dem.reshape(-1), cap, ka.pred_ptr, ka.pred_dat, ka.succ_ptr, ka.succ_dat,
             req.reshape(-1).view(np.int32), capw.view(np.int32), lptr, ldat]
    hdr = np.zeros(32, np.int32)
    off = 32
    for slot, arr in zip(range(16, 27), parts):
        hdr[slot] = off
        off += len(arr)
    sink_free = int(dur[n - 1]) == 0
    fan = max([len(s) for s in inst.successors]
              + [len(p) for i, p in enumerate(inst.predecessors) if not (sink_free and i == n - 1)]
              + [0])
    lbres = max([-(-int((dur.astype(np.int64) * dem[:, k]).sum()) // int(cap[k]))
                 for k in range(m) if cap[k] > 0] + [0])
    hdr[:14] = [0x52435053, n, m, int(ka.horizon), len(ka.pred_dat), W, lb,
                max(1, top), critical_path_length(inst), off, len(levels),
                int(int(dur.max()) > 32 or fan > 32), int(cap.sum()), lbres]
    return np.concatenate([hdr] + [np.asarray(p, np.int32) for p in parts])


def _instances(ginst):
    out = list(ginst.values())
    out += synth.benchmark_batch("j30p", 6) + synth.benchmark_batch("j120p", 6)
    out += synth.benchmark_batch("act300", 2)
    out.append(chain_instance([40, 3, 7]))                       # B_BIG by duration
    hub = make_instance("hub", [0] + [1] * 40 + [0], [5], [[0]] + [[1]] * 40 + [[0]],
                        [list(range(1, 41))] + [[41]] * 40 + [[]])  # fan-out 40
    out.append(hub)
    out.append(make_instance("wide", [0, 2, 3, 0], [10] * 9,
                             [[0] * 9, [3] * 9, [1] * 9, [0] * 9], [[1, 2], [3], [3], []]))
    out.append(make_instance("roomy16", [0, 2, 3, 0], [999, 40000 // 2, 7],
                             [[0, 0, 0], [500, 1, 7], [1, 20000, 0], [0, 0, 0]],
                             [[1, 2], [3], [3], []]))
    return out


def test_pack_matches_layout_restatement(ginst):
    for inst in _instances(ginst):
        got = device.pack_instance(inst)
        want = reference_blob(inst)
        assert got.dtype == np.int32
        assert got.tolist() == want.tolist(), inst.name
        sh = device.blob_shape(got)
        assert (sh.n, sh.m, sh.horizon, sh.edges, sh.words, sh.rmax, sh.cpm, sh.len, sh.big,
                sh.sumcap) == (got[1], got[2], got[3], got[4], got[5], got[7], got[8], len(got),
                               got[11], got[12])


def test_pack_errors():
    over = make_instance("over", [0, 2, 0], [2], [[0], [3], [0]], [[1], [2], []])
    with pytest.raises(ValueError, match="demands 3 of resource 0 with capacity 2"):
        device.pack_instance(over)
    L = _native.host_lib()
    z = np.zeros(4, np.int32)
    ptr = np.array([0, 0, 1, 2], np.int32)
    dat = np.array([0, 1], np.int32)
    # cycle 1 -> 2 -> 1 (pred lists) with matching successor lists
    pp = np.array([0, 0, 1, 2], np.int32)
    pd = np.array([2, 1], np.int32)
    sp = np.array([0, 0, 1, 2], np.int32)
    sd = np.array([2, 1], np.int32)
    dur = np.array([0, 1, 1], np.int32)
    cap = np.array([1], np.int32)
    dem = np.zeros(3, np.int32)
    assert L.rcpsp_blob_words(dur.ctypes.data, dem.ctypes.data, cap.ctypes.data, 3, 1,
                              pp.ctypes.data, pd.ctypes.data, sp.ctypes.data, sd.ctypes.data,
                              2) == -1
    assert b"cycle" in L.rcpsp_pack_last_error()
    # a buffer that is too small is refused
    ok = device.pack_instance(chain_instance([1, 2]))
    inst = chain_instance([1, 2])
    n, m, arrs, horizon = device._c_arrays(inst)
    a = [x.ctypes.data for x in arrs]
    small = np.zeros(len(ok) - 1, np.int32)
    assert L.rcpsp_pack_instance(*a[:3], n, m, *a[3:], horizon, small.ctypes.data,
                                 len(small)) == -1
    assert b"words <" in L.rcpsp_pack_last_error()
    del z, ptr, dat


def test_blob_shape_rejects_bad_magic():
    bad = np.zeros(32, np.int32)
    with pytest.raises(ValueError, match="magic"):
        device.blob_shape(bad)
