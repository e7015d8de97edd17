"""Single-step resource-state API on the GPU (reference evaluator.py:30-107,
test_evaluator.py TestCapacityState / TestTimeState), through rcpsp_state_op,
which runs the same device functions as the SGS (cap_es/cap_commit,
warp_window/warp_commit)."""

import numpy as np
import pytest

import oracle
from conftest import random_topological_order

pytestmark = pytest.mark.gpu

from paper_1711_04556_b200 import device, make_instance, synth  # noqa: E402
from paper_1711_04556_b200.evaluator import (CapacityResourceState,  # noqa: E402
                                             TimeResourceState, cap_earliest_start, cap_update,
                                             time_earliest_start, time_update)


def one_resource(cap, durations, demands, successors):
    return make_instance("one-res", durations, [cap], [[d] for d in demands], successors)


def figure_state():
    # capacity 7 holding {7,7,5,5,5,5,4}; activity 1 needs 3 units for 3 time units
    inst = one_resource(7, [0, 3, 0], [0, 3, 0], [[1], [2], []])
    st = CapacityResourceState(inst)
    st.levels[0, :] = [7, 7, 5, 5, 5, 5, 4]
    return inst, st


def test_capacity_worked_example():
    inst, st = figure_state()
    assert cap_earliest_start(st, 1, inst) == 5
    assert cap_earliest_start(st, 0, inst) == 0
    cap_update(st, 1, 5, inst)                       # test_evaluator.py:49-53 (Fig. 4)
    assert st.levels[0].tolist() == [8, 8, 8, 7, 7, 5, 4]
    assert st.rows_descending()
    with pytest.raises(ValueError):
        figure = figure_state()
        cap_update(figure[1], 1, 4, figure[0])       # earliest is 5
    two = one_resource(2, [0, 5, 0], [0, 2, 0], [[1], [2], []])
    s2 = CapacityResourceState(two)
    cap_update(s2, 1, 5, two)                        # test_evaluator.py:61-65
    assert s2.levels[0].tolist() == [10, 10]


def gap_state():
    inst = one_resource(2, [0, 5, 3, 5, 0], [0, 2, 2, 0, 0], [[1, 2, 3], [4], [4], [4], []])
    st = TimeResourceState(inst)
    time_update(st, 1, 5, inst)                      # books [5, 10) fully
    return inst, st


def test_time_worked_examples():
    inst, st = gap_state()
    assert (st.free[0, 5:10] == 0).all() and (st.free[0, :5] == 2).all()
    fresh = TimeResourceState(inst)
    assert time_earliest_start(fresh, 2, 4, inst) == 4
    assert time_earliest_start(st, 2, 0, inst) == 0
    assert time_earliest_start(st, 2, 4, inst) == 10
    before = st.free.copy()
    time_update(st, 0, 3, inst)                      # zero demand: no change
    assert (st.free == before).all()
    over = one_resource(2, [0, 5, 3, 0], [0, 2, 2, 0], [[1, 2], [3], [3], []])
    so = TimeResourceState(over)
    time_update(so, 1, 0, over)
    with pytest.raises(ValueError):
        time_update(so, 2, 2, over)


def test_state_ops_fuzz_vs_oracle():
    """Replay random SGS passes step by step; every intermediate state and
    earliest start equals the oracle's (both schemes, 1-5 resources)."""
    rng = np.random.default_rng(5)
    for seed in range(12):
        m = int(rng.integers(1, 6))
        inst = synth.random_instance(int(rng.integers(4, 14)), m, seed=seed, cap_lo=3,
                                     cap_hi=12, demand_density=0.7)
        order = random_topological_order(inst, rng)
        cs, co = CapacityResourceState(inst), CapacityResourceState(inst).levels.copy()
        ts = TimeResourceState(inst)
        to = ts.free.copy()
        starts_c, starts_t = {}, {}
        for act in map(int, order):
            es = max((starts_c[p] + int(inst.durations[p]) for p in inst.predecessors[act]),
                     default=0)
            e_dev = cap_earliest_start(cs, act, inst)
            assert e_dev == oracle.cap_earliest_start(inst, co, act)
            s = max(es, e_dev)
            cap_update(cs, act, s, inst)
            oracle.cap_update(inst, co, act, s)
            assert (cs.levels == co).all(), (seed, act)
            starts_c[act] = s
            es_t = max((starts_t[p] + int(inst.durations[p]) for p in inst.predecessors[act]),
                       default=0)
            st = time_earliest_start(ts, act, es_t, inst)
            assert st == oracle.time_earliest_start(inst, to, act, es_t)
            time_update(ts, act, st, inst)
            oracle.time_update(inst, to, act, st)
            assert (ts.free == to).all(), (seed, act)
            starts_t[act] = st


def test_cap_update_closed_form_random_rows():
    """Alg. 4 on arbitrary descending rows -- runs of equal entries, rows
    longer than a warp (up to 120 entries), demands above 32 -- through
    rcpsp_state_op (the SGS's warp-wide closed form, sgs.cuh:cap_update_row)
    against the reference's loop (oracle.cap_update, kernels.py:81-110).
    Starts are at or above the Eq. 7 bound, as the SGS guarantees."""
    rng = np.random.default_rng(11)
    for trial in range(1500):
        cap = int(rng.choice([3, 17, 31, 32, 33, 40, 64, 75, 120]))
        m = int(rng.integers(1, 4))
        caps = [cap] + [int(rng.integers(1, cap + 1)) for _ in range(m - 1)]
        dur = int(rng.integers(1, 13))
        dem = [int(rng.integers(1, c + 1)) if rng.random() < 0.8 else 0 for c in caps]
        inst = make_instance("row", [0, dur, 0], caps, [[0] * m, dem, [0] * m],
                             [[1], [2], []])
        st = CapacityResourceState(inst)
        hi = int(rng.choice([2, 6, 40]))
        for k, c in enumerate(caps):
            st.levels[k, :c] = np.sort(rng.integers(0, hi + 1, c))[::-1]
        ref = st.levels.copy()
        es = cap_earliest_start(st, 1, inst)
        assert es == oracle.cap_earliest_start(inst, ref, 1)
        s = es + int(rng.choice([0, 0, 1, 3]))
        cap_update(st, 1, s, inst)
        oracle.cap_update(inst, ref, 1, s)
        assert (st.levels == ref).all(), (trial, caps, dem, dur, s)
        assert st.rows_descending()


def test_cap_update_below_bound_refused():
    """A cap_update start below Eq. 7's bound (no SGS produces one) is refused
    loudly with the state untouched, instead of a silently different row."""
    inst = one_resource(4, [0, 3, 2, 0], [0, 3, 2, 0], [[1, 2], [3], [3], []])
    st = CapacityResourceState(inst)
    cap_update(st, 1, 0, inst)
    es = cap_earliest_start(st, 2, inst)
    assert es == 3
    before = st.levels.copy()
    with pytest.raises(ValueError, match="below the earliest resource start"):
        cap_update(st, 2, es - 1, inst)          # the host mirror refuses first
    with pytest.raises(ValueError, match="below the capacity bound"):
        device.state_op(inst, "cap_update", st.levels, 2, es - 1)  # the C ABI itself
    assert (st.levels == before).all()
    cap_update(st, 2, es, inst)
    ref = before.copy()
    oracle.cap_update(inst, ref, 2, es)
    assert (st.levels == ref).all()
