"""Host-side logic that needs no GPU: instance model and PSPLIB I/O, the
Gen-R generator, device packing, rules, parameters, the host tabu mirror and
the C-ABI library's exported symbols (dlopen only, no CUDA call)."""

import ctypes
import io
import re
from pathlib import Path

import numpy as np
import pytest

from conftest import ROOT, chain_instance
from paper_1711_04556_b200 import (DEFAULT_RULES, EvalMode, PsplibParseError, SearchParams,
                                   TabuState, compute_levels, critical_path_length,
                                   extract_features, generate_reduced_neighborhood,
                                   initial_order, is_order_valid, load_psplib, make_instance,
                                   parse_psplib, parse_rules, validate, write_psplib)
from paper_1711_04556_b200 import decide_static, device, synth
from paper_1711_04556_b200.cooperation import WorkingSetEntry, assigned_iterations
from paper_1711_04556_b200.moves import neighborhood_size

EXAMPLE_ORDER = [0, 1, 2, 3, 4, 6, 5, 7, 9, 10, 8, 11]


def test_golden_instances_regenerate(golden):
    """synth.random_instance reproduces the reference's helpers.random_instance."""
    for name, d in golden["instances"].items():
        r = d.get("recipe")
        if not r:
            continue
        inst = synth.random_instance(r["n_real"], r["m"], seed=r["seed"],
                                     cap_lo=r["cap_lo"], cap_hi=r["cap_hi"],
                                     demand_density=r["demand_density"])
        assert inst.durations.tolist() == d["durations"], name
        assert inst.capacities.tolist() == d["capacities"], name
        assert inst.demands.tolist() == d["demands"], name
        assert [list(s) for s in inst.successors] == d["successors"], name
        assert inst.name == d["name"]


def test_psplib_roundtrip(ginst):
    for name in ("example12", "genr30s0", "fuzz4"):
        inst = ginst[name]
        back = parse_psplib(write_psplib(inst), name=inst.name)
        assert back.durations.tolist() == inst.durations.tolist()
        assert back.demands.tolist() == inst.demands.tolist()
        assert back.successors == inst.successors
        assert back.capacities.tolist() == inst.capacities.tolist()


def test_psplib_errors():
    with pytest.raises(PsplibParseError, match="missing section"):
        parse_psplib("nothing here")
    bad = write_psplib(chain_instance([1, 2])).replace("   1        1            1",
                                                       "   1        2            1")
    with pytest.raises(PsplibParseError, match=r"line \d+: .*modes"):
        parse_psplib(bad)


def test_load_psplib_file(tmp_path, ginst):
    path = tmp_path / "ex12.sm"
    path.write_text(write_psplib(ginst["example12"]))
    inst = load_psplib(path)
    assert inst.name == "ex12" and inst.n_activities == 12


def test_example_graph_quantities(ginst):
    ex = ginst["example12"]
    assert critical_path_length(ex) == 16
    assert initial_order(ex, shuffle=False).tolist() == [0, 1, 2, 3, 4, 6, 5, 7, 8, 9, 10, 11]
    assert is_order_valid(ex, np.array(EXAMPLE_ORDER))
    assert not is_order_valid(ex, np.array([0, 3, 2, 1, 4, 6, 5, 7, 9, 10, 8, 11]))
    assert validate(ex) == []
    assert compute_levels(ex)[0] == [0]
    f = extract_features(ex)
    assert f.max_capacity == 6 and f.critical_path_length == 16
    assert decide_static(f) == EvalMode.CAPACITY          # capacities 6, 6


def test_initial_order_matches_reference_rng(golden, ginst):
    for rec in golden["initial_order"]:
        rng = np.random.default_rng(rec["seed"])
        inst = ginst[rec["instance"]]
        got = [initial_order(inst, True, rng).tolist() for _ in rec["orders"]]
        assert got == rec["orders"]


def test_validate_detects_problems():
    inst = make_instance("bad", [1, 2, 0], [2], [[1], [3], [0]], [[1], [2], []])
    msgs = validate(inst)
    assert any("dummy activity 0" in m for m in msgs)
    assert any("demands 3" in m for m in msgs)


def test_neighbourhood_counts():
    order = np.arange(12, dtype=np.int32)
    assert len(generate_reduced_neighborhood(order, 1)) == 9
    assert len(generate_reduced_neighborhood(order, 60)) == 45
    assert len(generate_reduced_neighborhood(order, 2)) == 17
    for n in (5, 12, 32, 62, 122):
        for delta in (1, 2, 30, 60):
            assert neighborhood_size(n, delta) == device.neighborhood_size(n, delta)
            assert neighborhood_size(n, delta) == len(
                generate_reduced_neighborhood(np.arange(n), delta))


def test_search_params_defaults():
    assert (SearchParams.defaults_for(32).delta, SearchParams.defaults_for(32).tabu_size) == (30, 60)
    assert SearchParams.defaults_for(62).tabu_size == 250
    assert SearchParams.defaults_for(92).tabu_size == 600
    assert SearchParams.defaults_for(122).tabu_size == 800
    assert SearchParams(total_iters=10, workers=3).block_iters == 4


def test_rules():
    rules = parse_rules("# c\nmax_capacity <= 6 -> CAPACITY\navg_duration >= 15 -> capacity\n"
                        "default time\n")
    assert len(rules.predicates) == 2 and rules.default == EvalMode.TIME
    with pytest.raises(ValueError, match="default"):
        parse_rules("max_capacity <= 6 -> CAPACITY\n")
    with pytest.raises(ValueError, match="unknown feature"):
        parse_rules("banana <= 6 -> CAPACITY\ndefault TIME\n")
    with pytest.raises(ValueError, match="expected"):
        parse_rules("max_capacity <= -> CAPACITY\ndefault TIME\n")
    for cfg in ("j30", "j60", "j120", "act300"):
        inst = synth.benchmark_batch(cfg, 1)[0]
        assert decide_static(extract_features(inst), DEFAULT_RULES) == EvalMode.TIME


def test_assigned_iterations_host(golden):
    def e(c, ic):
        return WorkingSetEntry(order=np.zeros(2, np.int32), cmax=c,
                               tabu_entries=np.zeros((1, 2), np.int32), tabu_head=0,
                               iter_count=ic)
    assert assigned_iterations(e(100, 0), 1000, 100) == 200
    assert assigned_iterations(e(101, 1000), 1000, 100) == 59
    for cmax, ic, bi, best, want in golden["assigned_iterations"]:
        assert assigned_iterations(e(cmax, ic), bi, best) == want


def test_tabu_mirror():
    st = TabuState(10, size=4)
    st.add(2, 5); st.add(2, 5); st.add(1, 2); st.add(1, 3)
    st.add(1, 4)
    assert st.is_tabu(2, 5)
    st.add(1, 5)
    assert not st.is_tabu(2, 5)
    entries, head = st.snapshot()
    other = TabuState(10, 4)
    other.load(entries, head)
    assert (other.counts == st.counts).all() and other.head == st.head


def test_pack_instance_layout(ginst):
    inst = ginst["genr120s0"]
    blob = device.pack_instance(inst)
    assert blob[device.B_MAGIC] == device.BLOB_MAGIC
    n, m = inst.n_activities, inst.n_resources
    assert blob[device.B_N] == n and blob[device.B_M] == m
    assert blob[device.B_W] == 1 and blob[device.B_LB] == 8
    assert blob[device.B_CPM] == critical_path_length(inst)
    req = blob[blob[device.B_OFF_REQ]:blob[device.B_OFF_REQ] + n].view(np.uint32)
    for act in (0, 5, n - 2):
        for k in range(m):
            assert (int(req[act]) >> (8 * k)) & 0xFF == int(inst.demands[act, k])
    assert blob[device.B_LEN] == len(blob)
    roomy = ginst["roomy"]           # capacities 999 -> 16-bit lanes
    assert device.packing_for(roomy.capacities) == (16, 1)
    assert device.packing_for(np.array([10] * 5)) == (8, 2)
    # no TIME packing: the blob still builds (CAPACITY mode), TIME is refused
    assert device.packing_for(np.array([10] * 9)) == (0, 0)
    assert device.packing_for(np.array([200] * 5)) == (0, 0)
    wide = make_instance("wide", [0, 2, 0], [10] * 9, [[0] * 9, [3] * 9, [0] * 9],
                         [[1], [2], []])
    blob = device.pack_instance(wide)
    assert blob[device.B_W] == 0 and blob[device.B_LB] == 0
    with pytest.raises(device.UnsupportedInstance, match="CAPACITY"):
        device.require_time_packing(blob, device.MODE_TIME)
    device.require_time_packing(blob, device.MODE_CAPACITY)


def test_pack_rejects_overload():
    inst = make_instance("over", [0, 2, 0], [2], [[0], [3], [0]], [[1], [2], []])
    with pytest.raises(ValueError, match="demands 3"):
        device.pack_instance(inst)


def test_library_exports_every_declared_symbol():
    """The C ABI library loads (dlopen) and exports every function the header
    declares; no CUDA call is made."""
    from paper_1711_04556_b200 import _native
    header = (ROOT / "include" / "rcpsp_tabu_b200.h").read_text()
    declared = set(re.findall(r"^\s*(?:int|int64_t|const char \*)\s*\*?(rcpsp_\w+)\(", header,
                              re.M))
    assert declared, "no declarations parsed"
    assert declared == set(_native.EXPORTED)
    if not _native.LIB_PATH.exists():
        pytest.skip("library not built")
    lib = ctypes.CDLL(str(_native.LIB_PATH))
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.rcpsp_abi_version() == _native.ABI_VERSION


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1711_04556_b200 import _native, evaluate
    from paper_1711_04556_b200.instance import make_instance as mk
    inst = mk("t", [0, 1, 0], [1], [[0], [1], [0]], [[1], [2], []])
    with pytest.raises(_native.NativeLibraryError):
        evaluate(np.array([0, 1, 2]), inst, 1)


def test_product_never_imports_oracle():
    """The product package must not import, link or call the CPU oracle."""
    pkg = ROOT / "paper_1711_04556_b200"
    for path in list(pkg.rglob("*.py")) + list(pkg.rglob("*.cu")) + list(pkg.rglob("*.cuh")):
        text = path.read_text()
        assert not re.search(r"^\s*(import|from)\s+oracle\b", text, re.M), path
        assert "liboracle" not in text, path


def test_b200_rules_match_measurements():
    """B200_RULES pick the mode the device measured faster on every family
    of profiles/r2/mode_rules_b200.json (tools/derive_rules.py)."""
    import json
    from types import SimpleNamespace
    from paper_1711_04556_b200 import B200_RULES, DEFAULT_RULES, EvalMode, decide_static
    rows = json.loads((ROOT / "profiles" / "r2" / "mode_rules_b200.json").read_text())["rows"]
    hits = 0
    for r in rows:
        f = SimpleNamespace(max_capacity=r["cap"][1], avg_duration=r["avg_duration"],
                            min_capacity=r["cap"][0], avg_capacity=sum(r["cap"]) / 2,
                            avg_branch_factor=1.5, critical_path_length=0)
        got = decide_static(f, B200_RULES)
        hits += got == (EvalMode.CAPACITY if r["faster"] == "capacity" else EvalMode.TIME)
    assert hits == len(rows) == 15
    # the Gen-R benchmark configs keep TIME under both rule sets
    f = SimpleNamespace(max_capacity=16, avg_duration=5.5, min_capacity=10, avg_capacity=13,
                        avg_branch_factor=1.5, critical_path_length=0)
    assert decide_static(f, B200_RULES) == decide_static(f, DEFAULT_RULES) == EvalMode.TIME


def test_bench_reference_arm_contract():
    """`bench.py --impl reference` (the reference algorithm on the host cores)
    prints one JSON line with the driver's keys; it needs no GPU."""
    import json
    import subprocess
    import sys
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                          "--config", "j30p", "--instances", "40", "--steps", "1",
                          "--warmup", "0", "--cpu-sample", "2", "--iters", "50"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "dtype", "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0


def test_operator_instance_cache_follows_content(ginst):
    """The operator layer's instance cache is keyed by array content: mutating
    the caller's demands / capacities in place (same buffer addresses) must
    give a new instance, not the cached one (kernels.py cache)."""
    from paper_1711_04556_b200 import kernels
    inst = ginst["genr30s0"]
    ka = inst.kernel_arrays
    dur = np.array(ka.durations, np.int32)
    dem = np.array(ka.demands, np.int32)
    cap = np.array(ka.capacities, np.int32)
    pp, pd = np.array(ka.pred_ptr, np.int32), np.array(ka.pred_dat, np.int32)
    first = kernels._instance(dur, dem, cap, pp, pd)
    assert first.demands.tolist() == inst.demands.tolist()
    assert kernels._instance(dur, dem, cap, pp, pd) is first   # same content: cached
    dem[:] = 0
    cap += 5
    second = kernels._instance(dur, dem, cap, pp, pd)
    assert second is not first
    assert int(second.demands.sum()) == 0
    assert second.capacities.tolist() == cap.tolist()


def test_tabu_state_mirror_semantics():
    """TabuState: eviction, duplicate moves, snapshot/load, reference views."""
    st = TabuState(12, size=3)
    for mv in [(1, 2), (3, 5), (1, 2)]:
        st.add(*mv)
    assert st.is_tabu(1, 2) and st.is_tabu(3, 5) and len(st) == 3 and st.head == 0
    st.add(4, 6)                       # evicts the first (1, 2); the copy keeps it tabu
    assert st.is_tabu(1, 2) and st.counts[1, 2] == 1 and st.head == 1
    st.add(7, 8)                       # evicts (3, 5)
    assert not st.is_tabu(3, 5)
    assert st.entries.tolist() == [[4, 6], [7, 8], [1, 2]]
    ent, head = st.snapshot()
    other = TabuState(12, 3)
    other.load(ent, head)
    assert other.entries.tolist() == st.entries.tolist() and other.head == st.head
    assert (other.counts == st.counts).all()
    assert other.packed.tolist() == [(4 << 16) | 6, (7 << 16) | 8, (1 << 16) | 2]
    st.reset()
    assert len(st) == 0 and not st.counts.any()
    with pytest.raises(ValueError):
        TabuState(5, 0)


def test_moves_host_helpers(ginst):
    """moves.py: validity, neighbourhood generation, swap feasibility (position
    bounds) against brute force over the direct edges."""
    from paper_1711_04556_b200 import apply_swap, is_swap_feasible
    from conftest import random_topological_order
    inst = ginst["genr30s0"]
    rng = np.random.default_rng(3)
    order = random_topological_order(inst, rng)
    assert is_order_valid(inst, order)
    nb = generate_reduced_neighborhood(order, 7)
    want = [(u, v) for u in range(1, len(order) - 2)
            for v in range(u + 1, min(u + 7, len(order) - 2) + 1)]
    assert [tuple(x) for x in nb.tolist()] == want
    for u, v in want[::5]:
        sw = apply_swap(order, (u, v))
        assert sw[u] == order[v] and sw[v] == order[u]
        assert is_swap_feasible(order, (u, v), inst) == is_order_valid(inst, sw)
    with pytest.raises(ValueError):
        is_swap_feasible(order, (0, 3), inst)
