"""GPU parity: the sm_100a kernels against the reference's golden vectors and
the CPU oracle, bit-exact (integer work -- no tolerance anywhere)."""

import numpy as np
import pytest

import oracle
from conftest import chain_instance, random_topological_order, random_topological_orders

pytestmark = pytest.mark.gpu

from paper_1711_04556_b200 import (EvalMode, SearchParams, check_schedule_feasible,  # noqa: E402
                                   critical_path_length, device, evaluate, initial_order,
                                   orchestrate, orchestrate_batch, synth)
from paper_1711_04556_b200.cooperation import initialize_working_set  # noqa: E402

GROUPS = (32, 16, 8)        # TIME lanes per schedule
CAP_GROUPS = (32, 1)        # CAPACITY: warp per schedule / thread per schedule


@pytest.mark.parametrize("group", GROUPS)
def test_eval_golden(golden, ginst, group):
    by_inst: dict = {}
    for rec in golden["evaluate"]:
        by_inst.setdefault(rec["instance"], []).append(rec)
    for name, recs in by_inst.items():
        orders = np.array([r["order"] for r in recs], np.int32)
        for mode in (0, 1):
            c, s = device.eval_batch(ginst[name], orders, mode, group=group)
            assert c.tolist() == [r[f"cmax{mode}"] for r in recs], (name, mode)
            assert s.tolist() == [r[f"starts{mode}"] for r in recs], (name, mode)


def test_worked_example(ginst):
    ex = ginst["example12"]
    s = evaluate(np.array([0, 1, 2, 3, 4, 6, 5, 7, 9, 10, 8, 11]), ex, 1)
    assert s.cmax == 22 and s.starts.tolist() == [0, 0, 4, 4, 7, 12, 9, 12, 20, 15, 16, 22]
    assert check_schedule_feasible(ex, s)[0]
    gap = ginst["gap"]
    assert evaluate(np.arange(5), gap, 1).cmax == 10
    assert evaluate(np.arange(5), gap, 0).cmax == 13
    d2 = ginst["dummy2"]
    for mode in (0, 1):
        sch = evaluate(np.array([0, 1]), d2, mode)
        assert sch.cmax == 0 and sch.starts.tolist() == [0, 0]
    roomy = ginst["roomy"]
    for mode in (0, 1):
        assert evaluate(initial_order(roomy, False), roomy, mode).cmax == critical_path_length(roomy)


FUZZ_CONFIGS = ("j30", "j60", "j120", "act300", "j30p", "j60p", "j120p")


def _oracle_parallel(inst, orders, mode, reverse=False, chunks=16):
    """oracle.evaluate_batch over row chunks in threads (ctypes drops the GIL)."""
    from concurrent.futures import ThreadPoolExecutor
    parts = np.array_split(orders, min(chunks, max(1, len(orders))))
    with ThreadPoolExecutor(max_workers=chunks) as ex:
        res = list(ex.map(lambda o: oracle.evaluate_batch(inst, o, mode, reverse=reverse), parts))
    return np.concatenate([c for c, _ in res]), np.concatenate([s for _, s in res])


def _fuzz(cfg, per_inst, n_inst, groups_time, groups_cap, seed):
    insts = synth.benchmark_batch(cfg, n_inst, first_seed=11)
    rng = np.random.default_rng(seed)
    for inst in insts:
        orders = random_topological_orders(inst, rng, per_inst)
        orders[: min(50, per_inst)] = np.stack(
            [random_topological_order(inst, rng) for _ in range(min(50, per_inst))])
        for mode in (0, 1):
            want_c, want_s = _oracle_parallel(inst, orders, mode)
            for group in groups_time if mode == 1 else groups_cap:
                got_c, got_s = device.eval_batch(inst, orders, mode, group=group)
                assert np.array_equal(got_c, want_c), (cfg, mode, group)
                assert np.array_equal(got_s, want_s), (cfg, mode, group)
        # reversed project (FBI backward pass): orders topological on the reverse graph
        rev = orders[:, ::-1].copy()
        for mode in (0, 1):
            want_c, want_s = _oracle_parallel(inst, rev, mode, reverse=True)
            got_c, got_s = device.eval_batch(inst, rev, mode, reverse=True)
            assert np.array_equal(got_c, want_c) and np.array_equal(got_s, want_s)


@pytest.mark.parametrize("cfg", FUZZ_CONFIGS)
def test_eval_fuzz_vs_oracle(cfg):
    """10^4 precedence-feasible orders per config (2 instances x 5000; Gen-R
    and the benchmarked Gen-P), both modes, every group size, start times
    included; plus reversed-project evaluation."""
    _fuzz(cfg, 5000, 2, GROUPS, CAP_GROUPS, 5)


@pytest.mark.slow
@pytest.mark.parametrize("cfg", FUZZ_CONFIGS)
def test_eval_fuzz_1e5_vs_oracle(cfg):
    """10^5 orders per config (4 instances x 25000), both modes, the search's
    evaluator groups (TIME 32, CAPACITY 32 and 1), starts included."""
    _fuzz(cfg, 25000, 4, (32,), CAP_GROUPS, 6)


def test_eval_fuzz_small_shapes():
    """Varied shapes: 1-8 resources, 8/16-bit lanes, tiny and long durations."""
    rng = np.random.default_rng(17)
    for seed in range(40):
        m = int(rng.integers(1, 9))
        cap_hi = int(rng.choice([6, 20, 127, 300]))
        if m > 4 and cap_hi > 127:
            cap_hi = 127
        inst = synth.random_instance(int(rng.integers(3, 40)), m, seed=seed,
                                     cap_lo=max(1, cap_hi // 3), cap_hi=cap_hi,
                                     max_dur=int(rng.choice([3, 10, 40])),
                                     demand_density=float(rng.choice([0.3, 1.0])))
        orders = np.stack([random_topological_order(inst, rng) for _ in range(60)])
        for mode in (0, 1):
            want_c, want_s = oracle.evaluate_batch(inst, orders, mode)
            g = int(rng.choice(GROUPS if mode == 1 else CAP_GROUPS))
            got_c, got_s = device.eval_batch(inst, orders, mode, group=g)
            assert np.array_equal(got_c, want_c), (seed, mode)
            assert np.array_equal(got_s, want_s), (seed, mode)


def test_filter_golden(golden, ginst):
    for rec in golden["filter"]:
        got = device.filter_batch(ginst[rec["instance"]], np.array([rec["order"]]), rec["delta"])
        assert got[0].tolist() == rec["kept"], (rec["instance"], rec["delta"])


def test_filter_fuzz_vs_oracle():
    rng = np.random.default_rng(3)
    for seed in range(20):
        inst = synth.random_instance(int(rng.integers(4, 60)), 2, seed=seed)
        orders = np.stack([random_topological_order(inst, rng) for _ in range(20)])
        for delta in (1, 7, 30, inst.n_activities):
            got = device.filter_batch(inst, orders, delta)
            moves = oracle.neighborhood(inst.n_activities, delta)
            for b in range(len(orders)):
                assert got[b].tolist() == oracle.filter_moves(inst, orders[b], moves).tolist()


@pytest.mark.parametrize("group", GROUPS + (1,))
def test_run_chunk_golden(golden, ginst, group):
    for rec in golden["run_chunk"]:
        if group == 1 and rec["mode"] == 1:
            continue  # group 1 is the thread-per-schedule CAPACITY evaluator
        inst = ginst[rec["instance"]]
        res = device.run_chunk_batch(inst, rec["mode"], rec["delta"], np.array([rec["order"]]),
                                     [np.array(rec["tabu_list"])], [rec["tabu_head"]],
                                     rec["budget"], rec["adopted_cmax"], rec["start_cmax"],
                                     rec["best_known_cmax"], rec["floor_cmax"], group=group)
        st = res["stats"][0]
        iters = int(st[0])
        assert st[:7].tolist() == rec["out_stats"], (rec["instance"], rec["mode"])
        assert res["trace"][0][:iters].tolist() == rec["out_trace"]
        assert res["order"][0].tolist() == rec["out_order"]
        assert res["best_order"][0].tolist() == rec["out_best_order"]
        assert res["tabu"][0].tolist() == rec["out_tabu_list"]


def _swap_rows(order, moves):
    out = np.repeat(order[None], len(moves), 0)
    r = np.arange(len(moves))
    out[r, moves[:, 0]] = order[moves[:, 1]]
    out[r, moves[:, 1]] = order[moves[:, 0]]
    return out


def _check_neighbourhood(inst, orders, mode, delta, group, key):
    """One run_chunk iteration per order: every evaluated swap's makespan ==
    the oracle's full SGS of the swapped order (kernels.py:350-362)."""
    S = len(orders)
    T = 8
    tl = [np.zeros((T, 2), np.int32) for _ in range(S)]
    cm, _ = oracle.evaluate_batch(inst, orders, mode)
    res = device.run_chunk_batch(inst, mode, delta, orders, tl, [0] * S, 1, 0, cm, cm, 0,
                                 group=group)
    nb = oracle.neighborhood(inst.n_activities, delta)
    for b in range(S):
        moves, got = res["neighbourhood"][b]
        want_moves = oracle.filter_moves(inst, orders[b], nb)
        assert moves.tolist() == want_moves.tolist(), key
        if len(moves):
            want, _ = oracle.evaluate_batch(inst, _swap_rows(orders[b], moves), mode)
            assert got.tolist() == want.tolist(), (key, b)


@pytest.mark.parametrize("cfg", ["j30", "j60", "j120", "act300", "j30p", "j60p", "j120p"])
def test_neighbourhood_makespans_vs_oracle(cfg):
    """Prefix-reusing (group 32) and full-SGS (group 16) neighbourhood
    evaluation inside the search kernel, every move checked."""
    rng = np.random.default_rng(21)
    for inst in synth.benchmark_batch(cfg, 2, first_seed=40):
        orders = np.stack([random_topological_order(inst, rng) for _ in range(6)])
        # also orders the search actually visits: FBI-improved ones are denser
        for group in (32, 16):
            _check_neighbourhood(inst, orders, 1, 60, group, (cfg, group))
        for group in CAP_GROUPS if cfg != "act300" else (32,):
            _check_neighbourhood(inst, orders[:3], 0, 60, group, (cfg, "cap", group))


def test_neighbourhood_makespans_shapes():
    """Wide packings (W = 2), long durations, tiny instances, delta = n."""
    rng = np.random.default_rng(23)
    for seed in range(24):
        m = int(rng.integers(1, 9))
        cap_hi = int(rng.choice([6, 20, 127, 300]))
        if m > 4 and cap_hi > 127:
            cap_hi = 127
        inst = synth.random_instance(int(rng.integers(3, 50)), m, seed=100 + seed,
                                     cap_lo=max(1, cap_hi // 3), cap_hi=cap_hi,
                                     max_dur=int(rng.choice([3, 10, 40])),
                                     demand_density=float(rng.choice([0.3, 1.0])))
        orders = np.stack([random_topological_order(inst, rng) for _ in range(4)])
        delta = int(rng.choice([3, 30, inst.n_activities]))
        _check_neighbourhood(inst, orders, 1, delta, 32, seed)
        _check_neighbourhood(inst, orders, 0, delta, int(rng.choice(CAP_GROUPS)), (seed, "cap"))


def _edge_instances():
    """Shapes the prefix-reusing evaluators must survive: zero durations, one
    unit of one resource (fully serial), demand == capacity everywhere, a hub
    with 40 successors (fan-out > 32 -> the multi-round push path), durations
    above 32 (multi-round booking / windows), no resource use at all."""
    from paper_1711_04556_b200 import make_instance
    rng = np.random.default_rng(31)
    out = []
    # zero durations sprinkled in, single resource of capacity 1
    n = 24
    durs = [0] + [int(x) if rng.random() < 0.7 else 0 for x in rng.integers(1, 6, n - 2)] + [0]
    succ = [[1, 2, 3]] + [[min(n - 1, i + 1 + int(rng.integers(0, 3)))] for i in range(1, n - 1)] + [[]]
    out.append(make_instance("serial1", durs, [1], [[0]] + [[1]] * (n - 2) + [[0]], succ))
    # demand == capacity for every used resource
    dem = [[0, 0]] + [[3, 0] if i % 2 else [0, 5] for i in range(1, n - 1)] + [[0, 0]]
    out.append(make_instance("full", [0] + [int(x) for x in rng.integers(1, 8, n - 2)] + [0],
                             [3, 5], dem, succ))
    # hub: activity 1 precedes 40 activities
    n = 46
    succ = ([[1]] + [list(range(2, 42))] + [[42 + (i % 3)] for i in range(2, 42)]
            + [[n - 1] for _ in range(42, n - 1)] + [[]])
    dem = [[0, 0]] + [[int(x) for x in rng.integers(0, 6, 2)] for _ in range(n - 2)] + [[0, 0]]
    out.append(make_instance("hub40", [0] + [int(x) for x in rng.integers(1, 9, n - 2)] + [0],
                             [6, 7], dem, succ))
    # long durations (> 32)
    out.append(synth.random_instance(30, 3, seed=77, cap_lo=4, cap_hi=9, max_dur=70,
                                     demand_density=0.8))
    # no resource demand at all (the SGS is the critical-path schedule)
    out.append(synth.random_instance(25, 2, seed=78, demand_density=0.0))
    return out


def test_neighbourhood_makespans_edge_shapes():
    rng = np.random.default_rng(37)
    for inst in _edge_instances():
        orders = np.stack([random_topological_order(inst, rng) for _ in range(4)])
        for mode, group in ((1, 32), (1, 16), (0, 32), (0, 1)):
            _check_neighbourhood(inst, orders, mode, inst.n_activities, group,
                                 (inst.name, mode, group))


def test_run_chunk_batch_independent(ginst):
    """Several searches in one launch give the same results as one each."""
    inst = ginst["genr60s0"]
    rng = np.random.default_rng(9)
    orders = np.stack([random_topological_order(inst, rng) for _ in range(5)])
    cm, _ = device.eval_batch(inst, orders, 1, want_starts=False)
    T = 250
    tl = [np.zeros((T, 2), np.int32) for _ in orders]
    floor = critical_path_length(inst)
    batch = device.run_chunk_batch(inst, 1, 60, orders, tl, [0] * 5, 7, 0, cm, cm + 3, floor)
    for b in range(5):
        want = oracle.run_chunk(inst, orders[b], tl[b], 0, 7, 0, int(cm[b]), int(cm[b]) + 3,
                                floor, 60, 1)
        assert batch["stats"][b][:7].tolist() == list(want["stats"])
        assert batch["trace"][b][:int(want["stats"][0])].tolist() == want["trace"].tolist()


def test_orchestrate_golden(golden, ginst):
    """B = 1 full trajectories, identical to the reference."""
    for rec in golden["orchestrate"]:
        inst = ginst[rec["instance"]]
        p = SearchParams.defaults_for(inst.n_activities, total_iters=rec["total_iters"],
                                      workers=1, seed=rec["seed"], mode=EvalMode(rec["mode"]),
                                      collect_trace=True, **rec["extra"])
        st = orchestrate(inst, p)
        key = (rec["instance"], rec["total_iters"], rec["mode"])
        assert st.best_cmax == rec["best_cmax"], key
        assert st.evaluations == rec["evaluations"], key
        assert st.exchanges == rec["exchanges"], key
        assert st.diversifications == rec["diversifications"], key
        assert st.forced_tabu_picks == rec["forced_tabu_picks"], key
        assert st.iterations == rec["iterations"], key
        assert st.stop_reason == rec["stop_reason"], key
        assert st.critical_path == rec["critical_path"], key
        assert [t.tolist() for t in st.traces] == rec["traces"], key
        assert st.schedule.starts.tolist() == rec["starts"], key
        assert st.feasible


def test_orchestrate_batch_equals_single(ginst):
    """B = 1 per instance inside a mixed-mode batch == each solved alone (oracle)."""
    names = ["genr30s0", "genr30s1", "example12", "fuzz3", "genr60s0"]
    insts = [ginst[k] for k in names]
    modes = [EvalMode.TIME, EvalMode.CAPACITY, EvalMode.TIME, EvalMode.CAPACITY, EvalMode.TIME]
    p = SearchParams(total_iters=150, workers=1, delta=30, tabu_size=60, seed=4,
                     collect_trace=True)
    out = orchestrate_batch(insts, p, modes)
    for inst, mode, run in zip(insts, modes, out.runs):
        want = oracle.orchestrate(inst, 150, 1, 4, int(mode), delta=30, tabu_size=60,
                                  collect_trace=True)
        assert run.best_cmax == want["best_cmax"]
        assert run.evaluations == want["evaluations"]
        assert [t.tolist() for t in run.traces] == [t.tolist() for t in want["traces"]]


def test_pool_init_matches_oracle(ginst):
    for name, mode in (("genr30s0", 1), ("example12", 0), ("genr120s0", 1)):
        inst = ginst[name]
        p = SearchParams.defaults_for(inst.n_activities, pool_size=16, seed=4)
        counters: dict = {}
        ws = initialize_working_set(inst, p, np.random.default_rng(4), EvalMode(mode),
                                    critical_path_length(inst), counters)
        rng = np.random.default_rng(4)
        evals = 0
        for i, e in enumerate(ws.entries):
            raw = initial_order(inst, True, rng)
            if i % 2 == 0:
                fo, _, _, ev = oracle.fbi(inst, raw, mode)
                evals += ev
            else:
                fo = raw
            assert e.order.tolist() == fo.tolist(), (name, i)
            assert e.cmax == int(oracle.evaluate_batch(inst, fo[None], mode)[0][0])
            evals += 1
        assert counters["evaluations"] == evals


def test_diversify_golden(golden, ginst):
    from paper_1711_04556_b200 import diversify
    for rec in golden["diversify"]:
        rng = np.random.default_rng(rec["seed"])
        out = diversify(np.array(rec["order"]), rec["phi_steps"], ginst[rec["instance"]], rng)
        assert out.tolist() == rec["out"]
        # the caller's rng continues exactly like numpy's after the same draws
        ref = np.random.default_rng(rec["seed"])
        st = oracle.rng_state(rec["seed"])
        oracle.diversify(ginst[rec["instance"]], rec["order"], rec["phi_steps"], st)
        assert rng.integers(1 << 30) == oracle.pcg_integers(st, 1 << 30)
        del ref


def test_rng_probe_golden(golden):
    for rec in golden["rng"]:
        ops = [(0, n) if kind == "int" else (1, n) for kind, n, _ in rec["seq"]]
        out, _ = device.rng_probe(device.rng_words(rec["seed"]), ops)
        flat = []
        for kind, _, want in rec["seq"]:
            flat.extend([want] if kind == "int" else want)
        assert out.tolist() == flat


def test_eq8_probe(golden):
    quads = np.array([[c, ic, bi, best] for c, ic, bi, best, _ in golden["assigned_iterations"]])
    got = device.eq8_probe(quads)
    assert got.tolist() == [w for *_, w in golden["assigned_iterations"]]
    # a dense grid against the host double-precision formula
    import math
    rng = np.random.default_rng(1)
    q = np.stack([rng.integers(50, 400, 20000), rng.integers(0, 30000, 20000),
                  rng.integers(1, 12000, 20000), np.zeros(20000, np.int64)], 1)
    q[:, 3] = q[:, 0] - rng.integers(0, 30, 20000)
    q[:, 3] = np.maximum(q[:, 3], 1)
    got = device.eq8_probe(q)
    want = [math.floor((bi / 5.0) * (0.8 * math.exp(-100.0 * (c / b - 1.0))
                                     + 0.2 * math.exp(-4.0 * (ic / bi))))
            for c, ic, bi, b in q.tolist()]
    assert got.tolist() == want


def test_edge_cases(ginst):
    ex = ginst["example12"]
    st = orchestrate(ex, SearchParams.defaults_for(12, total_iters=0, workers=1, seed=1))
    assert st.iterations == 0 and st.feasible
    chain = chain_instance([2, 2, 2, 2])
    st = orchestrate(chain, SearchParams.defaults_for(6, total_iters=50, workers=1, seed=1,
                                                      collect_trace=True))
    want = oracle.orchestrate(chain, 50, 1, 1, 1, collect_trace=True)
    assert st.evaluations == want["evaluations"] and st.best_cmax == want["best_cmax"]
    roomy = ginst["roomy"]
    st = orchestrate(roomy, SearchParams.defaults_for(12, total_iters=5000, workers=4, seed=2))
    assert st.best_cmax == critical_path_length(roomy) and st.stop_reason == "critical_path"


def test_multi_worker_solve(ginst):
    """B > 1 CTAs share one working set: budget accounting and feasibility."""
    inst = ginst["genr60s0"]
    for workers in (2, 8):
        st = orchestrate(inst, SearchParams.defaults_for(inst.n_activities, total_iters=400,
                                                         workers=workers, seed=3))
        assert st.iterations == 400
        assert st.best_cmax >= critical_path_length(inst)
        assert st.feasible and st.exchanges >= workers
        assert st.evaluations > 400


def test_merge_elites_model(ginst):
    """k_export_elites / k_merge_elites follow the host model in test_multigpu.py."""
    import torch
    from paper_1711_04556_b200.device import BatchSolver, SolveConfig
    from test_multigpu import merge_model
    insts = [ginst["genr30s0"], ginst["genr30s1"]]
    cfg = SolveConfig(total_iters=10, workers=1, pool_size=6, tabu_size=60, delta=30,
                      phi_steps=20, phi_max=3, seed=3)
    s = BatchSolver(insts, [1, 1], cfg)
    s.upload()
    s.pool_init()
    torch.cuda.synchronize()
    I, n_max = 2, s.n_max
    mine = torch.zeros((I, n_max), dtype=torch.int32, device="cuda")
    mine_c = torch.zeros(I, dtype=torch.int32, device="cuda")
    s.export_elites(mine, mine_c)
    pool_c = s.ent_cmax.cpu().numpy().copy()
    pool_o = s.ent_order.cpu().numpy().copy()
    best = s.ws_hdr.cpu().numpy()[:, 5].copy()
    best_o = s.best_order.cpu().numpy().copy()
    assert mine_c.cpu().numpy().tolist() == best.tolist()
    assert (mine.cpu().numpy() == best_o).all()
    # two foreign sources: one better than everything, one duplicate makespan
    rng = np.random.default_rng(0)
    src_c = np.stack([best - 3, pool_c[:, 1]]).astype(np.int32)          # [src, inst]
    src_o = np.stack([[rng.permutation(n_max) for _ in range(I)] for _ in range(2)]).astype(np.int32)
    s.merge_elites(torch.from_numpy(src_o.reshape(2 * I, n_max)).cuda(),
                   torch.from_numpy(src_c.reshape(-1)).cuda(), 2)
    got_c = s.ent_cmax.cpu().numpy()
    got_o = s.ent_order.cpu().numpy()
    got_b = s.ws_hdr.cpu().numpy()[:, 5]
    for i in range(I):
        n = insts[i].n_activities
        pc, po, b, bo = merge_model(pool_c[i], pool_o[i, :, :n], int(best[i]), best_o[i, :n],
                                    src_o[:, i, :n], src_c[:, i])
        assert got_c[i].tolist() == pc
        assert got_o[i, :, :n].tolist() == po
        assert int(got_b[i]) == b
        assert s.best_order.cpu().numpy()[i, :n].tolist() == bo


def test_full_sgs_equals_prefix_reuse():
    """The whole batch solve gives identical trajectories with and without
    prefix reuse (B = 1 per instance, traces compared)."""
    from paper_1711_04556_b200.device import BatchSolver, SolveConfig
    insts = synth.benchmark_batch("j120", 4, first_seed=7)
    modes = [1, 0, 1, 0]
    out = []
    for full, cap_group in ((False, 32), (True, 32), (False, 1), (True, 1)):
        cfg = SolveConfig(total_iters=120, workers=1, pool_size=8, tabu_size=800, delta=60,
                          phi_steps=20, phi_max=3, seed=1, collect_trace=True, full_sgs=full,
                          cap_group=cap_group)
        r = BatchSolver(insts, modes, cfg).run()
        out.append((r.best_cmax.tolist(), r.evaluations.tolist(),
                    [[t.tolist() for t in tr] for tr in r.traces]))
    assert out[0] == out[1] == out[2] == out[3]


def test_cluster_workers_equal_single_cta():
    """A worker spread over a thread-block cluster (2..8 CTAs sharing the
    neighbourhood over distributed shared memory) follows the same trajectory
    as a single-CTA worker (B = 1, traces compared); the multi-worker launch
    with steals keeps its budget accounting."""
    from paper_1711_04556_b200.device import BatchSolver, SolveConfig
    insts = synth.benchmark_batch("j120p", 3, first_seed=150) + \
        synth.benchmark_batch("j60", 1, first_seed=3)
    # two-word packing (6 resources) with durations > 32 (the multi-round paths)
    wide = synth.random_instance(50, 6, seed=91, cap_lo=20, cap_hi=60, max_dur=45,
                                 demand_density=0.6)
    for modes, cap_group in (([1] * 4, None), ([1, 0, 0, 1], 32), ([0, 1, 0, 0], 1)):
        out = []
        for cl in (1, 2, 8):
            cfg = SolveConfig(total_iters=80, workers=1, pool_size=8, tabu_size=800, delta=60,
                              phi_steps=20, phi_max=3, seed=2, collect_trace=True, cluster=cl,
                              cap_group=cap_group)
            r = BatchSolver(insts, modes, cfg).run()
            out.append((r.best_cmax.tolist(), r.evaluations.tolist(),
                        [[t.tolist() for t in tr] for tr in r.traces]))
        assert out[0] == out[1] == out[2], (modes, cap_group)
    for mode in (1, 0):
        out = []
        for cl in (1, 4):
            cfg = SolveConfig(total_iters=60, workers=1, pool_size=8, tabu_size=250, delta=60,
                              phi_steps=20, phi_max=3, seed=5, collect_trace=True, cluster=cl)
            r = BatchSolver([wide], [mode], cfg).run()
            out.append((r.best_cmax.tolist(), r.evaluations.tolist(),
                        [[t.tolist() for t in tr] for tr in r.traces]))
        assert out[0] == out[1], ("wide", mode)
        want = oracle.orchestrate(wide, 60, 1, 5, mode, delta=60, tabu_size=250,
                                  pool_size=8, collect_trace=True)
        assert out[0][0] == [want["best_cmax"]] and out[0][1] == [want["evaluations"]]
        assert out[0][2][0] == [t.tolist() for t in want["traces"]], ("wide", mode)
    cfg = SolveConfig(total_iters=300, workers=3, pool_size=8, tabu_size=800, delta=60,
                      phi_steps=20, phi_max=3, seed=2, cluster=4)
    r = BatchSolver(insts, [1] * 4, cfg).run()
    assert ((r.iterations == 300) | (r.best_cmax == r.critical_path)).all()


def test_time_limited_solve_stops_on_the_device_clock():
    """SolveConfig.time_limit_s: the search stops on %globaltimer -- well before
    the iteration budget, close to the time limit -- and the result is a valid
    schedule (the budget's only effect is where the search stops)."""
    from paper_1711_04556_b200.device import BatchSolver, SolveConfig
    insts = synth.benchmark_batch("j120p", 6, first_seed=20)
    cfg = SolveConfig(total_iters=10 ** 7, workers=4, pool_size=8, tabu_size=800, delta=60,
                      phi_steps=20, phi_max=3, seed=1, time_limit_s=0.4)
    r = BatchSolver(insts, [1] * 6, cfg).run()
    assert r.search_ms * 1e-3 < 1.0
    # it ran to the limit unless every instance reached the critical path first
    assert r.search_ms * 1e-3 > 0.3 or (r.best_cmax == r.critical_path).all()
    assert (r.iterations < 10 ** 7).all()
    # an instance the pool already solved to the critical path never searches
    assert ((r.iterations > 0) | (r.best_cmax == r.critical_path)).all()
    for i, inst in enumerate(insts):
        from paper_1711_04556_b200 import evaluate
        n = inst.n_activities
        assert evaluate(r.best_order[i, :n], inst, 1).cmax == int(r.best_cmax[i])


def test_batch_solve_shapes_vs_oracle():
    """Full B = 1 solves of varied shapes (1-8 resources, 8/16-bit packings,
    long durations, sparse demand) in one mixed batch: traces, evaluations and
    best makespans equal the oracle's for every instance and mode."""
    from paper_1711_04556_b200.device import BatchSolver, SolveConfig
    rng = np.random.default_rng(43)
    insts, modes = [], []
    for seed in range(12):
        m = int(rng.integers(1, 9))
        cap_hi = int(rng.choice([6, 20, 127, 300]))
        if m > 4 and cap_hi > 127:
            cap_hi = 127
        insts.append(synth.random_instance(int(rng.integers(8, 60)), m, seed=300 + seed,
                                           cap_lo=max(1, cap_hi // 3), cap_hi=cap_hi,
                                           max_dur=int(rng.choice([5, 10, 40])),
                                           demand_density=float(rng.choice([0.3, 0.7]))))
        modes.append(seed % 2)
    cfg = SolveConfig(total_iters=40, workers=1, pool_size=6, tabu_size=60, delta=30,
                      phi_steps=20, phi_max=3, seed=7, collect_trace=True)
    r = BatchSolver(insts, modes, cfg).run()
    for i, (inst, mode) in enumerate(zip(insts, modes)):
        want = oracle.orchestrate(inst, 40, 1, 7, mode, delta=30, tabu_size=60, pool_size=6,
                                  collect_trace=True)
        assert int(r.best_cmax[i]) == want["best_cmax"], (i, mode)
        assert int(r.evaluations[i]) == want["evaluations"], (i, mode)
        assert [t.tolist() for t in r.traces[i]] == [t.tolist() for t in want["traces"]], i


def test_multi_worker_batch_shapes_feasible():
    """B > 1 with steals (and clusters where the launch is small) over varied
    shapes: every instance consumes exactly its budget (or stops at the
    critical path) and its best order's schedule is feasible with the
    reported makespan."""
    from paper_1711_04556_b200 import evaluate
    from paper_1711_04556_b200.device import BatchSolver, SolveConfig
    rng = np.random.default_rng(47)
    insts, modes = [], []
    for seed in range(10):
        m = int(rng.integers(1, 7))
        cap_hi = int(rng.choice([8, 30, 120]))
        insts.append(synth.random_instance(int(rng.integers(10, 70)), m, seed=400 + seed,
                                           cap_lo=max(1, cap_hi // 3), cap_hi=cap_hi,
                                           max_dur=int(rng.choice([8, 36])),
                                           demand_density=0.6))
        modes.append(int(rng.integers(0, 2)))
    for cluster in (None, 1):
        cfg = SolveConfig(total_iters=150, workers=3, pool_size=6, tabu_size=60, delta=30,
                          phi_steps=20, phi_max=3, seed=11, cluster=cluster)
        r = BatchSolver(insts, modes, cfg).run()
        for i, (inst, mode) in enumerate(zip(insts, modes)):
            assert r.iterations[i] == 150 or r.best_cmax[i] == r.critical_path[i], i
            n = inst.n_activities
            sched = evaluate(r.best_order[i, :n], inst, mode)
            assert sched.cmax == int(r.best_cmax[i]), (i, mode)
            ok, problems = check_schedule_feasible(inst, sched)
            assert ok, (i, problems[:3])


def test_reference_backend_fingerprint(golden):
    """The reference's own backend-parity harness (helpers.py:190-223,
    test_backends.py:36-41) with this package as the backend: the same digest
    -- evaluations in both modes, filters, forward-backward improvement and a
    200-iteration seeded search trace -- recomputed through this package's
    API on the GPU equals the one the reference produced with numba
    (tests/golden/fingerprint.json, tests/golden/make_fingerprint.py)."""
    import json
    from conftest import ROOT
    from paper_1711_04556_b200 import (filter_infeasible, forward_backward_improve,
                                       generate_reduced_neighborhood)
    want = json.loads((ROOT / "tests" / "golden" / "fingerprint.json").read_text())
    out: dict = {}
    rng = np.random.default_rng(2024)
    evals, filters = [], []
    for seed in range(6):
        inst = synth.random_instance(12, 2, seed=seed)
        order = random_topological_order(inst, rng)
        for mode in (0, 1):
            sched = evaluate(order, inst, mode)
            evals.append([sched.cmax] + sched.starts.tolist())
        moves = generate_reduced_neighborhood(order, 8)
        filters.append(filter_infeasible(moves, order, inst).tolist())
        improved, sched = forward_backward_improve(inst, order, 1)
        evals.append([sched.cmax] + improved.tolist())
    out["evals"] = evals
    out["filters"] = filters
    inst = synth.random_instance(14, 3, seed=99)
    params = SearchParams.defaults_for(16, total_iters=200, workers=1, seed=5,
                                       collect_trace=True)
    stats = orchestrate(inst, params)
    out["search_best"] = stats.best_cmax
    out["search_evals"] = stats.evaluations
    out["search_trace"] = [int(x) for chunk in stats.traces for x in chunk]
    assert json.loads(json.dumps(out)) == want


def test_sized_profile_trajectories_match_oracle():
    """TIME with per-warp profiles sized by a makespan bound (SolveConfig.
    profile_slots forced): moves that would book past the profile are
    abandoned and evaluated exactly on the CTA's full-horizon region.  B = 1
    trajectories equal the oracle's with a generous size (overflow rare), a
    tight one (frequent fallbacks) and one below the current schedule's
    makespan (every move on the fallback)."""
    from paper_1711_04556_b200.device import BatchSolver, SolveConfig
    insts = synth.benchmark_batch("j60p", 2, first_seed=0) + \
        synth.benchmark_batch("j120p", 1, first_seed=3)
    want = [oracle.orchestrate(x, 60, 1, 3, 1, delta=60, tabu_size=250, pool_size=8,
                               collect_trace=True) for x in insts]
    for slots in (400, 160, 96):
        cfg = SolveConfig(total_iters=60, workers=1, pool_size=8, tabu_size=250, delta=60,
                          phi_steps=20, phi_max=3, seed=3, collect_trace=True, cluster=1,
                          profile_slots=slots)
        r = BatchSolver(insts, [1] * len(insts), cfg).run()
        for i, w in enumerate(want):
            assert int(r.best_cmax[i]) == w["best_cmax"], (slots, i)
            assert int(r.evaluations[i]) == w["evaluations"], (slots, i)
            assert [t.tolist() for t in r.traces[i]] == [t.tolist() for t in w["traces"]], \
                (slots, i)
    # the auto choice on a 300-activity batch keeps the budget accounting and
    # valid best schedules
    big = synth.benchmark_batch("act300", 4, first_seed=9)
    cfg = SolveConfig(total_iters=20, workers=2, pool_size=8, tabu_size=800, delta=60,
                      phi_steps=20, phi_max=3, seed=1)
    r = BatchSolver(big, [1] * 4, cfg).run()
    for i, inst in enumerate(big):
        assert r.iterations[i] == 20 or r.best_cmax[i] == r.critical_path[i]
        n = inst.n_activities
        assert evaluate(r.best_order[i, :n], inst, 1).cmax == int(r.best_cmax[i])


def test_capacity_beyond_time_packing():
    """CAPACITY has no packing limit (kernels.py:68-110 works on any m and
    capacity): instances with 9-24 resources, or more than 4 resources with
    capacities above 127, evaluate and search in CAPACITY mode equal to the
    oracle, while TIME is refused loudly (its packed profile cannot hold them)."""
    from paper_1711_04556_b200.device import BatchSolver, SolveConfig
    rng = np.random.default_rng(29)
    insts = [synth.random_instance(30, 12, seed=1, cap_lo=5, cap_hi=20, demand_density=0.5),
             synth.random_instance(40, 6, seed=2, cap_lo=100, cap_hi=250, demand_density=0.6),
             synth.random_instance(25, 24, seed=3, cap_lo=2, cap_hi=9, demand_density=0.3)]
    for inst in insts:
        orders = np.stack([random_topological_order(inst, rng) for _ in range(40)])
        want_c, want_s = oracle.evaluate_batch(inst, orders, 0)
        for g in CAP_GROUPS:
            got_c, got_s = device.eval_batch(inst, orders, 0, group=g)
            assert np.array_equal(got_c, want_c) and np.array_equal(got_s, want_s), inst.name
        with pytest.raises(ValueError):
            device.eval_batch(inst, orders, 1)
    cfg = SolveConfig(total_iters=30, workers=1, pool_size=6, tabu_size=60, delta=30,
                      phi_steps=20, phi_max=3, seed=3, collect_trace=True)
    r = BatchSolver(insts, [0] * len(insts), cfg).run()
    for i, inst in enumerate(insts):
        want = oracle.orchestrate(inst, 30, 1, 3, 0, delta=30, tabu_size=60, pool_size=6,
                                  collect_trace=True)
        assert int(r.best_cmax[i]) == want["best_cmax"], i
        assert int(r.evaluations[i]) == want["evaluations"], i
        assert [t.tolist() for t in r.traces[i]] == [t.tolist() for t in want["traces"]], i


def test_decide_dynamic_on_the_device():
    """The measured mode choice (selector.py decide_dynamic, the reference's
    'auto-measure', cooperation.py:204-225): both modes timed on the GPU, a
    CAPACITY-only instance picks CAPACITY, and a B = 1 solve under the
    re-measuring controller returns a feasible, re-evaluated best schedule."""
    from paper_1711_04556_b200.cooperation import choose_mode
    from paper_1711_04556_b200.selector import decide_dynamic, measure_modes
    from paper_1711_04556_b200 import moves as hmoves
    inst = synth.benchmark_batch("j30p", 1, first_seed=5)[0]
    probe = hmoves.initial_order(inst, shuffle=False)
    t = measure_modes(inst, probe, 10)
    assert set(t) == {EvalMode.TIME, EvalMode.CAPACITY} and all(0 < x < 1 for x in t.values())
    assert decide_dynamic(inst, probe, 10) in (EvalMode.TIME, EvalMode.CAPACITY)
    wide = synth.random_instance(30, 12, seed=1, cap_lo=5, cap_hi=20, demand_density=0.5)
    assert decide_dynamic(wide, hmoves.initial_order(wide, shuffle=False), 10) == EvalMode.CAPACITY
    hard = synth.benchmark_batch("j120p", 1, first_seed=0)[0]  # not solved to its CPM early
    p = SearchParams.defaults_for(hard.n_activities, total_iters=300, workers=1, seed=2)
    p.measure_window = 100
    mode, ctl = choose_mode(hard, p, "auto-measure")
    st = orchestrate(hard, p, mode, mode_controller=ctl)
    # (orchestrate re-evaluates the stored best order and checks it feasible)
    assert ctl.measurements >= 2 and st.feasible
    assert st.iterations <= 300 and st.best_cmax >= st.critical_path


def test_large_project_kernel_shapes_vs_oracle():
    """The large-project search kernel (projects above 64 activities: 20-warp
    CTAs, long-suffix phase-B loop) on both TIME packings (one and two words
    per slot) and on CAPACITY: B = 1 trajectories equal to the oracle's."""
    from paper_1711_04556_b200.device import BatchSolver, SolveConfig
    insts = [synth.random_instance(90, 3, seed=71, cap_lo=6, cap_hi=20),           # W = 1
             synth.random_instance(80, 6, seed=72, cap_lo=6, cap_hi=20),           # W = 2
             synth.benchmark_batch("j120p", 1, first_seed=77)[0]]
    for mode in (1, 0):
        cfg = SolveConfig(total_iters=40, workers=1, pool_size=6, tabu_size=60, delta=30,
                          phi_steps=20, phi_max=3, seed=9, collect_trace=True)
        for inst in insts:  # one launch per packing (TIME groups by words)
            r = BatchSolver([inst], [mode], cfg).run()
            want = oracle.orchestrate(inst, 40, 1, 9, mode, delta=30, tabu_size=60, pool_size=6,
                                      collect_trace=True)
            assert int(r.best_cmax[0]) == want["best_cmax"], (inst.name, mode)
            assert int(r.evaluations[0]) == want["evaluations"], (inst.name, mode)
            assert [t.tolist() for t in r.traces[0]] == [t.tolist() for t in want["traces"]]
