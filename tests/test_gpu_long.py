"""Long B = 1 trajectories on the benchmarked workload (Gen-P j120), device vs
the pinned fixture tests/golden/long_trajectories.json (made by
tests/golden/make_long_trajectories.py: the CPU oracle and, in the build
container, the reference package itself agree on every case).  1000-1500
iterations with a pool of 16; the cases include diversification and forced
tabu picks, in both evaluation modes.  Bit-exact: traces (sha256 of the
int32 trace + chunk lengths = the exchange structure), evaluations,
exchanges, diversifications, forced picks, best makespan and schedule."""

import hashlib
import json

import numpy as np
import pytest

from conftest import ROOT
from paper_1711_04556_b200 import EvalMode, SearchParams, orchestrate, synth

pytestmark = pytest.mark.gpu

FIXTURE = ROOT / "tests" / "golden" / "long_trajectories.json"
CASES = json.loads(FIXTURE.read_text())["cases"]


def _sha(chunks) -> tuple[str, int]:
    flat = np.concatenate([np.asarray(c, np.int32) for c in chunks]) if chunks else \
        np.zeros(0, np.int32)
    return hashlib.sha256(flat.astype("<i4").tobytes()).hexdigest(), int(len(flat))


def test_fixture_covers_the_hard_paths():
    assert len(CASES) >= 3
    assert all(c["total_iters"] >= 1000 and c["pool_size"] == 16 for c in CASES)
    assert sum(c["diversifications"] for c in CASES) > 0
    assert sum(c["forced_tabu_picks"] for c in CASES) > 0
    assert {c["mode"] for c in CASES} == {0, 1}


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c['config']}-{c['index']}-m{c['mode']}-d{c['delta']}")
def test_long_trajectory_matches(case):
    inst = synth.benchmark_batch(case["config"], 1, first_seed=case["index"])[0]
    p = SearchParams.defaults_for(inst.n_activities, total_iters=case["total_iters"], workers=1,
                                  seed=case["seed"], mode=EvalMode(case["mode"]),
                                  collect_trace=True, delta=case["delta"],
                                  tabu_size=case["tabu_size"], phi_max=case["phi_max"],
                                  pool_size=case["pool_size"])
    st = orchestrate(inst, p)
    key = (case["index"], case["mode"], case["delta"])
    sha, ln = _sha(st.traces)
    assert st.best_cmax == case["best_cmax"], key
    assert st.evaluations == case["evaluations"], key
    assert st.exchanges == case["exchanges"], key
    assert st.diversifications == case["diversifications"], key
    assert st.forced_tabu_picks == case["forced_tabu_picks"], key
    assert st.iterations == case["iterations"], key
    assert st.critical_path == case["critical_path"], key
    assert [len(c) for c in st.traces] == case["chunk_lens"], key
    assert (sha, ln) == (case["trace_sha256"], case["trace_len"]), key
    if "starts" in case:
        assert st.schedule.starts.tolist() == case["starts"], key
    assert st.feasible


def test_long_trajectory_single_cta_equals_cluster():
    """The same trajectory with one CTA per worker (no cluster) -- the
    batch path's mapping -- as with the single-instance cluster default."""
    from paper_1711_04556_b200.device import BatchSolver, SolveConfig
    case = CASES[1]
    inst = synth.benchmark_batch(case["config"], 1, first_seed=case["index"])[0]
    cfg = SolveConfig(total_iters=case["total_iters"], workers=1, pool_size=16,
                      tabu_size=case["tabu_size"], delta=case["delta"], phi_steps=20,
                      phi_max=case["phi_max"], seed=case["seed"], collect_trace=True, cluster=1)
    r = BatchSolver([inst], [case["mode"]], cfg).run()
    assert int(r.best_cmax[0]) == case["best_cmax"]
    assert int(r.evaluations[0]) == case["evaluations"]
    assert _sha(r.traces[0]) == (case["trace_sha256"], case["trace_len"])
