"""CLI (reference cli.py): parsing on CPU; solve/bench end to end on the GPU."""

import json

import pytest

from paper_1711_04556_b200 import cli, synth, write_psplib


def test_bounds_and_aggregates(tmp_path):
    p = tmp_path / "b.csv"
    p.write_text("instance,bound\na,10\nb,12\n")
    assert cli.load_bounds(p) == {"a": 10, "b": 12}
    p.write_text("instance,bound\na,10\na,11\n")
    with pytest.raises(ValueError, match="duplicate"):
        cli.load_bounds(p)
    rows = [dict(instance="a", cmax=12, critical_path=10, bound=12, error="", wall_time_s=1.0,
                 evaluations=100),
            dict(instance="b", cmax=11, critical_path=10, bound="", error="", wall_time_s=1.0,
                 evaluations=300)]
    agg = cli.aggregate_rows(rows)
    assert agg["cpm_dev"] == pytest.approx(15.0) and agg["best_sol"] == 1
    assert agg["sched_sec"] == pytest.approx(200.0)


def test_missing_instance_fails(tmp_path):
    with pytest.raises(SystemExit, match="not found"):
        cli.main(["solve", str(tmp_path / "nope.sm")])


@pytest.mark.gpu
def test_solve_deterministic_and_bench(tmp_path, capsys):
    inst = synth.random_instance(12, 2, seed=3)
    path = tmp_path / "x.sm"
    path.write_text(write_psplib(inst))
    argv = ["solve", str(path), "--iters", "300", "--workers", "1", "--seed", "11",
            "--eval", "time", "--trace", str(tmp_path / "t.csv")]
    assert cli.main(argv) == 0
    first = capsys.readouterr().out
    cli.main(argv)
    assert capsys.readouterr().out == first
    assert "feasible: yes" in first
    assert (tmp_path / "t.csv").read_text().startswith("iteration,cmax")
    for s in range(3):
        (tmp_path / f"r{s}.sm").write_text(write_psplib(synth.random_instance(20, 3, seed=s)))
    cli.main(["bench", str(tmp_path), "--iters", "200", "--workers", "2", "--format", "json"])
    out = json.loads(capsys.readouterr().out)
    assert out["aggregates"]["solved"] == 4 and out["aggregates"]["failures"] == 0
    assert all(r["feasible"] for r in out["rows"])
