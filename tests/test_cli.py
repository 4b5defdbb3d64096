"""CLI harness (reference cli.py:185-209, test_cli.py:54-65 shape)."""
import pytest

from paper_1308_1343_b200.cli import build_parser, main


def test_parser_defaults_match_reference():
    a = build_parser().parse_args(["stencil-bench"])
    assert (a.extent, a.iters, a.seed) == (64, 100, 20130715)
    b = build_parser().parse_args(["config-bench", "--config", "4", "--tune", "0"])
    assert (b.config, b.tune) == (4, 0)


def test_bad_flag_exits_2():
    with pytest.raises(SystemExit) as e:
        main(["stencil-bench", "--bogus"])
    assert e.value.code == 2


@pytest.mark.gpu
def test_stencil_bench_bit_identical_and_csv(tmp_path, capsys):
    out = tmp_path / "bench.csv"
    rc = main(["stencil-bench", "--extent", "16", "--iters", "8", "--threads", "2", "--out", str(out)])
    assert rc == 0
    assert "bit-identical: True" in capsys.readouterr().out
    lines = out.read_text().splitlines()
    assert lines[0] == "impl,iter,elapsed_ns,phase,is_best"
    assert all(len(l.split(",")) == 5 for l in lines)
    impls = {l.split(",")[0] for l in lines[1:]}
    assert impls == {"serial", "naive", "tuned", "graphed", "persistent"}
    phases = {l.split(",")[3] for l in lines[1:] if l.startswith("tuned")}
    assert phases <= {"warmup", "initial", "climbing", "excursion"}


@pytest.mark.gpu
@pytest.mark.parametrize("config", [1, 2, 3, 4, 5])
def test_config_bench_runs(config, capsys):
    import json
    assert main(["config-bench", "--config", str(config), "--iters", "3", "--tune", "6"]) == 0
    rec = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert rec["config"] == config and rec["gpts"] > 0


def test_tune_sim(tmp_path, capsys):
    from paper_1308_1343_b200.cli import main
    out = tmp_path / "sim.csv"
    assert main(["tune-sim", "--seeds", "20", "--iters", "50", "--out", str(out)]) == 0
    assert "seeds within 10%" in capsys.readouterr().out
    rows = out.read_text().splitlines()
    assert rows[0] == "seed,best_cost,evals_to_within_10pct,total_cost" and len(rows) == 21


@pytest.mark.gpu
def test_quickstart_example_runs():
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    r = subprocess.run([sys.executable, str(root / "examples" / "quickstart.py")], capture_output=True, text=True,
                       timeout=600, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    out = r.stdout
    assert "jacobi:" in out and "level: 3 boxes" in out and "wave:" in out and "derivatives: 10 outputs" in out
