"""The B200 benchmark harness and CLI: the reference
CLI's flags and exit codes (clothsim/cli.py:26-165), its sweep CSV header
(bench.py:256-321) and FrameStats rows (io.py:29-74)."""

import csv

import pytest

from paper_2507_11794_b200 import cli, harness


def test_sweep_header_and_grid_rule_match_the_reference():
    assert harness.SWEEP_FIELDS == (
        "nodes_requested", "nx", "ny", "nodes", "springs", "cpu_mean_wall_ms", "cpu_mean_fps",
        "cpu_below_30fps", "gpu_mean_wall_ms", "gpu_mean_fps", "gpu_below_30fps",
        "cpu_over_gpu_ratio", "status", "reason")
    assert harness.grid_for_nodes(640000) == (800, 800)
    assert harness.grid_for_nodes(100000) == (316, 316)
    with pytest.raises(ValueError):
        harness.grid_for_nodes(3)
    row = harness.SweepRow(4096, 64, 64, 4096, 23938, gpu_mean_wall_ms=0.05, gpu_mean_fps=20000.0,
                           gpu_below_30fps=False)
    assert row.as_row() == ["4096", "64", "64", "4096", "23938", "", "", "", "0.050", "20000.00",
                            "no", "", "ok", ""]


def test_usage_errors_exit_2(capsys):
    assert cli.main(["--grid", "1x5"]) == cli.EXIT_USAGE
    assert cli.main(["--grid", "abc"]) == cli.EXIT_USAGE
    assert cli.main(["--sweep", "64,x"]) == cli.EXIT_USAGE
    assert cli.main(["--scene", "hanging", "--obstacle", "icosphere:1"]) == cli.EXIT_USAGE
    with pytest.raises(SystemExit) as e:
        cli.main(["--probe-limits", "--sweep", "64"])
    assert e.value.code == 2


def test_no_adapter_exits_3(monkeypatch, capsys):
    monkeypatch.setenv("CLOTHSIM_ADAPTER", "none")
    assert cli.main(["--grid", "8x8", "--frames", "2"]) == cli.EXIT_NO_ADAPTER
    assert cli.main(["--probe-limits"]) == cli.EXIT_NO_ADAPTER
    assert "no compute adapter" in capsys.readouterr().err


def test_probe_arithmetic_matches_the_engine_census():
    """probe_limits sizes grids with the same byte census Engine.layout
    checks against free device memory (engine.py)."""
    import numpy as np

    from paper_2507_11794_b200.engine import Layout  # noqa: F401  (the census owner)

    side = 800
    pitch_nodes = ((side + 31) // 32 * 32) * side
    want = 2 * 6 * pitch_nodes * 4 + 3 * pitch_nodes * 4 + 24 * pitch_nodes + 12 * 2 * (side - 1) ** 2
    assert harness._grid_engine_bytes(side) == want
    assert np.isclose(harness._grid_engine_bytes(4096) / 4096 ** 2, 108, rtol=0.01)


@pytest.mark.gpu
def test_single_run_writes_reference_stats_csv(tmp_path, capsys):
    out = tmp_path / "s.csv"
    rc = cli.main(["--scene", "drop", "--grid", "24x24", "--obstacle", "icosphere:2",
                   "--frames", "30", "--out", str(out), "--snapshot-every", "15"])
    assert rc == cli.EXIT_OK
    rows = list(csv.reader(open(out)))
    assert rows[0][:8] == ["frame", "wall_ms", "fps", "nodes", "springs", "obstacle_triangles",
                           "collision_hits", "backend"]
    assert len(rows) == 31 and rows[-1][0] == "29" and rows[1][7] == "cuda"
    assert len(list(tmp_path.glob("s_cuda_*.png"))) == 2
    assert "mean device" in capsys.readouterr().out


@pytest.mark.gpu
def test_sweep_and_probe(tmp_path, capsys):
    out = tmp_path / "sweep.csv"
    rc = cli.main(["--scene", "hanging", "--dt", "0.004", "--frames", "20",
                   "--sweep", "4096,65536,640000", "--out", str(out)])
    assert rc == cli.EXIT_OK
    rows = list(csv.reader(open(out)))
    assert tuple(rows[0]) == harness.SWEEP_FIELDS and len(rows) == 4
    assert [r[3] for r in rows[1:]] == ["4096", "65536", "640000"]
    assert all(r[12] == "ok" and float(r[9]) > 30 for r in rows[1:])
    assert cli.main(["--probe-limits"]) == cli.EXIT_OK
    text = capsys.readouterr().out
    assert "largest square cloth that fits" in text
    rep, _ = harness.probe_limits()
    assert rep.max_side > 4096 and rep.free_bytes > 0
