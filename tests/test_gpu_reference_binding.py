"""curvipat's own CLI driving the B200 engine through the Option-B binding
(``interop.run_simulation``), against the same CLI on the reference's CPU
path -- the unmodified reference, pip-installed into the git-ignored
``baseline/_ref`` (it travels to the GPU box with the snapshot; the tests
skip when it is absent and never read /root/reference).

- ``cmd_run`` writes the same snapshot CSVs and time series (within the
  north_star fp64 tolerance) whether run_simulation is the reference's or the
  engine's;
- a diverging run exits 3 from both, naming the same step, with the partial
  outputs kept;
- the reference's own build_system output runs through the engine with no
  manual descriptor (the closure is recognised).
"""

from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def cli():
    from oracle import ref_configs

    try:
        ref_configs.load_curvipat()  # baseline/_ref only
    except ImportError:
        pytest.skip("reference not installed into baseline/_ref")
    import curvipat.cli as cli

    return cli


def _snapshot(path):
    """The numeric rows of a snapshot / time-series CSV (comment lines and the
    column header skipped)."""
    rows = [ln for ln in Path(path).read_text().splitlines() if ln and not ln.startswith("#")]
    return np.array([[float(x) for x in ln.split(",")] for ln in rows[1:]])


def _run(cli, monkeypatch, engine, argv, out):
    from paper_2604_11558_b200 import interop

    with monkeypatch.context() as mp:
        if engine:
            mp.setattr(cli, "run_simulation", interop.run_simulation)
        return cli.main(argv + ["--out", str(out)])


@pytest.mark.parametrize("model,dims,m,tstar", [
    ("bvam_disk", ["--n-rho", "12", "--n-theta", "16"], 40, 0.4),
    ("schnakenberg_anomalous_disk", ["--n-rho", "16", "--n-theta", "32"], 40, 0.004),
    ("dib_sphere", ["--n-theta", "16", "--n-phi", "12"], 40, 0.04),
    ("bulk_surface_schnakenberg_ball", ["--n-rho", "6", "--n-theta", "8", "--n-phi", "6"], 20, 0.002),
])
def test_cmd_run_outputs_match_reference(cli, monkeypatch, tmp_path, model, dims, m, tstar):
    argv = ["run", "--model", model, *dims, "--m", str(m), "--tstar", str(tstar), "--snapshots", "10"]
    assert _run(cli, monkeypatch, False, argv, tmp_path / "cpu") == 0
    assert _run(cli, monkeypatch, True, argv, tmp_path / "gpu") == 0
    cpu_files = sorted(p.name for p in (tmp_path / "cpu").iterdir())
    assert cpu_files == sorted(p.name for p in (tmp_path / "gpu").iterdir())
    for name in cpu_files:
        a, b = _snapshot(tmp_path / "cpu" / name), _snapshot(tmp_path / "gpu" / name)
        assert a.shape == b.shape, name
        assert np.array_equal(a[:, :-1 if name != "timeseries.csv" else 1], b[:, :-1 if name != "timeseries.csv"
                                                                              else 1]), name  # indices, grid, t
        # north_star's tolerances: the step-0 snapshot is the initial state
        # itself, later snapshots (steps 10..40) get the <= 1e-8 bound of 100 steps
        tol = 0.0 if name.endswith("_0000000.csv") else 1e-8
        for col in range(a.shape[1] - 1 if name != "timeseries.csv" else 1, a.shape[1]):
            assert np.max(np.abs(a[:, col] - b[:, col])) <= tol * max(np.max(np.abs(a[:, col])), 1e-300), name


def test_divergence_exit_code_and_step_match_reference(cli, monkeypatch, tmp_path, capsys):
    argv = ["run", "--model", "schnakenberg_anomalous_disk", "--n-rho", "12", "--n-theta", "16", "--m", "40",
            "--tstar", "0.04", "--snapshots", "10", "--set", "params.alpha1=1e7"]
    assert _run(cli, monkeypatch, False, argv, tmp_path / "cpu") == 3
    err_cpu = capsys.readouterr().err
    assert _run(cli, monkeypatch, True, argv, tmp_path / "gpu") == 3
    err_gpu = capsys.readouterr().err
    assert "DIVERGED at step" in err_cpu and err_cpu == err_gpu
    assert sorted(p.name for p in (tmp_path / "gpu").iterdir()) == \
        sorted(p.name for p in (tmp_path / "cpu").iterdir())


def test_reference_built_system_runs_on_engine(cli):
    import curvipat.integrators as ri
    import curvipat.models as rm

    from paper_2604_11558_b200 import interop

    sysm = rm.build_system("schnakenberg_anomalous_disk", {"n_rho": 16, "n_theta": 32}, 5)
    ref = ri.run_simulation(sysm, 30, 0.003)
    got = interop.run_simulation(sysm, 30, 0.003)
    for c in sysm.components:
        a, b = got.fields[c.name] + c.lift, ref.fields[c.name] + c.lift
        assert np.max(np.abs(a - b)) / np.max(np.abs(b)) <= 1e-10
    with pytest.raises(ri.DivergenceError):
        interop.run_simulation(rm.build_system(rm.model_spec("schnakenberg_anomalous_disk", {"alpha1": 1e7}),
                                               {"n_rho": 12, "n_theta": 16}, 1), 40, 0.04)
