"""Convergence study (cmd_converge's split-EE column, cli.py:258-346) on the
GPU against the reference's own tables (tests/golden/converge.json); argument
checks on the CPU."""

import json
from pathlib import Path

import numpy as np
import pytest

from paper_2604_11558_b200.converge import convergence_study, relative_error
from paper_2604_11558_b200.models import model_spec

GOLD = json.loads((Path(__file__).resolve().parent / "golden" / "converge.json").read_text())
DIM_KEYS = ("n_rho", "n_theta", "n_phi", "n_z")


def _args(cfg):
    dims = {k: cfg[k] for k in DIM_KEYS if k in cfg}
    return model_spec(cfg["model"]), dims, cfg["tstar"], cfg["m_list"]


def test_relative_error_formula():
    ref = {"u": np.array([3.0, 4.0]), "v": np.array([1.0, 0.0])}
    got = {"u": np.array([3.0, 4.0]) + np.array([0.0, 5.0]), "v": np.array([1.0, 1.0])}
    assert relative_error(got, ref) == pytest.approx(np.sqrt(1.0 + 1.0))


@pytest.mark.parametrize("bad", [dict(m_list=[10, 5]), dict(m_list=[5, 10], m_ref=30), dict(m_list=[])])
def test_usage_errors(bad):
    spec, dims, t, _ = _args(GOLD[1]["cfg"])
    with pytest.raises(ValueError):
        convergence_study(spec, dims, t, bad.pop("m_list"), **bad)


@pytest.mark.gpu
@pytest.mark.parametrize("case", GOLD, ids=[c["cfg"]["model"] for c in GOLD])
def test_convergence_tables_match_reference(case):
    cfg = case["cfg"]
    spec, dims, t, m_list = _args(cfg)
    res = convergence_study(spec, dims, t, m_list, m_ref=cfg.get("m_ref"), seed=cfg["seed"])
    assert [e["m"] for e in res["table"]] == [e["m"] for e in case["table"]]
    for got, ref in zip(res["table"], case["table"]):
        assert got["err_split"] == pytest.approx(ref["err_split"], rel=1e-8)
    assert res["slope"] == pytest.approx(case["slope"], rel=1e-8, abs=1e-10)
