"""Host logic of the reference drivers (runner.hpp:276-492) without a GPU: a stand-in solver
returns fixed summaries and exports, and the files must come out in the reference's layout,
column order, aggregation (median/mean) and number formatting."""
import csv
import os

import numpy as np
import pytest

from paper_2412_19207_b200 import frontend as F

from test_frontend import small_config


class FakeSolver:
    """Deterministic stand-in for rdd.Solver: iterations and errors depend on the seed."""

    def __init__(self):
        self.calls = []
        self.kind = None

    def run_single(self, cfg, seed=None):
        s = int(cfg.seed)
        self.calls.append((s, int(cfg.precond), int(cfg.gmres_restart), int(cfg.counts[0]), int(cfg.colloc[0])))
        none = cfg.precond < 0
        return {"seed": s, "J": int(cfg.counts[0] * cfg.counts[1]), "DoF": 80 + (s % 3), "N": int(cfg.colloc[0] ** 2),
                "p": 80, "iterations": (300 if none else 1 + (s % 2)), "converged": 0 if none else 1,
                "breakdown": 0, "e_l2": 0.01 * (1 + (s % 5)), "e_l1n": 0.005 * (1 + (s % 4)),
                "t_assemble": 0.001, "t_precond": 0.0005, "t_solve": 0.0002, "t_evaluate": 0.0001,
                "t_pca": 0.0008, "final_residual": 1e-9}

    def getd(self, what, index=0):
        if what == "hist":
            return np.array([1.0, 6.19860877913e-09])
        if what == "true_hist":
            return np.array([1.0, 2.94228937369e-10])
        if what == "sigma":
            return np.array([3.0, 1.0, 1e-5])
        if what == "local_cond":
            return np.array([8.590612345e6, 1.5, 2.25, 3.0])
        raise KeyError(what)

    def geti(self, what, index=0):
        if what == "local_rank":
            return np.array([24, 24, 23, 24])
        if what == "set":
            return np.arange(24)
        if what == "p":
            return np.array([32])
        raise KeyError(what)

    def build_instance(self, cfg, seed=None):
        self.calls.append(("build", int(cfg.seed)))
        return self

    def assemble(self, eq=True):
        return self

    def build_preconditioner(self, kind):
        self.kind = kind
        return self

    def spectra(self, with_precond=True, cap=0):
        normal = np.array([4.0, 1.0, 2.0, 3.0]) + 0j
        pre = np.array([2.0 + 1j, 1.0, 2.0 - 1j, 0.5]) if with_precond else None
        return normal, pre, 1.2345678901e6, 1.0


def _rows(path):
    with open(path) as f:
        return list(csv.DictReader(f))


def test_run_files(tmp_path):
    out = str(tmp_path / "o")
    cfg = F.parse_config_text(small_config(out) + "[run]\nnum_seeds = 3\n")
    dev = FakeSolver()
    rows = F.run(cfg, solver=dev)
    assert [c[0] for c in dev.calls] == [77, 78, 79]
    assert open(os.path.join(out, "config_echo.ini")).read() == F.config_echo(cfg)
    s = _rows(os.path.join(out, "summary.csv"))
    assert list(s[0].keys()) == F.K_SUMMARY_HEADER.split(",")
    assert [r["seed"] for r in s] == ["77", "78", "79"]
    assert s[0]["tau"] == "off" and s[0]["precond"] == "AS" and s[0]["solver"] == "gmres"
    assert s[0]["e_l2"] == "0.03" and s[0]["t_solve"] == "0.0002"
    agg = {r["metric"]: r for r in _rows(os.path.join(out, "aggregate.csv"))}
    its = [r["iterations"] for r in rows]
    assert float(agg["iter"]["median"]) == np.median(its) and float(agg["iter"]["mean"]) == pytest.approx(np.mean(its))
    assert float(agg["e_l2"]["median"]) == pytest.approx(np.median([r["e_l2"] for r in rows]))
    res = open(os.path.join(out, "residuals.csv")).read().splitlines()
    assert res == ["iter,preconditioned_residual,true_residual", "0,1,1", "1,6.19860877913e-09,2.94228937369e-10"]


def test_singular_values_dump(tmp_path):
    out = str(tmp_path / "sv")
    cfg = F.parse_config_text(small_config(out).replace("tau = off", "tau = 1e-3")
                              + "[run]\nnum_seeds = 1\ndump_diagnostics = on\n")
    F.run(cfg, solver=FakeSolver())
    lines = open(os.path.join(out, "singular_values.csv")).read().splitlines()
    assert lines[0] == "subdomain,index,sigma"
    assert lines[1:4] == ["0,0,3", "0,1,1", "0,2,1e-05"]  # reduction.hpp:158-165, default precision
    assert len(lines) == 1 + 4 * 3


def test_spectrum_csv_sorted_by_real_part(tmp_path):
    out = str(tmp_path / "spec")
    cfg = F.parse_config_text(small_config(out))
    F.spectrum_cmd(cfg, solver=FakeSolver())
    pre = open(os.path.join(out, "spectrum_preconditioned.csv")).read().splitlines()
    assert pre[0] == "index,real,imag"
    assert [float(l.split(",")[1]) for l in pre[1:]] == [0.5, 1.0, 2.0, 2.0]
    normal = _rows(os.path.join(out, "spectrum_normal.csv"))
    assert [r["real"] for r in normal] == ["1", "2", "3", "4"] and all(r["imag"] == "0" for r in normal)


def test_sweep_tau_medians(tmp_path):
    out = str(tmp_path / "sweep")
    cfg = F.parse_config_text(small_config(out))
    rows = F.sweep_tau(cfg, [1e-4, 1e-2], solver=FakeSolver())
    got = _rows(os.path.join(out, "sweep_tau.csv"))
    assert list(got[0].keys()) == ["tau", "DoF", "cond_HtH", "cond_precond", "iter", "e_l2"]
    assert [r["tau"] for r in got] == ["0.0001", "0.01"]
    assert got[0]["cond_HtH"] == "1234567.89" and got[0]["cond_precond"] == "1"
    assert float(got[0]["DoF"]) == rows[0]["DoF"] == np.median([80 + (77 % 3), 80 + (78 % 3)])


def test_scaling_schedule(tmp_path):
    out = str(tmp_path / "scaling")
    cfg = F.parse_config_text(small_config(out) + "[run]\nnum_seeds = 5\n")
    dev = FakeSolver()
    rows = F.scaling_cmd(cfg, [2, 3], solver=dev)
    # runner.hpp:443-454: l = 2^(n-1), (5·2^n)² points, m = 32, τ = 1e-3; preconditioned rows on the
    # configured seeds, unpreconditioned GMRES(30) rows on at most 3 seeds
    assert [r["precond"] for r in rows] == ["AS", "none", "AS", "none"]
    runs = [c for c in dev.calls if c[0] != "build"]
    assert sum(1 for c in runs if c[3] == 2 and c[1] >= 0) == 5 and sum(1 for c in runs if c[3] == 2 and c[1] < 0) == 3
    assert all(c[2] == 30 for c in runs if c[1] < 0)
    assert {c[4] for c in runs if c[3] == 2} == {20} and {c[4] for c in runs if c[3] == 4} == {40}
    got = _rows(os.path.join(out, "scaling.csv"))
    assert list(got[0].keys()) == ["n", "J", "precond", "DoF", "N", "iter", "converged_fraction", "e_l1n", "t_assemble",
                                   "t_precond", "t_solve"]
    assert got[1]["converged_fraction"] == "0" and got[0]["converged_fraction"] == "1"


def test_local_diagnostics_csv(tmp_path):
    path = str(tmp_path / "d.csv")
    F.write_local_diagnostics_csv(path, FakeSolver())
    assert open(path).read().splitlines() == ["subdomain,size,rank,cond_estimate", "0,24,24,8.59061e+06",
                                              "1,24,24,1.5", "2,24,23,2.25", "3,24,24,3"]
