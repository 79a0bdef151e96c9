"""The reference's data formats either side of the solve path, on the device.

* ``parse_config_text`` / ``parse_config_file`` / ``config_echo`` — the flat sectioned key=value
  run description of config.hpp:23-262 (strict schema: unknown sections and keys are rejected with
  the reference's messages; errors are ValueError, the binding's std::invalid_argument).
* ``run`` — runner.hpp:296-330: one device pipeline per seed, then config_echo.ini, summary.csv,
  residuals.csv (first seed), aggregate.csv and, with dump_diagnostics, singular_values.csv
  (reduction.hpp:158-165), in the reference's column order and number formatting.
* ``spectrum_cmd`` / ``sweep_tau`` / ``scaling_cmd`` — runner.hpp:344-492 with the dense
  diagnostics on the device (``Solver.spectra``).

Every solve runs through librdd.so (``rdd.Solver``); there is no host fallback. The reference's
``override_caps`` stays a call argument (it is command-line only, config.hpp:61).
"""
from __future__ import annotations

import dataclasses
import math
import os
import re
import statistics
from typing import Optional

from . import abi as A

SCHEMA = {  # config.hpp:139-147
    "problem": {"name", "n", "ref_resolution"},
    "decomposition": {"counts", "delta"},
    "basis": {"m", "activation", "seed"},
    "points": {"collocation", "test"},
    "pca": {"tau", "matrix"},
    "solver": {"method", "preconditioner", "rel_tol", "max_iter", "gmres_restart"},
    "run": {"num_seeds", "out_dir", "dump_diagnostics"},
}
_SOLVERS = {"qr_direct": A.SOLVER_QR, "cg": A.SOLVER_CG, "cgs": A.SOLVER_CGS, "bicg": A.SOLVER_BICG,
            "gmres": A.SOLVER_GMRES}
_PRECONDS = {"none": None, "AS": "AS", "SAS": "SAS", "RAS": "RAS"}
_PRECOND_ID = {None: A.PRECOND_NONE, "AS": A.PRECOND_AS, "SAS": A.PRECOND_SAS, "RAS": A.PRECOND_RAS}
_PROBLEM_ID = {"example1": A.PROBLEM_EXAMPLE1, "example2": A.PROBLEM_EXAMPLE2, "example3": A.PROBLEM_EXAMPLE3}
K_SUMMARY_HEADER = "seed,problem,J,DoF,N,solver,precond,tau,iter,converged,e_l2,e_l1n,t_assemble,t_precond,t_solve"


@dataclasses.dataclass
class RunConfig:
    """config.hpp:23-70 RunConfig with the reference's defaults."""
    problem: str = "example1"
    n: int = 2
    ref_resolution: int = 2001
    counts: list = dataclasses.field(default_factory=lambda: [4, 4])
    delta: float = 2.0
    m: int = 16
    activation: str = "tanh"
    seed: int = 1000
    collocation: list = dataclasses.field(default_factory=lambda: [40, 40])
    test: list = dataclasses.field(default_factory=lambda: [350, 350])
    tau_on: bool = False
    tau: float = 0.0
    pca_matrix: str = "operator"
    solver: str = "gmres"
    preconditioner: Optional[str] = "AS"
    rel_tol: float = 1e-5
    max_iter: int = 0
    gmres_restart: int = 0
    num_seeds: int = 10
    out_dir: str = "out"
    dump_diagnostics: bool = False

    def tau_label(self) -> str:  # config.hpp:63-68 (ostream default precision)
        return _g(self.tau, 6) if self.tau_on else "off"

    def precond_label(self) -> str:
        return self.preconditioner or "none"

    def to_abi(self, seed: Optional[int] = None) -> A.Config:
        """The device-side description of the same run (geometry.hpp:109 decomposition, absolute τ)."""
        return A.make_config(
            _PROBLEM_ID[self.problem], list(self.counts), self.m, list(self.collocation), n=self.n,
            decomposition=A.DECOMP_REFERENCE, delta=self.delta, activation=0 if self.activation == "tanh" else 1,
            seed=self.seed if seed is None else seed, test=list(self.test),
            tau_mode=A.TAU_ABSOLUTE if self.tau_on else A.TAU_OFF, tau=self.tau,
            pca_matrix=A.PCA_OP_APPLIED if self.pca_matrix == "operator" else A.PCA_PSI,
            solver=_SOLVERS[self.solver], precond=_PRECOND_ID[self.preconditioner], rel_tol=self.rel_tol,
            max_iter=self.max_iter, gmres_restart=self.gmres_restart, ref_resolution=self.ref_resolution)


def _g(v: float, prec: int) -> str:
    """std::ostream << double with precision(prec), default floatfield (%g)."""
    if isinstance(v, float) and math.isnan(v):
        return "nan" if math.copysign(1.0, v) > 0 else "-nan"
    if isinstance(v, float) and math.isinf(v):
        return "inf" if v > 0 else "-inf"
    return format(v, f".{prec}g")


def _parse_int_list(value: str, key: str) -> list:  # config.hpp:79-89 (stops at the first non-integer)
    out = []
    for tok in value.replace(",", " ").split():
        try:
            out.append(int(tok))
        except ValueError:
            break
    if not out:
        raise ValueError(f"config: empty integer list for '{key}'")
    return out


def _parse_int(value: str, key: str) -> int:  # std::stoi, whole string consumed, int range
    if re.fullmatch(r"[+-]?[0-9]+", value) and -2**31 <= int(value) < 2**31:
        return int(value)
    raise ValueError(f"config: '{key}' expects an integer, got '{value}'")


def _parse_double(value: str, key: str) -> float:  # std::stod, whole string consumed
    try:
        if "_" in value:
            raise ValueError
        return float(value)
    except ValueError:
        raise ValueError(f"config: '{key}' expects a number, got '{value}'") from None


def _parse_on_off(value: str, key: str) -> bool:
    if value in ("on", "true"):
        return True
    if value in ("off", "false"):
        return False
    raise ValueError(f"config: '{key}' expects on/off, got '{value}'")


def parse_config_text(text: str) -> RunConfig:
    """config.hpp:138-228 parse_config_text."""
    cfg = RunConfig()
    section = ""
    for lineno, line in enumerate(text.splitlines(), start=1):
        line = line.split("#", 1)[0].strip(" \t\r\n")
        if not line:
            continue
        if line[0] == "[":
            if line[-1] != "]":
                raise ValueError(f"config line {lineno}: bad section")
            section = line[1:-1].strip(" \t\r\n")
            if section not in SCHEMA:
                raise ValueError(f"config: unknown section '{section}'")
            continue
        if "=" not in line:
            raise ValueError(f"config line {lineno}: expected key = value")
        key, value = (s.strip(" \t\r\n") for s in line.split("=", 1))
        if not section:
            raise ValueError(f"config: key '{key}' outside any section")
        if key not in SCHEMA[section]:
            raise ValueError(f"config: unknown key '{key}' in section [{section}]")
        if section == "problem":
            if key == "name":
                cfg.problem = value
            elif key == "n":
                cfg.n = _parse_int(value, key)
            else:
                cfg.ref_resolution = _parse_int(value, key)
        elif section == "decomposition":
            if key == "counts":
                cfg.counts = _parse_int_list(value, key)
            else:
                cfg.delta = _parse_double(value, key)
        elif section == "basis":
            if key == "m":
                cfg.m = _parse_int(value, key)
            elif key == "activation":
                if value not in ("tanh", "sin"):
                    raise ValueError("config: activation must be tanh or sin")
                cfg.activation = value
            else:
                cfg.seed = int(value)
        elif section == "points":
            if key == "collocation":
                cfg.collocation = _parse_int_list(value, key)
            else:
                cfg.test = _parse_int_list(value, key)
        elif section == "pca":
            if key == "matrix":
                if value not in ("operator", "psi"):
                    raise ValueError("config: pca matrix must be operator or psi")
                cfg.pca_matrix = value
            elif value == "off":
                cfg.tau_on, cfg.tau = False, 0.0
            else:
                cfg.tau_on, cfg.tau = True, _parse_double(value, key)
                if cfg.tau < 0.0:
                    raise ValueError("config: tau must be >= 0 or off")
        elif section == "solver":
            if key == "method":
                if value not in _SOLVERS:
                    raise ValueError(f"config: unknown solver '{value}'")
                cfg.solver = value
            elif key == "preconditioner":
                if value not in _PRECONDS:
                    raise ValueError(f"config: unknown preconditioner '{value}'")
                cfg.preconditioner = _PRECONDS[value]
            elif key == "rel_tol":
                cfg.rel_tol = _parse_double(value, key)
            elif key == "max_iter":
                cfg.max_iter = _parse_int(value, key)
            else:
                cfg.gmres_restart = _parse_int(value, key)
        elif section == "run":
            if key == "num_seeds":
                cfg.num_seeds = _parse_int(value, key)
            elif key == "out_dir":
                cfg.out_dir = value
            else:
                cfg.dump_diagnostics = _parse_on_off(value, key)
    if cfg.problem not in _PROBLEM_ID:
        raise ValueError(f"config: unknown problem '{cfg.problem}'")
    if not cfg.rel_tol > 0.0:
        raise ValueError("config: rel_tol must be positive")
    if cfg.num_seeds < 1:
        raise ValueError("config: num_seeds must be >= 1")
    if cfg.m < 1:
        raise ValueError("config: m must be >= 1")
    return cfg


def parse_config_file(path: str) -> RunConfig:
    try:
        with open(path) as f:
            text = f.read()
    except OSError:
        raise RuntimeError(f"cannot open config file {path}") from None
    return parse_config_text(text)


def config_echo(cfg: RunConfig) -> str:
    """config.hpp:232-260: canonical echo (precision 17), parseable by parse_config_text."""
    g = lambda v: _g(float(v), 17)  # noqa: E731
    return (f"[problem]\nname = {cfg.problem}\nn = {cfg.n}\nref_resolution = {cfg.ref_resolution}\n\n"
            f"[decomposition]\ncounts =" + "".join(f" {c}" for c in cfg.counts) + f"\ndelta = {g(cfg.delta)}\n\n"
            f"[basis]\nm = {cfg.m}\nactivation = {cfg.activation}\nseed = {cfg.seed}\n\n"
            "[points]\ncollocation =" + "".join(f" {c}" for c in cfg.collocation)
            + "\ntest =" + "".join(f" {c}" for c in cfg.test) + "\n\n"
            f"[pca]\ntau = {cfg.tau_label()}\nmatrix = {cfg.pca_matrix}\n\n"
            f"[solver]\nmethod = {cfg.solver}\npreconditioner = {cfg.precond_label()}\n"
            f"rel_tol = {g(cfg.rel_tol)}\nmax_iter = {cfg.max_iter}\ngmres_restart = {cfg.gmres_restart}\n\n"
            f"[run]\nnum_seeds = {cfg.num_seeds}\nout_dir = {cfg.out_dir}\n"
            f"dump_diagnostics = {'on' if cfg.dump_diagnostics else 'off'}\n")


def summary_row(cfg: RunConfig, s: dict) -> str:
    """runner.hpp:158-168 (precision 10)."""
    g = lambda v: _g(float(v), 10)  # noqa: E731
    precond = "none" if cfg.solver == "qr_direct" else cfg.precond_label()
    conv = 1 if cfg.solver == "qr_direct" or s["converged"] else 0
    return ",".join([str(s["seed"]), cfg.problem, str(s["J"]), str(s["DoF"]), str(s["N"]), cfg.solver, precond,
                     cfg.tau_label(), str(s["iterations"]), str(conv), g(s["e_l2"]), g(s["e_l1n"]),
                     g(s["t_assemble"]), g(s["t_precond"]), g(s["t_solve"])])


def _solver(solver=None):
    if solver is not None:
        return solver
    from . import rdd
    return rdd.Solver(0)


def run(cfg: RunConfig, solver=None) -> list:
    """runner.hpp:296-330 run: per-seed pipelines on the device and the reference's output files."""
    dev = _solver(solver)
    os.makedirs(cfg.out_dir, exist_ok=True)
    with open(os.path.join(cfg.out_dir, "config_echo.ini"), "w") as f:
        f.write(config_echo(cfg))
    rows = []
    with open(os.path.join(cfg.out_dir, "summary.csv"), "w") as summary:
        summary.write(K_SUMMARY_HEADER + "\n")
        for k in range(cfg.num_seeds):
            s = dev.run_single(cfg.to_abi(cfg.seed + k))
            summary.write(summary_row(cfg, s) + "\n")
            rows.append(s)
            if k == 0 and cfg.solver != "qr_direct":
                hist, true_hist = dev.getd("hist", 0), dev.getd("true_hist", 0)
                with open(os.path.join(cfg.out_dir, "residuals.csv"), "w") as f:  # runner.hpp:276-283
                    f.write("iter,preconditioned_residual,true_residual\n")
                    for i, (a, b) in enumerate(zip(hist, true_hist)):
                        f.write(f"{i},{_g(float(a), 12)},{_g(float(b), 12)}\n")
            if k == 0 and cfg.dump_diagnostics:
                with open(os.path.join(cfg.out_dir, "singular_values.csv"), "w") as f:  # reduction.hpp:158-165
                    f.write("subdomain,index,sigma\n")
                    if cfg.tau_on:
                        for j in range(s["J"]):
                            for i, v in enumerate(dev.getd("sigma", j)):
                                f.write(f"{j},{i},{_g(float(v), 6)}\n")
    with open(os.path.join(cfg.out_dir, "aggregate.csv"), "w") as agg:
        agg.write("metric,median,mean\n")
        for name, key in (("iter", "iterations"), ("e_l2", "e_l2"), ("e_l1n", "e_l1n")):
            vals = [float(r[key]) for r in rows]
            agg.write(f"{name},{_g(statistics.median(vals), 10)},{_g(statistics.fmean(vals), 10)}\n")
    return rows


def write_local_diagnostics_csv(path: str, solver) -> None:
    """schwarz.hpp:217-225: per-subdomain set size, local rank and condition estimate of the
    preconditioner built on the device context (default stream precision)."""
    ranks, conds = solver.geti("local_rank"), solver.getd("local_cond")
    with open(path, "w") as f:
        f.write("subdomain,size,rank,cond_estimate\n")
        for i, (r, k) in enumerate(zip(ranks, conds)):
            f.write(f"{i},{len(solver.geti('set', i))},{int(r)},{_g(float(k), 6)}\n")


def _precond_kind(cfg: RunConfig) -> int:
    return _PRECOND_ID[cfg.preconditioner or "AS"]  # value_or(AS), runner.hpp:354/385


def write_spectrum_csv(path: str, eigs) -> None:
    """runner.hpp:332-341: sorted by real part, precision 12."""
    eigs = sorted(eigs, key=lambda z: z.real)
    with open(path, "w") as f:
        f.write("index,real,imag\n")
        for i, z in enumerate(eigs):
            f.write(f"{i},{_g(float(z.real), 12)},{_g(float(z.imag), 12)}\n")


def spectrum_cmd(cfg: RunConfig, solver=None, override_caps: bool = False):
    """runner.hpp:344-362: spectra of HᵀH and M⁻¹HᵀH for the first seed."""
    dev = _solver(solver)
    os.makedirs(cfg.out_dir, exist_ok=True)
    cap = 1 << 20 if override_caps else 0
    dev.build_instance(cfg.to_abi(cfg.seed))
    dev.assemble(True)
    dev.build_preconditioner(_precond_kind(cfg))
    normal, pre, _, _ = dev.spectra(True, cap=cap)
    write_spectrum_csv(os.path.join(cfg.out_dir, "spectrum_normal.csv"), normal)
    write_spectrum_csv(os.path.join(cfg.out_dir, "spectrum_preconditioned.csv"), pre)
    return normal, pre


def sweep_tau(base: RunConfig, taus, solver=None, override_caps: bool = False) -> list:
    """runner.hpp:375-417: median-over-seeds DoF, condition numbers, iterations and error per τ."""
    dev = _solver(solver)
    os.makedirs(base.out_dir, exist_ok=True)
    cap = 1 << 20 if override_caps else 0
    rows = []
    for tau in taus:
        cfg = dataclasses.replace(base, tau_on=True, tau=float(tau))
        dof, cn, cp, iters, el2 = [], [], [], [], []
        for k in range(cfg.num_seeds):
            s = dev.run_single(cfg.to_abi(cfg.seed + k))
            dof.append(s["DoF"])
            iters.append(s["iterations"])
            el2.append(s["e_l2"])
            dev.build_instance(cfg.to_abi(cfg.seed + k))
            dev.assemble(True)
            dev.build_preconditioner(_precond_kind(cfg))
            _, _, c1, c2 = dev.spectra(True, cap=cap)
            cn.append(c1)
            cp.append(c2)
        med = statistics.median
        rows.append({"tau": float(tau), "DoF": med(dof), "cond_HtH": med(cn), "cond_precond": med(cp),
                     "iter": med(iters), "e_l2": med(el2)})
    with open(os.path.join(base.out_dir, "sweep_tau.csv"), "w") as f:
        f.write("tau,DoF,cond_HtH,cond_precond,iter,e_l2\n")
        for r in rows:
            f.write(",".join(_g(float(r[k]), 10) for k in ("tau", "DoF", "cond_HtH", "cond_precond", "iter", "e_l2"))
                    + "\n")
    return rows


def scaling_cmd(base: RunConfig, ns, solver=None, override_caps: bool = False) -> list:
    """runner.hpp:434-492: weak-scaling schedule, configured preconditioner vs none."""
    for n in ns:
        if n < 2:
            raise ValueError("scaling: n must be >= 2")
        if n > 4 and not override_caps:
            raise ValueError("scaling: n > 4 exceeds the desk-scale cap; pass --override-caps")
    dev = _solver(solver)
    os.makedirs(base.out_dir, exist_ok=True)
    rows = []
    for n in ns:
        l, npts = 1 << (n - 1), 5 * (1 << n)
        cfg = dataclasses.replace(base, problem="example1", n=n, counts=[l, l], collocation=[npts, npts], m=32,
                                  tau_on=True, tau=1e-3)
        for variant in (0, 1):
            vc, seeds = cfg, cfg.num_seeds
            if variant == 1:
                vc = dataclasses.replace(cfg, preconditioner=None)
                if vc.solver == "gmres" and vc.gmres_restart == 0:
                    vc = dataclasses.replace(vc, gmres_restart=30)
                seeds = min(seeds, 3)
            res = [dev.run_single(vc.to_abi(vc.seed + k)) for k in range(seeds)]
            med = lambda key: statistics.median([float(r[key]) for r in res])  # noqa: E731
            rows.append({"n": n, "J": res[-1]["J"], "precond": vc.precond_label(), "DoF": med("DoF"),
                         "N": res[-1]["N"], "iter": med("iterations"),
                         "converged_fraction": sum(1 for r in res if r["converged"]) / seeds,
                         "e_l1n": med("e_l1n"), "t_assemble": med("t_assemble"), "t_precond": med("t_precond"),
                         "t_solve": med("t_solve")})
    with open(os.path.join(base.out_dir, "scaling.csv"), "w") as f:
        f.write("n,J,precond,DoF,N,iter,converged_fraction,e_l1n,t_assemble,t_precond,t_solve\n")
        for r in rows:
            f.write(f"{r['n']},{r['J']},{r['precond']}," + ",".join(
                _g(float(r[k]), 10) for k in ("DoF", "N", "iter", "converged_fraction", "e_l1n", "t_assemble",
                                              "t_precond", "t_solve")) + "\n")
    return rows
