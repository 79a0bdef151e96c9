"""Full-size oracle fixtures for BASELINE.json's configurations (test infrastructure).

Runs the CPU oracle (oracle/, the C++ restatement of the reference) at the configs' full sizes
and writes small .npz fixtures that `tests/test_fullsize_gpu.py` compares the device with on the
GPU box (where /root/reference and the hours of CPU time are not available):

  pca_<C>.npz   (C2, C3, C4, C5)  the PCA of every subdomain (reduction.hpp:89-109):
                p_j (bit-exact bar), the leading singular values σ_0..σ_{p_j+3}, one seeded
                probe per subdomain pushed through the kept projector (P_j·x_j, x_j ~ N(0,1)
                from default_rng(PROBE_SEED + j)), and for a few subdomains the whole kept
                basis or its orthogonal complement (whichever is smaller) for the exact
                projector 2-norm.
  run_<C>.npz   (C2, C4, AS-PCG to 1e-10)  run_single (runner.hpp:202-275): iterations,
                convergence, e_L2, e_L1n, final residual, both residual histories, the
                coefficients W and the approximation at the test points (the exact values are
                recomputed on the device bit-identically, so they are not stored).

The per-subdomain PCAs are independent, so `pca` mode runs them concurrently on all cores
(Oracle.set_option("parallel_pca", 1)); `run` mode is the oracle's run_single exactly as the
bench's CPU leg runs it (the reference's serial PCA loop). Timings and the core count go to
profiles/oracle_fullsize_r02.jsonl.

  ref_run_<C>.npz (C2, C4)  the same run_single on the reference itself (oracle/_ref: the unmodified
                headers on the Eigen-subset shim, the BASELINE objects built from its own types):
                p_j, iterations, errors, final residual, residual history.

usage: python tests/golden/make_fullsize.py pca C5 [C3 ...] | run C2 [C4] | refrun C2 [C4]
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

from oracle import Oracle, lib  # noqa: E402
from paper_2412_19207_b200 import configs  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "fullsize")
PROBE_SEED = 20250
N_SIGMA_EXTRA = 4


def subset(J: int) -> list[int]:
    return sorted({0, J // 3, J // 2 + 1, J - 1})


def pca_payload(o: Oracle, m: int) -> dict:
    J = int(o.geti("J")[0])
    pj = o.geti("p_j").astype(np.int32)
    sig_off = np.zeros(J + 1, dtype=np.int64)
    sig, probes = [], np.zeros((J, m))
    for j in range(J):
        s = o.getd("sigma", j)
        k = min(len(s), int(pj[j]) + N_SIGMA_EXTRA)
        sig.append(s[:k])
        sig_off[j + 1] = sig_off[j] + k
        V = o.getd("V", j).reshape(int(pj[j]), m).T
        x = np.random.default_rng(PROBE_SEED + j).standard_normal(m)
        probes[j] = V @ (V.T @ x)
    out = {"p_j": pj, "sigma": np.concatenate(sig), "sigma_off": sig_off, "probe_px": probes,
           "subset": np.array(subset(J), dtype=np.int32)}
    for j in subset(J):
        Vf = o.getd("V_full", j)
        k = Vf.size // m
        Vf = Vf.reshape(k, m).T
        p = int(pj[j])
        if p <= m - p:
            out[f"basis_{j}"] = Vf[:, :p]
            out[f"basis_kind_{j}"] = np.array(0)  # kept basis
        else:
            # complement of the kept subspace inside R^m: the discarded right vectors (k = min(rows, m)
            # of them) plus, when rows < m, the null space of S that the thin SVD leaves implicit
            comp = Vf[:, p:]
            if k < m:
                q, _ = np.linalg.qr(np.concatenate([Vf, np.random.default_rng(j).standard_normal((m, m - k))], 1))
                comp = np.concatenate([comp, q[:, k:]], 1)
            out[f"basis_{j}"] = comp
            out[f"basis_kind_{j}"] = np.array(1)  # orthogonal complement
    return out


def log(rec: dict):
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", "oracle_fullsize_r02.jsonl"), "a") as f:
        f.write(json.dumps(rec) + "\n")


def do_pca(name: str):
    cfg = configs.BASELINE[name]()
    Oracle.set_option("parallel_pca", 1)
    Oracle.set_option("keep_samples", 0)
    o = Oracle(threads=os.cpu_count() or 1)
    t0 = time.perf_counter()
    o.build_instance(cfg)
    t = time.perf_counter() - t0
    pay = pca_payload(o, cfg.m)
    os.makedirs(OUT, exist_ok=True)
    np.savez_compressed(os.path.join(OUT, f"pca_{name}.npz"), **pay)
    log({"mode": "pca", "config": name, "J": int(o.geti("J")[0]), "p": int(o.geti("p")[0]),
         "wall_s": t, "threads": lib().orc_max_threads(), "parallel_over_subdomains": True,
         "host": os.uname().nodename})
    print(name, "pca", f"{t:.1f}s", "p =", int(o.geti("p")[0]), flush=True)
    o.close()


def do_run(name: str):
    cfg = configs.aspcg(name)
    Oracle.set_option("parallel_pca", 0)
    Oracle.set_option("keep_samples", 0)
    o = Oracle(threads=os.cpu_count() or 1)
    t0 = time.perf_counter()
    s = o.run_single(cfg)
    t = time.perf_counter() - t0
    pay = pca_payload(o, cfg.m)
    pay.update({
        "iterations": np.array(s["iterations"]), "converged": np.array(s["converged"]),
        "e_l2": np.array(s["e_l2"]), "e_l1n": np.array(s["e_l1n"]), "final_residual": np.array(s["final_residual"]),
        "DoF": np.array(s["DoF"]), "N": np.array(s["N"]),
        "hist": o.getd("hist", 0), "true_hist": o.getd("true_hist", 0),
        "W": o.getd("W", 0), "approx": o.getd("approx"),
    })
    os.makedirs(OUT, exist_ok=True)
    np.savez_compressed(os.path.join(OUT, f"run_{name}.npz"), **pay)
    log({"mode": "run_single", "config": name, "solver": "AS-PCG", "rel_tol": cfg.rel_tol,
         "J": s["J"], "DoF": s["DoF"], "N": s["N"], "iterations": s["iterations"], "e_l2": s["e_l2"],
         "wall_s": t, "phases_s": {k: s[k] for k in ("t_assemble", "t_precond", "t_solve", "t_evaluate")},
         "threads": lib().orc_max_threads(), "host": os.uname().nodename,
         "note": "oracle run_single as the reference: serial PCA loop, OpenMP at the reference's sites, "
                 "LAPACK single-threaded"})
    print(name, "run", f"{t:.1f}s", {k: s[k] for k in ("iterations", "e_l2", "DoF")}, flush=True)
    o.close()


def do_refrun(name: str):
    import ref as refmod
    cfg = configs.aspcg(name)
    os.environ.setdefault("OMP_NUM_THREADS", str(os.cpu_count() or 1))
    r = refmod.Reference()
    t0 = time.perf_counter()
    s = r.run_baseline(cfg)
    t = time.perf_counter() - t0
    pay = {"p_j": r.geti("p_j").astype(np.int32), "iterations": np.array(s["iterations"]),
           "converged": np.array(s["converged"]), "e_l2": np.array(s["e_l2"]), "e_l1n": np.array(s["e_l1n"]),
           "final_residual": np.array(s["final_residual"]), "DoF": np.array(s["DoF"]), "N": np.array(s["N"]),
           "hist": r.getd("hist", 0)}
    os.makedirs(OUT, exist_ok=True)
    np.savez_compressed(os.path.join(OUT, f"ref_run_{name}.npz"), **pay)
    log({"mode": "reference run_single (oracle/_ref)", "config": name, "solver": "AS-PCG", "rel_tol": cfg.rel_tol,
         "J": s["J"], "DoF": s["DoF"], "N": s["N"], "iterations": s["iterations"], "e_l2": s["e_l2"], "wall_s": t,
         "phases_s": {k: s[k] for k in ("t_assemble", "t_precond", "t_solve")}, "threads": os.environ["OMP_NUM_THREADS"],
         "host": os.uname().nodename})
    print(name, "refrun", f"{t:.1f}s", {k: s[k] for k in ("iterations", "e_l2", "DoF")}, flush=True)
    r.close()


if __name__ == "__main__":
    mode, names = sys.argv[1], sys.argv[2:]
    for n in names:
        {"pca": do_pca, "run": do_run, "refrun": do_refrun}[mode](n)
