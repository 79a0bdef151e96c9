"""Measured device-vs-oracle deviations for every parity case of tests/test_parity_gpu.py (the
tests assert bars; this records how far inside them the device lands) -> JSON lines.

    python tools/parity_report.py > profiles/parity_r02.jsonl
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle import Oracle  # noqa: E402
from paper_2412_19207_b200 import abi as A, rdd  # noqa: E402
from test_parity_gpu import CASES  # noqa: E402


def rel(a, b):
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / nb) if nb > 0 else float(np.linalg.norm(a - b))


def main():
    dev, orc = rdd.Solver(0), Oracle()
    for name, cfg0 in CASES.items():
        cfg = A.Config.from_buffer_copy(cfg0)
        out = {"case": name}
        dev.build_instance(cfg)
        orc.build_instance(cfg)
        J = int(orc.geti("J")[0])
        out["points_bitexact"] = bool(np.array_equal(dev.getd("points"), orc.getd("points")))
        out["rows_bitexact"] = all(np.array_equal(dev.geti("rows", j), orc.geti("rows", j)) for j in range(J))
        out["pca_ranks_bitexact"] = bool(np.array_equal(dev.geti("p_j"), orc.geti("p_j")))
        if cfg.tau_mode != A.TAU_OFF and out["pca_ranks_bitexact"]:
            m, pj = cfg.m, orc.geti("p_j")
            proj = 0.0
            for j in range(J):
                Vd = dev.getd("V", j).reshape(pj[j], m).T
                Vo = orc.getd("V", j).reshape(pj[j], m).T
                proj = max(proj, float(np.linalg.norm(Vd @ Vd.T - Vo @ Vo.T, 2)))
            out["pca_projector_diff_max"] = proj
        eq = cfg.precond >= 0
        dev.assemble(eq)
        orc.assemble(eq)
        out["H_rel_max"] = max(rel(dev.block(j), orc.block(j)) for j in range(J))
        rng = np.random.default_rng(3)
        p, N = int(orc.geti("p")[0]), int(orc.geti("N")[0])
        w = rng.standard_normal(p)
        out["normal_operator_rel"] = rel(dev.normal_apply(w), orc.matvec_transpose(orc.matvec(w)))
        if cfg.precond >= 0:
            dev.build_preconditioner(cfg.precond)
            orc.build_preconditioner(cfg.precond)
            out["local_ranks_bitexact"] = bool(np.array_equal(dev.geti("local_rank"), orc.geti("local_rank")))
            v = rng.standard_normal(p)
            out["precond_apply_rel"] = rel(dev.precond_apply(v), orc.precond_apply(v))
            out["local_cond_max"] = float(orc.getd("local_cond").max())
        run = A.Config.from_buffer_copy(cfg0)
        if run.precond < 0:
            run.precond = A.PRECOND_AS
        sd, so = dev.run_single(run), orc.run_single(run)
        out.update({"iterations_dev": sd["iterations"], "iterations_oracle": so["iterations"], "rel_tol": run.rel_tol})
        # the e_L2 bars are checked at rel_tol 1e-10 (tests/test_parity_gpu.py::test_run_single)
        run.rel_tol = 1e-10
        so = orc.run_single(run)
        uo = orc.getd("approx")
        sd = dev.run_single(run)
        ud, ue = dev.getd("approx"), dev.getd("exact")
        out.update({"iterations_dev_1e-10": sd["iterations"], "iterations_oracle_1e-10": so["iterations"],
                    "e_l2_dev": sd["e_l2"], "e_l2_oracle": so["e_l2"], "e_l2_abs_diff": abs(sd["e_l2"] - so["e_l2"]),
                    "e_l2_rel_diff": abs(sd["e_l2"] - so["e_l2"]) / so["e_l2"],
                    "u_rel_diff": float(np.linalg.norm(ud - uo) / np.linalg.norm(ue)),
                    "final_residual_dev": sd["final_residual"], "final_residual_oracle": so["final_residual"]})
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
