"""Diagnostic sweep (no asserts): per-stage GPU-vs-oracle deltas for the parity cases."""
import sys, os, time, traceback
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]
import numpy as np
from oracle import Oracle
from paper_2412_19207_b200 import rdd, abi as A
import test_parity_gpu as T

dev = rdd.Solver(0)
orc = Oracle()
names = sys.argv[1:] or list(T.CASES)
for name in names:
    cfg = T.CASES[name]
    print(f"=== {name}", flush=True)
    try:
        t = time.time(); dev.build_instance(cfg); t1 = time.time() - t
        orc.build_instance(cfg)
        J = int(orc.geti("J")[0])
        rows_ok = all(np.array_equal(dev.geti("rows", j), orc.geti("rows", j)) for j in range(J))
        pd, po = dev.geti("p_j"), orc.geti("p_j")
        print(f" build {t1:.3f}s rows_exact={rows_ok} p_dev={pd.tolist()} p_orc={po.tolist()}")
        if cfg.tau_mode != A.TAU_OFF:
            worst = 0.0; sw = 0.0
            for j in range(J):
                pj = int(po[j]); m = cfg.m
                if pd[j] != po[j]:
                    continue
                Vd = dev.getd("V", j).reshape(pj, m).T; Vo = orc.getd("V", j).reshape(pj, m).T
                worst = max(worst, np.linalg.norm(Vd @ Vd.T - Vo @ Vo.T, 2))
                sd, so = dev.getd("sigma", j), orc.getd("sigma", j)
                thr = cfg.tau * so[0] if cfg.tau_mode == A.TAU_RELATIVE else cfg.tau
                big = so > max(1e-8 * so[0], 0.2 * thr)
                sw = max(sw, np.max(np.abs(sd[big] - so[big]) / so[big]))
            print(f" projector max {worst:.2e}  sigma rel max {sw:.2e}")
        eq = cfg.precond >= 0
        dev.assemble(eq); orc.assemble(eq)
        hd = max(np.linalg.norm(dev.block(j) - orc.block(j)) / max(1e-300, np.linalg.norm(orc.block(j))) for j in range(J))
        Fd, Fo = dev.getd("F"), orc.getd("F")
        print(f" H rel max {hd:.2e}  F max abs {np.abs(Fd-Fo).max():.2e} (|F| {np.abs(Fo).max():.2e})  scales rel {np.max(np.abs(dev.getd('scales')-orc.getd('scales'))/orc.getd('scales')):.2e}")
        rng = np.random.default_rng(3)
        p, N = int(orc.geti("p")[0]), int(orc.geti("N")[0])
        w, r = rng.standard_normal(p), rng.standard_normal(N)
        yo, yd = orc.matvec(w), dev.matvec(w)
        to, td = orc.matvec_transpose(r), dev.matvec_transpose(r)
        print(f" matvec rel {np.linalg.norm(yd-yo)/np.linalg.norm(yo):.2e}  matvec_t rel {np.linalg.norm(td-to)/np.linalg.norm(to):.2e}")
        if cfg.precond >= 0:
            dev.build_preconditioner(cfg.precond); orc.build_preconditioner(cfg.precond)
            Ad, Ao = dev.getd("nb_dense"), orc.getd("nb_dense")
            print(f" nb pairs equal {np.array_equal(dev.geti('nb_pairs'), orc.geti('nb_pairs'))}  nb rel {np.linalg.norm(Ad-Ao)/np.linalg.norm(Ao):.2e}")
            print(f" ranks dev {dev.geti('local_rank').tolist()} orc {orc.geti('local_rank').tolist()}")
            v = rng.standard_normal(p)
            for tr in (False, True):
                zo, zd = orc.precond_apply(v, tr), dev.precond_apply(v, tr)
                print(f" precond(tr={tr}) rel {np.linalg.norm(zd-zo)/np.linalg.norm(zo):.2e}")
        c2 = A.Config.from_buffer_copy(cfg)
        if c2.precond < 0: c2.precond = A.PRECOND_AS
        t = time.time(); sd = dev.run_single(c2); t2 = time.time() - t
        so = orc.run_single(c2)
        print(f" run dev it={sd['iterations']} conv={sd['converged']} e_l2={sd['e_l2']:.10g} ({t2:.3f}s)  orc it={so['iterations']} conv={so['converged']} e_l2={so['e_l2']:.10g}")
    except Exception:
        traceback.print_exc()
