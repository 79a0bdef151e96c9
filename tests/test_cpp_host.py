"""The C++ host interface (include/rannddm_gpu.hpp) and its driver (examples/rdd_run.cpp): the
header compiles standalone; the driver reports the reference's exception classes; on a GPU its
summary rows equal the Python binding's run_single on the same config (same library, bit-identical
reruns)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "examples", "rdd_run")


def _build():
    subprocess.run(["make", "-C", os.path.join(ROOT, "paper_2412_19207_b200", "csrc"), "-s"], check=True,
                   capture_output=True)
    assert os.path.exists(EXE)


def test_header_compiles_standalone(tmp_path):
    src = tmp_path / "h.cpp"
    src.write_text('#include "rannddm_gpu.hpp"\nint main() { auto c = rannddm::gpu::baseline_config("C2");'
                   ' return c.m == 300 && c.counts[0] == 16 && c.colloc[1] == 960 ? 0 : 1; }\n')
    exe = tmp_path / "h"
    subprocess.run(["g++", "-std=c++17", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
                    str(src), "-o", str(exe)], check=True)
    assert subprocess.run([str(exe)]).returncode == 0


def test_driver_errors_map_to_reference_exceptions():
    _build()
    r = subprocess.run([EXE, "C9"], capture_output=True, text=True)
    assert r.returncode == 1 and "invalid_argument: unknown config 'C9'" in r.stderr
    r = subprocess.run([EXE, "C1", "--solver", "lsqr"], capture_output=True, text=True)
    assert r.returncode == 1 and "invalid_argument: unknown solver" in r.stderr
    r = subprocess.run([EXE], capture_output=True, text=True)
    assert r.returncode == 2 and "usage" in r.stderr


def test_driver_without_device_fails_loudly():
    _build()
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is visible")
    except ImportError:
        pass
    r = subprocess.run([EXE, "C1"], capture_output=True, text=True)
    assert r.returncode == 1 and "rdd_create" in r.stderr


def _rows(out):
    lines = out.strip().splitlines()
    hdr = lines[0].split(",")
    return [dict(zip(hdr, ln.split(","))) for ln in lines[1:]]


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["C1", "C5s"])
def test_driver_matches_python_binding(name):
    from paper_2412_19207_b200 import configs, rdd
    _build()
    r = subprocess.run([EXE, name, "--reps", "2", "--resident"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    rows = _rows(r.stdout)
    assert len(rows) == 2
    cfg = configs.c1() if name == "C1" else configs.c5(counts=(2, 2, 2))
    s = rdd.Solver(0)
    ref = s.run_single(cfg)
    for row in rows:
        assert int(row["J"]) == ref["J"] and int(row["DoF"]) == ref["DoF"] and int(row["N"]) == ref["N"]
        assert int(row["iter"]) == ref["iterations"] and int(row["converged"]) == 1
        assert float(row["e_l2"]) == pytest.approx(ref["e_l2"], rel=1e-9)
    s.close()
