"""Extract the reference's committed test artefacts into tests/golden/reference_artefacts.json.

Run in the build container (where /root/reference exists):  python tests/golden/make_golden.py
The artefacts are outputs of the reference's own Catch2 tests:
  proj/h_export.txt, proj/ata_export.txt        test_assembly.cpp:188-210
  proj/runner_out/{summary,residuals,aggregate}.csv  test_runner.cpp:91-125
  proj/runner_out_scaling/scaling.csv           test_runner.cpp:173-184
  proj/runner_out_sweep/sweep_tau.csv           test_runner.cpp:162-171
  proj/runner_out_spec/spectrum_*.csv           test_runner.cpp:139-160
  proj/schwarz_diag.csv                         test_schwarz.cpp:190-203
  proj/runner_out/config_echo.ini               test_runner.cpp:91-125 (config.hpp:232-260)
"""
import csv
import json
import os

REF = "/root/reference/proj"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_artefacts.json")


def rows(path):
    with open(os.path.join(REF, path)) as f:
        return list(csv.DictReader(f))


def main():
    g = {}
    lines = open(os.path.join(REF, "h_export.txt")).read().split("\n")
    r, c = map(int, lines[0].split())
    g["h_export"] = {"rows": r, "cols": c,
                     "triples": [[int(a), int(b), float(v)] for a, b, v in (l.split() for l in lines[1:] if l.strip())]}
    lines = open(os.path.join(REF, "ata_export.txt")).read().split("\n")
    g["ata_export"] = [[float(x) for x in l.split()] for l in lines[1:] if l.strip()]
    g["runner_summary"] = rows("runner_out/summary.csv")
    g["runner_residuals"] = rows("runner_out/residuals.csv")
    g["runner_aggregate"] = rows("runner_out/aggregate.csv")
    g["scaling"] = rows("runner_out_scaling/scaling.csv")
    g["sweep_tau"] = rows("runner_out_sweep/sweep_tau.csv")
    g["spectrum_normal"] = [float(r["real"]) for r in rows("runner_out_spec/spectrum_normal.csv")]
    g["spectrum_preconditioned"] = [float(r["real"]) for r in rows("runner_out_spec/spectrum_preconditioned.csv")]
    g["schwarz_diag"] = rows("schwarz_diag.csv")
    # config.hpp:232-260 config_echo of test_runner.cpp's small_config (runner_out/config_echo.ini)
    g["runner_config_echo"] = open(os.path.join(REF, "runner_out/config_echo.ini")).read()
    with open(OUT, "w") as f:
        json.dump(g, f, indent=0)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
