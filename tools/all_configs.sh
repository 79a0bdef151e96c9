#!/bin/bash
# One resident rerun per BASELINE config (and the variants the configs name); JSON lines to stdout.
run() { timeout 300 python tools/run_named.py "$@" 2>/dev/null | tail -1; }
run C1
run C2
run C3 "" "" solver=1 precond=0
run C3 "" "" max_iter=500
run C4 "" "" solver=1 precond=0
run C4 "" "" max_iter=2000
run C5
run C5 2,2,2 20
