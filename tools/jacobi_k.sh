#!/bin/bash
# C2 PCA time with the stage-2 Jacobi cluster size forced to 2/4/8
for k in 2 4 8; do
  RDD_JACOBI_K=$k timeout 120 python tools/phase_stats.py C2 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('K=$k', d['families_ms']['syevj'], d['families_ms']['pca_total'])"
done
