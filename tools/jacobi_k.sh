#!/bin/bash
# C2 PCA time with the stage-2 Jacobi cluster size forced to 2/4/8
for k in 2 4 8; do
  RDD_JACOBI_K=$k timeout 120 python tools/phase_stats.py C2 > /tmp/jk.json 2> /tmp/jk.err || tail -5 /tmp/jk.err
  python -c "import json,sys; d=json.load(open('/tmp/jk.json')); print('K=$k', d['families_ms']['syevj'], d['families_ms']['pca_total'], d['families_ms']['schwarz_build'])"
done
