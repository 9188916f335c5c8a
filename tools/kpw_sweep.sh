#!/bin/bash
# Sweep kernels-per-warp for k_decompile on C2/C3/C4 samples.
O=gpurun_out/${1:-kpw}
mkdir -p $O
for k in ${KPWS:-1 2 4 32}; do
  for c in "C4 100000" "C2 10000" "C3 10000"; do
    set -- $c
    OCLDEC_B200_KPW=$k timeout 300 python tools/gpu_prof.py $1 $2 > $O/kpw${k}_$1.json 2>&1
  done
done
grep -h instr_per_s $O/*.json | python3 -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['cfg'], d['kernels'], round(d['instr_per_s']/1e6,2), 'M/s', d['ms'])
"
