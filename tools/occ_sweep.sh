#!/bin/bash
# Occupancy sweep (blocks of 4 warps per SM) for the lower / emit phases on a C4 sample.
O=gpurun_out/${1:-occ}
mkdir -p $O
for occ in 0 1 2 4; do
  OCLDEC_B200_OCC_LOWER=$occ OCLDEC_B200_OCC_EMIT=$occ OCLDEC_B200_OCC_FRONT=$occ timeout 300 python tools/gpu_prof.py C4 100000 > $O/occ$occ.json 2>&1
  echo "occ $occ $(python3 -c "import json;d=json.load(open('$O/occ$occ.json'));print(round(d['instr_per_s']/1e6,2),'M/s', d['phase_share'])")"
done
