#!/bin/bash
O=gpurun_out/${1:-grp}
mkdir -p $O
for g in 1 2; do
  OCLDEC_B200_GROUP=$g timeout 300 python tools/gpu_prof.py C4 100000 > $O/g$g.json 2>&1
  echo "group=$g $(python3 -c "import json;d=json.load(open('$O/g$g.json'));print(round(d['instr_per_s']/1e6,2),'M/s',{k:round(v) for k,v in d['ms'].items()})")"
done
