#!/bin/bash
O=gpurun_out/${1:-kpwr}
mkdir -p $O
for combo in "1 2 1" "1 1 2" "2 1 1" "1 4 4"; do
  set -- $combo
  OCLDEC_B200_KPW_FRONT=$1 OCLDEC_B200_KPW_LOWER=$2 OCLDEC_B200_KPW_EMIT=$3 \
    timeout 300 python tools/gpu_prof.py C4 100000 > $O/f$1_l$2_e$3.json 2>&1
  echo "f$1 l$2 e$3 $(python3 -c "import json;d=json.load(open('$O/f$1_l$2_e$3.json'));print(round(d['instr_per_s']/1e6,2),'M/s',{k:round(v) for k,v in d['ms'].items()})")"
done
NK=30000 bash tools/ncu_phases.sh $1/ncu
