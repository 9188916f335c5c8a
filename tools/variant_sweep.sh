#!/bin/bash
# Compares library variants (paper_2107_07809_b200/libocldec_b200*.so) on a C4 sample.
O=gpurun_out/${1:-variants}
mkdir -p $O
for f in paper_2107_07809_b200/libocldec_b200*.so; do
  v=$(basename $f .so)
  OCLDEC_B200_LIB=$PWD/$f timeout 300 python tools/gpu_prof.py C4 ${NK:-100000} > $O/$v.json 2>&1
  echo "$v $(python3 -c "import json;d=json.load(open('$O/$v.json'));print(round(d['instr_per_s']/1e6,2),'M/s',{k:round(v) for k,v in d['ms'].items()})")"
done
