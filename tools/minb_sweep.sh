#!/bin/bash
# Register-cap (min blocks per SM) variants of the phase kernels on a C4 sample.
O=gpurun_out/${1:-minb}
mkdir -p $O
for v in "" _minb14 _minb16; do
  OCLDEC_B200_LIB=$PWD/paper_2107_07809_b200/libocldec_b200$v.so timeout 300 python tools/gpu_prof.py C4 100000 > $O/c4$v.json 2>&1
  echo "$v $(python3 -c "import json;d=json.load(open('$O/c4$v.json'));print(round(d['instr_per_s']/1e6,2),'M/s',{k:round(v) for k,v in d['ms'].items()})")"
done
