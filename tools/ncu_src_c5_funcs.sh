#!/bin/bash
# Per-function summary of k_lower / k_front / k_emit on a C5 sample (source
# counters; summaries only travel back):  tools/ncu_src_c5_funcs.sh OUTDIR
O=gpurun_out/${1:-ncu_src_c5f}
mkdir -p $O
NK=${NK:-1500} bash tools/ncu_src_c5.sh ${1:-ncu_src_c5f}/raw > /dev/null 2>&1
for k in k_front k_lower k_emit; do
  python tools/ncu_funcs.py $O/raw/cs_$k.csv 30 > $O/funcs_c5_$k.txt 2>&1
done
/usr/local/cuda/bin/ncu -i $O/raw/c5.ncu-rep --page details --csv > $O/details_c5.csv 2>/dev/null
rm -rf $O/raw
ls -la $O
