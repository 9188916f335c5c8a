#!/bin/bash
# Source-level ncu capture of k_semcheck on one fuel-exhausting kernel
# (one warp, ~1M interpreted steps per lane):  tools/ncu_sem_one.sh OUTDIR
O=gpurun_out/${1:-ncu_sem_one}
mkdir -p $O
timeout 900 /usr/local/cuda/bin/ncu --section SourceCounters --section WarpStateStats --section LaunchStats \
  --section InstructionStats --clock-control none --import-source on -k regex:k_semcheck -c 1 -o $O/sem \
  python tools/sem_one.py > $O/ncu.log 2>&1
/usr/local/cuda/bin/ncu -i $O/sem.ncu-rep --page source --csv --print-source cuda > $O/src_k_semcheck.csv 2>/dev/null
/usr/local/cuda/bin/ncu -i $O/sem.ncu-rep --page source --csv --print-source sass > $O/sass_k_semcheck.csv 2>/dev/null
/usr/local/cuda/bin/ncu -i $O/sem.ncu-rep --page details --csv > $O/details.csv 2>/dev/null
rm -f $O/sem.ncu-rep
ls -la $O
