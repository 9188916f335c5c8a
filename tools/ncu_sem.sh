#!/bin/bash
# Source-level ncu capture of one k_semcheck launch (the batched semantic
# check) on a C4 sample:  tools/ncu_sem.sh OUTDIR
O=gpurun_out/${1:-ncu_sem}
mkdir -p $O
timeout 1500 /usr/local/cuda/bin/ncu --section SourceCounters --section WarpStateStats --section SpeedOfLight \
  --section LaunchStats --section Occupancy --section InstructionStats --section MemoryWorkloadAnalysis \
  --clock-control none --import-source on -k regex:k_semcheck -c 1 -o $O/sem \
  python bench.py --kernels ${NK:-4096} --steps 1 --warmup 3 --no-e2e --no-cpu --semantic > $O/ncu.log 2>&1
/usr/local/cuda/bin/ncu -i $O/sem.ncu-rep --page source --csv --print-source cuda,sass 2>/dev/null | python tools/ncu_funcs.py /dev/stdin 30 > $O/funcs_k_semcheck.txt 2>/dev/null
/usr/local/cuda/bin/ncu -i $O/sem.ncu-rep --page details --csv > $O/details.csv 2>/dev/null
rm -f $O/sem.ncu-rep
ls -la $O
