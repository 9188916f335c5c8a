#!/bin/bash
# Source-level ncu capture (stall samples per SASS / CUDA line) of the
# decompile phase kernels on a C4 sample; one launch each.
#   tools/ncu_src.sh OUTDIR [regex]
O=gpurun_out/${1:-ncu_src}
mkdir -p $O
K=${2:-"k_front|k_lower|k_emit|k_fold"}
timeout 1500 /usr/local/cuda/bin/ncu --section SourceCounters --section WarpStateStats --section SpeedOfLight \
  --section LaunchStats --section Occupancy --section InstructionStats --section MemoryWorkloadAnalysis \
  --clock-control none --import-source on -k "regex:$K" -c 4 -o $O/phases \
  python bench.py --kernels ${NK:-30000} --steps 1 --warmup 3 --no-e2e --no-cpu > $O/ncu.log 2>&1
for k in k_front k_lower k_fold k_emit; do
  /usr/local/cuda/bin/ncu -i $O/phases.ncu-rep -k $k --page source --csv --print-source cuda > $O/src_$k.csv 2>/dev/null
done
ls -la $O
