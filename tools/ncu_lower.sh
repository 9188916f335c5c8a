#!/bin/bash
# Focused ncu capture of one phase kernel (KERNEL, default k_lower) with source counters.
O=gpurun_out/${1:-ncu_lower}
mkdir -p $O
K=${KERNEL:-k_lower}
timeout 900 /usr/local/cuda/bin/ncu --section SourceCounters --section WarpStateStats --section SpeedOfLight \
  --section LaunchStats --section Occupancy --section InstructionStats --section MemoryWorkloadAnalysis \
  --clock-control none --import-source on -k regex:$K -c 1 -o $O/$K \
  python bench.py --kernels ${NK:-30000} --steps 1 --warmup 3 --no-e2e --no-cpu > $O/ncu.log 2>&1
ls -la $O
