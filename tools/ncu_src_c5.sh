#!/bin/bash
# Source-level ncu capture of k_front / k_lower on a C5 sample (streamed run).
O=gpurun_out/${1:-ncu_src_c5}
mkdir -p $O
timeout 1500 /usr/local/cuda/bin/ncu --section SourceCounters --section WarpStateStats --section SpeedOfLight \
  --section LaunchStats --section Occupancy --section InstructionStats --section MemoryWorkloadAnalysis \
  --clock-control none --import-source on -k "regex:k_front|k_lower|k_emit" -c 3 -o $O/c5 \
  python -c "
import paper_2107_07809_b200 as P
s = P.Session(0)
st, _, _ = s.run_generated('C5', ${NK:-1500}, seed=0x210707809C5)
print(st, s.stats())
" > $O/ncu.log 2>&1
for k in k_front k_lower k_emit; do
  /usr/local/cuda/bin/ncu -i $O/c5.ncu-rep -k $k --page source --csv --print-source cuda,sass > $O/cs_$k.csv 2>/dev/null
done
ls -la $O
