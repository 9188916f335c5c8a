#!/bin/bash
# Source-level ncu capture of the parse kernels (k_classify, k_decode) on a C4 sample.
O=gpurun_out/${1:-ncu_parse_src}
mkdir -p $O
timeout 1500 /usr/local/cuda/bin/ncu --section SourceCounters --section WarpStateStats --section SpeedOfLight \
  --section LaunchStats --section Occupancy --section InstructionStats --section MemoryWorkloadAnalysis \
  --clock-control none --import-source on -k "regex:k_decode|k_classify|k_nl_count|k_nl_write" -c 4 -o $O/parse \
  python bench.py --kernels ${NK:-100000} --steps 1 --warmup 0 --no-e2e --no-cpu > $O/ncu.log 2>&1
for k in k_decode k_classify; do
  /usr/local/cuda/bin/ncu -i $O/parse.ncu-rep -k $k --page source --csv --print-source cuda,sass > $O/cs_$k.csv 2>/dev/null
done
/usr/local/cuda/bin/ncu -i $O/parse.ncu-rep --page details --csv > $O/details.csv 2>/dev/null
ls -la $O
