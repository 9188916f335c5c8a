#!/bin/bash
# Full ncu capture of the three decompile phase kernels on a sample.
O=gpurun_out/${1:-ncu_phases}
mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
timeout 1200 $NCU --set full --clock-control none --import-source on -k regex:'k_front|k_lower|k_fold|k_emit' -c 4 \
  -o $O/phases_${CFG:-C4} python bench.py --config ${CFG:-C4} --kernels ${NK:-50000} --steps 1 --warmup 3 --no-e2e --no-cpu \
  > $O/ncu.log 2>&1
ls -la $O
