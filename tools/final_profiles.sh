#!/bin/bash
# Round-end evidence: full ncu capture of the decompile phases and the parse
# kernels on C4 samples, plus the launch list of one bench-shaped run.
O=gpurun_out/${1:-final}
mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
timeout 1200 $NCU --set full --clock-control none --import-source on -k regex:'k_front|k_lower|k_fold|k_emit' -c 4 \
  -o $O/phases python bench.py --kernels 30000 --steps 1 --warmup 3 --no-e2e --no-cpu > $O/ncu_phases.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on \
  -k regex:'k_nl_count|k_nl_write|k_classify|k_decode|k_gather|k_ksize' -c 7 \
  -o $O/parse python bench.py --kernels 200000 --steps 1 --warmup 3 --no-e2e --no-cpu > $O/ncu_parse.log 2>&1
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches.csv python bench.py --kernels 50000 --steps 1 --warmup 3 --no-e2e --no-cpu \
  > $O/ncu_launch.log 2>&1
ls -la $O
