#!/bin/bash
# Bench line + ncu launch list (same command, 50k-kernel sample) on one GPU.
TAG=${1:-bench}
O=gpurun_out/$TAG
mkdir -p $O
timeout 1500 python bench.py --steps ${STEPS:-3} --warmup 3 > $O/bench.json 2> $O/bench.err
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches.csv python bench.py --kernels 50000 --steps 1 --warmup 3 --no-e2e --no-cpu \
  > $O/ncu_launch.log 2>&1
ls -la $O
