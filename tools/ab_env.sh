#!/bin/bash
# A/B of the C4 bench under environment settings: tools/ab_env.sh OUT "VAR=val ..." ["VAR=val ..."]
O=gpurun_out/$1; shift
mkdir -p $O
for rep in 1 2; do
  timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu > $O/base_$rep.json 2>/dev/null
  i=0
  for e in "$@"; do
    i=$((i+1))
    env $e timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu > $O/env${i}_$rep.json 2>/dev/null
  done
done
