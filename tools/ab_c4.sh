#!/bin/bash
# A/B of the C4 bench between the in-tree library and variants/<name>/libocldec_b200.so
O=gpurun_out/$1; shift
mkdir -p $O
for rep in 1 2; do
  timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > $O/base_$rep.json 2>/dev/null
  for v in "$@"; do
    OCLDEC_B200_LIB=variants/$v/libocldec_b200.so timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > $O/${v}_$rep.json 2>/dev/null
  done
done
