#!/bin/bash
# One gpurun call: GPU parity suite, smoke, phase profile, bench line, ncu
# launch list and one full ncu capture per hot kernel.  Usage (from here):
#   gpurun --timeout 2400 -- 'bash tools/gpu_round.sh TAG [quick]'
TAG=${1:-r1}
MODE=${2:-full}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/gpu.txt 2>&1
nproc > $O/nproc.txt; lscpu | grep -i 'model name' >> $O/nproc.txt
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $O/pytest_gpu.log
timeout 300 python __graft_entry__.py > $O/smoke.log 2>&1; echo "smoke rc $?" >> $O/smoke.log
for c in C2 C3; do
  timeout 300 python tools/gpu_prof.py $c 10000 > $O/prof_$c.json 2>&1
done
timeout 600 python tools/gpu_prof.py C4 100000 > $O/prof_C4.json 2>&1
if [ "$MODE" = "full" ]; then
  timeout 1500 python bench.py --steps 3 --warmup 3 > $O/bench.json 2> $O/bench.err
fi
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches.csv python bench.py --kernels 50000 --steps 1 --warmup 3 --no-e2e --no-cpu \
  > $O/ncu_launch.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_decompile -c 1 \
  -o $O/k_decompile python bench.py --kernels 20000 --steps 1 --warmup 3 --no-e2e --no-cpu \
  > $O/ncu_dec.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on \
  -k regex:'k_nl_write|k_classify|k_decode|k_gather|k_nl_count' -c 6 \
  -o $O/k_parse python bench.py --kernels 200000 --steps 1 --warmup 3 --no-e2e --no-cpu \
  > $O/ncu_parse.log 2>&1
ls -la $O
