#!/bin/bash
# Round-end evidence of the last round-2 build (session 3):
#   gputest.log, bench_c4.json (default bench: C4 1M, 5 steps), bench_ref_c4.json
#   (the reference arm), launches.csv (ncu launch list, bench-shaped C4 run),
#   phases/c5/parse ncu --set full summaries, k_fold counters (a targeted
#   metric list: its --set full replay returns nan).
O=gpurun_out/${1:-final_r2b}
mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
timeout 1200 python -m pytest tests -m gpu -q > $O/gputest.log 2>&1; echo rc=$? >> $O/gputest.log
timeout 900 python bench.py > $O/bench_c4.json 2> $O/bench_c4.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref_c4.json 2> $O/bench_ref_c4.err
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches.csv python bench.py --kernels 50000 --steps 1 --warmup 3 --no-e2e --no-cpu \
  > $O/ncu_launch.log 2>&1
timeout 1500 $NCU --set full --clock-control none --import-source on -k regex:'k_front|k_lower|k_fold|k_emit' -c 4 \
  -o $O/phases python bench.py --kernels 30000 --steps 1 --warmup 3 --no-e2e --no-cpu > $O/ncu_phases.log 2>&1
timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__thread_inst_executed_per_inst_executed.ratio,smsp__sass_average_branch_targets_threads_uniform.pct \
  --clock-control none -k regex:'k_fold' -c 2 --csv --log-file $O/k_fold_metrics.csv \
  python bench.py --kernels 30000 --steps 1 --warmup 3 --no-e2e --no-cpu > $O/ncu_fold.log 2>&1
timeout 1500 $NCU --set full --clock-control none --import-source on -k regex:'k_front|k_lower|k_fold|k_emit' -c 4 \
  -o $O/c5 python -c "
import paper_2107_07809_b200 as P, json
s = P.Session(0)
st, _, _ = s.run_generated('C5', 1500, seed=0x210707809C5)
print(json.dumps(st))
" > $O/ncu_c5.log 2>&1
timeout 1200 $NCU --set full --clock-control none --import-source on \
  -k regex:'k_nl_count|k_nl_write|k_classify|k_decode|k_gather|k_ksize' -c 6 \
  -o $O/parse python bench.py --kernels 200000 --steps 1 --warmup 0 --no-e2e --no-cpu > $O/ncu_parse.log 2>&1
for r in phases c5 parse; do
  [ -f $O/$r.ncu-rep ] && $NCU -i $O/$r.ncu-rep --page details --csv > $O/${r}_details.csv 2>/dev/null
done
OUT=$O/dram_traffic.json python tools/traffic_json.py $O/phases.ncu-rep $O/ncu_phases.log > /dev/null 2>&1
OUT=$O/dataflow_ncu.json python tools/dataflow_json.py $O/phases.ncu-rep $O/c5.ncu-rep > /dev/null 2>&1
for k in k_front k_lower k_emit; do
  $NCU -i $O/phases.ncu-rep -k $k --page source --csv --print-source cuda,sass 2>/dev/null | python tools/ncu_funcs.py /dev/stdin 25 > $O/funcs_$k.txt 2>&1
done
rm -f $O/*.ncu-rep
du -sh $O
