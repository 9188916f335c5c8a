#!/bin/bash
# One GPU round trip for a build: GPU suite, C4 bench (short), C5 sample phases,
# launch list of the C5 sample.   tools/r2_check.sh OUTDIR [skip-tests]
O=gpurun_out/$1
mkdir -p $O
if [ -z "$2" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q > $O/gputest.log 2>&1; echo rc=$? >> $O/gputest.log
fi
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu > $O/bench_c4.json 2> $O/bench_c4.err
timeout 600 python -c "
import paper_2107_07809_b200 as P, json
s = P.Session(0)
st, _, _ = s.run_generated('C5', 3000, seed=0x210707809C5)
ss = s.stats()
print(json.dumps({'stream': st, 'front': ss['ms_front'], 'lower': ss['ms_lower'], 'fold': ss['ms_fold'], 'emit': ss['ms_render'], 'parse': ss['ms_parse'], 'gather': ss['ms_emit']}))
" > $O/c5_phases.json 2>&1
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/c5_launches.csv python -c "
import paper_2107_07809_b200 as P
s = P.Session(0)
s.run_generated('C5', 1000, seed=0x210707809C5)
" > /dev/null 2>&1
