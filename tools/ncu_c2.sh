#!/bin/bash
# Full ncu capture of k_decompile on a C2/C4 sample at a given KPW.
O=gpurun_out/${1:-ncu}
mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
for k in ${KPWS:-1 32}; do
  OCLDEC_B200_KPW=$k timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_decompile -c 1 \
    -o $O/dec_${CFG:-C2}_kpw$k python bench.py --config ${CFG:-C2} --kernels ${NK:-10000} --steps 1 --warmup 3 --no-e2e --no-cpu \
    > $O/ncu_kpw$k.log 2>&1
done
ls -la $O
