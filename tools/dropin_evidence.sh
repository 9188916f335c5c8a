#!/bin/bash
# The drop-in evidence of the current build: the reference's acceptance
# harness through the GPU drop-in (and with the body withheld), and the
# DecompiledKernel::cfg field-by-field check on several corpora.
#   tools/dropin_evidence.sh OUTDIR
O=gpurun_out/${1:-dropin}
mkdir -p $O
export LD_LIBRARY_PATH=$PWD/paper_2107_07809_b200
timeout 900 oracle/_ref/acceptance_b200 > $O/acceptance_b200.txt 2>&1; echo "rc=$?" >> $O/acceptance_b200.txt
OCLDEC_B200_DROPIN_NO_BODY=1 timeout 900 oracle/_ref/acceptance_b200 > $O/acceptance_b200_nobody.txt 2>&1; echo "rc=$?" >> $O/acceptance_b200_nobody.txt
python - "$O" <<'PY'
import os, subprocess, sys
sys.path.insert(0, os.getcwd())
from oracle import oracle as O
out = sys.argv[1]
cases = [("corpus", b"".join(x[1] for x in O.corpus())),
         ("nests300", b"".join(O.make_nest(s) for s in range(1, 301)))]
for shape, stress, count in (("C2", 1, 300), ("C3", 0, 300), ("C3", 1, 300), ("C4", 0, 300)):
    cases.append((f"{shape}-stress{stress}-{count}", O.generate_corpus(shape, count, seed=91 + count, stress=bool(stress))[0]))
with open(os.path.join(out, "cfg_check.txt"), "w") as f:
    for name, listing in cases:
        p = os.path.join(out, name + ".s")
        open(p, "wb").write(listing)
        r = subprocess.run(["oracle/_ref/cfg_check_b200", p], capture_output=True, text=True)
        f.write(f"{name}: {r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-300:]} (rc {r.returncode})\n")
        os.remove(p)
PY
cat $O/cfg_check.txt
