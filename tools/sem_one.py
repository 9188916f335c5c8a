"""One semantic-check launch on a single fuel-exhausting kernel (C4 bench
corpus kernel 4619 as kernel 0): the target of tools/ncu_sem_one.sh."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_07809_b200 as P  # noqa: E402

listing, _, _ = P.generate_corpus("C4", 1, seed=0x210707809C4, k0=4619)
r = P.decompile_listing(listing, P.DecompileOptions(semantic_check=True, semantic_seed=0x5E3A171C))
print(r.kernels[0].semantic)
