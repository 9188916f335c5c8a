import sys; sys.path.insert(0,'.')
import paper_2107_07809_b200 as P
r=P.decompile_listing(open('tests/golden/copy.asm','rb').read())
print(r.combined[:200])
