for t in uniform normal cauchy; do PCB_RANK_PROFILE=1 python - <<PY 2>&1 | grep "rank profile" | tail -1
import numpy as np, torch, ctypes as C, sys
sys.path.insert(0,'.')
import paper_1609_05530_b200 as pcb
from scipy.special import ndtri
n=200_000_000//4; K=n//125000
g=np.random.default_rng(1)
u=g.random(n)
f={'uniform':lambda u:u,'normal':ndtri,'cauchy':lambda u: np.tan(np.pi*(u-0.5))}['$t']
x=f(u); y=f(g.random(n))
ctx=pcb.Context(0)
off=np.linspace(0,n,K+1).astype(np.uint64)
for i in range(2): U=pcb.normalized_ranks(pcb.DataMatrix(x,y),off,ctx=ctx)
print('$t', ctx.rank_paths(), file=sys.stderr)
PY
done
