# per-phase SM cycles of the rank cluster kernel (PCB_RANK_PROFILE) on 1e8 uniform
# keys per column, once per environment setting given as arguments
for S in "$@"; do env $S PCB_RANK_PROFILE=1 python - <<PY 2>&1 | grep "rank profile" | tail -1 | sed "s|^|[$S] |"
import numpy as np, sys
sys.path.insert(0,'.')
import paper_1609_05530_b200 as pcb
n=100_000_000; K=n//125000
g=np.random.default_rng(1)
x=g.random(n); y=g.random(n)
ctx=pcb.Context(0)
off=np.linspace(0,n,K+1).astype(np.uint64)
for i in range(2): U=pcb.normalized_ranks(pcb.DataMatrix(x,y),off,ctx=ctx)
PY
done
