# A/B of rank-kernel variants: uniform-data cycles per phase + parity of ranks vs the default build
for L in "" paper_1609_05530_b200/libparcop_b200_exp_a.so paper_1609_05530_b200/libparcop_b200_exp_b.so ; do
PCB_LIB_PATH=$L PCB_RANK_PROFILE=1 python - <<PY 2>&1 | grep -v "^$" | cut -c1-220
import numpy as np, sys, hashlib
sys.path.insert(0,'.')
import paper_1609_05530_b200 as pcb
n=50_000_000; K=n//125000
g=np.random.default_rng(1)
x=g.random(n); y=g.random(n)
ctx=pcb.Context(0)
off=np.linspace(0,n,K+1).astype(np.uint64)
for i in range(2): U=pcb.normalized_ranks(pcb.DataMatrix(x,y),off,ctx=ctx)
print('$L', ctx.stage_times().get('rank'), hashlib.sha256(U.u1.tobytes()+U.u2.tobytes()).hexdigest()[:16], file=sys.stderr)
PY
done
