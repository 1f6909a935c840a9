# A/B of rank-kernel variants (PCB_LIB_PATH libraries built with `make exp`):
# uniform-data cycles per phase + rank hashes (uniform and tie-heavy) vs the default build
for L in "" ${AB_LIBS:-paper_1609_05530_b200/libparcop_b200_exp_a.so paper_1609_05530_b200/libparcop_b200_exp_b.so}; do
PCB_LIB_PATH=$L PCB_RANK_PROFILE=1 python - <<PY 2>&1 | grep -v "^$" | cut -c1-200
import numpy as np, sys, hashlib
sys.path.insert(0,'.')
import paper_1609_05530_b200 as pcb
n=50_000_000; K=n//125000
g=np.random.default_rng(1)
ctx=pcb.Context(0)
off=np.linspace(0,n,K+1).astype(np.uint64)
x=g.random(n); y=np.round(g.random(n),4)
T=pcb.normalized_ranks(pcb.DataMatrix(x,y),off,ctx=ctx)
h1=hashlib.sha256(T.u1.tobytes()+T.u2.tobytes()).hexdigest()[:12]
y=g.random(n)
for i in range(2): U=pcb.normalized_ranks(pcb.DataMatrix(x,y),off,ctx=ctx)
print('$L', 'ties', h1, 'uniform', hashlib.sha256(U.u1.tobytes()+U.u2.tobytes()).hexdigest()[:12], file=sys.stderr)
PY
done
