"""fp32 likelihood path (precision=1) at edge parameters against the fp64 oracle:
Gumbel just above theta = 1, Frank at small |theta| and large |theta|, Gaussian
near 0 and +-1. Reports cases outside the 1e-5 bar (Known limits).

    python tools/fp32_edges.py
"""
import numpy as np, sys
sys.path.insert(0,'.')
import paper_1609_05530_b200 as pcb
from oracle.oracle import oracle_lib
orc=oracle_lib(); ctx=pcb.Context(0)
g=np.random.default_rng(5); worst=0; bad=0; cases=0
for fam, thetas in ((2,[1.001,1.003,1.006,1.01,1.05]), (1,[-0.3,-0.05,0.05,0.3,1.0,1.5,1.9,2.1,3.0,25.0,-30.0]), (0,[0.0,0.97,-0.97])):
    for th in thetas:
        for rep in range(3):
            n=int(g.integers(2000,200000)); k=int(g.integers(1,5))
            X=pcb.sample_matrix(fam, th, n, k, base_seed=int(g.integers(1,2**62)), ctx=ctx)
            off=orc.partition(n,k)
            got=pcb.fit_blocks(fam, X, off, precision=pcb.Precision.fp32, ctx=ctx)
            want=orc.fit_blocks(fam, X.col1, X.col2, off)
            for a,b in zip(got,want):
                cases+=1
                if bool(a.converged)!=bool(b.converged): bad+=1; print('CONV', fam, th, n, a.converged, b.converged, a.theta_hat, b.theta_hat); continue
                if not b.converged: continue
                e=max(abs(a.theta_hat-b.theta_hat)/abs(b.theta_hat), abs(a.sigma2-b.sigma2)/abs(b.sigma2))
                worst=max(worst,e)
                if e>1e-5: bad+=1; print('TOL', fam, th, n, a.theta_hat, b.theta_hat, a.sigma2, b.sigma2, e)
print('fp32 edge cases', cases, 'bad', bad, 'worst', worst)
