"""Rank-kernel occupancy probe: device time of the rank stage at a given
subset size with the full (1 CTA/SM) and lean (2 CTAs/SM) cluster kernels at
the same cluster size. Usage: python tools/rank_occ_probe.py n_m CL"""
import os, sys, subprocess, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
n_m, cl = int(sys.argv[1]), sys.argv[2]
code = r'''
import sys, numpy as np, torch, json
sys.path.insert(0,'.')
import paper_1609_05530_b200 as pcb
n_m=%d; n=(200_000_000//n_m)*n_m; K=n//n_m
ctx=pcb.Context(0); s=torch.cuda.current_stream(); ctx.set_stream(s.cuda_stream)
X=pcb.sample_matrix(1, 5.0, n, K, device_out=True, ctx=ctx)
off=np.arange(K+1,dtype=np.uint64)*np.uint64(n_m)
for _ in range(2): U=pcb.normalized_ranks(X, off, ctx=ctx)
e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
e0.record(s)
for _ in range(3): U=pcb.normalized_ranks(X, off, ctx=ctx)
e1.record(s); torch.cuda.synchronize()
print(json.dumps({"n_m":n_m,"ms_per_call":e0.elapsed_time(e1)/3,"paths":ctx.rank_paths()}))
''' % n_m
for lean in ("0", "1"):
    env = dict(os.environ, PCB_RANK_CL=cl, PCB_RANK_LEAN=lean)
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print("lean", lean, "CL", cl, out.stdout.strip() or out.stderr[-500:])
