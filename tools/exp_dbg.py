import ctypes as C, sys, numpy as np, torch
sys.path.insert(0,'.')
import paper_1609_05530_b200 as pcb
n=200_000_000; K=n//125000
ctx=pcb.Context(0); s=torch.cuda.current_stream(); ctx.set_stream(s.cuda_stream)
u1=torch.empty(n,dtype=torch.float64,device='cuda'); u2=torch.empty_like(u1)
ctx.check(ctx.lib.pcb_sample(ctx.ptr,1,5.0,n,K,0,K,pcb.BASE_SEED,u1.data_ptr(),u2.data_ptr()))
off=(np.arange(K+1,dtype=np.uint64)*np.uint64(n//K)); off[-1]=n
offp=off.ctypes.data_as(C.POINTER(C.c_uint64))
for name,f in [('uniform',lambda u:u),('exponential',lambda u:-torch.log1p(-u)),('normal',torch.special.ndtri)]:
    x1,x2=f(u1).contiguous(),f(u2).contiguous()
    rec=torch.zeros((K,6),dtype=torch.int64,device='cuda')
    for it in range(3):
        e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
        e0.record(s)
        ctx.check(ctx.lib.pcb_fit_blocks(ctx.ptr,1,0,x1.data_ptr(),x2.data_ptr(),n,offp,K,rec.data_ptr()))
        e1.record(s); torch.cuda.synchronize()
        print(name, it, round(e0.elapsed_time(e1),2), {k:round(v,2) for k,v in ctx.stage_times().items()}, ctx.rank_paths())
    r=rec.cpu().numpy().view(np.float64) if False else rec.cpu().numpy()
    print(' converged', (r[:,3]!=0).sum() if r.shape[1]>3 else None)
