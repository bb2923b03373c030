import sys; sys.path[:0]=['.','tests']
import numpy as np, scipy.sparse as sp, torch, oracle, pscgen
import paper_2406_19754_b200 as psc
n=8
A=sp.diags([-np.ones(n-1),2*np.ones(n),-np.ones(n-1)],[-1,0,1],format='csr'); A.sort_indices()
h=pscgen.csr_hierarchy(A, max_levels=1)
print("oracle", oracle.pcg(h, np.ones(n), tol=1e-30, maxit=3, pre=1, post=1, coarse=3)[1:])
for env in ({}, {"PSC_NO_DENSE_COARSE":"1"}):
    import os
    os.environ.update(env)
    ctx=psc.Context(); d=psc.Descriptor(ctx,n,[0,n]); m=psc.Matrix(ctx,d,d,A.indptr,A.indices,A.data); d.assemble(); m.assemble()
    H=psc.Hierarchy(ctx,[m],[],[],pre=1,post=1,coarse=3)
    b=torch.ones(n,dtype=torch.float64,device='cuda')
    z=torch.zeros(n,dtype=torch.float64,device='cuda'); H.vcycle(b,z); print(env, "vcycle", z.cpu().numpy(), oracle.vcycle(h, np.ones(n), pre=1, post=1, coarse=3))
    try:
        x=torch.zeros(n,dtype=torch.float64,device='cuda'); print(H.solve(b,x,tol=1e-30,maxit=3)[::2])
    except Exception as e: print("ERR", e)
    ctx.close()
