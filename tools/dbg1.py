import numpy as np, torch, ctypes as C, sys
sys.path.insert(0,'/root/repo')
from paper_1712_09005_b200 import optimizer as opt, _lib, affinities as aff
z=np.load('/root/repo/tests/golden/reference_golden.npz')
r,c,v=z['run_fft_rows'],z['run_fft_cols'],z['run_fft_vals']
P=aff.SparseAffinities(n=1500,rows=r,cols=c,values=v)
for dt in (torch.float64, torch.float32):
    y0=opt.np.random.default_rng(np.random.SeedSequence(5).spawn(3)[1]).normal(0,1e-4,(1500,2))
    ctx,_=opt._ctx_with_P(P,0,2,dt,3,50,1.0)
    ya=torch.from_numpy(y0).to(device=0,dtype=dt); yb=torch.empty_like(ya)
    vel=torch.zeros_like(ya); gains=torch.ones_like(ya)
    kl=torch.zeros(10,dtype=torch.float64,device=0); st=torch.zeros(10,dtype=torch.int32,device=0)
    bb=(C.c_double*4)()
    print(dt, "bbox rc", ctx.lib.fitsne_bbox(ctx.h,_lib.ptr(ya),1500,bb,ctx.stream), list(bb), _lib.last_error())
    for it in range(3):
        rc=ctx.lib.fitsne_iterate(ctx.h,_lib.ptr(ya),_lib.ptr(yb),_lib.ptr(vel),_lib.ptr(gains),12.0,0.5,200.0,C.c_void_p(kl.data_ptr()+8*it),C.c_void_p(st.data_ptr()+4*it),ctx.stream)
        print(it, rc, _lib.last_error(), kl[:3].tolist(), st[:3].tolist(), yb[:2].tolist())
        ya,yb=yb,ya
