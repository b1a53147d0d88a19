import sys, numpy as np
sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/oracle')
import paper_2501_17779_b200 as cva
from pyoracle import Oracle
O=Oracle()
rng=np.random.default_rng(0)
for n in [4,8,16,32,64,65,100,127,128,200,256,300,511,512,1000,2000,3000]:
    phi=np.sort(rng.uniform(0,2*np.pi,n)); r=1+0.3*np.cos(3*phi)
    raw=np.stack([r*np.cos(phi),r*np.sin(phi)],1)
    row=[]
    for nout in [8,100,128,1024]:
        g=cva.resample_uniform(raw,nout); w=O.resample_uniform(raw,nout)
        e=np.abs(g-w).max(axis=0)
        row.append("%d:%.1e/%.1e"%(nout,e[0],e[1]))
    print(n, " ".join(row))
