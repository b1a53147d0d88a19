import sys, numpy as np
sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/oracle')
import paper_2501_17779_b200 as cva
from pyoracle import Oracle
O=Oracle()
g=np.load('/root/repo/tests/golden/curve_core_kat.npz')
h=g['hippo100']
for nout in (8,64,128,1024):
    r=cva.resample_uniform(h,nout); ro=O.resample_uniform(h,nout)
    p=cva.preprocess(h,nout); po=O.preprocess(h,nout)
    print(nout, np.abs(r-ro).max(axis=0), np.abs(p-po).max(axis=0))
    c=ro.mean(0); L=np.sum(np.hypot(*(np.roll(ro,-1,0)-ro).T))
    print('  centroid/len oracle', c, L, ' gpu implied', ((r-p/ (1/L))[:3]))
