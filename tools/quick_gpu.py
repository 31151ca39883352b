import sys, time
sys.path.insert(0, '.')
import numpy as np
import oracle
import paper_1909_09825_b200 as fgt
ys=[0.0,0.1,0.35,0.5,0.75,1.0]; a=[0.5,-0.25,1.0,0.8,-0.6,0.9]; xs=[0.0,0.5,1.0]
gold=np.array([0.53026354628615822,1.3078174711896560,0.66552744606900788])
print("golden", np.array(fgt.gauss_transform(xs,ys,a,0.02,ne=6))-gold, flush=True)
print("direct", np.array(fgt.direct_transform(xs,ys,a,0.02))-gold, flush=True)
for (n,m,delta,ne,srt) in [(1000,1000,1e-2,6,True),(100000,100000,1e-2,6,True),(200000,300000,1e-3,6,False),(100000,100000,1e-6,6,True),(50000,50000,1.0,4,False)]:
    x=fgt.uniform_points_array(n,1,3); y=fgt.uniform_points_array(m,1,0); al=2*fgt.uniform_points_array(m,1,1)-1
    if srt: x=np.sort(x); y=np.sort(y)
    t=time.time(); u=np.array(fgt.gauss_transform(x,y,al,delta,ne=ne)); tg=time.time()-t
    ref=oracle.transform(x,y,al,delta,ne=ne)
    print(n,m,delta,ne,srt,"err/sum|a|",np.abs(u-ref).max()/np.abs(al).sum(), "t",tg, flush=True)
