import numpy as np, sys
sys.path.insert(0,'/root/repo')
from paper_2604_10187_b200 import capi, synthetic as S
cfg=S.config_space(False); t=S.synthetic_tables(cfg); reg=S.registry_arrays(cfg)
P=capi.prune_plan(t, reg, 148); masks=P['masks']; R=P['R']; cls_cfg=P['cls_cfg']; seg_pos=P['seg_pos']; seg_n=P['seg_n']
C=len(cfg['id']); W=40
theta=t['coeff_theta'].reshape(C,W,4); ext=t['theta_ext'].reshape(C,4)
rows=np.concatenate([theta, ext[:,None,:]],1)  # [C][R=41][4]: row r -> wave r+1, last = ext
rng=np.random.default_rng(1); n=100_000
dec=rng.random(n)<0.5
M=np.where(dec, rng.integers(1,257,n), rng.integers(257,8193,n)).astype(np.int64)
N=rng.integers(256,32769,n).astype(np.int64); K=rng.integers(256,32769,n).astype(np.int64)
nseg=len(seg_pos)
segbest=np.full((n,nseg),np.inf); LB=np.full((n,nseg),-np.inf)
S_=148
for s in range(nseg):
    cfgs=cls_cfg[seg_pos[s]:seg_pos[s]+seg_n[s]]
    tm,tn,tk=cfg['t_m'][cfgs[0]],cfg['t_n'][cfgs[0]],cfg['t_k'][cfgs[0]]
    G=((M+tm-1)//tm)*((N+tn-1)//tn); L=(K+tk-1)//tk
    r=np.minimum((G+S_-1)//S_, R)-1; lb=np.minimum(np.floor(np.log2(L)).astype(int),15)
    m=masks[s, r, lb]
    # cell box
    G0=r*S_+1.0; G1=np.where(r==R-1, np.inf, (r+1)*S_*1.0); L0=2.0**lb; L1=np.where(lb==15, np.inf, 2.0**(lb+1)-1)
    for j,c in enumerate(cfgs):
        alive=(m>>j)&1
        th=rows[c][r]  # [n,4]
        f=th[:,0]*G*L+th[:,1]*G+th[:,2]*L+th[:,3]
        segbest[:,s]=np.where(alive==1, np.minimum(segbest[:,s], f), segbest[:,s])
        # lower bound over the cell box: bilinear min at corners (all coeffs here positive -> (G0,L0))
        lbv=th[:,0]*G0*L0+th[:,1]*G0+th[:,2]*L0+th[:,3]
        neg=(th<0).any(1)
        lbv=np.where(neg, -np.inf, lbv)
        LB[:,s]=np.where(alive==1, np.where(LB[:,s]==-np.inf, lbv, np.minimum(LB[:,s], lbv)), LB[:,s])
best=segbest.min(1)
skip=(LB>best[:,None]*(1+1e-9))
print("segments", nseg, "max skippable fraction (oracle best known)", skip.mean())
# realistic: evaluate segments in ascending LB order, skip when LB > running best
order=np.argsort(LB,1)
runs=0
for q in range(0,n,1):
    b=np.inf; cnt=0
    for s in order[q]:
        if LB[q,s] > b*(1+1e-9): continue
        cnt+=1; b=min(b, segbest[q,s])
    runs+=cnt
print("evaluated segments per query in LB order", runs/n, "of", nseg)
