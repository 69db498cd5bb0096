import sys, numpy as np
sys.path.insert(0,'/root/repo/tests'); sys.path.insert(0,'/root/repo')
import helpers
from paper_2501_10689_b200.channel import generate
T=200
tot={'index':[], 'vrsort':[], 'full':[], 'need':[]}
for s in range(4):
    r = helpers.oracle_cfg2_philox_task((s,'vr-ogrk',2024,T))
    rows = r['rows']  # (K,T)
    ch = generate('cfg2',[s])
    st, ln = ch.start[0], ch.length[0]
    K = len(st)
    c0 = st//32; c1=(st+ln-1)//32
    # coupled: rows overlapping VR of row i
    ov = (st[:,None] < (st+ln)[None,:]) & (st[None,:] < (st+ln)[:,None])
    pieces = c1-c0+1
    full = pieces.sum()
    for name, order in (('index', np.arange(K)), ('vrsort', np.argsort(st, kind='stable'))):
        w=0; n=0
        for t in range(1,T):
            for g in range(0,K,32):
                grp = order[g:g+32]
                prev = rows[grp, t-1]
                prev = prev[prev>=0]
                if len(prev)==0: continue
                need = ov[prev].any(axis=0)   # rows needed by any rhs of the group
                w += pieces[need].sum(); n += full
        tot[name].append(w/n)
    # algorithmic need per rhs
    a=0;n=0
    for t in range(1,T):
        prev = rows[:, t-1]; prev=prev[prev>=0]
        a += pieces[ov[prev]].sum() if False else sum(pieces[ov[p]].sum() for p in prev); n += full*len(prev)
    tot['need'].append(a/n)
print({k: np.mean(v) for k,v in tot.items() if v})
