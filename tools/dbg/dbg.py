import sys, numpy as np
sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/oracle')
import oracle as O
from paper_2604_15765_b200 import hermsim as H, harness as HS
orc=O.Oracle()
n,m=8,5
psi=HS.rank_psi(n,5,4); base=HS.rho_payload(n,psi,m)
st=H.TiledHermitian(n,m)
for name,spec,och,tg in [("haar2",H.make_generic("u",HS.haar(2,3)),O.generic(HS.haar(2,3)),[5,7]), ("ident",H.make_generic("u",np.eye(4)),O.generic(np.eye(4)),[5,7])]:
    want=base.copy(); orc.apply(want,n,m,och,tg)
    st.upload(base); H.apply(st,spec,tg); got=st.download()
    G=got.reshape(-1,32,32); W=want.reshape(-1,32,32); B=base.reshape(-1,32,32)
    for t in (12,13,17,18,14):
        g,w,b=G[t],W[t],B[t]
        print(name,t,'ok',np.abs(g-w).max()<1e-12,'conj',np.abs(g-w.conj()).max()<1e-12,'T',np.abs(g-w.T).max()<1e-12,'cT',np.abs(g-w.conj().T).max()<1e-12,'=base',np.abs(g-b).max()<1e-15)
        for q in range(2):
          for r in range(2):
            blk=(slice(16*q,16*q+16),slice(16*r,16*r+16))
            print('   sub',q,r,'ok',np.abs(g[blk]-w[blk]).max()<1e-12, 'cT-of-other', [np.abs(g[blk]-w[16*a:16*a+16,16*c:16*c+16].conj().T).max()<1e-12 for a in range(2) for c in range(2)])
