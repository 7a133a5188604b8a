import sys, ctypes, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2604_15765_b200 import hermsim as H, _native as nat
from paper_2604_15765_b200.multigpu import ShardGroup
grp = ShardGroup(10, 5, 4)
L = nat.engine()
for s in range(4):
    st = grp.shards[s]
    for tbl, tg in (([0,1,3,2],[8,9]), ([0,2,1,3],[8,9]), ([0,1,3,2],[9,8])):
        t = (ctypes.c_uint32*2)(*tg); tb = (ctypes.c_uint32*4)(*tbl)
        rc = L.hs_apply_permutation(st.handle, 2, tb, t, None)
        print(s, tbl, tg, rc, L.hs_last_error())
    try:
        H.apply(st, H.native_gate("cnot"), [9, 8]); print("apply ok")
    except Exception as e:
        print("apply raised", e)
