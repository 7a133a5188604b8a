"""Diagnostics: compare each shard of a freshly filled ShardGroup with the layout's scatter of the
single-GPU payload (python tools/shard_debug.py N P)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_15765_b200 import harness as HS  # noqa: E402
from paper_2604_15765_b200 import hermsim as H  # noqa: E402
from paper_2604_15765_b200.multigpu import ShardGroup  # noqa: E402

n, P = int(sys.argv[1]), int(sys.argv[2])
psi = HS.rank_psi(n, 42, 4)
ref = H.TiledHermitian(n)
ref.fill_mixture(psi)
grp = ShardGroup(n, 5, P)
grp.fill_mixture(psi)
parts = grp.layout.scatter(ref.download())
for s, st in enumerate(grp.shards):
    got = st.download()
    bad = np.nonzero(np.any((got != parts[s]).reshape(-1, 1024), axis=1))[0]
    print(s, st.element_count() // 1024, "tiles; mismatching local tiles:", bad[:16].tolist(),
          [grp.layout.decode(s, int(t)) for t in bad[:4]])
