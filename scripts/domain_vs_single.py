"""Tile build / order / force kernel times of the decomposed engine against
the single-domain engine on the same lattice (one rank, 1x1x1, and 2x2x2 in
process), for an ncu launch list:
  ncu --profile-from-start off --metrics gpu__time_duration.sum --csv \\
      --log-file out.csv python scripts/domain_vs_single.py 64
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2109_09056_b200 as pc  # noqa: E402
from paper_2109_09056_b200.dist import FabricMD  # noqa: E402

cells = int(sys.argv[1]) if len(sys.argv) > 1 else 64
which = sys.argv[2] if len(sys.argv) > 2 else "all"
kw = dict(lattice_cells=cells, density=0.8442, temperature=1.44, dt=0.005, cutoff=2.5,
          skin=0.3, rebuild_stride=20, seed=1, steps=0)
if which in ("all", "single"):
    drv = pc.md.MDDriver(pc.md.MDConfig(**kw), time_phases=False)
    for s in range(1, 21):
        drv.step(s)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    drv._rebuild()
    drv._force_step(kick_dtm=drv._dtm)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("single", drv.n, drv._ntiles)
    del drv
for dims in ((1, 1, 1), (2, 2, 2)):
    if which not in ("all", "x".join(map(str, dims))):
        continue
    fab = FabricMD(pc.md.MDConfig(**kw, rank_dims=dims))
    for s in range(1, 21):
        fab.step(s)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    fab._rebuild_all()
    fab._forces(fab._dtm)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    e = fab.engines[0]
    print("x".join(map(str, dims)), e.n_owned, e.n_total, e._ntiles)
    del fab
