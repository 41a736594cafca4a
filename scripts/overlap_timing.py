"""In-process cost of the interior/boundary force split:
FabricMD (all ranks on one GPU, sequential) with the force as one pass vs as
interior + boundary tile passes around the ghost refresh.  On one GPU there
is no transfer to hide, so this measures the split's overhead (a second
launch and CTA tail per rank); on N GPUs the interior pass overlaps the
NCCL all-to-all (DistMD)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2109_09056_b200 as pc  # noqa: E402
from paper_2109_09056_b200.dist import FabricMD  # noqa: E402

cells = int(sys.argv[1]) if len(sys.argv) > 1 else 128
dims = tuple(int(t) for t in (sys.argv[2] if len(sys.argv) > 2 else "2,2,2").split(","))
cfg = pc.md.MDConfig(lattice_cells=cells, density=0.8442, temperature=1.44, dt=0.005, cutoff=2.5,
                     skin=0.3, rebuild_stride=20, seed=1, steps=0, rank_dims=dims)
fab = FabricMD(cfg)
for e in fab.engines:
    nt, ni = e._ntiles, int(e._tbounds[1].item())
    print(f"rank {e.rank}: owned {e.n_owned} ghosts {e.n_total - e.n_owned} tiles {nt} "
          f"interior {ni} ({ni / nt:.2f})")
s = 0
for overlap in (False, True, False, True):
    fab.overlap = overlap
    for _ in range(5):
        s += 1
        fab.step(s)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # steps between rebuilds only (the split applies to refresh steps)
    while (s + 1) % cfg.rebuild_stride == 0:
        s += 1
        fab.step(s)
    k = 0
    a.record()
    while k < 15:
        s += 1
        if s % cfg.rebuild_stride == 0:
            fab.step(s)
            continue
        fab.step(s)
        k += 1
    b.record()
    b.synchronize()
    print(f"overlap={overlap}: {a.elapsed_time(b) / 15:.3f} ms per step (8 ranks in sequence, "
          f"incl. any rebuild in the window)")
