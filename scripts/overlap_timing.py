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
R = cfg.rebuild_stride
for overlap in (False, True, False, True):
    fab.overlap = overlap
    # advance to just after a rebuild, then time R - 1 refresh steps (the
    # split applies to them; rebuild steps run the force in one pass)
    while True:
        s += 1
        fab.step(s)
        if s % R == 0:
            break
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(R - 1):
        s += 1
        fab.step(s)
    b.record()
    b.synchronize()
    print(f"overlap={overlap}: {a.elapsed_time(b) / (R - 1):.3f} ms per refresh step "
          f"({len(fab.engines)} ranks in sequence on one GPU)")
