"""One steady-state rebuild (migrate + halo + sort/build, 8 in-process ranks of
a 2x2x2 fabric) inside a profiler range, for an ncu launch list:

  ncu --profile-from-start off --metrics gpu__time_duration.sum --csv \\
      --log-file gpurun_out/rebuild_launches.csv python scripts/rebuild_launches.py 128
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2109_09056_b200 as pc  # noqa: E402
from paper_2109_09056_b200.dist import FabricMD  # noqa: E402

cells = int(sys.argv[1]) if len(sys.argv) > 1 else 128
cfg = pc.md.MDConfig(lattice_cells=cells, density=0.8442, temperature=1.44, dt=0.005, cutoff=2.5,
                     skin=0.3, rebuild_stride=20, seed=1, steps=0, rank_dims=(2, 2, 2))
fab = FabricMD(cfg)
for s in range(1, 21):
    fab.step(s)
torch.cuda.synchronize()
torch.cuda.profiler.start()
fab._rebuild_all()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
