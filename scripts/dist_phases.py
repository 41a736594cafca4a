"""Phase times of the decomposed engine with one rank (gloo): where the
per-rebuild overhead over MDDriver goes."""
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2109_09056_b200 as pc  # noqa: E402
from paper_2109_09056_b200.dist import DistMD  # noqa: E402

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29537")
dist.init_process_group("gloo", rank=0, world_size=1)
kw = dict(lattice_cells=64, density=0.8442, temperature=1.44, dt=0.005, cutoff=2.5, skin=0.3,
          rebuild_stride=20, seed=1, steps=0)
drv = DistMD(pc.md.MDConfig(**kw), time_phases=True)
for s in range(1, 21):
    drv.step(s)
torch.cuda.synchronize()
drv.engine.timer.reset()
t0 = time.perf_counter()
for s in range(21, 121):
    drv.step(s)
torch.cuda.synchronize()
wall = time.perf_counter() - t0
tot = drv.engine.timer.resolve()
print(f"100 steps wall {wall * 1e3:.1f} ms; device phase totals (ms):",
      {k: round(v * 1e3, 2) for k, v in tot.items()})
# host time of one rebuild
torch.cuda.synchronize()
t0 = time.perf_counter()
drv._rebuild_all()
torch.cuda.synchronize()
print(f"one rebuild wall {(time.perf_counter() - t0) * 1e3:.2f} ms")
dist.destroy_process_group()
