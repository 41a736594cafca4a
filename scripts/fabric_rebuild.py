"""Wall time of one rebuild (migrate + halo + sort/build, all ranks) of the
in-process 2x2x2 fabric at full size: the per-peer host work of the
decomposed engine's rebuild."""
import os
import sys
import time

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
for e in fab.engines:
    e._time = True
    e.timer.reset()
t0 = time.perf_counter()
for s in range(21, 41):
    fab.step(s)
torch.cuda.synchronize()
wall = time.perf_counter() - t0
tot = {}
for e in fab.engines:
    for k, v in e.timer.resolve().items():
        tot[k] = tot.get(k, 0.0) + v
print(f"20 steps (1 rebuild) of 8 ranks: wall {wall * 1e3:.1f} ms; summed phase ms:",
      {k: round(v * 1e3, 2) for k, v in tot.items()})
torch.cuda.synchronize()
t0 = time.perf_counter()
fab._rebuild_all()
torch.cuda.synchronize()
print(f"one rebuild (8 ranks) wall {(time.perf_counter() - t0) * 1e3:.1f} ms")
for e in fab.engines:
    e.timer.reset()
torch.cuda.synchronize()
fab._rebuild_all()
torch.cuda.synchronize()
tot = {}
for e in fab.engines:
    for k, v in e.timer.resolve().items():
        tot[k] = tot.get(k, 0.0) + v
print("rebuild phases summed over 8 ranks (ms):", {k: round(v * 1e3, 2) for k, v in tot.items()})
import cProfile, pstats  # noqa: E402,E401
pr = cProfile.Profile()
pr.enable()
fab._rebuild_all()
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("cumulative").print_stats(18)
