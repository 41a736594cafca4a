"""Work per CTA of the force kernel's static tile assignment (tile t -> CTA
t % grid): sum of rounds over the tile's row-warps; max / mean."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2109_09056_b200 as pc  # noqa: E402

cells = int(sys.argv[1]) if len(sys.argv) > 1 else 64
drv = pc.md.MDDriver(pc.md.MDConfig(lattice_cells=cells, density=0.8442, temperature=1.44,
                                    dt=0.005, cutoff=2.5, skin=0.3, rebuild_stride=20, seed=1,
                                    steps=0))
for s in range(1, 41):
    drv.step(s)
torch.cuda.synchronize()
nt = drv._ntiles
rw0 = drv._rw0.cpu().numpy()
rounds = drv._rounds[: int(rw0[nt])].cpu().numpy().astype(np.int64)
tile_work = np.add.reduceat(rounds, rw0[:-1]) if nt else np.zeros(0)
tile_work[np.diff(rw0) == 0] = 0
grid = min(nt, 148)
cta = np.bincount(np.arange(nt) % grid, weights=tile_work, minlength=grid)
print(f"cells {cells} tiles {nt} per CTA {nt / grid:.1f}  tile work mean {tile_work.mean():.0f} "
      f"std {tile_work.std():.0f}  CTA work max/mean {cta.max() / cta.mean():.3f} "
      f"min/mean {cta.min() / cta.mean():.3f}")
