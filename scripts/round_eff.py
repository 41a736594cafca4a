"""Lane efficiency of the tile lists: sum of row lengths / (32 * sum of rounds)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2109_09056_b200 as pc  # noqa: E402

cells = int(sys.argv[1]) if len(sys.argv) > 1 else 64
drv = pc.md.MDDriver(pc.md.MDConfig(lattice_cells=cells, density=0.8442, temperature=1.44,
                                    dt=0.005, cutoff=2.5, skin=0.3, rebuild_stride=20, seed=1,
                                    steps=0))
for s in range(1, 201):
    drv.step(s)
torch.cuda.synchronize()
cnt, _ = drv._tile_rows()
nrw = int(drv._rw0[drv._ntiles].item())
rounds = drv._rounds[:nrw].double()
tot = float(cnt.double().sum().item())
print(f"rows {drv.n} row-warps {nrw} mean count {tot / drv.n:.2f} "
      f"sum rounds*32 {float(rounds.sum()) * 32:.4g} efficiency {tot / (float(rounds.sum()) * 32):.3f}")
c = cnt.double()
print(f"count std {float(c.std()):.2f} min {int(c.min())} max {int(c.max())}")
# ideal: rows sorted by count within each tile
rw0 = drv._rw0.cpu()
ri = drv._rowidx[: nrw * 32].view(nrw, 32).cpu()
cc = cnt.cpu()
srt_rounds = 0
import numpy as np
for t in range(drv._ntiles):
    a, b = int(rw0[t]), int(rw0[t + 1])
    rows = ri[a:b].reshape(-1)
    rows = rows[rows >= 0]
    v = np.sort(cc[rows.long()].numpy())[::-1]
    for g in range(0, len(v), 32):
        srt_rounds += v[g]
print(f"sorted-within-tile efficiency {tot / (srt_rounds * 32):.3f}")
