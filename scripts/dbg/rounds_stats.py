import numpy as np, torch, sys
sys.path.insert(0,'.')
import paper_2109_09056_b200 as pc
from paper_2109_09056_b200 import _lib
for cells,temp in ((10,3.0),(64,1.44)):
    cfg = pc.md.MDConfig(lattice_cells=cells, density=0.8442, temperature=temp, cutoff=2.5, skin=0.3, rebuild_stride=20, seed=5, steps=0)
    drv = pc.md.MDDriver(cfg)
    print(cells, "mode", drv.mode, "flag", drv.build_flag.cpu().numpy(), "q8", drv._q8, "grid nc", list(drv._grid.nc))
    if drv.mode != "tile": continue
    tot = int(drv._rw0[-1].item())
    R = drv._rounds[:tot].cpu().numpy()
    cnt, _ = drv._tile_rows()
    rowidx = drv._rowidx[:tot*32].cpu().numpy().reshape(tot,32)
    c = cnt.cpu().numpy()
    cc = np.where(rowidx>=0, c[np.maximum(rowidx,0)], 0)
    mx = cc.max(1)
    print(" rows", (rowidx>=0).sum(), "n", drv.n, "rounds/atom", R.sum()*32/drv.n, "maxlen/atom", mx.sum()*32/drv.n, "mean", c.mean(), "R/maxlen", R.sum()/mx.sum(), "active lanes frac", (rowidx>=0).mean())
