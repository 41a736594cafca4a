import numpy as np, torch, sys
sys.path.insert(0,'.')
import paper_2109_09056_b200 as pc
from paper_2109_09056_b200 import md as mdm
orig = mdm.MDDriver._tile_build
def wrapped(self, cs):
    r = orig(self, cs)
    print("tile_build ->", r, "flags", self.build_flag.cpu().numpy(), "q8", self._q8)
    return r
mdm.MDDriver._tile_build = wrapped
for cells,temp in ((10,3.0),(12,1.44)):
    cfg = pc.md.MDConfig(lattice_cells=cells, density=0.8442, temperature=temp, cutoff=2.5, skin=0.3, rebuild_stride=20, seed=5, steps=0)
    drv = pc.md.MDDriver(cfg)
    print(cells, drv.mode, list(drv._grid.nc))
