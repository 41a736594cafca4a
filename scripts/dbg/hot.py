import sys, time, torch
sys.path.insert(0, '.')
import paper_2109_09056_b200 as pc
from paper_2109_09056_b200 import md as mdm
orig = mdm.MDDriver._tile_build
def wrapped(self, cs):
    r = orig(self, cs)
    if not r: print("tile_build -> False flags", self.build_flag.cpu().numpy(), "q8", self._q8)
    return r
mdm.MDDriver._tile_build = wrapped
cfg = pc.md.MDConfig(lattice_cells=64, density=0.8442, temperature=3.0, cutoff=2.5, skin=0.3, rebuild_stride=5, seed=1, steps=0)
drv = pc.md.MDDriver(cfg, time_phases=True)
for s in range(1, 101):
    drv.step(s)
torch.cuda.synchronize()
drv.timings = {k: 0.0 for k in drv.timings}
t0 = time.time()
for s in range(101, 301):
    drv.step(s)
torch.cuda.synchronize()
print("mode", drv.mode, "q8", drv._q8, "wall per step ms", (time.time() - t0) / 200 * 1e3)
print({k: round(v / 200 * 1e3, 4) for k, v in drv.timings.items()})
print("mean nbr", drv.mean_neighbors())
