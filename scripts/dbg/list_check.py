"""Build the tile lists of the half-filled-box case and report list entries
that are not slot byte offsets (not multiples of 8) within each row-warp's
rounds: which row-warp / lane / round / tile."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
import paper_2109_09056_b200 as pc
cells = int(sys.argv[1]) if len(sys.argv) > 1 else 28
a = (4.0 / 0.8442) ** (1.0 / 3.0)
x = pc.md.fcc_lattice(cells, a)
v = pc.md.initial_velocities(x.shape[0], 1.44, 1.0, 3)
cfg = pc.md.MDConfig(lattice_cells=cells, density=0.4221, temperature=1.44, cutoff=2.5,
                     skin=0.3, rebuild_stride=3, seed=3, steps=0)
os.environ["PC_TILE_ORDER"] = "0"
drv = pc.md.MDDriver.__new__(pc.md.MDDriver)
try:
    pc.md.MDDriver.__init__(drv, cfg, state=(x, v))
except Exception as e:
    print("init raised", type(e).__name__, str(e)[:100])
torch.cuda.synchronize()
rounds = drv._rounds.cpu().numpy()
rw0 = drv._rw0.cpu().numpy()
nt = drv._ntiles
nrw = int(rw0[nt])
q8 = drv._q8
lst = drv._tlist.view(torch.int16).cpu().numpy().view(np.uint16)
rowidx = drv._rowidx.cpu().numpy()
bad = 0
for rw in range(nrw):
    R = int(rounds[rw])
    if R <= 0:
        continue
    for lane in range(32):
        for r in range(R):
            val = int(lst[((rw * q8 + r // 8) * 32 + lane) * 8 + r % 8])
            if val % 8:
                bad += 1
                if bad <= 10:
                    t = int(np.searchsorted(rw0[:nt + 1], rw, side="right") - 1)
                    print(f"rw {rw} tile {t} lane {lane} r {r}/{R} val {val} row {rowidx[rw*32+lane]}")
print("row-warps", nrw, "bad entries", bad, "flags", drv.build_flag.cpu().numpy()[:3])
