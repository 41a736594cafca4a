"""Repro of test_md_engine_empty_tiles (half-filled box) for one build variant."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2109_09056_b200 as pc
cells = 28
a = (4.0 / 0.8442) ** (1.0 / 3.0)
x = pc.md.fcc_lattice(cells, a)
v = pc.md.initial_velocities(x.shape[0], 1.44, 1.0, 3)
cfg = pc.md.MDConfig(lattice_cells=cells, density=0.4221, temperature=1.44, cutoff=2.5,
                     skin=0.3, rebuild_stride=10, seed=3, steps=0)
drv = pc.md.MDDriver(cfg, state=(x, v))
torch.cuda.synchronize()
print("ok", drv.mode, drv.tile_failures)
