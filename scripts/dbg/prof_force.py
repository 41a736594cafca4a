import sys, ctypes, torch
sys.path.insert(0, '.')
import paper_2109_09056_b200 as pc
from paper_2109_09056_b200 import _lib
lib = ctypes.CDLL(_lib.LIB_PATH)
buf = (ctypes.c_ulonglong * 8)()
cfg = pc.md.MDConfig(lattice_cells=64, density=0.8442, temperature=1.44, cutoff=2.5, skin=0.3, rebuild_stride=20, seed=1, steps=0)
drv = pc.md.MDDriver(cfg, time_phases=False)
for s in range(1, 21): drv.step(s)
torch.cuda.synchronize(); lib.pc_tile_prof(buf, 1)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for s in range(21, 40): drv.step(s)
e1.record(); torch.cuda.synchronize()
lib.pc_tile_prof(buf, 0)
ms = e0.elapsed_time(e1)
n = buf[3]
print("row-warps", n, "per step", n / 19)
tot = ms * 1e-3 * 1.965e9 * 148 * 32 / 19   # warp-cycles per step (32 warps/SM)
print("avg cycles per row-warp: prologue %.0f spin %.0f  mbar %.0f  compute %.0f release %.0f stores %.0f partials %.0f" % (buf[4] / n, buf[0] / n, buf[1] / n, buf[2] / n, buf[6] / n, buf[7] / n, buf[5] / n))
print("fraction of warp-time per step: spin %.3f mbar %.3f compute %.3f" % (buf[0] / 19 / tot, buf[1] / 19 / tot, buf[2] / 19 / tot))
