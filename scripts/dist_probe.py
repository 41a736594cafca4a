"""Per-step cost of the decomposed engine on one GPU: DistMD with one rank
(gloo, no peers) and FabricMD 2x1x1 (two ranks in-process, ghosts), vs the
single-domain MDDriver; phase times from the engines' CUDA-event timers."""
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2109_09056_b200 as pc                       # noqa: E402
from paper_2109_09056_b200.dist import DistMD, FabricMD  # noqa: E402

cells = int(sys.argv[1]) if len(sys.argv) > 1 else 64
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
kw = dict(lattice_cells=cells, density=0.8442, temperature=1.44, dt=0.005, cutoff=2.5,
          skin=0.3, rebuild_stride=20, seed=1, steps=steps)


def timed(drv, label, n):
    for s in range(1, 21):
        drv.step(s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for s in range(21, 21 + steps):
        drv.step(s)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / steps
    print(f"{label:28s} {ms:.4f} ms/step  {n / ms / 1e6:.3e} atom-steps/s", flush=True)


os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
dist.init_process_group("gloo", rank=0, world_size=1)
drv = pc.md.MDDriver(pc.md.MDConfig(**kw))
timed(drv, "MDDriver (tile, fused)", drv.n)
del drv
d1 = DistMD(pc.md.MDConfig(**kw))
print("DistMD x1 mode", d1.engine.mode, "tile failures", d1.engine.tile_failures)
timed(d1, "DistMD x1 (gloo)", d1.n)
del d1
fab = FabricMD(pc.md.MDConfig(**dict(kw, rank_dims=(2, 1, 1))))
print("Fabric 2x1x1 modes", [e.mode for e in fab.engines],
      "ghosts", [e.n_total - e.n_owned for e in fab.engines])
timed(fab, "FabricMD 2x1x1 (both ranks)", fab.n)
fab = FabricMD(pc.md.MDConfig(**dict(kw, rank_dims=(2, 2, 2))))
print("Fabric 2x2x2 ghosts", [e.n_total - e.n_owned for e in fab.engines][:2])
timed(fab, "FabricMD 2x2x2 (all ranks)", fab.n)
dist.destroy_process_group()
