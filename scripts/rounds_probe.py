"""Longest neighbour rows of the tile lists (rounds per row-warp = its longest
row) at C3 for T = 1.44 and the hot T = 3.0, over several rebuilds: the
headroom of the build's per-lane hit capacity (kHitCap)."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402
import paper_2109_09056_b200 as pc  # noqa: E402

for temp, rb in ((1.44, 20), (3.0, 5)):
    cfg = pc.md.MDConfig(lattice_cells=128, density=0.8442, temperature=temp, cutoff=2.5,
                         skin=0.3, rebuild_stride=rb, steps=100)
    drv = pc.md.MDDriver(cfg, time_phases=False)
    worst = 0
    hist = torch.zeros(129, dtype=torch.int64)
    for s in range(1, 101):
        drv.step(s)
        if s % rb == 0:
            nrw = int(drv._rw0[-1].item()) if hasattr(drv, "_rw0") else drv._rounds.numel()
            r = drv._rounds[:nrw].to(torch.int64).clamp(0, 128).cpu()
            worst = max(worst, int(r.max()))
            hist += torch.bincount(r, minlength=129)
    tail = {k: int(hist[k:].sum()) for k in (88, 92, 96, 100, 104, 108)}
    print(f"T={temp} rebuild {rb}: mode {drv.mode}, longest row-warp {worst} rounds, "
          f"row-warps with >= k rounds {tail} of {int(hist.sum())}", flush=True)
