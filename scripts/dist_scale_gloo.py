"""bench.py --gpus 2's DistMD construction at full size (2 x 64^3 cells,
local_init, rank_dims 2x1x1) with two processes sharing one GPU over gloo:
checks the decomposed tile path runs at scale (ghost counts, modes, energy
drift) where NCCL cannot be used (one GPU)."""
import os
import sys
import time

import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def worker(rank, world, port, steps):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_2109_09056_b200 as pc
    from paper_2109_09056_b200.dist import DistMD, rank_dims_for
    cfg = pc.md.MDConfig(lattice_cells=64, density=0.8442, temperature=1.44, dt=0.005, cutoff=2.5,
                         skin=0.3, rebuild_stride=20, seed=1, steps=steps)
    dims = rank_dims_for(world)
    cfg.rank_dims = dims
    drv = DistMD(cfg, cells=[64 * d for d in dims], local_init=True)
    e = drv.engine
    e0 = drv.diagnostics()["E_total"]
    t0 = time.perf_counter()
    for s in range(1, steps + 1):
        drv.step(s)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    e1 = drv.diagnostics()["E_total"]
    owned = torch.tensor([e.n_owned], dtype=torch.int64)
    dist.all_reduce(owned)
    if rank == 0:
        print(f"n {drv.n} owned-sum {int(owned)} mode {e.mode} ghosts {e.n_total - e.n_owned} "
              f"tile_failures {e.tile_failures} rebuilds {e.rebuilds} mean_nbr "
              f"{e.mean_neighbors():.2f} drift {abs(e1 - e0) / abs(e0):.2e} "
              f"{steps} steps {dt:.1f}s (gloo host-staged)", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    mp.spawn(worker, args=(2, 29561, int(sys.argv[1]) if len(sys.argv) > 1 else 45), nprocs=2)
