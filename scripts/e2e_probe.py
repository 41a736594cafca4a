"""End-to-end leg breakdown at C3: MDDriver construction (H2D + allocations +
sort + first list + first force) vs the step loop, with events, repeated in
one process -- after empty_cache (fresh cudaMallocs, bench.py's e2e leg) and
with a warm caching allocator."""
import sys
import time

sys.path.insert(0, ".")
import torch
import paper_2109_09056_b200 as pc

kw = dict(lattice_cells=128, density=0.8442, temperature=1.44, cutoff=2.5, skin=0.3,
          rebuild_stride=20, seed=12345)
n = 4 * 128 ** 3
a = (4.0 / kw["density"]) ** (1.0 / 3.0)
x = torch.as_tensor(pc.md.fcc_lattice(128, a)).pin_memory()
v = torch.as_tensor(pc.md.initial_velocities(n, 1.44, 1.0, kw["seed"])).pin_memory()
for rep in range(4):
    if rep < 2:
        torch.cuda.empty_cache()
    torch.cuda.synchronize()
    cfg = pc.md.MDConfig(**kw, steps=200)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    t0 = time.perf_counter()
    ev[0].record()
    drv = pc.md.MDDriver(cfg, state=(x, v), time_phases=False)
    ev[1].record()
    t1 = time.perf_counter()
    for s in range(1, 201):
        drv.step(s)
    ev[2].record()
    ev[2].synchronize()
    t2 = time.perf_counter()
    print(f"rep {rep} ({'empty_cache' if rep < 2 else 'warm allocator'}): setup "
          f"{ev[0].elapsed_time(ev[1]):.1f} ms (host {1e3 * (t1 - t0):.1f}), 200 steps "
          f"{ev[1].elapsed_time(ev[2]):.1f} ms (host {1e3 * (t2 - t1):.1f}), mode {drv.mode}",
          flush=True)
    del drv
