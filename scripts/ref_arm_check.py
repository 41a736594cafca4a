"""Rate of the reference package itself vs the oracle port (both numpy, one
thread) on the same 16^3 MD run -- run HERE (needs /root/reference; the GPU box
has no reference).  Shows that the port with the per-cell loop restatement
(oracle.neighbor_pairs_cell_loop, what bench.py's reference arm times) runs at
the reference's own rate; output kept in profiles/r02aw/ref_arm_check.txt."""
import sys
import time

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ".")
import particula.md as ref  # noqa: E402
from oracle import particula_oracle as orc  # noqa: E402

KW = dict(lattice_cells=16, density=0.8442, temperature=1.44, cutoff=2.5, skin=0.3,
          rebuild_stride=20)
STEPS = 25
n = 4 * 16 ** 3
for rep in range(2):
    t = time.perf_counter()
    d = ref.MDDriver(ref.MDConfig(**KW, steps=STEPS))
    t1 = time.perf_counter()
    for s in range(1, STEPS + 1):
        d.step(s)
    t2 = time.perf_counter()
    print(f"reference particula      init {t1 - t:.2f} s  {n * STEPS / (t2 - t1):.3g} atom-steps/s")
    for cl in (False, True):
        t = time.perf_counter()
        o = orc.MDOracle(orc.MDConfig(**KW, steps=STEPS), cell_loop=cl)
        t1 = time.perf_counter()
        for s in range(1, STEPS + 1):
            o.step(s)
        t2 = time.perf_counter()
        print(f"oracle cell_loop={cl!s:5}   init {t1 - t:.2f} s  {n * STEPS / (t2 - t1):.3g} atom-steps/s")
