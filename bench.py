#!/usr/bin/env python
"""Benchmark of the LJ short-range MD hot path (BASELINE.json metric:
atom-timesteps/sec, LJ rc = 2.5 sigma, at 1/2/4/8 B200, plus % of the HBM
roofline).

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]
                    [--scaling strong|weak] [--cells C]

Workload (BASELINE configs[2], the configuration the metric is quoted on):
fcc 128^3 cells = 8,388,608 atoms, rho = 0.8442, T = 1.44, rc = 2.5,
skin 0.3, neighbor rebuild every 20 steps, full neighbor list.  At N = 1 the
whole system runs on one B200.  Under torchrun (N > 1):

* ``--scaling strong`` (default, configs[2]): the same 8.4M-atom system
  decomposed over rank_dims 2x1x1 / 2x2x1 / 2x2x2;
* ``--scaling weak`` (configs[4]): a 128^3-cell block (8.4M atoms) per GPU,
  67M atoms at N = 8.

One rank per GPU, tile path on every rank's local grid, ghost refresh every
step and migrate + halo rebuild every 20 steps over NCCL
(paper_2109_09056_b200.dist).  A "step" is one velocity-Verlet
MD step (integrate, rebuild on schedule, force + final kick).  Timing: W
untimed warm-up steps, then exactly K steps between CUDA events on the
launching stream, barrier + synchronize on both sides, max over ranks.  The
working set (Verlet list ~1.4 GB at 8.4M atoms) exceeds the 126 MB L2, so no
explicit L2 flush is done between steps.

``--impl reference`` times the CPU oracle port of the reference
(oracle/particula_oracle.py: numpy, single-threaded like the reference) on a
bounded sample of the same workload (rank 0 only).
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "atom-timesteps/sec (LJ, rc=2.5σ)"
UNIT = "atom-steps/s"

# SURVEY §8(d) algorithmic bytes per atom (FP64 x/v, 4-B index per list
# entry, FP64 force): K6 full-list force 4k + 8 + 24 + 12, K8 integrate 168,
# rebuild (K1 28 + K3 112 + K4/5 24 + 4k + 8) per rebuild
def k6_bytes(k):
    return 4.0 * k + 8 + 24 + 12


def build_bytes(k):
    return 24.0 + 4.0 * k + 8


def rebuild_bytes(k):
    return 28.0 + 112.0 + build_bytes(k)


def step_bytes(k, rebuild):
    return k6_bytes(k) + 168.0 + rebuild_bytes(k) / rebuild


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--cells", type=int, default=128,
                    help="fcc cells per axis: of the global system (strong) or per GPU (weak)")
    ap.add_argument("--scaling", choices=["strong", "weak"], default="strong")
    ap.add_argument("--temperature", type=float, default=1.44)
    ap.add_argument("--rebuild", type=int, default=20)
    ap.add_argument("--list", choices=["full", "half"], default="full")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=0,
                    help="steps of the end-to-end leg (0: max(K, 200))")
    ap.add_argument("--path", choices=["tile", "sell"], default="tile",
                    help="MD force/list path: TMA-staged tile rounds (default) or the "
                         "per-particle SELL list")
    ap.add_argument("--gather", choices=["planar", "pos4"], default="planar",
                    help="SELL force-kernel neighbor gather layout")
    ap.add_argument("--transport", choices=["nccl", "p2p"], default="nccl",
                    help="N > 1: per-step ghost refresh as one NCCL all_to_all_single "
                         "(default) or direct peer-memory stores between the ranks' "
                         "processes (dist.P2PTransport: CUDA IPC windows over NVLink)")
    return ap.parse_args()


def make_transport(args):
    """The N-rank transport: None (DistMD's NCCLTransport) or P2PTransport."""
    if getattr(args, "transport", "nccl") != "p2p":
        return None
    from paper_2109_09056_b200.dist import P2PTransport
    return P2PTransport()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def md_kwargs(args, cells):
    return dict(lattice_cells=cells, density=0.8442, temperature=args.temperature, dt=0.005,
                cutoff=2.5, skin=0.3, rebuild_stride=args.rebuild, seed=1)


def global_cells(args, world):
    """fcc cells per axis of the global system (strong: fixed; weak: grows
    with the rank grid)."""
    if world == 1 or args.scaling == "strong":
        return [args.cells] * 3
    from paper_2109_09056_b200.dist import rank_dims_for
    return [args.cells * d for d in rank_dims_for(world)]


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def _force_capture():
    p = os.path.join(ROOT, "profiles", "force_traffic.json")
    try:
        with open(p) as f:
            return json.load(f), p
    except Exception:
        return None, p


def static_traffic():
    """ncu DRAM read+write per launch per atom of the force kernel, from the
    committed capture (an ncu replay cannot run inside the timed region)."""
    d, p = _force_capture()
    if d is None:
        return None, None
    return float(d["bytes_per_launch_per_atom"]), d.get("source", p)


def static_build_capture():
    """ncu warp instructions and DRAM bytes per atom of one rebuild's build +
    order kernels (profiles/build_traffic.json)."""
    p = os.path.join(ROOT, "profiles", "build_traffic.json")
    try:
        with open(p) as f:
            return json.load(f)
    except (OSError, ValueError):
        return None


def static_inst_per_atom():
    """ncu warp instructions per atom of one force launch (same capture)."""
    d, _ = _force_capture()
    return None if d is None else d.get("warp_instructions_per_atom")


class ClockSampler:
    """NVML sampling of SM clock + throttle reasons during the timed region."""

    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4,
        "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
        "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
        "display_clock_setting": 0x100,
    }

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self._nv.nvmlDeviceGetClockInfo(self._h,
                                                                    self._nv.NVML_CLOCK_SM))
                r = self._nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for name, bit in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self._nv is not None:
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._nv is not None:
            self._t.join()

    def summary(self):
        import statistics
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons - {"gpu_idle"}), "samples": len(self.samples)}


def cpu_oracle_rate(kw, cells, steps):
    """Oracle port of the reference MD (numpy, 1 thread) on a bounded sample."""
    from oracle import particula_oracle as orc
    cfg = orc.MDConfig(**dict(kw, lattice_cells=cells, steps=steps))
    drv = orc.MDOracle(cfg, cell_loop=True)
    t0 = time.perf_counter()
    for s in range(1, steps + 1):
        drv.step(s)
    dt = time.perf_counter() - t0
    return drv.n * steps / dt, drv.n, dt


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    kw = md_kwargs(args, args.cells)
    gc = global_cells(args, world)
    # size the sample so warmup+steps finish in ~2 minutes of CPU time; at
    # most 48^3 cells (442k atoms): the port's vectorised pair arrays and its
    # setup (lattice, first list and force) grow with the sample too
    probe_rate, _, _ = cpu_oracle_rate(kw, 8, 2)
    budget_atoms = probe_rate * 120.0 / max(1, args.steps + args.warmup)
    cells = max(6, min(gc[0], 48, int((budget_atoms / 4) ** (1 / 3))))
    from oracle import particula_oracle as orc
    cfg = orc.MDConfig(**dict(kw, lattice_cells=cells, steps=args.steps))
    drv = orc.MDOracle(cfg, cell_loop=True)
    for s in range(1, args.warmup + 1):
        drv.step(s)
    t0 = time.perf_counter()
    for s in range(args.warmup + 1, args.warmup + args.steps + 1):
        drv.step(s)
    dt = time.perf_counter() - t0
    value = drv.n * args.steps / dt
    ncpu = os.cpu_count()
    sample = (f"oracle port of the reference MD (numpy, 1 thread: the reference is "
              f"single-threaded; 1 of {ncpu} host cores; neighbor lists through the "
              f"reference's per-cell loop) on fcc {cells}^3 = {drv.n} atoms, "
              f"same rho/T/rc/skin/rebuild as the fcc {'x'.join(map(str, gc))} workload")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": 0, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dt * 1e3 / args.steps, "higher_is_better": True,
            "scaling": args.scaling if world > 1 else "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"LJ fcc {'x'.join(map(str, gc))} "
                                   f"({4 * gc[0] * gc[1] * gc[2]} atoms)",
                       "sample_atoms": drv.n, "rebuild_stride": args.rebuild, "list": "full",
                       "host_cores": ncpu},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "port",
                             "host_cores": ncpu, "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def _avg_ms(pairs):
    import numpy as np
    return float(np.mean([a.elapsed_time(b) for a, b in pairs])) if pairs else None


def _sum_ms(pairs):
    return float(sum(a.elapsed_time(b) for a, b in pairs))


def _sm_count():
    import torch
    return torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    torch.cuda.set_device(local % max(1, torch.cuda.device_count()))
    if world > 1:
        # NCCL over NVLink; PC_BENCH_BACKEND=gloo runs the same N-rank path with
        # several ranks on one GPU (tests/test_bench_contract.py)
        dist.init_process_group(os.environ.get("PC_BENCH_BACKEND", "nccl"))
    import paper_2109_09056_b200 as pc
    from paper_2109_09056_b200 import _lib

    gc = global_cells(args, world)
    kw = md_kwargs(args, gc[0])
    cfg = pc.md.MDConfig(**kw, steps=args.steps)
    if world > 1:
        # spatial decomposition, ghost halo over NCCL (paper_2109_09056_b200.dist)
        from paper_2109_09056_b200.dist import DistMD, rank_dims_for
        dims = rank_dims_for(world)
        cfg.rank_dims = dims
        drv = DistMD(cfg, cells=gc, local_init=True, transport=make_transport(args))
        eng = drv.engine
    else:
        drv = pc.md.MDDriver(cfg, time_phases=False, planar_gather=args.gather == "planar",
                             tile=args.path == "tile", half_list=args.list == "half")
        eng = drv
    n_global = int(drv.n)
    W, K = args.warmup, args.steps
    for s in range(1, W + 1):
        drv.step(s)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    lib = _lib.load()
    eng.force_events = []
    eng.rebuild_events = []
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = lib.pc_launch_count()
    with ClockSampler(local) as clk:
        ev0.record()
        for s in range(W + 1, W + K + 1):
            drv.step(s)
        ev1.record()
        ev1.synchronize()
    torch.cuda.synchronize()
    launches = lib.pc_launch_count() - launches0
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.barrier()
        ms = float(t.item())
    value = n_global * K / (ms * 1e-3)
    diag = drv.diagnostics()
    # force time per step: one launch per step on one GPU; two (interior +
    # boundary tiles around the ghost refresh) on a decomposed rank
    n_force = len(eng.force_events)
    force_ms = _sum_ms(eng.force_events) / K
    rb = eng.rebuild_events
    build_ms = _avg_ms([(e[1], e[2]) for e in rb])
    rebuild_ms = _avg_ms([(e[0], e[2]) for e in rb])
    eng.force_events = None
    eng.rebuild_events = None
    n_local = int(eng.n_owned) if world > 1 else n_global
    kmean = eng.mean_neighbors()
    mode = getattr(eng, "mode", "sell")
    peak, peak_kind = measured_peak()
    # dominant kernel: the force pass.  Algorithmic bytes per launch = the
    # §8(d) K6 figure x the atoms the launch processes (this rank's owned
    # atoms); the fused final kick / next integrate are NOT counted
    b_force = k6_bytes(kmean)
    if mode == "half":
        kname = "lj_force_sell_half_kernel (Newton-3, FP64 atomics; kick separate)"
    elif mode == "tile":
        kname = ("tile_force_kernel (TMA-staged smem neighbourhood, 16-bit slot rounds, "
                 "fused final kick + next integrate)")
    else:
        kname = "lj_force_sell_kernel (+fused final kick)"
    achieved = n_local * b_force / (force_ms * 1e-3) / 1e9
    tr_atom, tr_src = static_traffic()
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak,
                "traffic": None if tr_atom is None else tr_atom * n_local,
                "traffic_source": None if tr_src is None else
                f"static: ncu DRAM read+write per launch per atom from {tr_src}, x {n_local} "
                f"atoms (an ncu replay cannot run inside the timed region)",
                "kernel": kname, "bytes_per_atom": b_force,
                "bytes_model": "SURVEY §8(d) K6: 4k + 8 + 24 + 12, k = mean list length",
                "peak_kind": peak_kind, "avg_launch_us": force_ms * 1e3,
                "force_launches": n_force, "per": "force pass per step (sum of its launches)",
                "limiter": "not HBM: instruction issue and shared-memory wavefronts of the "
                           "exact FP64 pair test (ncu, profiles/, DESIGN.md §5)"}
    # the force kernel is instruction-issue bound, not HBM bound: its issue
    # roofline = warp instructions per launch (ncu count per atom x atoms)
    # / live launch time, against 4 warp instructions per clock per SM
    ipa = static_inst_per_atom()
    if ipa is not None and mode == "tile":
        sm_clk = (clk.summary().get("sm_mhz") or 1965.0) * 1e6
        peak_i = _sm_count() * 4 * sm_clk
        ach_i = ipa * n_local / (force_ms * 1e-3)
        roofline["issue"] = {"achieved_warp_inst_per_s": ach_i, "peak_warp_inst_per_s": peak_i,
                             "frac": ach_i / peak_i,
                             "source": "static: ncu smsp__inst_executed.sum per atom "
                                       "(profiles/force_traffic.json) x atoms / live launch "
                                       "time; peak = SMs x 4 schedulers x median SM clock"}
    per_gpu_rate = value / world
    b_step = step_bytes(kmean, args.rebuild)
    roofline_step = {"bound": "hbm", "achieved": per_gpu_rate * b_step / 1e9, "peak": peak,
                     "unit": "GB/s", "frac": per_gpu_rate * b_step / 1e9 / peak,
                     "bytes_per_atom_step": b_step,
                     "bytes_model": "SURVEY §8(d): K6 + K8 168 + rebuild/R"}
    roofline_build = None
    if build_ms:
        bb = build_bytes(kmean)
        roofline_build = {"bound": "hbm", "kernel": "tile_build_kernel + tile_order_kernel"
                          if mode == "tile" else "nbr build (SELL)",
                          "achieved": n_local * bb / (build_ms * 1e-3) / 1e9, "peak": peak,
                          "unit": "GB/s",
                          "frac": n_local * bb / (build_ms * 1e-3) / 1e9 / peak,
                          "bytes_per_atom": bb, "bytes_model": "SURVEY §8(d) K4/5: 24 + 4k + 8",
                          "avg_launch_us": build_ms * 1e3,
                          "rebuild_us": rebuild_ms * 1e3, "rebuilds": len(rb)}
        bc = static_build_capture()
        if bc is not None and mode == "tile":
            # like the force kernel, the build is not HBM bound: its issue
            # roofline from the committed ncu instruction count
            sm_clk = (clk.summary().get("sm_mhz") or 1965.0) * 1e6
            peak_i = _sm_count() * 4 * sm_clk
            ach_i = bc["warp_instructions_per_atom"] * n_local / (build_ms * 1e-3)
            roofline_build["issue"] = {
                "achieved_warp_inst_per_s": ach_i, "peak_warp_inst_per_s": peak_i,
                "frac": ach_i / peak_i,
                "traffic_bytes_per_atom": bc["dram_bytes_per_atom"],
                "source": "static: ncu smsp__inst_executed.sum of the build + order kernels "
                          "per atom (profiles/build_traffic.json) x atoms / live build time"}

    # the device leg's engine goes back to PyTorch's caching allocator, so the
    # end-to-end leg (a fresh engine through the public API) allocates from a
    # warm pool, as a process calling run_md repeatedly does (after an
    # empty_cache the leg's setup paid ~20 ms of fresh cudaMallocs and varied
    # run to run: profiles/r02aw/e2e_probe.txt)
    del drv, eng
    e2e = None
    if not args.no_e2e and world == 1:
        e2e = run_e2e(pc, kw, args.e2e_steps or max(K, 200),
                      dict(tile=args.path == "tile", half_list=args.list == "half",
                           planar_gather=args.gather == "planar"))
    elif not args.no_e2e:
        e2e = run_e2e_dist(pc, kw, args.e2e_steps or max(K, 100), gc, world, args)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, natoms, secs = cpu_oracle_rate(kw, 16, 20)
        cpu = {"value": rate, "unit": UNIT, "cores": 1, "kind": "port",
               "host_cores": os.cpu_count(),
               "sample": f"oracle port (numpy, 1 thread, as the single-threaded reference; "
                         f"1 of {os.cpu_count()} host cores; neighbor lists through the "
                         f"reference's per-cell loop) 20 MD steps on fcc 16^3 = "
                         f"{natoms} atoms, same rho/T/rc/skin/rebuild ({secs:.1f} s)"}
    if rank == 0:
        shape = "x".join(map(str, gc))
        if world == 1:
            workload = (f"LJ fcc {shape} ({n_global} atoms) on one GPU, rho=0.8442 "
                        f"T={args.temperature} rc=2.5 skin=0.3 rebuild={args.rebuild} "
                        f"{args.list} list")
        else:
            workload = (f"LJ fcc {shape} ({n_global} atoms) over {world} GPUs "
                        f"({args.scaling} scaling, ~{n_global // world} atoms per GPU), "
                        f"rho=0.8442 T={args.temperature} rc=2.5 skin=0.3 "
                        f"rebuild={args.rebuild} {args.list} list")
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
                "warmup": W, "ms_per_step": ms / K, "higher_is_better": True,
                "scaling": args.scaling if world > 1 else "strong", "vs_baseline": None,
                "dtype": "f64+f32(LJ magnitude)",
                "data": "synthetic fcc lattice, seeded Gaussian velocities",
                "config": {"workload": workload, "global_atoms": n_global,
                           "atoms_per_gpu": n_global / world, "rank0_owned_atoms": n_local,
                           "parallelism": f"domain x{world}" if world > 1 else "single domain",
                           "halo_transport": args.transport if world > 1 else None,
                           "l2": "working set > L2 (Verlet list ~170 B/atom), no flush",
                           "mean_neighbors": kmean},
                "roofline": roofline, "roofline_step": roofline_step,
                "roofline_build": roofline_build,
                "gpu_launches": int(launches),
                "clocks": clk.summary(),
                "e2e": e2e, "cpu_baseline": cpu,
                "check": {"E_total": diag["E_total"], "temperature": diag["temperature"]}}
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def run_e2e(pc, kw, steps, driver_options=None):
    """Same metric through the public API with host buffers: pinned host x, v
    uploaded inside the timed region, then `pc.md.run_md` (the reference's
    run_md contract: every step's KE/PE/E_total/temperature row, returned to
    the host at the end -- 40 B of diagnostics per step)."""
    import torch
    n = 4 * kw["lattice_cells"] ** 3
    a = (4.0 / kw["density"]) ** (1.0 / 3.0)
    x = torch.as_tensor(pc.md.fcc_lattice(kw["lattice_cells"], a)).pin_memory()
    v = torch.as_tensor(pc.md.initial_velocities(n, kw["temperature"], 1.0,
                                                 kw["seed"])).pin_memory()
    cfg = pc.md.MDConfig(**kw, steps=steps)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rows, _ = pc.md.run_md(cfg, state=(x, v), time_phases=False, **(driver_options or {}))
    e1.record()
    e1.synchronize()
    assert len(rows) == steps + 1
    ms = e0.elapsed_time(e1)
    return {"value": n * steps / (ms * 1e-3), "unit": UNIT,
            "h2d_bytes_per_step": n * 48 / steps, "d2h_bytes_per_step": 40,
            "steps": steps, "includes": "H2D of x, v + engine setup (sort, list build, first "
                                        "force) + the steps + run_md's per-step diagnostics "
                                        "rows (D2H at the end)"}


def run_e2e_dist(pc, kw, steps, cells, world, args=None):
    """The N-GPU end-to-end leg through the public multi-GPU API: every rank
    uploads its own block of the lattice from pinned host memory
    (DistMD(state=...)) inside the timed region, runs the steps keeping each
    step's (KE, PE, px, py, pz) partial row on the device, and the per-step
    rows are summed over ranks and read back to the host at the end (40 B of
    diagnostics per step, as run_md).  Time = max over ranks."""
    import torch
    import torch.distributed as dist
    from paper_2109_09056_b200.dist import DistMD, local_block, rank_dims_for
    rank = dist.get_rank()
    cfg = pc.md.MDConfig(**kw, steps=steps)
    cfg.rank_dims = rank_dims_for(world)
    x, v, ids = (torch.as_tensor(t).pin_memory()
                 for t in local_block(cfg, cells, cfg.rank_dims, rank))
    dev = torch.device("cuda", torch.cuda.current_device())
    hist = torch.zeros((steps + 1, 5), dtype=torch.float64, device=dev)
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    drv = DistMD(cfg, cells=cells, state=(x, v, ids), transport=make_transport(args))
    hist[0] = drv.engine.local_diagnostics()
    for s in range(1, steps + 1):
        drv.step(s)
        hist[s] = drv.engine.local_diagnostics()
    dist.all_reduce(hist)
    rows = hist.cpu()
    e1.record()
    e1.synchronize()
    ms = torch.tensor([e0.elapsed_time(e1)], device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    assert rows.shape[0] == steps + 1 and bool(torch.isfinite(rows).all())
    n = int(drv.n)
    h2d = int(x.numel() * 8 + v.numel() * 8 + ids.numel() * 8)
    del drv
    return {"value": n * steps / (float(ms.item()) * 1e-3), "unit": UNIT,
            "h2d_bytes_per_step": h2d / steps, "d2h_bytes_per_step": 40, "steps": steps,
            "includes": "per rank: H2D of its block's x, v, ids (pinned) + DistMD setup "
                        "(migrate, halo, sort, list build, first force) + the steps, each "
                        "step's energy row kept on the device; rows summed over ranks and "
                        "read back at the end; h2d bytes are rank 0's; max over ranks"}


def main():
    args = parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
