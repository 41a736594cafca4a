"""Multi-process DistMD (one process per rank, torch.distributed) on one GPU:
two ranks share cuda:0 with the gloo backend (host-staged blocks; NCCL needs
distinct GPUs).  The decomposed run must reproduce the single-domain energy
series (within the tile path's 1e-6 energy tolerance) -- the same engine code
the N-GPU bench runs over NCCL."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

KW = dict(lattice_cells=6, density=0.8442, temperature=1.44, cutoff=2.5, skin=0.3,
          rebuild_stride=5, seed=1, steps=0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, steps, det=False, overlap=None, kw=None, half=False,
            p2p=False, state=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import paper_2109_09056_b200 as pc
        from paper_2109_09056_b200.dist import DistMD, P2PTransport
        tr = P2PTransport() if p2p else None
        drv = DistMD(pc.md.MDConfig(**(kw or KW)), deterministic=det, half_list=half,
                     transport=tr)
        if overlap is not None:
            drv.overlap = overlap
        es = [drv.diagnostics()["E_total"]]
        for s in range(1, steps + 1):
            drv.step(s)
            es.append(drv.diagnostics()["E_total"])
        if state:
            gid, x, v = drv.engine.owned_state()
            o = np.argsort(gid)
            q.put((rank, np.array(es), gid[o], x[o], v[o]))
        elif overlap is None:
            q.put((rank, np.array(es), drv.engine.n_owned))
        else:
            gid, x, v = drv.engine.owned_state()
            o = np.argsort(gid)
            q.put((rank, np.array(es), gid[o], x[o], v[o]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_distmd_two_processes(world):
    import paper_2109_09056_b200 as pc
    steps = 25
    drv = pc.md.MDDriver(pc.md.MDConfig(**KW))
    ref = [drv.diagnostics()["E_total"]]
    for s in range(1, steps + 1):
        drv.step(s)
        ref.append(drv.diagnostics()["E_total"])
    ref = np.array(ref)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, steps)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    owned = sum(o[2] for o in out)
    assert owned == drv.n
    for _, es, _ in out:
        assert np.max(np.abs(es - ref) / np.abs(ref)) < 1e-6     # tile path: FP32 pair energies summed in slot order


def test_distmd_deterministic_bitwise():
    """Two processes, deterministic=True: energy series bitwise equal to the
    single-domain deterministic run."""
    import paper_2109_09056_b200 as pc
    steps = 15
    drv = pc.md.MDDriver(pc.md.MDConfig(**KW), deterministic=True)
    ref = [drv.diagnostics()["E_total"]]
    for s in range(1, steps + 1):
        drv.step(s)
        ref.append(drv.diagnostics()["E_total"])
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, steps, True)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=600) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for _, es, _ in out:
        assert np.array_equal(es, np.array(ref))


@pytest.mark.parametrize("world,det", [(4, True), (4, False), (8, True)])
def test_distmd_four_processes(world, det):
    """Four / eight processes (rank grids 2x2x1 and 2x2x2, the 8-GPU bench's:
    up to seven neighbour ranks, several halo images per neighbour) through
    the same all-to-all refresh and vectorised halo plan as the 8-GPU run:
    bitwise equal to the single-domain run in deterministic mode, within the
    tile path's 1e-6 otherwise."""
    import paper_2109_09056_b200 as pc
    steps = 12
    drv = pc.md.MDDriver(pc.md.MDConfig(**KW), deterministic=det)
    ref = [drv.diagnostics()["E_total"]]
    for s in range(1, steps + 1):
        drv.step(s)
        ref.append(drv.diagnostics()["E_total"])
    ref = np.array(ref)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, steps, det))
             for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert sum(o[2] for o in out) == drv.n
    for _, es, _ in out:
        if det:
            assert np.array_equal(es, ref)
        else:
            assert np.max(np.abs(es - ref) / np.abs(ref)) < 1e-6


@pytest.mark.parametrize("world", [2, 4])
def test_distmd_overlap_split_bitwise(world):
    """Across processes: the step with the interior-tile force overlapping the
    ghost all-to-all (then unpack, then boundary tiles) gives positions and
    velocities bitwise equal to the one-pass step on every rank, energies to
    1e-12 (on a GPU box the all-to-all is NCCL on its own
    stream, here gloo)."""
    kw = dict(KW, lattice_cells=10)
    res = {}
    for overlap in (False, True):
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        port = _free_port()
        procs = [ctx.Process(target=_worker, args=(r, world, port, q, 12, False, overlap, kw))
                 for r in range(world)]
        for p in procs:
            p.start()
        out = sorted([q.get(timeout=600) for _ in range(world)], key=lambda t: t[0])
        for p in procs:
            p.join(timeout=120)
            assert p.exitcode == 0
        res[overlap] = out
    for a, b in zip(res[False], res[True]):
        assert np.array_equal(a[2], b[2])
        assert np.array_equal(a[3], b[3]) and np.array_equal(a[4], b[4])
        assert np.max(np.abs(a[1] - b[1]) / np.abs(a[1])) < 1e-12


def test_distmd_half_list_two_processes():
    """Two processes, half list + reverse halo over the transport (the
    transpose of the refresh all-to-all): the energy series matches the
    single-domain half-list engine within 1e-9."""
    import paper_2109_09056_b200 as pc
    steps = 15
    drv = pc.md.MDDriver(pc.md.MDConfig(**KW), half_list=True, tile=False)
    ref = [drv.diagnostics()["E_total"]]
    for s in range(1, steps + 1):
        drv.step(s)
        ref.append(drv.diagnostics()["E_total"])
    ref = np.array(ref)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, steps, False, None, None, True))
             for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=600) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for _, es, _ in out:
        assert np.max(np.abs(es - ref) / np.abs(ref)) < 1e-9


def _run(world, **kw):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    args = dict(kw)
    steps = args.pop("steps")
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, steps), kwargs=args)
             for r in range(world)]
    for p in procs:
        p.start()
    out = sorted([q.get(timeout=600) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return out


@pytest.mark.parametrize("world,half,overlap", [(2, False, False), (2, False, True),
                                                 (4, False, False), (2, True, False),
                                                 (8, False, False)])
def test_distmd_p2p_transport_bitwise(world, half, overlap):
    """The per-step refresh (and the half list's reverse halo) as direct
    peer-memory stores between the ranks' processes (P2PTransport: CUDA IPC
    windows, device-side arrival / acknowledgement flags; here two / four
    processes on one GPU) gives positions and velocities bitwise equal to the
    all-to-all transport on every rank, and the same energy series (1e-12),
    over several rebuilds (rebuild every 5 steps: the channels are re-planned
    each time); the half list (FP64 atomics on both sides of a pair, not
    bitwise reproducible run to run) within 1e-10."""
    kw = dict(KW, lattice_cells=8)
    res = {}
    for p2p in (False, True):
        res[p2p] = _run(world, steps=17, kw=kw, half=half, p2p=p2p, state=True,
                        overlap=overlap)
    for a, b in zip(res[False], res[True]):
        assert np.array_equal(a[2], b[2])
        if half:
            # the half list accumulates both sides of a pair with FP64
            # atomics: not bitwise reproducible between two runs
            assert np.max(np.abs(a[3] - b[3])) < 1e-10 and np.max(np.abs(a[4] - b[4])) < 1e-9
            assert np.max(np.abs(a[1] - b[1]) / np.abs(a[1])) < 1e-10
            continue
        assert np.array_equal(a[3], b[3]) and np.array_equal(a[4], b[4])
        assert np.max(np.abs(a[1] - b[1]) / np.abs(a[1])) < 1e-12
