"""Multi-process exchange protocol of the multi-GPU engine, on CPU with gloo
(world size 2 and 3): counts first, then batched point-to-point blocks,
delivered per source -- the transport dist.DistMD uses over NCCL."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2109_09056_b200.dist import NCCLTransport
        t = NCCLTransport()
        # rank r sends (r+1)*(d+1) rows to every d != r, rows encode (src, dst, k)
        out = {}
        for d in range(world):
            if d == rank:
                continue
            m = (rank + 1) * (d + 1)
            rows = torch.zeros((m, 3), dtype=torch.float64)
            rows[:, 0] = rank
            rows[:, 1] = d
            rows[:, 2] = torch.arange(m, dtype=torch.float64)
            out[d] = rows
        out_full = dict(out)
        if rank == world - 1:
            out.pop(0, None)          # a rank that sends nothing to rank 0
        inbox = t.exchange(out, 3, torch.device("cpu"))
        got = {s: b.numpy().copy() for s, b in inbox.items()}
        # the per-step ghost refresh path: receive sizes known, no counts round
        recv = {s: b.shape[0] for s, b in inbox.items()}
        again = t.exchange(out, 3, torch.device("cpu"), recv_counts=recv)
        assert sorted(again) == sorted(inbox)
        for s_ in again:
            assert torch.equal(again[s_], inbox[s_])
        # the per-step refresh path: one all-to-all with per-rank split sizes
        send_split = [0 if d == rank else (rank + 1) * (d + 1) for d in range(world)]
        recv_split = [0 if s_ == rank else (s_ + 1) * (rank + 1) for s_ in range(world)]
        send = torch.cat([out_full[d] for d in range(world) if d != rank])
        got_a2a = t.alltoall(send, send_split, recv_split, torch.device("cpu"))
        expect = torch.cat([torch.stack([torch.full(((s_ + 1) * (rank + 1),), float(s_)),
                                         torch.full(((s_ + 1) * (rank + 1),), float(rank)),
                                         torch.arange((s_ + 1) * (rank + 1),
                                                      dtype=torch.float64)], 1)
                            for s_ in range(world) if s_ != rank])
        assert torch.equal(got_a2a, expect)
        red = t.allreduce(torch.tensor([float(rank), 1.0], dtype=torch.float64))
        q.put((rank, got, red.numpy().copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_transport_exchange_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        rank, got, red = q.get(timeout=120)
        res[rank] = (got, red)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, (got, red) in res.items():
        assert red.tolist() == [sum(range(world)), float(world)]
        for src in range(world):
            if src == rank or (src == world - 1 and rank == 0):
                assert src not in got
                continue
            m = (src + 1) * (rank + 1)
            b = got[src]
            assert b.shape == (m, 3)
            assert np.all(b[:, 0] == src) and np.all(b[:, 1] == rank)
            assert np.array_equal(b[:, 2], np.arange(m))


def test_rank_dims_for():
    from paper_2109_09056_b200.dist import rank_dims_for
    assert rank_dims_for(1) == (1, 1, 1)
    assert rank_dims_for(2) == (2, 1, 1)
    assert rank_dims_for(4) == (2, 2, 1)
    assert rank_dims_for(8) == (2, 2, 2)
    assert int(np.prod(rank_dims_for(6))) == 6


@pytest.mark.parametrize("dims", [(2, 1, 1), (2, 2, 1), (2, 2, 2)])
def test_local_blocks_tile_the_lattice(dims):
    """dist.local_block (the per-rank host input of DistMD(local_init=True) and
    of the bench's N-GPU end-to-end leg): the blocks of all ranks are the
    reference's fcc lattice (md.py:67-74) split by owner, ids = lattice order."""
    from paper_2109_09056_b200.dist import local_block
    from paper_2109_09056_b200.md import MDConfig, fcc_lattice
    cfg = MDConfig(lattice_cells=6, temperature=1.44, skin=0.3, rebuild_stride=5)
    cells = np.array([6, 6, 6])
    a = (4.0 / cfg.density) ** (1.0 / 3.0)
    ref = fcc_lattice(6, a)
    bl = cells * a / np.array(dims)
    seen = np.zeros(ref.shape[0], bool)
    for r in range(int(np.prod(dims))):
        x, v, ids = local_block(cfg, cells, dims, r)
        assert x.shape == v.shape == (ids.size, 3)
        assert np.array_equal(x, ref[ids])
        # owner by the reference formula (decomp.py:58-66), host-side
        c = np.minimum(np.floor(x / bl).astype(np.int64), np.array(dims) - 1)
        assert np.all(np.ravel_multi_index(tuple(c.T), dims) == r)
        assert not seen[ids].any()
        seen[ids] = True
        assert np.abs(v.mean(axis=0)).max() < 1e-12
    assert seen.all()


def test_p2p_plan_matches_all_to_all_layout():
    """The peer-memory all-to-all's addressing (dist.p2p_plan: each rank's puts
    from its destination-ordered send rows into every destination's
    source-ordered window) reproduces all_to_all_single's result for random
    split matrices, self-sends and empty pairs included (host logic of
    P2PTransport; the device path is tests/test_gpu_distmd.py)."""
    import numpy as np
    from paper_2109_09056_b200.dist import p2p_plan
    rng = np.random.default_rng(3)
    for world in (1, 2, 4, 8):
        for _ in range(5):
            C = rng.integers(0, 6, (world, world)) * (rng.random((world, world)) < 0.7)
            send = []
            for s in range(world):         # row (s, d, k), destination order
                send.append([(s, d, k) for d in range(world) for k in range(C[s, d])])
            windows = [[None] * int(C[:, d].sum()) for d in range(world)]
            for s in range(world):
                for d, src0, cnt, dst0 in p2p_plan(C, s)["puts"]:
                    windows[d][dst0:dst0 + cnt] = send[s][src0:src0 + cnt]
            for d in range(world):
                want = [(s, d, k) for s in range(world) for k in range(C[s, d])]
                assert windows[d] == want
                assert p2p_plan(C, d)["srcs"] == [s for s in range(world) if C[s, d] > 0]
