"""Multi-rank host logic on CPU (world size 2, gloo): the row-block partition of
the dense operator, the padded all-gather layout the CUDA path uses after every
sharded matvec, and the NCCL unique-id exchange of bench.py.  (The GPU sessions of
this run expose one GPU, so the NCCL path itself is exercised on CPU only through
its host-side pieces.)"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import fde_inputs as fi


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_rows_cover_and_balance():
    from paper_1808_02937_b200 import fde
    for N, P in [(8, 4), (1024, 8), (4096, 8), (13, 3), (5, 1)]:
        n = N * P - 1
        for G in (1, 2, 3, 4, 8):
            if G > N:
                continue
            spans = [fde.shard_rows(N, P, G, g) for g in range(G)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            for g in range(G - 1):
                assert spans[g][1] == spans[g + 1][0]            # contiguous, disjoint
            rm = max(b - a for a, b, _ in spans)
            assert all(s[2] == max(rm, 1) for s in spans)
            for a, b, _ in spans:                                 # shards start at element boundaries
                assert a % P == 0
            sizes = [b - a for a, b, _ in spans]
            assert max(sizes) - min(sizes) <= P * (1 + N // G - N // G)   # balanced to one element


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1808_02937_b200 import fde
        import oracle as O
        p = fi.config2(1.5, N=12, P=4)
        N, P, n = p.N, p.P, p.n
        r0, r1, rmax = fde.shard_rows(N, P, world, rank)
        # internal (element-interleaved) order of the oracle's operator
        so = O.assemble_system(p)
        perm = fde.internal_to_paper_index(N, P)
        Ai = so.A[np.ix_(perm, perm)]
        x = np.random.default_rng(3).standard_normal(n)
        y_loc = np.zeros(rmax)
        y_loc[: r1 - r0] = Ai[r0:r1] @ x                     # this rank's rows (padded shard)
        out = [torch.zeros(rmax, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(out, torch.tensor(y_loc))
        starts = [fde.shard_rows(N, P, world, g)[0] for g in range(world)]
        y = np.empty(n)
        for r in range(n):                                   # compaction as in k_compact_gather
            g = max(gg for gg in range(world) if starts[gg] <= r)
            y[r] = out[g][r - starts[g]].item()
        err = np.abs(y - Ai @ x).max() / np.abs(Ai @ x).max()
        # NCCL unique id exchange (bench.py): rank 0 creates, everyone receives the same bytes
        try:
            uid = fde.nccl_unique_id() if rank == 0 else None
        except Exception:
            uid = b"\0" * 128 if rank == 0 else None
        obj = [uid]
        dist.broadcast_object_list(obj, src=0)
        q.put((rank, float(err), len(obj[0]), obj[0][:16]))
    finally:
        dist.destroy_process_group()


def test_two_rank_sharded_matvec_gather_matches_full_matvec():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
    assert all(pr.exitcode == 0 for pr in procs)
    for rank, err, ln, head in res:
        assert err < 1e-13
        assert ln == 128
    assert res[0][3] == res[1][3]
