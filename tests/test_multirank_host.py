"""Multi-rank host logic on CPU: two gloo processes each run the product's
host-side setup (host_only) for their rank and check, against each other and
against the oracle's reordered matrix, everything that decides what the NCCL
halo exchange moves: rank ranges (count-balanced contiguous subdomains, R32),
ghost rows and owners, send lists (peer's ghost order), and a gloo halo
exchange driven by those lists delivering exactly x[ghost_rows]."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import paper_2508_04917_b200 as dd
from inputs.gen import random_block_grid

GRID, TILES = (12, 8, 8), (4, 4, 4)   # 18 subdomains: 9 per rank


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        rp, ci, v = random_block_grid(*GRID, seed=21)
        ctx = dd.dd_setup(rp, ci, v, grid=GRID, tiles=TILES, host_only=True, rank=rank, world=world)
        ghosts, owners = ctx.halo()
        mine = dict(rank=rank, first=ctx.row_first, n=ctx.n_local, ghosts=ghosts.tolist(),
                    owners=owners.tolist(), send={p: ctx.send_rows(p).tolist() for p in range(world)},
                    stats=ctx.stats())
        allinfo = [None] * world
        dist.all_gather_object(allinfo, mine)
        S = oracle.setup(rp, ci, v, grid=GRID, tiles=TILES)
        N = S["n"]
        # 1. ranges: contiguous, disjoint, cover [0, N), count-balanced subdomains
        starts = sorted((a["first"], a["n"]) for a in allinfo)
        pos = 0
        for f, n in starts:
            assert f == pos
            pos += n
        assert pos == N
        nsub = S["n_sub"]
        for a in allinfo:
            r = a["rank"]
            s0, s1 = nsub * r // world, nsub * (r + 1) // world
            assert a["first"] == S["sub_ptr"][s0] and a["n"] == S["sub_ptr"][s1] - S["sub_ptr"][s0]
        # 2. ghosts = columns of my rows (reordered A_r, all couplings) outside my range
        a0, n0 = mine["first"], mine["n"]
        cols = S["ci_r"][S["rp_r"][a0]:S["rp_r"][a0 + n0]]
        expect = np.unique(cols[(cols < a0) | (cols >= a0 + n0)])
        assert np.array_equal(np.array(mine["ghosts"], dtype=np.int64), expect)
        for g, o in zip(mine["ghosts"], mine["owners"]):
            b = allinfo[o]
            assert b["first"] <= g < b["first"] + b["n"]
        # 3. my send list to peer p == p's ghosts owned by me, in p's order
        for p in range(world):
            if p == rank:
                assert mine["send"][p] == []
                continue
            theirs = [g for g, o in zip(allinfo[p]["ghosts"], allinfo[p]["owners"]) if o == rank]
            assert [a0 + x for x in mine["send"][p]] == theirs
        # 4. a halo exchange driven by the lists delivers x[ghost_rows]
        import torch
        x = np.random.default_rng(5).uniform(-1, 1, 3 * N)
        xl = x.reshape(-1, 3)[a0:a0 + n0]
        reqs, recv = [], {}
        for p in range(world):
            if p == rank:
                continue
            sb = torch.from_numpy(np.ascontiguousarray(xl[mine["send"][p]]).ravel())
            nr = sum(1 for o in mine["owners"] if o == p)
            recv[p] = torch.empty(3 * nr, dtype=torch.float64)
            reqs.append(dist.isend(sb, p))
            reqs.append(dist.irecv(recv[p], p))
        for rq in reqs:
            rq.wait()
        got = np.concatenate([recv[p].numpy().reshape(-1, 3) for p in sorted(recv)]) if recv else np.zeros((0, 3))
        assert np.array_equal(got, x.reshape(-1, 3)[np.array(mine["ghosts"], dtype=np.int64)])
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, traceback.format_exc()))


@pytest.mark.parametrize("world", [2, 3])
def test_multirank_host_logic_gloo(world):
    ctx_mp = mp.get_context("spawn")
    q = ctx_mp.Queue()
    port = _free_port()
    procs = [ctx_mp.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, msg in res:
        assert msg == "ok", f"rank {rank}: {msg}"
