"""Host logic of the multi-GPU x-slab path on CPU (gloo, world_size 2).

The CUDA side of the decomposition is checked bit for bit on one GPU by
tests/test_slab_gpu.py (in-process rank emulation); here the pieces that run
per process under torchrun are exercised with real processes: partition,
ghost/owned ranges, slab slicing and reassembly, probe ownership, and the
NCCL unique-id broadcast over torch.distributed.
"""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2510_22221_b200 import parallel


def test_partition_balanced_and_complete():
    for nx in (4, 7, 12, 1024, 8192):
        for n in (1, 2, 3, 4, 8):
            if nx < 2 * n:
                with pytest.raises(ValueError):
                    parallel.partition(nx, n)
                continue
            parts = parallel.partition(nx, n)
            assert parts[0][0] == 0 and parts[-1][1] == nx
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            sizes = [h - l for l, h in parts]
            assert max(sizes) - min(sizes) <= 1 and min(sizes) >= 2


def test_slab_ranges():
    slabs = parallel.make_slabs(12, 3)
    assert [s.owned_fields for s in slabs] == [(0, 4), (4, 8), (8, 13)]
    assert [s.field_range for s in slabs] == [(0, 5), (3, 9), (7, 13)]
    assert [s.cell_range for s in slabs] == [(0, 5), (3, 9), (7, 12)]
    # owned field planes tile [0, F) exactly once
    covered = np.zeros(13, int)
    for s in slabs:
        covered[slice(*s.owned_fields)] += 1
    assert (covered == 1).all()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    try:
        rng = np.random.default_rng(7)
        nx, ny, nz = 10, 4, 3
        field = rng.standard_normal((nx + 1, ny + 1, nz + 1))
        m = rng.standard_normal((3, nx, ny, nz))
        slab = parallel.make_slabs(nx, world)[rank]
        loc_f = parallel.local_fields(slab, field)
        loc_m = parallel.local_cells(slab, m, axis=1)
        # reassemble owned parts on every rank (what bench/run gather does)
        parts = [None] * world
        dist.all_gather_object(parts, (slab.owned_fields, parallel.owned_part(slab, loc_f),
                                       (slab.x_lo, slab.x_hi),
                                       parallel.owned_cells(slab, loc_m)))
        back = np.empty_like(field)
        mback = np.empty_like(m)
        for (c0, c1), arr, (x0, x1), marr in parts:
            back[c0:c1] = arr
            mback[:, x0:x1] = marr
        ok_fields = np.array_equal(back, field) and np.array_equal(mback, m)
        # ghost planes hold the neighbours' boundary planes
        f0, f1 = slab.field_range
        ok_ghost = np.array_equal(loc_f, field[f0:f1])
        # probe ownership: exactly one rank owns each field plane
        owned = [slab.owned_fields[0] <= i < slab.owned_fields[1] for i in range(nx + 1)]
        cnt = torch.tensor([int(o) for o in owned])
        dist.all_reduce(cnt)
        ok_probe = bool((cnt == 1).all())
        # NCCL id from rank 0 reaches every rank unchanged
        nid = parallel.nccl_unique_id(dist)
        ids = [None] * world
        dist.all_gather_object(ids, nid)
        ok_id = len(nid) == 128 and all(x == nid for x in ids)
        q.put((rank, ok_fields, ok_ghost, ok_probe, ok_id))
    finally:
        dist.destroy_process_group()


def test_two_rank_slab_host_logic():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, *oks in res:
        assert all(oks), (rank, oks)
