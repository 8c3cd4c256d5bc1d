"""World-size-2 gloo test of the multi-rank bench path (one process per GPU,
independent blocks per rank, max-over-ranks timing, rank-0 reporting) on
CPU."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    import numpy as np
    import oracle as O
    import paper_2509_26475_b200 as P
    # each rank evaluates its own independent block (replicas, weak scaling):
    # a different seed per rank, checked against the oracle's serial result
    wl = P.workload(1, 64)
    op = O.csr_from_arrays(wl.n, wl.rp, wl.ci, wl.av)
    ss = O.select_parameters(op, 61, wl.tol)
    V = O.Rng(100 + rank).matrix(wl.n, wl.p + 1)
    W, rec = O.phimv_block(op, wl.t, wl.alpha, V, wl.tol, ss)
    elapsed = 1.0 + rank  # per-rank clock
    m = bench.max_over_ranks(elapsed, dist, "cpu")
    sums = bench.max_over_ranks(float(np.abs(W).sum()), dist, "cpu")
    out[rank] = (m, rec.series_len_S, sums)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_max_over_ranks():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    assert out[0][0] == out[1][0] == 2.0  # slowest rank's clock
    assert out[0][1] == out[1][1]          # same operator -> same series length
    assert out[0][2] == out[1][2]
