"""Multi-process (world_size 2, gloo on CPU) coverage of the sharded step's
host logic: contiguous shard ranges, per-rank field generation from the
global LCG stream, and the all-reduce(MAX) that yields a bit-identical
global eigenvalue / dt.  The per-rank compute here is the CPU oracle (the
checker); on the GPU box the same driver runs the CUDA kernel per rank."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2306_16731_b200.distributed import shard_range


def test_shard_range_partitions():
    for total in (1, 7, 64, 1000):
        for world in (1, 2, 3, 8):
            if world > total:
                continue
            spans = [shard_range(total, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, d, p, total, result):
    import torch
    import torch.distributed as dist

    from oracle import oracle
    from paper_2306_16731_b200 import _lib

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard_range(total, rank, world)
    n, M, Mi = oracle.sizes(d, p, hi - lo)
    # generate this shard straight from the global stream (jump-ahead)
    qs = np.zeros(n * total * M)
    oracle.lib().fvo_init_field_soa(d, p, total, 0, 1.4, qs.ctypes.data, lo, hi - lo, 1)
    q = np.ascontiguousarray(qs.reshape(n, total, M)[:, lo:hi, :]).reshape(-1)
    out, red = oracle.step_c(d, p, hi - lo, q, threads=1)
    lam = torch.tensor([red], dtype=torch.float64)
    dist.all_reduce(lam, op=dist.ReduceOp.MAX)
    dt = _lib.load().fvb_admissible_dt(float(lam.item()), 0.1, 0.5)
    result[rank] = (float(lam.item()), dt, out.tobytes())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("d,p,total", [(2, 16, 9), (3, 4, 5)])
def test_two_rank_allreduce_max_matches_single_process(d, p, total):
    from oracle import oracle

    ctx = mp.get_context("spawn")
    manager = ctx.Manager()
    result = manager.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, d, p, total, result)) for r in range(2)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(120)
        assert pr.exitcode == 0
    q = oracle.init_field_soa(d, p, total, 0)
    out, red = oracle.step_c(d, p, total, q, threads=1)
    assert result[0][0] == result[1][0] == red
    assert result[0][1] == result[1][1] == 0.5 * 0.1 / red
    n, _, Mi = oracle.sizes(d, p, total)
    whole = out.reshape(n, total, Mi)
    for rank in range(2):
        lo, hi = shard_range(total, rank, 2)
        part = np.frombuffer(result[rank][2]).reshape(n, hi - lo, Mi)
        assert part.tobytes() == np.ascontiguousarray(whole[:, lo:hi, :]).tobytes()
