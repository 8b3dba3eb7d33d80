"""CPU, world size 2 over gloo: the multi-GPU decomposition the device plan
uses -- contiguous ordinal ranges of the outer loop by the reference's chunk
rule (dxc_chunk_range == eval.cpp:323-330), each rank evaluating its range,
Accum deltas all-gathered and folded into the cells in rank order
(cell = ((cell + d_0) + d_1), the Merge step) -- reproduces the reference's
own chunked evaluation (EvalOptions.chunks = world).  Each rank also lowers
its sharded device plan (compile only) and checks it has exactly that shape:
one Merge step, no all-reduce.  The per-rank evaluation is the reference
evaluator (oracle) on the rank's slice (no GPU here); the device side of the
same plan is tests/test_gpu_comm.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, q):
    import sys
    sys.path.insert(0, ROOT)
    import oracle
    import paper_2104_05372_b200 as dx
    from paper_2104_05372_b200 import programs as P
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    d, k = 8, 5
    pts, asg, cs = P.kmeans_inputs(n, d, k, seed=17)
    for src in (P.kmeans_cost_grad(n, d, k), P.histogram(n, 7)):
        plan = dx.Program(src, ctx=None, rank=rank, world=world).plan.split("---")[0]
        assert plan.count("merge ") == 1 and "allreduce" not in plan, plan

    def merged(delta):
        # all-gather the per-rank deltas, fold them into the (zero) cell in rank order
        parts = [torch.zeros_like(delta) for _ in range(world)]
        dist.all_gather(parts, delta)
        cell = torch.zeros_like(delta)
        for p in parts:
            cell = cell + p
        return cell.numpy()

    lo, hi = dx.chunk_range(n, world, rank)
    m = hi - lo
    cost, dC = oracle.RefProgram(P.kmeans_cost_grad(m, d, k))(pts[lo:hi], asg[lo:hi], cs)
    t = merged(torch.tensor(np.concatenate([cost, dC]), dtype=torch.float64))
    keys = P.histogram_inputs(n, 7, seed=18)
    (h,) = oracle.RefProgram(P.histogram(m, 7))(keys[lo:hi])
    th = merged(torch.tensor(h, dtype=torch.float64))
    if rank == 0:
        full_cost, full_dC = oracle.RefProgram(P.kmeans_cost_grad(n, d, k))(pts, asg, cs, chunks=world)
        (full_h,) = oracle.RefProgram(P.histogram(n, 7))(keys, chunks=world)
        q.put((oracle.rel_diff(t, np.concatenate([full_cost, full_dC])), bool(np.array_equal(th, full_h)),
               bool(np.array_equal(t[:1], full_cost))))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n", [1000, 1001])
def test_sharded_kmeans_and_histogram_gloo_world2(n):
    import oracle
    if not oracle.available():
        pytest.skip("oracle/_ref not built")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    diff, hist_exact, cost_exact = q.get(timeout=10)
    assert diff <= 1e-12
    assert hist_exact
    assert cost_exact  # forward-loop cell: same chunks, same left fold, same bits as the reference
