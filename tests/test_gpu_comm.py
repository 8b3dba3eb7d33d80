"""GPU: the multi-rank plumbing on one device -- NCCL (dlopen'ed, the copy
torch maps) communicator of one rank through dxc_comm_init, and an in-place
dxc_allreduce_sum of a device buffer (identity at world size 1).  The
world-size-2 merge logic itself is covered on CPU with gloo
(tests/test_distributed.py)."""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_single_rank_nccl_allreduce_is_identity():
    import paper_2104_05372_b200 as dx
    lib = dx._lib
    ctx = dx.Context(0)
    ctx.init_comm(dx.nccl_unique_id(), 1, 0)
    vals = np.arange(1000, dtype=np.float64) * 0.5 - 7.0
    buf = ctypes.c_void_p()
    lib.dxc_buf_alloc.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_void_p)]
    lib.dxc_buf_upload.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_size_t]
    lib.dxc_buf_download.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_size_t]
    lib.dxc_buf_ptr.argtypes = [ctypes.c_void_p]
    lib.dxc_buf_ptr.restype = ctypes.c_void_p
    lib.dxc_buf_free.argtypes = [ctypes.c_void_p]
    assert lib.dxc_buf_alloc(ctx.handle, vals.nbytes, ctypes.byref(buf)) == 0
    try:
        assert lib.dxc_buf_upload(buf, 0, vals.ctypes.data, vals.nbytes) == 0
        assert lib.dxc_allreduce_sum(ctx.handle, lib.dxc_buf_ptr(buf), vals.size, dx.DXC_F64) == 0
        ctx.sync()
        out = np.empty_like(vals)
        assert lib.dxc_buf_download(buf, 0, out.ctypes.data, out.nbytes) == 0
        assert np.array_equal(out, vals)
    finally:
        lib.dxc_buf_free(buf)


@pytest.mark.parametrize("which", ["kmeans", "histogram"])
def test_world2_shards_through_nccl_sum_to_the_whole(which):
    """Both ranks of a world-size-2 sharded plan run on this device, each with
    its Accum cells all-reduced over a one-rank NCCL communicator (the
    plan's Allreduce steps execute for real, as identities); the two shard
    results summed on the host equal the unsharded result."""
    import oracle
    import paper_2104_05372_b200 as dx
    from paper_2104_05372_b200 import programs as P
    ctx = dx.Context(0)
    ctx.init_comm(dx.nccl_unique_id(), 1, 0)
    if which == "kmeans":
        n, d, k = 50_000, 16, 64
        src, args = P.kmeans_cost_grad(n, d, k), P.kmeans_inputs(n, d, k)
    else:
        n, k = 1 << 20, 4096
        src, args = P.histogram(n, k), (P.histogram_inputs(n, k, seed=5),)
    whole = dx.Program(src, ctx=ctx)(*args)
    parts = []
    for rank in (0, 1):
        prog = dx.Program(src, ctx=ctx, rank=rank, world=2, flags=dx.F_TEST_COMM_MISMATCH)
        assert "merge " in prog.plan
        parts.append(prog(*args))
    for w, p0, p1 in zip(whole, parts[0], parts[1]):
        got = np.asarray(p0, dtype=np.float64) + np.asarray(p1, dtype=np.float64)
        if which == "histogram":
            assert np.array_equal(got, np.asarray(w, dtype=np.float64))  # integer counts: exact
        else:
            assert oracle.rel_diff(got, np.asarray(w, dtype=np.float64)) <= 1e-5


def test_gmm_moments_allreduce_path():
    """The GMM plan all-reduces its lse sum and fp64 moments when a
    communicator is set: at one rank the results equal the local ones."""
    import paper_2104_05372_b200 as dx
    from oracle import gmm as G
    n, k = 5000, 7
    a, mu, icf, x = G.gmm_inputs(n, 64, k, seed=9)
    plain = dx.GMM(dx.Context(0), 64, k, n)(a, mu, icf, x)
    ctx = dx.Context(0)
    ctx.init_comm(dx.nccl_unique_id(), 1, 0)
    comm = dx.GMM(ctx, 64, k, n, n)(a, mu, icf, x)
    assert plain[0] == comm[0]
    for u, v in zip(plain[1:], comm[1:]):
        assert np.array_equal(u, v)


def test_sharded_plan_without_communicator_fails_loudly():
    import paper_2104_05372_b200 as dx
    from paper_2104_05372_b200 import programs as P
    ctx = dx.Context(0)
    n, k = 4096, 64
    prog = dx.Program(P.histogram(n, k), ctx=ctx, rank=0, world=2)
    with pytest.raises(dx.DexError):
        prog(P.histogram_inputs(n, k, seed=1))


def test_sharded_plan_with_wrong_communicator_fails_loudly():
    """A world-2 plan over a one-rank communicator would all-reduce nothing:
    refused before anything is launched (unless the test-only flag is set)."""
    import paper_2104_05372_b200 as dx
    from paper_2104_05372_b200 import programs as P
    ctx = dx.Context(0)
    ctx.init_comm(dx.nccl_unique_id(), 1, 0)
    n, k = 4096, 64
    prog = dx.Program(P.histogram(n, k), ctx=ctx, rank=1, world=2)
    with pytest.raises(dx.DexError) as e:
        prog(P.histogram_inputs(n, k, seed=1))
    assert e.value.code == dx.DXC_E_ARG


def test_sharded_gmm_without_communicator_fails_loudly():
    import paper_2104_05372_b200 as dx
    from paper_2104_05372_b200 import programs as P
    n, k = 1000, 3
    a, mu, icf, x = P.gmm_inputs(n, 64, k, seed=2)
    g = dx.GMM(dx.Context(0), 64, k, n, 2 * n)
    with pytest.raises(dx.DexError) as e:
        g(a, mu, icf, x)
    assert e.value.code == dx.DXC_E_ARG


def test_input_size_mismatch_is_e_size():
    import paper_2104_05372_b200 as dx
    from paper_2104_05372_b200 import programs as P
    ctx = dx.Context(0)
    n, k = 4096, 64
    prog = dx.Program(P.histogram(n, k), ctx=ctx)
    with pytest.raises(dx.DexError) as e:
        prog(P.histogram_inputs(n - 1, k, seed=1))
    assert e.value.code == dx.DXC_E_SIZE


def test_unread_index_leaf_is_range_checked_on_upload():
    """An index input passed straight to the output is checked at upload
    (fromOrdinal's check, index_set.cpp:99-106), not only where kernels read it."""
    import paper_2104_05372_b200 as dx
    ctx = dx.Context(0)
    prog = dx.Program("main = \\p:((Fin 8)=>(Fin 4)). p\n", ctx=ctx)
    keys = np.array([0, 1, 2, 3, 4, 0, 1, 2], dtype=np.int32)
    prog.set_input(0, 0, keys)
    prog.run()
    with pytest.raises(dx.DexError) as e:
        prog.check()
    assert e.value.code == dx.DXC_E_BOUNDS
    prog.set_input(0, 0, keys % 4)
    prog.run()
    prog.check()


def test_mlp_world2_shards_sum_to_the_whole():
    """configs[4] data-parallel on one device: ranks 0 and 1 of a world-2
    plan (tcgen05 GEMMs on each rank's batch rows, one fused merge through a
    one-rank NCCL communicator) each return their batch shard's loss and
    weight gradients; the two summed equal the unsharded program."""
    import oracle
    import paper_2104_05372_b200 as dx
    from paper_2104_05372_b200 import programs as P
    ctx = dx.Context(0)
    ctx.init_comm(dx.nccl_unique_id(), 1, 0)
    b, i, h, o = 2048, 256, 256, 128
    x, w1, w2 = P.mlp_inputs(b, i, h, o)
    src = P.mlp_grad(b, i, h, o)
    whole = dx.Program(src, ctx=ctx)(x, [w1, w2])
    parts = []
    for rank in (0, 1):
        prog = dx.Program(src, ctx=ctx, rank=rank, world=2, flags=dx.F_TEST_COMM_MISMATCH)
        assert "tcgen05 gemm" in prog.plan and "allreduce" not in prog.plan.split("---")[0]
        parts.append(prog(x, [w1, w2]))
    for w, p0, p1 in zip(whole, parts[0], parts[1]):
        got = np.asarray(p0, dtype=np.float64) + np.asarray(p1, dtype=np.float64)
        assert oracle.rel_diff(got, np.asarray(w, dtype=np.float64)) <= 1e-4


def test_rank_local_input_shards():
    """dxl_program_set_input_rows: each rank of a world-2 k-means plan uploads
    only its chunk of the points and assignments (the rows its kernel reads)
    and gets the same shard result as with the whole inputs uploaded."""
    import paper_2104_05372_b200 as dx
    from paper_2104_05372_b200 import programs as P
    ctx = dx.Context(0)
    ctx.init_comm(dx.nccl_unique_id(), 1, 0)
    n, d, k = 30_001, 16, 64
    pts, asg, cs = P.kmeans_inputs(n, d, k)
    src = P.kmeans_cost_grad(n, d, k)
    for rank in (0, 1):
        full = dx.Program(src, ctx=ctx, rank=rank, world=2, flags=dx.F_TEST_COMM_MISMATCH)(pts, asg, cs)
        prog = dx.Program(src, ctx=ctx, rank=rank, world=2, flags=dx.F_TEST_COMM_MISMATCH)
        lo, hi = dx.chunk_range(n, 2, rank)
        prog.set_input_rows(0, 0, pts[lo:hi], lo)
        prog.set_input_rows(1, 0, asg[lo:hi].astype(np.int32), lo)
        prog.set_input(2, 0, cs)
        prog.run()
        got = [prog.get_output(0), prog.get_output(1)]
        for a, b in zip(full, got):
            assert np.array_equal(a, b)
