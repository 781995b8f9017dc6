"""World-size-2 CPU (gloo) tests of the multi-GPU decomposition.

The CUDA path shards A by columns with mnb_shard_columns and exchanges:
  * per CG iteration: one allreduce (sum) of [s = A_J(A_J^H w), ||A_J^H w||^2,
    <r_J, t_J>, ||r_J||^2]  (solver.cu: fused_pass + allreduce_sum);
  * per sketch: one all-to-all turning column shards into row blocks
    A[rows_h, :], a local sketch of the row block, and an allgather of the
    sketch columns (srft_gpu.cu: sketch_matrix).
These tests run exactly that exchange pattern over torch.distributed (gloo)
with numpy local compute, and check the results against the unsharded
computation -- using the product's own partition function.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as tmp  # noqa: E402


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _instance():
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    from tests.instances import make_instance
    return make_instance(12, 1000, 1e3, seed=11)


def _worker(rank, world, port, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_0905_4745_b200 as mn
        from oracle import minnorm_oracle as O
        A, b = _instance()
        m, n = A.shape
        cb, cn = mn.shard_columns(n, world, rank)
        AJ = np.asfortranarray(A[:, cb:cb + cn])
        rng = np.random.default_rng(5)
        w = rng.standard_normal(m) + 1j * rng.standard_normal(m)
        r = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        # ---- the per-iteration allreduce of the fused pass
        tJ = O.AH_v(AJ, w)
        red = np.concatenate([O.A_r(AJ, tJ).view(np.float64),
                              [np.vdot(tJ, tJ).real, np.vdot(r[cb:cb + cn], tJ).real,
                               np.vdot(r[cb:cb + cn], r[cb:cb + cn]).real, 0.0]])
        tr = torch.from_numpy(red.copy())
        dist.all_reduce(tr, op=dist.ReduceOp.SUM)
        red_all = tr.numpy()
        # ---- the sketch all-to-all into row blocks, laid out by the library's own table
        # (mnb_redistribute_plan: the offsets srft_gpu.cu redistribute_rows packs and receives at)
        plan = mn.redistribute_plan(m, n, world, rank)
        my_rows = int(plan[rank, 1])
        pack = np.zeros(m * cn, np.complex128)
        for h in range(world):
            r0, rc, off = plan[h, 0], plan[h, 1], plan[h, 2]
            pack[off:off + rc * cn] = AJ[r0:r0 + rc, :].ravel(order="F")  # column-major, ld rc
        slab = np.zeros(my_rows * n, np.complex128)
        send = [torch.from_numpy(pack[plan[h, 2]:plan[h, 2] + plan[h, 1] * cn].view(np.float64).copy())
                for h in range(world)]
        recv = [torch.zeros(my_rows * int(plan[h, 4]) * 2, dtype=torch.float64) for h in range(world)]
        # grouped point-to-point, as the CUDA path's ncclGroupStart/ncclSend/ncclRecv (srft_gpu.cu)
        ops = []
        for h in range(world):
            if h == rank:
                recv[h].copy_(send[h])
                continue
            ops.append(dist.P2POp(dist.isend, send[h], h))
            ops.append(dist.P2POp(dist.irecv, recv[h], h))
        for req in dist.batch_isend_irecv(ops):
            req.wait()
        for h in range(world):
            off, cnt = plan[h, 5], my_rows * plan[h, 4]
            slab[off:off + cnt] = recv[h].numpy().view(np.complex128)
        block = slab.reshape(n, my_rows).T  # my_rows x n, column-major (ld my_rows)
        rows = [mn.shard_columns(m, world, h) for h in range(world)]
        rb, rc = rows[rank]
        assert (rb, rc) == (plan[rank, 0], my_rows)
        op = O.Srft.build(48, n, O.derive_seed(42, 11))
        S_local = op.sketch(block, threads=1)  # l x rc
        gathered = [torch.zeros(48 * rows[h][1] * 2, dtype=torch.float64) for h in range(world)]
        dist.all_gather(gathered, torch.from_numpy(S_local.ravel(order="F").view(np.float64).copy()))
        S = np.concatenate([g.numpy().view(np.complex128).reshape(48, rows[h][1], order="F")
                            for h, g in enumerate(gathered)], axis=1)
        q.put((rank, red_all, np.array_equal(block, A[rb:rb + rc, :]), S))
    except Exception as e:  # surface worker failures instead of a queue timeout
        q.put((rank, repr(e), False, None))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_pass_and_sketch_redistribution_match_unsharded(world):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    from oracle import minnorm_oracle as O
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    A, _ = _instance()
    m, n = A.shape
    rng = np.random.default_rng(5)
    w = rng.standard_normal(m) + 1j * rng.standard_normal(m)
    r = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    t = O.AH_v(A, w)
    s = O.A_r(A, t)
    S_full = O.Srft.build(48, n, O.derive_seed(42, 11)).sketch(A, threads=1)
    for rank, red, block_ok, S in sorted(results, key=lambda x: x[0]):
        assert not isinstance(red, str), red
        assert block_ok, "all-to-all did not reproduce the row block"
        assert np.allclose(red[:2 * m].view(np.complex128), s, rtol=1e-13, atol=1e-13 * np.abs(s).max())
        assert red[2 * m] == pytest.approx(np.vdot(t, t).real, rel=1e-13)
        assert red[2 * m + 1] == pytest.approx(np.vdot(r, t).real, rel=1e-12)
        assert red[2 * m + 2] == pytest.approx(np.vdot(r, r).real, rel=1e-13)
        assert np.array_equal(S, S_full), "gathered sketch differs from the single-rank sketch"
