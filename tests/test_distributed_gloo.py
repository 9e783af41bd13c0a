"""The multi-GPU orchestration (partitioned mapping + H all-gather, tile-range sharding, result
gather + unpack on rank 0) under gloo with world_size 2 on CPU.  The per-step compute is the
fp64 oracle (test stand-in); the partition / exchange / assembly code is the product's."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from asot_inputs import make_inputs
from oracle import asot_oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_steps(inp):
    import paper_2310_16123_b200 as asot
    from paper_2310_16123_b200.distributed import DistSteps

    def map_range(lo, hi):
        s, e = inp.offsets[lo], inp.offsets[hi]
        _, H = O.map_and_histogram(inp.points[s:e], inp.offsets[lo:hi + 1] - s, inp.weights[s:e],
                                   inp.anchors)
        return torch.from_numpy(H.astype(np.float32))

    def tiles(H, t0, t1):
        i, j, v = asot.tile_pairs(inp.n_dist, t0, t1)
        out = np.zeros(i.shape[0], np.float32)
        if v.any():
            c, _ = O.pair_costs(H.numpy().astype(np.float64), inp.cost, inp.eps, inp.iters,
                                i[v].astype(np.int64), j[v].astype(np.int64))
            out[v] = c
        return torch.from_numpy(out)

    def unpack(packed, t0, t1, D):
        i, j, v = asot.tile_pairs(inp.n_dist, t0, t1)
        p = packed.numpy()
        D[i[v], j[v]] = torch.from_numpy(p[v])
        D[j[v], i[v]] = torch.from_numpy(p[v])

    def zero_diag(D):
        D.fill_diagonal_(0.0)

    return DistSteps(map_range, tiles, unpack, zero_diag)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2310_16123_b200 as asot
        from paper_2310_16123_b200.distributed import distance_matrix_distributed

        inp = make_inputs("c1", n_dist=37)
        D = distance_matrix_distributed(inp.n_dist, inp.n_anchors, inp.offsets,
                                        asot.num_tiles(inp.n_dist), _oracle_steps(inp))
        if rank == 0:
            q.put(D.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_distributed_matches_single_process(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    D = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    inp = make_inputs("c1", n_dist=37)
    Do, _, _ = O.distance_matrix(inp.points, inp.offsets, inp.weights, inp.anchors, inp.cost,
                                 inp.eps, inp.iters)
    np.testing.assert_allclose(D, Do.astype(np.float32), rtol=1e-6, atol=0)
    assert np.all(np.diag(D) == 0)


class _SharedP2P:
    """Stand-in for P2PResult: the 'symmetric memory' is CPU shared memory visible to both
    processes; h_peers / root_ptr are the peer tensors themselves (the stand-in steps below
    interpret them)."""

    def __init__(self, H_list, D, rank):
        self.H = H_list[rank]
        self.h_peers = H_list
        self.root_ptr = D
        self.D = D


def _p2p_worker(rank, world, port, q, H_list, D):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2310_16123_b200 as asot
        from paper_2310_16123_b200.distributed import distance_matrix_distributed_p2p

        inp = make_inputs("c1", n_dist=37)
        steps = _oracle_steps(inp)

        def map_range_bcast(lo, hi, peers):      # this rank's rows -> every rank's H
            rows = steps.map_range(lo, hi)
            for Hp in peers:
                Hp[lo:hi] = rows

        def tiles_into(H, t0, t1, Droot):        # this rank's pairs -> rank 0's matrix
            packed = steps.tiles(H, t0, t1)
            steps.unpack(packed, t0, t1, Droot)

        steps.map_range_bcast = map_range_bcast
        steps.tiles_into = tiles_into
        out = distance_matrix_distributed_p2p(inp.n_dist, inp.n_anchors, inp.offsets,
                                              asot.num_tiles(inp.n_dist), steps,
                                              _SharedP2P(H_list, D, rank), device=torch.device("cpu"))
        q.put((rank, None if out is None else out.numpy().copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_p2p_orchestration(world):
    """The fused-exchange path (histogram rows stored into every rank's H, pair results stored into
    rank 0's matrix, barriers, rank-0 diagonal) under gloo with shared-memory stand-ins."""
    inp = make_inputs("c1", n_dist=37)
    H_list = [torch.zeros((inp.n_dist, inp.n_anchors), dtype=torch.float32).share_memory_()
              for _ in range(world)]
    D = torch.full((inp.n_dist, inp.n_dist), -1.0, dtype=torch.float32).share_memory_()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_p2p_worker, args=(r, world, port, q, H_list, D)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(res[r] is None for r in range(1, world))
    Do, _, H_o = O.distance_matrix(inp.points, inp.offsets, inp.weights, inp.anchors, inp.cost,
                                   inp.eps, inp.iters)
    for Hr in H_list:                             # every rank holds the full H
        np.testing.assert_array_equal(Hr.numpy(), H_o.astype(np.float32))
    np.testing.assert_allclose(res[0], Do.astype(np.float32), rtol=1e-6, atol=0)
    assert np.all(np.diag(res[0]) == 0)


def test_partitions():
    from paper_2310_16123_b200.distributed import partition_by_points, partition_even
    for n in (0, 1, 7, 100):
        for w in (1, 2, 3, 8):
            r = partition_even(n, w)
            assert r[0][0] == 0 and r[-1][1] == n
            assert all(a <= b for a, b in r) and all(r[k][1] == r[k + 1][0] for k in range(w - 1))
            assert max(b - a for a, b in r) - min(b - a for a, b in r) <= 1
    offs = np.concatenate([[0], np.cumsum(np.random.default_rng(0).integers(1, 50, 200))])
    for w in (1, 2, 4, 8):
        r = partition_by_points(offs, w)
        assert r[0][0] == 0 and r[-1][1] == 200
        loads = [offs[b] - offs[a] for a, b in r]
        assert max(loads) - min(loads) <= 2 * 50 + offs[-1] // w // 10 + 1
