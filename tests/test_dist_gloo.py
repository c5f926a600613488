"""N>1 host path on CPU: world_size-2 gloo process group, shards computed by the oracle, one
all_reduce, finalised by the library's host-side sre_finalize (no GPU needed)."""
import os
import socket

import numpy as np
import pytest

import sre_inputs as si

torch = pytest.importorskip("torch")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, alphas, out_q):
    import torch.distributed as dist

    import oracle
    import paper_2601_07824_b200 as sre
    from paper_2601_07824_b200 import dist as sdist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    psi = si.haar(n, 777)

    def part(lo, hi):
        return torch.from_numpy(oracle.sums_fwht(psi, alphas, a_range=(lo, hi))).reshape(1, -1)

    def allreduce(t):
        dist.all_reduce(t, op=dist.ReduceOp.SUM)

    m, ln = sdist.exact_sharded(n, alphas, rank, world, part, allreduce, lambda s: sre.finalize(s.numpy(), n, alphas))
    out_q.put((rank, m.tolist(), float(ln[0])))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_sharded_equals_single(world):
    import torch.multiprocessing as mp

    import oracle
    oracle.build()
    n, alphas = 9, [1.0, 2.0, 3.0]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, alphas, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref_m, ref_ln = oracle.sre(si.haar(n, 777), alphas, "fwht")
    for _, m, ln in res:
        assert np.max(np.abs(np.array(m[0]) - np.array(ref_m))) < 1e-12
        assert abs(ln - ref_ln) < 1e-13


def test_shard_plan_partitions():
    from paper_2601_07824_b200.dist import shard_range
    for n in (1, 3, 10, 20):
        for world in (1, 2, 3, 4, 5, 8):
            if world > (1 << n):
                continue
            rs = [shard_range(n, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == 1 << n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in rs]
            assert max(sizes) - min(sizes) <= 1


def _mana_worker(rank, world, port, n, out_q):
    import torch.distributed as dist

    from oracle import mana as om
    from paper_2601_07824_b200 import dist as sdist
    import sre_inputs.qutrit as sq

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    psi = sq.brickwall(n, 3, 778)

    def part(lo, hi):
        return torch.from_numpy(om.sums_fwht(psi, (lo, hi)))

    def allreduce(t):
        dist.all_reduce(t, op=dist.ReduceOp.SUM)

    m, n2 = sdist.mana_sharded(n, rank, world, part, allreduce)
    out_q.put((rank, m, n2))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_mana_sharded_equals_single(world):
    """NEXT-3 shards: 3^N X-strings split over ranks, one all_reduce of the two sums."""
    import torch.multiprocessing as mp

    from oracle import mana as om
    import sre_inputs.qutrit as sq
    from paper_2601_07824_b200 import dist as sdist
    n = 5
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_mana_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    ref = om.mana(sq.brickwall(n, 3, 778))
    for _, m, n2 in res:
        assert m == pytest.approx(ref, abs=1e-12) and n2 == pytest.approx(1.0, abs=1e-12)
    bounds = [sdist.shard_bounds(3 ** n, r, world) for r in range(world)]
    assert bounds[0][0] == 0 and bounds[-1][1] == 3 ** n
    assert all(bounds[i][1] == bounds[i + 1][0] for i in range(world - 1))


def _batch_worker(rank, world, port, n, b, alphas, out_q):
    import torch.distributed as dist

    import oracle
    import paper_2601_07824_b200 as sre
    from paper_2601_07824_b200 import dist as sdist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    batch = si.haar_batch(n, b, 779)
    seen = []

    def part(s0, s1):
        seen.append((s0, s1))
        return torch.from_numpy(np.stack([oracle.sums_fwht(batch[s], alphas) for s in range(s0, s1)]))

    def allreduce(t):
        dist.all_reduce(t, op=dist.ReduceOp.SUM)

    m, ln = sdist.exact_batched_sharded(n, b, alphas, rank, world, part, allreduce,
                                        lambda s: sre.finalize(s.numpy(), n, alphas),
                                        lambda bb, k: torch.zeros((bb, k), dtype=torch.float64))
    out_q.put((rank, m.tolist(), ln.tolist(), seen))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_state_sharded_batch(world):
    """Batched variant sharded by state: 5 states over 2 or 3 ranks (ragged shards), one
    all_reduce of the zero-padded [B, n_alpha+2] sums; every rank returns the whole batch's M."""
    import torch.multiprocessing as mp

    import oracle
    oracle.build()
    n, b, alphas = 6, 5, [1.0, 2.0]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_batch_worker, args=(r, world, port, n, b, alphas, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    batch = si.haar_batch(n, b, 779)
    ref = [oracle.sre(batch[s], alphas, "fwht") for s in range(b)]
    shards = sorted(sh for _, _, _, seen in res for sh in seen)
    assert shards[0][0] == 0 and shards[-1][1] == b and all(shards[i][1] == shards[i + 1][0] for i in range(len(shards) - 1))
    for _, m, ln, _ in res:
        for s in range(b):
            assert np.max(np.abs(np.array(m[s]) - np.array(ref[s][0]))) < 1e-12
            assert abs(ln[s] - ref[s][1]) < 1e-13
