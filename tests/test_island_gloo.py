"""Island-model host logic on CPU: world_size 2 over gloo.  Each rank owns a
stand-in colony (the device colony exposes the same best()/set_best()
contract); after the exchange every rank holds the strictly best tour, ties go
to the lowest rank, and a worse import is never adopted."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1605_02669_b200.island import NO_KEY, decode_key, exchange_host, exchange_key


class FakeColony:
    def __init__(self, order, length):
        self.order, self.length, self.adopted = np.asarray(order, np.uint32), int(length), 0

    def best(self):
        return self.order.copy(), self.length

    def set_best(self, order, length):
        if length < self.length:
            self.order, self.length = np.asarray(order, np.uint32), int(length)
            self.adopted += 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, lens, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n = 12
    rng = np.random.default_rng(rank)
    col = FakeColony(rng.permutation(n), lens[rank])
    g1 = exchange_host(col, dist)
    order1, len1 = col.best()
    col.length = lens[rank] + 1000 if rank == 0 else col.length  # rank 0 degrades locally...
    g2 = exchange_host(col, dist)                                 # ...and re-imports the best
    q.put((rank, g1, len1, order1.tolist(), g2, col.length, col.adopted))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("lens", [(500, 400), (400, 500), (450, 450)])
def test_exchange_two_ranks(lens):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, lens, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    best = min(lens)
    winner = int(np.argmin(lens))  # ties -> lowest rank
    for rank, g1, len1, order1, g2, len2, adopted in res:
        # strict adoption: on a tie every colony keeps its own tour
        keep = lens[rank] == best
        want_tour = np.random.default_rng(rank if keep else winner).permutation(12).tolist()
        assert g1 == best and len1 == best and order1 == want_tour
        assert g2 == best and len2 == best


def test_exchange_key_order():
    assert exchange_key(5, 3) < exchange_key(6, 0)
    assert exchange_key(5, 0) < exchange_key(5, 1)
    assert exchange_key(5, 300) < exchange_key(6, 0)  # 16-bit ranks (> 256 ranks)
    assert decode_key(exchange_key(12345, 4000)) == (4000, 12345)
    with pytest.raises(ValueError):
        exchange_key(5, 1 << 16)
    # a colony without a tour (LLONG_MAX sentinel) never wins and adopts nothing
    assert exchange_key((1 << 63) - 1, 0) == NO_KEY
    assert exchange_key(10**9, 7) < NO_KEY
    assert decode_key(NO_KEY) == (None, None)


def _worker_empty(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # rank 1 has not iterated yet (sentinel length); rank 0 has a tour
    length = 700 if rank == 0 else (1 << 63) - 1
    col = FakeColony(np.arange(10)[::-1] if rank == 0 else np.zeros(10), length)
    g = exchange_host(col, dist)
    q.put((rank, g, col.length, col.best()[0].tolist()))
    dist.barrier()
    dist.destroy_process_group()


def test_exchange_before_first_iteration():
    """a rank still holding the LLONG_MAX sentinel must not win."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_empty, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, g, length, order in res:
        assert g == 700 and length == 700 and order == list(range(10))[::-1]
