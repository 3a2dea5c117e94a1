"""One rank of test_gpu_island.test_two_rank_real_colonies_gloo: a real
Colony on cuda:0, host exchange over gloo (RANK / WORLD_SIZE / MASTER_* from
the environment, as torchrun sets them).  Writes its observations as JSON."""
import json
import os
import sys

import torch.distributed as dist  # first: torch before anything that could load another libnccl

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
import paper_1605_02669_b200 as acs  # noqa: E402
from paper_1605_02669_b200.island import exchange_host  # noqa: E402


def main(out_path):
    dist.init_process_group("gloo")
    rank = dist.get_rank()
    I = O.load("pcb442")
    inst = acs.TspInstance(I.name, I.type, I.xs.copy(), I.ys.copy())
    out = {}
    with acs.Colony(inst, acs.AcsParams(variant="relaxed", seed=100 + rank, m=64)) as col:
        st = col.iterate(2 + 3 * rank)  # rank 1 runs longer
        out["own"] = int(col.best()[1])
        g = exchange_host(col, dist)
        order, ln = col.best()
        out["g"], out["len"], out["tour"] = int(g), int(ln), order.tolist()
        st2 = col.iterate(3)
        out["trace"] = st["global_best_len"].tolist() + st2["global_best_len"].tolist()
        # a tie: both ranks hold the same (better) length -> nobody adopts (strict)
        ident = np.arange(I.n, dtype=np.uint32)
        col.set_best(ident if rank == 0 else ident[::-1].copy(), 1000)
        out["tie_g"] = int(exchange_host(col, dist))
        out["tie_tour0"] = int(col.best()[0][0])
    with open(out_path, "w") as f:
        json.dump(out, f)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1])
