"""One rank of the sharded two-level AT-MGRIT cycle over torch.distributed
(gloo, CPU).  The SCHEDULE -- owned ranges, halo partners, window payload
blocks -- comes from the product library's host code (atm_rank_ranges,
atm_window_recvs); the arithmetic is the oracle's.  This restates the
reference's WorkerExecution (parallel.cpp:198-310): halo before every
F-sweep, one window exchange per iteration, per-point squares gathered to
rank 0 and summed in point order.

Usage (spawned by tests/test_dist_gloo.py):
    python tests/dist_worker.py RANK WORLD PORT OUT.json
"""
import json
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2107_09596_b200 as T  # noqa: E402
from helpers import oracle_driver  # noqa: E402

CASE = dict(problem="heat1d", n=9, tf=2.0, n_points=65, m=4, k=3, guess="random", seed=71,
            tol=1e-9, max_iters=40)


def main():
    rank, world, port, out = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], sys.argv[4]
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    hier = T.build_hierarchy(T.TimeGrid.make(0.0, CASE["tf"], CASE["n_points"]), [CASE["m"]],
                             CASE["k"])
    rr = T.rank_ranges(hier, world, rank)
    recvs = {q: T.window_recvs(hier, world, q) for q in range(world)}
    orc = oracle_driver(CASE)
    orc.setup()
    u0, r1 = orc.array(0), orc.array(1, "r")
    m = CASE["m"]
    lo0, hi0 = rr["lo"][0], rr["hi"][0]
    lo1, hi1 = rr["lo"][1], rr["hi"][1]

    def halo():
        # sync_left_edge (parallel.cpp:236-249)
        reqs = []
        if rr["right_dst"][0] >= 0:
            reqs.append(dist.isend(torch.from_numpy(u0[hi0].copy()), rr["right_dst"][0]))
        if lo0 > 0 and rr["left_src"][0] >= 0:
            buf = torch.zeros(u0.shape[1], dtype=torch.float64)
            dist.recv(buf, rr["left_src"][0])
            u0[lo0 - 1] = buf.numpy()
        for q in reqs:
            q.wait()

    def window_exchange():
        reqs = []
        for q, triples in recvs.items():
            for (src, first, count) in triples:
                if src == rank:
                    reqs.append(dist.isend(torch.from_numpy(r1[first:first + count].copy()), q))
        for (src, first, count) in recvs[rank]:
            buf = torch.zeros((count, r1.shape[1]), dtype=torch.float64)
            dist.recv(buf, src)
            r1[first:first + count] = buf.numpy()
        for q in reqs:
            q.wait()

    def norm():
        # reduce_norm (parallel.cpp:279-295): per-point squares in point order
        res = orc.residual(0, lo0, hi0 - lo0 + 1)
        sq = []
        for row in res:
            s = 0.0
            for v in row:
                s += v * v
            sq.append(s)
        parts = [None] * world
        dist.all_gather_object(parts, sq)
        tot = 0.0
        for part in parts:
            for v in part:
                tot += v
        return math.sqrt(tot)

    history = []
    for _ in range(CASE["max_iters"]):
        halo()
        orc.f_relax(0, rr["iv_first"][0], rr["iv_count"][0])
        for j in range(rr["c_first"][0], rr["c_first"][0] + rr["c_count"][0]):
            r1[j] = orc.residual(0, j * m, 1)[0]
        window_exchange()
        for p in range(lo1, hi1 + 1):
            lo = max(0, p - CASE["k"] + 1)
            u0[p * m] += orc.window_linear(1, lo, r1[lo:p + 1])
        halo()
        orc.f_relax(0, rr["iv_first"][0], rr["iv_count"][0])
        nv = norm()
        history.append(nv)
        if nv <= CASE["tol"]:
            break
    parts = [None] * world
    dist.all_gather_object(parts, u0[lo0:hi0 + 1].tolist())
    if rank == 0:
        json.dump(dict(history=history, u=[row for part in parts for row in part]), open(out, "w"))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
