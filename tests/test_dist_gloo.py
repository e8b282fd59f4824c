"""Host-side logic of the N > 1 path, world_size 2 over gloo on CPU (-m "not gpu").

The GPU exchange itself (k_pack -> ncclAllGather -> k_select) is covered on one GPU by
tests/test_gpu_parity.py (virtual ranks and a real 1-rank NCCL communicator).  Here:
  * the NCCL id hand-off the binding performs (share_nccl_id over a process group);
  * every rank derives the same column partition and the parts tile the columns;
  * the per-rank Step-1 candidates folded lexicographically equal the sequential
    Step 1 over the whole row, i.e. the protocol
    the device implements is exact, with the oracle's Step 1 on each rank's slab;
  * bench.py's max-over-ranks timing reduction, its sum and gather helpers, and the rank-0-only
    oracle cpu_baseline leg with the other ranks waiting at a barrier.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import lpgen
        import oracle
        import paper_2211_10979_b200 as sx
        out = {}
        # (1) NCCL id hand-off
        nid = sx.share_nccl_id(dist.group.WORLD)
        ids = [None] * world
        dist.all_gather_object(ids, nid)
        out["ids_equal"] = all(i == ids[0] for i in ids) and len(nid) == 128
        # (2) partition of the n+m columns of an LP
        m, n = 37, 53
        c0, w = sx.partition(n + m, world, rank)
        parts = [None] * world
        dist.all_gather_object(parts, (c0, w))
        out["parts"] = parts
        # (3) distributed Step 1 == sequential Step 1, on successive row-0s of a real solve
        A, b, c = lpgen.dense_lp(m, n, 5)
        T, _ = oracle.build_tableau(A, b, c)
        ok = True
        for _ in range(15):
            row0 = T[0, : n + m]
            kk, vv = oracle.price(row0[c0: c0 + w])
            cand = (vv, c0 + kk) if kk >= 0 else (float("inf"), 1 << 62)
            cands = [None] * world
            dist.all_gather_object(cands, cand)
            best = min(cands)                     # lexicographic (value, column) fold
            k_seq, _ = oracle.price(row0)
            k_dist = best[1] if best[0] != float("inf") else -1
            ok &= (k_dist == k_seq)
            if k_seq < 0:
                break
            r, _ = oracle.ratio(T, k_seq)
            oracle.pivot(T, r, k_seq)
        out["fold_ok"] = ok
        # (4) bench timing reduction: max over ranks
        import bench
        out["tmax"] = bench.reduce_max(10.0 * (rank + 1), world, torch.device("cpu"))
        out["tsum"] = bench.reduce_sum(1.5 * (rank + 1), world, torch.device("cpu"))
        # (5) the per-rank roofline fractions gathered to every rank (bench.gather_list)
        out["fracs"] = bench.gather_list(0.9 + 0.01 * rank, world)
        # (6) the cpu_baseline leg runs on rank 0 only while the others wait at a barrier
        if rank == 0:
            A0, b0, c0_ = lpgen.dense_lp(64, 64, 1)
            out["cpu"] = bench.cpu_baseline(A0, b0, c0_, 0.3)["kind"]
        dist.barrier()
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_world2(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        out = res[r]
        assert out["ids_equal"]
        assert out["fold_ok"]
        assert out["tmax"] == 10.0 * world
        assert out["tsum"] == 1.5 * world * (world + 1) / 2
        assert out["fracs"] == [0.9 + 0.01 * q for q in range(world)]
        assert (out.get("cpu") == "oracle") == (r == 0)
        parts = out["parts"]
        assert parts == res[0]["parts"]
        assert parts[0][0] == 0 and sum(w for _, w in parts) == 37 + 53
        assert all(parts[i][0] + parts[i][1] == parts[i + 1][0] for i in range(world - 1))
