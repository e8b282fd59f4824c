"""Worker of tests/test_gpu_multi.py (test infrastructure): one process per GPU under
torch.distributed.run; every rank solves the same LPs with its column slab and rank 0 compares
the replicated results with the CPU oracle bit for bit.  Exit code 0 = all equal."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import lpgen  # noqa: E402
import oracle  # noqa: E402
import paper_2211_10979_b200 as sx  # noqa: E402
from lpgen import fixtures as F  # noqa: E402


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cases = [("dense", lpgen.dense_lp(300, 400, 3)), ("klee_minty", F.klee_minty(8))]
    A, b, c = lpgen.dense_lp(120, 150, 7)
    b = b.copy()
    b[::5] = -b[::5] / 40.0                                  # Phase I rows
    cases.append(("phase1", (A, b, c)))
    failed = []
    for exchange in (0, 1):                                  # peer memory (auto), NCCL allgather
        for look in (1, 16):
            for overlap in (True, False):
                for name, (A, b, c) in cases:
                    with sx.Simplex(A, b, c, group=dist.group.WORLD, device=local, lookahead=look,
                                    exchange=exchange, overlap=overlap) as s:
                        st = s.solve()
                        x, y, obj, piv, _ = s.solution()
                        k, r = s.trace()
                    if rank == 0:
                        o = oracle.solve_2phase(A, b, c) if (b < 0).any() else oracle.solve(A, b, c)
                        ok = (st == o.status and piv == o.pivots and np.array_equal(k, o.trace_k)
                              and np.array_equal(r, o.trace_r) and obj == o.objective
                              and np.array_equal(x, o.x) and np.array_equal(y, o.y))
                        if not ok:
                            failed.append((name, exchange, look, overlap))
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0:
        print("FAILED" if failed else "OK", failed, flush=True)
        sys.exit(1 if failed else 0)


if __name__ == "__main__":
    main()
