"""World-size-2 gloo tests (CPU) of the multi-rank glue: the in-place bracket
all-gather, the cluster-whole column partition computed identically on every
rank, and the all-gather of variable column ranges of w."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        import oracle
        import paper_1304_1864_b200 as mr3
        import synth
        from paper_1304_1864_b200.distributed import BRK_REC as RB
        from paper_1304_1864_b200.distributed import exchange_brackets, gather_columns

        p = synth.glued_wilkinson(6, 21)
        n = p.n
        cap = (n + world - 1) // world
        buf = torch.full((world * cap * RB,), float("nan"), dtype=torch.float64)
        # this rank's static slice: brackets from the oracle's eigenvalues (stand-in for K2)
        first, cnt = rank * cap, min(cap, n - rank * cap)
        lh, ll = oracle.eigvals(p.d, p.e, np.arange(first + 1, first + cnt + 1))
        rec = buf[rank * cap * RB:(rank * cap + cnt) * RB].view(cnt, RB)
        rec[:, 0] = torch.from_numpy(lh - 1e-12 * np.abs(lh))
        rec[:, 2] = torch.from_numpy(lh + 1e-12 * np.abs(lh))
        rec[:, 1] = 0
        rec[:, 3] = 0
        rec[:, 4] = torch.from_numpy(lh)  # Newton estimate
        rec[:, 5] = 0
        exchange_brackets(buf, rank, world, cap, None)
        allrec = buf[:n * RB].view(n, RB).numpy()
        assert np.all(np.isfinite(allrec))
        # classification (reldist >= gaptol) of the gathered brackets, identical on all ranks
        lo, hi = allrec[:, 0], allrec[:, 2]
        gap = lo[1:] - hi[:-1]
        den = np.maximum.reduce([np.abs(lo[1:]), np.abs(hi[1:]), np.abs(lo[:-1]), np.abs(hi[:-1])])
        starts = np.concatenate([[0], np.nonzero(gap >= 1e-10 * den)[0] + 1])
        sb = np.concatenate([starts, [n]])
        sizes = np.diff(sb)
        cost = sizes * np.where(sizes > 1, 3.0, 1.0)
        cb = mr3.partition_columns(sb, cost, world)
        allcb = [torch.zeros(world + 1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(allcb, torch.from_numpy(cb))
        for c in allcb:
            assert c.tolist() == cb.tolist()
        assert set(cb.tolist()) <= set(sb.tolist())  # never inside a cluster
        c0, c1 = int(cb[rank]), int(cb[rank + 1])
        w = torch.zeros(n, dtype=torch.float64)
        w[c0:c1] = torch.from_numpy(lo[c0:c1])
        wf = gather_columns(w, c0, c1, None)
        assert np.array_equal(wf.numpy(), lo)
        q.put((rank, "ok", int(sizes.max())))
    except Exception as ex:  # pragma: no cover
        import traceback
        q.put((rank, traceback.format_exc(), 0))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_exchange_partition_gather():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
    for r, msg, big in res:
        assert msg == "ok", msg
        assert big > 1  # glued Wilkinson has clusters at gaptol 1e-10
