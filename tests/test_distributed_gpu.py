"""The one-call multi-rank solve executed end to end: two processes on the one GPU of the
test box, a gloo process group, and the library's exchange callback staging the bracket
records and the eigenvalues through host memory (distributed.host_exchange) -- the same
library path an NCCL communicator takes, with the all-gather done by the callback.  The
union of the ranks' columns must equal the single-process solve bit for bit.
Also: an in-library NCCL communicator (mr3_nccl_comm_init) at world size 1."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _make(name):
    import synth
    return {"legendre3000": lambda: synth.legendre(3000),
            "glued30": lambda: synth.glued_wilkinson(30, 21),
            "uniform2000": lambda: synth.random_uniform(2000, 5),
            "f32": lambda: synth.random_normal_f32(4000, 2, 1, 600)}[name]()


def _worker(rank, world, port, name, exchange, params, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1304_1864_b200 as mr3
        torch.cuda.set_device(0)
        for k, v in params.items():
            mr3.set_param(k, v, 1 if name == "f32" else 0)
        p = _make(name)
        d = torch.from_numpy(p.d).cuda()
        e = torch.from_numpy(p.e).cuda()
        w, Z, (c0, c1), st = mr3.solve_distributed(d, e, "V", p.range, p.il, p.iu,
                                                   exchange=exchange)
        torch.cuda.synchronize()
        q.put((rank, w.cpu().numpy(), Z.cpu().numpy(), c0, c1, None))
    except Exception as ex:  # pragma: no cover
        import traceback
        q.put((rank, None, None, 0, 0, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def _run_world(name, world, exchange, params=None):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, exchange, params or {}, q))
             for r in range(world)]
    for pr in procs:
        pr.start()
    out = [q.get(timeout=600) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=120)
    for r in out:
        assert r[5] is None, r[5]
    return sorted(out, key=lambda t: t[0])


@pytest.mark.parametrize("name,params,exchange", [("legendre3000", {"GROUPS": 1}, "host"),
                                                  ("glued30", {}, "host"),
                                                  ("uniform2000", {}, "torch"),
                                                  ("f32", {}, "host")])
def test_two_process_solve_bitwise(name, params, exchange):
    import paper_1304_1864_b200 as mr3
    p = _make(name)
    mode = 1 if name == "f32" else 0
    for k, v in params.items():
        mr3.set_param(k, v, mode)
    try:
        fn = mr3.mr3_sstemr_d if mode else mr3.mr3_dstemr_dd
        w1, Z1, _ = fn(torch.from_numpy(p.d).cuda(), torch.from_numpy(p.e).cuda(), "V", p.range,
                       p.il, p.iu)
        w1, Z1 = w1.cpu().numpy(), Z1.cpu().numpy()
    finally:
        for k in params:
            mr3.set_param(k, -1, mode)
    res = _run_world(name, 2, exchange, params)
    m = w1.shape[0]
    cols = np.zeros((p.n, m), dtype=Z1.dtype)
    prev = 0
    for rank, w, Z, c0, c1, _ in res:
        np.testing.assert_array_equal(w, w1)  # every rank holds all eigenvalues
        assert c0 == prev and Z.shape == (p.n, c1 - c0)
        cols[:, c0:c1] = Z
        prev = c1
    assert prev == m
    np.testing.assert_array_equal(cols, Z1)


def test_nccl_communicator_world1():
    """An in-library NCCL communicator (lazily loaded libnccl.so.2) on a one-rank context
    gives the plain single-GPU result."""
    import ctypes

    import paper_1304_1864_b200 as mr3
    import synth
    L = mr3.lib()
    uid = ctypes.create_string_buffer(128)
    assert L.mr3_nccl_unique_id(uid) == 0
    comm = ctypes.c_void_p()
    assert L.mr3_nccl_comm_init(ctypes.byref(comm), uid, 0, 1, 0) == 0
    h = ctypes.c_void_p()
    st = torch.cuda.current_stream()
    assert L.mr3_create(ctypes.byref(h), 0, ctypes.c_void_p(int(st.cuda_stream) or 1), comm, 0,
                        1) == 0
    p = synth.random_uniform(600, 3)
    d = torch.from_numpy(p.d).cuda()
    e = torch.from_numpy(p.e).cuda()
    w = torch.zeros(p.n, dtype=torch.float64, device="cuda")
    Zs = torch.zeros((p.n, p.n), dtype=torch.float64, device="cuda")
    m, zb, ze = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    rc = L.mr3_dstemr_dd(h, b"V", b"A", p.n, ctypes.c_void_p(d.data_ptr()),
                         ctypes.c_void_p(e.data_ptr()), 0.0, 0.0, 1, p.n, ctypes.byref(m),
                         ctypes.c_void_p(w.data_ptr()), ctypes.c_void_p(Zs.data_ptr()), p.n, p.n,
                         ctypes.byref(zb), ctypes.byref(ze), None)
    assert rc == 0 and m.value == p.n and (zb.value, ze.value) == (0, p.n)
    w0, Z0, _ = mr3.mr3_dstemr_dd(d, e)
    assert torch.equal(w, w0) and torch.equal(Zs.T, Z0)
    L.mr3_destroy(h)
    assert L.mr3_nccl_comm_destroy(comm) == 0


def test_bench_two_ranks_gloo_json_line():
    """The driver's N > 1 launch of bench.py (torch.distributed.run, one rank per process) on
    the multi-rank path, as a logic test: two ranks share the one GPU over gloo (host-staged
    exchange).  Rank 0 prints ONE JSON line with the contract's keys, the N-rank e2e among them."""
    import json
    import subprocess
    import sys
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "2", "--warmup", "1",
           "--backend", "gloo", "--config", "2", "--no-cpu"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    j = json.loads(lines[0])
    assert j["n_gpus"] == 2 and j["steps"] == 2 and j["value"] > 0
    assert j["unit"] == "eigenpairs/s" and j["scaling"] == "strong"
    assert j["config"]["parallelism"].endswith("x2")
    e = j["e2e"]
    n, m = j["config"]["n"], j["config"]["m"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == 2 * (2 * n - 1) * 8
    # both ranks read all of w and, together, every column of Z exactly once
    assert e["d2h_bytes_per_step"] == (2 * m + m * n) * 8
    assert j["gpu_launches"] > 0 and "roofline" in j and "clocks" in j
