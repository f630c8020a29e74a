"""Index-set partition of the solve over ranks (one GPU per rank).

SURVEY.md 8(e) / BJ:5: every rank builds the same root representation, bisects a static
slice of the requested index set, the bracket records are all-gathered, every rank
classifies the whole set identically and takes a cluster-whole range of output columns,
and finally the eigenvalues are all-gathered.  No eigenvector data crosses GPUs: each rank
owns its columns of Z.

Both all-gathers run INSIDE the library's one-call solver (mr3_dstemr_dd / mr3_sstemr_d on
a context created with the rank, the world size and a communicator):
  * NCCL process groups: an in-library NCCL communicator (mr3_nccl_comm_init; the unique id
    is broadcast once per group with torch.distributed), ncclAllGather over NVLink;
  * other backends (gloo; the CPU tests and a one-GPU two-process run): an exchange callback
    (mr3_set_exchange) that all-gathers the library's device buffer through host memory with
    torch.distributed.
The two-phase form (mr3_plan / mr3_execute with the all-gathers done here by
torch.distributed) is kept as `exchange="torch"`.  Nothing numeric happens in this module.
"""
from __future__ import annotations

import ctypes

import torch
import torch.distributed as dist

BRK_REC = 6  # doubles per bracket record (MR3_BRK_REC in include/mr3.h)


class _DevPtr:
    """__cuda_array_interface__ view of a library-owned device buffer."""

    def __init__(self, ptr, n, typestr="<f8"):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


def wrap_device(ptr: int, n: int, device, typestr="<f8") -> torch.Tensor:
    return torch.as_tensor(_DevPtr(ptr, n, typestr), device=device)


def exchange_brackets(buf: torch.Tensor, rank: int, world: int, cap: int, group=None):
    """All-gather equal slices of `buf` (world*cap records of BRK_REC float64) in place."""
    if world == 1:
        return buf
    rec = BRK_REC * cap
    mine = buf[rank * rec:(rank + 1) * rec].clone()
    dist.all_gather_into_tensor(buf[:world * rec], mine, group=group)
    return buf


def gather_columns(w: torch.Tensor, c0: int, c1: int, group=None) -> torch.Tensor:
    """Every rank holds w[c0:c1] (its own column range) of a length-m vector;
    returns the full vector on every rank (all-gather of padded slices)."""
    world = dist.get_world_size(group)
    if world == 1:
        return w
    dev = w.device
    rng = torch.tensor([c0, c1], dtype=torch.int64, device=dev)
    allr = torch.empty(2 * world, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(allr, rng, group=group)
    allr = allr.view(world, 2).cpu().tolist()
    cap = max(max(b - a for a, b in allr), 1)
    mine = torch.zeros(cap, dtype=w.dtype, device=dev)
    mine[:c1 - c0] = w[c0:c1]
    buf = torch.empty(world * cap, dtype=w.dtype, device=dev)
    dist.all_gather_into_tensor(buf, mine, group=group)
    out = w.clone()
    for r, (a, b) in enumerate(allr):
        out[a:b] = buf[r * cap:r * cap + (b - a)]
    return out


def host_exchange(group=None):
    """An mr3_allgather_fn that all-gathers the library's device buffer through host memory
    with torch.distributed (any backend; gloo in the tests).  Keep the returned object alive
    while the context uses it."""

    def fn(user, buf, nbytes, rank, world, stream):
        try:
            torch.cuda.synchronize()  # the library's work on its stream is complete
            dev = torch.device("cuda", torch.cuda.current_device())
            full = wrap_device(buf, world * nbytes, dev, "|u1")
            mine = full[rank * nbytes:(rank + 1) * nbytes].cpu()
            parts = [torch.empty(nbytes, dtype=torch.uint8) for _ in range(world)]
            dist.all_gather(parts, mine, group=group)
            full.copy_(torch.cat(parts).to(dev))
            torch.cuda.synchronize()
            return 0
        except Exception:  # pragma: no cover - reported as MR3_ERR_NCCL by the library
            return 1

    from . import EXCHANGE_FN
    return EXCHANGE_FN(fn)


_dist_ctx: dict = {}


def _dist_context(device, group, exchange):
    """A library context for this rank of `group` (cached): NCCL communicator or callback."""
    from . import MR3Error, _params, lib, PARAMS
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    backend = dist.get_backend(group)
    if exchange == "auto":
        exchange = "nccl" if backend == "nccl" else "host"
    dev = torch.cuda.current_device() if device is None else int(device)
    st = torch.cuda.current_stream(dev)
    sh = int(st.cuda_stream) or 1
    key = (dev, sh, id(group), rank, world, exchange)
    ent = _dist_ctx.get(key)
    if ent is None:
        L = lib()
        comm = ctypes.c_void_p()
        keep = None
        if exchange == "nccl" and world > 1:
            uid = ctypes.create_string_buffer(128)
            if rank == 0:
                rc = L.mr3_nccl_unique_id(uid)
                if rc:
                    raise MR3Error(rc, "mr3_nccl_unique_id")
            obj = [uid.raw if rank == 0 else None]
            dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group else 0,
                                       group=group)
            uid = ctypes.create_string_buffer(obj[0], 128)
            rc = L.mr3_nccl_comm_init(ctypes.byref(comm), uid, rank, world, dev)
            if rc:
                raise MR3Error(rc, "mr3_nccl_comm_init")
        h = ctypes.c_void_p()
        rc = L.mr3_create(ctypes.byref(h), dev, ctypes.c_void_p(sh),
                          comm if comm.value else None, rank, world)
        if rc:
            raise MR3Error(rc, "mr3_create")
        if exchange == "host" and world > 1:
            keep = host_exchange(group)
            L.mr3_set_exchange(h, keep, None)
        ent = (h, comm, keep)
        _dist_ctx[key] = ent
    h = ent[0]
    for mode in (0, 1):
        for k, v in _params[mode].items():
            lib().mr3_set_param(h, mode, PARAMS[k], float(v))
    return h


def solve_distributed(d, e, jobz="V", range="A", il=1, iu=0, vl=0.0, vu=0.0, group=None,
                      exchange="auto"):
    """Multi-rank solve: one library call per rank.  Returns (w[m] on every rank,
    Z_local[n, c1-c0] (this rank's columns c0..c1-1 of the global m), (c0, c1), stats).

    exchange: "auto" (NCCL communicator for NCCL groups, host callback otherwise), "nccl",
    "host", or "torch" (two-phase mr3_plan / mr3_execute with torch.distributed all-gathers).
    """
    if exchange == "torch":
        return _solve_two_phase(d, e, jobz, range, il, iu, vl, vu, group)
    from . import MR3Error, Stats, _err, lib
    if not dist.is_initialized():
        from . import _solve
        w, Z, st = _solve(0 if d.dtype == torch.float64 else 1, d, e, jobz, range, il, iu, vl, vu)
        return w, Z, (0, w.numel()), st
    mode = 0 if d.dtype == torch.float64 else 1
    d = d.contiguous()
    e = e.contiguous()
    n = d.numel()
    from . import _used
    c = _used(_dist_context(d.device.index, group, exchange))
    fn = lib().mr3_dstemr_dd if mode == 0 else lib().mr3_sstemr_d
    w = torch.zeros(max(n, 1), dtype=d.dtype, device=d.device)
    m = ctypes.c_int64(0)
    zb, ze = ctypes.c_int64(0), ctypes.c_int64(0)
    st = Stats()

    def call(Zt, zcap):
        return fn(c, jobz.encode(), range.encode(), n, ctypes.c_void_p(d.data_ptr()),
                  ctypes.c_void_p(e.data_ptr() if n > 1 else d.data_ptr()), vl, vu, il, iu,
                  ctypes.byref(m), ctypes.c_void_p(w.data_ptr()),
                  ctypes.c_void_p(Zt.data_ptr() if Zt is not None else 0), max(n, 1), zcap,
                  ctypes.byref(zb), ctypes.byref(ze), ctypes.byref(st))

    Zs = None
    if jobz == "V":
        # a rank's cluster-whole share is at most ceil(m/world) + the largest cluster; start
        # from twice the even share and size exactly on MR3_ERR_ZCAP (every rank retries
        # together: the partition is identical on all ranks)
        world = dist.get_world_size(group)
        mcap = n if range != "I" else max(0, min(iu, n) - max(il, 1) + 1)
        cap = min(mcap, 2 * ((mcap + world - 1) // world) + 64)
        Zs = torch.empty((max(cap, 1), max(n, 1)), dtype=d.dtype, device=d.device)
        rc = call(Zs, cap)
        if rc == 6:  # (collective: every rank returns MR3_ERR_ZCAP together, ranges filled)
            cap = max(ze.value - zb.value, 1)
            Zs = torch.empty((cap, max(n, 1)), dtype=d.dtype, device=d.device)
            rc = call(Zs, cap)
    else:
        rc = call(None, 0)
    _err(c, rc, "mr3_dstemr_dd" if mode == 0 else "mr3_sstemr_d")
    mm = m.value
    Z = Zs[:ze.value - zb.value].T if Zs is not None else None
    if MR3Error is None:  # pragma: no cover
        pass
    return w[:mm], Z, (zb.value, ze.value), st.asdict()


def _solve_two_phase(d, e, jobz, range, il, iu, vl, vu, group):
    """mr3_plan + torch.distributed all-gather of the bracket records + mr3_execute + all-gather
    of w (the collectives in Python; kept for comparison and for callers that own them)."""
    from . import Stats, _ctx, _err, lib

    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    mode = 0 if d.dtype == torch.float64 else 1
    d = d.contiguous()
    e = e.contiguous()
    n = d.numel()
    from . import _used
    c = _used(_ctx(d.device.index))
    m = ctypes.c_int64(0)
    brk = ctypes.c_void_p()
    cap = ctypes.c_int64(0)
    cnt = ctypes.c_int64(0)
    rc = lib().mr3_plan(c, mode, range.encode(), n, ctypes.c_void_p(d.data_ptr()),
                        ctypes.c_void_p(e.data_ptr()), float(vl), float(vu), il, iu, rank, world,
                        ctypes.byref(m), ctypes.byref(brk), ctypes.byref(cap), ctypes.byref(cnt))
    _err(c, rc, "mr3_plan")
    if brk.value and world > 1:
        torch.cuda.synchronize()
        buf = wrap_device(brk.value, world * cap.value * BRK_REC, d.device)
        if dist.get_backend(group) == "nccl":
            exchange_brackets(buf, rank, world, cap.value, group)
        else:  # host staging for CPU backends
            hb = buf.cpu()
            exchange_brackets(hb, rank, world, cap.value, group)
            buf.copy_(hb.to(d.device))
        torch.cuda.synchronize()
    w = torch.zeros(max(n, 1), dtype=d.dtype, device=d.device)
    zb, ze = ctypes.c_int64(0), ctypes.c_int64(0)
    st = Stats()
    Z = None
    if jobz == "V":
        rc = lib().mr3_execute(c, b"V", ctypes.c_void_p(w.data_ptr()), None, max(n, 1), 0,
                               ctypes.byref(zb), ctypes.byref(ze), ctypes.byref(st))
        if rc not in (0, 6):
            _err(c, rc, "mr3_execute")
        if rc == 6:
            Zs = torch.empty((max(ze.value - zb.value, 1), max(n, 1)), dtype=d.dtype,
                             device=d.device)
            rc = lib().mr3_execute(c, b"V", ctypes.c_void_p(w.data_ptr()),
                                   ctypes.c_void_p(Zs.data_ptr()), max(n, 1), ze.value - zb.value,
                                   ctypes.byref(zb), ctypes.byref(ze), ctypes.byref(st))
            _err(c, rc, "mr3_execute")
            Z = Zs[:ze.value - zb.value].T
        else:
            Z = torch.empty((n, 0), dtype=d.dtype, device=d.device)
    else:
        rc = lib().mr3_execute(c, b"N", ctypes.c_void_p(w.data_ptr()), None, max(n, 1), 0,
                               ctypes.byref(zb), ctypes.byref(ze), ctypes.byref(st))
        _err(c, rc, "mr3_execute")
    mm = m.value if m.value >= 0 else ze.value
    if dist.is_initialized() and world > 1:
        mt = torch.tensor([ze.value], dtype=torch.int64)
        if dist.get_backend(group) == "nccl":
            mt = mt.to(d.device)
        dist.all_reduce(mt, op=dist.ReduceOp.MAX, group=group)
        mm = max(mm, int(mt.item()))
        if dist.get_backend(group) == "nccl":
            w = gather_columns(w[:mm], zb.value, ze.value, group)
        else:
            w = gather_columns(w[:mm].cpu(), zb.value, ze.value, group).to(d.device)
    else:
        w = w[:mm]
    return w, Z, (zb.value, ze.value), st.asdict()
