"""Index-set partition of the solve over ranks (one GPU per rank).

SURVEY.md 8(e) / BJ:5: every rank builds the same root representation, bisects
a static slice of the requested index set (mr3_plan), the bracket records are
all-gathered (NCCL over NVLink via torch.distributed), every rank classifies the
whole set identically and takes a cluster-whole range of output columns
(mr3_execute), and finally the eigenvalues are all-gathered.  No eigenvector
data crosses GPUs: each rank owns its columns of Z.

The collectives are the only thing done here; everything numeric runs in the
library.  `exchange_brackets` and `gather_columns` work with any backend (gloo
on CPU tensors in the tests, NCCL on CUDA tensors in production).
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


def wrap_device(ptr: int, n: int, device) -> torch.Tensor:
    return torch.as_tensor(_DevPtr(ptr, n), device=device)


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


def solve_distributed(d, e, jobz="V", range="A", il=1, iu=0, vl=0.0, vu=0.0, group=None):
    """Multi-rank solve.  Returns (w[m] on every rank, Z_local[n, c1-c0], (c0, c1), stats)."""
    from . import MR3Error, Stats, _ctx, _err, lib

    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    mode = 0 if d.dtype == torch.float64 else 1
    d = d.contiguous()
    e = e.contiguous()
    n = d.numel()
    c = _ctx(d.device.index)
    m = ctypes.c_int64(0)
    brk = ctypes.c_void_p()
    cap = ctypes.c_int64(0)
    cnt = ctypes.c_int64(0)
    rc = lib().mr3_plan(c, mode, range.encode(), n, ctypes.c_void_p(d.data_ptr()),
                        ctypes.c_void_p(e.data_ptr()), float(vl), float(vu), il, iu, rank, world,
                        ctypes.byref(m), ctypes.byref(brk), ctypes.byref(cap), ctypes.byref(cnt))
    _err(c, rc, "mr3_plan")
    if brk.value and world > 1:
        buf = wrap_device(brk.value, world * cap.value * BRK_REC, d.device)
        exchange_brackets(buf, rank, world, cap.value, group)
        torch.cuda.current_stream(d.device).synchronize()
    w = torch.zeros(max(n, 1), dtype=d.dtype, device=d.device)
    zb, ze = ctypes.c_int64(0), ctypes.c_int64(0)
    st = Stats()
    Z = None
    zptr, zcap = 0, 0
    if jobz == "V":
        rc = lib().mr3_execute(c, b"V", ctypes.c_void_p(w.data_ptr()), None, max(n, 1), 0,
                               ctypes.byref(zb), ctypes.byref(ze), ctypes.byref(st))
        if rc not in (0, 6):
            _err(c, rc, "mr3_execute")
        if rc == 6:
            Zs = torch.empty((max(ze.value - zb.value, 1), max(n, 1)), dtype=d.dtype,
                             device=d.device)
            zptr, zcap = Zs.data_ptr(), ze.value - zb.value
            rc = lib().mr3_execute(c, b"V", ctypes.c_void_p(w.data_ptr()), ctypes.c_void_p(zptr),
                                   max(n, 1), zcap, ctypes.byref(zb), ctypes.byref(ze),
                                   ctypes.byref(st))
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
        # m for the split case is only known after execute: take it from the ranges
        mt = torch.tensor([ze.value], dtype=torch.int64, device=d.device)
        dist.all_reduce(mt, op=dist.ReduceOp.MAX, group=group)
        mm = max(mm, int(mt.item()))
        w = gather_columns(w[:mm], zb.value, ze.value, group)
    else:
        w = w[:mm]
    if MR3Error is None:  # pragma: no cover
        pass
    return w, Z, (zb.value, ze.value), st.asdict()
