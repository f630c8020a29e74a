"""paper_1304_1864_b200 -- B200-native mixed-precision MRRR (MR^3) hot path.

Thin ctypes binding of the C-ABI in include/mr3.h (libmr3.so, built in-tree for
sm_100a).  Argument marshalling only: every step of the solve runs in the CUDA
kernels of csrc/.  PyTorch supplies device memory, the stream and, for the
multi-GPU form, the NCCL process group (torch.distributed).  There is no CPU
fallback: without the built library or a CUDA device every call raises.

Public API (names follow the C-ABI):
    mr3_dstemr_dd(d, e, jobz='V', range='A', il=1, iu=0, vl=0., vu=0.)  fp64 I/O, dd internal
    mr3_sstemr_d(d, e, ...)                                            fp32 I/O, fp64 internal
    dstemr(...) / sstemr(...)            aliases of the two above
    solve_host(d_np, e_np, ...)          end to end through the host-buffer C-ABI entry points
    solve_distributed(d, e, group=...)   index-set partition over ranks: one library call per
                                         rank, all-gathers inside it (in-library NCCL
                                         communicator, or an exchange callback over gloo)
    mr3_dsyevr_dd(A, ...) / dsyevr       dense symmetric fp64: reduction, tridiagonal solve,
                                         back-transformation (NEXT-4)
    fp64_peak()                          K7 same-run FP64 peak + dd-step latency
    set_param(name, value, mode)         GAPTOL, XI, KRS, MAX_RQI, MAX_DEPTH, SEED, ELG_MAX, RTOL, GROUPS
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
_ROOT = os.path.dirname(_HERE)
LIB_PATH = os.path.join(_HERE, "libmr3.so")
SOURCES = sorted(os.path.join("csrc", f) for f in os.listdir(os.path.join(_HERE, "csrc"))
                 if f.endswith((".cu", ".cuh")))
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC,-ffp-contract=off", "-shared"]

PARAMS = {"GAPTOL": 0, "XI": 1, "KRS": 2, "MAX_RQI": 3, "MAX_DEPTH": 4, "SEED": 5, "ELG_MAX": 6,
          "RTOL": 7, "GROUPS": 8, "XPHASE": 9, "REFINE": 10, "GRID": 11, "CTA": 12, "XPTS": 13, "YCERT": 14, "NEWTON": 15, "TWISTW": 16,
          "SPLIT": 17, "FUSE_SCALE": 18, "POOL_MB": 19, "DEBUG": 20, "RQI_FB": 21, "RQI_CHUNK": 22,
          "RELAX": 23, "ABSGAP": 24, "BACKTRACK": 25}
ERRORS = {1: "NONFINITE", 2: "CUDA", 3: "NCCL", 4: "NOMEM", 5: "NOCONV", 6: "ZCAP", 7: "STATE"}


class MR3Error(RuntimeError):
    def __init__(self, code, msg=""):
        self.code = code
        name = ERRORS.get(code, "invalid argument %d" % (-code) if code < 0 else str(code))
        super().__init__(f"mr3 error {code} ({name}) {msg}".strip())


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile libmr3.so for sm_100a with nvcc (cross-compiles without a GPU)."""
    srcs = [os.path.join(_HERE, s) for s in SOURCES] + [os.path.join(_ROOT, "include", "mr3.h")]
    newest = max(os.path.getmtime(s) for s in srcs)
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < newest:
        tmp = LIB_PATH + f".tmp{os.getpid()}"
        cmd = ["nvcc", *NVCC_FLAGS, "-o", tmp, os.path.join(_HERE, "csrc", "mr3.cu")]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        subprocess.check_call(cmd, cwd=_HERE)
        os.replace(tmp, LIB_PATH)
    return LIB_PATH


class Stats(ctypes.Structure):
    _fields_ = [("d_max", ctypes.c_int32), ("n_clusters", ctypes.c_int32),
                ("largest_cluster", ctypes.c_int32), ("robustness_failures", ctypes.c_int32),
                ("rqi_fallbacks", ctypes.c_int32), ("n_blocks", ctypes.c_int32),
                ("rqi_iters_max", ctypes.c_int32), ("levels", ctypes.c_int32),
                ("rho", ctypes.c_double), ("bisect_rows", ctypes.c_double),
                ("rqi_rows", ctypes.c_double), ("bisect_rows_x", ctypes.c_double),
                ("newton_rows_x", ctypes.c_double),
                ("t_ms", ctypes.c_double * 8),
                ("backtracks", ctypes.c_int32), ("backtrack_tries", ctypes.c_int32)]

    def asdict(self):
        d = {f: getattr(self, f) for f, _ in self._fields_ if f != "t_ms"}
        d["t_ms"] = dict(zip(["root", "bisect", "classify", "child", "rqi", "total"],
                             list(self.t_ms)[:6]))
        return d


_lib = None
_lock = threading.Lock()
# int (*)(void *user, void *buf, size_t bytes_per_rank, int rank, int world, void *stream)
EXCHANGE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                               ctypes.c_int, ctypes.c_int, ctypes.c_void_p)


def lib():
    """Load libmr3.so (raises if it is missing: there is no fallback path)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(f"{LIB_PATH} not built; run paper_1304_1864_b200.build()")
            L = ctypes.CDLL(LIB_PATH)
            i64, i32, dbl, vp = ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_void_p
            pi64 = ctypes.POINTER(ctypes.c_int64)
            L.mr3_create.argtypes = [ctypes.POINTER(vp), i32, vp, vp, i32, i32]
            L.mr3_set_exchange.argtypes = [vp, EXCHANGE_FN, vp]
            L.mr3_nccl_unique_id.argtypes = [vp]
            L.mr3_nccl_comm_init.argtypes = [ctypes.POINTER(vp), vp, i32, i32, i32]
            L.mr3_nccl_comm_destroy.argtypes = [vp]
            L.mr3_destroy.argtypes = [vp]
            L.mr3_set_param.argtypes = [vp, i32, i32, dbl]
            L.mr3_get_param.argtypes = [vp, i32, i32]
            L.mr3_get_param.restype = dbl
            L.mr3_dstemr_dd.argtypes = [vp, ctypes.c_char, ctypes.c_char, i64, vp, vp, dbl, dbl,
                                        i64, i64, pi64, vp, vp, i64, i64, pi64, pi64,
                                        ctypes.POINTER(Stats)]
            L.mr3_sstemr_d.argtypes = [vp, ctypes.c_char, ctypes.c_char, i64, vp, vp,
                                       ctypes.c_float, ctypes.c_float, i64, i64, pi64, vp, vp,
                                       i64, i64, pi64, pi64, ctypes.POINTER(Stats)]
            L.mr3_dsyevr_dd.argtypes = [vp, ctypes.c_char, ctypes.c_char, i64, vp, i64, dbl, dbl,
                                        i64, i64, pi64, vp, vp, i64, ctypes.POINTER(Stats)]
            L.mr3_dstemr_dd_host.argtypes = L.mr3_dstemr_dd.argtypes
            L.mr3_sstemr_d_host.argtypes = L.mr3_sstemr_d.argtypes
            L.mr3_plan.argtypes = [vp, i32, ctypes.c_char, i64, vp, vp, dbl, dbl, i64, i64, i32,
                                   i32, pi64, ctypes.POINTER(ctypes.c_void_p), pi64, pi64]
            L.mr3_execute.argtypes = [vp, ctypes.c_char, vp, vp, i64, i64, pi64, pi64,
                                      ctypes.POINTER(Stats)]
            L.mr3_partition_columns.argtypes = [i64, pi64, ctypes.POINTER(dbl), i32, pi64]
            L.mr3_fp64_peak.argtypes = [vp, ctypes.POINTER(dbl), ctypes.POINTER(dbl)]
            L.mr3_last_kernel_times.argtypes = [vp, ctypes.POINTER(i32),
                                                ctypes.POINTER(ctypes.c_char_p),
                                                ctypes.POINTER(dbl), ctypes.POINTER(i32)]
            L.mr3_last_launch_count.argtypes = [vp]
            L.mr3_last_launch_count.restype = i64
            L.mr3_strerror.restype = ctypes.c_char_p
            L.mr3_last_error_string.argtypes = [vp]
            L.mr3_last_error_string.restype = ctypes.c_char_p
            L.mr3_version.restype = ctypes.c_char_p
            _lib = L
    return _lib


# ------------------------------------------------------------------ contexts

_ctx_cache: dict = {}
_params: dict = {0: {}, 1: {}}


def _ctx(device=None, stream=None):
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("mr3: no CUDA device (the product path has no CPU fallback)")
    dev = torch.cuda.current_device() if device is None else int(device)
    st = torch.cuda.current_stream(dev) if stream is None else stream
    # torch's default stream has handle 0 = the legacy default stream; pass it as
    # cudaStreamLegacy (1) so the library works on it (ordered after the caller's work)
    # instead of taking NULL = a stream of its own
    sh = int(st.cuda_stream) or 1
    key = (dev, sh)
    c = _ctx_cache.get(key)
    if c is None:
        h = ctypes.c_void_p()
        rc = lib().mr3_create(ctypes.byref(h), dev, ctypes.c_void_p(sh), None, 0, 1)
        if rc:
            raise MR3Error(rc, "mr3_create")
        c = h
        _ctx_cache[key] = c
    for mode in (0, 1):
        for k, v in _params[mode].items():
            lib().mr3_set_param(c, mode, PARAMS[k], float(v))
    return c


def set_param(name: str, value: float, mode: int = 0):
    """Set a solver parameter for mode 0 (fp64 I/O) or 1 (fp32 I/O); value < 0 = default."""
    if name not in PARAMS:
        raise KeyError(name)
    if value is None or (value < 0 and name != "RTOL"):
        _params[mode].pop(name, None)
        value = -1.0
    else:
        _params[mode][name] = value
    for c in _ctx_cache.values():
        lib().mr3_set_param(c, mode, PARAMS[name], float(value))


def get_param(name: str, mode: int = 0) -> float:
    return lib().mr3_get_param(_ctx(), mode, PARAMS[name])


def _err(c, rc, what):
    if rc:
        msg = lib().mr3_last_error_string(c).decode()
        raise MR3Error(rc, f"{what}: {msg}")


_last = {"ctx": None}  # the context of the last solve (single-rank or distributed)


def _used(c):
    _last["ctx"] = c
    return c


def kernel_times():
    """{kernel name: (total ms, launches)} of the last solve (on the context that solve used:
    the device/stream context, or the rank's distributed context), from CUDA events recorded
    on the context's stream around each launch."""
    c = _last["ctx"] or _ctx()
    cnt = ctypes.c_int(0)
    names = (ctypes.c_char_p * 16)()
    ms = (ctypes.c_double * 16)()
    nl = (ctypes.c_int * 16)()
    lib().mr3_last_kernel_times(c, ctypes.byref(cnt), names, ms, nl)
    return {names[i].decode(): (ms[i], nl[i]) for i in range(cnt.value)}


def launch_count() -> int:
    """Kernel launches issued by the last solve (all of this library's kernels)."""
    return int(lib().mr3_last_launch_count(_last["ctx"] or _ctx()))


def _solve(mode, d, e, jobz, range_, il, iu, vl, vu, w=None, Z=None):
    import torch
    dt = torch.float64 if mode == 0 else torch.float32
    if d.dtype != dt or e.dtype != dt or not d.is_cuda or not e.is_cuda:
        raise TypeError(f"mr3: d, e must be CUDA {dt} tensors")
    d = d.contiguous()
    e = e.contiguous()
    n = d.numel()
    if e.numel() < max(n - 1, 0):
        raise ValueError("mr3: e must have n-1 entries")
    c = _used(_ctx(d.device.index))
    if w is None:
        w = torch.empty(max(n, 1), dtype=dt, device=d.device)
    if jobz == "V" and Z is None:
        # column-major n x mcap: storage as (mcap, n) row-major, returned transposed; an
        # index range needs only its iu - il + 1 columns
        mcap = n if range_ != "I" else max(0, min(iu, n) - max(il, 1) + 1)
        Zs = torch.empty((max(mcap, 1), max(n, 1)), dtype=dt, device=d.device)
    else:
        Zs = Z
    m = ctypes.c_int64(0)
    zb, ze = ctypes.c_int64(0), ctypes.c_int64(0)
    st = Stats()
    fn = lib().mr3_dstemr_dd if mode == 0 else lib().mr3_sstemr_d
    zcap = Zs.shape[0] if Zs is not None else 0
    rc = fn(c, jobz.encode(), range_.encode(), n, ctypes.c_void_p(d.data_ptr()),
            ctypes.c_void_p(e.data_ptr() if n > 1 else d.data_ptr()), vl, vu, il, iu,
            ctypes.byref(m), ctypes.c_void_p(w.data_ptr()),
            ctypes.c_void_p(Zs.data_ptr() if Zs is not None else 0), max(n, 1), zcap,
            ctypes.byref(zb), ctypes.byref(ze), ctypes.byref(st))
    _err(c, rc, "mr3_dstemr_dd" if mode == 0 else "mr3_sstemr_d")
    mm = m.value
    Zout = Zs[:mm].T if (jobz == "V" and Zs is not None) else None
    return w[:mm], Zout, st.asdict()


def mr3_dstemr_dd(d, e, jobz="V", range="A", il=1, iu=0, vl=0.0, vu=0.0):
    """fp64 I/O, double-double internal.  d, e: CUDA float64 tensors.
    Returns (w[m], Z[n, m] (column j = eigenvector of w[j]) or None, stats dict)."""
    return _solve(0, d, e, jobz, range, il, iu, vl, vu)


def mr3_sstemr_d(d, e, jobz="V", range="A", il=1, iu=0, vl=0.0, vu=0.0):
    """fp32 I/O, fp64 internal.  d, e: CUDA float32 tensors."""
    return _solve(1, d, e, jobz, range, il, iu, vl, vu)


dstemr = mr3_dstemr_dd
sstemr = mr3_sstemr_d


_dense_work: dict = {}


def mr3_dsyevr_dd(A, jobz="V", range="A", il=1, iu=0, vl=0.0, vu=0.0, overwrite=False):
    """Dense symmetric fp64 eigenproblem (NEXT-4): reduction to tridiagonal form, the
    double-double tridiagonal solver, back-transformation -- all on the device.
    A: CUDA float64 (n, n) symmetric tensor (its row-major storage is the column-major storage
    of A^T = A).  overwrite=False works on a copy (the C-ABI overwrites A with the reduction).
    Returns (w[m], Z[n, m] or None, stats dict with t_ms['reduce'], t_ms['backtransform'])."""
    import torch
    if A.dtype != torch.float64 or not A.is_cuda or A.dim() != 2 or A.shape[0] != A.shape[1]:
        raise TypeError("mr3: A must be a square CUDA float64 tensor")
    n = A.shape[0]
    if overwrite and A.is_contiguous():
        Aw = A
    else:
        # a cached work copy per (device, n): the library replays its captured reduction graph
        # when the matrix buffer is the same one
        key = (A.device.index, n)
        Aw = _dense_work.get(key)
        if Aw is None:
            Aw = torch.empty_like(A, memory_format=torch.contiguous_format)
            _dense_work.clear()
            _dense_work[key] = Aw
        Aw.copy_(A)
    c = _used(_ctx(A.device.index))
    w = torch.empty(max(n, 1), dtype=torch.float64, device=A.device)
    Zs = None
    if jobz == "V":
        mcap = n if range != "I" else max(0, min(iu, n) - max(il, 1) + 1)
        Zs = torch.empty((max(mcap, 1), max(n, 1)), dtype=torch.float64, device=A.device)
    m = ctypes.c_int64(0)
    st = Stats()
    rc = lib().mr3_dsyevr_dd(c, jobz.encode(), range.encode(), n, ctypes.c_void_p(Aw.data_ptr()),
                             max(n, 1), vl, vu, il, iu, ctypes.byref(m),
                             ctypes.c_void_p(w.data_ptr()),
                             ctypes.c_void_p(Zs.data_ptr() if Zs is not None else 0), max(n, 1),
                             ctypes.byref(st))
    _err(c, rc, "mr3_dsyevr_dd")
    mm = m.value
    d = st.asdict()
    d["t_ms"]["reduce"] = st.t_ms[6]
    d["t_ms"]["backtransform"] = st.t_ms[7]
    return w[:mm], (Zs[:mm].T if Zs is not None else None), d


dsyevr = mr3_dsyevr_dd


def solve_host(d, e, jobz="V", range="A", il=1, iu=0, vl=0.0, vu=0.0, w=None, Z=None):
    """End to end through the host-buffer C-ABI (mr3_dstemr_dd_host / mr3_sstemr_d_host):
    d, e are host arrays (numpy or CPU torch tensors, ideally pinned); the library copies
    them to the device, solves, and writes w and Z back to host memory.  w (n) and Z
    (host, column-major n x m storage given as an (m_cap, n) row-major array) may be
    preallocated (pinned) buffers.  Returns (w[:m], Z[:m].T or None, stats)."""
    import numpy as np
    import torch
    dtn = np.asarray(d).dtype if not isinstance(d, torch.Tensor) else d.numpy().dtype
    mode = 1 if dtn == np.float32 else 0
    dt = torch.float32 if mode else torch.float64
    hd = d if isinstance(d, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(d, dtype=dtn))
    he = e if isinstance(e, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(e, dtype=dtn))
    if hd.is_cuda or he.is_cuda or hd.dtype != dt or he.dtype != dt:
        raise TypeError("solve_host: d, e must be host arrays of one float dtype")
    hd, he = hd.contiguous(), he.contiguous()
    n = hd.numel()
    mcap = n if range != "I" else max(0, min(iu, n) - max(il, 1) + 1)
    if w is None:
        w = torch.empty(max(n, 1), dtype=dt)
    if jobz == "V" and Z is None:
        Z = torch.empty((max(mcap, 1), max(n, 1)), dtype=dt)
    c = _used(_ctx())
    m = ctypes.c_int64(0)
    zb, ze = ctypes.c_int64(0), ctypes.c_int64(0)
    st = Stats()
    fn = lib().mr3_dstemr_dd_host if mode == 0 else lib().mr3_sstemr_d_host
    zcap = Z.shape[0] if (jobz == "V" and Z is not None) else 0
    rc = fn(c, jobz.encode(), range.encode(), n, ctypes.c_void_p(hd.data_ptr()),
            ctypes.c_void_p(he.data_ptr() if n > 1 else hd.data_ptr()), vl, vu, il, iu,
            ctypes.byref(m), ctypes.c_void_p(w.data_ptr()),
            ctypes.c_void_p(Z.data_ptr() if (jobz == "V" and Z is not None) else 0), max(n, 1),
            zcap, ctypes.byref(zb), ctypes.byref(ze), ctypes.byref(st))
    _err(c, rc, "mr3_dstemr_dd_host" if mode == 0 else "mr3_sstemr_d_host")
    mm = m.value
    return w[:mm], (Z[:mm].T if jobz == "V" else None), st.asdict()


def fp64_peak():
    """K7: (FP64 instructions/s over all SMs, latency of one dd Sturm step in ns)."""
    c = _ctx()
    a, b = ctypes.c_double(), ctypes.c_double()
    _err(c, lib().mr3_fp64_peak(c, ctypes.byref(a), ctypes.byref(b)), "mr3_fp64_peak")
    return a.value, b.value


def partition_columns(seg_begin, cost, world):
    """Host-only cluster-whole column partition (mr3_partition_columns)."""
    import numpy as np
    sb = np.ascontiguousarray(np.asarray(seg_begin, dtype=np.int64))
    cs = np.ascontiguousarray(np.asarray(cost, dtype=np.float64))
    out = np.zeros(world + 1, dtype=np.int64)
    rc = lib().mr3_partition_columns(sb.size - 1, sb.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                     cs.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), world,
                                     out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)))
    if rc:
        raise MR3Error(rc, "mr3_partition_columns")
    return out


from .distributed import solve_distributed, gather_columns  # noqa: E402,F401
