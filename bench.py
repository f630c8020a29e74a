#!/usr/bin/env python3
"""Benchmark of the mixed-precision MRRR hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--impl reference]

metric : eigenpairs/s, fp64 I/O dd-internal, n = 50000 (config 5: Legendre-type,
         all eigenpairs, Z = 20 GB); one step = one full solve (root, bisection,
         classification, RQI + Z store) through the C-ABI, inputs resident in HBM.
e2e    : the same metric from pinned host d, e to host w and Z (H2D + solve + D2H).
N > 1  : launched by torchrun, one rank per GPU; the index set is partitioned
         (mr3_plan -> NCCL all-gather of brackets -> mr3_execute -> all-gather
         of w); total work is fixed -> "scaling": "strong".
--impl reference : the binary128 oracle (oracle/) timed on the host cores on a
         bounded sample of the same workload (the "reference arm" of this tier).
"""
import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

# Algorithmic FP64 instructions (DADD/DMUL/DFMA) per unit of work, from the operation
# counts of the recurrences in the arithmetic of dd.cuh (pair add 11,
# pair mul 7, pair fma 15, pair div 14 + one MUFU.RCP64H):
#   Sturm row, binary_y projective (2 pair fma + 1 pair mul)          37
#   Sturm row, binary_x projective (2 DFMA + 1 DMUL + rescale/8)      3.25
#   Sturm row, fp64-internal mode (projective, binary64)              3.25
#   Newton/Laguerre pass row, binary_x (value + two x-derivatives)    11
#   RQI row (rqi_rows: 2 fixed-twist passes of n rows each; projective F or B row: pair fma
#   15 + pair dot product 19 + prefix norm 6 (+ rescale/8) = 40.5 on the non-storing pass; the
#   storing pass replaces the prefix norm by the product-form z component and its compensated
#   square, 6 (R9e); SASS of k_rqi_fb: 40.5 / 40.5)
#   dd 40.5, fp64-internal 9.25 (9.25 / 9.25)
FP64_INST_PER_BISECT_ROW = {"dd": 37.0, "f64": 3.25, "x": 3.25, "newton": 11.0}
FP64_INST_PER_RQI_ROW = {"dd": 40.5, "f64": 9.25}
DERIVED_FP64_PEAK = 148 * 64 * 1.965e9  # SMs x FP64 lanes x max SM clock (inst/s)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--impl", default="mr3", choices=["mr3", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=0)
    ap.add_argument("--other-configs", default="1,2,3,4",
                    help="BASELINE configs also timed (with roofline and the full oracle run "
                         "as CPU baseline), reported under 'other_configs'; '' = none")
    ap.add_argument("--emulate-world", default="2,4,8",
                    help="world sizes whose ranks (mr3_plan + mr3_execute) are emulated one "
                         "after another on this GPU; per-rank device times under "
                         "'emulated_world' (an emulation, not a multi-GPU measurement)")
    ap.add_argument("--no-zstore", action="store_true")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend for --gpus > 1 (gloo: logic tests of the multi-rank "
                         "path with several ranks sharing one GPU and the host-staged exchange; "
                         "never a measurement)")
    ap.add_argument("--dense", default="4096",
                    help="NEXT-4 dense pipeline line (mr3_dsyevr_dd on A = Q T Q^T of this size, "
                         "T the config-2 recipe) under 'dense'; '' = none")
    return ap.parse_args()


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class Clocks:
    """SM clocks and throttle reasons sampled DURING the timed region (in-process NVML,
    every 200 ms; nvidia-smi in a subprocess would fork this large process)."""

    def __init__(self, dev):
        self.dev = dev
        self.samples = []
        self.stop = threading.Event()
        self.t = threading.Thread(target=self.run, daemon=True)
        self.nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(dev)
        except Exception:
            self.nvml = None

    def run(self):
        nv = self.nvml
        if nv is None:
            return
        while not self.stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                mx = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h) \
                    if hasattr(nv, "nvmlDeviceGetCurrentClocksEventReasons") \
                    else nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                pw = nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0
                self.samples.append((sm, mx, rs, pw))
            except Exception:
                pass
            self.stop.wait(0.2)

    def __enter__(self):
        self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.t.join(timeout=10)
        if self.nvml is not None and not self.samples:
            self.sample_once()

    def sample_once(self):
        self.stop.clear()
        self.stop.set()
        try:
            nv = self.nvml
            self.samples.append((nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM),
                                 nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM),
                                 nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h),
                                 nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0))
        except Exception:
            pass

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        bits = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
                "sw_power_cap": 0x4}
        reasons = set()
        for _, _, rs, _ in self.samples:
            for nm, bit in bits.items():
                if rs & bit:
                    reasons.add(nm)
        return {"sm_mhz": float(np.median([s[0] for s in self.samples])),
                "sm_max_mhz": float(max(s[1] for s in self.samples)),
                "reasons": sorted(reasons), "samples": len(self.samples),
                "power_w_max": float(max(s[3] for s in self.samples))}


def cpu_baseline_run(p, n_idx, seed=0, idx=None):
    """The oracle (binary128 bisection + inverse iteration) on a bounded sample of
    eigenpairs of the same matrix (or the given 1-based indices), on all host cores."""
    import oracle
    rng = np.random.default_rng(seed)
    if idx is None:
        idx = np.unique(np.concatenate([[1, p.n], rng.choice(np.arange(2, p.n), n_idx - 2,
                                                              replace=False)]))
    d, e = p.d.astype(np.float64), p.e.astype(np.float64)
    t0 = time.perf_counter()
    lh, ll = oracle.eigvals(d, e, idx)
    oracle.eigvecs(d, e, lh, ll, group_tol_rel=1e-9)
    dt = time.perf_counter() - t0
    return idx.size, dt, oracle.num_threads()


def run_reference(args, p, rank, world):
    if rank != 0:
        return
    import oracle
    oracle.build()
    cores = oracle.num_threads()
    per_step = args.cpu_sample or max(8 * cores, 16)
    for _ in range(args.warmup):
        cpu_baseline_run(p, min(per_step, 4))
    tot_n, tot_t = 0, 0.0
    for s in range(args.steps):
        k, dt, _ = cpu_baseline_run(p, per_step, seed=s + 1)
        tot_n += k
        tot_t += dt
    v = tot_n / tot_t
    line = {"impl": "reference", "metric": metric_name(p), "value": v, "unit": "eigenpairs/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * tot_t / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "binary128 (oracle)",
            "data": "synthetic", "config": {"workload": p.name, "n": p.n, "sample_per_step": per_step},
            "cpu_baseline": {"value": v, "unit": "eigenpairs/s", "cores": cores, "kind": "oracle",
                             "cpu": cpu_model(),
                             "sample": f"{per_step} eigenpairs of the n={p.n} workload per step "
                                       "(bisection on T + inverse iteration, binary128)"},
            "e2e": {"value": v, "unit": "eigenpairs/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def make_roof(ktot, stats, steps, mode, traffic_tab, peak_ips):
    """roofline(kname): algorithmic FP64 instructions per launch of kname (DESIGN.md section 5
    counts x the units the solve processed) / its CUDA-event time per launch."""

    def roof(kname):
        ms, nl = ktot.get(kname, (0.0, 0))
        if kname == "k_bisect":
            rows = stats["bisect_rows"] if stats else 0.0
            rows_x = stats.get("bisect_rows_x", 0.0) if stats else 0.0
            rows_n = stats.get("newton_rows_x", 0.0) if stats else 0.0
            inst = (rows * FP64_INST_PER_BISECT_ROW[mode] +
                    (rows_x - rows_n) * FP64_INST_PER_BISECT_ROW["x"] +
                    rows_n * FP64_INST_PER_BISECT_ROW["newton"])
            per = {"binary_y_row": FP64_INST_PER_BISECT_ROW[mode],
                   "binary_x_row": FP64_INST_PER_BISECT_ROW["x"],
                   "binary_x_newton_row": FP64_INST_PER_BISECT_ROW["newton"]}
            units = {"binary_y_rows": rows, "binary_x_rows": rows_x - rows_n,
                     "binary_x_newton_rows": rows_n}
        else:
            rows = stats["rqi_rows"] if stats else 0.0
            inst = rows * FP64_INST_PER_RQI_ROW[mode]
            per = {"rqi_row": FP64_INST_PER_RQI_ROW[mode]}
            units = {"rqi_rows": rows}
        t_launch = ms / max(nl, 1) * 1e-3  # average launch duration
        inst_launch = inst / max(nl / steps, 1)
        ach = inst_launch / t_launch if t_launch else 0.0
        return {"bound": "alu", "kernel": kname, "achieved": ach / 1e12,
                "peak": DERIVED_FP64_PEAK / 1e12, "unit": "T FP64-inst/s",
                "frac": ach / DERIVED_FP64_PEAK, "traffic": traffic_tab.get(kname),
                "peak_source": "derived: 148 SMs x 64 FP64 lanes x 1.965 GHz (MEASURED_PEAKS.json "
                               "has no FP64 entry); measured_peak_same_run = K7 DFMA microbenchmark",
                "measured_peak_same_run": peak_ips / 1e12,
                "frac_of_measured": ach / peak_ips if peak_ips else None,
                "inst_per_unit": per, "units_per_step": units,
                "launches_per_step": nl / steps, "ms_per_launch": t_launch * 1e3}
    return roof


def hbm_peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]), \
            "MEASURED_PEAKS.json hbm_gbs (copy, burst)"
    except Exception:
        return 6546.2, "fallback: B200_PROFILING.md measured copy bandwidth"


def timed_solves(mr3, fn, d, e, p, il, iu, steps, warmup, flush, stream):
    """Device-timed solves of one config (inputs resident, L2 flushed between steps)."""
    import torch
    for _ in range(warmup):
        out = fn(d, e, "V", p.range, il, iu)
        del out
    torch.cuda.synchronize()
    times, ktot, launches, stats = [], {}, 0, None
    for s in range(steps):
        flush.fill_(s)
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        w, Z, stats = fn(d, e, "V", p.range, il, iu)
        b.record(stream)
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b))
        for k, (ms, nl) in mr3.kernel_times().items():
            t0, n0 = ktot.get(k, (0.0, 0))
            ktot[k] = (t0 + ms, n0 + nl)
        launches += mr3.launch_count()
        del w, Z
    return times, ktot, launches, stats


def other_config_line(mr3, cfg, args, flush, stream, peak_ips, cpu):
    """Timing, roofline and CPU baseline of another BASELINE config (a secondary line)."""
    import torch
    p = synth.config(cfg)
    il, iu = p.index_range()
    m_req = iu - il + 1
    fn = mr3.mr3_sstemr_d if p.io == "f32" else mr3.mr3_dstemr_dd
    d = torch.from_numpy(p.d).cuda()
    e = torch.from_numpy(p.e).cuda()
    steps = max(3, min(args.steps, 5))
    times, ktot, launches, stats = timed_solves(mr3, fn, d, e, p, il, iu, steps, 2, flush, stream)
    t = float(np.mean(times))
    mode = "f64" if p.io == "f32" else "dd"
    roof = make_roof(ktot, stats, steps, mode, {}, peak_ips)
    cand = [k for k in ("k_bisect", "k_rqi") if k in ktot]
    dom = max(cand, key=lambda k: ktot[k][0]) if cand else "k_rqi"
    line = {"config": cfg, "metric": metric_name(p), "value": m_req / (t * 1e-3),
            "unit": "eigenpairs/s", "ms_per_step": t, "steps": steps, "n": p.n, "m": m_req,
            "io": p.io, "roofline": roof(dom),
            "kernels": {k: {"ms_per_step": v[0] / steps, "launches_per_step": v[1] / steps}
                        for k, v in ktot.items()},
            "gpu_launches": launches,
            "stats": {k: v for k, v in (stats or {}).items()}}
    if cpu:
        # the oracle in full (north_star: the full run for n <= 20000)
        idx = np.arange(il, iu + 1)
        cnt, dt_cpu, cores = cpu_baseline_run(p, 0, idx=idx)
        line["cpu_baseline"] = {"value": cnt / dt_cpu, "unit": "eigenpairs/s", "cores": cores,
                                "cpu": cpu_model(), "kind": "oracle",
                                "sample": f"full run: all {cnt} requested eigenpairs, binary128 "
                                          f"bisection on T + inverse iteration, {dt_cpu:.1f} s"}
    del d, e
    torch.cuda.empty_cache()
    return line


def dense_line(mr3, n, steps, warmup, flush, stream, cpu):
    """NEXT-4: the dense symmetric pipeline (reduction, tridiagonal solve, back-transformation)
    through mr3_dsyevr_dd, A = Q T Q^T resident in HBM (copied into the library's work buffer
    inside the timed region: the call overwrites A).  Roofline of the reduction (both of its
    kernels, the dominant phase): algorithmic bytes = one read of the trailing block per
    reflector and one write from the second on, sum_j 8 (n - j - 1)^2 (1 + [j >= 1])."""
    import torch
    p = synth.dense_config(n, 0)
    A = torch.from_numpy(np.ascontiguousarray(p.A)).cuda()
    times, ktot, launches = [], {}, 0
    st = None
    for it in range(warmup + steps):
        flush.fill_(it)
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        w, Z, st = mr3.mr3_dsyevr_dd(A)
        b.record(stream)
        torch.cuda.synchronize()
        if it >= warmup:
            times.append(a.elapsed_time(b))
            for k, (ms, nl) in mr3.kernel_times().items():
                t0, n0 = ktot.get(k, (0.0, 0))
                ktot[k] = (t0 + ms, n0 + nl)
            launches += mr3.launch_count()
        del w, Z
    t = float(np.mean(times))
    j = np.arange(n - 1, dtype=np.float64)
    red_bytes = float(np.sum(8.0 * (n - j - 1) ** 2 * np.where(j >= 1, 2.0, 1.0)))
    red_ms = ktot.get("k_sytrd", (float("nan"), 0))[0] / steps
    peak, peak_src = hbm_peak()
    ach = red_bytes / (red_ms * 1e-3) / 1e9
    line = {"metric": f"eigenpairs/s, dense symmetric fp64 I/O (A = Q T Q^T), n={n}",
            "value": n / (t * 1e-3), "unit": "eigenpairs/s", "ms_per_step": t, "steps": steps,
            "n": n, "m": n, "io": "f64",
            "config": {"workload": p.name, "n": n, "range": "A",
                       "pipeline": "Householder reduction (k_sytd_col + k_sytd_fused, one CUDA "
                                   "graph) -> mr3_dstemr_dd -> blocked back-transformation "
                                   "(k_build_v, k_larft, cuBLAS DGEMM)"},
            "roofline": {"bound": "hbm", "kernel": "k_sytrd (k_sytd_fused + k_sytd_col)",
                         "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                         "traffic": None, "bytes_per_launch": red_bytes,
                         "ms_per_launch": red_ms,
                         "peak_source": peak_src,
                         "note": "the trailing block is L2-resident once below ~126 MB "
                                 "(n - j < ~3970): later sweeps run from L2"},
            "kernels": {k: {"ms_per_step": v[0] / steps, "launches_per_step": v[1] / steps}
                        for k, v in ktot.items()},
            "gpu_launches": launches,
            "stats": {k: v for k, v in (st or {}).items()}}
    if cpu:
        from oracle import dense as odense
        import oracle
        ns = 512
        q = synth.dense_config(ns, 0)
        t0 = time.time()
        odense.eig_dense(q.A)
        dt_cpu = time.time() - t0
        line["cpu_baseline"] = {"value": ns / dt_cpu, "unit": "eigenpairs/s",
                                "cores": oracle.num_threads(), "cpu": cpu_model(),
                                "kind": "oracle",
                                "sample": f"full run at n={ns} (same recipe): numpy Householder "
                                          f"reduction + binary128 tridiagonal oracle + Q y, "
                                          f"{dt_cpu:.1f} s (the n^3 reduction makes n={n} "
                                          f"~{(n / ns) ** 3:.0f}x longer)"}
    del A
    torch.cuda.empty_cache()
    return line


def emulate_world(mr3, p, world, stream):
    """Ranks of the two-phase form run one after another on this GPU: per rank, device time of
    mr3_plan (root + its slice's bisection) and of mr3_execute (classification, its columns'
    child representations and eigenvectors); the bracket all-gather is a device copy."""
    import ctypes

    import torch
    L = mr3.lib()
    d = torch.from_numpy(p.d).cuda()
    e = torch.from_numpy(p.e).cuda()
    n = p.n
    ctxs, bufs, caps, tplan = [], [], [], []
    for r in range(world):
        h = ctypes.c_void_p()
        assert L.mr3_create(ctypes.byref(h), torch.cuda.current_device(),
                            ctypes.c_void_p(int(stream.cuda_stream) or 1), None, 0, 1) == 0
        ctxs.append(h)
        m, brk = ctypes.c_int64(), ctypes.c_void_p()
        cap, cnt = ctypes.c_int64(), ctypes.c_int64()
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        rc = L.mr3_plan(h, 0 if p.io == "f64" else 1, p.range.encode(), n,
                        ctypes.c_void_p(d.data_ptr()), ctypes.c_void_p(e.data_ptr()), 0.0, 0.0,
                        1, n, r, world, ctypes.byref(m), ctypes.byref(brk), ctypes.byref(cap),
                        ctypes.byref(cnt))
        b.record(stream)
        torch.cuda.synchronize()
        assert rc == 0, rc
        tplan.append(a.elapsed_time(b))
        bufs.append(mr3.distributed.wrap_device(brk.value, world * cap.value * 6, d.device))
        caps.append(cap.value)
    rec = 6 * caps[0]
    full = torch.cat([bufs[r][r * rec:(r + 1) * rec] for r in range(world)])
    for r in range(world):
        bufs[r][:world * rec].copy_(full)
    torch.cuda.synchronize()
    dt = torch.float64 if p.io == "f64" else torch.float32
    texec, cols = [], []
    for r in range(world):
        w = torch.zeros(n, dtype=dt, device="cuda")
        zb, ze = ctypes.c_int64(), ctypes.c_int64()
        rc = L.mr3_execute(ctxs[r], b"V", ctypes.c_void_p(w.data_ptr()), None, n, 0,
                           ctypes.byref(zb), ctypes.byref(ze), None)
        Zs = torch.empty((max(ze.value - zb.value, 1), n), dtype=dt, device="cuda")
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        rc = L.mr3_execute(ctxs[r], b"V", ctypes.c_void_p(w.data_ptr()),
                           ctypes.c_void_p(Zs.data_ptr()), n, Zs.shape[0], ctypes.byref(zb),
                           ctypes.byref(ze), None)
        b.record(stream)
        torch.cuda.synchronize()
        assert rc == 0, rc
        texec.append(a.elapsed_time(b))
        cols.append(ze.value - zb.value)
        del Zs, w
    for h in ctxs:
        L.mr3_destroy(h)
    per_rank = [a + b for a, b in zip(tplan, texec)]
    torch.cuda.empty_cache()
    return {"world": world, "per_rank_ms": [round(x, 3) for x in per_rank],
            "plan_ms": [round(x, 3) for x in tplan], "execute_ms": [round(x, 3) for x in texec],
            "columns": cols, "max_rank_ms": max(per_rank),
            "note": "ranks emulated sequentially on one GPU (each alone on the device); the "
                    "all-gathers are device copies; not a multi-GPU measurement"}


def metric_name(p):
    io = "fp32 I/O fp64-internal" if p.io == "f32" else "fp64 I/O dd-internal"
    return f"eigenpairs/s, {io}, {p.name} n={p.n}"


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    p = synth.config(args.config)

    if args.impl == "reference":
        if world > 1:
            import torch.distributed as dist
            dist.init_process_group("gloo")
        run_reference(args, p, rank, world)
        return

    import torch
    import torch.distributed as dist

    import paper_1304_1864_b200 as mr3

    local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    if world > 1:
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    rdev = "cuda" if args.backend == "nccl" else "cpu"  # where the timing reductions live

    def allreduce(v, op):
        t = torch.tensor([v], dtype=torch.float64, device=rdev)
        dist.all_reduce(t, op=op)
        return float(t.item())

    mr3.lib()
    dt = torch.float32 if p.io == "f32" else torch.float64
    d = torch.from_numpy(p.d).cuda()
    e = torch.from_numpy(p.e).cuda()
    n = p.n
    il, iu = p.index_range()
    m_req = iu - il + 1
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")  # > L2

    exch = {"mode": "auto"}  # in-library NCCL communicator (mr3_nccl_comm_init + ncclAllGather)

    def solve():
        if world > 1:
            return mr3.solve_distributed(d, e, "V", p.range, il, iu, exchange=exch["mode"])
        fn = mr3.mr3_sstemr_d if p.io == "f32" else mr3.mr3_dstemr_dd
        w, Z, st = fn(d, e, "V", p.range, il, iu)
        return w, Z, (0, w.numel()), st

    # K7: same-run FP64 peak
    peak_ips, dd_step_ns = mr3.fp64_peak()

    if world > 1:
        # one untimed solve decides the exchange for every rank together: if the in-library
        # communicator cannot be set up on this box (no usable libnccl.so.2 for the library),
        # all ranks fall back to the two-phase form whose all-gathers torch.distributed issues
        # (still NCCL); the line says which one ran
        bad = 0
        try:
            out = solve()
            del out
        except Exception as ex:  # noqa: BLE001
            bad = 1
            print(f"[rank {rank}] in-library NCCL exchange failed: {ex}", file=sys.stderr)
        if allreduce(float(bad), dist.ReduceOp.MAX) > 0:
            exch["mode"] = "torch"

    for _ in range(args.warmup):
        out = solve()
        del out
    torch.cuda.synchronize()

    stream = torch.cuda.current_stream()
    times = []
    ktot = {}
    launches = 0
    stats = None
    with Clocks(local) as clk:
        for s in range(args.steps):
            flush.fill_(s)  # L2 flush between timed steps (outside the events)
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            w, Z, rng, stats = solve()
            b.record(stream)
            torch.cuda.synchronize()
            times.append(a.elapsed_time(b))
            for k, (ms, nl) in mr3.kernel_times().items():
                t0, n0 = ktot.get(k, (0.0, 0))
                ktot[k] = (t0 + ms, n0 + nl)
            launches += mr3.launch_count()
            del w, Z
    t_step = float(np.mean(times))
    t_max = t_step
    if world > 1:
        t_max = allreduce(t_step, dist.ReduceOp.MAX)
    value = m_req / (t_max * 1e-3)  # all ranks together produce the m eigenpairs of one solve

    # roofline of the dominant kernel (the larger of k_bisect and k_rqi): algorithmic FP64
    # instructions per launch / its CUDA-event time inside the timed region
    mode = "f64" if p.io == "f32" else "dd"
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    traffic_tab = {}
    if os.path.exists(tp):
        try:
            traffic_tab = json.load(open(tp)).get(f"config{args.config}", {})
        except Exception:
            traffic_tab = {}

    roof = make_roof(ktot, stats, args.steps, mode, traffic_tab, peak_ips)
    cand = [k for k in ("k_bisect", "k_rqi") if k in ktot]
    dom = max(cand, key=lambda k: ktot[k][0]) if cand else "k_bisect"
    roofs = {k: roof(k) for k in cand}

    result = None
    if rank == 0:
        kt = {k: {"ms_per_step": v[0] / args.steps, "launches_per_step": v[1] / args.steps}
              for k, v in ktot.items()}
        result = {
            "metric": metric_name(p), "value": value, "unit": "eigenpairs/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_max,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64" if p.io == "f32" else "dd (f64 pairs)", "data": "synthetic",
            "config": {"workload": p.name, "n": n, "m": m_req, "range": p.range,
                       "io": p.io, "parallelism": f"index-set partition x{world}",
                       "exchange": ("none" if world == 1 else
                                    "host-staged callback (gloo logic test)"
                                    if args.backend != "nccl" else
                                    "in-library ncclAllGather" if exch["mode"] == "auto" else
                                    "torch.distributed all_gather (two-phase)"),
                       "l2": "512 MB buffer written between timed steps; Z output > L2"},
            "roofline": roofs.get(dom, {}),
            "roofline_other": {k: v for k, v in roofs.items() if k != dom},
            "kernels": kt,
            "dd_step_latency_ns": dd_step_ns,
            "step_ms": [round(t, 3) for t in times],
            "gpu_launches": launches,
            "stats": {k: v for k, v in (stats or {}).items()},
            "clocks": clk.summary(),
        }

    # e2e: the host-buffer C-ABI call (mr3_dstemr_dd_host / mr3_sstemr_d_host): pinned host
    # d, e -> device, solve, device -> pinned host w and Z, all inside the timed region
    if not args.no_e2e and world == 1:
        es = torch.float32 if p.io == "f32" else torch.float64
        hd = torch.from_numpy(p.d).pin_memory()
        he = torch.from_numpy(p.e).pin_memory()
        hw = torch.empty(n, dtype=es).pin_memory()
        hZ = torch.empty((m_req, n), dtype=es).pin_memory()
        et = []
        mr3.solve_host(hd, he, "V", p.range, il, iu, w=hw, Z=hZ)  # warm-up (scratch allocation)
        for s in range(max(1, min(args.steps, 2))):
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            wv, Zv, st = mr3.solve_host(hd, he, "V", p.range, il, iu, w=hw, Z=hZ)
            b.record(stream)
            torch.cuda.synchronize()
            et.append(a.elapsed_time(b))
            assert wv.shape[0] == m_req
        esz = 4 if p.io == "f32" else 8
        if rank == 0:
            result["e2e"] = {"value": m_req / (np.mean(et) * 1e-3), "unit": "eigenpairs/s",
                             "h2d_bytes_per_step": (2 * n - 1) * esz,
                             "d2h_bytes_per_step": (m_req + m_req * n) * esz,
                             "ms_per_step": float(np.mean(et)),
                             "api": "mr3_sstemr_d_host" if p.io == "f32" else "mr3_dstemr_dd_host"}
        del hZ

    if not args.no_e2e and world > 1:
        # e2e at N ranks: every rank copies d, e from pinned host memory, runs the multi-rank
        # solve and reads w and ITS columns of Z back into pinned host memory inside the timed
        # region (barrier + synchronize on both sides, max over ranks)
        hd = torch.from_numpy(p.d).pin_memory()
        he = torch.from_numpy(p.e).pin_memory()
        w0, Z0, rng0, _ = solve()
        ncol = Z0.shape[1]
        del w0, Z0
        hw = torch.empty(m_req, dtype=dt).pin_memory()
        hZ = torch.empty((max(ncol, 1), n), dtype=dt).pin_memory()
        et = []
        for s in range(max(1, min(args.steps, 2))):
            dist.barrier()
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            dd_ = hd.cuda(non_blocking=True)
            ee_ = he.cuda(non_blocking=True)
            wv, Zv, rg, st = mr3.solve_distributed(dd_, ee_, "V", p.range, il, iu,
                                                   exchange=exch["mode"])
            hw.copy_(wv, non_blocking=True)
            hZ[:Zv.shape[1]].copy_(Zv.T, non_blocking=True)
            b.record(stream)
            torch.cuda.synchronize()
            et.append(a.elapsed_time(b))
            del wv, Zv, dd_, ee_
        esz = 4 if p.io == "f32" else 8
        te = allreduce(float(np.mean(et)), dist.ReduceOp.MAX)
        nb = allreduce(float((m_req + ncol * n) * esz), dist.ReduceOp.SUM)
        if rank == 0:
            result["e2e"] = {"value": m_req / (te * 1e-3), "unit": "eigenpairs/s",
                             "h2d_bytes_per_step": (2 * n - 1) * esz * world,
                             "d2h_bytes_per_step": nb,
                             "ms_per_step": te,
                             "api": "solve_distributed (one C-ABI call per rank; pinned host "
                                    "d, e in, w and the rank's Z columns out)"}
        del hZ

    if rank == 0 and not args.no_cpu:
        import oracle
        oracle.build()
        k = args.cpu_sample or max(32 * oracle.num_threads(), 64)
        cnt, dt_cpu, cores = cpu_baseline_run(p, k)
        result["cpu_baseline"] = {"value": cnt / dt_cpu, "unit": "eigenpairs/s", "cores": cores,
                                  "kind": "oracle", "cpu": cpu_model(),
                                  "sample": f"{cnt} eigenpairs (incl. both spectrum ends) of the "
                                            f"n={n} workload: binary128 bisection on T + "
                                            f"inverse iteration, {dt_cpu:.1f} s"}
    if rank == 0 and world == 1 and not args.no_zstore and p.io == "f64":
        # the Z normalisation pass as its own HBM-bound kernel (MR3_FUSE_SCALE = 0: k_zscale reads
        # and writes every written column once): bytes / its CUDA-event time vs the measured HBM
        # peak; with the default fused epilogue the same traffic runs inside k_rqi
        mr3.set_param("FUSE_SCALE", 0, 0)
        try:
            zt, rt, rrows = [], [], 0.0
            for s in range(2):
                flush.fill_(s)
                w, Z, st = mr3.mr3_dstemr_dd(d, e, "V", p.range, il, iu)
                torch.cuda.synchronize()
                kts = mr3.kernel_times()
                kz = kts.get("k_zscale")
                if kz:
                    zt.append(kz[0])
                if kts.get("k_rqi"):
                    rt.append(kts["k_rqi"][0])
                    rrows = float(st["rqi_rows"])
                del w, Z
        finally:
            mr3.set_param("FUSE_SCALE", -1, 0)
        pk, src = hbm_peak()
        if zt:
            tz = min(zt) * 1e-3
            zbytes = 2.0 * 8.0 * n * m_req  # read + write of every element of Z
            result["roofline_other"]["z_store"] = {
                "bound": "hbm", "kernel": "k_zscale (MR3_FUSE_SCALE=0)",
                "achieved": zbytes / tz / 1e9, "peak": pk, "unit": "GB/s",
                "frac": zbytes / tz / 1e9 / pk, "peak_source": src,
                "bytes_per_launch": zbytes, "ms_per_launch": tz * 1e3,
                "traffic": (traffic_tab.get("k_zscale") if traffic_tab else None),
                "z_algorithmic_bytes": 8.0 * n * m_req,
                "k_rqi_dram_bytes_fused": traffic_tab.get("k_rqi"),
                "note": "Z is written once by the storing RQI pass (8 n m bytes) and read + "
                        "written once more by the exact normalisation (DESIGN.md section 5): 3x "
                        "the algorithmic bytes in total"}
        if rt and rrows:
            # the same launch without its HBM-bound epilogue: the two factorization passes alone
            tr = min(rt) * 1e-3
            ach = rrows * FP64_INST_PER_RQI_ROW[mode] / tr
            result["roofline_other"]["k_rqi_passes_only"] = {
                "bound": "alu", "kernel": "k_rqi (MR3_FUSE_SCALE=0: no normalisation epilogue)",
                "achieved": ach / 1e12, "peak": DERIVED_FP64_PEAK / 1e12, "unit": "T FP64-inst/s",
                "frac": ach / DERIVED_FP64_PEAK,
                "measured_peak_same_run": peak_ips / 1e12,
                "frac_of_measured": ach / peak_ips if peak_ips else None,
                "inst_per_unit": {"rqi_row": FP64_INST_PER_RQI_ROW[mode]},
                "units_per_launch": {"rqi_rows": rrows}, "ms_per_launch": tr * 1e3,
                "note": "k_rqi_fb timed with the normalisation in its own kernel (k_zscale, "
                        "z_store above); the headline roofline keeps the fused launch"}
    if rank == 0 and world == 1 and args.other_configs:
        oc = []
        for cfg in [int(x) for x in args.other_configs.split(",") if x.strip()]:
            if cfg == args.config:
                continue
            oc.append(other_config_line(mr3, cfg, args, flush, stream, peak_ips,
                                        cpu=not args.no_cpu))
        result["other_configs"] = oc
    if rank == 0 and world == 1 and args.dense:
        result["dense"] = dense_line(mr3, int(args.dense), max(3, min(args.steps, 5)), 2, flush,
                                     stream, not args.no_cpu)
    if rank == 0 and world == 1 and args.emulate_world:
        em = []
        for wv in [int(x) for x in args.emulate_world.split(",") if x.strip()]:
            r = emulate_world(mr3, p, wv, stream)
            r["emulated_value"] = m_req / (r["max_rank_ms"] * 1e-3)
            r["unit"] = "eigenpairs/s"
            em.append(r)
        result["emulated_world"] = em
    if rank == 0:
        print(json.dumps(result), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
