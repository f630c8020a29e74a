"""CPU-only checks of the C-ABI library: it loads, exports every symbol that
include/mr3.h declares, and its host-only logic (column partition, error
strings) behaves.  No compute call needs a GPU here."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_1304_1864_b200 as mr3

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    mr3.build()
    return mr3.lib()


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "mr3.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mr3_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported(L):
    syms = declared_symbols()
    assert len(syms) >= 12
    for s in syms:
        assert hasattr(L, s), s


def test_version_and_strerror(L):
    assert b"sm_100a" in L.mr3_version()
    assert L.mr3_strerror(0) == b"ok"
    assert b"NaN" in L.mr3_strerror(1)
    assert L.mr3_strerror(-3) == b"invalid argument"


def test_built_for_sm100a():
    out = os.popen(f"cuobjdump --list-elf {mr3.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out, out


def test_partition_basic():
    # 10 singletons of cost 1 over 2 ranks -> 5 + 5
    sb = list(range(11))
    cb = mr3.partition_columns(sb, [1.0] * 10, 2)
    assert cb.tolist() == [0, 5, 10]


def test_partition_never_cuts_a_cluster():
    # segments: singles, a cluster of 6 columns [3, 9), singles
    sb = [0, 1, 2, 3, 9, 10, 11, 12]
    cost = [1, 1, 1, 18, 1, 1, 1]
    for world in (1, 2, 3, 4, 8):
        cb = mr3.partition_columns(sb, cost, world)
        assert cb[0] == 0 and cb[-1] == 12 and np.all(np.diff(cb) >= 0)
        for c in cb:
            assert not (3 < c < 9), (world, cb)


def test_partition_balances_cost():
    rng = np.random.default_rng(0)
    sizes = rng.integers(1, 4, 200)
    sb = np.concatenate([[0], np.cumsum(sizes)])
    cost = sizes * np.where(sizes > 1, 3.0, 1.0)
    cb = mr3.partition_columns(sb, cost, 4)
    seg_of = {int(c): i for i, c in enumerate(sb)}
    loads = [cost[seg_of[int(cb[r])]:seg_of[int(cb[r + 1])]].sum() for r in range(4)]
    assert max(loads) <= cost.sum() / 4 + cost.max() + 1e-9


def test_partition_bad_args(L):
    out = (ctypes.c_int64 * 3)()
    sb = (ctypes.c_int64 * 2)(0, 1)
    cs = (ctypes.c_double * 1)(1.0)
    assert L.mr3_partition_columns(1, sb, cs, 0, out) == -1


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    d = torch.ones(4, dtype=torch.float64)
    with pytest.raises((RuntimeError, TypeError)):
        mr3.mr3_dstemr_dd(d, torch.ones(3, dtype=torch.float64))


def test_bracket_record_size_matches_header():
    src = open(os.path.join(ROOT, "include", "mr3.h")).read()
    m = re.search(r"#define\s+MR3_BRK_REC\s+(\d+)", src)
    assert m is not None
    from paper_1304_1864_b200.distributed import BRK_REC
    assert int(m.group(1)) == BRK_REC
