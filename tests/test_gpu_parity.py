"""GPU parity: the CUDA path (through the C-ABI) against the binary128 oracle.

Sizes: small matrices the oracle finishes in seconds that still span several
checkpoint blocks / output tiles and a ragged tail, edge cases, and the
BASELINE.json configurations at full size on sampled outputs (oracle per index)
plus size-independent properties (residuals of every column, exact
orthogonality of every pair, eigenvalue ordering).
"""
import numpy as np
import pytest
import torch

import oracle
import paper_1304_1864_b200 as mr3
import synth
from mr3check import assert_parity, check_solution, exact_gram, exact_orthogonality

pytestmark = pytest.mark.gpu


def run(p, jobz="V", rng=None, il=1, iu=0, vl=0.0, vu=0.0):
    d = torch.from_numpy(p.d).cuda()
    e = torch.from_numpy(p.e).cuda()
    rng = rng or p.range
    if p.io == "f32":
        w, Z, st = mr3.mr3_sstemr_d(d, e, jobz, rng, il or p.il, iu or p.iu, vl, vu)
    else:
        w, Z, st = mr3.mr3_dstemr_dd(d, e, jobz, rng, il or p.il, iu or p.iu, vl, vu)
    torch.cuda.synchronize()
    return w.cpu().numpy(), (Z.cpu().numpy() if Z is not None else None), st


@pytest.mark.parametrize("n", [1, 2, 3, 7, 8, 9, 31, 33, 100, 257])
@pytest.mark.parametrize("kind", ["uniform", "graded", "integer"])
def test_small_random_full(n, kind):
    p = synth.random_small(n, n + 7, kind)
    w, Z, st = run(p)
    assert w.shape == (n,) and Z.shape == (n, n)
    assert np.all(np.diff(w) >= 0)
    res = check_solution(p, w, Z, np.arange(1, n + 1))
    assert_parity(res)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_random_uniform_1200(seed):
    """Several checkpoint blocks, 10 output tiles, ragged tail (1200 = 37*32 + 16)."""
    p = synth.random_uniform(1200, seed)
    w, Z, st = run(p)
    res = check_solution(p, w, Z, np.arange(1, p.n + 1), verbose=True)
    assert_parity(res)
    assert st["d_max"] == 0 and st["largest_cluster"] == 1


def test_config1_121_full():
    """BASELINE config 1 at full size, every pair against the oracle."""
    p = synth.config(1)
    w, Z, st = run(p)
    res = check_solution(p, w, Z, np.arange(1, p.n + 1), verbose=True)
    assert_parity(res)
    assert st["d_max"] == 0  # d_max = 0 for non-Wilkinson types
    k = np.arange(1, p.n + 1)
    assert np.max(np.abs(w - (2 - 2 * np.cos(k * np.pi / (p.n + 1))))) < 4e-16 * 4 + 1e-15


@pytest.mark.parametrize("copies", [2, 5, 12])
def test_glued_wilkinson_small(copies):
    """Clustered spectrum: child representations (tree depth >= 1)."""
    p = synth.glued_wilkinson(copies, 21)
    w, Z, st = run(p)
    res = check_solution(p, w, Z, np.arange(1, p.n + 1), verbose=True)
    assert_parity(res)
    assert st["d_max"] >= 1


def test_index_and_value_ranges():
    p = synth.random_uniform(500, 4)
    w, Z, st = run(p, rng="I", il=37, iu=211)
    assert w.shape == (175,)
    assert_parity(check_solution(p, w, Z, np.arange(37, 212)))
    lh, _ = oracle.eigvals(p.d, p.e)
    vl, vu = 0.5 * (lh[99] + lh[100]), 0.5 * (lh[299] + lh[300])
    w2, Z2, _ = run(p, rng="V", vl=vl, vu=vu)
    assert w2.shape == (200,)
    assert_parity(check_solution(p, w2, Z2, np.arange(101, 301)))
    # upper-half subset uses the right-end root
    w3, Z3, _ = run(p, rng="I", il=450, iu=500)
    assert_parity(check_solution(p, w3, Z3, np.arange(450, 501)))


def test_values_only_matches_vectors_run():
    p = synth.random_uniform(300, 9)
    wn, Zn, _ = run(p, jobz="N")
    wv, Zv, _ = run(p, jobz="V")
    assert Zn is None
    np.testing.assert_array_equal(wn, wv)
    assert_parity(check_solution(p, wn, None, np.arange(1, 301)))


def test_split_matrix():
    """Exact zeros in e split T into blocks."""
    p = synth.split_matrix(90, 3, split_at=(20, 21, 60))
    w, Z, st = run(p)
    assert st["n_blocks"] == 4
    assert np.all(np.diff(w) >= 0)
    assert_parity(check_solution(p, w, Z, np.arange(1, p.n + 1)))
    w2, Z2, _ = run(p, rng="I", il=10, iu=70)
    assert_parity(check_solution(p, w2, Z2, np.arange(10, 71)))


def _interleaved_blocks(io):
    """Blocks whose spectra interleave far below the bisection tolerance: copies of one block
    (equal eigenvalues across blocks), copies shifted by a few ulps of ||T||, and a strongly
    graded tail of tiny blocks -- cut by exact zeros in e."""
    rng = np.random.default_rng(11)
    dt = np.float32 if io == "f32" else np.float64
    ulp = float(np.finfo(dt).eps)
    d0 = rng.standard_normal(37)
    e0 = rng.random(36) + 0.1
    ds, es = [], []
    for c in range(12):
        ds.append(d0 + (c % 4) * 3.0 * ulp * (c % 3 - 1))
        es.append(np.concatenate([e0, [0.0]]))
    k = np.arange(60)
    ds.append(10.0 ** (-k / 6.0))
    es.append(np.where(k % 3 == 2, 0.0, 10.0 ** (-k / 6.0) * 0.2))
    d = np.concatenate(ds).astype(dt)
    e = np.concatenate(es)[:-1].astype(dt)
    return synth.Problem("interleaved-blocks", d, e)


@pytest.mark.parametrize("io", ["f64", "f32"])
def test_split_blocks_interleaved_spectra_sorted(io):
    """include/mr3.h: w ascending.  Eigenvalues of different blocks that agree to within the
    bisection tolerance get their columns from the bracket order; the final stable sort of w
    (k_sort_keys .. k_permute_cols) must put w in order and carry the Z columns along."""
    p = _interleaved_blocks(io)
    w, Z, st = run(p)
    assert st["n_blocks"] > 12
    assert np.all(np.diff(w) >= 0), int(np.sum(np.diff(w) < 0))
    assert_parity(check_solution(p, w, Z, np.arange(1, p.n + 1), io=io, oracle_vectors=False,
                                 gate_angles=False), io=io, gate_angles=False)
    # every column still belongs to its eigenvalue: residual per column in binary64
    d64, e64 = p.d.astype(np.float64), p.e.astype(np.float64)
    Zd, wd = Z.astype(np.float64), w.astype(np.float64)
    TZ = d64[:, None] * Zd
    TZ[:-1] += e64[:, None] * Zd[1:]
    TZ[1:] += e64[:, None] * Zd[:-1]
    eps = 2.0 ** -53 if io == "f64" else 2.0 ** -24
    nrm = oracle.norm1(d64, e64)
    assert np.max(np.linalg.norm(TZ - wd[None, :] * Zd, axis=0)) <= 4 * p.n * eps * nrm
    # values only: the same eigenvalues, ascending
    w2, _, _ = run(p, jobz="N")
    assert np.all(np.diff(w2) >= 0)
    np.testing.assert_allclose(w2, w, rtol=0, atol=8 * eps * nrm)


@pytest.mark.parametrize("lg", [-1045, -1030, 1022])
def test_extreme_norms(lg):
    """||T||_1 subnormal (2^-1047: every entry subnormal) and close to overflow: the power-of-2
    scaling keeps both the scale and its inverse finite.  Checked in a rescaled copy of the
    problem (exact: powers of 2), with the output quantum of w at that magnitude allowed for."""
    base = synth.random_uniform(80, 9)
    d, e = np.ldexp(base.d, lg - 2), np.ldexp(base.e, lg - 2)  # (rounded where subnormal: the input)
    p = synth.Problem("extreme", d, e)
    w, Z, st = run(p)
    dd_, ee_, ww = np.ldexp(d, -lg), np.ldexp(e, -lg), np.ldexp(w, -lg)
    lh, ll = oracle.eigvals(dd_, ee_)
    nrm = oracle.norm1(dd_, ee_)
    quantum = 2.0 ** (-1074 - lg) if lg < -1022 else 0.0
    assert np.all(np.isfinite(w)) and np.all(np.diff(w) >= 0)
    assert np.max(np.abs(ww - (lh + ll))) <= 4e-16 * nrm + quantum
    TZ = dd_[:, None] * Z
    TZ[:-1] += ee_[:, None] * Z[1:]
    TZ[1:] += ee_[:, None] * Z[:-1]
    assert np.max(np.linalg.norm(TZ - ww[None, :] * Z, axis=0)) <= 1e-15 * p.n * nrm + 4 * quantum
    o, dev = exact_orthogonality(torch.from_numpy(Z).cuda())
    assert o <= 1e-14 and dev <= 1e-14


def test_degenerate_inputs():
    # n = 1
    p = synth.Problem("one", np.array([3.5]), np.zeros(0))
    w, Z, _ = run(p)
    assert w.tolist() == [3.5] and Z.tolist() == [[1.0]]
    # diagonal (all splits) with repeated values
    p = synth.Problem("diag", np.array([3.0, 1.0, 2.0, 1.0]), np.zeros(3))
    w, Z, _ = run(p)
    np.testing.assert_array_equal(w, [1.0, 1.0, 2.0, 3.0])
    assert np.allclose(np.abs(Z).sum(0), 1.0) and exact_orthogonality(torch.from_numpy(Z))[0] == 0
    # zero matrix
    p = synth.Problem("zero", np.zeros(5), np.zeros(4))
    w, Z, _ = run(p)
    assert np.all(w == 0) and exact_orthogonality(torch.from_numpy(Z))[0] == 0
    # n = 0
    w, Z, _ = mr3.mr3_dstemr_dd(torch.zeros(0, dtype=torch.float64, device="cuda"),
                                torch.zeros(0, dtype=torch.float64, device="cuda"))
    assert w.numel() == 0


def test_error_codes():
    d = torch.ones(10, dtype=torch.float64, device="cuda")
    e = torch.ones(9, dtype=torch.float64, device="cuda")
    d[3] = float("nan")
    with pytest.raises(mr3.MR3Error) as ex:
        mr3.mr3_dstemr_dd(d, e)
    assert ex.value.code == 1
    d[3] = 1.0
    with pytest.raises(mr3.MR3Error) as ex:
        mr3.mr3_dstemr_dd(d, e, "V", "I", 5, 3)
    assert ex.value.code < 0
    with pytest.raises(mr3.MR3Error):
        mr3.mr3_dstemr_dd(d, e, "V", "V", 1, 1, 2.0, 1.0)


def test_fp32_small_full():
    p = synth.random_normal_f32(1000, 5, 1, 1000)
    p.range = "A"
    w, Z, st = run(p)
    res = check_solution(p, w, Z, np.arange(1, 1001), io="f32")
    assert_parity(res, io="f32")


def test_fp32_subset():
    p = synth.random_normal_f32(3000, 1, 1, 300)
    w, Z, st = run(p)
    res = check_solution(p, w, Z, np.arange(1, 301), io="f32")
    assert_parity(res, io="f32")


def test_deterministic_repeat():
    p = synth.glued_wilkinson(4, 21)
    w1, Z1, _ = run(p)
    w2, Z2, _ = run(p)
    np.testing.assert_array_equal(w1, w2)
    np.testing.assert_array_equal(Z1, Z2)


def _emulate_world(p, world, params=None):
    """Ranks of the plan/execute form emulated one after another on one GPU (each with its
    own context and stream); returns the world-1 solution and the union of the ranks'
    columns, both on the device."""
    import ctypes
    d = torch.from_numpy(p.d).cuda()
    e = torch.from_numpy(p.e).cuda()
    w1, Z1, _ = mr3.mr3_dstemr_dd(d, e)
    L = mr3.lib()
    ctxs, bufs, caps = [], [], []
    streams = [torch.cuda.Stream() for _ in range(world)]
    for r in range(world):
        h = ctypes.c_void_p()
        assert L.mr3_create(ctypes.byref(h), 0, ctypes.c_void_p(streams[r].cuda_stream), None, 0,
                            1) == 0
        for k, v in (params or {}).items():
            L.mr3_set_param(h, 0, mr3.PARAMS[k], float(v))
        ctxs.append(h)
        m = ctypes.c_int64()
        brk = ctypes.c_void_p()
        cap, cnt = ctypes.c_int64(), ctypes.c_int64()
        rc = L.mr3_plan(h, 0, b"A", p.n, ctypes.c_void_p(d.data_ptr()),
                        ctypes.c_void_p(e.data_ptr()), 0.0, 0.0, 1, p.n, r, world,
                        ctypes.byref(m), ctypes.byref(brk), ctypes.byref(cap), ctypes.byref(cnt))
        assert rc == 0
        torch.cuda.synchronize()
        bufs.append(mr3.distributed.wrap_device(brk.value, world * cap.value * mr3.distributed.BRK_REC,
                                                   d.device))
        caps.append(cap.value)
    rec = mr3.distributed.BRK_REC * caps[0]
    full = torch.cat([bufs[r][r * rec:(r + 1) * rec] for r in range(world)])
    for r in range(world):
        bufs[r][:world * rec].copy_(full)
    torch.cuda.synchronize()
    wall = torch.zeros(p.n, dtype=torch.float64, device="cuda")
    Zall = torch.zeros((p.n, p.n), dtype=torch.float64, device="cuda")
    ranges = []
    for r in range(world):
        w = torch.zeros(p.n, dtype=torch.float64, device="cuda")
        zb, ze = ctypes.c_int64(), ctypes.c_int64()
        st = mr3.Stats()
        # size Z from MR3_ERR_ZCAP (the partition is known after classification)
        rc = L.mr3_execute(ctxs[r], b"V", ctypes.c_void_p(w.data_ptr()), None, p.n, 0,
                           ctypes.byref(zb), ctypes.byref(ze), ctypes.byref(st))
        if rc == 6:
            Zs = torch.zeros((ze.value - zb.value, p.n), dtype=torch.float64, device="cuda")
            rc = L.mr3_execute(ctxs[r], b"V", ctypes.c_void_p(w.data_ptr()),
                               ctypes.c_void_p(Zs.data_ptr()), p.n, Zs.shape[0], ctypes.byref(zb),
                               ctypes.byref(ze), ctypes.byref(st))
        assert rc == 0, rc
        torch.cuda.synchronize()
        a, b = zb.value, ze.value
        ranges.append((a, b))
        wall[a:b] = w[a:b]
        if b > a:
            Zall[:, a:b] = Zs[:b - a].T
    for h in ctxs:
        L.mr3_destroy(h)
    assert ranges[0][0] == 0 and ranges[-1][1] == p.n
    assert all(ranges[i][1] == ranges[i + 1][0] for i in range(world - 1))
    return w1, Z1, wall, Zall, ranges


@pytest.mark.parametrize("world", [2, 3, 4])
def test_two_phase_world_emulation_bitwise(world):
    """Ranks of the plan/execute form emulated one after another on one GPU: the
    union of their columns equals the world=1 solve bit for bit."""
    w1, Z1, wall, Zall, _ = _emulate_world(synth.glued_wilkinson(8, 21), world)
    assert torch.equal(wall, w1) and torch.equal(Zall, Z1)


@pytest.mark.slow
@pytest.mark.parametrize("make,world", [(lambda: synth.legendre(20000), 2),
                                        (lambda: synth.legendre(20000), 8),
                                        (lambda: synth.glued_wilkinson(1000, 21), 4)])
def test_world_emulation_bitwise_large(make, world):
    """The same at sizes where the default large-n path runs across ranks: the shared grid
    (>= 512 items), the Newton/Laguerre binary_x phase (one lane per eigenvalue above ~19k
    items) and its fixed-lane multisection tail, the refinement, k_rqi_fb and the k_rqi
    hand-off; and (glued Wilkinson) clusters that must stay whole on one rank."""
    p = make()
    w1, Z1, wall, Zall, ranges = _emulate_world(p, world)
    assert torch.equal(wall, w1)
    assert torch.equal(Zall, Z1)
    del Z1, Zall
    torch.cuda.empty_cache()


def test_fp64_peak_microbenchmark():
    ips, lat = mr3.fp64_peak()
    assert 1e12 < ips < 1e14, ips
    assert 1.0 < lat < 1e4, lat


# ------------------------------------------------------------ full-size configs

def _sample_indices(n, m, k=24, seed=0):
    rng = np.random.default_rng(seed)
    base = [1, 2, 3, m - 2, m - 1, m]
    rest = rng.choice(np.arange(4, m - 2), size=k - len(base), replace=False)
    return np.unique(np.concatenate([base, rest]))


@pytest.mark.slow
def test_config2_full_size():
    p = synth.config(2)
    w, Z, st = run(p)
    assert np.all(np.diff(w) >= 0)
    o, dd = exact_orthogonality(torch.from_numpy(Z).cuda())
    assert o <= 1e-14 and dd <= 1e-14
    r1, r2, _ = oracle.residuals(p.d, p.e, w, Z)
    assert r2.max() <= 1e-15
    idx = _sample_indices(p.n, p.n)
    res = check_solution(p, w[idx - 1], Z[:, idx - 1], idx, full_orth=False, verbose=True)
    assert_parity(res)


@pytest.mark.slow
def test_config3_full_size():
    p = synth.config(3)
    w, Z, st = run(p)
    assert st["d_max"] >= 1
    o, dd = exact_orthogonality(torch.from_numpy(Z).cuda())
    assert o <= 1e-14 and dd <= 1e-14, (o, dd)
    r1, r2, _ = oracle.residuals(p.d, p.e, w, Z)
    assert r2.max() <= 1e-15
    # Weyl: eigenvalues within 2^-26 of the W21 multiset (test_oracle_pins pins the oracle)
    db, eb = synth.wilkinson_block(21)
    jh, jl, _, _ = oracle.jacobi(db, eb)
    ref = np.sort(np.repeat(jh + jl, 200))
    assert np.max(np.abs(w - ref)) <= 2.0 ** -26 * 1.0001
    # every eigenvalue against the oracle
    lh, ll = oracle.eigvals(p.d, p.e)
    assert np.max(np.abs(w - (lh + ll))) <= 4e-16 * oracle.norm1(p.d, p.e)
    # eigenvectors of whole groups against the oracle (R1 floor, per-column angles, subspace
    # angles of the degenerate / glue-split groups; Gap-theorem and Davis-Kahan bounds, SURVEY.md
    # c5): the 200 copies of the lowest and of the highest W21 eigenvalue (the glue-split top
    # pair included), 400 columns -- the whole set in the oracle's binary128 CGS2 takes minutes
    for lo_i, hi_i in ((1, 200), (4001, 4200)):
        idx = np.arange(lo_i, hi_i + 1)
        res = check_solution(p, w[idx - 1], Z[:, idx - 1], idx, full_orth=False, verbose=True)
        assert res["n_groups"] >= 1
        assert_parity(res)


@pytest.mark.slow
def test_config4_full_size():
    p = synth.config(4)
    w, Z, st = run(p)
    assert w.shape == (2000,)
    o, dd = exact_orthogonality(torch.from_numpy(Z).cuda())
    assert o <= 5e-6 and dd <= 5e-6
    # every column: R1 (Eq. (1.1)) and R2 in binary128
    r1, r2, _ = oracle.residuals(p.d.astype(np.float64), p.e.astype(np.float64),
                                 w.astype(np.float64), Z.astype(np.float64))
    print("config 4: R1 max %.3g R2 max %.3g" % (r1.max(), r2.max()))
    assert r1.max() <= 5e-7
    idx = _sample_indices(p.n, 2000, k=64)
    res = check_solution(p, w[idx - 1], Z[:, idx - 1], idx, io="f32", full_orth=False,
                         verbose=True)
    assert_parity(res, io="f32")


@pytest.mark.slow
def test_config5_full_size_sampled():
    """Legendre n = 50000 (Z = 20 GB): the bench workload, sampled against the oracle."""
    p = synth.config(5)
    d = torch.from_numpy(p.d).cuda()
    e = torch.from_numpy(p.e).cuda()
    w, Z, st = mr3.mr3_dstemr_dd(d, e)
    torch.cuda.synchronize()
    assert st["d_max"] == 0 and st["largest_cluster"] == 1  # rho = 1/n (Table 2)
    wc = w.cpu().numpy()
    assert np.all(np.diff(wc) > 0)
    # 512 indices against the oracle: 64 from each dense end of the spectrum (the
    # Gauss-Legendre nodes cluster at +-1) and 384 spread over the interior
    rng = np.random.default_rng(5)
    idx = np.unique(np.concatenate([np.arange(1, 65), np.arange(p.n - 63, p.n + 1),
                                    rng.choice(np.arange(65, p.n - 63), 384, replace=False)]))
    assert idx.size == 512
    Zs = Z[:, torch.from_numpy(idx - 1).cuda()]
    res = check_solution(p, wc[idx - 1], Zs.cpu().numpy(), idx, full_orth=True, verbose=True)
    assert_parity(res)
    # R2 of every column (binary128 residuals, chunked through host memory)
    r2max, r1max = 0.0, 0.0
    for c0 in range(0, p.n, 2500):
        r1, r2, _ = oracle.residuals(p.d, p.e, wc[c0:c0 + 2500], Z[:, c0:c0 + 2500].cpu().numpy())
        r2max, r1max = max(r2max, float(r2.max())), max(r1max, float(r1.max()))
    print("config 5: all columns R2 max %.3g R1 max %.3g" % (r2max, r1max))
    assert r2max <= 1e-15
    # orthogonality of the sample against every column, exactly (c7)
    omax = 0.0
    for c0 in range(0, p.n, 5000):
        G = exact_gram(Zs, Z[:, c0:c0 + 5000])
        for j, k in enumerate(idx - 1):
            if c0 <= k < c0 + 5000:
                G[j, k - c0] -= 1.0
        omax = max(omax, float(G.abs().max()))
        del G
    assert omax <= 1e-14, omax
    del Z
    torch.cuda.empty_cache()


@pytest.mark.parametrize("io", ["f64", "f32"])
def test_host_buffer_abi_matches_device_abi(io):
    """mr3_*_host (host d, e, w, Z; copies inside the call) == the device-pointer call,
    bit for bit, including an index subset."""
    if io == "f64":
        p = synth.random_uniform(700, 5)
        fn = mr3.mr3_dstemr_dd
    else:
        p = synth.random_normal_f32(700, 2, 1, 120)
        fn = mr3.mr3_sstemr_d
    for rng, il, iu in (("A", 1, p.n), ("I", 37, 160)):
        w1, Z1, _ = fn(torch.from_numpy(p.d).cuda(), torch.from_numpy(p.e).cuda(), "V", rng, il, iu)
        hd = torch.from_numpy(p.d).pin_memory()
        he = torch.from_numpy(p.e).pin_memory()
        w2, Z2, _ = mr3.solve_host(hd, he, "V", rng, il, iu)
        np.testing.assert_array_equal(w1.cpu().numpy(), w2.numpy())
        np.testing.assert_array_equal(Z1.cpu().numpy(), Z2.numpy())
        w3, Z3, _ = mr3.solve_host(p.d, p.e, "N", rng, il, iu)  # pageable, values only
        assert Z3 is None
        np.testing.assert_array_equal(w1.cpu().numpy(), w3.numpy())


@pytest.mark.parametrize("make", [lambda: synth.random_uniform(900, 11), lambda: synth.one_two_one(700),
                                  lambda: synth.glued_wilkinson(12, 21),
                                  lambda: synth.legendre(3000)])
def test_root_certification_modes_agree(make):
    """Reading R8d: the binary_x root brackets widened by the definite root's relative
    robustness bound (MR3_YCERT = 0, default) give the same eigenvalues, bit for bit, as
    certifying every bracket with binary_y Sturm counts (MR3_YCERT = 1), and the same
    eigenvectors up to sign and rounding (reading R10: the RQI of the default path starts
    from the Newton estimate of its binary_x phase, the certified path from the midpoint)."""
    p = make()
    d = torch.from_numpy(p.d).cuda()
    e = torch.from_numpy(p.e).cuda()
    try:
        mr3.set_param("YCERT", 1)
        w1, Z1, s1 = mr3.mr3_dstemr_dd(d, e)
        mr3.set_param("YCERT", 0)
        w0, Z0, s0 = mr3.mr3_dstemr_dd(d, e)
    finally:
        mr3.set_param("YCERT", -1)
    assert s1["bisect_rows"] > s0["bisect_rows"]
    np.testing.assert_array_equal(w1.cpu().numpy(), w0.cpu().numpy())
    # (the twist, located at the RQI start, fixes the sign z_r > 0: a different start may
    # pick another twist, i.e. the other sign)
    z1, z0 = Z1.cpu().numpy(), Z0.cpu().numpy()
    sgn = np.where(np.sum(z1 * z0, axis=0) < 0, -1.0, 1.0)  # columns are the vectors
    dz = np.abs(z1 - sgn[None, :] * z0)
    assert dz.max() <= 1e-13, dz.max()


def _with_params(params, fn, mode=0):
    try:
        for k, v in params.items():
            mr3.set_param(k, v, mode)
        return fn()
    finally:
        for k in params:
            mr3.set_param(k, -1, mode)


def test_default_needs_no_rqi_fallback():
    """The located twists and RQI starts converge for representative matrices without the
    bisection fallback (P:L720-L727 keep it for the rare failures): a regression guard for
    the twist location (R9b) -- a poor twist leaves |gamma_r| large at every iteration."""
    for p in (synth.random_uniform(900, 11), synth.glued_wilkinson(12, 21), synth.legendre(3000),
              synth.one_two_one(700)):
        _, _, st = run(p)
        assert st["rqi_fallbacks"] == 0, (p.name, st["rqi_fallbacks"])


@pytest.mark.parametrize("params", [
    {"MAX_RQI": 1},            # every singleton takes the bisection fallback + sweep-form z
    {"REFINE": 1e12},          # all starts refined: many converge in the first (non-storing)
                               # pass and join the second as store-only
    {"KRS": 1e-4},             # tighter stopping: third and later iterations, as split passes
    {"KRS": 1e-4, "SPLIT": 0},  # the same iterations as serial passes
    {"SPLIT": 2},              # small sets: every iteration a split pass, one eigenpair per CTA
    {"TWISTW": 0},             # unweighted argmin twist
    {"NEWTON": 1},             # almost every item through the many-lane multisection tail
    {"XPTS": 1},               # plain bisection in the binary_x phase
    {"XPTS": 2},               # two points per lane
    {"GRID": 0},               # no shared grid start
    {"REFINE": 0},             # midpoints as RQI starts
    {"RELAX": 0},              # every bracket to rtol (no NEXT-1b relaxed stop)
    {"ABSGAP": 1e-12},         # absolute-gap splitting (NEXT-3)
])
def test_rare_paths_parity(params):
    """The paths the default workload rarely takes, forced by parameters, against the oracle."""
    for p in (synth.random_uniform(700, 4), synth.glued_wilkinson(4, 21), synth.legendre(1500)):
        w, Z, st = _with_params(params, lambda: run(p))
        res = check_solution(p, w, Z, np.arange(1, p.n + 1))
        assert_parity(res)
        if params.get("MAX_RQI") == 1 and not p.name.startswith("glued"):
            assert st["rqi_fallbacks"] > 0


@pytest.mark.parametrize("make", [lambda: synth.legendre(3000), lambda: synth.random_uniform(1500, 3),
                                  lambda: synth.random_uniform(700, 8),
                                  lambda: synth.glued_wilkinson(30, 21)])
@pytest.mark.parametrize("params", [{"GROUPS": 1}, {"GROUPS": 1, "NEWTON": 1}])
def test_newton_path_parity(make, params):
    """The bench workload's own bisection path -- one lane per eigenvalue, the
    Newton/Laguerre-accelerated binary_x phase (R8e) and its multisection tail -- which the
    automatic lane choice takes only above ~19k items, forced at small n (GROUPS = 1) and
    checked against the oracle on every pair."""
    p = make()
    w, Z, st = _with_params(params, lambda: run(p))
    assert st["newton_rows_x"] > 0, st  # the Newton passes really ran
    res = check_solution(p, w, Z, np.arange(1, p.n + 1))
    assert_parity(res)


def test_fused_scale_off_bitwise():
    """MR3_FUSE_SCALE = 0 (one k_zscale launch after the RQI phase) computes exactly what the
    fused epilogue of k_rqi computes: same bits."""
    for p in (synth.random_uniform(900, 2), synth.glued_wilkinson(12, 21),
              synth.random_normal_f32(1200, 3, 1, 200)):
        w1, Z1, _ = run(p)
        w0, Z0, _ = _with_params({"FUSE_SCALE": 0}, lambda: run(p))
        np.testing.assert_array_equal(w1, w0)
        np.testing.assert_array_equal(Z1, Z0)


@pytest.mark.parametrize("make", [lambda: synth.glued_wilkinson(12, 21),
                                  lambda: synth.glued_wilkinson(40, 21)])
def test_pool_batches_bitwise(make):
    """Clusters processed in depth-first batches (child-pool budget MR3_POOL_MB forced to one
    cluster per batch) give the same eigenpairs, bit for bit, as one batch per level."""
    p = make()
    w1, Z1, s1 = run(p)
    w0, Z0, s0 = _with_params({"POOL_MB": 1e-9}, lambda: run(p))
    assert s1["n_clusters"] == s0["n_clusters"] and s1["d_max"] == s0["d_max"] >= 1
    np.testing.assert_array_equal(w1, w0)
    np.testing.assert_array_equal(Z1, Z0)
    res = check_solution(p, w0, Z0, np.arange(1, p.n + 1))
    assert_parity(res)


def test_index_range_z_columns():
    """An index range allocates and returns exactly iu - il + 1 columns."""
    p = synth.random_uniform(800, 6)
    w, Z, _ = run(p, rng="I", il=101, iu=164)
    assert Z.shape == (800, 64) and w.shape == (64,)
    assert_parity(check_solution(p, w, Z, np.arange(101, 165)))


@pytest.mark.parametrize("make", [lambda: synth.random_uniform(1200, 1), lambda: synth.legendre(3000),
                                  lambda: synth.glued_wilkinson(20, 21),
                                  lambda: synth.random_normal_f32(3000, 4, 1, 700),
                                  lambda: synth.split_matrix(500, 5, split_at=(100, 101, 333))])
@pytest.mark.parametrize("params", [{}, {"MAX_RQI": 1}, {"KRS": 1e-4}, {"GROUPS": 1}])
def test_rqi_fb_matches_single_thread_rqi(make, params):
    """k_rqi_fb (the two halves of every twisted factorization in two threads, iterations 1-2,
    then k_rqi from the saved state) computes exactly what k_rqi alone computes (MR3_RQI_FB = 0):
    same bits, including eigenpairs continued after the hand-off (KRS = 1e-4 forces third
    iterations, MAX_RQI = 1 the bisection fallback)."""
    p = make()
    # (RQI_CHUNK = 0: small sets take k_rqi_fb too, with the stragglers in serial k_rqi)
    w1, Z1, s1 = _with_params(dict(params, RQI_CHUNK=0), lambda: run(p))
    w0, Z0, s0 = _with_params(dict(params, RQI_FB=0, RQI_CHUNK=0), lambda: run(p))
    np.testing.assert_array_equal(w1, w0)
    np.testing.assert_array_equal(Z1, Z0)
    assert s1["rqi_fallbacks"] == s0["rqi_fallbacks"]


@pytest.mark.parametrize("make", [lambda: synth.random_uniform(1200, 1), lambda: synth.legendre(3000),
                                  lambda: synth.glued_wilkinson(20, 21),
                                  lambda: synth.random_normal_f32(2000, 4, 1, 300),
                                  lambda: synth.split_matrix(500, 5, split_at=(100, 101, 333)),
                                  lambda: synth.random_uniform(5000, 7)])
@pytest.mark.parametrize("params", [{}, {"MAX_RQI": 1}, {"KRS": 1e-4}])
def test_rqi_chunk_parity(make, params):
    """k_rqi_chunk (every RQI iteration chunk-parallel over a CTA, one eigenpair per CTA: the
    small-index-set path, default up to 8192 singletons) against the oracle on every pair, and
    against the serial k_rqi_fb path to the accuracy of the method (different rounding of the
    same recurrences)."""
    p = make()
    io = p.io
    w1, Z1, s1 = _with_params(params, lambda: run(p))
    il, iu = p.index_range()
    res = check_solution(p, w1, Z1, np.arange(il, iu + 1), io=io)
    assert_parity(res, io=io)
    w0, Z0, _ = _with_params(dict(params, RQI_CHUNK=0), lambda: run(p))
    nrm = float(np.abs(p.d).max() + 2 * np.abs(p.e).max())
    tolw = (4e-16 if io == "f64" else 4 * 2.0 ** -24) * nrm * 2
    assert np.max(np.abs(w1.astype(np.float64) - w0)) <= tolw



@pytest.mark.parametrize("make", [lambda: synth.random_uniform(1200, 2), lambda: synth.one_two_one(900),
                                  lambda: synth.glued_wilkinson(10, 21),
                                  lambda: synth.random_normal_f32(3000, 1, 1, 400)])
def test_relaxed_isolation_stop(make):
    """NEXT-1b (R20): bisection of eigenvalues that their own
    Sturm counts isolate stops at c gap sqrt(eps_x sqrt(n) / C) instead of rtol.  Fewer Sturm
    rows, the same classification, parity with the oracle, and RQI from the wider brackets
    without the bisection fallback."""
    p = make()
    w1, Z1, s1 = run(p)                                      # default: RELAX = 0.5
    w0, Z0, s0 = _with_params({"RELAX": 0}, lambda: run(p),  # every bracket to rtol
                              mode=1 if p.io == "f32" else 0)
    ks = np.arange(p.il, p.iu + 1) if p.range == "I" else np.arange(1, p.n + 1)
    for w, Z in ((w1, Z1), (w0, Z0)):
        assert_parity(check_solution(p, w, Z, ks, io=p.io), io=p.io)
    rows1 = s1["bisect_rows"] + s1["bisect_rows_x"]
    rows0 = s0["bisect_rows"] + s0["bisect_rows_x"]
    assert rows1 < rows0, (rows1, rows0)
    assert s1["n_clusters"] == s0["n_clusters"] and s1["d_max"] == s0["d_max"]
    assert s1["rqi_fallbacks"] == 0


def test_absolute_gap_splitting():
    """NEXT-3 (R21): glued Wilkinson's top W21 pairs
    are split by the glue by ~5.6e-11 (relative gap ~4e-12 < gaptol = 1e-10, so they form
    clusters); with MR3_ABSGAP = 1e-12 the absolute gap >= 1e-12 ||T||_1 separates them at
    the root.  Fewer clusters, the same parity with the oracle."""
    p = synth.glued_wilkinson(2, 21)
    w0, Z0, s0 = run(p)
    w1, Z1, s1 = _with_params({"ABSGAP": 1e-12}, lambda: run(p))
    ks = np.arange(1, p.n + 1)
    assert_parity(check_solution(p, w0, Z0, ks))
    assert_parity(check_solution(p, w1, Z1, ks))
    assert s1["n_clusters"] < s0["n_clusters"], (s1["n_clusters"], s0["n_clusters"])


@pytest.mark.slow
def test_backtracking_from_grandparent():
    """NEXT-3 backtracking (R22): a child at depth >= 2 that
    fails the acceptance tests is redone from its grandparent.  The test hook MR3_BACKTRACK = 2
    fails every depth->=2 child first, so each such cluster of config 3 (glued Wilkinson, the
    one matrix here with a depth-2 tree) takes the backtracking path; the solve keeps the
    config-3 parity bar.  By default no child fails, so nothing backtracks."""
    p = synth.config(3)
    _, _, s0 = run(p)
    assert s0["d_max"] >= 2 and s0["backtrack_tries"] == 0 and s0["robustness_failures"] == 0
    w, Z, st = _with_params({"BACKTRACK": 2}, lambda: run(p))
    assert st["backtrack_tries"] > 0 and st["backtracks"] == st["backtrack_tries"], st
    assert st["robustness_failures"] == 0, st
    o, dd = exact_orthogonality(torch.from_numpy(Z).cuda())
    assert o <= 1e-14 and dd <= 1e-14, (o, dd)
    r1, r2, _ = oracle.residuals(p.d, p.e, w, Z)
    assert r2.max() <= 1e-15
    lh, ll = oracle.eigvals(p.d, p.e)
    assert np.max(np.abs(w - (lh + ll))) <= 4e-16 * oracle.norm1(p.d, p.e)
    for lo_i, hi_i in ((1, 200), (4001, 4200)):
        idx = np.arange(lo_i, hi_i + 1)
        res = check_solution(p, w[idx - 1], Z[:, idx - 1], idx, full_orth=False)
        assert_parity(res)


_STRAGGLER_SCRIPT = r"""
import sys
import numpy as np
import torch
sys.path.insert(0, {root!r})
import paper_1304_1864_b200 as mr3
k = np.arange(3000)
d = 2.0 ** (-k / 4.0)
e = 2.0 ** (-(k[:-1] + 0.5) / 4.0) * 0.3
mr3.set_param("RQI_CHUNK", 1, 0)   # m > 1: the k_rqi_fb path, its stragglers to k_rqi_chunk
w, Z, st = mr3.mr3_dstemr_dd(torch.from_numpy(d).cuda(), torch.from_numpy(e).cuda(), "V", "A")
torch.cuda.synchronize()
np.savez({out!r}, w=w.cpu().numpy(), Z=Z.cpu().numpy(), fb=st["rqi_fallbacks"], nb=st["n_blocks"])
"""


def test_fb_stragglers_that_never_converge(tmp_path):
    """Strongly graded T (d_k = 2^(-k/4)): three eigenpairs at the small end of its leading block
    use every RQI iteration and end in the bisection fallback.  On the k_rqi_fb path they
    continue in k_rqi_chunk from a saved state; its loop must start at the same iteration in
    every thread (a CTA-wide barrier sits inside) -- with the owner thread's private count the
    kernel never returned (found by tools/stress.py --large).  Run in a child process with a
    time limit so that a regression fails instead of hanging the suite."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = str(tmp_path / "res.npz")
    r = subprocess.run([sys.executable, "-c", _STRAGGLER_SCRIPT.format(root=root, out=out)],
                       capture_output=True, text=True, timeout=240)
    assert r.returncode == 0, r.stderr[-2000:]
    f = np.load(out)
    w, Z = f["w"], f["Z"]
    assert int(f["nb"]) > 2000 and int(f["fb"]) >= 1
    k = np.arange(3000)
    d = 2.0 ** (-k / 4.0)
    e = 2.0 ** (-(k[:-1] + 0.5) / 4.0) * 0.3
    p = synth.Problem("graded-down", d, e)
    assert np.all(np.diff(w) >= 0)
    assert_parity(check_solution(p, w, Z, np.arange(1, p.n + 1), oracle_vectors=False,
                                 gate_angles=False), gate_angles=False)
