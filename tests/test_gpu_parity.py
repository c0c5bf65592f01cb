"""GPU parity: the C-ABI path (libcyclicot.so on an sm_100a B200) against the fp64 oracle.

Bars (BASELINE.json north_star):
  * G, argmin and the d x d expansion: bit-exact.
  * C-EROT: objective (transport cost), dual and regularised primal within 1e-6 relative; marginal
    residuals and the plan within 1e-5 in L1 (full scale); the fp64 template (C1) within 1e-10.
Iteration parity is iterate-for-iterate: same start (z = 0), same order (p then q), same count.
"""
import math

import numpy as np
import pytest
import torch

import oracle
import synthetic

pytestmark = pytest.mark.gpu

cot = pytest.importorskip("paper_2311_13147_b200")
DEV = torch.device("cuda:0")


@pytest.fixture(scope="module", autouse=True)
def _built():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    from paper_2311_13147_b200 import build
    build.build()
    cot.lib()


def _dev(x):
    return torch.as_tensor(np.ascontiguousarray(x), device=DEV)


# ------------------------------------------------------------------------------- A2: aggregation
def _agg_cases():
    rng = np.random.default_rng(0)
    ties = rng.integers(0, 3, size=(5, 37, 37)).astype(np.float32)
    signed = np.zeros((3, 4, 4), np.float32)
    signed[1] = -0.0
    signed[2, 0, 0] = -1.0
    return [
        ("C1", synthetic.c1_tiny().C),
        ("C2", synthetic.c2_ring().C),
        ("C3", synthetic.c3_image().C),
        ("C5x8", synthetic.c5_batched(B=8).C),
        ("ties_odd_m", ties),
        ("ties_fp64_odd", ties.astype(np.float64)[:, :7, :7].copy()),
        ("signed_zero", signed),
        ("n1", rng.random((1, 9, 9)).astype(np.float32)),
        ("m1", rng.random((6, 1, 1)).astype(np.float32)),
    ]


@pytest.mark.parametrize("name,C", _agg_cases(), ids=[c[0] for c in _agg_cases()])
def test_aggregate_bitexact(name, C):
    G, A = cot.clot_aggregate(_dev(C))
    Go, Ao = oracle.aggregate(C)
    Gg = G.cpu().numpy()
    assert Gg.dtype == Go.dtype
    assert np.array_equal(Gg.view(np.uint32 if Gg.dtype == np.float32 else np.uint64),
                          Go.view(np.uint32 if Go.dtype == np.float32 else np.uint64))   # sign of zero too
    assert np.array_equal(A.cpu().numpy(), Ao)


def test_aggregate_nonfinite_rejected():
    C = np.random.default_rng(1).random((4, 8, 8)).astype(np.float32)
    for bad in (np.nan, np.inf, -np.inf):
        C2 = C.copy()
        C2[2, 3, 5] = bad
        with pytest.raises(cot.CotError) as e:
            cot.clot_aggregate(_dev(C2))
        assert e.value.code == -2


# ------------------------------------------------------------------------------- A6: expansion
def test_expand_clot_c1_bitexact():
    p = synthetic.c1_tiny()
    r = oracle.clot(p.alpha, p.beta, p.C)
    _, A = cot.clot_aggregate(_dev(p.C))
    T = cot.clot_expand(_dev(r["S"]), p.n, argmin=A).cpu().numpy()
    ref = oracle.expand_plan(oracle.lift(r["S"], r["A"], p.n))
    assert np.array_equal(T, ref)
    # Theorem 1: the expanded plan is feasible and optimal for the explicit problem
    Cf = oracle.expand_cost(p.C)
    assert abs((Cf * T).sum() - r["value"]) < 1e-12


@pytest.mark.parametrize("B,n,m,dt", [(1, 8, 128, np.float32), (3, 4, 37, np.float32), (1, 5, 16, np.float64),
                                      (2, 1, 24, np.float32), (1, 3, 1, np.float64), (2, 6, 130, np.float32)])
def test_expand_blocks_and_lift_bitexact(B, n, m, dt):
    rng = np.random.default_rng(B * 100 + n * 10 + m)
    blocks = rng.random((B, n, m, m)).astype(dt)
    T = cot.clot_expand(_dev(blocks), n).cpu().numpy()
    for b in range(B):
        assert np.array_equal(T[b], oracle.expand_plan(blocks[b]))
    S = rng.random((B, m, m)).astype(dt)
    A = rng.integers(0, n, size=(B, m, m)).astype(np.int32)
    T2 = cot.clot_expand(_dev(S), n, argmin=_dev(A)).cpu().numpy()
    for b in range(B):
        assert np.array_equal(T2[b], oracle.expand_plan(oracle.lift(S[b], A[b], n)))


def test_clot_pipeline_c5_sample():
    """C5 sample: clot_aggregate -> host LP -> clot_expand per problem; value n<G,S> equals the oracle's
    Alg. 1 value and the expanded plan equals the oracle's expansion of the same S (bit-exact)."""
    from paper_2311_13147_b200 import host_lp
    p = synthetic.c5_batched(B=4)
    for b in range(p.B):
        q = p.single(b)
        res = host_lp.clot_solve(_dev(q.C), q.alpha, q.beta)
        ro = oracle.clot(q.alpha, q.beta, q.C)
        assert abs(res["value"] - ro["value"]) <= 1e-9 * max(1.0, abs(ro["value"]))
        S32 = res["S"].cpu().numpy()
        assert np.array_equal(res["argmin"].cpu().numpy(), ro["A"])
        ref = oracle.expand_plan(oracle.lift(S32, ro["A"], q.n))
        assert np.array_equal(res["T_full"].cpu().numpy(), ref)


# ------------------------------------------------------------------------------- A3-A5: C-EROT
def _gpu_run(p, iters, tol=0.0, check_every=1, T_blocks=True, flags=0):
    prob = cot.CerotProblem(_dev(p.C), _dev(p.alpha), _dev(p.beta), _dev(p.eps))
    prob.init().iterate(iters, tol=tol, check_every=check_every, flags=flags)
    T, rep = prob.plan(T_blocks=T_blocks)
    torch.cuda.synchronize()
    it, conv, res = prob.state()
    return prob, (T.cpu().numpy() if T is not None else None), rep.cpu().numpy(), it, conv


def _compare(p, rep_gpu, T_gpu, w, z, obj_rtol=1e-6, l1_tol=1e-5):
    eps = float(p.eps[0])
    ro = oracle.report(w, z, p.alpha, p.beta, p.C, eps)
    g = cot.report_dict(rep_gpu)
    for key in ("objective", "dual", "reg_primal"):
        assert math.isclose(g[key], ro[key], rel_tol=obj_rtol, abs_tol=1e-300), (key, g[key], ro[key])
    for key in ("row_l1", "col_l1"):
        assert abs(g[key] - ro[key]) <= l1_tol, (key, g[key], ro[key])
    assert abs(g["mass"] - ro["mass"]) <= l1_tol
    if T_gpu is not None:
        To = oracle.plan_blocks(w, z, p.C, eps)
        l1 = p.n * np.abs(T_gpu.astype(np.float64) - To).sum()
        assert l1 <= l1_tol, ("plan L1", l1)
        # marginal vectors of the returned plan (full scale, L1)
        r_g, c_g = T_gpu.astype(np.float64).sum(axis=(0, 2)), T_gpu.astype(np.float64).sum(axis=(0, 1))
        assert p.n * np.abs(r_g - ro["r"]).sum() <= l1_tol
        assert p.n * np.abs(c_g - ro["c"]).sum() <= l1_tol
    return g, ro


def test_c1_fp64_to_tolerance():
    """C1 (configs[0]): fp64 template, run to n*sum|c - beta| <= 1e-9 checked every iteration; the GPU stops at
    the same iteration as the oracle and matches it to 1e-10."""
    p = synthetic.c1_tiny()
    w, z, t, _ = oracle.cyclic_sinkhorn(p.alpha, p.beta, p.C, float(p.eps[0]), 100000, tol=p.tol)
    prob, T, rep, it, conv = _gpu_run(p, t + 25, tol=p.tol)
    assert conv[0] == 1 and it[0] == t
    _compare(p, rep[0], T, w, z, obj_rtol=1e-10, l1_tol=1e-10)
    w_g, z_g = prob.w_hat.cpu().numpy(), prob.z_hat.cpu().numpy()
    eps = float(p.eps[0])
    assert np.abs(w_g * eps - w).max() < 1e-10 and np.abs(z_g * eps - z).max() < 1e-10


def test_c1_solve_api():
    p = synthetic.c1_tiny()
    w, z, t, _ = oracle.cyclic_sinkhorn(p.alpha, p.beta, p.C, float(p.eps[0]), 100000, tol=p.tol)
    wg, zg, T, reps = cot.cerot_solve(_dev(p.C), _dev(p.alpha), _dev(p.beta), p.eps, tol=p.tol, max_iter=10000,
                                      check_every=1, T_blocks=True)
    assert reps[0]["converged"] and reps[0]["iters"] == t and reps[0]["status"] == "COT_OK"
    _compare(p, np.array([reps[0][f] for f in cot.REPORT_FIELDS]), T.cpu().numpy(), w, z, 1e-10, 1e-10)


_PATH_FLAGS = {"cluster": 0, "tma": 0x8, "ldg": 0x2}   # default (cluster-resident), COT_FORCE_TMA, COT_FORCE_LDG
_PATH_CODE = {"cluster": 3, "tma": 1, "ldg": 0}        # 3: k_batch_chain (m <= 128)


@pytest.mark.parametrize("eps_factor", [1e-1, 1e-2, 1e-3])
@pytest.mark.parametrize("path", ["cluster", "tma", "ldg"])
def test_c2_500_iterations(eps_factor, path):
    """C2 (configs[1]): ring, fp32, 500 iterations at each eps; iterate parity (not converged at 1e-3).
    Every row path: the cluster-resident kernel C2 takes by default, the persistent TMA kernel (COT_FORCE_TMA)
    and the generic LDG kernels (COT_FORCE_LDG); the path taken is asserted."""
    p = synthetic.c2_ring(eps_factor=eps_factor)
    flags = _PATH_FLAGS[path]
    assert cot.lib().cot_iter_path(1, p.n, p.m, 0, flags) == _PATH_CODE[path]
    w, z, _, _ = oracle.cyclic_sinkhorn(p.alpha, p.beta, p.C, float(p.eps[0]), 500, form="kernel")
    _, T, rep, it, _ = _gpu_run(p, 500, flags=flags)
    assert it[0] == 500
    _compare(p, rep[0], T, w, z)


@pytest.mark.parametrize("kernel", ["res", "tma"])
def test_c3_image_500_iterations(kernel, monkeypatch):
    """C3 (configs[2]): 64x64 rotation-symmetric histograms (stand-in for Table 2's NYU images), eps = 1e-2; on the
    on-chip-resident kernel (k_iter_res, the default) and the streaming persistent kernel (COT_RES=0)."""
    if kernel == "tma":
        monkeypatch.setenv("COT_RES", "0")
    p = synthetic.c3_image(pair=0)
    assert cot.lib().cot_iter_path(1, p.n, p.m, 0, 0) == (4 if kernel == "res" else 1)
    w, z, _, _ = oracle.cyclic_sinkhorn(p.alpha, p.beta, p.C, float(p.eps[0]), 500, form="kernel")
    _, T, rep, _, _ = _gpu_run(p, 500)
    _compare(p, rep[0], T, w, z)


def test_c3_converges_like_oracle():
    p = synthetic.c3_image(pair=1)
    w, z, t, _ = oracle.cyclic_sinkhorn(p.alpha, p.beta, p.C, float(p.eps[0]), 5000, tol=1e-9, form="kernel",
                                        check_every=10)
    assert t < 4000
    _, T, rep, it, conv = _gpu_run(p, t + 50, tol=1e-9, check_every=10)
    assert conv[0] == 1 and it[0] == t
    _compare(p, rep[0], T, w, z)


def test_c4_full_size_500_iterations():
    """C4 (configs[3]) at full size (n = 64, m = 1024, 256 MiB of cost), 500 iterations, the bench's
    launch configuration; the oracle runs Alg. 2 with K precomputed (pinned equal to the streaming form)."""
    p = synthetic.c4_large()
    w, z, _, _ = oracle.cyclic_sinkhorn(p.alpha, p.beta, p.C, float(p.eps[0]), 500, form="kernel")
    _, T, rep, it, _ = _gpu_run(p, 500, T_blocks=False)
    g, ro = _compare(p, rep[0], None, w, z)
    assert g["row_l1"] > 1e-4    # not converged at 500 iterations: the comparison is iterate-for-iterate


def test_c4_full_size_3_iterations_stream_oracle():
    p = synthetic.c4_large()
    w, z, _, _ = oracle.cyclic_sinkhorn(p.alpha, p.beta, p.C, float(p.eps[0]), 3, form="stream")
    _, T, rep, _, _ = _gpu_run(p, 3, T_blocks=True)
    _compare(p, rep[0], T, w, z)


def test_c5_sample_batched_200_iterations():
    """C5 (configs[4]) sample: 8 problems with their own eps in one batched call, 200 iterations."""
    p = synthetic.c5_batched(B=8, first=100)
    prob = cot.CerotProblem(_dev(p.C), _dev(p.alpha), _dev(p.beta), _dev(p.eps))
    prob.init().iterate(200)
    T, rep = prob.plan(T_blocks=True)
    T = T.cpu().numpy()
    rep = rep.cpu().numpy()
    for b in range(p.B):
        q = p.single(b)
        w, z, _, _ = oracle.cyclic_sinkhorn(q.alpha, q.beta, q.C, float(q.eps[0]), 200, form="kernel")
        _compare(q, rep[b], T[b], w, z)


@pytest.mark.parametrize("n,m,dt", [(3, 1, np.float64), (1, 24, np.float32), (5, 37, np.float32),
                                    (4, 130, np.float32), (2, 7, np.float64), (7, 300, np.float32)])
def test_edge_shapes(n, m, dt):
    """Ragged tails (m not a multiple of the vector width or of the CTA), n = 1, m = 1."""
    p = synthetic.random_cyclic(seed=n * 1000 + m, n=n, m=m, dtype=dt, eps=0.05)
    w, z, _, _ = oracle.cyclic_sinkhorn(p.alpha, p.beta, p.C, 0.05, 30)
    _, T, rep, _, _ = _gpu_run(p, 30)
    tol = 1e-10 if dt == np.float64 else 1e-6
    _compare(p, rep[0], T, w, z, obj_rtol=tol, l1_tol=1e-5 if dt == np.float32 else 1e-10)


def test_batch_freeze_rule_matches_oracle():
    """tol > 0 in a batch: each problem stops at its own iteration (rule of SURVEY Q1), others continue."""
    p = synthetic.random_cyclic(seed=5, n=4, m=20, B=3, eps=0.1)
    p.eps = np.array([0.1, 0.05, 0.2])
    prob = cot.CerotProblem(_dev(p.C), _dev(p.alpha), _dev(p.beta), _dev(p.eps))
    prob.init().iterate(3000, tol=1e-8, check_every=5)
    T, rep = prob.plan(T_blocks=True)
    it, conv, _ = prob.state()
    for b in range(3):
        q = p.single(b)
        w, z, t, _ = oracle.cyclic_sinkhorn(q.alpha, q.beta, q.C, float(q.eps[0]), 3000, tol=1e-8, check_every=5)
        assert conv[b] == 1 and it[b] == t
        _compare(q, rep.cpu().numpy()[b], T.cpu().numpy()[b], w, z, obj_rtol=1e-8, l1_tol=1e-8)


def test_warm_start_and_validation():
    p = synthetic.c2_ring(eps_factor=1e-2)
    prob = cot.CerotProblem(_dev(p.C), _dev(p.alpha), _dev(p.beta), _dev(p.eps))
    prob.init().iterate(20)
    prob.init(cold=False).iterate(30)        # warm start: continue from the current z_hat
    T, rep = prob.plan(T_blocks=True)
    w, z, _, _ = oracle.cyclic_sinkhorn(p.alpha, p.beta, p.C, float(p.eps[0]), 50, form="kernel")
    _compare(p, rep.cpu().numpy()[0], T.cpu().numpy(), w, z)
    bad = p.alpha.copy()
    bad[3] = 0.0
    prob2 = cot.CerotProblem(_dev(p.C), _dev(bad), _dev(p.beta), _dev(p.eps))
    prob2.init().iterate(2)
    with pytest.raises(cot.CotError) as e:
        prob2.state()
    assert e.value.code == -3


def test_split_rows_cols_api_matches_iter():
    """cerot_rows + cerot_cols (the split used by the sharded path) == cerot_iter's iterate."""
    p = synthetic.c2_ring(eps_factor=1e-2)
    prob = cot.CerotProblem(_dev(p.C), _dev(p.alpha), _dev(p.beta), _dev(p.eps)).init()
    for t in range(25):
        prob.rows(t & 1)
        prob.cols(t & 1)
    T, rep = prob.plan(T_blocks=True)
    w, z, _, _ = oracle.cyclic_sinkhorn(p.alpha, p.beta, p.C, float(p.eps[0]), 25, form="kernel")
    _compare(p, rep.cpu().numpy()[0], T.cpu().numpy(), w, z)
    it, _, _ = prob.state()
    assert it[0] == 25


def check_stop_iteration(q, it_g, tol, check_every, iters_max, run_fixed, rep_g=None, T_g=None, rel_band=1e-3):
    """Freeze-rule parity for fp32 problems, with no silent skip:
      * the GPU's stopping iteration equals the oracle's, or it is one check away AND the oracle's fp64 monitor at
        the two checks involved lies within `rel_band` of tol (the only case where fp32 rounding of the monitor
        may legitimately decide the other way);
      * the GPU's tol-run state (rep_g, T_g) is compared with the oracle run for exactly it_g iterations;
      * the plan and report at the ORACLE's stopping iteration are always compared too: run_fixed(t) runs the GPU
        for exactly t iterations (no tol) and returns (rep, T)."""
    eps = float(q.eps[0])
    w, z, t, hist = oracle.cyclic_sinkhorn(q.alpha, q.beta, q.C, eps, iters_max, tol=tol, check_every=check_every,
                                           form="kernel", record=True)
    assert t < iters_max, "oracle did not converge"
    it_g = int(it_g)
    if it_g != t:
        assert abs(it_g - t) == check_every, (it_g, t)
        res = {k + 1: h[2] for k, h in enumerate(hist)}
        edge = min(it_g, t)                 # the check at which the two decisions differ
        assert abs(res[edge] / tol - 1) < rel_band, ("stop iteration differs without a borderline monitor",
                                                     it_g, t, res[edge], tol)
    if rep_g is not None:
        wg, zg, _, _ = oracle.cyclic_sinkhorn(q.alpha, q.beta, q.C, eps, it_g, form="kernel")
        _compare(q, rep_g, T_g, wg, zg)
    rep_t, T_t = run_fixed(t)
    _compare(q, rep_t, T_t, w, z)
    return t


def test_cluster_path_batch_freeze_fp32():
    """The cluster-resident path (fp32, m <= 256): per-problem freeze rule in a batch with mixed eps."""
    p = synthetic.random_cyclic(seed=6, n=6, m=32, B=4, eps=0.1, dtype=np.float32)
    p.eps = np.array([0.1, 0.05, 0.2, 0.08])
    prob = cot.CerotProblem(_dev(p.C), _dev(p.alpha), _dev(p.beta), _dev(p.eps))
    prob.init().iterate(4000, tol=1e-7, check_every=5)
    T, rep = prob.plan(T_blocks=True)
    it, conv, _ = prob.state()
    T, rep = T.cpu().numpy(), rep.cpu().numpy()
    for b in range(p.B):
        q = p.single(b)
        assert conv[b] == 1

        def run_fixed(t, q=q):
            _, Tq, rq, itq, _ = _gpu_run(q, t)
            assert itq[0] == t
            return rq[0], Tq
        check_stop_iteration(q, it[b], 1e-7, 5, 4000, run_fixed, rep[b], T[b])


def test_chain_batch_freeze_six_cta_clusters():
    """k_batch_chain in the 6-CTA schedule C5 runs (26-row producers): per-problem freeze rule with mixed eps --
    the problems stop at iterations 20..70 while their producers run up to two iterations ahead of the chain
    CTA and must leave through the stop flag, not a buffer hand-back."""
    p = synthetic.random_cyclic(seed=9, n=4, m=128, B=4, eps=0.1, dtype=np.float32)
    p.eps = np.array([0.01, 0.004, 0.02, 0.007])
    with _env(COT_CHAIN_NCL="6"):
        assert cot.lib().cot_iter_path(p.B, p.n, p.m, 0, 0) == 3
        prob = cot.CerotProblem(_dev(p.C), _dev(p.alpha), _dev(p.beta), _dev(p.eps))
        prob.init().iterate(4000, tol=1e-7, check_every=5)
        T, rep = prob.plan(T_blocks=True)
        it, conv, _ = prob.state()
    T, rep = T.cpu().numpy(), rep.cpu().numpy()
    assert len(set(int(x) for x in it)) > 1
    for b in range(p.B):
        q = p.single(b)
        assert conv[b] == 1

        def run_fixed(t, q=q):
            _, Tq, rq, itq, _ = _gpu_run(q, t)
            assert itq[0] == t
            return rq[0], Tq
        check_stop_iteration(q, it[b], 1e-7, 5, 4000, run_fixed, rep[b], T[b])


@pytest.mark.parametrize("maker,path", [(lambda: synthetic.c2_ring(eps_factor=1e-2), "cluster"),
                                        (lambda: synthetic.c2_ring(eps_factor=1e-2), "ldg"),
                                        (lambda: synthetic.c4_large(m=512, n=32), "tma"),
                                        (lambda: synthetic.c1_tiny(), "ldg"),
                                        (lambda: synthetic.c5_batched(B=3, first=11), "cluster")])
def test_precomputed_mode_matches_alg2(maker, path):
    """NEXT-1: Alg. 2 as written (K precomputed once; O(m^2) per iteration) against the oracle's
    precomputed-K form, iterate for iterate; S itself against the oracle's log K (G-shifted)."""
    p = maker()
    iters = 150
    prob = cot.CerotProblem(_dev(p.C), _dev(p.alpha), _dev(p.beta), _dev(p.eps)).init()
    prob.precompute()
    for b in range(p.B):
        q = p.single(b)
        Go, _ = oracle.aggregate(q.C)
        logK = oracle.lse(-np.asarray(q.C, np.float64) / float(q.eps[0]), axis=0)
        S_ref = np.exp(logK + Go.astype(np.float64) / float(q.eps[0]))     # S = K e^{G/eps} in [1, n]
        S_g = prob.S.cpu().numpy().reshape(p.B, p.m, p.m)[b].astype(np.float64)
        assert np.abs(S_g / S_ref - 1).max() < (1e-12 if q.C.dtype == np.float64 else 2e-6)
    prob.iterate_precomputed(iters, flags=cot.COT_FORCE_LDG if path == "ldg" else 0)
    T, rep = prob.plan(T_blocks=True)
    T = T.cpu().numpy().reshape((p.B,) + p.C.shape[-3:])
    rep = rep.cpu().numpy()
    for b in range(p.B):
        q = p.single(b)
        w, z, _, _ = oracle.cyclic_sinkhorn(q.alpha, q.beta, q.C, float(q.eps[0]), iters, form="kernel")
        fp64 = q.C.dtype == np.float64
        _compare(q, rep[b], T[b], w, z, obj_rtol=1e-10 if fp64 else 1e-6, l1_tol=1e-10 if fp64 else 1e-5)


def test_c5_full_batch_in_the_bench_launch_configuration_sampled():
    """C5 (configs[4]) at full size -- 4096 problems, one batched launch of each step exactly as bench.py times
    it (clot_aggregate, cerot_init, 200 iterations, cerot_plan with T blocks, clot_expand of the C-EROT blocks
    to the 68.7 GB dense plans) -- checked on a sample of problems the oracle computes one by one: G and argmin
    bit-exact, the report and the plan blocks within the bar, the expanded plans bit-exact."""
    p = synthetic.c5_batched(B=4096)
    C = _dev(p.C)
    G, A = cot.clot_aggregate(C)
    prob = cot.CerotProblem(C, _dev(p.alpha), _dev(p.beta), _dev(p.eps))
    prob.init().iterate(200)
    T, rep = prob.plan(T_blocks=True)
    Tfull = cot.clot_expand(T, p.n)
    torch.cuda.synchronize()
    rep = rep.cpu().numpy()
    for b in (0, 1, 777, 2048, 4000, 4095):
        q = p.single(b)
        Go, Ao = oracle.aggregate(q.C)
        assert np.array_equal(G[b].cpu().numpy().view(np.uint32), Go.view(np.uint32))
        assert np.array_equal(A[b].cpu().numpy(), Ao)
        w, z, _, _ = oracle.cyclic_sinkhorn(q.alpha, q.beta, q.C, float(q.eps[0]), 200, form="kernel")
        Tb = T[b].cpu().numpy()
        _compare(q, rep[b], Tb, w, z)
        assert np.array_equal(Tfull[b].cpu().numpy(), oracle.expand_plan(Tb))
    del Tfull, T, C, prob
    torch.cuda.empty_cache()


@pytest.mark.parametrize("n,m,R_seed", [(1, 4, 1), (3, 12, 2), (5, 64, 3), (17, 132, 4), (33, 256, 5), (2, 1020, 6),
                                        (40, 512, 7)])
def test_tma_kernel_shapes(n, m, R_seed):
    """The persistent TMA kernel (forced on shapes the cluster kernel would take) on ragged shapes: n = 1, n not a
    multiple of the slot's k-rows, m not a multiple of the warp width, m up to 1020; 25 iterations against the
    oracle, and a second launch continuing from the first (the epoch / reference hand-over across launches)."""
    p = synthetic.random_cyclic(seed=100 + R_seed, n=n, m=m, dtype=np.float32, eps=0.05)
    prob = cot.CerotProblem(_dev(p.C), _dev(p.alpha), _dev(p.beta), _dev(p.eps)).init()
    prob.iterate(15, flags=cot.COT_FORCE_TMA)
    prob.iterate(10, flags=cot.COT_FORCE_TMA)
    T, rep = prob.plan(T_blocks=True)
    w, z, _, _ = oracle.cyclic_sinkhorn(p.alpha, p.beta, p.C, 0.05, 25, form="kernel")
    _compare(p, rep.cpu().numpy()[0], T.cpu().numpy(), w, z)
    it, _, _ = prob.state()
    assert it[0] == 25


class _env:
    def __init__(self, **kv):
        self.kv = kv

    def __enter__(self):
        import os
        self.old = {k: os.environ.get(k) for k in self.kv}
        os.environ.update({k: str(v) for k, v in self.kv.items()})

    def __exit__(self, *a):
        import os
        for k, v in self.old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


@pytest.mark.parametrize("kernel", ["chain", "cluster"])
@pytest.mark.parametrize("n,m,B", [(1, 8, 1), (3, 12, 1), (5, 36, 2), (17, 128, 1), (16, 128, 20), (4, 132, 1),
                                   (7, 132, 20), (2, 256, 3), (16, 128, 40), (8, 124, 3)])
def test_cluster_kernel_shapes(kernel, n, m, B):
    """The cluster-resident kernels on ragged shapes, in each of their schedules. kernel = "chain": k_batch_chain
    (m <= 128; one CTA runs the iteration chain, the others stream the Gibbs terms), 8-CTA clusters while B fits
    one wave, 6-CTA clusters beyond (B = 20, 40: several waves); kernel = "cluster": k_batch_cluster
    (COT_BATCH_CHAIN=0, and m > 128), warp-specialised for m <= 128, interleaved beyond. n = 1 and n not a
    multiple of 4, rows not a multiple of the warp count. 30 iterations in two launches, every problem against
    the oracle."""
    if kernel == "chain" and m > 128:
        pytest.skip("k_batch_chain holds the m x m problem in one CTA: m <= 128")
    env = {"COT_BATCH_CHAIN": "0"} if kernel == "cluster" else {}
    p = synthetic.random_cyclic(seed=7 * n + m, n=n, m=m, dtype=np.float32, eps=0.05, B=B)
    with _env(**env):
        prob = cot.CerotProblem(_dev(p.C), _dev(p.alpha), _dev(p.beta), _dev(p.eps)).init()
        assert cot.lib().cot_iter_path(B, n, m, 0, 0) == (3 if kernel == "chain" else 2)
        prob.iterate(18)
        prob.iterate(12)
        T, rep = prob.plan(T_blocks=True)
    T, rep = T.cpu().numpy(), rep.cpu().numpy()
    it, _, _ = prob.state()
    assert (np.asarray(it) == 30).all()
    for b in range(B):
        pb = synthetic.Problem("b", p.C[b], p.alpha[b], p.beta[b], p.eps[b:b + 1], iters=0, tol=0.0, meta={})
        w, z, _, _ = oracle.cyclic_sinkhorn(pb.alpha, pb.beta, pb.C, 0.05, 30, form="kernel")
        _compare(pb, rep[b], T[b], w, z)


def test_chain_kernel_launch_boundaries_bitwise():
    """k_batch_chain carries nothing across launches but z_hat (the row shift is the exact maximum every
    iteration): 30 iterations in one launch and in launches of 7 + 11 + 12 give bitwise identical potentials."""
    p = synthetic.c5_batched(B=30, first=200)
    out = []
    for split in ([30], [7, 11, 12]):
        prob = cot.CerotProblem(_dev(p.C), _dev(p.alpha), _dev(p.beta), _dev(p.eps)).init()
        for k in split:
            prob.iterate(k)
        torch.cuda.synchronize()
        out.append((prob.w_hat.cpu().numpy(), prob.z_hat.cpu().numpy()))
    assert cot.lib().cot_iter_path(30, p.n, p.m, 0, 0) == 3
    for a, b in zip(out[0], out[1]):
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64))


@pytest.mark.parametrize("nch", [1, 2, 4])
def test_chain_kernel_split_chain_ctas(nch):
    """k_batch_chain with one chain CTA per problem and with two or four (rows split, the parts of the column
    sums exchanged through DSMEM every iteration: the default while a batch of m = 128 problems fits one wave of
    8-CTA clusters, as C2): the C2 sweep batch against the oracle after 40 iterations, and launch boundaries
    (40 = 13 + 27) bitwise."""
    p = synthetic.c2_sweep()
    out = []
    with _env(COT_CHAIN_NCH=str(nch)):
        assert cot.lib().cot_iter_path(p.B, p.n, p.m, 0, 0) == 3
        for split in ([40], [13, 27]):
            prob = cot.CerotProblem(_dev(p.C), _dev(p.alpha), _dev(p.beta), _dev(p.eps)).init()
            for k in split:
                prob.iterate(k)
            T, rep = prob.plan(T_blocks=True)
            torch.cuda.synchronize()
            out.append((prob.w_hat.cpu().numpy(), prob.z_hat.cpu().numpy(), T.cpu().numpy(), rep.cpu().numpy()))
    for a, b in zip(out[0][:2], out[1][:2]):
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
    T, rep = out[0][2], out[0][3]
    for b in range(p.B):
        q = p.single(b)
        w, z, _, _ = oracle.cyclic_sinkhorn(q.alpha, q.beta, q.C, float(q.eps[0]), 40, form="kernel")
        _compare(q, rep[b], T[b], w, z)


@pytest.mark.parametrize("maker,path,env", [(lambda: synthetic.c1_tiny(), 0, None),
                                            (lambda: synthetic.c3_image(pair=1), 4, None),
                                            (lambda: synthetic.c3_image(pair=1), 1, "0"),
                                            (lambda: synthetic.c2_ring(eps_factor=1e-1), 3, None)],
                         ids=["C1_ldg_graph_loop", "C3_res_one_launch", "C3_tma_one_launch", "C2_chain_one_launch"])
def test_solve_to_tolerance_on_device(maker, path, env, monkeypatch):
    """cerot_solve: "until convergence" on the device -- one persistent launch, or (fp64 / generic path) one
    CUDA graph with a device-side while loop -- stops at the oracle's stopping iteration with the freeze rule
    checked every check_every iterations, and the report matches the oracle there. C3 on the on-chip-resident
    kernel (default) and on the streaming persistent kernel (COT_RES=0)."""
    if env is not None:
        monkeypatch.setenv("COT_RES", env)
    p = maker()
    tol = p.tol if p.tol > 0 else 1e-7
    ce = 1 if path == 0 else 5
    assert cot.lib().cot_iter_path(p.B, p.n, p.m, 1 if p.C.dtype == np.float64 else 0, 0) == path
    w, z, t, _ = oracle.cyclic_sinkhorn(p.alpha, p.beta, p.C, float(p.eps[0]), 20000, tol=tol, check_every=ce,
                                        form="kernel")
    wg, zg, T, reps = cot.cerot_solve(_dev(p.C), _dev(p.alpha), _dev(p.beta), p.eps, tol=tol, max_iter=20000,
                                      check_every=ce, T_blocks=True)
    fp64 = p.C.dtype == np.float64
    assert reps[0]["converged"]
    if fp64:
        assert reps[0]["iters"] == t
        _compare(p, np.array([reps[0][f] for f in cot.REPORT_FIELDS]), T.cpu().numpy(), w, z, 1e-10, 1e-10)
    else:
        def run_fixed(tt):
            _, Tq, rq, itq, _ = _gpu_run(p, tt)
            return rq[0], Tq
        check_stop_iteration(p, reps[0]["iters"], tol, ce, 20000, run_fixed,
                             np.array([reps[0][f] for f in cot.REPORT_FIELDS]), T.cpu().numpy())
