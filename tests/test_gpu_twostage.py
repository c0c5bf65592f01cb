"""GPU parity of NEXT-2, the two-stage Sinkhorn algorithm (Algorithm 3), through the C ABI
(cerot_two_stage) against the oracle (oracle.two_stage_sinkhorn) iterate for iterate from the same start.
Bars as DESIGN.md §4: fp32 costs -- plan L1 and marginals 1e-5, objective / dual 1e-6 relative; fp64 costs
-- 1e-10."""
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


def _full_report(f, g, a, b, C, eps):
    T = oracle.plan_full(f, g, C, eps)
    return {"objective": float((C * T).sum()), "row_l1": float(np.abs(T.sum(1) - a).sum()),
            "col_l1": float(np.abs(T.sum(0) - b).sum()), "dual": float(f @ a + g @ b - eps * T.sum()),
            "mass": float(T.sum())}, T


@pytest.mark.parametrize("dtype,tol", [(np.float32, 1e-5), (np.float64, 1e-10)], ids=["f32", "f64"])
@pytest.mark.parametrize("H,noise", [(16, 0.1), (8, 0.3)])
def test_two_stage_matches_oracle(dtype, tol, H, noise):
    p = synthetic.c3_image(H=H)
    a, b = synthetic.approx_symmetric(p, noise=noise)
    C = p.C.astype(dtype)
    eps = 0.05
    f, g, w, z, rep = cot.two_stage_sinkhorn(_dev(a), _dev(b), _dev(C), eps, 15, 25)
    assert (rep["iters1"], rep["iters2"]) == (15, 25)
    fo, go, _, _ = oracle.two_stage_sinkhorn(a, b, C, eps, 15, 25)
    Cf = oracle.expand_cost(C.astype(np.float64))
    ro, To = _full_report(fo, go, a, b, Cf, eps)
    Tg = oracle.plan_full(f.cpu().numpy() * eps, g.cpu().numpy() * eps, Cf, eps)
    assert np.abs(Tg - To).sum() < tol
    rel = 1e-6 if dtype == np.float32 else 1e-10
    assert abs(rep["objective"] - ro["objective"]) <= rel * abs(ro["objective"])
    assert abs(rep["dual"] - ro["dual"]) <= rel * abs(ro["dual"])
    assert abs(rep["row_l1"] - ro["row_l1"]) <= tol
    assert abs(rep["col_l1"] - ro["col_l1"]) <= tol
    # stage-1 potentials: the cyclic Sinkhorn of the fold averages (gauge-invariant: the reduced plan)
    wo, zo, _, _ = oracle.cyclic_sinkhorn(oracle.fold_average(a, p.n), oracle.fold_average(b, p.n), C, eps, 15)
    Tr = oracle.plan_blocks(w.cpu().numpy() * eps, z.cpu().numpy() * eps, C, eps)
    assert p.n * np.abs(Tr - oracle.plan_blocks(wo, zo, C, eps)).sum() < tol


def test_two_stage_exact_symmetry_continues_the_cyclic_iteration():
    p = synthetic.c2_ring(eps_factor=1e-1)
    eps = float(p.eps[0])
    a = oracle.expand_vector(p.alpha, p.n)
    b = oracle.expand_vector(p.beta, p.n)
    f, g, w, z, rep = cot.two_stage_sinkhorn(_dev(a), _dev(b), _dev(p.C), eps, 10, 5)
    prob = cot.CerotProblem(_dev(p.C), _dev(p.alpha), _dev(p.beta), p.eps).init().iterate(15)
    torch.cuda.synchronize()
    C = oracle.expand_cost(p.C.astype(np.float64))
    Tg = oracle.plan_full(f.cpu().numpy() * eps, g.cpu().numpy() * eps, C, eps)
    Tc = oracle.expand_plan(oracle.plan_blocks(prob.w_hat.cpu().numpy() * eps, prob.z_hat.cpu().numpy() * eps,
                                               p.C, eps))
    assert np.abs(Tg - Tc).sum() < 1e-5


def test_two_stage_converges_with_the_oracle():
    """Stage 2 to the marginal tolerance: tol2 is placed at the geometric mean of the oracle's residuals of two
    consecutive iterations (a factor >= 1.02 from each, asserted), so both sides must stop at exactly the same
    iteration, and the plans are compared there (no +-1 allowance)."""
    p = synthetic.c3_image(H=16)
    a, b = synthetic.approx_symmetric(p, noise=0.1)
    C = p.C.astype(np.float64)
    eps = 0.05
    Cf = oracle.expand_cost(C)
    _, zo, _, _ = oracle.cyclic_sinkhorn(oracle.fold_average(a, p.n), oracle.fold_average(b, p.n), C, eps, 30,
                                         form="kernel")
    _, _, _, hist = oracle.sinkhorn_full(a, b, Cf, eps, 40, record=True, g0=oracle.expand_vector(zo, p.n))
    res = [h[2] for h in hist]
    k = next(i for i in range(20, 39) if res[i] > 1.04 * res[i + 1] and all(r > res[i] for r in res[:i]))
    tol2 = float(np.sqrt(res[k] * res[k + 1]))
    fo, go, t1, t2 = oracle.two_stage_sinkhorn(a, b, C, eps, 30, 2000, tol2=tol2)
    assert t2 == k + 2
    f, g, w, z, rep = cot.two_stage_sinkhorn(_dev(a), _dev(b), _dev(C), eps, 30, 2000, tol2=tol2)
    assert rep["converged"] and (rep["iters1"], rep["iters2"]) == (t1, t2)
    assert rep["residual"] <= tol2 and abs(rep["residual"] - res[k + 1]) <= 1e-10
    Tg = oracle.plan_full(f.cpu().numpy() * eps, g.cpu().numpy() * eps, Cf, eps)
    assert np.abs(Tg - oracle.plan_full(fo, go, Cf, eps)).sum() < 1e-10


@pytest.mark.parametrize("dtype", [np.float32, np.float64], ids=["f32", "f64"])
@pytest.mark.parametrize("check_every", [1, 2])
def test_two_stage_gap_rule_matches_oracle(dtype, check_every):
    """App. F's stage-2 stopping rule through cerot_two_stage_gap against oracle.two_stage_sinkhorn_gap:
    the reference value is the oracle's directly solved objective; both stop at the same stage-2 iteration
    (tol_obj sits a factor >= 1.5 away from the gaps of the neighbouring checks, asserted on the oracle side, so
    fp32 cost rounding cannot move the decision) and return the same plan."""
    p = synthetic.c3_image(H=8)
    a, b = synthetic.approx_symmetric(p, noise=0.9)
    C = p.C.astype(dtype)
    C64 = C.astype(np.float64)
    eps = float(p.eps[0]) * 5
    Cf = oracle.expand_cost(C64)
    f0, g0, _, _ = oracle.sinkhorn_full(a, b, Cf, eps, 20000, tol=1e-13)
    ref = oracle.entropic_objective_full(oracle.plan_full(f0, g0, Cf, eps), Cf, eps)
    tol_obj = 5e-5
    fo, go, t1, t2, gap_o = oracle.two_stage_sinkhorn_gap(a, b, C64, eps, 2, 400, ref, tol_obj, check_every=check_every)
    assert 1 < t2 < 400 and gap_o < tol_obj / 1.5
    _, _, _, tprev, gap_prev = oracle.two_stage_sinkhorn_gap(a, b, C64, eps, 2, t2 - check_every, ref, 0.0,
                                                             check_every=check_every)
    assert tprev == t2 - check_every and gap_prev > tol_obj * 1.5
    f, g, w, z, rep = cot.two_stage_sinkhorn(_dev(a), _dev(b), _dev(C), eps, 2, 400, check_every=check_every,
                                             obj_ref=ref, tol_obj=tol_obj)
    assert rep["converged"] and rep["status"] == "COT_OK"
    assert (rep["iters1"], rep["iters2"]) == (t1, t2)
    bar = 1e-5 if dtype == np.float32 else 1e-10           # DESIGN §4 bars
    assert abs(rep["residual"] - gap_o) <= bar            # the measured |objective - obj_ref|
    assert abs(rep["reg_primal"] - (oracle.entropic_objective_full(oracle.plan_full(fo, go, Cf, eps), Cf, eps))) <= bar
    Tg = oracle.plan_full(f.cpu().numpy() * eps, g.cpu().numpy() * eps, Cf, eps)
    assert np.abs(Tg - oracle.plan_full(fo, go, Cf, eps)).sum() < bar


def test_two_stage_gap_rule_not_reached_and_argument_errors():
    p = synthetic.c3_image(H=8)
    a, b = synthetic.approx_symmetric(p, noise=0.5)
    eps = float(p.eps[0]) * 5
    C = p.C.astype(np.float64)
    f, g, w, z, rep = cot.two_stage_sinkhorn(_dev(a), _dev(b), _dev(C), eps, 5, 7, obj_ref=1e3, tol_obj=1e-4)
    assert not rep["converged"] and rep["status"] == "COT_NOT_CONVERGED" and rep["iters2"] == 7
    # the iterates are those of the plain two-stage run (the rule only decides when to stop)
    f2, g2, _, _, _ = cot.two_stage_sinkhorn(_dev(a), _dev(b), _dev(C), eps, 5, 7)
    assert torch.equal(f, f2) and torch.equal(g, g2)
    with pytest.raises(Exception):
        cot.two_stage_sinkhorn(_dev(a), _dev(b), _dev(C), eps, 5, 7, obj_ref=0.0, tol_obj=0.0)
    with pytest.raises(Exception):
        cot.two_stage_sinkhorn(_dev(a), _dev(b), _dev(C), eps, 5, 7, obj_ref=float("nan"), tol_obj=1e-4)
