"""Pins of the NEXT-2 oracle (two-stage Sinkhorn, Algorithm 3).

* Exact symmetry: if a, b are exactly n-periodic, stage 2 continues stage 1 iterate for iterate -- the full
  Sinkhorn iterates from tiled potentials are the tiled cyclic iterates (P:161-168 with P:398-411) -- so
  two_stage(t1, t2) equals cyclic Sinkhorn run t1 + t2 iterations, tiled ("the time complexity of this
  algorithm is the same as that of the cyclic Sinkhorn algorithm").
* Approximate symmetry: the EROT optimum is unique (strict convexity), so at convergence the two-stage
  result equals the original Sinkhorn run from scratch on the explicit problem (a textbook routine), and the
  plan has the marginals a, b.
* The fold average keeps mass and is the identity on periodic vectors."""
import numpy as np

import oracle
import synthetic


def test_exact_symmetry_reduces_to_cyclic_sinkhorn():
    p = synthetic.random_cyclic(seed=5, n=4, m=9, eps=0.1)
    eps = float(p.eps[0])
    a = oracle.expand_vector(p.alpha, p.n)
    b = oracle.expand_vector(p.beta, p.n)
    f, g, t1, t2 = oracle.two_stage_sinkhorn(a, b, p.C, eps, 7, 11)
    assert (t1, t2) == (7, 11)
    w, z, _, _ = oracle.cyclic_sinkhorn(p.alpha, p.beta, p.C, eps, 18)
    assert np.abs(f - oracle.expand_vector(w, p.n)).max() < 1e-12
    assert np.abs(g - oracle.expand_vector(z, p.n)).max() < 1e-12


def test_approximate_symmetry_converges_to_the_unique_optimum():
    p = synthetic.c3_image(H=8)            # n = 4, m = 16, d = 64
    a, b = synthetic.approx_symmetric(p, noise=0.2)
    eps = float(p.eps[0]) * 5
    C = oracle.expand_cost(p.C)
    f2, g2, t1, t2 = oracle.two_stage_sinkhorn(a, b, p.C, eps, 50, 5000, tol2=1e-13)
    assert t2 < 5000
    f0, g0, t0, _ = oracle.sinkhorn_full(a, b, C, eps, 20000, tol=1e-13)
    T2 = oracle.plan_full(f2, g2, C, eps)
    T0 = oracle.plan_full(f0, g0, C, eps)
    assert np.abs(T2 - T0).sum() < 1e-10
    assert np.abs(T2.sum(1) - a).sum() < 1e-10 and np.abs(T2.sum(0) - b).sum() < 1e-12
    # the warm start from the symmetric stage-1 solution needs fewer stage-2 iterations than a cold start
    assert t2 < t0


def test_fold_average_mass_and_periodic_identity():
    rng = np.random.default_rng(0)
    v = rng.random(24)
    al = oracle.fold_average(v, 4)
    assert abs(al.sum() - v.sum() / 4) < 1e-15
    assert np.allclose(oracle.fold_average(oracle.expand_vector(al, 4), 4), al, atol=0, rtol=1e-15)


def test_stage2_warm_start_is_alg3_line11():
    """Stage 2 starts from q = concatenated q^: with zero stage-2 iterations allowed to change
    nothing, one stage-2 iteration from the tiled stage-1 potentials is a plain p-update of the explicit
    problem (eq. P:403-411 with n = 1), evaluated here by brute force."""
    p = synthetic.random_cyclic(seed=9, n=3, m=5, eps=0.2)
    eps = float(p.eps[0])
    a, b = synthetic.approx_symmetric(p, noise=0.3, seed=2)
    C = oracle.expand_cost(p.C)
    w, z, _, _ = oracle.cyclic_sinkhorn(oracle.fold_average(a, 3), oracle.fold_average(b, 3), p.C, eps, 4,
                                        form="kernel")
    f, g, _, _ = oracle.two_stage_sinkhorn(a, b, p.C, eps, 4, 1)
    zt = oracle.expand_vector(z, 3)
    f_bf = np.array([eps * (np.log(a[I]) - np.log(sum(np.exp((zt[J] - C[I, J]) / eps) for J in range(15))))
                     for I in range(15)])
    assert np.abs(f - f_bf).max() < 1e-12


def test_entropic_objective_closed_form_and_duality():
    """Pins of entropic_objective_full (eq. problem_CROT + eq. reg_for_entropy_ROT): (i) closed form for the
    independent coupling with zero cost, eps (sum a log a + sum b log b - 1); (ii) strong duality at the
    Sinkhorn optimum (eq. dual_problem_cyclic_ROT with n = 1): primal = <f,a> + <g,b> - eps sum T, a value
    computed without the entropy term, so a wrong sign or a dropped '-1' fails."""
    rng = np.random.default_rng(3)
    a = rng.random(6); a /= a.sum()
    b = rng.random(7); b /= b.sum()
    T = np.outer(a, b)
    want = 0.3 * ((a * np.log(a)).sum() + (b * np.log(b)).sum() - 1.0)
    assert abs(oracle.entropic_objective_full(T, np.zeros((6, 7)), 0.3) - want) < 1e-14
    C = rng.random((6, 7))
    f, g, _, _ = oracle.sinkhorn_full(a, b, C, 0.2, 5000, tol=1e-14)
    Topt = oracle.plan_full(f, g, C, 0.2)
    dual = f @ a + g @ b - 0.2 * Topt.sum()
    assert abs(oracle.entropic_objective_full(Topt, C, 0.2) - dual) < 1e-11
    # suboptimal feasible plan: primal above the optimum (the objective is minimised)
    assert oracle.entropic_objective_full(T, C, 0.2) > dual + 1e-6


def test_gap_rule_stops_at_the_first_iteration_within_tol():
    """App. F: stage 2 stops at the first checked iteration whose objective is within tol_obj of the
    directly solved value. Checked against the recorded iterates of the plain original Sinkhorn from the same
    start (sinkhorn_full(record=True)): the stop index is the first one below tol, the one before is not, and
    the returned potentials are that iterate; a tol never reached runs all iters2; a huge tol stops at once."""
    p = synthetic.c3_image(H=8)
    a, b = synthetic.approx_symmetric(p, noise=0.5)
    eps = float(p.eps[0]) * 5
    C = oracle.expand_cost(p.C)
    f0, g0, _, _ = oracle.sinkhorn_full(a, b, C, eps, 20000, tol=1e-13)          # "directly solving"
    ref = oracle.entropic_objective_full(oracle.plan_full(f0, g0, C, eps), C, eps)
    f, g, t1, t2, gap = oracle.two_stage_sinkhorn_gap(a, b, p.C, eps, 5, 400, ref, 1e-8)
    assert t1 == 5 and 1 < t2 < 400 and gap < 1e-8
    w, z, _, _ = oracle.cyclic_sinkhorn(oracle.fold_average(a, p.n), oracle.fold_average(b, p.n), p.C, eps, 5,
                                        form="kernel")
    _, _, _, hist = oracle.sinkhorn_full(a, b, C, eps, t2, record=True, g0=oracle.expand_vector(z, p.n))
    gaps = [abs(oracle.entropic_objective_full(oracle.plan_full(fh, gh, C, eps), C, eps) - ref)
            for fh, gh, _ in hist]
    assert all(x >= 1e-8 for x in gaps[:-1]) and gaps[-1] < 1e-8
    assert np.array_equal(f, hist[-1][0]) and np.array_equal(g, hist[-1][1])
    # check_every = 3: stops at the first multiple of 3 at or after t2
    _, _, _, t3, _ = oracle.two_stage_sinkhorn_gap(a, b, p.C, eps, 5, 400, ref, 1e-8, check_every=3)
    assert t3 % 3 == 0 and t2 <= t3 < t2 + 3
    _, _, _, tn, _ = oracle.two_stage_sinkhorn_gap(a, b, p.C, eps, 5, 20, ref, 1e-300)
    assert tn == 20
    _, _, _, th, _ = oracle.two_stage_sinkhorn_gap(a, b, p.C, eps, 5, 20, ref, 1e300)
    assert th == 1
