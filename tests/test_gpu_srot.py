"""GPU parity of NEXT-3 (C-SROT, squared regulariser) against the oracle's alternating maximisation."""
import numpy as np
import pytest
import torch

import oracle
import synthetic

pytestmark = pytest.mark.gpu
cot = pytest.importorskip("paper_2311_13147_b200")
DEV = torch.device("cuda:0")


def _dev(x):
    return torch.as_tensor(np.ascontiguousarray(x), device=DEV)


@pytest.mark.parametrize("maker,gam,sweeps", [
    (lambda: synthetic.random_cyclic(seed=11, n=4, m=7), 0.5, 12),
    (lambda: synthetic.random_cyclic(seed=12, n=6, m=33, dtype=np.float32), 0.3, 20),
    (lambda: synthetic.c2_ring(eps_factor=1e-2), 1.0, 15),
])
def test_srot_fixed_sweeps(maker, gam, sweeps):
    p = maker()
    reg = ("squared", gam)
    w, z, _, _ = oracle.alternating_maximize(p.alpha, p.beta, p.C, reg, sweeps)
    wg, zg, T, reps = cot.csrot_solve(_dev(p.C), _dev(p.alpha), _dev(p.beta), gam, max_sweeps=sweeps, T_blocks=True)
    wg, zg = wg.cpu().numpy(), zg.cpu().numpy()
    assert np.abs(wg - w).max() < 1e-9 * max(1.0, np.abs(w).max())
    assert np.abs(zg - z).max() < 1e-9 * max(1.0, np.abs(z).max())
    ro = oracle.srot_report(w, z, p.alpha, p.beta, p.C, reg)
    g = reps[0]
    for key in ("objective", "reg_primal", "dual"):
        assert abs(g[key] - ro[key]) <= 1e-8 * abs(ro[key]) + 1e-14, (key, g[key], ro[key])
    for key in ("row_l1", "col_l1", "mass"):
        assert abs(g[key] - ro[key]) <= 1e-9, (key, g[key], ro[key])
    To = oracle.srot_plan(w, z, p.C, reg)
    assert np.abs(T.cpu().numpy().astype(np.float64) - To).max() <= 1e-6 * To.max()


def test_srot_converges_with_duality():
    p = synthetic.random_cyclic(seed=13, n=3, m=16, B=3)
    wg, zg, T, reps = cot.csrot_solve(_dev(p.C), _dev(p.alpha), _dev(p.beta), 0.4, tol=1e-12, max_sweeps=5000,
                                      check_every=4)
    for b in range(3):
        q = p.single(b)
        w, z, t, _ = oracle.alternating_maximize(q.alpha, q.beta, q.C, ("squared", 0.4), 5000, tol=1e-12,
                                                 check_every=4)
        assert reps[b]["converged"] and reps[b]["iters"] == t
        assert abs(reps[b]["reg_primal"] - reps[b]["dual"]) < 1e-9
