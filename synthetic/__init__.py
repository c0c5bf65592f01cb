"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle.

This module builds INPUTS only: cost blocks C[k][i][j], reduced marginals alpha/beta and eps.
It holds none of the method's arithmetic (no aggregation, no Sinkhorn, no LP, no expansion),
so it may be imported by both sides (tests, bench) without coupling the oracle to the kernels.

Conventions (PAPER.md = P, SURVEY.md §8(d) = the recipes, BASELINE.json configs C1..C5):
  * Assumption 1: a = (alpha; ...; alpha), b = (beta; ...; beta), d = n*m, and the
    d x d cost is block-circulant: block (r, s) = C_{(s - r) mod n}.
  * Cost blocks are stored [n][m][m] (or [B][n][m][m]), row-major per block, blocks in k order.
  * alpha, beta sum to 1/n each, so the tiled a, b lie in the simplex Delta^d.
  * Every generator is deterministic given its seed (numpy PCG64 `default_rng`).

Point-cloud configs: base points x_0..x_{m-1}; the d points are y_{s*m+j} = R^s x_j with R^n = I.
Then cost((r,i),(s,j)) = ||R^r x_i - R^s x_j||^2 = ||x_i - R^{s-r} x_j||^2, which is exactly the
block-circulant form with C_k[i][j] = ||x_i - R^k x_j||^2.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional

import numpy as np

__all__ = [
    "Problem", "c1_tiny", "c2_ring", "c3_image", "c4_large", "c5_batched", "appd_synthetic",
    "counter_example", "random_cyclic", "approx_symmetric", "CONFIGS", "make",
]


@dataclasses.dataclass
class Problem:
    """One (or a batch of) cyclic problem(s) in reduced form (Assumption 1)."""
    name: str
    C: np.ndarray            # [n][m][m] or [B][n][m][m]; float32 or float64
    alpha: np.ndarray        # [m] or [B][m]; float64, sums to 1/n
    beta: np.ndarray         # [m] or [B][m]; float64, sums to 1/n
    eps: np.ndarray          # [B] float64 (B = 1 for a single problem)
    iters: int               # fixed iteration count (0 = run to tol)
    tol: float               # convergence tolerance on n*sum|c - beta|; 0 = fixed iters
    meta: dict = dataclasses.field(default_factory=dict)

    @property
    def batched(self) -> bool:
        return self.C.ndim == 4

    @property
    def B(self) -> int:
        return self.C.shape[0] if self.batched else 1

    @property
    def n(self) -> int:
        return self.C.shape[-3]

    @property
    def m(self) -> int:
        return self.C.shape[-1]

    @property
    def d(self) -> int:
        return self.n * self.m

    @property
    def dtype(self) -> str:
        return "f64" if self.C.dtype == np.float64 else "f32"

    def single(self, b: int) -> "Problem":
        """Problem b of a batch as a stand-alone problem (same arrays, no copy of method data)."""
        if not self.batched:
            assert b == 0
            return self
        return Problem(f"{self.name}[{b}]", self.C[b], self.alpha[b], self.beta[b],
                       self.eps[b:b + 1].copy(), self.iters, self.tol, dict(self.meta))


# ----------------------------------------------------------------------------------------------
# helpers: points, rotations, marginals (input construction only)
# ----------------------------------------------------------------------------------------------
def _rot2(theta: float) -> np.ndarray:
    c, s = math.cos(theta), math.sin(theta)
    return np.array([[c, -s], [s, c]])


def _rot3_z(theta: float) -> np.ndarray:
    c, s = math.cos(theta), math.sin(theta)
    return np.array([[c, -s, 0.0], [s, c, 0.0], [0.0, 0.0, 1.0]])


def _rot3_axis(axis: np.ndarray, theta: float) -> np.ndarray:
    """Rodrigues rotation about a unit axis."""
    u = axis / np.linalg.norm(axis)
    K = np.array([[0.0, -u[2], u[1]], [u[2], 0.0, -u[0]], [-u[1], u[0], 0.0]])
    return np.eye(3) + math.sin(theta) * K + (1.0 - math.cos(theta)) * (K @ K)


def _sqdist_blocks(x: np.ndarray, R: np.ndarray, n: int) -> np.ndarray:
    """C_k[i][j] = ||x_i - R^k x_j||^2 for k = 0..n-1 (float64). Rotating by R^k is done by
    repeated matrix products so that R^n returns (up to rounding) to the identity."""
    m = x.shape[0]
    C = np.empty((n, m, m), dtype=np.float64)
    y = x.copy()
    xx = (x * x).sum(1)
    for k in range(n):
        if k == 0:
            y = x.copy()
        else:
            y = y @ R.T
        # direct difference form (not the |x|^2 + |y|^2 - 2xy expansion) so C_0 has an exact zero diagonal
        diff = x[:, None, :] - y[None, :, :]
        C[k] = (diff * diff).sum(-1)
    del xx
    return C


def _unit_ball(rng: np.random.Generator, m: int, dim: int = 3) -> np.ndarray:
    g = rng.standard_normal((m, dim))
    g /= np.linalg.norm(g, axis=1, keepdims=True)
    r = rng.random(m) ** (1.0 / dim)
    return g * r[:, None]


def _dirichlet_over_n(rng: np.random.Generator, m: int, n: int, conc: float = 1.0) -> np.ndarray:
    v = rng.dirichlet(np.full(m, conc))
    v = v / v.sum()
    return v / n


def _renorm(v: np.ndarray, n: int) -> np.ndarray:
    return (v / v.sum()) / n


# ----------------------------------------------------------------------------------------------
# BASELINE.json configs
# ----------------------------------------------------------------------------------------------
def c1_tiny(seed: int = 1) -> Problem:
    """C1 (configs[0]): d=64, n=4, m=16, fp64. 16 points uniform in the unit disc (r = sqrt(U),
    theta = 2 pi U), copies rotated by 2 pi k / 4; squared Euclidean cost; alpha, beta = Dir(1)/4;
    eps = 0.05 * mean(C) (mean over the n*m^2 block entries = mean of the full d x d C); tol 1e-9."""
    n, m = 4, 16
    rng = np.random.default_rng(seed)
    r = np.sqrt(rng.random(m))
    th = 2.0 * np.pi * rng.random(m)
    x = np.stack([r * np.cos(th), r * np.sin(th)], axis=1)
    C = _sqdist_blocks(x, _rot2(2.0 * np.pi / n), n)
    alpha = _dirichlet_over_n(rng, m, n)
    beta = _dirichlet_over_n(rng, m, n)
    eps = 0.05 * float(C.mean())
    return Problem("C1_tiny", C, alpha, beta, np.array([eps]), iters=0, tol=1e-9,
                   meta={"points": x, "seed": seed})


def c2_ring(seed: int = 2, eps_factor: float = 1e-2) -> Problem:
    """C2 (configs[1]): d=1024, n=8, m=128, fp32. 128 points ~ N((1,0), 0.2^2 I), 8 copies rotated by
    2 pi k / 8; squared Euclidean cost; alpha, beta = (0.5 * uniform + 0.5 * Dir(0.5)) / 8;
    eps in {1e-1, 1e-2, 1e-3} * mean(C); exactly 500 iterations."""
    n, m = 8, 128
    rng = np.random.default_rng(seed)
    x = np.array([1.0, 0.0]) + 0.2 * rng.standard_normal((m, 2))
    C64 = _sqdist_blocks(x, _rot2(2.0 * np.pi / n), n)
    C = C64.astype(np.float32)
    mix = lambda: 0.5 * np.full(m, 1.0 / m) + 0.5 * rng.dirichlet(np.full(m, 0.5))
    alpha = _renorm(mix(), n)
    beta = _renorm(mix(), n)
    eps = eps_factor * float(C.astype(np.float64).mean())
    return Problem(f"C2_ring_eps{eps_factor:g}", C, alpha, beta, np.array([eps]), iters=500, tol=0.0,
                   meta={"seed": seed, "eps_factor": eps_factor})


def rotation_quadrant_order(H: int) -> np.ndarray:
    """Pixel ordering for 90-degree rotational symmetry (n = 4):
    block 0 = top-left quadrant in row-major order; block k = rho^k(block 0) with
    rho(r, c) = (c, H - 1 - r). Returns [4][m][2] integer pixel coordinates, m = (H/2)^2."""
    h = H // 2
    base = np.array([(r, c) for r in range(h) for c in range(h)], dtype=np.int64)
    out = [base]
    cur = base
    for _ in range(3):
        cur = np.stack([cur[:, 1], H - 1 - cur[:, 0]], axis=1)
        out.append(cur)
    return np.stack(out, 0)


def _rotation_symmetric_histogram(rng: np.random.Generator, H: int, n_gauss: int = 5) -> np.ndarray:
    """Sum of n_gauss anisotropic Gaussians (centres uniform on the grid, sigma_x, sigma_y ~ U[2,8] px,
    orientation ~ U[0, pi)), summed with its 3 rotations, normalised, then mixed 0.999 : 0.001 with the
    uniform histogram so that every pixel has positive mass (SURVEY Q10 rejects zero marginals)."""
    rr, cc = np.meshgrid(np.arange(H, dtype=np.float64), np.arange(H, dtype=np.float64), indexing="ij")
    img = np.zeros((H, H))
    for _ in range(n_gauss):
        cy, cx = rng.random(2) * (H - 1)
        sx, sy = 2.0 + 6.0 * rng.random(2)
        th = np.pi * rng.random()
        c, s = math.cos(th), math.sin(th)
        dy, dx = rr - cy, cc - cx
        u = c * dx + s * dy
        v = -s * dx + c * dy
        img += np.exp(-0.5 * ((u / sx) ** 2 + (v / sy) ** 2))
    sym = img.copy()
    cur = img
    for _ in range(3):
        # rho(r, c) = (c, H-1-r): value at rho(p) of the rotated image equals value at p
        cur = np.rot90(cur, k=1)
        sym += cur
    sym /= sym.sum()
    sym = 0.999 * sym + 0.001 / (H * H)
    return sym


def c3_image(seed: int = 3, H: int = 64, pair: int = 0) -> Problem:
    """C3 (configs[2]): 64x64 grid with 4-fold rotational symmetry, n=4, m=1024, d=4096, fp32.
    Cost = squared pixel distance normalised to [0,1] by the max 2*(H-1)^2; histograms = 5 random
    anisotropic Gaussians + their 3 rotations, normalised. eps = 1e-2. Stands in for Table 2's 64x64
    NYU workload, whose dataset is not available; rotation (n=4) instead of mirror (n=2)."""
    n = 4
    order = rotation_quadrant_order(H)                       # [4][m][2]
    m = order.shape[1]
    rng = np.random.default_rng(seed * 1000 + pair)
    A = _rotation_symmetric_histogram(rng, H)
    Bimg = _rotation_symmetric_histogram(rng, H)
    alpha = np.array([A[r, c] for r, c in order[0]])
    beta = np.array([Bimg[r, c] for r, c in order[0]])
    alpha = _renorm(alpha, n)
    beta = _renorm(beta, n)
    p0 = order[0].astype(np.float64)
    C64 = np.empty((n, m, m))
    for k in range(n):
        pk = order[k].astype(np.float64)
        diff = p0[:, None, :] - pk[None, :, :]
        C64[k] = (diff * diff).sum(-1) / (2.0 * (H - 1) ** 2)
    C = C64.astype(np.float32)
    return Problem(f"C3_image_pair{pair}", C, alpha, beta, np.array([1e-2]), iters=500, tol=0.0,
                   meta={"seed": seed, "pair": pair, "H": H})


def approx_symmetric(p: Problem, noise: float = 0.05, seed: int = 7):
    """NEXT-2 inputs (Alg. 3): full-length marginals a, b in Delta^d that are only
    APPROXIMATELY periodic -- the tiled alpha, beta of `p` times (1 + noise * U(-1, 1)) per entry,
    renormalised to sum 1 (images with "slight noise and displacement"). The cost blocks of `p` stay
    strictly block-circulant. Stands in for Table 2's NYU mirror images (not available). Returns (a, b)."""
    rng = np.random.default_rng(seed)
    out = []
    for v in (p.alpha, p.beta):
        t = np.tile(np.asarray(v, dtype=np.float64), p.n)
        t = t * (1.0 + noise * rng.uniform(-1.0, 1.0, size=t.shape))
        out.append(t / t.sum())
    return out[0], out[1]


def c4_large(seed: int = 4, m: int = 1024, n: int = 64) -> Problem:
    """C4 (configs[3]): d=65536, n=64, m=1024, fp32 (256 MiB of cost blocks). 1024 points uniform in
    the 3-D unit ball; 64 rotations about the z axis by 2 pi k / 64; squared Euclidean cost;
    alpha, beta = Dir(1)/64; eps = 5e-3; fixed 500 iterations. m, n can be shrunk for parity runs."""
    rng = np.random.default_rng(seed)
    x = _unit_ball(rng, m)
    C = _sqdist_blocks(x, _rot3_z(2.0 * np.pi / n), n).astype(np.float32)
    alpha = _dirichlet_over_n(rng, m, n)
    beta = _dirichlet_over_n(rng, m, n)
    return Problem(f"C4_large_n{n}_m{m}", C, alpha, beta, np.array([5e-3]), iters=500, tol=0.0,
                   meta={"seed": seed})


def c5_problem(b: int, base_seed: int = 5000, n: int = 16, m: int = 128):
    """Problem b of C5: seed = base + b; 128 points uniform in the unit ball; rotation axis uniform on
    S^2; R = rotation by 2 pi / 16 about it; C_k = ||x_i - R^k x_j||^2 (fp32); alpha, beta = Dir(1)/16;
    eps = 1e-2 * mean(C_b)."""
    rng = np.random.default_rng(base_seed + b)
    x = _unit_ball(rng, m)
    axis = rng.standard_normal(3)
    axis /= np.linalg.norm(axis)
    C = _sqdist_blocks(x, _rot3_axis(axis, 2.0 * np.pi / n), n).astype(np.float32)
    alpha = _dirichlet_over_n(rng, m, n)
    beta = _dirichlet_over_n(rng, m, n)
    eps = 1e-2 * float(C.astype(np.float64).mean())
    return C, alpha, beta, eps


def c5_batched(B: int = 4096, base_seed: int = 5000, first: int = 0) -> Problem:
    """C5 (configs[4]): B independent problems, d=2048, n=16, m=128, fp32; 200 iterations each.
    `first` selects a contiguous window [first, first+B) of the 4096 seeds (for sampled parity)."""
    n, m = 16, 128
    C = np.empty((B, n, m, m), dtype=np.float32)
    alpha = np.empty((B, m))
    beta = np.empty((B, m))
    eps = np.empty(B)
    for t in range(B):
        C[t], alpha[t], beta[t], eps[t] = c5_problem(first + t, base_seed, n, m)
    return Problem(f"C5_batched_B{B}", C, alpha, beta, eps, iters=200, tol=0.0,
                   meta={"base_seed": base_seed, "first": first})


# ----------------------------------------------------------------------------------------------
# the paper's own synthetic workload (App. D) and the App. A counter-example
# ----------------------------------------------------------------------------------------------
def appd_synthetic(seed: int, d: int = 5000, n_max: int = 50, dtype=np.float64) -> Problem:
    """App. D: alpha, beta ~ U[0,1)^m, tiled and normalised to sum 1; blocks
    C_0..C_{n-1} ~ N(3, 5^2)^{m x m}, shifted by |global minimum| so that all costs are >= 0.
    Generated at order n_max (m = d / n_max); lambda = 0.5. The RNG sampling order is not
    specified by the paper: we draw alpha, beta, then the blocks."""
    m = d // n_max
    rng = np.random.default_rng(seed)
    alpha = rng.random(m)
    beta = rng.random(m)
    blocks = rng.normal(3.0, 5.0, size=(n_max, m, m))
    blocks = blocks + abs(blocks.min())
    return Problem(f"AppD_d{d}_seed{seed}", blocks.astype(dtype), _renorm(alpha, n_max),
                   _renorm(beta, n_max), np.array([0.5]), iters=0, tol=1e-9,
                   meta={"seed": seed, "n_max": n_max})


def counter_example(metric: str = "euclidean") -> Problem:
    """App. A: 4x4 grid, 90-degree rotational symmetry (n = 4), quadrant
    ordering. Left image: mass 0.25 at pixel (0,1) and its 3 rotations; right image: 0.25 at (0,2)
    and its rotations. Pixel-wise Euclidean (or squared) cost."""
    H, n = 4, 4
    order = rotation_quadrant_order(H)                       # [4][4][2]
    m = order.shape[1]
    base = [tuple(p) for p in order[0]]
    alpha = np.zeros(m)
    beta = np.zeros(m)
    # (0,1) is in the top-left quadrant; (0,2) is not, but its rotation rho^3(0,2) = (1,0) is
    # (rho(r,c) = (c, H-1-r): rho(1,0) = (0,2)), so the right image's block-0 pixel is (1,0).
    alpha[base.index((0, 1))] = 0.25
    beta[base.index((1, 0))] = 0.25
    p0 = order[0].astype(np.float64)
    C = np.empty((n, m, m))
    for k in range(n):
        diff = p0[:, None, :] - order[k].astype(np.float64)[None, :, :]
        sq = (diff * diff).sum(-1)
        C[k] = np.sqrt(sq) if metric == "euclidean" else sq
    return Problem(f"counter_example_{metric}", C, alpha, beta, np.array([1.0]), iters=0, tol=0.0,
                   meta={"order": order})


def random_cyclic(seed: int, n: int, m: int, dtype=np.float64, integer: bool = False,
                  eps: float = 0.1, B: Optional[int] = None) -> Problem:
    """Small random strictly-symmetric instance for brute-force tests (SPEC acceptance 1):
    uniform costs in [0,1) (or small integers to create ties), Dirichlet(1) marginals / n."""
    rng = np.random.default_rng(seed)
    shape = (n, m, m) if B is None else (B, n, m, m)
    if integer:
        C = rng.integers(0, 4, size=shape).astype(np.float64)
    else:
        C = rng.random(shape)
    if B is None:
        alpha = _dirichlet_over_n(rng, m, n)
        beta = _dirichlet_over_n(rng, m, n)
        e = np.array([eps])
    else:
        alpha = np.stack([_dirichlet_over_n(rng, m, n) for _ in range(B)])
        beta = np.stack([_dirichlet_over_n(rng, m, n) for _ in range(B)])
        e = np.full(B, eps)
    return Problem(f"random_n{n}_m{m}_s{seed}", C.astype(dtype), alpha, beta, e, iters=0, tol=0.0,
                   meta={"seed": seed})


def c2_sweep(seed: int = 2) -> Problem:
    """C2 as configs[1] states it: the ring problem at eps in {1e-1, 1e-2, 1e-3} * mean(C), 500 iterations
    each -- three independent problems (same C, alpha, beta), one batch of B = 3."""
    ps = [c2_ring(seed=seed, eps_factor=f) for f in (1e-1, 1e-2, 1e-3)]
    return Problem("C2_ring_eps_sweep", np.stack([q.C for q in ps]), np.stack([q.alpha for q in ps]),
                   np.stack([q.beta for q in ps]), np.concatenate([q.eps for q in ps]), iters=ps[0].iters, tol=0.0,
                   meta={"eps_factors": [1e-1, 1e-2, 1e-3]})


CONFIGS = {
    "C1": c1_tiny,
    "C2": c2_ring,
    "C3": c3_image,
    "C4": c4_large,
    "C5": c5_batched,
}


def make(name: str, **kw) -> Problem:
    return CONFIGS[name](**kw)
