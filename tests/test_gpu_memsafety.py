"""Memory-safety checks of every kernel, standing in for compute-sanitizer (closed on this GPU pool: "runs under it
have left GPUs needing a reset"). Each case runs every input, output and workspace buffer inside a larger
allocation with 64 KiB guard bands, twice: once with the guards and the workspace filled with 0x00 bytes, once with
0xFF bytes (NaN for fp32/fp64). Checked:
  * out-of-bounds WRITES: the guard bands are unchanged after the run (memcheck's write side);
  * out-of-bounds READS that reach a result, and reads of uninitialised workspace: the outputs of the two runs are
    bitwise identical (a NaN read would propagate) and finite (memcheck's read side, initcheck);
  * races that change results: the two runs, and a third with the same fill, agree bit for bit (the kernels'
    sums have fixed orders, so any difference is a race or an uninitialised read).
Results against the oracle are the other test files' job."""
import ctypes

import numpy as np
import pytest
import torch

import synthetic

pytestmark = pytest.mark.gpu

cot = pytest.importorskip("paper_2311_13147_b200")
from paper_2311_13147_b200 import dist as cdist  # noqa: E402

DEV = torch.device("cuda:0")
GUARD = 65536
F32, F64 = 0, 1


@pytest.fixture(scope="module", autouse=True)
def _built():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    from paper_2311_13147_b200 import build
    build.build()
    cot.lib()


class Arena:
    """Guarded device buffers for one run; every guard band and uninitialised byte is `fill`."""

    def __init__(self, fill):
        self.fill = fill
        self.bufs = []

    def _alloc(self, numel, dtype):
        esz = torch.tensor([], dtype=dtype).element_size()
        g = GUARD // esz
        raw = torch.empty(numel + 2 * g, dtype=dtype, device=DEV)
        raw.view(torch.uint8).fill_(self.fill)
        self.bufs.append((raw, g, numel, esz))
        return raw[g:g + numel]

    def out(self, shape, dtype):
        n = int(np.prod(shape)) if len(shape) else 1
        return self._alloc(n, dtype).view(*shape)

    def inp(self, x):
        x = np.ascontiguousarray(x)
        t = torch.as_tensor(x)
        v = self._alloc(t.numel(), t.dtype).view(*t.shape)
        v.copy_(t.to(DEV))
        return v

    def workspace(self, nbytes):
        return self._alloc(int(nbytes), torch.uint8)

    def check_guards(self):
        torch.cuda.synchronize()
        for raw, g, numel, esz in self.bufs:
            b = raw.view(torch.uint8)
            head, tail = b[:g * esz], b[(g + numel) * esz:]
            assert bool((head == self.fill).all()) and bool((tail == self.fill).all()), "guard band overwritten"


P = lambda t: None if t is None else t.data_ptr()  # noqa: E731
S = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731


def _ck(code, fn):
    assert code in (0, 1), f"{fn}: {code} {cot.lib().cot_last_error().decode()}"


def run_aggregate(A, C):
    L = cot.lib()
    Cd = A.inp(C)
    B, n, m = (1, C.shape[0], C.shape[1]) if C.ndim == 3 else C.shape[:3]
    dt = torch.float32 if C.dtype == np.float32 else torch.float64
    G, Am = A.out((B, m, m), dt), A.out((B, m, m), torch.int32)
    nf = A.out((1,), torch.int32)
    _ck(L.clot_aggregate(P(Cd), B, n, m, F32 if dt == torch.float32 else F64, P(G), P(Am), P(nf), S()), "agg")
    return [G, Am]


def run_expand(A, n, m, B, dt, argmin, seed):
    rng = np.random.default_rng(seed)
    L = cot.lib()
    npdt = np.float32 if dt == F32 else np.float64
    tdt = torch.float32 if dt == F32 else torch.float64
    if argmin:
        Sd = A.inp(rng.random((B, m, m)).astype(npdt))
        Ad = A.inp(rng.integers(0, n, size=(B, m, m)).astype(np.int32))
    else:
        Sd = A.inp(rng.random((B, n, m, m)).astype(npdt))
        Ad = None
    d = n * m
    T = A.out((B, d, d), tdt)
    _ck(L.clot_expand(P(Sd), P(Ad), B, n, m, dt, P(T), S()), "expand")
    return [T]


def run_cerot(A, p, iters, flags=0, pre=False):
    """aggregate -> init -> iterations -> plan with T blocks and the device report, all buffers guarded."""
    L = cot.lib()
    dt = F32 if p.C.dtype == np.float32 else F64
    tdt = torch.float32 if dt == F32 else torch.float64
    B, n, m = p.B, p.n, p.m
    Cd, ad, bd, ed = A.inp(p.C), A.inp(p.alpha), A.inp(p.beta), A.inp(np.asarray(p.eps, np.float64))
    G, Am, nf = A.out((B, m, m), tdt), A.out((B, m, m), torch.int32), A.out((1,), torch.int32)
    _ck(L.clot_aggregate(P(Cd), B, n, m, dt, P(G), P(Am), P(nf), S()), "agg")
    w, z = A.out((B, m), torch.float64), A.out((B, m), torch.float64)
    ws = A.workspace(L.cot_workspace_bytes(B, n, m, dt))
    _ck(L.cerot_init(P(ad), P(bd), B, m, 1, P(z), P(ws), ws.numel(), S()), "init")
    src, nn = Cd, n
    if pre:
        Sd = A.out((B, 1, m, m), tdt)
        _ck(L.cerot_precompute(P(Cd), P(G), B, n, m, dt, P(ed), P(Sd), S()), "precompute")
        src, nn, flags = Sd, 1, flags | cot.COT_PRECOMPUTED
    _ck(L.cerot_iter(P(ad), P(bd), P(src), P(G), B, nn, m, dt, P(ed), iters, 0.0, 1, flags, P(w), P(z), P(ws),
                     ws.numel(), S()), "iter")
    T, rep = A.out((B, n, m, m), tdt), A.out((B, 8), torch.float64)
    _ck(L.cerot_plan(P(ad), P(bd), P(Cd), P(G), B, n, m, dt, P(ed), P(w), P(z), P(T), P(rep), P(ws), ws.numel(),
                     S()), "plan")
    return [w, z, T, rep]


def run_fused(A, world):
    L = cot.lib()
    p = synthetic.c4_large(m=256, n=8)
    V, m, n = world, p.m, p.n
    ad, bd, ed = A.inp(p.alpha), A.inp(p.beta), A.inp(np.asarray(p.eps, np.float64))
    Cs, Gs, ws_, w_, z_, rb, Rs = [], [], [], [], [], [], []
    for r in range(V):
        b0, R = cdist.row_partition(m, V, r)
        Cl = A.inp(p.C[:, b0:b0 + R, :])
        Gl, Al, nf = A.out((R, m), torch.float32), A.out((R, m), torch.int32), A.out((1,), torch.int32)
        _ck(L.clot_aggregate_shard(P(Cl), n, R, m, F32, P(Gl), P(Al), P(nf), S()), "agg_shard")
        ws = A.workspace(L.cot_workspace_bytes_sharded(n, m, R, F32))
        w, z = A.out((m,), torch.float64), A.out((m,), torch.float64)
        _ck(L.cerot_init(P(ad), P(bd), 1, m, 1, P(z), P(ws), ws.numel(), S()), "init")
        Cs.append(Cl), Gs.append(Gl), ws_.append(ws), w_.append(w), z_.append(z), rb.append(b0), Rs.append(R)
    xb = []
    for _ in range(V):
        b = ctypes.c_void_p()
        _ck(L.cot_xchg_alloc(m, V, ctypes.byref(b), None), "xchg_alloc")
        xb.append(b.value)
    arr = lambda xs: (ctypes.c_void_p * V)(*xs)  # noqa: E731
    _ck(L.cerot_iter_fused_emulated(V, P(ad), P(bd), arr([P(c) for c in Cs]), arr([P(g) for g in Gs]), n, m,
                                    (ctypes.c_int64 * V)(*rb), (ctypes.c_int64 * V)(*Rs), F32, P(ed), 4, 0.0, 1, 0,
                                    arr([P(w) for w in w_]), arr([P(z) for z in z_]), arr([P(s) for s in ws_]),
                                    (ctypes.c_size_t * V)(*[s.numel() for s in ws_]), arr(xb), S()), "fused_emu")
    torch.cuda.synchronize()
    for b in xb:
        L.cot_xchg_free(b)
    return [w[rb[i]:rb[i] + Rs[i]] for i, w in enumerate(w_)] + z_


def run_two_stage(A):
    L = cot.lib()
    p = synthetic.random_cyclic(seed=6, n=4, m=32, dtype=np.float32, eps=0.1)
    a, b = synthetic.approx_symmetric(p)
    n, m = p.n, p.m
    ad, bd, Cd, ed = A.inp(a), A.inp(b), A.inp(p.C), A.inp(np.array([0.1]))
    f, g = A.out((n * m,), torch.float64), A.out((n * m,), torch.float64)
    w, z = A.out((m,), torch.float64), A.out((m,), torch.float64)
    ws = A.workspace(L.cot_two_stage_workspace_bytes(n, m, F32))
    rep = cot.cot_report()
    its = (ctypes.c_int64 * 2)()
    _ck(L.cerot_two_stage(P(ad), P(bd), P(Cd), n, m, F32, P(ed), 5, 0.0, 5, 0.0, 1, P(f), P(g), P(w), P(z), P(ws),
                          ws.numel(), ctypes.byref(rep), its, S()), "two_stage")
    return [f, g, w, z]


def run_two_stage_gap(A):
    """App. F's stage-2 rule (cerot_two_stage_gap): the report passes run inside the loop, every 2nd iteration;
    the reference value is never reached (obj_ref = 1e3), so all 6 iterations and 3 checks run."""
    L = cot.lib()
    p = synthetic.random_cyclic(seed=6, n=4, m=32, dtype=np.float32, eps=0.1)
    a, b = synthetic.approx_symmetric(p)
    n, m = p.n, p.m
    ad, bd, Cd, ed = A.inp(a), A.inp(b), A.inp(p.C), A.inp(np.array([0.1]))
    f, g = A.out((n * m,), torch.float64), A.out((n * m,), torch.float64)
    w, z = A.out((m,), torch.float64), A.out((m,), torch.float64)
    ws = A.workspace(L.cot_two_stage_workspace_bytes(n, m, F32))
    rep = cot.cot_report()
    its = (ctypes.c_int64 * 2)()
    code = L.cerot_two_stage_gap(P(ad), P(bd), P(Cd), n, m, F32, P(ed), 5, 0.0, 6, 1e3, 1e-4, 2, P(f), P(g), P(w),
                                 P(z), P(ws), ws.numel(), ctypes.byref(rep), its, S())
    assert code == 1 and its[1] == 6, (code, its[1])        # COT_NOT_CONVERGED
    return [f, g, w, z]


def run_srot(A):
    L = cot.lib()
    p = synthetic.random_cyclic(seed=7, n=4, m=32, dtype=np.float32, eps=0.1)
    n, m = p.n, p.m
    Cd, ad, bd = A.inp(p.C), A.inp(p.alpha), A.inp(p.beta)
    gam = A.inp(np.array([0.5]))
    w, z = A.out((1, m), torch.float64), A.out((1, m), torch.float64)
    T = A.out((1, n, m, m), torch.float32)
    ws = A.workspace(L.cot_workspace_bytes(1, n, m, F32))
    rep = (cot.cot_report * 1)()
    _ck(L.csrot_solve(P(ad), P(bd), P(Cd), 1, n, m, F32, cot.COT_REG_SQUARED, P(gam), 0.0, 4, 1, cot.COT_COLD_START,
                      P(w), P(z), P(T), P(ws), ws.numel(), rep, S()), "csrot")
    return [w, z, T]


def _env(kv, fn):
    import os
    old = {k: os.environ.get(k) for k in kv}
    os.environ.update(kv)
    try:
        return fn()
    finally:
        for k, v in old.items():
            if v is None:
                del os.environ[k]
            else:
                os.environ[k] = v


CASES = {
    "aggregate_f32": lambda A: run_aggregate(A, synthetic.c2_ring().C),
    "aggregate_f64": lambda A: run_aggregate(A, synthetic.c1_tiny().C),
    "expand_rows": lambda A: run_expand(A, 16, 128, 2, F32, False, 1) + run_expand(A, 16, 128, 2, F32, True, 2),
    "expand_bulk": lambda A: run_expand(A, 7, 512, 1, F32, False, 3) + run_expand(A, 7, 512, 1, F32, True, 4),
    "expand_generic": lambda A: run_expand(A, 3, 37, 2, F32, False, 5) + run_expand(A, 3, 37, 1, F64, True, 6),
    "chain_c2_sweep": lambda A: run_cerot(A, synthetic.c2_sweep(), 6),
    "chain_c5_batch": lambda A: run_cerot(A, synthetic.c5_batched(B=24), 4),
    "chain_ragged": lambda A: run_cerot(A, synthetic.random_cyclic(seed=8, n=5, m=36, dtype=np.float32, eps=0.05,
                                                                   B=3), 6),
    "cluster_interleaved": lambda A: run_cerot(A, synthetic.random_cyclic(seed=4, n=3, m=192, dtype=np.float32,
                                                                          eps=0.05, B=2), 5),
    "tma_forced_small": lambda A: run_cerot(A, synthetic.random_cyclic(seed=5, n=9, m=256, dtype=np.float32,
                                                                       eps=0.05), 5, flags=cot.COT_FORCE_TMA),
    "res_c3": lambda A: run_cerot(A, synthetic.c3_image(), 4),
    "res_h2_ragged": lambda A: _env({"COT_RES_H": "2"}, lambda: run_cerot(A, synthetic.c4_large(m=768, n=8), 4)),
    "res_h4": lambda A: _env({"COT_RES_H": "4"}, lambda: run_cerot(A, synthetic.c4_large(m=512, n=12), 4)),
    "res_smem_only": lambda A: run_cerot(A, synthetic.random_cyclic(seed=9, n=6, m=256, dtype=np.float32,
                                                                    eps=0.05), 5),
    "tma_c3": lambda A: run_cerot(A, synthetic.c3_image(), 4, flags=cot.COT_FORCE_TMA),
    "tma_deterministic": lambda A: run_cerot(A, synthetic.c4_large(m=256, n=8), 4, flags=cot.COT_DETERMINISTIC),
    "ldg_fp64": lambda A: run_cerot(A, synthetic.c1_tiny(), 6),
    "ldg_forced_f32": lambda A: run_cerot(A, synthetic.c2_ring(), 4, flags=cot.COT_FORCE_LDG),
    "precomputed": lambda A: run_cerot(A, synthetic.c2_ring(), 4, pre=True),
    "fused_emulated_2": lambda A: run_fused(A, 2),
    "fused_emulated_2_tma": lambda A: _env({"COT_RES": "0"}, lambda: run_fused(A, 2)),
    "two_stage": run_two_stage,
    "two_stage_gap": run_two_stage_gap,
    "srot": run_srot,
}


@pytest.mark.parametrize("name", list(CASES))
def test_guards_and_poisoned_memory(name):
    outs = []
    for fill in (0x00, 0xFF, 0xFF):
        A = Arena(fill)
        res = CASES[name](A)
        A.check_guards()
        outs.append([r.detach().cpu().numpy().copy() for r in res])
        del A
    for a, b in zip(outs[0], outs[1]):
        assert np.array_equal(a.view(np.uint8), b.view(np.uint8)), f"{name}: result depends on memory it should not read"
    for a, b in zip(outs[1], outs[2]):
        assert np.array_equal(a.view(np.uint8), b.view(np.uint8)), f"{name}: run-to-run difference"
    for a in outs[0]:
        if a.dtype.kind == "f":
            assert np.isfinite(a).all(), name
