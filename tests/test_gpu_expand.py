"""GPU parity of A6, the dense d x d block-circulant expansion (Lemma 1; Alg. 1 lines 3-6, P:340-343;
Alg. 2 line 10), in every kernel launch_expand selects -- in particular k_expand_bulk, the kernel the C3
and C4 headline steps run (cot_expand_path == 1) -- against the oracle's placement (oracle.expand_plan for
plans the host can hold, oracle.expand_plan_rows on seeded row samples for C4's 17.2 GB plan). Pure placement,
so the bar is bit-exact (fp32 / fp64 bit patterns). Inputs are seeded (synthetic/ and numpy), never GPU output.
"""
import ctypes

import numpy as np
import pytest
import torch

import oracle
import synthetic

pytestmark = pytest.mark.gpu

cot = pytest.importorskip("paper_2311_13147_b200")
DEV = torch.device("cuda:0")
F32, F64 = 0, 1


@pytest.fixture(scope="module", autouse=True)
def _built():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    from paper_2311_13147_b200 import build
    build.build()
    cot.lib()


def _dev(x):
    return torch.as_tensor(np.ascontiguousarray(x), device=DEV)


def _bits(x):
    x = np.ascontiguousarray(x)
    return x.view(np.uint32 if x.dtype == np.float32 else np.uint64)


def _same(a, b):
    assert a.dtype == b.dtype and a.shape == b.shape
    return np.array_equal(_bits(a), _bits(b))


def _blocks(seed, n, m, dt):
    """Seeded plan blocks with signed zeros and exact zeros mixed in (placement must keep bit patterns)."""
    rng = np.random.default_rng(seed)
    T = rng.random((n, m, m)).astype(dt)
    T[rng.random((n, m, m)) < 0.05] = 0.0
    T[rng.random((n, m, m)) < 0.01] = -0.0
    return T


def _sample_rows(seed, n, m, count):
    rng = np.random.default_rng(seed)
    rows = set(rng.choice(n * m, size=count, replace=False).tolist())
    rows |= {0, m - 1, m, n * m - 1, (n - 1) * m}          # first / last row of the first and last block rows
    return sorted(rows)


def test_path_selection():
    L = cot.lib()
    assert L.cot_expand_path(4, 1024, F32) == 1      # C3: k_expand_bulk
    assert L.cot_expand_path(64, 1024, F32) == 1     # C4: k_expand_bulk
    assert L.cot_expand_path(16, 128, F32) == 2      # C5: k_expand_rows
    assert L.cot_expand_path(16, 256, F64) == 1
    assert L.cot_expand_path(4, 130, F32) == 0       # 520 B segments: not 16-byte multiples


def test_bulk_c3_full_blocks_bitexact():
    """C3 (configs[2]) shape n = 4, m = 1024: the whole 64 MiB dense plan of seeded blocks, bit-exact."""
    n, m = 4, 1024
    assert cot.lib().cot_expand_path(n, m, F32) == 1
    T = _blocks(30, n, m, np.float32)
    got = cot.clot_expand(_dev(T), n).cpu().numpy()
    assert _same(got, oracle.expand_plan(T))


def test_bulk_c3_full_clot_lift_bitexact():
    """C-LOT mode through k_expand_bulk at C3 size: argmin of the actual C3 cost (oracle.aggregate, the smallest
    minimiser), a seeded S in the problem dtype; the dense plan equals the oracle's lift + expansion."""
    p = synthetic.c3_image(pair=0)
    _, Ao = oracle.aggregate(p.C)
    S = _blocks(31, 1, p.m, np.float32)[0]
    got = cot.clot_expand(_dev(S), p.n, argmin=_dev(Ao)).cpu().numpy()
    assert _same(got, oracle.expand_plan(oracle.lift(S, Ao, p.n)))
    # the device argmin feeds the same kernel in the pipeline: identical to the oracle's on C3
    _, A = cot.clot_aggregate(_dev(p.C))
    assert np.array_equal(A.cpu().numpy(), Ao)


def test_bulk_fp64_full_bitexact():
    n, m = 16, 256
    assert cot.lib().cot_expand_path(n, m, F64) == 1
    T = _blocks(32, n, m, np.float64)
    got = cot.clot_expand(_dev(T), n).cpu().numpy()
    assert _same(got, oracle.expand_plan(T))
    S = _blocks(33, 1, m, np.float64)[0]
    A = np.random.default_rng(34).integers(0, n, size=(m, m)).astype(np.int32)
    got = cot.clot_expand(_dev(S), n, argmin=_dev(A)).cpu().numpy()
    assert _same(got, oracle.expand_plan(oracle.lift(S, A, n)))


def test_bulk_batched_bitexact():
    """B > 1 through k_expand_bulk (the (b, k, i) unit decomposition and the b * d * d output offset)."""
    B, n, m = 3, 7, 512
    assert cot.lib().cot_expand_path(n, m, F32) == 1
    T = np.stack([_blocks(40 + b, n, m, np.float32) for b in range(B)])
    got = cot.clot_expand(_dev(T), n).cpu().numpy()
    for b in range(B):
        assert _same(got[b], oracle.expand_plan(T[b]))


def _c4_rows_check(out, expected_fn, rows):
    d = out.shape[-1]
    idx = torch.as_tensor(rows, device=DEV, dtype=torch.long)
    got = out.view(d, d).index_select(0, idx).cpu().numpy()
    assert _same(got, expected_fn(rows))


def test_bulk_c4_full_size_sampled_rows():
    """C4 (configs[3]) shape n = 64, m = 1024: the 17.2 GB dense plan (blocks mode and C-LOT mode, one
    buffer), compared on >= 64 seeded rows r*m + i (plus the first and last rows of the outer block rows)
    against oracle.expand_plan_rows -- the host cannot hold the whole plan."""
    n, m = 64, 1024
    d = n * m
    assert cot.lib().cot_expand_path(n, m, F32) == 1
    rows = _sample_rows(50, n, m, 64)
    T = _blocks(51, n, m, np.float32)
    out = torch.empty((d, d), dtype=torch.float32, device=DEV)
    cot.clot_expand(_dev(T), n, out=out)
    _c4_rows_check(out, lambda r: oracle.expand_plan_rows(T, r), rows)
    # C-LOT lift at the same size: argmin of the actual C4 cost
    p = synthetic.c4_large()
    _, Ao = oracle.aggregate(p.C)
    S = _blocks(52, 1, m, np.float32)[0]
    out.fill_(7.0)
    cot.clot_expand(_dev(S), n, argmin=_dev(Ao), out=out)
    lifted = oracle.lift(S, Ao, n)
    _c4_rows_check(out, lambda r: oracle.expand_plan_rows(lifted, r), rows)
    # G / argmin at the C4 shape itself, bit-exact (the aggregation feeding this lift)
    G, A = cot.clot_aggregate(_dev(p.C))
    Go, _ = oracle.aggregate(p.C)
    assert _same(G.cpu().numpy(), Go) and np.array_equal(A.cpu().numpy(), Ao)
    del out
    torch.cuda.empty_cache()


def _expand_shard(src, argmin, n, R, m, out):
    L = cot.lib()
    code = L.clot_expand_shard(src.data_ptr(), argmin.data_ptr() if argmin is not None else None, n, R, m,
                               F32 if src.dtype == torch.float32 else F64, out.data_ptr(),
                               torch.cuda.current_stream().cuda_stream)
    assert code == 0, L.cot_last_error()


@pytest.mark.parametrize("world,rank", [(8, 0), (8, 5), (4, 3)])
def test_bulk_c4_shard_rows(world, rank):
    """clot_expand_shard at the C4 row-shard shapes (R = m / world rows of every block, R < m): shard row
    (r, i) is dense row r*m + row_begin + i; blocks mode and C-LOT mode, sampled rows bit-exact."""
    from paper_2311_13147_b200 import dist
    n, m = 64, 1024
    d = n * m
    b0, R = dist.row_partition(m, world, rank)
    T = _blocks(60 + rank, n, m, np.float32)
    out = torch.empty((n, R, d), dtype=torch.float32, device=DEV)
    _expand_shard(_dev(T[:, b0:b0 + R, :]), None, n, R, m, out)
    rng = np.random.default_rng(61)
    local = sorted(set(rng.choice(n * R, size=64, replace=False).tolist()) | {0, R - 1, n * R - 1})
    dense_rows = [(q // R) * m + b0 + q % R for q in local]
    idx = torch.as_tensor(local, device=DEV, dtype=torch.long)
    got = out.view(n * R, d).index_select(0, idx).cpu().numpy()
    assert _same(got, oracle.expand_plan_rows(T, dense_rows))
    S = _blocks(62, 1, m, np.float32)[0]
    A = np.random.default_rng(63).integers(0, n, size=(m, m)).astype(np.int32)
    out.zero_()
    _expand_shard(_dev(S[b0:b0 + R]), _dev(A[b0:b0 + R]), n, R, m, out)
    got = out.view(n * R, d).index_select(0, idx).cpu().numpy()
    assert _same(got, oracle.expand_plan_rows(oracle.lift(S, A, n), dense_rows))
    del out
    torch.cuda.empty_cache()


def test_bulk_shard_ragged_rows_full():
    """A ragged shard (R = 300 of m = 1024 rows, n = 4, the C3 shape) through k_expand_bulk, the whole output."""
    n, m, b0, R = 4, 1024, 417, 300
    d = n * m
    T = _blocks(70, n, m, np.float32)
    out = torch.empty((n, R, d), dtype=torch.float32, device=DEV)
    _expand_shard(_dev(T[:, b0:b0 + R, :]), None, n, R, m, out)
    dense_rows = [r * m + b0 + i for r in range(n) for i in range(R)]
    assert _same(out.view(n * R, d).cpu().numpy(), oracle.expand_plan_rows(T, dense_rows))
