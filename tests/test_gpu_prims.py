"""The library's own device primitives (slm_prim.cu): stable onesweep LSD radix sort and
decoupled look-back scans, against numpy.  These carry the CSR build and the aggregation
(graph.py:97-116 stable lexsort + reduceat offsets, 266-280), so stability and exactness
are tested directly, at sizes spanning one tile to many."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_1702_04645_b200 import _lib
    return _lib.Context(0)


SIZES = [0, 1, 2, 31, 511, 8191, 8192, 8193, 100_003, 1 << 20, (1 << 22) + 17]


@pytest.mark.parametrize("n", SIZES)
def test_sort_u64_f64_stable(ctx, n):
    rng = np.random.default_rng(n)
    for end_bit in (64, 48, 20, 9, 1):
        hi = (1 << min(end_bit + 3, 63))
        keys = rng.integers(0, hi, n, dtype=np.uint64)
        if n > 10:
            keys[rng.integers(0, n, n // 3)] = keys[0]   # heavy duplicates
        vals = np.arange(n, dtype=np.float64) + 0.5
        k2, v2, _ = ctx.debug_sort(keys, vals, end_bit)
        mask = np.uint64((1 << end_bit) - 1) if end_bit < 64 else np.uint64(~0 & ((1 << 64) - 1))
        order = np.argsort(keys & mask, kind="stable")
        np.testing.assert_array_equal(k2, keys[order])
        np.testing.assert_array_equal(v2, vals[order])


@pytest.mark.parametrize("n", SIZES)
def test_sort_u32_i32_stable(ctx, n):
    rng = np.random.default_rng(n + 1)
    for end_bit in (32, 25, 8, 3):
        keys = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
        vals = np.arange(n, dtype=np.int32)
        k2, v2, _ = ctx.debug_sort(keys, vals, end_bit)
        order = np.argsort(keys & np.uint32((1 << end_bit) - 1 if end_bit < 32 else 0xFFFFFFFF),
                           kind="stable")
        np.testing.assert_array_equal(k2, keys[order])
        np.testing.assert_array_equal(v2, vals[order])


@pytest.mark.parametrize("n", SIZES)
def test_scans(ctx, n):
    rng = np.random.default_rng(n + 2)
    x64 = rng.integers(-1000, 1000, n).astype(np.int64)
    ex = np.concatenate([[0], np.cumsum(x64)[:-1]]) if n else x64
    np.testing.assert_array_equal(ctx.debug_scan(x64), ex)
    x32 = x64.astype(np.int32)
    np.testing.assert_array_equal(ctx.debug_scan(x32), ex.astype(np.int32))
    np.testing.assert_array_equal(ctx.debug_scan(x32, out_dtype=np.int64), ex)
    xf = x64.astype(np.float64)   # integer-valued: every order is exact
    np.testing.assert_array_equal(ctx.debug_scan(xf), ex.astype(np.float64))
    keys = np.sort(rng.integers(0, max(1, n // 5), n)).astype(np.uint32)
    keys[::7] = np.maximum.accumulate(keys[::7]) if n else keys[::7]
    exp = np.zeros(n, np.int32)
    run = 0
    for i in range(n) if n <= 200_000 else []:
        if i == 0 or keys[i] != keys[i - 1]:
            run = 0
        exp[i] = run
        run += int(x32[i])
    if n <= 200_000:
        np.testing.assert_array_equal(ctx.debug_scan(x32, keys=keys), exp)


def test_sort_speed_vs_torch_cub(ctx):
    """Informational bar: our onesweep vs torch.sort (CUB radix sort) on 2^26 48-bit keys."""
    import torch
    n = 1 << 26
    rng = np.random.default_rng(3)
    keys = rng.integers(0, 1 << 48, n, dtype=np.uint64)
    vals = rng.random(n)
    ctx.debug_sort(keys[:1 << 20], vals[:1 << 20], 48)
    _, _, ms = ctx.debug_sort(keys, vals, 48)
    kt = torch.from_numpy(keys.view(np.int64)).cuda()
    torch.sort(kt, stable=True)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    _, idx = torch.sort(kt, stable=True)
    vt = torch.from_numpy(vals).cuda()
    vt[idx]
    b.record()
    b.synchronize()
    ms_t = a.elapsed_time(b)
    print(f"\nonesweep pairs 2^26 x 48 bit: {ms:.2f} ms; torch.sort + gather: {ms_t:.2f} ms")
    assert ms < 3 * ms_t + 5
