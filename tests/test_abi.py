"""CPU checks of the drop-in boundary and the host-side logic (no GPU needed)."""

import os
import re

import numpy as np
import pytest

from tests.conftest import ROOT


def _declared_symbols():
    text = open(os.path.join(ROOT, "include", "slm.h")).read()
    return sorted(set(re.findall(r"SLM_API\s+[\w\s\*]*?\b(slm_\w+)\s*\(", text)))


def test_library_loads_and_exports_every_declared_symbol():
    from paper_1702_04645_b200 import _lib
    L = _lib.load()
    declared = _declared_symbols()
    assert len(declared) >= 25
    for name in declared:
        assert hasattr(L, name), name
    # the ctypes signature table covers exactly the header
    assert sorted(_lib.SIGNATURES) == declared


def test_library_is_sm100a():
    import subprocess
    lib = os.path.join(ROOT, "paper_1702_04645_b200", "libslm.so")
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_runconfig_validation():
    from paper_1702_04645_b200 import RunConfig
    RunConfig(threads=2, seed=5, accept_prob=1.0)
    for kw in (dict(threads=0), dict(accept_prob=0.0), dict(accept_prob=1.5),
               dict(max_outer_iters=0), dict(scc_cut_cap=1), dict(resolution=0.0)):
        with pytest.raises(ValueError):
            RunConfig(**kw)


def test_graph_validation_errors_before_device():
    from paper_1702_04645_b200 import Graph
    with pytest.raises(ValueError):
        Graph.from_edges(3, [0, 1], [1], [1.0])
    with pytest.raises(ValueError):
        Graph.from_edges(3, [0], [3], [1.0])
    with pytest.raises(ValueError):
        Graph.from_edges(3, [0], [1], [-1.0])
    with pytest.raises(ValueError):
        Graph.from_edges(3, [0], [1], [np.inf])
    g = Graph.from_edges(0, np.empty(0, np.int64), np.empty(0, np.int64), np.empty(0))
    from paper_1702_04645_b200 import run
    with pytest.raises(ValueError):
        run(g)


def test_label_helpers():
    # canonicalize_labels runs on the device (tests/test_gpu_surface.py); compose is a gather
    from paper_1702_04645_b200 import compose_labels
    np.testing.assert_array_equal(compose_labels([0, 1, 1, 2], [1, 0, 1]), [1, 0, 0, 1])


def test_host_generators_deterministic_and_symmetric():
    import workloads as GN
    n, s, d, w = GN.rmat(10, 8, 1, 4)
    n2, s2, d2, w2 = GN.rmat(10, 8, 1, 4)
    assert np.array_equal(s, s2) and np.array_equal(d, d2) and np.array_equal(w, w2)
    assert n == 1024 and s.size % 2 == 0
    assert (s != d).all()
    h = s.size // 2
    # emitted in (u,v), (v,u) pairs with equal weights
    np.testing.assert_array_equal(s[0::2], d[1::2])
    np.testing.assert_array_equal(w[0::2], w[1::2])
    assert w.min() >= 1 and w.max() <= 100 and (w == np.floor(w)).all()
    assert h > 0
    n, s, d, w = GN.rgg(2048, 8.0, 3)
    key = set(zip(s.tolist(), d.tolist()))
    assert all((b, a) in key for a, b in key)
    assert abs(s.size / n - 8.0) < 1.5
    n, s, d, w = GN.sbm()
    assert n == 1000 and s.size == 14502


def test_dcsbm_shape():
    import workloads as GN
    n, s, d, w = GN.dcsbm(n=5000, k=20, size_lo=50, size_hi=500, seed=1)
    assert n == 5000 and (s != d).all()
    assert 10 < s.size / n < 30
