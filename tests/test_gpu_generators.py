"""Device generators (slm_gen.cu) against their host twins (workloads/gen_host.c): the
same edge multiset, so the level-0 CSRs agree bit for bit -- R-MAT, RGG, and the pair-model
SBM / DC-SBM (one counter-hash Bernoulli draw per node pair)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _same_csr(ctx_a, ctx_b):
    for x, y in zip(ctx_a.csr(), ctx_b.csr()):
        np.testing.assert_array_equal(x, y)


def test_pair_models_match_host():
    import workloads as W
    from paper_1702_04645_b200 import _lib
    cases = [(0, dict(n=1000, blocks=10, p_in=0.10, p_out=0.005, seed=0), None),
             (0, dict(n=3001, blocks=7, p_in=0.05, p_out=0.001, seed=5), None),
             (1, dict(n=6000, k=20, seed=1), W.dcsbm_params(n=6000, k=20, size_lo=100,
                                                          size_hi=1000, seed=1))]
    for mode, kw, params in cases:
        ctx_d = _lib.Context(0)
        if mode == 0:
            ctx_d.build_pairs(0, kw["n"], kw["blocks"], kw["p_in"], kw["p_out"], seed=kw["seed"])
            n, s, d, w = W.sbm_hash(**kw)
        else:
            ctx_d.build_pairs(1, kw["n"], params=params, seed=kw["seed"])
            n, s, d, w = W._pairs(1, kw["n"], 0, 0.0, 0.0, params, kw["seed"])
        assert s.size > 0
        ctx_h = _lib.Context(0)
        ctx_h.build_graph(n, s, d, w)
        _same_csr(ctx_d, ctx_h)


def test_pair_model_configs_run(oracle):
    """C1's pair-model twin generated on the device runs the full hierarchy identically to
    the oracle on the host twin's edges."""
    import workloads as W
    import paper_1702_04645_b200 as P
    from paper_1702_04645_b200 import _lib
    spec = W.CONFIGS["c1_sbm_hash"]
    ctx = _lib.Context(0)
    ctx.build_pairs(0, spec["n"], spec["blocks"], spec["p_in"], spec["p_out"], seed=spec["seed"])
    g = P.Graph(spec["n"], None, None, None)
    g._ctx = ctx
    r = P.run(g, P.RunConfig())
    n, s, d, w = W.generate("c1_sbm_hash")
    o = oracle.run(n, s, d, w)
    assert len(r.hierarchy.levels) == len(o.levels)
    for x, y in zip(r.hierarchy.levels, o.levels):
        np.testing.assert_array_equal(x, y)
