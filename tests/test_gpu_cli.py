"""The CLI end to end on the device (reference test_cli.py semantics): partition files in
the reference's format, identical to the oracle's hierarchy; bench's runs.csv/phases.tsv;
generate -> detect round trip through the text format."""

import numpy as np
import pytest

from paper_1702_04645_b200 import io
from paper_1702_04645_b200.cli import main

pytestmark = pytest.mark.gpu

TRIANGLES = "0 1 1.0\n1 2 1.0\n2 0 1.0\n3 4 1.0\n4 5 1.0\n5 3 1.0\n"


def test_detect_two_triangles(tmp_path, capsys, monkeypatch):
    f = tmp_path / "tri.edges"
    f.write_text(TRIANGLES)
    out = tmp_path / "out"
    assert main(["detect", str(f), "--out-dir", str(out), "--seed", "7"]) == 0
    np.testing.assert_array_equal(io.read_partition(str(out / "tri.flat")), [0, 0, 0, 1, 1, 1])
    assert (out / "tri.level0").exists() and (out / "tri.level1").exists()
    summary = capsys.readouterr().out
    assert "score=0.5" in summary and "levels=2" in summary
    out2 = tmp_path / "out2"
    monkeypatch.setenv("SYNCLOUVAIN_THREADS", "2")
    assert main(["detect", str(f), "--out-dir", str(out2), "--seed", "7"]) == 0
    assert "threads=2" in capsys.readouterr().out
    for name in ("tri.flat", "tri.level0", "tri.level1"):
        assert (out / name).read_bytes() == (out2 / name).read_bytes()


def test_detect_matches_oracle_and_binary(tmp_path, oracle):
    import workloads as W
    n, s, d, w = W.rmat(12, 8, 1, 4)
    txt = tmp_path / "g.edges"
    txt.write_text(f"# nodes {n}\n" + "".join("%d %d %.17g\n" % t for t in zip(s, d, w)))
    binf = tmp_path / "gb.sle"
    io.write_edge_binary(str(binf), n, s, d, w)
    assert main(["detect", str(txt), "--out-dir", str(tmp_path)]) == 0
    assert main(["detect", str(binf), "--out-dir", str(tmp_path)]) == 0
    r = oracle.run(n, s, d, w, seed=0)
    for t, lv in enumerate(r.levels):
        np.testing.assert_array_equal(io.read_partition(str(tmp_path / f"g.level{t}")), lv)
        assert (tmp_path / f"g.level{t}").read_bytes() == (tmp_path / f"gb.level{t}").read_bytes()
    np.testing.assert_array_equal(io.read_partition(str(tmp_path / "g.flat")), r.flat)


def test_bench_writes_runs_and_phases(tmp_path, capsys):
    import workloads as W
    n, s, d, w = W.rmat(11, 8, 0, 2)
    binf = tmp_path / "g.sle"
    io.write_edge_binary(str(binf), n, s, d, w)
    assert main(["bench", "--input", str(binf), "--repeats", "2", "--out-dir", str(tmp_path)]) == 0
    rows = (tmp_path / "runs.csv").read_text().splitlines()
    assert rows[0] == ("threads,repeat,wall_seconds,score,levels,seed,p,union_entries,"
                       "plan_gteps,plan_hbm_frac")
    assert len(rows) == 3 and float(rows[1].split(",")[8]) > 0
    ph = (tmp_path / "phases.tsv").read_text().splitlines()
    assert ph[0] == "threads\tphase\tmean_seconds" and len(ph) == 6


def test_generate_roundtrip(tmp_path):
    from paper_1702_04645_b200 import _lib, generators as GN
    out = tmp_path / "r.edges"
    assert main(["generate", "--kind", "rmat", "--scale", "10", "--edge-factor", "8",
                 "--weights", "int100", "--seed", "4", "--out", str(out)]) == 0
    g = io.load_edge_list(str(out))
    ctx = _lib.Context(0)
    GN.rmat_device(ctx, 10, 8, 1, 4)
    for x, y in zip(g.context().csr(), ctx.csr()):
        np.testing.assert_array_equal(x, y)
