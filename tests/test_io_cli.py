"""CPU checks of the on-disk formats and the CLI plumbing (io.py, cli.py), mirroring the
reference's own tests (test_graph.py:22-70, 165-172; test_cli.py)."""

import numpy as np
import pytest

from paper_1702_04645_b200 import io
from paper_1702_04645_b200.cli import main
from paper_1702_04645_b200.graph import GraphFormatError


def test_load_basic_and_defaults(tmp_path):
    p = tmp_path / "g.txt"
    p.write_text("# a comment\n0 1 2.5\n\n1 2\n2 0 1e0\n")
    g = io.load_edge_list(str(p))
    assert g.n == 3
    np.testing.assert_array_equal(g._src, [0, 1, 2])
    np.testing.assert_array_equal(g._w, [2.5, 1.0, 1.0])


def test_nodes_header(tmp_path):
    p = tmp_path / "g.txt"
    p.write_text("# nodes 5\n0 1 1.0\n")
    assert io.load_edge_list(str(p)).n == 5
    p.write_text("# nodes 2\n0 3 1.0\n")
    with pytest.raises(GraphFormatError):
        io.load_edge_list(str(p))


@pytest.mark.parametrize(
    "line", ["0 1 0.0", "0 1 -2", "0 1 nan", "0 1 inf", "0 x 1.0", "0 1.5 1.0", "-1 2 1.0",
             "0 1 2 3"])
def test_bad_lines_report_line_number(tmp_path, line):
    p = tmp_path / "g.txt"
    p.write_text("0 1 1.0\n%s\n" % line)
    with pytest.raises(GraphFormatError) as err:
        io.load_edge_list(str(p))
    assert "line 2" in str(err.value)


def test_fast_and_line_parsers_agree(tmp_path):
    rng = np.random.default_rng(3)
    s = rng.integers(0, 500, 4000)
    d = rng.integers(0, 500, 4000)
    w = rng.uniform(0.1, 3.0, 4000)
    p = tmp_path / "g.txt"
    p.write_text("# nodes 600\n" + "".join("%d %d %.17g\n" % t for t in zip(s, d, w)))
    fast = io._parse_fast(str(p))
    slow = io._parse_lines(str(p))
    assert fast is not None and fast[0] == slow[0] == 600
    for x, y in zip(fast[1:], slow[1:]):
        np.testing.assert_array_equal(x, y)
    np.testing.assert_array_equal(slow[3], w)   # %.17g round-trips bit for bit
    # mixed 2- and 3-column lines are valid in the reference: the fast path defers
    p.write_text("0 1 2.0\n1 2\n")
    assert io._parse_fast(str(p)) is None
    n, s2, d2, w2 = io._parse_lines(str(p))
    np.testing.assert_array_equal(w2, [2.0, 1.0])


def test_partition_roundtrip(tmp_path):
    labels = np.array([0, 0, 1, 2, 1])
    p = tmp_path / "x.flat"
    io.write_partition(labels, str(p))
    assert p.read_text() == "0 0\n1 0\n2 1\n3 2\n4 1\n"
    np.testing.assert_array_equal(io.read_partition(str(p)), labels)
    p.write_text("0 0\n0 1\n")
    with pytest.raises(GraphFormatError):
        io.read_partition(str(p))
    p.write_text("0 0\n1\n")
    with pytest.raises(GraphFormatError) as err:
        io.read_partition(str(p))
    assert "line 2" in str(err.value)


def test_binary_edge_list_roundtrip(tmp_path):
    rng = np.random.default_rng(9)
    s = rng.integers(0, 1000, 5000)
    d = rng.integers(0, 1000, 5000)
    w = rng.integers(1, 100, 5000).astype(float)
    p = tmp_path / "g.sle"
    io.write_edge_binary(str(p), 1000, s, d, w)
    g = io.load_graph(str(p))
    assert g.n == 1000
    for x, y in zip((g._src, g._dst, g._w), (s, d, w)):
        np.testing.assert_array_equal(x, y)
    p.write_bytes(b"NOTMAGIC" + b"\0" * 24)
    with pytest.raises(GraphFormatError):
        io.load_edge_binary(str(p))


def test_cli_errors_and_amdahl(tmp_path, capsys):
    assert main(["detect", str(tmp_path / "nope.edges")]) == 2
    assert "nope.edges" in capsys.readouterr().err
    bad = tmp_path / "bad.edges"
    bad.write_text("0 1 1.0\n0 1 -3.0\n")
    assert main(["detect", str(bad)]) == 2
    assert "line 2" in capsys.readouterr().err
    empty = tmp_path / "empty.edges"
    empty.write_text("# nodes 0\n")
    assert main(["detect", str(empty)]) == 2
    assert main(["amdahl", "--p", "0.95", "--threads", "1,12"]) == 0
    out = capsys.readouterr().out
    assert "12\t7.741935" in out
