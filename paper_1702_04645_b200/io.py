"""On-disk formats of the reference (graph.py:178-332) plus a binary edge list.

Text formats are the reference's, byte for byte:
  * edge list: ``src dst [weight]`` lines, ``#`` comments, ``# nodes N`` header
    (load_edge_list graph.py:178-242; dump_edge_list graph.py:245-254 writes ``%.17g``);
  * partition: ``node community`` lines (write_partition / read_partition graph.py:301-332).
Errors are ``GraphFormatError`` (a ValueError) with the offending line number, like the
reference.  Well-formed files take a vectorised fast path; anything the fast path rejects
is re-parsed line by line for the reference's exact message.

Binary edge list (``.sle``): 8-byte magic ``SLMEDGE1``, int64 n, int64 m, int64 flags
(bit 0: weights present, bit 1: int32 ids), then src[m], dst[m] (int64 or int32) and w[m]
(float64).  Read with one ``np.fromfile`` per array -- the ingest path for 1e9-edge graphs,
where the text parser would dominate setup.
"""

from __future__ import annotations

import math
import os

import numpy as np

from .graph import Graph, GraphFormatError

__all__ = ["load_edge_list", "dump_edge_list", "write_partition", "read_partition",
           "load_edge_binary", "write_edge_binary", "load_graph"]

MAGIC = b"SLMEDGE1"


def _parse_lines(path):
    """The reference's line-by-line parser (graph.py:178-242) -> (n, src, dst, w)."""
    srcs, dsts, ws = [], [], []
    declared = -1
    max_id = -1
    with open(path, "r", encoding="utf-8") as handle:
        for lineno, raw in enumerate(handle, start=1):
            line = raw.strip()
            if not line:
                continue
            if line.startswith("#"):
                parts = line[1:].split()
                if len(parts) == 2 and parts[0] == "nodes":
                    try:
                        declared = max(declared, int(parts[1]))
                    except ValueError:
                        raise GraphFormatError(f"line {lineno}: bad node-count header: {line!r}")
                continue
            parts = line.split()
            if len(parts) not in (2, 3):
                raise GraphFormatError(f"line {lineno}: expected 'src dst [weight]', got {line!r}")
            try:
                s = int(parts[0])
                d = int(parts[1])
            except ValueError:
                raise GraphFormatError(f"line {lineno}: node ids must be integers: {line!r}")
            if s < 0 or d < 0:
                raise GraphFormatError(f"line {lineno}: node ids must be non-negative: {line!r}")
            if len(parts) == 3:
                try:
                    weight = float(parts[2])
                except ValueError:
                    raise GraphFormatError(f"line {lineno}: bad weight: {line!r}")
            else:
                weight = 1.0
            if not math.isfinite(weight) or weight <= 0.0:
                raise GraphFormatError(f"line {lineno}: weight must be finite and > 0: {line!r}")
            srcs.append(s)
            dsts.append(d)
            ws.append(weight)
            max_id = max(max_id, s, d)
    if declared >= 0 and declared < max_id + 1:
        raise GraphFormatError(
            f"node-count header declares {declared} nodes but ids reach {max_id}")
    n = max(declared, max_id + 1, 0)
    return (n, np.array(srcs, dtype=np.int64), np.array(dsts, dtype=np.int64),
            np.array(ws, dtype=np.float64))


def _parse_fast(path):
    """Vectorised parse of a well-formed file; None when anything needs the slow path."""
    with open(path, "rb") as fh:
        data = fh.read()
    declared = -1
    body = []
    for line in data.split(b"\n"):
        t = line.strip()
        if not t:
            continue
        if t.startswith(b"#"):
            parts = t[1:].split()
            if len(parts) == 2 and parts[0] == b"nodes":
                try:
                    declared = max(declared, int(parts[1]))
                except ValueError:
                    return None
            continue
        body.append(t)
    if not body:
        return (max(declared, 0), np.empty(0, np.int64), np.empty(0, np.int64),
                np.empty(0, np.float64))
    toks = [t.split() for t in body]
    ncols = len(toks[0])
    if ncols not in (2, 3) or any(len(t) != ncols for t in toks):
        return None
    try:
        arr = np.array(toks, dtype=bytes)
        src = arr[:, 0].astype(np.int64)
        dst = arr[:, 1].astype(np.int64)
        w = arr[:, 2].astype(np.float64) if ncols == 3 else np.ones(len(body), np.float64)
    except (ValueError, OverflowError):
        return None
    if (src < 0).any() or (dst < 0).any() or not np.isfinite(w).all() or (w <= 0).any():
        return None
    max_id = int(max(src.max(), dst.max()))
    if declared >= 0 and declared < max_id + 1:
        return None
    return max(declared, max_id + 1, 0), src, dst, w


def load_edge_list(path) -> Graph:
    """graph.py:178-242: parse ``src dst [weight]`` lines into a Graph (weight default 1.0)."""
    parsed = _parse_fast(path)
    if parsed is None:
        parsed = _parse_lines(path)
    n, src, dst, w = parsed
    return Graph.from_edges(n, src, dst, w)


def dump_edge_list(graph: Graph, path, header_lines=()) -> None:
    """graph.py:245-254: ``# nodes N`` then the canonical ``src dst %.17g`` rows."""
    rows = graph.edge_rows()
    lines = [f"# {h}" for h in header_lines]
    lines.append(f"# nodes {graph.n}")
    lines.extend("%d %d %.17g" % (s, d, w) for s, d, w in
                 zip(rows.tolist(), graph.out_dst.tolist(), graph.out_w.tolist()))
    lines.append("")
    with open(path, "w", encoding="utf-8") as handle:
        handle.write("\n".join(lines))


def write_partition(labels, path) -> None:
    """graph.py:301-305: one ``node community`` line per node."""
    labels = np.asarray(labels, dtype=np.int64)
    with open(path, "w", encoding="utf-8") as handle:
        handle.write("\n".join(f"{i} {c}" for i, c in enumerate(labels.tolist())))
        handle.write("\n")


def read_partition(path) -> np.ndarray:
    """graph.py:308-332 (same errors)."""
    nodes, comms = [], []
    with open(path, "r", encoding="utf-8") as handle:
        for lineno, raw in enumerate(handle, start=1):
            line = raw.strip()
            if not line or line.startswith("#"):
                continue
            parts = line.split()
            if len(parts) != 2:
                raise GraphFormatError(f"line {lineno}: expected 'node community', got {line!r}")
            try:
                nodes.append(int(parts[0]))
                comms.append(int(parts[1]))
            except ValueError:
                raise GraphFormatError(f"line {lineno}: bad integer: {line!r}")
    labels = np.full(len(nodes), -1, dtype=np.int64)
    for node, comm in zip(nodes, comms):
        if node < 0 or node >= len(nodes) or labels[node] != -1:
            raise GraphFormatError(
                f"partition file must list each node 0..n-1 exactly once (offending node {node})")
        labels[node] = comm
    return labels


def write_edge_binary(path, n, src, dst, w=None) -> None:
    """Binary edge list (module docstring): int32 ids when they fit, weights when given."""
    src = np.asarray(src)
    dst = np.asarray(dst)
    m = src.size
    small = n < (1 << 31)
    flags = (1 if w is not None else 0) | (2 if small else 0)
    it = np.int32 if small else np.int64
    with open(path, "wb") as fh:
        fh.write(MAGIC)
        np.array([n, m, flags], np.int64).tofile(fh)
        np.ascontiguousarray(src, it).tofile(fh)
        np.ascontiguousarray(dst, it).tofile(fh)
        if w is not None:
            np.ascontiguousarray(w, np.float64).tofile(fh)


def load_edge_binary(path) -> Graph:
    """Read a binary edge list into a Graph (validated like Graph.from_edges)."""
    with open(path, "rb") as fh:
        if fh.read(8) != MAGIC:
            raise GraphFormatError(f"{path}: not a binary edge list (bad magic)")
        hdr = np.fromfile(fh, np.int64, 3)
        if hdr.size != 3:
            raise GraphFormatError(f"{path}: truncated header")
        n, m, flags = (int(x) for x in hdr)
        it = np.int32 if flags & 2 else np.int64
        src = np.fromfile(fh, it, m)
        dst = np.fromfile(fh, it, m)
        w = np.fromfile(fh, np.float64, m) if flags & 1 else np.ones(m, np.float64)
        if src.size != m or dst.size != m or w.size != m:
            raise GraphFormatError(f"{path}: truncated edge arrays")
    return Graph.from_edges(n, src, dst, w)


def load_graph(path) -> Graph:
    """Binary edge list by magic, text edge list otherwise."""
    with open(path, "rb") as fh:
        head = fh.read(8)
    if head == MAGIC:
        return load_edge_binary(path)
    return load_edge_list(path)


def stem(path) -> str:
    return os.path.splitext(os.path.basename(str(path)))[0]
