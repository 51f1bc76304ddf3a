"""Text file formats of the command-line tool.

* nodes: one node per line, ``d`` whitespace-separated coordinates;
* complex vectors: one ``re im`` pair per line, written with 17 significant
  digits so a round trip is exact.

Blank lines are ignored.  Files are parsed in bulk (one ``float`` conversion
of all tokens); only when that fails, or a line has the wrong field count, is
the file scanned again to name the first offending line -- with the
reference CLI's messages (cli.py:177-222), which tests compare verbatim.
"""

import numpy as np


class FormatError(Exception):
    """A malformed or unreadable input file."""


def _lines(path, what):
    try:
        with open(path) as fh:
            text = fh.read()
    except OSError as exc:
        raise FormatError(f"cannot open {what} file {path}: {exc}") from exc
    # (line number, fields) of every non-blank line
    return [(no, ln.split()) for no, ln in enumerate(text.splitlines(), start=1) if ln.strip()]


def _table(path, rows, width, count_msg):
    """Stack the rows' fields as float64 (rows of ``width`` fields)."""
    for no, fields in rows:
        if len(fields) != width:
            raise FormatError(f"{path}:{no}: {count_msg(len(fields))}")
    try:
        return np.array([f for _, fields in rows for f in fields], dtype=np.float64).reshape(-1, width)
    except ValueError:
        for no, fields in rows:
            try:
                [float(f) for f in fields]
            except ValueError:
                raise FormatError(f"{path}:{no}: malformed number") from None
        raise


def read_nodes(path, d):
    """(M, d) float64 node coordinates."""
    rows = _lines(path, "nodes")
    table = _table(path, rows, d, lambda k: f"expected {d} coordinates, got {k}")
    if table.shape[0] == 0:
        raise FormatError(f"{path}: no nodes found")
    return table


def read_complex_vector(path):
    """complex128 vector from 're im' lines."""
    rows = _lines(path, "vector")
    pairs = _table(path, rows, 2, lambda k: f"expected 're im' pair, got {k} fields")
    return np.ascontiguousarray(pairs).view(np.complex128).reshape(-1)


def write_complex_vector(path, values):
    """'re im' lines, 17 significant digits."""
    v = np.asarray(values, dtype=np.complex128).reshape(-1)
    with open(path, "w") as fh:
        fh.writelines(f"{z.real:.17g} {z.imag:.17g}\n" for z in v)
