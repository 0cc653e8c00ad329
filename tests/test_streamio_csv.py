"""Native CSV reader (stgn_read_stream) against the Python restatement of
S/streamio.py:53-79: identical arrays on written streams (with and without
features, sorted and unsorted), and identical errors (the native path declines
and the reference-faithful parser reports them). CPU only."""

import numpy as np
import pytest

from paper_2603_21090_b200.streamio import (StreamParseError, generate_stream, read_stream,
                                            write_stream)


def _same(a, b):
    (ea, da), (eb, db) = a, b
    assert da == db
    for f in ("src", "dst", "t", "feat"):
        np.testing.assert_array_equal(getattr(ea, f), getattr(eb, f))


@pytest.mark.parametrize("d_e", [0, 3])
def test_native_equals_python_on_written_stream(tmp_path, d_e):
    s = generate_stream(4, 50, 700, attachment="preferential", d_e=d_e, native=False)
    p = tmp_path / "s.csv"
    write_stream(s, d_e, str(p))
    _same(read_stream(str(p)), read_stream(str(p), native=False))


def test_sort_and_spellings(tmp_path):
    p = tmp_path / "s.csv"
    p.write_text("# streamtgn-edges v1 d_e=1\n0,1,2.0,0.5\n\n 3 , 4 ,1.0, -1e-3 \n5,6,2.0,inf\n")
    _same(read_stream(str(p), sort=True), read_stream(str(p), sort=True, native=False))
    with pytest.raises(StreamParseError) as ei:
        read_stream(str(p))
    assert ei.value.line_no == 4


@pytest.mark.parametrize("body,line", [
    ("0,1\n", 2),                 # too few fields
    ("0,1,2.0,9\n", 2),           # too many
    ("-1,1,2.0\n", 2),            # negative id
    ("0,1,2.0\n1,x,3.0\n", 3),    # not an integer
    ("0,1,0x10\n", 2),            # hex float (Python rejects)
])
def test_errors_match_reference_parser(tmp_path, body, line):
    p = tmp_path / "s.csv"
    p.write_text("# streamtgn-edges v1 d_e=0\n" + body)
    with pytest.raises(StreamParseError) as ei:
        read_stream(str(p))
    with pytest.raises(StreamParseError) as ej:
        read_stream(str(p), native=False)
    assert ei.value.line_no == ej.value.line_no == line
    assert str(ei.value) == str(ej.value)


def test_bad_header(tmp_path):
    p = tmp_path / "s.csv"
    p.write_text("# something else\n0,1,2.0\n")
    with pytest.raises(StreamParseError) as ei:
        read_stream(str(p))
    assert ei.value.line_no == 1
