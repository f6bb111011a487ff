"""Policy CSV formatted and parsed on the device (pvi_policy_csv_format /
pvi_policy_csv_parse) with the semantics of runner.cpp:90-148 and
io.cpp:53-92 (parse_csv): byte-identical rows, row-count / field-count /
non-numeric FormatError and tuple-range IndexingError for the first bad row
in file order, std::stoi field parsing, last row wins for a repeated state,
unnamed states 0.  (tests/test_gpu_runner.py checks whole runner files
against the reference runner's own output.)"""
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _py_rows(m, actions):
    """The reference's row loop, restated in Python (decode + to_string)."""
    n = m.state_count()
    nb = m.info.max_order_b + 1 if m.scenario() == "b" else 0
    out = []
    for s in range(n):
        f = [str(d) for d in m.decode(s)]
        a = int(actions[s])
        f += [str(a // nb), str(a % nb)] if nb else [str(a)]
        out.append(",".join(f) + "\n")
    return "".join(out).encode()


def _header(m):
    from paper_2303_10672_b200 import runner
    return runner.csv_row(runner.state_column_names(m) + runner.action_column_names(m)).encode()


@pytest.mark.parametrize("preset", ["a/m2/exp1", "b/m2/exp1", "c/m3/exp1", "a/m3/exp5"])
def test_rows_match_reference_loop(pvi, preset):
    m = pvi.make_preset(preset)
    n = m.state_count()
    a = np.random.default_rng(3).integers(0, m.action_count(), n).astype(np.uint32)
    body = m.policy_csv_body(a)
    assert body == _py_rows(m, a)
    np.testing.assert_array_equal(m.policy_from_csv_text(_header(m) + body), a)


def test_headline_round_trip(pvi):
    m = pvi.make_preset("b/m3/exp1")
    n = m.state_count()
    a = np.random.default_rng(4).integers(0, 256, n).astype(np.uint32)
    t0 = time.perf_counter()
    body = m.policy_csv_body(a)
    t1 = time.perf_counter()
    back = m.policy_from_csv_text(_header(m) + body)
    t2 = time.perf_counter()
    np.testing.assert_array_equal(back, a)
    print(f"b/m3/exp1 policy CSV {len(body) / 1e6:.1f} MB: format {t1 - t0:.3f} s, parse {t2 - t1:.3f} s")
    # spot-check rows against the reference loop
    rows = body.split(b"\n")
    for s in (0, 1, 4095, 4096, n // 2 + 12345, n - 1):
        f = [str(d) for d in m.decode(s)] + [str(a[s] // 16), str(a[s] % 16)]
        assert rows[s] == ",".join(f).encode()


def _small(pvi):
    m = pvi.make_preset("a/m2/exp1")  # 121 states, tuple (x_1, x_2) in [0, 10]^2
    a = (np.arange(121) % 11).astype(np.uint32)
    return m, a, _header(m), m.policy_csv_body(a)


def test_parse_semantics(pvi):
    m, a, head, body = _small(pvi)
    rows = body.split(b"\n")[:-1]
    # CRLF line ends, no final newline
    txt = head.replace(b"\n", b"\r\n") + b"\r\n".join(rows)
    np.testing.assert_array_equal(m.policy_from_csv_text(txt), a)
    # std::stoi: leading blanks, '+', trailing garbage after the digits
    r = list(rows)
    r[5] = b" 0,+5,7xyz"
    got = m.policy_from_csv_text(head + b"\n".join(r) + b"\n")
    assert got[5] == 7
    # a state named twice: the last row wins; the state it displaced stays 0
    r = list(rows)
    r[7] = b"0,9,3"   # state 9 named again (row 10 also names it)
    got = m.policy_from_csv_text(head + b"\n".join(r) + b"\n")
    assert got[9] == a[9] and got[7] == 0
    r = list(rows)
    r[20] = b"0,7,4"  # state 7 named after its own row: this one wins
    got = m.policy_from_csv_text(head + b"\n".join(r) + b"\n")
    assert got[7] == 4 and got[20] == 0
    # quoted fields go through the host parse_csv restatement: same result
    q = head + b"\n".join(b'"' + x.replace(b",", b'","') + b'"' for x in rows) + b"\n"
    np.testing.assert_array_equal(m.policy_from_csv_text(q), a)


def test_parse_errors_in_file_order(pvi):
    m, a, head, body = _small(pvi)
    rows = body.split(b"\n")[:-1]

    def parse(rs):
        return m.policy_from_csv_text(head + b"\n".join(rs) + b"\n")

    with pytest.raises(pvi.FormatError, match="policy CSV has 121 rows, expected 122"):
        parse(rows[:-1])
    r = list(rows)
    r[4] = b"1,2"
    with pytest.raises(pvi.FormatError, match="policy CSV row 5 has 2 fields"):
        parse(r)
    r = list(rows)
    r[9] = b"1,x,3"
    with pytest.raises(pvi.FormatError, match="policy CSV row 10 is not numeric"):
        parse(r)
    r = list(rows)
    r[9] = b"1,99999999999,3"
    with pytest.raises(pvi.FormatError, match="policy CSV row 10 is not numeric"):
        parse(r)
    r = list(rows)
    r[2] = b"0,11,3"
    with pytest.raises(pvi.IndexingError, match=r"tuple component 1 = 11 outside \[0, 10\]"):
        parse(r)
    # the first bad row wins, whatever its kind
    r = list(rows)
    r[2] = b"0,-1,3"
    r[6] = b"1,2"
    with pytest.raises(pvi.IndexingError, match="tuple component 1 = -1"):
        parse(r)
    r[1] = b"a,b,c"
    with pytest.raises(pvi.FormatError, match="row 2 is not numeric"):
        parse(r)
