"""Pin the oracle's edge-list text restatement (oracle.c orc_parse_edge_list /
orc_write_edge_list, io.hpp:18-64) to the reference's own outputs
(tests/golden/reference_io.json) and, where oracle/_ref is built, to the
reference on fresh seeded texts."""
import hashlib
import random

import numpy as np
import pytest

from oracle import binding as O


def _msg(e):
    return str(e).split("\x00")[0]  # what() is a C string


def test_parse_against_golden(io_golden):
    for case in io_golden["parse"]:
        text = case["text"].encode("latin-1")
        if "error" in case:
            with pytest.raises(O.ParseError) as ei:
                O.parse_edge_list(text)
            assert ei.value.line == case["error_line"]
            assert _msg(ei.value) == case["error"]
        else:
            assert O.parse_edge_list(text).reshape(-1).tolist() == case["pairs"]


def test_reference_test_cases(io_golden):
    # test_io.cpp:12-35
    assert O.parse_edge_list(b"0 1\n1 2\n").tolist() == [[0, 1], [1, 2]]
    assert O.parse_edge_list(b"# comment\n3 4\n").tolist() == [[3, 4]]
    assert O.parse_edge_list(b"").size == 0
    with pytest.raises(O.ParseError) as ei:
        O.parse_edge_list(b"0 1\n\n2 y\n")
    assert ei.value.line == 3


def test_write_against_golden(io_golden):
    from paper_1706_05151_b200 import trigraph as T  # host generators only

    g5 = O.build_graph([[0, 1], [0, 2], [1, 2], [1, 3], [2, 3], [3, 4]])
    assert O.write_edge_list(g5).decode() == io_golden["write_g5"]["text"]
    for name, pairs in (("pa20000", T.gen_pa(20000, 20, 3)),
                        ("rmat12", T.gen_rmat(12, 8, 0.57, 0.19, 0.19, 5))):
        txt = O.write_edge_list(O.build_graph(pairs))
        assert hashlib.sha256(txt).hexdigest() == io_golden[f"write_{name}"]["sha256"]
        # round trip (test_io.cpp:37-46)
        back = O.build_graph(O.parse_edge_list(txt))
        assert O.write_edge_list(back) == txt


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_parse_against_reference_fuzz():
    rng = random.Random(99)
    alphabet = [b" ", b"\t", b"\r", b"\n", b"\v", b"\f", b"#", b"+", b"-", b"0", b"1", b"9",
                b"x", b",", b"\x00", b"\xff", b"12", b"4294967296", b"18446744073709551616"]
    for _ in range(3000):
        text = b"".join(rng.choice(alphabet) for _ in range(rng.randint(0, 14)))
        r = O.ref_parse_edge_list(text)
        if isinstance(r, tuple):
            with pytest.raises(O.ParseError) as ei:
                O.parse_edge_list(text)
            assert (ei.value.line, _msg(ei.value)) == r
        else:
            assert np.array_equal(O.parse_edge_list(text), r)
