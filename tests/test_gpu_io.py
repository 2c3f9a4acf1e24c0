"""Edge-list text on the device (io.hpp:18-64) through the C ABI:
parse_edge_list / build_graph_from_text / write_edge_list, bit-exact against
the reference's outputs (tests/golden/reference_io.json) and the oracle, plus
size-independent round trips at larger sizes."""
import hashlib
import random

import numpy as np
import pytest

from oracle import binding as O
from paper_1706_05151_b200 import trigraph as T

pytestmark = pytest.mark.gpu


def test_parse_against_golden(io_golden):
    for case in io_golden["parse"]:
        text = case["text"].encode("latin-1")
        if "error" in case:
            with pytest.raises(T.ParseError) as ei:
                T.parse_edge_list(text)
            assert ei.value.line == case["error_line"], case
            assert str(ei.value) == case["error"], case
            with pytest.raises(T.ParseError):
                T.build_graph_from_text(text)
        else:
            got = T.parse_edge_list(text)
            assert got.reshape(-1).tolist() == case["pairs"], case


def test_reference_io_cases(io_golden):
    # test_io.cpp:12-46
    assert T.parse_edge_list(b"0 1\n1 2\n").tolist() == [[0, 1], [1, 2]]
    assert T.parse_edge_list(b"# comment\n3 4\n").tolist() == [[3, 4]]
    assert T.parse_edge_list(b"").size == 0
    assert T.parse_edge_list(b"\n  \n# only comments\n").size == 0
    with pytest.raises(T.ParseError) as ei:
        T.parse_edge_list(b"0 1\n\n2 y\n")
    assert ei.value.line == 3
    g5 = T.build_graph([[0, 1], [0, 2], [1, 2], [1, 3], [2, 3], [3, 4]])
    text = T.write_edge_list(g5)
    assert text.decode() == io_golden["write_g5"]["text"]
    g2 = T.build_graph_from_text(text)
    assert (g2.num_nodes(), g2.num_edges()) == (5, 6)
    assert T.write_edge_list(g2) == text
    assert T.write_edge_list(T.build_graph(np.zeros((0, 2), np.uint32))) == b""


def test_write_against_golden(io_golden):
    for name, pairs in (("pa20000", T.gen_pa(20000, 20, 3)),
                        ("rmat12", T.gen_rmat(12, 8, 0.57, 0.19, 0.19, 5))):
        with T.build_graph(pairs) as g:
            txt = T.write_edge_list(g)
            rec = io_golden[f"write_{name}"]
            assert len(txt) == rec["len"]
            assert hashlib.sha256(txt).hexdigest() == rec["sha256"]
            with T.build_graph_from_text(txt) as g2:
                o1, a1 = g.csr()
                o2, a2 = g2.csr()
                assert np.array_equal(o1, o2) and np.array_equal(a1, a2)


def test_random_texts_against_oracle():
    rng = random.Random(7)
    ws = [b"", b" ", b"\t", b"\r", b"\v", b"\f", b"  "]
    nums = [b"0", b"5", b"+9", b"-2", b"4294967296", b"18446744073709551616", b"0012", b"77"]
    for _ in range(400):
        lines = []
        for _ in range(rng.randint(0, 30)):
            r = rng.random()
            if r < 0.1:
                lines.append(rng.choice(ws) + b"#" + rng.choice(nums))
            elif r < 0.15:
                lines.append(rng.choice(ws))
            else:
                lines.append(rng.choice(ws) + rng.choice(nums) + rng.choice(ws[1:]) +
                             rng.choice(nums) + rng.choice(ws) +
                             (rng.choice([b" x", b"y", b" 3", b","]) if rng.random() < 0.01
                              else b""))
        text = b"\n".join(lines) + (b"\n" if rng.random() < 0.5 else b"")
        try:
            want = O.parse_edge_list(text)
        except O.ParseError as e:
            with pytest.raises(T.ParseError) as ei:
                T.parse_edge_list(text)
            assert ei.value.line == e.line and str(ei.value) == str(e).split("\x00")[0]
            continue
        assert np.array_equal(T.parse_edge_list(text), want)


def test_large_round_trip_and_chunk_boundaries():
    """PA(3e5): ~100 MB of text spans many 64 KB newline-count chunks; lines
    with comments, CRLF and padding are interleaved so lines straddle chunk
    ends at every offset.  write -> parse -> build reproduces the CSR, and the
    parse equals the oracle's."""
    pairs = T.gen_pa(300_000, 20, 9)
    with T.build_graph(pairs) as g:
        txt = T.write_edge_list(g)
        off, adj = g.csr()
    ref = O.build_graph(pairs)
    assert txt == O.write_edge_list(ref)
    lines = txt.split(b"\n")
    rng = random.Random(3)
    noisy = []
    for ln in lines[:-1]:
        r = rng.random()
        if r < 0.05:
            noisy.append(b"# " + b"c" * rng.randint(0, 200))
        if r < 0.02:
            noisy.append(b" " * rng.randint(0, 70000))  # a blank line longer than a chunk
        noisy.append((b"\t" if r < 0.3 else b"") + ln + (b"\r" if r > 0.7 else b""))
    text = b"\n".join(noisy)  # no final newline
    want = O.parse_edge_list(text)
    got = T.parse_edge_list(text)
    assert np.array_equal(got, want)
    with T.build_graph_from_text(text, n_override=300_005) as g2:
        o2, a2 = g2.csr()
        assert g2.num_nodes() == 300_005
        assert np.array_equal(o2[:len(off)], off) and np.array_equal(a2, adj)
    # an error deep in the text reports the exact line
    bad = text + b"\n12 x"
    with pytest.raises(T.ParseError) as ei:
        T.parse_edge_list(bad)
    assert ei.value.line == bad.count(b"\n") + 1


def test_device_text_input():
    import torch

    text = b"0 1\n1 2\n2 0\n# c\n2 3\n"
    buf = torch.tensor(list(text), dtype=torch.uint8, device="cuda")
    assert T.parse_edge_list(buf).tolist() == [[0, 1], [1, 2], [2, 0], [2, 3]]
    with T.build_graph_from_text(buf) as g:
        assert T.count_node_iterator_n(g) == 1


@pytest.mark.parametrize("kind", ["rmat", "ws"])
def test_device_generators_match_host(kind):
    """R-MAT / Watts-Strogatz generated on the device build the same graph as
    the host harness's pair stream."""
    if kind == "rmat":
        pairs, n = T.gen_rmat(15, 8, 0.57, 0.19, 0.19, 11), 1 << 15
        g = T.graph_rmat(15, 8, 0.57, 0.19, 0.19, 11)
    else:
        pairs, n = T.gen_ws(200_003, 10, 0.1, 11), 200_003
        g = T.graph_ws(200_003, 10, 0.1, 11)
    with T.build_graph(pairs, n) as ref, g:
        o1, a1 = ref.csr()
        o2, a2 = g.csr()
        assert np.array_equal(o1, o2) and np.array_equal(a1, a2)
        assert T.count_node_iterator_n(g) == T.count_node_iterator_n(ref)
    with pytest.raises(ValueError):
        T.graph_ws(10, 3, 0.1, 1)
