"""Pins the CPU oracle (oracle/ra_oracle.c) to the reference.

Two anchors: (1) golden fixtures produced by the unmodified reference
(tests/golden/make_golden.py) and the reference's own golden splitmix64
vector (test_util.cpp:13-19); (2) when oracle/_ref is available, bit-for-bit
agreement with the reference library on fresh random cases.
"""
import os

import numpy as np
import pytest

from conftest import GOLDEN, load_golden
from oracle.ffi import BuildParams, OracleError


def test_splitmix64_golden(port):
    # test_util.cpp:13-19
    assert port.splitmix64(1234567, 3) == [6457827717110365317, 3203168211198807973,
                                          9817491932198370423]
    with open(os.path.join(GOLDEN, "splitmix64.txt")) as f:
        assert [int(x) for x in f.read().split()] == port.splitmix64(1234567, 3)


@pytest.mark.parametrize("name", ["d32", "d128"])
def test_port_matches_golden_workload(port, name):
    g = load_golden(f"workload_{name}.npz")
    n, dm, dh, H, G, seed, nd = (int(x) for x in g["spec"])
    w = port.generate_workload(n, dm, dh, H, G, seed=seed, n_decode=nd)
    for key in ("prefill_q", "decode_q", "keys", "values"):
        np.testing.assert_array_equal(w[key], g[key])


GOLD_PARAMS = {
    "d32": BuildParams(k_train=32, max_degree=16, ef_construction=64),
    "d128": BuildParams(k_train=128, max_degree=24, ef_construction=256, edge_window=8),
}


@pytest.mark.parametrize("name,heads", [("d32", 2), ("d128", 1)])
def test_port_matches_golden_graph_and_search(port, name, heads):
    w = load_golden(f"workload_{name}.npz")
    H, G = int(w["spec"][3]), int(w["spec"][4])
    W, _ = port.static_partition(int(w["spec"][0]), 128, 512)
    for h in range(heads):
        keys = w["keys"][h // (H // G)]
        blob = port.graph_build(keys, w["prefill_q"][h], GOLD_PARAMS[name])
        with open(os.path.join(GOLDEN, f"graph_{name}_h{h}.oodg"), "rb") as f:
            assert blob == f.read()
        s = load_golden(f"search_{name}_h{h}.npz")
        gr = port.graph(keys, blob)
        for i in range(len(s["qi"])):
            q = w["decode_q"][h][s["qi"][i]]
            r = gr.search(q, int(s["k"][i]), W if s["mask"][i] else None, int(s["ef"][i]))
            n = len(r.ids)
            np.testing.assert_array_equal(r.ids, s["ids"][i][:n])
            np.testing.assert_array_equal(r.scores, s["scores"][i][:n])
            assert r.scanned == s["scanned"][i]
            assert r.truncated == bool(s["truncated"][i])


@pytest.mark.parametrize("name,h", [("d32", 0), ("d32", 1), ("d128", 0)])
def test_port_matches_golden_attention(port, name, h):
    w = load_golden(f"workload_{name}.npz")
    a = load_golden(f"attn_{name}_h{h}.npz")
    H, G, dh = int(w["spec"][3]), int(w["spec"][4]), int(w["spec"][2])
    g = h // (H // G)
    W, _ = port.static_partition(int(w["spec"][0]), 128, 512)
    for qi in range(len(a["out"])):
        q = w["decode_q"][h][qi]
        om = a["omega"][qi]
        om = om[om != 0xFFFFFFFF]
        pw = port.partial_attention(q, w["keys"][g], w["values"][g], W)
        po = port.partial_attention(q, w["keys"][g], w["values"][g], om)
        assert pw[1] == a["zw"][qi] and pw[2] == a["sw"][qi]
        assert po[1] == a["zo"][qi] and po[2] == a["so"][qi]
        out, _, _ = port.merge(pw, po, dh)
        np.testing.assert_array_equal(out, a["out"][qi])


def test_port_matches_reference_random_builds(port, ref):
    rng = np.random.default_rng(3)
    for n, d, nq, bp in [
        (257, 8, 64, BuildParams(k_train=8, max_degree=4, ef_construction=8)),
        (1000, 16, 200, BuildParams(k_train=16, max_degree=8, ef_construction=16)),
        (600, 16, 150, BuildParams(k_train=16, max_degree=8, prune_inner_product=True)),
        (500, 16, 100, BuildParams(k_train=16, max_degree=8, entry_maxnorm=True)),
        (100, 4, 0, BuildParams(max_degree=3)),          # no training queries
        (64, 8, 4, BuildParams(k_train=8, edge_window=0)),
        (1, 4, 1, BuildParams()),                          # single key
        (300, 12, 40, BuildParams(k_train=20, max_degree=1)),  # cap 1 forces repair
    ]:
        keys = rng.standard_normal((n, d)).astype(np.float32)
        tq = rng.standard_normal((nq, d)).astype(np.float32)
        assert port.graph_build(keys, tq, bp) == ref.graph_build(keys, tq, bp), (n, d, nq)


def test_port_matches_reference_search_and_attention(port, ref, small_workload):
    w = small_workload
    keys, vals = w["keys"][0], w["values"][0]
    bp = BuildParams(k_train=32, max_degree=16, ef_construction=64)
    blob = ref.graph_build(keys, w["prefill_q"][0], bp)
    gp, gr = port.graph(keys, blob), ref.graph(keys, blob)
    W, pool = port.static_partition(2048, 128, 512)
    for qi in range(16):
        q = w["decode_q"][0][qi]
        for mask in (None, W, W[:37]):
            for ef, k in ((16, 10), (100, 100), (300, 50), (2048, 2048 - 640)):
                a, b = gp.search(q, k, mask, ef), gr.search(q, k, mask, ef)
                np.testing.assert_array_equal(a.ids, b.ids)
                np.testing.assert_array_equal(a.scores, b.scores)
                assert (a.scanned, a.truncated) == (b.scanned, b.truncated)
        ids = pool[qi * 7: qi * 7 + 50]
        pa, pb = port.partial_attention(q, keys, vals, ids), ref.partial_attention(q, keys, vals, ids)
        np.testing.assert_array_equal(pa[0], pb[0])
        assert pa[1:] == pb[1:]


def test_port_error_messages_match_reference(port, ref):
    keys = np.ones((4, 2), np.float32)
    for o in (port, ref):
        blob = o.graph_build(keys, np.ones((1, 2), np.float32), BuildParams(k_train=3))
        g = o.graph(keys, blob)
        with pytest.raises(OracleError, match="k must be >= 1"):
            g.search(np.ones(2, np.float32), 0, None, 4)
        with pytest.raises(OracleError, match="ef must be >= k"):
            g.search(np.ones(2, np.float32), 5, None, 4)
        with pytest.raises(OracleError, match="k_train must be >= 1"):
            o.graph_build(keys, np.ones((1, 2), np.float32), BuildParams(k_train=0))
        with pytest.raises(OracleError, match="bad graph magic"):
            o.graph(keys, b"XODG" + blob[4:])
        with pytest.raises(OracleError, match="empty attention support"):
            o.merge(None, None, 2)
