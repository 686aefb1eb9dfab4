"""Pin the CPU oracle against the reference's own outputs and known answers.

CPU-only.  The golden fixtures were produced by running the reference
package (tests/golden/make_golden.py); the murmur3 vectors are the
reference's frozen known-answer tests (reference tests/test_hashing.py:31-56).
"""

import hashlib
import struct

import numpy as np
import pytest

from conftest import golden_names, load_golden

ALL = golden_names()


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("data,seed,expected", [
    (b"", 0x00000000, 0x00000000),
    (b"", 0x00000001, 0x514E28B7),
    (b"", 0xFFFFFFFF, 0x81F16F39),
    (b"test", 0x00000000, 0xBA6BD213),
    (b"hello", 0x00000000, 0x248BFA47),
    (b"a", 0x00000000, 0x3C2569B2),
    (b"ab", 0x00000000, 0x9BBFD75F),
    (b"abc", 0x00000000, 0xB3DD93FA),
    (b"abcd", 0x00000000, 0x43ED676A),
    (b"The quick brown fox jumps over the lazy dog", 0x00000000, 0x2E4FF723),
    (b"Hello, world!", 0x9747B28C, 0x24884CBA),
])
def test_oracle_murmur3_reference_vectors(orc, data, seed, expected):
    assert orc.murmur3_bytes(data, seed) == expected


def test_oracle_pair_digests(orc):
    for lo, hi, expected in [(0, 1, 0x3AD85688), (3, 7, 0x2C37C8F7), (123, 456, 0x33BE5BF3)]:
        assert orc.lib().oracle_murmur3_pair(lo, hi) == expected
        assert orc.murmur3_bytes(struct.pack("<II", lo, hi)) == expected
    # masked values quoted in SURVEY 8(c)
    assert [orc.lib().oracle_murmur3_pair(a, b) & 0x7FFFFFFF
            for a, b in [(0, 1), (3, 7), (123, 456)]] == [987256456, 741853431, 868113395]


def test_oracle_randoms_first_words(orc):
    # first X words for seed 0 (this numpy); prefix stability
    assert orc.randoms(8, 0).tolist() == [1826701615, 1367864807, 1097657232, 579362556,
                                         661058652, 87989972, 161576974, 35492827]
    assert np.array_equal(orc.randoms(1024, 0)[:128], orc.randoms(128, 0))
    assert orc.randoms(20, 3).shape == (24,)


@pytest.mark.parametrize("name", ALL)
def test_oracle_csr_and_sampler_tables(orc, name):
    z = load_golden(name)
    xadj, adj, _ = orc.csr_from_edges(int(z["n"]), z["edges"].astype(np.int64))
    if "xadj" in z:
        assert np.array_equal(xadj, z["xadj"]) and np.array_equal(adj, z["adj"])
        hashes = orc.hash_table(xadj, adj)
        assert np.array_equal(hashes, z["hashes"])
        assert np.array_equal(orc.thresholds(z["weights"], orc.reciprocal(xadj, adj)), z["thr"])
    else:
        assert sha(xadj) == str(z["xadj_sha"]) and sha(adj) == str(z["adj_sha"])
        assert sha(orc.hash_table(xadj, adj)) == str(z["hashes_sha"])
    assert np.array_equal(orc.randoms(int(z["R"]), int(z["master_seed"])), z["X"])


def _golden_weights(orc, z, xadj, adj):
    if "weights" in z:
        return z["weights"]
    # config fixtures: constant schemes only (C1/C2)
    scheme = str(z["scheme"])
    assert scheme.startswith("const:")
    w = np.full(len(adj), float(scheme.split(":")[1]))
    assert sha(w) == str(z["weights_sha"])
    return w


@pytest.mark.parametrize("name", ALL)
def test_oracle_full_pipeline_matches_reference(orc, name):
    z = load_golden(name)
    n = int(z["n"])
    xadj, adj, _ = orc.csr_from_edges(n, z["edges"].astype(np.int64))
    w = _golden_weights(orc, z, xadj, adj)
    R, k = int(z["R"]), int(z["k"])
    out = orc.run_fused(xadj, adj, w, k, R, int(z["master_seed"]), nthreads=4)
    if "labels" in z:
        assert np.array_equal(out["labels"], z["labels"])
        assert np.array_equal(out["sizes"], z["sizes"])
    assert sha(out["labels"]) == str(z["labels_sha"])
    assert sha(out["sizes"]) == str(z["sizes_sha"])
    assert np.array_equal(out["gains"], z["gains"])
    assert out["seeds"].tolist() == z["seeds"].tolist()
    assert out["seed_gains"].tolist() == z["seed_gains"].tolist()
    assert out["sigma"] == int(z["sigma"])
    assert out["spread"] == float(z["spread"])
    assert out["spread_se"] == pytest.approx(float(z["spread_se"]), rel=1e-12, abs=1e-15)
    assert np.array_equal(out["trace"], z["trace"])


def test_oracle_thread_count_invariance(orc):
    z = load_golden("er_big_1000")
    xadj, adj, _ = orc.csr_from_edges(int(z["n"]), z["edges"])
    thr = orc.thresholds(z["weights"], orc.reciprocal(xadj, adj))
    h = orc.hash_table(xadj, adj)
    one, _ = orc.propagate(xadj, adj, h, thr, z["X"], nthreads=1, lane_block=8)
    many, _ = orc.propagate(xadj, adj, h, thr, z["X"], nthreads=8, lane_block=16)
    assert np.array_equal(one, many)
    assert np.array_equal(one, z["labels"])


def test_oracle_celf_equals_stepwise_argmax(orc):
    # CELF commits the step-wise lexicographic argmax of fresh gains
    z = load_golden("er_mid_300")
    labels, sizes = z["labels"], z["sizes"]
    ns = int(z["R"])
    n = labels.shape[0]
    owned = np.zeros((n, ns), bool)
    cols = np.arange(ns)
    seeds = []
    for _ in range(int(z["k"])):
        lu = labels[:, :ns]
        fresh = np.where(owned[lu, cols], 0, sizes[lu, cols]).sum(axis=1)
        fresh[seeds] = -1
        u = int(np.argmax(fresh))
        seeds.append(u)
        owned[labels[u, :ns], cols] = True
    assert seeds == z["seeds"].tolist()


# ---- the config-scale checker, pinned on every fixture ----

@pytest.mark.parametrize("name", ALL)
def test_oracle_uf_labels_match_reference(orc, name):
    """Per-lane union-find labels == the reference's propagate labels."""
    z = load_golden(name)
    xadj, adj, _ = orc.csr_from_edges(int(z["n"]), z["edges"].astype(np.int64))
    w = _golden_weights(orc, z, xadj, adj)
    thr = orc.thresholds(w, orc.reciprocal(xadj, adj))
    uni = len(thr) > 0 and bool((thr == thr[0]).all())
    labels = orc.uf_labels(xadj, adj, orc.hash_table(xadj, adj), int(thr[0]) if uni else thr,
                           z["X"], nthreads=4)
    if "labels" in z:
        assert np.array_equal(labels, z["labels"])
    assert sha(labels) == str(z["labels_sha"])


@pytest.mark.parametrize("chunks", ["one", "ragged", "reversed"])
@pytest.mark.parametrize("name", ALL)
def test_oracle_selection_check_matches_reference(orc, name, chunks):
    """Lane-chunked sizes + fresh-gain table + heap == the reference's
    sizes, initial gains, seeds, seed gains, trace and spread_se, for any
    lane chunking (the checker used at config scale on the GPU box)."""
    z = load_golden(name)
    n, R, k = int(z["n"]), int(z["R"]), int(z["k"])
    xadj, adj, _ = orc.csr_from_edges(n, z["edges"].astype(np.int64))
    w = _golden_weights(orc, z, xadj, adj)
    thr = orc.thresholds(w, orc.reciprocal(xadj, adj))
    labels = orc.uf_labels(xadj, adj, orc.hash_table(xadj, adj), thr, z["X"], nthreads=4)
    W = labels.shape[1]
    cuts = {"one": [0, W], "ragged": sorted({0, min(W, 3), min(W, 11), W}),
            "reversed": [0, W // 2, W]}[chunks]
    spans = list(zip(cuts[:-1], cuts[1:]))
    if chunks == "reversed":
        spans = spans[::-1]
    chk = orc.SelectionCheck(n, k, z["seeds"], R)
    sizes = np.empty_like(labels)
    for a, b in spans:
        sizes[:, a:b] = chk.add_chunk(labels[:, a:b], a, nthreads=3)
    out = chk.result()
    assert sha(sizes) == str(z["sizes_sha"])
    assert np.array_equal(out["gains"], z["gains"])
    assert out["seeds"].tolist() == z["seeds"].tolist()
    assert out["seed_gains"].tolist() == z["seed_gains"].tolist()
    assert out["sigma"] == int(z["sigma"])
    assert np.array_equal(out["trace"], z["trace"])
    assert out["spread_se"] == pytest.approx(float(z["spread_se"]), rel=1e-12, abs=1e-15)


def test_oracle_selection_check_flags_a_wrong_seed(orc):
    """A claimed sequence that deviates at step t yields the reference's
    seeds up to t and a different seed at t (so the comparison fails)."""
    z = load_golden("er_mid_300")
    n, R, k = int(z["n"]), int(z["R"]), int(z["k"])
    claimed = z["seeds"].copy()
    other = next(v for v in range(n) if v not in set(claimed.tolist()))
    claimed[2] = other
    chk = orc.SelectionCheck(n, k, claimed, R)
    chk.add_chunk(z["labels"], 0)
    out = chk.result()
    assert out["seeds"][:3].tolist() == z["seeds"][:3].tolist()
    assert out["seeds"].tolist() != claimed.tolist()


@pytest.mark.parametrize("kind,n,m,draws,extra", [
    (0, 1000, 3000, 0, {}),
    (1, 1 << 12, 0, 16 << 12, {"probs": (0.57, 0.19, 0.19, 0.05)}),
    (1, 1 << 11, 5000, 0, {"probs": (0.45, 0.22, 0.22, 0.11)}),
    (2, 3000, 8000, 0, {"gamma": 2.5}),
])
def test_oracle_config_csr_equals_numpy_generator(orc, kind, n, m, draws, extra):
    """The C restatement of the config generator + sorted-key CSR equals the
    numpy generator (generators.edges) + Graph.from_edges restatement."""
    from paper_2008_03095_b200 import generators as gen
    cdf = gen.chung_lu_cdf(n, extra["gamma"]) if "gamma" in extra else None
    probs = extra.get("probs")
    xadj, adj = orc.config_csr(kind, n, m, 11, draws, probs, cdf)
    wx, wa, _ = orc.csr_from_edges(n, gen.edges(kind, n, m, 11, draws, probs, cdf))
    assert np.array_equal(xadj, wx) and np.array_equal(adj, wa)
