"""Graph file formats vs the reference (tests/golden/io_*, made by running the
reference's load_edge_list / write_edge_list / save_csr; make_golden_io.py).

CPU: the native parser (host code in libinfuser_b200.so) against the
reference's CSR (rebuilt with the oracle's numpy from_edges), its error
messages, write_edge_list text and save_csr bytes.  GPU: the full
load_edge_list / load_csr / load_graph path."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden_names, load_golden

IO = golden_names("io_")
OK = [n for n in IO if not n.startswith("io_err")]
ERR = [n for n in IO if n.startswith("io_err")]


def _write(tmp_path, z, name):
    p = tmp_path / f"{name}.txt"
    p.write_bytes(z["content"].tobytes())
    return p


def test_fixtures_present():
    assert len(OK) >= 10 and len(ERR) >= 10


@pytest.mark.parametrize("name", OK)
def test_native_parser_matches_reference_csr(orc, tmp_path, name):
    from paper_2008_03095_b200.io import _parse_edge_list
    z = load_golden(name)
    edges, w, orig = _parse_edge_list(_write(tmp_path, z, name))
    assert np.array_equal(orig, z["orig_ids"])
    xadj, adj, ww = orc.csr_from_edges(len(orig), edges, w)
    assert np.array_equal(xadj, z["xadj"]) and np.array_equal(adj, z["adj"])
    assert np.array_equal(ww, z["weights"])


@pytest.mark.parametrize("name", ERR)
def test_parser_errors_match_reference(tmp_path, name):
    import paper_2008_03095_b200 as imx
    z = load_golden(name)
    p = _write(tmp_path, z, name)
    with pytest.raises(Exception) as ei:
        imx.load_edge_list(p)
    assert type(ei.value).__name__ == str(z["error_type"])
    assert str(ei.value) == str(z["error_msg"]).replace("{path}", str(p))


def test_missing_file_is_a_format_error(tmp_path):
    import paper_2008_03095_b200 as imx
    with pytest.raises(imx.GraphFormatError, match="cannot open"):
        imx.load_edge_list(tmp_path / "absent.txt")
    with pytest.raises(imx.GraphFormatError, match="cannot open"):
        imx.load_csr(tmp_path / "absent.csr")


@pytest.mark.parametrize("name", OK)
def test_write_edge_list_and_save_csr_bytes(tmp_path, name):
    import paper_2008_03095_b200 as imx
    z = load_golden(name)
    g = imx.Graph(z["xadj"], z["adj"], z["weights"], z["orig_ids"])
    imx.write_edge_list(g, tmp_path / "out.txt")
    assert (tmp_path / "out.txt").read_bytes() == z["written"].tobytes()
    imx.save_csr(g, tmp_path / "g.csr")
    assert (tmp_path / "g.csr").read_bytes() == z["csr_bytes"].tobytes()
    h = imx.load_csr(tmp_path / "g.csr")
    for key in ("xadj", "adj", "weights", "orig_ids"):
        assert np.array_equal(getattr(h, key), z[key])


def test_csr_cache_validation(tmp_path):
    import paper_2008_03095_b200 as imx
    (tmp_path / "bad").write_bytes(b"NOTACSR!" + bytes(40))
    with pytest.raises(imx.GraphFormatError, match="bad magic"):
        imx.load_csr(tmp_path / "bad")
    z = load_golden("io_basic")
    (tmp_path / "cut").write_bytes(z["csr_bytes"].tobytes()[:-3])
    with pytest.raises(imx.GraphFormatError, match="truncated"):
        imx.load_csr(tmp_path / "cut")


@pytest.mark.gpu
@pytest.mark.parametrize("name", OK)
def test_load_edge_list_and_load_graph_on_device(gpu, tmp_path, name):
    z = load_golden(name)
    p = _write(tmp_path, z, name)
    for g in (gpu.load_edge_list(p), gpu.load_graph(p)):
        for key in ("xadj", "adj", "weights", "orig_ids"):
            assert np.array_equal(getattr(g, key), z[key])
    (tmp_path / "g.csr").write_bytes(z["csr_bytes"].tobytes())
    h = gpu.load_graph(tmp_path / "g.csr")
    assert np.array_equal(h.adj, z["adj"])
    assert np.array_equal(h.reciprocal_slots[h.reciprocal_slots], np.arange(h.m))
