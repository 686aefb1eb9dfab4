"""Golden fixtures for the graph file formats, made by running the REFERENCE
package (graph.py:269-437) in the build container:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_io.py

Every case is a text edge list (bytes) fed to the reference's load_edge_list;
the fixture stores the resulting CSR + orig ids, the reference's
write_edge_list text and save_csr bytes -- or the exception type and message
(with the file path replaced by "{path}").
"""

from __future__ import annotations

import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent

from infmax.graph import load_edge_list, save_csr, write_edge_list  # noqa: E402


def cases():
    rng = np.random.default_rng(7)
    big = []
    ids = rng.integers(-10**12, 10**12, size=3000)
    for _ in range(20000):
        a, b = rng.integers(0, len(ids), size=2)
        w = rng.random()
        form = rng.integers(0, 4)
        if form == 0:
            big.append(f"{ids[a]} {ids[b]}")
        elif form == 1:
            big.append(f"{ids[a]}\t{ids[b]}\t{w!r}")
        elif form == 2:
            big.append(f"  {ids[a]}  {ids[b]}  {w:.3f}  ")
        else:
            big.append(f"{ids[a]} {ids[b]} {w:.6e}")
        if rng.random() < 0.02:
            big.append("# comment " + str(rng.integers(0, 100)))
        if rng.random() < 0.02:
            big.append("")
    return {
        "basic": b"0 1\n1 2\n2 3\n",
        "weights_comments": b"# header\n10 20 0.5\n\n20 30 0.25\n  # indented comment\n30 10 1.0\n",
        "dupes_selfloops": b"5 6 0.1\n6 5 0.9\n5 5 0.3\n7 7\n6 7 0.2\n5 6 0.4\n",
        "crlf_cr_tabs": b"1\t2\t0.5\r\n2 3\r3 4 0.75\r\n\r\n4\x1c5\n",
        "underscores_signs": b"1_000 +2 0.5\n-3 1_000 1_0e-1\n+2 -3 .5\n",
        "inf_nan_words": b"1 2 1\n2 3 0e0\n",
        "large_ids": b"9223372036854775807 -9223372036854775808 0.5\n-9223372036854775808 0\n",
        "first_appearance": b"9 8\n7 9\n8 7\n1 9\n",
        "isolated_by_selfloop": b"4 4\n1 2\n",
        "random_20k": ("\n".join(big) + "\n").encode(),
        # error cases
        "err_fields": b"0 1\n1 2 3 4\n",
        "err_one_field": b"0 1\n\n7\n",
        "err_nonnumeric": b"0 1\n1 x\n",
        "err_float_word": b"0 1 0.5\n1 2 abc\n",
        "err_hex": b"0 1 0x1p-2\n",
        "err_weight_range": b"0 1 0.5\n1 2 1.5\n",
        "err_weight_neg": b"0 1 -0.25\n",
        "err_weight_nan": b"0 1 nan\n",
        "err_weight_inf": b"0 1 inf\n",
        "err_bad_underscore": b"1__0 2\n",
        "err_no_edges": b"# nothing\n3 3\n\n",
        "err_empty": b"",
    }


def main():
    out = {}
    with tempfile.TemporaryDirectory() as td:
        for name, content in cases().items():
            p = Path(td) / f"{name}.txt"
            p.write_bytes(content)
            rec = {"content": np.frombuffer(content, np.uint8)}
            try:
                g = load_edge_list(p)
            except Exception as exc:      # recorded, not raised
                rec["error_type"] = np.array(type(exc).__name__)
                rec["error_msg"] = np.array(str(exc).replace(str(p), "{path}"))
            else:
                rec.update(xadj=g.xadj, adj=g.adj, weights=g.weights, orig_ids=g.orig_ids)
                wp = Path(td) / f"{name}.out"
                write_edge_list(g, wp)
                rec["written"] = np.frombuffer(wp.read_bytes(), np.uint8)
                cp = Path(td) / f"{name}.csr"
                save_csr(g, cp)
                rec["csr_bytes"] = np.frombuffer(cp.read_bytes(), np.uint8)
            np.savez_compressed(HERE / f"io_{name}.npz", **rec)
            print(name, rec.get("error_type", "ok"), rec.get("error_msg", ""))


if __name__ == "__main__":
    sys.exit(main())
