"""Golden fixtures for edge-list ingestion.

Runs the REFERENCE's own parser, trawl.graph.load_edge_list
(graph.py:132-188), on edge-list texts that cover its rules: universal
newlines, comments and blank lines, ASCII and Unicode whitespace, 2/3 fields,
PEP 515 underscores, float spellings (exponents, inf, nan, signed zero,
mantissas beyond the device's exact fast path), non-ASCII digits, sparse and
huge ids, undirected doubling, keyed default weights, and every error it
raises (line number and message).  Writes tests/golden/ingest.json (arguments,
expected error) and tests/golden/ingest.npz (the texts as UTF-8 bytes and the
expected CSR arrays).

    python tests/golden/make_golden_ingest.py      # needs /root/reference
"""

from __future__ import annotations

import json
import os
import random
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import import_reference  # noqa: E402


def big_text(seed: int, n: int) -> str:
    """Random file mixing every spelling the device parses plus a few host lines."""
    rnd = random.Random(seed)
    lines = []
    fmts = [lambda w: f"{w:.3f}", lambda w: f"{w:.17g}", lambda w: f"{w:e}", lambda w: repr(w),
            lambda w: f"{int(w)}", lambda w: f"{w:.1f}".rstrip("0"), lambda w: f"{w * 1000:.0f}e-3"]
    for i in range(n):
        r = rnd.random()
        s, d = rnd.randrange(0, 5000) * 7919, rnd.randrange(0, 5000) * 7919
        if r < 0.02:
            lines.append("# comment " + str(i))
        elif r < 0.03:
            lines.append("   ")
        elif r < 0.40:
            lines.append(f"{s} {d}")
        elif r < 0.41:
            lines.append(f"{s}\t{d}\t{rnd.uniform(0, 9):.40f}")  # 40 digits: host path
        else:
            lines.append(f"{s} {d} {rnd.choice(fmts)(rnd.uniform(0, 9))}")
    seps = ["\n", "\r\n", "\r"]
    out = []
    for ln in lines:
        out.append(ln + rnd.choice(seps) if rnd.random() < 0.05 else ln + "\n")
    return "".join(out)


CASES = [
    ("basic", "0 1\n0 2\n1 2\n", {}),
    ("comment_weighted", "# comment\n0 1 2.5\n", {"weighted": True}),
    ("keyed_weights", "0 1\n1 2\n2 0 3.5\n\n3 1\n", {"weighted": True, "seed": 3}),
    ("newlines", "0 1\r\n1 2\r2 3\n\r\n3 4\r\r5 6", {}),
    ("whitespace", "  0\t1  \n\x0b2 3\x0c\n4\x1c5\n 6 \x1f 7 \n", {}),
    ("sparse_ids", "500 10\n10 7\n1000000000000 7\n", {}),
    ("undirected", "0 1\n1 2\n2 2\n", {"undirected": True}),
    ("dups_selfloops", "0 1\n0 1\n1 1\n", {}),
    ("float_spellings",
     "0 1 1e-3\n1 2 .5\n2 3 5.\n3 4 1_000.25\n4 5 +3\n5 6 inf\n6 7 nan\n7 8 -0.0\n"
     "8 9 0.1\n9 10 7E2\n10 11 1_2e1_0\n11 12 Infinity\n12 13 -nan\n13 14 0e999\n"
     "14 15 123456789012345678901234.5\n15 16 1.000000000000000000001\n16 17 4.9e-324\n"
     "17 18 1.7976931348623157e308\n18 19 2.2250738585072014e-308\n19 20 9007199254740993\n",
     {"weighted": True}),
    ("int_spellings", "+5 007\n-0 1_000\n00 12\n", {}),
    ("unicode_lines", "1 2\n٣ 4\n5 6 7.5\n", {"weighted": True}),
    ("third_field_ignored", "0 1 notaweight\n1 2 -5\n", {}),
    ("no_trailing_newline", "0 1\n1 2", {}),
    ("trailing_cr", "0 1\r", {}),
    ("err_fields", "0 1\nbroken line here extra\n", {}),
    ("err_one_field", "0 1\n7\n", {}),
    ("err_bad_id", "0 x\n", {}),
    ("err_bad_id_underscore", "0 1\n1__0 2\n", {}),
    ("err_bad_first_id", "y 1\n", {}),
    ("err_neg_id", "0 1\n-3 2\n", {}),
    ("err_bad_weight", "0 1 notaweight\n", {"weighted": True}),
    ("err_neg_weight", "0 1 -2.0\n", {"weighted": True}),
    ("err_neg_inf_weight", "0 1 3\n1 2 -inf\n", {"weighted": True}),
    ("err_weight_dot", "0 1 .\n", {"weighted": True}),
    ("err_after_host_line", "0 1\n1 2\n2 x\n", {}),
    ("err_in_host_line", "0 1\n٣ x \n2 y\n", {}),
    ("err_first_of_two", "0 1\n1 z\n2 w\n", {}),
    ("empty", "", {}),
    ("only_comments", "# only comments\n\n   \n", {}),
    ("huge_id", "0 1\n9223372036854775808 2\n", {}),
    ("big_mixed", big_text(11, 60_000), {"weighted": True, "seed": 5}),
    ("big_mixed_undirected", big_text(12, 20_000), {"weighted": True, "undirected": True}),
]


def main():
    trawl = import_reference()
    from trawl.graph import load_edge_list
    meta, store = [], {}
    with tempfile.TemporaryDirectory() as td:
        for name, text, kw in CASES:
            path = os.path.join(td, name + ".txt")
            with open(path, "w", encoding="utf-8", newline="") as fh:
                fh.write(text)
            ent = {"name": name, "kwargs": kw}
            store[f"{name}/text"] = np.frombuffer(text.encode("utf-8"), dtype=np.uint8)
            try:
                g = load_edge_list(path, **kw)
                for k in ("row_offsets", "col_indices", "weights", "remap"):
                    store[f"{name}/{k}"] = np.asarray(getattr(g, k))
                ent["ok"] = True
            except trawl.errors.GraphParseError as e:
                ent.update(ok=False, error="GraphParseError", line_no=e.line_no, message=str(e))
            except trawl.errors.EmptyGraphError:
                ent.update(ok=False, error="EmptyGraphError")
            except OverflowError:
                ent.update(ok=False, error="OverflowError")
            meta.append(ent)
    with open(os.path.join(HERE, "ingest.json"), "w") as fh:
        json.dump(meta, fh, indent=0)
    np.savez_compressed(os.path.join(HERE, "ingest.npz"), **store)
    print(f"{len(meta)} cases, {sum(m['ok'] for m in meta)} graphs")


if __name__ == "__main__":
    main()
