"""Golden NDSO files (the reference's binary output, output.py:108-142): for
the first golden runs (tests/golden/runs.json), the reference's own
write_binary bytes in both layouts, as sha256 digests in ndso.json.

Run in the build container only (imports the reference as make_golden.py does):

    python tests/golden/make_golden_ndso.py
"""
import hashlib
import json
import os
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import import_reference  # noqa: E402

N_CASES = 10  # the SURVEY Appendix C table: one case per app


def main():
    import_reference()
    from trawl.apps import make_app
    from trawl.engine import EngineConfig, make_samples, tp_run
    from trawl.output import LAYOUT_FINAL, LAYOUT_PER_STEP, read_binary, write_binary
    from trawl.synth import make_synthetic
    metas = json.load(open(os.path.join(HERE, "runs.json")))[:N_CASES]
    out = []
    with tempfile.TemporaryDirectory() as td:
        for m in metas:
            assert not m["params"].get("unique")
            spec = m["graph"].split("|")[0]
            g = make_synthetic(spec, weighted=m["weighted"], seed=m["seed"])
            app = make_app(m["app"], **m["params"])
            res = tp_run(app, g, make_samples(app, g, m["n_samples"], m["seed"]),
                         EngineConfig(seed=m["seed"]))
            ent = {"idx": m["idx"]}
            for layout in (LAYOUT_FINAL, LAYOUT_PER_STEP):
                path = os.path.join(td, f"{m['idx']}.{layout}.ndso")
                write_binary(res, layout, path)
                read_binary(path)  # the reference reads its own file back
                ent[layout] = hashlib.sha256(open(path, "rb").read()).hexdigest()
            out.append(ent)
    with open(os.path.join(HERE, "ndso.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print(f"wrote {len(out)} NDSO digests")


if __name__ == "__main__":
    main()
