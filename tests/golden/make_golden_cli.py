"""Golden CLI outputs from the REFERENCE's own CLI (trawl/cli.py), run in the
build container (/tmp/trawl_ref, see make_golden.py).  Writes cli.json:
sha256 of the --output text file and of the .remap sidecar, plus the
deterministic report keys, per argument vector.

    python tests/golden/make_golden_cli.py
"""

import hashlib
import json
import os
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import REF_TMP, import_reference  # noqa: E402

CASES = [
    ["--app", "deepwalk", "--synth", "powerlaw:1000", "--weighted", "--samples", "64", "--seed", "3"],
    ["--app", "khop", "--synth", "powerlaw:1000", "--samples", "40", "--seed", "5", "--fanouts", "6,3",
     "--layout", "per-step"],
    ["--app", "ppr", "--synth", "path:300", "--weighted", "--samples", "50", "--seed", "2", "--term-prob", "0.1"],
    ["--app", "node2vec", "--synth", "powerlaw:1000", "--weighted", "--samples", "30", "--seed", "1",
     "--p", "0.5", "--q", "2", "--workers", "3"],
    ["--app", "mvs", "--synth", "powerlaw:1000", "--samples", "8", "--seed", "4", "--batch-size", "12"],
    ["--app", "layer", "--synth", "star:300", "--samples", "5", "--seed", "6", "--layer-max", "120",
     "--layer-step", "40", "--layout", "per-step"],
]
DET_KEYS = ("app", "paradigm", "samples", "seed", "workers", "steps", "adjacency_fetches",
            "groups.small", "groups.medium", "groups.large")


def sha(path):
    with open(path, "rb") as fh:
        return hashlib.sha256(fh.read()).hexdigest()[:16]


def main():
    import_reference()
    out = []
    env = dict(os.environ, PYTHONPATH=os.path.join(REF_TMP, "src"))
    for args in CASES:
        with tempfile.TemporaryDirectory() as d:
            o, r = os.path.join(d, "out.txt"), os.path.join(d, "rep.txt")
            subprocess.check_call([sys.executable, "-m", "trawl.cli", *args, "--output", o,
                                   "--report", r], env=env, stdout=subprocess.DEVNULL)
            rep = dict(line.split("=", 1) for line in open(r).read().splitlines())
            out.append({"args": args, "output": sha(o), "remap": sha(o + ".remap"),
                        "report": {k: rep[k] for k in DET_KEYS}})
    with open(os.path.join(HERE, "cli.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print(len(out), "cli cases")


if __name__ == "__main__":
    main()
