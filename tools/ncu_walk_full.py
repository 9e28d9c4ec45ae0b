"""profiles/<TAG>_ncu_walk_full.json from the raw page of the round's
`--set full` capture of the C2 SP step's walk launches (tools/ncu_round.sh):
per launch, time, DRAM bytes, hit rates, issue / warp activity and the
stall-reason shares of the PC samples.

  python tools/ncu_walk_full.py r02
"""
import csv
import json
import os
import sys

TAG = sys.argv[1] if len(sys.argv) > 1 else "r02"
KIND = sys.argv[2] if len(sys.argv) > 2 else "walk"  # walk | tw (TP k_tw_multi launches)
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
raw = os.path.join(REPO, "gpurun_out", f"ncu_{TAG}_{KIND}_full_raw.csv")
rows = list(csv.reader(open(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]
# the probe's launches in order: node2vec (one window), PPR window 1, PPR window 2
NAMES = (["node2vec (4,194,304 walkers x 100 steps)", "ppr window 1 (steps 0-127)",
          "ppr window 2 (the continuing walkers)"] if KIND == "walk" else
         [f"node2vec TP, k_tw_multi launch {k}" for k in range(16)])
STALL = "smsp__pcsamp_warps_issue_stalled_"
launches = []
for i, r in enumerate(data):
    d = dict(zip(hdr, r))
    u = dict(zip(hdr, units))
    out = {"name": NAMES[i] if i < len(NAMES) else f"launch {i}",
           "kernel": d.get("Kernel Name", "")[:60]}
    for k in KEYS:
        out[k] = d.get(k)
        if u.get(k):
            out[k + " unit"] = u[k]
    stalls = {}
    for h, v in d.items():
        if h.startswith(STALL) and not h.endswith("_not_issued"):
            try:
                stalls[h[len(STALL):]] = float(v.replace(",", ""))
            except ValueError:
                pass
    tot = sum(stalls.values())
    out["stall_share"] = {k: round(v / tot, 3) for k, v in sorted(stalls.items(), key=lambda x: -x[1])
                          if tot and v / tot >= 0.01}
    launches.append(out)
cap = ("ncu --set full --clock-control none --import-source on --profile-from-start off "
       "-k regex:k_walk_persistent -c 10 python tools/probe_ncu_round.py walk_sp (tools/ncu_round.sh)"
       if KIND == "walk" else
       "ncu --set full --clock-control none --profile-from-start off -k regex:k_tw_multi "
       "--launch-skip 8 -c 4 python tools/probe_tw_once.py node2vec")
res = {"round": TAG, "capture": cap, "report": f"gpurun_out/ncu_{TAG}_{KIND}_full.ncu-rep (not committed)",
       "launches": launches}
dst = os.path.join(REPO, "profiles", f"{TAG}_ncu_{KIND}_full.json")
json.dump(res, open(dst, "w"), indent=1)
print(dst)
for l in launches:
    print(l["name"], l["gpu__time_duration.sum"], l.get("gpu__time_duration.sum unit"), l["stall_share"])
