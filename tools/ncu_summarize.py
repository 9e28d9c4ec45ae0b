"""Summarise the round's ncu captures (tools/ncu_round.sh TAG) into
profiles/TAG_ncu_summary.json: per workload, per kernel name, the launch
count, device time, DRAM bytes (read + write), DRAM GB/s and its fraction of
the measured HBM peak, issue / warp activity; and `traffic_bytes_per_step`
= the DRAM bytes of k_walk_persistent over one C2 SP step (node2vec + PPR),
the number bench.py reports as roofline.traffic.

  python tools/ncu_summarize.py r02
"""
import collections
import csv
import json
import os
import shutil
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
        "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3,
        "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def launches(path):
    """{launch id: {"name":..., metric: value}} from a long-format ncu --csv log."""
    out = collections.OrderedDict()
    hdr = None
    with open(path, newline="") as fh:
        for r in csv.reader(fh):
            if r and r[0] == "ID":
                hdr = r
                continue
            if not hdr or len(r) != len(hdr):
                continue
            d = dict(zip(hdr, r))
            L = out.setdefault(d["ID"], {"name": d["Kernel Name"]})
            v = d["Metric Value"].replace(",", "")
            try:
                v = float(v) * UNIT.get(d["Metric Unit"], 1.0)
            except ValueError:
                pass
            L[d["Metric Name"]] = v
    return out


def short(name):
    n = name.split("(")[0]
    for p in ("void ", "nd::", "(anonymous namespace)::", "<unnamed>::"):
        n = n.replace(p, "")
    return n.strip()


def by_kernel(ls, peak):
    agg = collections.OrderedDict()
    for L in ls.values():
        k = short(L["name"])
        a = agg.setdefault(k, {"launches": 0, "ms": 0.0, "dram_bytes": 0.0, "_issue": 0.0,
                               "_warps": 0.0, "_l2": 0.0})
        ms = L.get("gpu__time_duration.sum", 0.0)
        a["launches"] += 1
        a["ms"] += ms
        a["dram_bytes"] += L.get("dram__bytes_read.sum", 0.0) + L.get("dram__bytes_write.sum", 0.0)
        a["_issue"] += ms * L.get("smsp__issue_active.avg.pct_of_peak_sustained_active", 0.0)
        a["_warps"] += ms * L.get("sm__warps_active.avg.pct_of_peak_sustained_active", 0.0)
        a["_l2"] += ms * L.get("lts__t_sector_hit_rate.pct", 0.0)
    tot = sum(a["ms"] for a in agg.values()) or 1.0
    for a in agg.values():
        ms = a["ms"] or 1e-9
        a["share_of_time"] = a["ms"] / tot
        a["dram_gbs"] = a["dram_bytes"] / (ms / 1e3) / 1e9
        a["dram_frac_of_peak"] = a["dram_gbs"] / peak
        a["issue_active_pct"] = a.pop("_issue") / ms
        a["warps_active_pct"] = a.pop("_warps") / ms
        a["l2_hit_pct"] = a.pop("_l2") / ms
    return dict(sorted(agg.items(), key=lambda kv: -kv[1]["ms"]))


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
    src = os.path.join(REPO, "gpurun_out")
    try:
        peak = float(json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        peak = 6650.0
    out = {"round": tag, "peak_hbm_gbs": peak,
           "capture": "tools/ncu_round.sh (ncu --metrics ... --clock-control none "
                      "--profile-from-start off python tools/probe_ncu_round.py <workload>)",
           "note": "ncu times are serialised and cold-cache; shares, bytes and rates are the "
                   "evidence, absolute times are not bench values",
           "workloads": {}}
    for w in ("walk_sp", "walk_tp", "khop", "dedup", "collective"):
        p = os.path.join(src, f"ncu_{tag}_{w}.csv")
        if not os.path.exists(p):
            continue
        ls = launches(p)
        out["workloads"][w] = by_kernel(ls, peak)
        if w == "walk_sp":
            walk = [L for L in ls.values() if "k_walk_persistent" in L["name"]]
            out["traffic_bytes_per_step"] = sum(
                L.get("dram__bytes_read.sum", 0.0) + L.get("dram__bytes_write.sum", 0.0) for L in walk)
            out["walk_launches"] = [{k: v for k, v in L.items() if k != "name"} for L in walk]
            out["walk_kernel_ms_per_step"] = sum(L.get("gpu__time_duration.sum", 0.0) for L in walk)
    dst = os.path.join(REPO, "profiles", f"{tag}_ncu_summary.json")
    with open(dst, "w") as fh:
        json.dump(out, fh, indent=1)
    lb = os.path.join(src, f"ncu_{tag}_launches_bench.csv")
    if os.path.exists(lb):
        shutil.copy(lb, os.path.join(REPO, "profiles", f"{tag}_launches_bench.csv"))
    print(dst)


if __name__ == "__main__":
    main()
