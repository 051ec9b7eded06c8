"""Summarise ncu outputs into profiles/: the launch list (per-kernel count,
total device time, share) and the --set full metrics of the captured
kernels (duration, DRAM bytes vs algorithmic bytes, occupancy).

    python scripts/ncu_summary.py launches.csv [prof.ncu-rep] --m M --j J --out profiles/x
"""

import argparse
import csv
import io
import json
import re
import subprocess
from collections import defaultdict

UNIT = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
        "s": 1e6, "second": 1e6}


def short(name):
    name = re.sub(r"^void\s+", "", name)
    name = re.sub(r"\(.*$", "", name)
    return name.replace("<unnamed>::", "")


def launches(path):
    t, n = defaultdict(float), defaultdict(int)
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(io.StringIO("".join(lines))):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = short(r["Kernel Name"])
        t[k] += float(r["Metric Value"].replace(",", "")) * UNIT[r["Metric Unit"]]
        n[k] += 1
    tot = sum(t.values())
    return [{"kernel": k, "launches": n[k], "total_us": t[k], "share": t[k] / tot}
            for k in sorted(t, key=lambda k: -t[k])]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__grid_size", "launch__block_size"]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
             "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1}
    res = []
    for r in rows[2:]:
        d = {"kernel": short(r[hdr.index("Kernel Name")])}
        for w in want:
            if w in hdr:
                i = hdr.index(w)
                v = float(r[i].replace(",", "")) * scale.get(units[i], 1)
                d[w] = v
        res.append(d)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("launches")
    ap.add_argument("report", nargs="?")
    ap.add_argument("--m", type=int, required=True)
    ap.add_argument("--j", type=int, required=True)
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    summary = {"launch_list": launches(a.launches)}
    if a.report:
        kern = full(a.report)
        algo = {"project_gram": 8 * a.m * (a.j + 2), "gram": 8 * a.m * (a.j + 2),
                "update": 8 * a.m * (a.j + 4), "stencil7": 16 * a.m, "mtm": 8 * a.m * (a.j + 2)}

        def family(name):
            for key in ("project_gram", "gram", "update", "stencil7", "mtm"):
                if key in name:
                    return key
            return None

        for d in kern:
            d["family"] = family(d["kernel"])
            d["algorithmic_bytes"] = algo.get(d["family"])
            dram = d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
            d["dram_bytes"] = dram
            if d["algorithmic_bytes"]:
                d["traffic_over_algorithmic"] = dram / d["algorithmic_bytes"]
                d["achieved_algorithmic_GBs"] = d["algorithmic_bytes"] / d["gpu__time_duration.sum"] / 1e9
        summary["ncu_full"] = kern
        summary["capture"] = {"m": a.m, "j": a.j}
        # per-kernel traffic entries bench.py reads
        for key in ("project_gram", "gram", "update", "stencil7", "mtm"):
            for d in kern:
                if d["family"] == key:
                    summary[key] = {"dram_bytes": d["dram_bytes"], "j": a.j,
                                    "algorithmic_bytes": d["algorithmic_bytes"],
                                    "traffic_over_algorithmic": d["traffic_over_algorithmic"]}
                    break
    with open(a.out + ".json", "w") as f:
        json.dump(summary, f, indent=1)
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main()
