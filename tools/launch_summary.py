"""Per-kernel summary of an ncu launch list (--metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum --csv): launches, mean duration,
share of GPU time, mean DRAM bytes per launch. Writes <out>_launch_summary.json
and profiles/ncu_traffic.json (the `traffic` field bench.py reports)."""
import csv
import io
import json
import sys
from collections import defaultdict


def main(path, out_prefix):
    rows = [l for l in open(path) if l.startswith('"')]
    per = defaultdict(lambda: defaultdict(float))
    for r in csv.DictReader(io.StringIO("".join(rows))):
        per[(r["ID"], r["Kernel Name"].split("(")[0])][r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    agg = defaultdict(lambda: {"launches": 0, "ns": 0.0, "bytes": 0.0})
    for (_, name), m in per.items():
        a = agg[name.replace("rfb::", "").split("::")[-1]]
        a["launches"] += 1
        a["ns"] += m["gpu__time_duration.sum"]
        a["bytes"] += m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]
    total = sum(a["ns"] for a in agg.values())
    summary = {k: {"launches": a["launches"], "mean_us": a["ns"] / a["launches"] / 1e3, "share": a["ns"] / total,
                   "dram_rw_bytes": a["bytes"] / a["launches"]}
               for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["ns"])}
    json.dump(summary, open(out_prefix + "_launch_summary.json", "w"), indent=1)
    names = {"track": "k_track", "fuse": "k_fuse", "allocate": "k_alloc", "cull": "k_cull"}
    traffic = {k: round(summary[v]["dram_rw_bytes"]) for k, v in names.items() if v in summary}
    traffic["_note"] = ("dram__bytes_read.sum + dram__bytes_write.sum per launch, mean over the launch list "
                        f"{path.split('/')[-1]} (ncu replays with a flushed L2: cold-cache upper bounds)")
    json.dump(traffic, open("profiles/ncu_traffic.json", "w"), indent=1)
    for k, v in summary.items():
        print(f"{k:24s} {v['launches']:5d} {v['mean_us']:9.1f} us  share {v['share']:.3f}  dram {v['dram_rw_bytes'] / 1e6:.2f} MB")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
