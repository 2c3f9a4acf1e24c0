"""Summarise ncu captures into profiles/ (tracked).  Usage:
    python profiles/summarize.py full   <report.ncu-rep> <tag>
    python profiles/summarize.py launches <launches.csv> <tag>
Writes profiles/<tag>.json (+ .md)."""
import collections
import csv
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "sm__inst_executed.sum",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "lts__t_sectors_srcunit_tex_op_read.sum"]


def full(rep, tag):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(h, r))
        k = {"kernel": d.get("Kernel Name", "")[:120]}
        for key in KEYS:
            if key in d:
                k[key] = d[key] + " " + dict(zip(h, units)).get(key, "")
        stalls = []
        for key in h:
            if key.startswith("smsp__average_warps_issue_stalled") and key.endswith(
                    "per_issue_active.ratio") and d[key] not in ("", "n/a"):
                stalls.append((float(d[key]), key.split("stalled_")[1].split("_per")[0]))
        k["top_stalls"] = [f"{n}={v:.2f}" for v, n in sorted(stalls, reverse=True)[:6]]
        res.append(k)
    with open(os.path.join(HERE, tag + ".json"), "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


def launches(path, tag):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, mi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) <= mi:
            continue
        v = float(r[mi].replace(",", ""))
        u = r[ui]
        v = v / 1e6 if u in ("ns", "nsecond") else v / 1e3 if u in ("us", "usecond") else v
        agg[r[ki][:100]].append(v)
    tot = sum(sum(v) for v in agg.values())
    res = [{"kernel": k, "launches": len(v), "total_ms": sum(v), "avg_ms": sum(v) / len(v),
            "share": sum(v) / tot} for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1]))]
    with open(os.path.join(HERE, tag + ".json"), "w") as f:
        json.dump(res, f, indent=1)
    for x in res[:20]:
        print(f"{x['total_ms']:9.3f} ms  n={x['launches']:3d}  avg={x['avg_ms']:8.4f}  "
              f"{100 * x['share']:5.1f}%  {x['kernel']}")


if __name__ == "__main__":
    {"full": full, "launches": launches}[sys.argv[1]](sys.argv[2], sys.argv[3])
