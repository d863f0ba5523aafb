"""Summarize ncu output into profiles/ (tracked).

  python tools/ncu_summary.py launches <launches.csv> <out.md>
      per-kernel launch count, device time, share of the captured time, DRAM bytes
      (ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv).
  python tools/ncu_summary.py traffic <launches.csv[.gz]> <traffic.json> <config/kernel> <name regex>
      mean DRAM traffic per launch of the matching kernels over the launch list -> traffic.json.
  python tools/ncu_summary.py full <report.ncu-rep> <out.md> [traffic.json class]
      key --set full metrics per captured launch; optionally records the mean DRAM traffic per
      launch under `class` ("config/kernel") in traffic.json (read by bench.py for roofline.traffic).
"""
import csv
import io
import json
import os
import re
import subprocess
import sys
from collections import OrderedDict, defaultdict


def short(name):
    name = re.sub(r"\(.*", "", name)
    name = name.replace("skc::", "").replace("(anonymous namespace)::", "").replace("unnamed>::", "")
    return name.replace("void ", "").strip()


def launches(path, out):
    rows = [l for l in open(path) if l.startswith('"')]
    rd = csv.DictReader(io.StringIO("".join(rows)))
    per = OrderedDict()
    for r in rd:
        k = (r["ID"], r["Kernel Name"])
        per.setdefault(k, {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    agg = defaultdict(lambda: dict(n=0, ns=0.0, rd=0.0, wr=0.0))
    for (i, name), m in per.items():
        a = agg[short(name)]
        a["n"] += 1
        a["ns"] += m.get("gpu__time_duration.sum", 0.0)
        a["rd"] += m.get("dram__bytes_read.sum", 0.0)
        a["wr"] += m.get("dram__bytes_write.sum", 0.0)
    total = sum(a["ns"] for a in agg.values()) or 1.0
    lines = [f"# ncu launch list summary ({os.path.basename(path)})", "",
             f"{len(per)} launches captured (cold-cache, serialised by ncu: compare shares, not absolutes).", "",
             "| kernel | launches | total us | share | mean us | DRAM read MB/launch | DRAM write MB/launch | DRAM GB/s |",
             "|---|---|---|---|---|---|---|---|"]
    for name, a in sorted(agg.items(), key=lambda kv: -kv[1]["ns"]):
        gbs = (a["rd"] + a["wr"]) / max(a["ns"], 1e-9)
        lines.append(f"| `{name}` | {a['n']} | {a['ns'] / 1e3:.1f} | {a['ns'] / total:.3f} | {a['ns'] / a['n'] / 1e3:.2f} | "
                     f"{a['rd'] / a['n'] / 1e6:.2f} | {a['wr'] / a['n'] / 1e6:.2f} | {gbs:.0f} |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "smsp__inst_executed.sum", "lts__t_sector_hit_rate.pct",
        "smsp__issue_active.avg.pct_of_peak_sustained_active"]


def full(path, out, traffic_json=None, klass=None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    lines = [f"# ncu --set full summary ({os.path.basename(path)})", ""]
    traffic = []
    for r in data:
        name = short(r[hdr.index("Kernel Name")])
        lines.append(f"## `{name}`")
        lines.append("")
        lines.append("| metric | value | unit |")
        lines.append("|---|---|---|")
        for w in WANT:
            if w in hdr:
                lines.append(f"| {w} | {r[hdr.index(w)]} | {units[hdr.index(w)]} |")
        st = [(hdr[i].replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""),
               float(r[i])) for i in range(len(hdr))
              if "warps_issue_stalled" in hdr[i] and hdr[i].endswith("_per_issue_active.ratio") and r[i] not in ("", "n/a")]
        st.sort(key=lambda t: -t[1])
        lines.append("")
        lines.append("top stall reasons (per issued instruction): " + ", ".join(f"{a} {b:.2f}" for a, b in st[:5]))
        lines.append("")
        try:
            rd = float(r[hdr.index("dram__bytes_read.sum")])
            wr = float(r[hdr.index("dram__bytes_write.sum")])
            unit = units[hdr.index("dram__bytes_read.sum")]
            scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1.0)
            traffic.append((rd + wr) * scale)
        except (ValueError, IndexError):
            pass
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    if traffic_json and klass and traffic:
        d = json.load(open(traffic_json)) if os.path.exists(traffic_json) else {}
        if "/" in klass:  # config/kernel (what bench.py reads: traffic[config][kernel])
            cfg, kern = klass.split("/", 1)
            d.setdefault(cfg, {})[kern] = sum(traffic) / len(traffic)
        else:
            d[klass] = sum(traffic) / len(traffic)
        json.dump(d, open(traffic_json, "w"), indent=1, sort_keys=True)


def traffic_from_launches(path, traffic_json, klass, pattern):
    """Mean DRAM read+write per launch of the kernels matching `pattern` over a launch list
    (hundreds of launches: every block step of the cycles, unlike the few --set full captures)."""
    op = __import__("gzip").open if path.endswith(".gz") else open
    rows = [l for l in op(path, "rt") if l.startswith('"')]
    per = defaultdict(dict)
    for r in csv.DictReader(io.StringIO("".join(rows))):
        if re.search(pattern, r["Kernel Name"]):
            per[r["ID"]][r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    vals = [m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0) for m in per.values()]
    d = json.load(open(traffic_json)) if os.path.exists(traffic_json) else {}
    cfg, kern = klass.split("/", 1)
    d.setdefault(cfg, {})[kern] = sum(vals) / max(1, len(vals))
    json.dump(d, open(traffic_json, "w"), indent=1, sort_keys=True)
    print(f"{klass}: {len(vals)} launches, mean DRAM traffic {d[cfg][kern] / 1e6:.1f} MB")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    elif sys.argv[1] == "traffic":
        traffic_from_launches(*sys.argv[2:6])
    else:
        full(sys.argv[2], sys.argv[3], *(sys.argv[4:6] if len(sys.argv) > 5 else (None, None)))
