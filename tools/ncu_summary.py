"""Summarise ncu artefacts (launch-list CSV and --set full reports) into
profiles/: per-kernel device-time shares and the key counters of the top kernel."""
import csv
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__cycles_elapsed.avg.per_second", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__m_xbar2l1tex_read_bytes.sum", "lts__t_sectors_srcunit_tex_lookup_hit.sum",
        "lts__t_sectors_srcunit_tex_lookup_miss.sum", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active"]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    per = {}
    for r in rows[hi + 1:]:
        name = r[ki].split("(")[0].replace("void ", "")
        per.setdefault(name, []).append(float(r[vi]))
    tot = sum(sum(v) for v in per.values())
    out = []
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        out.append({"kernel": k, "launches": len(v), "ns_total": sum(v),
                    "ns_per_launch": sum(v) / len(v), "share": sum(v) / tot})
    return out


def _report_row(h, units, vals):
    res = {}
    for k in KEYS:
        if k in h:
            i = h.index(k)
            res[k] = {"value": vals[i], "unit": units[i]}
    stalls = {}
    for i, k in enumerate(h):
        if "average_warps_issue_stalled" in k and k.endswith("per_issue_active.ratio"):
            try:
                if float(vals[i]) >= 0.2:
                    stalls[k.split("stalled_")[1].split("_per")[0]] = float(vals[i])
            except ValueError:
                pass
    res["stalls_per_issue_active"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1]))
    return res


def report(path):
    """Key counters of the first captured kernel; with several kernels in the
    report, a dict {kernel name: counters}."""
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, units = rows[0], rows[1]
    if len(rows) == 3:
        return _report_row(h, units, rows[2])
    ki = h.index("Kernel Name")
    return {f"{r[ki].split('(')[0]} #{n}": _report_row(h, units, r)
            for n, r in enumerate(rows[2:])}


def to_bytes(entry):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}[entry["unit"]]
    return float(entry["value"]) * scale


def traffic(summary_path, dst, label):
    d = json.load(open(summary_path))
    rd, wr = to_bytes(d["dram__bytes_read.sum"]), to_bytes(d["dram__bytes_write.sum"])
    json.dump({"kernel": label, "dram_bytes_per_launch": rd + wr, "dram_read_bytes": rd,
               "dram_write_bytes": wr, "source": summary_path}, open(dst, "w"), indent=1)


if __name__ == "__main__":
    # launches <csv> <out.json> | report <ncu-rep> <out.json> | traffic <summary.json> <out.json> <label>
    kind, src, dst = sys.argv[1], sys.argv[2], sys.argv[3]
    if kind == "traffic":
        traffic(src, dst, sys.argv[4])
        print(open(dst).read())
    else:
        data = launches(src) if kind == "launches" else report(src)
        with open(dst, "w") as fh:
            json.dump(data, fh, indent=1)
        print(json.dumps(data, indent=1)[:3000])
