"""Summarise ncu CSV outputs into profiles/ JSON (run here, after gpurun).

    python tools/ncu_summary.py launches <launches.csv> <out.json> <note>
    python tools/ncu_summary.py dram <dram.csv> <out.json> <note>
    python tools/ncu_summary.py capture <rep.ncu-rep> <out.json> <note> <key>   (adds/replaces entry <key>)
"""
import collections
import csv
import json
import sys


def rows(path):
    hdr, out = None, []
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            out.append(dict(zip(hdr, r)))
    return out


def val(d):
    v = float(d["Metric Value"].replace(",", ""))
    u = d["Metric Unit"]
    scale = {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6,
             "Gbyte": 1e9}
    return v * scale.get(u, 1.0)


def launches(path):
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in rows(path):
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        k = d["Kernel Name"].split("(")[0]
        agg[k][0] += 1
        agg[k][1] += val(d)
    tot = sum(x[1] for x in agg.values())
    return {k: {"launches": n, "total_us": round(t / 1e3, 1), "avg_us": round(t / n / 1e3, 2),
                "share": round(t / tot, 3)} for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])}


def dram(path):
    per = collections.defaultdict(lambda: collections.defaultdict(float))
    for d in rows(path):
        k = d["Kernel Name"].split("(")[0]
        per[(k, d["ID"])][d["Metric Name"]] += val(d)
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for (k, _), m in per.items():
        agg[k][0] += 1
        agg[k][1] += m.get("dram__bytes_read.sum", 0.0)
        agg[k][2] += m.get("dram__bytes_write.sum", 0.0)
    return {k: {"launches": n, "dram_read_bytes": r, "dram_write_bytes": w, "bytes_per_launch": (r + w) / n}
            for k, (n, r, w) in agg.items()}


def _page(rep, page):
    """One page of a capture: from the .ncu-rep, or from the <rep>.<page>.csv[.gz] exported on the GPU box
    (tools/ncu_export.sh; the reports themselves are too large to bring back)."""
    import gzip
    import os
    import subprocess

    base = rep[:-len(".ncu-rep")] if rep.endswith(".ncu-rep") else rep
    for ext, op in ((".csv", open), (".csv.gz", gzip.open)):
        if os.path.exists(f"{base}.{page}{ext}"):
            with op(f"{base}.{page}{ext}", "rt") as f:
                return f.read()
    args = ["--page", "details", "--csv"] if page == "details" else ["--page", "source", "--csv",
                                                                        "--print-source=cuda,sass"]
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def details(rep):
    """Key metrics of one `ncu --set full` capture (ncu -i <rep> --page details)."""
    out = _page(rep, "details")
    r = list(csv.reader(out.splitlines()))
    hdr = r[0]
    keep = {"Duration", "Elapsed Cycles", "SM Frequency", "DRAM Throughput", "Memory Throughput",
            "L1/TEX Hit Rate", "L2 Hit Rate", "Compute (SM) Throughput", "Executed Ipc Active",
            "Issue Slots Busy", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy",
            "Block Size", "Grid Size", "Dynamic Shared Memory Per Block", "Warp Cycles Per Issued Instruction",
            "No Eligible", "Executed Instructions"}
    res = {}
    for row in r[1:]:
        d = dict(zip(hdr, row))
        if d.get("Metric Name") in keep:
            res[d["Metric Name"]] = f'{d["Metric Value"]} {d["Metric Unit"]}'.strip()
    return res


def stalls(rep):
    """Warp-stall reasons summed over the source page of one capture."""
    out = _page(rep, "source")
    agg = collections.Counter()
    hdr = None
    for r in csv.reader(out.splitlines()):
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr and len(r) == len(hdr) and r[2] == "-":
            for i, h in enumerate(hdr):
                if h.startswith("stall_") and "Not Issued" not in h and r[i]:
                    try:
                        agg[h] += int(r[i])
                    except ValueError:
                        pass
    tot = sum(agg.values()) or 1
    return {k: round(v / tot, 3) for k, v in agg.most_common(8)}


if __name__ == "__main__":
    mode, src, dst, note = sys.argv[1:5]
    if mode == "capture":
        import os

        key = sys.argv[5]
        out = json.load(open(dst)) if os.path.exists(dst) else {}
        out[key] = {"note": note, "metrics": details(src), "stall_share": stalls(src)}
    else:
        out = {"note": note, "kernels": launches(src) if mode == "launches" else dram(src)}
    json.dump(out, open(dst, "w"), indent=1)
    print(json.dumps(out if mode != "capture" else out[key], indent=1)[:1500])
