"""Summarise ncu artefacts for profiles/ (run here, on the CPU box, after a gpurun call).

  python tools/summarize_ncu.py --rep gpurun_out/prof.ncu-rep --launches gpurun_out/launches.csv \
      --out profiles/round1_gemm --flops 68719476736 --bytes 0

Writes <out>.json (key metrics of the captured kernel + per-kernel launch shares) and <out>.md.
"""
import argparse
import csv
import io
import json
import subprocess
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__cluster_size",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg.per_second",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for h, u, v in zip(hdr, units, r):
            if h in KEYS or h in ("Kernel Name",):
                d[h] = (v, u)
        res.append(d)
    return res


def stalls(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return {}
    hdr = rows[1]
    tot = defaultdict(float)
    for r in rows[2:]:
        for h, v in zip(hdr, r):
            if h.startswith("stall_") and "Not Issued" not in h:
                try:
                    tot[h[6:]] += float(v)
                except ValueError:
                    pass
    s = sum(tot.values()) or 1.0
    return {k: round(v / s, 4) for k, v in sorted(tot.items(), key=lambda x: -x[1])[:8]}


def launches(path):
    per = defaultdict(list)
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(io.StringIO("".join(lines))):
        if r.get("Metric Name") == "gpu__time_duration.sum":
            full = r["Kernel Name"].replace("<unnamed>", "").replace("(anonymous namespace)", "")
            head = full.split("(")[0]
            depth, base = 0, ""
            for ch in head:  # drop template arguments, keep the last name component
                if ch == "<":
                    depth += 1
                elif ch == ">":
                    depth -= 1
                elif depth == 0:
                    base += ch
            name = base.replace("void ", "").strip().split("::")[-1]
            per[name].append(float(r["Metric Value"]) * (1e-3 if r["Metric Unit"] == "ns" else 1.0))
    tot = sum(sum(v) for v in per.values()) or 1.0
    return {k: {"launches": len(v), "us_total": round(sum(v), 2), "us_mean": round(sum(v) / len(v), 2),
                "share": round(sum(v) / tot, 4)} for k, v in sorted(per.items(), key=lambda x: -sum(x[1]))}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep")
    ap.add_argument("--launches")
    ap.add_argument("--out", required=True)
    ap.add_argument("--flops", type=float, default=0.0)
    ap.add_argument("--bytes", type=float, default=0.0)
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    res = {"note": a.note}
    if a.rep:
        kern = raw(a.rep)
        res["kernels_captured"] = [{k: v[0] + (" " + v[1] if v[1] else "") for k, v in d.items()} for d in kern]
        res["stall_mix"] = stalls(a.rep)
        if kern:
            d = kern[0]
            t = float(d["gpu__time_duration.sum"][0].replace(",", ""))
            unit = d["gpu__time_duration.sum"][1]
            t_s = t * {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "nsecond": 1e-9, "ms": 1e-3, "msecond": 1e-3}.get(unit, 1e-9)
            rd = float(d.get("dram__bytes_read.sum", ("0", ""))[0].replace(",", ""))
            wr = float(d.get("dram__bytes_write.sum", ("0", ""))[0].replace(",", ""))
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            rd *= scale.get(d.get("dram__bytes_read.sum", ("", "byte"))[1], 1)
            wr *= scale.get(d.get("dram__bytes_write.sum", ("", "byte"))[1], 1)
            res["dram_bytes_per_launch"] = rd + wr
            res["duration_s_under_ncu"] = t_s
            if a.flops:
                res["tflops_under_ncu"] = a.flops / t_s / 1e12
    if a.launches:
        res["launch_shares"] = launches(a.launches)
    with open(a.out + ".json", "w") as f:
        json.dump(res, f, indent=1)
    md = [f"# {a.out.split('/')[-1]}", "", a.note, ""]
    if "launch_shares" in res:
        md += ["| kernel | launches | mean us (ncu, cold, serialised) | share |", "|---|---|---|---|"]
        for k, v in res["launch_shares"].items():
            md.append(f"| {k[:70]} | {v['launches']} | {v['us_mean']} | {v['share']} |")
        md.append("")
    if "kernels_captured" in res:
        md += ["Captured kernel (ncu --set full):", ""]
        for k, v in res["kernels_captured"][0].items():
            md.append(f"- {k}: {v}")
        md += ["", f"stall mix: {res.get('stall_mix')}", f"DRAM bytes/launch: {res.get('dram_bytes_per_launch')}"]
    with open(a.out + ".md", "w") as f:
        f.write("\n".join(md) + "\n")
    print(json.dumps({k: v for k, v in res.items() if k != "kernels_captured"}, indent=1)[:3000])


if __name__ == "__main__":
    main()
