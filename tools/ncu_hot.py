"""Print the hottest SASS lines (warp-stall samples) of an ncu report: python tools/ncu_hot.py rep [kernel-regex] [thresh]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
if len(sys.argv) > 2 and sys.argv[2]:
    cmd += ["-k", "regex:" + sys.argv[2]]
th = float(sys.argv[3]) if len(sys.argv) > 3 else 0.01
rows = list(csv.reader(io.StringIO(subprocess.run(cmd, capture_output=True, text=True).stdout)))
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}; blocks.append(cur)
    elif r and r[0] == "Address":
        if cur is None:
            cur = {"name": "?", "rows": []}; blocks.append(cur)
        cur["hdr"] = r
    elif cur is not None and "hdr" in cur:
        cur["rows"].append(r)
for b in blocks:
    h = b["hdr"]; i = h.index("Warp Stall Sampling (All Samples)")
    tot = sum(float(r[i] or 0) for r in b["rows"] if len(r) > i) or 1
    print("==", b["name"][:100], "samples", tot)
    for j, r in enumerate(b["rows"]):
        v = float(r[i] or 0) / tot
        if v > th:
            print(f"{j:5d} {v:6.3f} {r[1][:110]}")
