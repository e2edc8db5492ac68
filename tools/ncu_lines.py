"""Top CUDA source lines of an ncu report by warp-stall samples and by
executed instructions (ncu -i <rep> --page source --csv --print-source
cuda,sass, which aggregates the SASS rows per CUDA line, file by file).

    python tools/ncu_lines.py <report.ncu-rep> [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows, fname, hdr = [], None, None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].isdigit():
        continue
    d = dict(zip(hdr[2:], r[2:]))
    try:
        s = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        ni = int(d.get("Warp Stall Sampling (Not-issued Samples)", "0") or 0)
        ie = int(d.get("Instructions Executed", "0") or 0)
    except ValueError:
        continue
    rows.append((s, ni, ie, f"{fname}:{r[0]}", r[1].strip()[:70]))
ts = sum(x[0] for x in rows) or 1
ti = sum(x[2] for x in rows) or 1
print(f"total samples {ts}, warp-instructions {ti}")
print("-- by stall samples: share samples | share instr | line")
for s, ni, ie, loc, src in sorted(rows, reverse=True)[:top]:
    print(f"{s / ts:6.3f} {ie / ti:6.3f}  {loc:24s} {src}")
print("-- by instructions")
for s, ni, ie, loc, src in sorted(rows, key=lambda x: -x[2])[:top]:
    print(f"{s / ts:6.3f} {ie / ti:6.3f}  {loc:24s} {src}")
