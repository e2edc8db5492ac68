"""Attribute an ncu SASS source page (CSV) to CUDA source lines.

    python tools/sass_lines.py <sass.csv> <cubin> <function-substring> [top]

The ncu CSV (ncu -i rep --page source --csv --print-source sass) lists one row
per SASS instruction with stall samples and executed-instruction counts; the
line table comes from `nvdisasm -g` of the same cubin (built -lineinfo)."""
import collections
import csv
import re
import subprocess
import sys

csv_path, cubin, fn = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
cur_fn, cur_line, lines, in_fn = None, None, {}, False
for ln in dis.splitlines():
    m = re.match(r"\s*\.text\.(\S+):", ln)
    if m:
        in_fn = fn in m.group(1)
        continue
    if not in_fn:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur_line = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
    if m and cur_line:
        lines[int(m.group(1), 16)] = cur_line
rows = list(csv.reader(open(csv_path)))
hdr, data = rows[1], rows[2:]
iS, iE = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
stall = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
base = int(data[0][0], 16)
agg = collections.defaultdict(lambda: [0, 0, collections.Counter()])
for r in data:
    key = lines.get(int(r[0], 16) - base, "?")
    a = agg[key]
    a[0] += int(r[iS] or 0)
    a[1] += int(r[iE] or 0)
    for i in stall:
        a[2][hdr[i][6:]] += int(r[i] or 0)
ts = sum(a[0] for a in agg.values()) or 1
te = sum(a[1] for a in agg.values()) or 1
print(f"samples {ts} instructions {te}  mapped lines {len(lines)}")
for k, a in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{k:28s} samp {100*a[0]/ts:5.1f}%  inst {100*a[1]/te:5.1f}%  {a[2].most_common(3)}")
