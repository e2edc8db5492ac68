"""Schedule quality of the exact-GEMM inner loops in a cubin, without a GPU.

    python tools/fadd_dist.py <cubin> <function-substring> [min_fadd]

For every straight-line SASS run (between branch targets) holding at least
`min_fadd` FADDs, prints the FADD count and how many instructions separate
each FADD from the FMUL producing its operand (mean, and how many are at
distance 1: those stall the warp ~4 cycles on the dependency).  A loop body
whose FADDs sit right behind their FMULs is register-starved: the fused-pe
beam kernel's joiner loop issued ~19% slower than the unfused kernel's for
exactly that reason (same instruction count, ncu "wait" stalls 2.3x)."""
import re
import subprocess
import sys

cubin, fn = sys.argv[1], sys.argv[2]
min_fadd = int(sys.argv[3]) if len(sys.argv) > 3 else 64
sass = subprocess.run(["cuobjdump", "-sass", cubin], capture_output=True, text=True).stdout
funcs, cur = {}, None
for ln in sass.splitlines():
    m = re.match(r"\s*Function : (\S+)", ln)
    if m:
        cur = m.group(1)
        funcs[cur] = []
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4})\*/\s+(.*?);", ln)
    if m and cur:
        funcs[cur].append((int(m.group(1), 16), m.group(2).strip()))

for name, ins in funcs.items():
    if fn not in name:
        continue
    # Split at branches and at branch targets.
    targets = set()
    for _, t in ins:
        m = re.search(r"BRA\S*\s+(?:`\(\.L_x_\d+\)|0x([0-9a-f]+))", t)
        if m and m.group(1):
            targets.add(int(m.group(1), 16))
    labels = {a for a, t in ins if False}
    runs, run = [], []
    for a, t in ins:
        if a in targets and run:
            runs.append(run)
            run = []
        run.append((a, t))
        if re.match(r"(@!?U?P\w+\s+)?(BRA|EXIT|RET|CALL|BAR)", t):
            runs.append(run)
            run = []
    if run:
        runs.append(run)
    print(name[:100])
    for r in runs:
        body = [t for _, t in r]
        nf = sum(1 for t in body if re.match(r"(@\S+\s+)?FADD\b", t))
        if nf < min_fadd:
            continue
        last_w = {}
        dists = []
        for i, t in enumerate(body):
            m = re.match(r"(?:@\S+\s+)?(\w+)(?:\.\S+)?\s+(R\d+),\s*(.*)", t)
            if not m:
                continue
            op, dst, srcs = m.group(1), m.group(2), re.findall(r"R\d+", m.group(3))
            if op == "FADD":
                ds = [i - last_w[s][0] for s in srcs if s in last_w and last_w[s][1] == "FMUL"]
                if ds:
                    dists.append(min(ds))
            last_w[dst] = (i, op)
        if dists:
            print(f"  @{r[0][0]:#07x} len {len(body):4d} FADD {nf:4d}  mean FMUL->FADD distance "
                  f"{sum(dists) / len(dists):5.2f}  at distance 1: {sum(1 for d in dists if d == 1):4d}")
