import sys, os
sys.path.insert(0, os.getcwd())
import os, sys, json, subprocess
os.environ["RNNTG_LIB"] = "paper_2211_00484_b200/variants/librnntg_pclk.so"
sys.argv = ["prof_fsa.py", sys.argv[1], "0", "500", "1"]
exec(open("tools/prof_fsa.py").read())
st = dec.stats()
ncta = {3: 128, 4: 128}[cfg]
tot = sum(st["phase_cycles"][:3])
print(json.dumps({"cfg": cfg, "per_frame_cycles_group0": {"setup+A": st["joiner_rows_computed"]/ncta/500, "B+prune": st["gather_cycles"]/ncta/500, "C+D": st["gemm_wait_cycles"]/ncta/500}, "frame_cycles": tot/ncta/500, "phase": [p/ncta/500 for p in st["phase_cycles"][:3]]}))
