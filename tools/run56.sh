# K1 occupancy A/B (launch-bounds min blocks): K1 time = gpu_ms - decode_ms on device frames; e2e
for v in "$@"; do
  L=paper_2211_00484_b200/variants/librnntg_$v.so
  RNNTG_LIB=$L RNNTG_SLICED=1 timeout 300 python tools/prof_beam.py 1024 1000 3 | python -c "import json,sys;d=json.load(sys.stdin);print('$v dev decode', round(min(d['decode_ms']),2), 'K1', round(d['gpu_ms']-d['decode_ms'][-1],2), d['checksum'])"
  RNNTG_LIB=$L timeout 300 python tools/prof_e2e.py 1024 1000 3 | python -c "import json,sys;d=json.load(sys.stdin);print('$v e2e', d['wall_ms'], d['gpu_ms'], round(d['e2e_fps']/1e6,3))"
done
