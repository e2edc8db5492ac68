for v in "$@"; do
  L=paper_2211_00484_b200/variants/librnntg_$v.so
  RNNTG_LIB=$L timeout 300 python tools/prof_beam.py 1024 1000 3 | python -c "import json,sys;d=json.load(sys.stdin);print('$v dev', [round(x,2) for x in d['decode_ms']], d['phase_share'], d['checksum'])"
  RNNTG_LIB=$L timeout 300 python tools/prof_e2e.py 1024 1000 4 | python -c "import json,sys;d=json.load(sys.stdin);print('$v e2e', d['wall_ms'], d['gpu_ms'], round(d['e2e_fps']/1e6,3), d['checksum'])"
done
