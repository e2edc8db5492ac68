# single-launch kernel code-generation variants: device-frame decode time
for pass in 1 2; do for v in "$@"; do
  RNNTG_LIB=paper_2211_00484_b200/variants/librnntg_$v.so timeout 300 python tools/prof_beam.py 1024 1000 3 | python -c "import json,sys;d=json.load(sys.stdin);print('$v dev', [round(x,2) for x in d['decode_ms']], d['phase_share'], d['checksum'])"
done; done
