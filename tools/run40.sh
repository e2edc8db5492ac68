# A/B of library builds (paper_2211_00484_b200/variants/*.so) on the bench
# workload's decode kernel (device frames, B=1024 T=1000).
for pass in 1; do
for v in "$@"; do
  RNNTG_LIB=paper_2211_00484_b200/variants/librnntg_$v.so timeout 300 python tools/prof_beam.py 1024 1000 3 > gpurun_out/pb_$v.json 2>gpurun_out/pb_$v.err
  python -c "
import json;d=json.load(open('gpurun_out/pb_$v.json'));print('$v', [round(x,2) for x in d['decode_ms']], d['phase_share'], round(d['gemm_mac_per_s_per_sm']/1e9,1), d['checksum'])"
done
done
