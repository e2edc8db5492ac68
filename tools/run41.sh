# A/B of library builds incl. the out-of-line GEMM (-rdc) variant; fused-pe
# kernel timing under each.
for v in "$@"; do
  RNNTG_LIB=paper_2211_00484_b200/variants/librnntg_$v.so timeout 300 python tools/prof_beam.py 1024 1000 3 > gpurun_out/pb_$v.json 2>gpurun_out/pb_$v.err
  python -c "
import json;d=json.load(open('gpurun_out/pb_$v.json'));print('$v', [round(x,2) for x in d['decode_ms']], d['phase_share'], round(d['gemm_mac_per_s_per_sm']/1e9,1), d['checksum'])" || tail -3 gpurun_out/pb_$v.err
  RNNTG_FUSED_PE=2 RNNTG_LIB=paper_2211_00484_b200/variants/librnntg_$v.so timeout 300 python tools/prof_beam.py 1024 1000 2 > gpurun_out/pbf_$v.json 2>gpurun_out/pbf_$v.err
  python -c "
import json;d=json.load(open('gpurun_out/pbf_$v.json'));print('$v fused', [round(x,2) for x in d['decode_ms']], d['phase_share'], d['fused_pe_share'], round(d['gemm_mac_per_s_per_sm']/1e9,1), d['checksum'])" || tail -3 gpurun_out/pbf_$v.err
done
