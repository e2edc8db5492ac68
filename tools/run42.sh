# Decode-kernel (device frames) and e2e (pinned host frames) timing per build.
for v in "$@"; do
  L=paper_2211_00484_b200/variants/librnntg_$v.so
  RNNTG_LIB=$L timeout 300 python tools/prof_beam.py 1024 1000 3 > gpurun_out/pb_$v.json 2>gpurun_out/pb_$v.err
  python -c "
import json;d=json.load(open('gpurun_out/pb_$v.json'));print('$v dev', [round(x,2) for x in d['decode_ms']], d['phase_share'], round(d['gemm_mac_per_s_per_sm']/1e9,1))" || tail -3 gpurun_out/pb_$v.err
  RNNTG_LIB=$L timeout 300 python tools/prof_e2e.py 1024 1000 3 > gpurun_out/pe_$v.json 2>gpurun_out/pe_$v.err
  python -c "
import json;d=json.load(open('gpurun_out/pe_$v.json'));print('$v e2e', d['wall_ms'], d['gpu_ms'], round(d['e2e_fps']/1e6,3), d['launches'], d['checksum'])" || tail -3 gpurun_out/pe_$v.err
done
