# Slice schedule with/without the K1 side stream.
for ov in 0 1; do
for v in "8 512" "4 512" "8 256"; do
  set -- $v
  RNNTG_SLICE_OVERLAP=$ov RNNTG_SLICE_FIRST=$1 RNNTG_SLICE_MAX=$2 timeout 300 python tools/prof_e2e.py 1024 1000 3 > gpurun_out/pe.json 2>gpurun_out/pe.err
  python -c "
import json;d=json.load(open('gpurun_out/pe.json'));print('ov=$ov $v', d['wall_ms'], d['gpu_ms'], round(d['e2e_fps']/1e6,3), d['launches'], d['checksum'])" || tail -3 gpurun_out/pe.err
done; done
