# GPU suite on the current build, then the host-frame path's slice schedule sweep.
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 2>&1 | tail -2
for v in "4 256" "8 256" "16 256" "8 512" "8 1024" "16 128" "32 512" "4 64"; do
  set -- $v
  RNNTG_SLICE_FIRST=$1 RNNTG_SLICE_MAX=$2 timeout 300 python tools/prof_e2e.py 1024 1000 3 > gpurun_out/pe.json 2>gpurun_out/pe.err
  python -c "
import json;d=json.load(open('gpurun_out/pe.json'));print('$v', d['wall_ms'], d['gpu_ms'], round(d['e2e_fps']/1e6,3), d['launches'])" || tail -3 gpurun_out/pe.err
done
