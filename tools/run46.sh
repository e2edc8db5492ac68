# Device-frame decode through the sliced path (RNNTG_SLICED=2) vs K1 + decode.
for v in 1 2; do
  RNNTG_SLICED=$v timeout 300 python tools/prof_beam.py 1024 1000 3 > gpurun_out/pb.json 2>gpurun_out/pb.err
  python -c "
import json;d=json.load(open('gpurun_out/pb.json'));print('sliced=$v', [round(x,2) for x in d['decode_ms']], d['gpu_ms'], d['checksum'])" || tail -3 gpurun_out/pb.err
done
timeout 300 python tools/prof_e2e.py 1024 1000 3
