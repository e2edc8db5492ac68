# Sliced path: K1 throttle on/off, host frames (e2e) and device frames.
for th in 0 1; do
  RNNTG_SLICE_THROTTLE=$th timeout 300 python tools/prof_e2e.py 1024 1000 3 | python -c "import json,sys;d=json.load(sys.stdin);print('host th=$th', d['wall_ms'], d['gpu_ms'], round(d['e2e_fps']/1e6,3))"
  RNNTG_SLICED=2 RNNTG_SLICE_THROTTLE=$th timeout 300 python tools/prof_beam.py 1024 1000 3 | python -c "import json,sys;d=json.load(sys.stdin);print('dev th=$th', d['decode_ms'], d['gpu_ms'])"
done
for fm in "4 512" "8 512" "8 1024" "16 512"; do set -- $fm
  RNNTG_SLICE_FIRST=$1 RNNTG_SLICE_MAX=$2 timeout 300 python tools/prof_e2e.py 1024 1000 3 | python -c "import json,sys;d=json.load(sys.stdin);print('host $fm', d['wall_ms'], d['gpu_ms'], round(d['e2e_fps']/1e6,3))"
  RNNTG_SLICED=2 RNNTG_SLICE_FIRST=$1 RNNTG_SLICE_MAX=$2 timeout 300 python tools/prof_beam.py 1024 1000 3 | python -c "import json,sys;d=json.load(sys.stdin);print('dev $fm', d['decode_ms'], d['gpu_ms'])"
done
RNNTG_SLICED=1 timeout 300 python tools/prof_beam.py 1024 1000 3 | python -c "import json,sys;d=json.load(sys.stdin);print('dev K1+decode', d['decode_ms'], d['gpu_ms'])"
