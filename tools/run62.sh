for th in 1 2 3 0; do
  RNNTG_SLICE_THROTTLE=$th timeout 300 python tools/prof_e2e.py 1024 1000 4 | python -c "import json,sys;d=json.load(sys.stdin);print('throttle=$th', d['wall_ms'], d['gpu_ms'], round(d['e2e_fps']/1e6,3))"
done
