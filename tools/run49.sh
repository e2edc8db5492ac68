timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 2>&1 | tail -2
RNNTG_SLICED=1 timeout 300 python tools/prof_beam.py 1024 1000 3 | python -c "import json,sys;d=json.load(sys.stdin);print('dev', d['decode_ms'], d['gpu_ms'])"
timeout 300 python tools/prof_e2e.py 1024 1000 3
