RNNTG_WS=1 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x --timeout 120 2>&1 | tail -2
RNNTG_WS=1 RNNTG_FUSED_PE=0 timeout 300 python tools/prof_beam.py 1024 1000 2 | cut -c1-200
RNNTG_FUSED_PE=0 timeout 300 python tools/prof_beam.py 1024 1000 2 | cut -c1-200
