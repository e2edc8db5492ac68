timeout 600 python -m pytest tests -m gpu -q -x --timeout 300 2>&1 | tail -2
RNNTG_FUSED_PE=0 timeout 300 python tools/prof_beam.py 1024 1000 2
RNNTG_FUSED_PE=1 timeout 300 python tools/prof_beam.py 1024 1000 2
