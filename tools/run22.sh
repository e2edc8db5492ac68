timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -2
RNNTG_WS=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
RNNTG_BEAM_IMPL=1 python tools/prof_beam.py 1024 1000 2
RNNTG_BEAM_IMPL=1 RNNTG_WS=1 python tools/prof_beam.py 1024 1000 2
