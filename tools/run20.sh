timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fsa.py -q -x --timeout 600 2>&1 | tail -3
for impl in 1; do RNNTG_BEAM_IMPL=$impl timeout 300 python tools/prof_beam.py 1024 1000 3; done
