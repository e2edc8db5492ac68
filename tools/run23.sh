timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -2
for i in 1 2; do RNNTG_BEAM_IMPL=1 python tools/prof_beam.py 1024 1000 2; done
