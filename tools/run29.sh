for i in 1 2; do RNNTG_FUSED_PE=2 timeout 300 python tools/prof_beam.py 1024 1000 3; done
RNNTG_FUSED_PE=0 timeout 300 python tools/prof_beam.py 1024 1000 3
