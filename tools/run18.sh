tools/probes/gemm_tiling
RNNTG_BEAM_IMPL=0 timeout 300 python tools/prof_beam.py 1024 1000 3
