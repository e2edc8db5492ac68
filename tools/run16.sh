mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 2>&1 | tail -3
for impl in 0 1; do RNNTG_BEAM_IMPL=$impl timeout 300 python tools/prof_beam.py 1024 1000 3; done
ncu --set full --clock-control none --import-source on -k regex:beam_dual -c 1 -o gpurun_out/prof_dual16 -f python tools/prof_beam.py 1024 200 1 > gpurun_out/prof_dual16.log 2>&1
tail -2 gpurun_out/prof_dual16.log
