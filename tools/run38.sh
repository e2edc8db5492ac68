RNNTG_FUSED_PE=2 ncu --set full --clock-control none --import-source on -k regex:beam_kernel -c 1 -o gpurun_out/prof_fpe38 -f python tools/prof_beam.py 1024 200 1 > gpurun_out/prof_fpe38.log 2>&1
RNNTG_FUSED_PE=0 ncu --set full --clock-control none --import-source on -k regex:beam_kernel -c 1 -o gpurun_out/prof_nf38 -f python tools/prof_beam.py 1024 200 1 > gpurun_out/prof_nf38.log 2>&1
tail -1 gpurun_out/prof_fpe38.log
