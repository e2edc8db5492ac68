RNNTG_BEAM_IMPL=1 ncu --set full --clock-control none --import-source on -k regex:beam_kernel -c 1 -o gpurun_out/prof_single21 -f python tools/prof_beam.py 1024 200 1 > gpurun_out/prof_single21.log 2>&1
tail -1 gpurun_out/prof_single21.log
