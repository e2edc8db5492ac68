mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:beam_kernel -c 1 -o gpurun_out/prof_beam15 -f python tools/quick_timing.py > gpurun_out/prof_beam15.log 2>&1
tail -3 gpurun_out/prof_beam15.log
