mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:beam_kernel -c 1 -o gpurun_out/prof_beam2 -f python tools/quick_timing.py > gpurun_out/prof_beam2.log 2>&1
timeout 600 python tools/quick_timing.py 2>&1 | tail -2
