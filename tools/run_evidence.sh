# Evidence capture: launch list of the bench command + one full ncu capture
# of the beam kernel at the bench size (B=1024, T=1000).  Outputs gpurun_out/.
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/launches_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:beam_kernel -c 1 -o gpurun_out/prof_beam_full -f python tools/prof_beam.py 1024 1000 1 > gpurun_out/prof_beam_full.log 2>&1
ncu -i gpurun_out/prof_beam_full.ncu-rep --page raw --csv > gpurun_out/prof_beam_full_raw.csv 2>&1
tail -2 gpurun_out/prof_beam_full.log
