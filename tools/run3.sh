mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt; lscpu | head -20 >> gpurun_out/nproc.txt
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_run.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:beam_kernel -s 3 -c 1 -o gpurun_out/prof_beam_bench -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_run.txt 2>&1
cat gpurun_out/bench.json gpurun_out/bench_ref.json; tail -3 gpurun_out/bench.err gpurun_out/bench_ref.err
