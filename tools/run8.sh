mkdir -p gpurun_out
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench4.json 2> gpurun_out/bench4.err
cat gpurun_out/bench4.json; tail -3 gpurun_out/bench4.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:beam_kernel -s 3 -c 1 -o gpurun_out/prof_beam4 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu4.txt 2>&1
tail -2 gpurun_out/ncu4.txt
