# ncu of the tcgen05 bf16 joiner variant of the beam kernel (bench workload),
# for the tensor-pipe evidence.  Outputs gpurun_out/.
mkdir -p gpurun_out
RNNTG_PROF_BF16=1 python tools/prof_beam.py 1024 1000 2 > gpurun_out/bf16_timing.json 2>&1; tail -1 gpurun_out/bf16_timing.json
RNNTG_PROF_BF16=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:beam_kernel -c 1 -o gpurun_out/ncu_bf16 -f python tools/prof_beam.py 1024 1000 1 > gpurun_out/ncu_bf16.log 2>&1
tail -2 gpurun_out/ncu_bf16.log
ncu -i gpurun_out/ncu_bf16.ncu-rep --page raw --csv > gpurun_out/ncu_bf16_raw.csv 2>&1
python tools/ncu_lines.py gpurun_out/ncu_bf16.ncu-rep 30 > gpurun_out/ncu_bf16_lines.txt 2>&1
