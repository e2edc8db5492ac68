mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:beam_cluster -c 1 -o gpurun_out/ncu_bc -f python tools/prof_beam.py 128 300 1 > gpurun_out/ncu_bc.log 2>&1
tail -3 gpurun_out/ncu_bc.log
python tools/ncu_lines.py gpurun_out/ncu_bc.ncu-rep 45 > gpurun_out/ncu_bc_lines.txt 2>&1
ncu -i gpurun_out/ncu_bc.ncu-rep --page raw --csv > gpurun_out/ncu_bc_raw.csv 2>&1
head -50 gpurun_out/ncu_bc_lines.txt
