# FSA evidence: timing/occupancy of configs 3 and 4 with device frames, and
# one ncu --set full capture of fsa_kernel per config (raw metrics + source
# page).  Outputs gpurun_out/.
mkdir -p gpurun_out
for c in 3 4; do
  timeout 600 python tools/prof_fsa.py $c > gpurun_out/prof_fsa$c.json 2> gpurun_out/prof_fsa$c.err; tail -1 gpurun_out/prof_fsa$c.json
done
for c in 3 4; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:fsa_kernel -c 1 -o gpurun_out/ncu_fsa$c -f python tools/prof_fsa.py $c 0 500 1 > gpurun_out/ncu_fsa$c.log 2>&1
  ncu -i gpurun_out/ncu_fsa$c.ncu-rep --page raw --csv > gpurun_out/ncu_fsa${c}_raw.csv 2>&1
  python tools/ncu_lines.py gpurun_out/ncu_fsa$c.ncu-rep 40 > gpurun_out/ncu_fsa${c}_lines.txt 2>&1
  tail -2 gpurun_out/ncu_fsa$c.log
done
ls -la gpurun_out/ncu_fsa*
