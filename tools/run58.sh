# ncu of one K1 launch (gemm_exact_kernel<0,0>) on the device-frame path
mkdir -p gpurun_out
ncu --set full --clock-control none --kernel-name-base demangled -k "regex:gemm_exact_kernel<\\(bool\\)0, \\(bool\\)0>" --launch-skip 2 -c 1 -o gpurun_out/prof_k1 -f env RNNTG_SLICED=1 python tools/prof_beam.py 1024 1000 1 > gpurun_out/prof_k1.log 2>&1
ncu -i gpurun_out/prof_k1.ncu-rep --page raw --csv > gpurun_out/prof_k1_raw.csv 2>&1
tail -n 2 gpurun_out/prof_k1.log
