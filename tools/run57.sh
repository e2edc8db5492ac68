# ncu evidence for the host-frame (sliced) path: the largest decode slice
# (beam_kernel<4,0,0,1>, frames 504..999) and one K1 launch (gemm_exact) of
# the device-frame path.
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:beam_kernel --launch-skip 6 -c 1 -o gpurun_out/prof_slice -f python tools/prof_e2e.py 1024 1000 1 > gpurun_out/prof_slice.log 2>&1
ncu -i gpurun_out/prof_slice.ncu-rep --page raw --csv > gpurun_out/prof_slice_raw.csv 2>&1
ncu --set full --clock-control none -k regex:gemm_exact_kernel --launch-skip 8 -c 1 -o gpurun_out/prof_k1 -f env RNNTG_SLICED=1 python tools/prof_beam.py 1024 1000 1 > gpurun_out/prof_k1.log 2>&1
ncu -i gpurun_out/prof_k1.ncu-rep --page raw --csv > gpurun_out/prof_k1_raw.csv 2>&1
tail -2 gpurun_out/prof_slice.log gpurun_out/prof_k1.log
