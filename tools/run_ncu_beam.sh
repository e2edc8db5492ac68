# ncu evidence for the bench workload (B=1024, T=1000): the beam kernel and
# K1 (the encoder-side projection GEMM: gemm_exact_kernel launched inside
# rnntg_beam_search_batch, selected by its NVTX range), each --set full with
# source correlation.  Outputs gpurun_out/.
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:beam_kernel -c 1 -o gpurun_out/ncu_beam -f python tools/prof_beam.py 1024 1000 1 > gpurun_out/ncu_beam.log 2>&1
tail -2 gpurun_out/ncu_beam.log
ncu -i gpurun_out/ncu_beam.ncu-rep --page raw --csv > gpurun_out/ncu_beam_raw.csv 2>&1
python tools/ncu_lines.py gpurun_out/ncu_beam.ncu-rep 40 > gpurun_out/ncu_beam_lines.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "rnntg_beam_search_batch/" -k regex:gemm_exact -c 1 -o gpurun_out/ncu_k1 -f python tools/prof_beam.py 1024 1000 1 > gpurun_out/ncu_k1.log 2>&1
tail -2 gpurun_out/ncu_k1.log
ncu -i gpurun_out/ncu_k1.ncu-rep --page raw --csv > gpurun_out/ncu_k1_raw.csv 2>&1
./tools/fp32_peak > gpurun_out/fp32_peak.json; cat gpurun_out/fp32_peak.json
