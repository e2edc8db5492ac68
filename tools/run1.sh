set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi.txt 2>&1
./tools/fp32_peak > gpurun_out/fp32_peak.json 2>&1
timeout 900 python -m pytest tests -m gpu -q -rf 2>&1 | tail -60 > gpurun_out/pytest1.txt
timeout 600 python tools/quick_timing.py > gpurun_out/timing1.txt 2>&1
cat gpurun_out/fp32_peak.json gpurun_out/pytest1.txt gpurun_out/timing1.txt
