timeout 900 python tools/perf_configs.py > gpurun_out/perf_configs32.log 2>&1; grep -E "config" gpurun_out/perf_configs32.log | cut -c1-330
bash tools/run_evidence.sh
