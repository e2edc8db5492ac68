# Round evidence: GPU tests, the contract bench (with CPU baseline), the
# reference arm, perf configs, launch list and one full ncu capture.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 2>&1 | tail -2
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench65.json 2> gpurun_out/bench65.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench65_ref.json 2> gpurun_out/bench65_ref.err
timeout 900 python tools/perf_configs.py > gpurun_out/perf_configs65.log 2>&1
bash tools/run_evidence.sh
python -c "
import json;d=json.load(open('gpurun_out/bench65.json'));print({k:d.get(k) for k in ['value','ms_per_step','decode_kernel_ms','e2e','cpu_baseline','clocks']}, d['roofline'])"
cat gpurun_out/bench65_ref.json
