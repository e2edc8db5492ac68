mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 2>&1 | tail -3
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench8.json 2> gpurun_out/bench8.err
python -c "
import json;d=json.load(open('gpurun_out/bench8.json'));print({k:d.get(k) for k in ['value','decode_kernel_ms','decode_phase_share','e2e']}, d['roofline']['frac'], d['bf16_variant'])"
tail -2 gpurun_out/bench8.err
timeout 900 python tools/perf_configs.py > gpurun_out/perf_configs3.log 2>&1; grep -E "config3|config4" gpurun_out/perf_configs3.log | cut -c1-600
