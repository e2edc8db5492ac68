mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 2>&1 | tail -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench13.json 2> gpurun_out/bench13.err
python -c "
import json;d=json.load(open('gpurun_out/bench13.json'));print({k:d.get(k) for k in ['value','decode_kernel_ms','decode_phase_share','e2e','cpu_baseline']}, d['roofline']['frac'], d['bf16_variant'])"
tail -2 gpurun_out/bench13.err
timeout 900 python tools/perf_configs.py > gpurun_out/perf_configs13.log 2>&1; grep -E "config" gpurun_out/perf_configs13.log | cut -c1-400
