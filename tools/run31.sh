timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 2>&1 | tail -2
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench31.json 2> gpurun_out/bench31.err; python -c "
import json;d=json.load(open('gpurun_out/bench31.json'));print({k:d.get(k) for k in ['value','ms_per_step','decode_kernel_ms','e2e','cpu_baseline']}, d['roofline']['frac'])"
