timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 2>&1 | tail -2
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b45.json 2> gpurun_out/b45.err
python -c "
import json;d=json.load(open('gpurun_out/b45.json'));print(round(d['value']/1e6,3), d['e2e'], d['decode_kernel_ms'], d['ms_per_step'], d['gpu_launches'])"
