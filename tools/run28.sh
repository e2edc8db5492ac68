timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_parity.py -q -x --timeout 300 2>&1 | tail -2
RNNTG_FUSED_PE=2 timeout 300 python tools/prof_beam.py 1024 1000 2
RNNTG_FUSED_PE=1 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench28.json 2> gpurun_out/bench28.err; python -c "
import json;d=json.load(open('gpurun_out/bench28.json'));print({k:d.get(k) for k in ['value','ms_per_step','decode_kernel_ms','e2e']})"
