mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bf16.py -q -x --timeout 300 2>&1 | tail -4
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench5.json 2> gpurun_out/bench5.err
python -c "
import json;d=json.load(open('gpurun_out/bench5.json'));print({k:d.get(k) for k in ['value','decode_kernel_ms','joiner_rows_per_stream_frame','e2e','roofline']})"
tail -3 gpurun_out/bench5.err
