mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bf16.py tests/test_gpu_fsa.py -q -x --timeout 300 2>&1 | tail -3
for ws in 1 0; do
RNNTG_WS=$ws timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench6_ws$ws.json 2> gpurun_out/bench6_ws$ws.err
python -c "
import json;d=json.load(open('gpurun_out/bench6_ws$ws.json'));print('ws=$ws', {k:d.get(k) for k in ['value','decode_kernel_ms','decode_phase_share','e2e']}, d['roofline']['frac'], d['bf16_variant']['value'])"
done
