mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_beam_cluster.py tests/test_gpu_parity.py tests/test_gpu_sliced.py tests/test_gpu_beam_multi.py -x -q -p no:cacheprovider > gpurun_out/gputest_j.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/gputest_j.log
timeout 900 python tools/perf_configs.py > gpurun_out/perf_configs_j.jsonl 2> gpurun_out/perf_configs_j.err
python - <<'PY'
import json
for l in open('gpurun_out/perf_configs_j.jsonl'):
    d=json.loads(l); print(d['name'], round(d['frames_per_s']/1e6,3), 'M', round(d['decode_ms'],2), 'ms')
PY
