mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=12 > gpurun_out/gputest_k.log 2>&1; echo "pytest rc=$?"
tail -22 gpurun_out/gputest_k.log
timeout 600 python bench.py > gpurun_out/bench_k.json 2> gpurun_out/bench_k.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_k.json')); print(d['value'], d['e2e']['value'], d['decode_kernel_ms'], d.get('cxx_dropin',{}).get('frames_per_s'), d['parity_sample']['scores_bit_equal'], d['cpu_baseline']['value'])"
timeout 900 python tools/perf_configs.py > gpurun_out/perf_configs_k.jsonl 2> gpurun_out/perf_configs_k.err
python - <<'PY'
import json
for l in open('gpurun_out/perf_configs_k.jsonl'):
    d=json.loads(l); print(d['name'], round(d['frames_per_s']/1e6,3), 'M', round(d['decode_ms'],2), 'ms')
PY
