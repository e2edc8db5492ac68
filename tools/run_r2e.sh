mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -x --durations=15 > gpurun_out/gputest_e.log 2>&1; echo "pytest rc=$?"
tail -25 gpurun_out/gputest_e.log
timeout 600 python bench.py > gpurun_out/bench_e.json 2> gpurun_out/bench_e.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_e.json')); print(d['value'], d['e2e']['value'], d['decode_kernel_ms'], d.get('cxx_dropin'), d.get('parity_sample'))"
