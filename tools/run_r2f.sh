mkdir -p gpurun_out
timeout 2000 python -m pytest tests/test_gpu_sanitize.py tests/test_gpu_sliced.py tests/test_tanhf.py tests/test_shard.py tests/test_synth.py -m gpu -q -p no:cacheprovider --durations=10 > gpurun_out/gputest_f.log 2>&1; echo "pytest rc=$?"
tail -22 gpurun_out/gputest_f.log
nvidia-smi --query-compute-apps=pid,name --format=csv
timeout 600 python bench.py > gpurun_out/bench_f.json 2> gpurun_out/bench_f.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_f.json')); print(d['value'], d['e2e']['value'], d['decode_kernel_ms'], d.get('cxx_dropin'), d['parity_sample']['scores_bit_equal'])"
