mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "glibc or lattice or test_gpu_parity or sliced" > gpurun_out/gputest_d.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/gputest_d.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_d.json 2> gpurun_out/bench_d.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_d.json')); print(d['value'], d['e2e']['value'], d['decode_kernel_ms'], d['decode_phase_share'], d['parity_sample']['tokens_identical'])"
