mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "glibc or lattice or test_gpu_parity" > gpurun_out/gputest_c.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/gputest_c.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_c.json 2> gpurun_out/bench_c.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_c.json')); print(d['value'], d['e2e']['value'], d['decode_kernel_ms'], d['decode_phase_share'])"
