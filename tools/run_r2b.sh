# GPU suite, bench, per-config throughput (round 2 evidence run)
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "glibc or lattice or parity or configs" > gpurun_out/gputest_b.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/gputest_b.log
timeout 600 python bench.py > gpurun_out/bench_b.json 2> gpurun_out/bench_b.err; echo "bench rc=$?"
cat gpurun_out/bench_b.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['decode_kernel_ms'], d['decode_phase_share'], d['parity_sample'])"
