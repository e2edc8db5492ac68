mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "fsa or lattice or config3 or config4 or sanitize" > gpurun_out/gputest_h.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/gputest_h.log
for c in 3 4; do timeout 600 python tools/prof_fsa.py $c > gpurun_out/prof_fsa$c.json 2>&1; tail -1 gpurun_out/prof_fsa$c.json; done
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_h.json 2> gpurun_out/bench_h.err
python -c "import json; d=json.load(open('gpurun_out/bench_h.json')); print(d['value'], d['e2e']['value'], d['decode_kernel_ms'], d['decode_phase_share'])"
