# Round evidence on one B200 (run under gpurun): the full GPU suite, the
# default bench line, per-config throughput, the greedy config-1 probe and an
# ncu capture of the greedy cluster kernel.  Outputs gpurun_out/.
#   gpurun --timeout 3000 -- bash tools/run_gpu_round.sh [suite|bench|configs|greedy|all]
what=${1:-all}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
if [ "$what" = suite ] || [ "$what" = all ]; then
  timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=12 > gpurun_out/gputest.log 2>&1
  echo "pytest rc=$?"; tail -16 gpurun_out/gputest.log
fi
if [ "$what" = bench ] || [ "$what" = all ]; then
  timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
  timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "bench ref rc=$?"
fi
if [ "$what" = configs ] || [ "$what" = all ]; then
  timeout 900 python tools/perf_configs.py > gpurun_out/perf_configs.jsonl 2> gpurun_out/perf_configs.err; echo "configs rc=$?"
fi
if [ "$what" = greedy ] || [ "$what" = all ]; then
  timeout 300 python tools/probes/greedy_cfg1.py > gpurun_out/greedy_cfg1.json 2>&1
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:greedy_cluster -c 1 \
    -o gpurun_out/ncu_greedy_cluster -f python tools/probes/greedy_cfg1.py > gpurun_out/ncu_greedy.log 2>&1
  echo "greedy rc=$?"
fi
