mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 --deselect tests/test_gpu_bf16.py::test_bf16_beam_runs_and_agrees 2>&1 | tail -5
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench3.json 2> gpurun_out/bench3.err
cat gpurun_out/bench3.json; tail -3 gpurun_out/bench3.err
timeout 180 python -m pytest tests/test_gpu_bf16.py -q -x -s 2>&1 | tail -15
