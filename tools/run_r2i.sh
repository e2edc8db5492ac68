mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_logadd.py tests/test_gpu_fsa.py tests/test_gpu_lattice.py -x -q -p no:cacheprovider > gpurun_out/gputest_i.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/gputest_i.log
timeout 1500 python -m pytest tests/test_gpu_configs.py -x -q -p no:cacheprovider -k logadd --durations=5 > gpurun_out/gputest_i2.log 2>&1; echo "pytest2 rc=$?"
tail -12 gpurun_out/gputest_i2.log
