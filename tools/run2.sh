mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -rf -x --timeout 600 2>&1 | tail -40 > gpurun_out/pytest2.txt
cat gpurun_out/pytest2.txt
