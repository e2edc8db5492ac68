mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -5
timeout 600 python tools/quick_timing.py 2>&1 | tail -6
